// d = 3 vMF mixtures on device, fp64 (proj/src/sphdist.cpp; its d = 3
// branches are pinned against the reference by tests/test_oracle.py through
// the oracle restatement): normalisation (Table 1, :287-310), mixture pdf
// (:176-185), inverse-CDF vMF sampling with the Duff et al. basis (:132-158),
// reflection at Neumann boundaries (:204-218), uniform sphere / hemisphere
// (:220-243), one-sample MIS (:245-270), and the raw-parameter gradient
// (mixture_grad, :315-381) with kl_grad / selection_grad
// (proj/src/guide_train.cpp:25-56). Operation order follows the oracle
// (oracle/wost_oracle.cpp) so the exact-MLP walk path matches it per walk.
#pragma once

#include "wg3_geom.cuh"
#include "wg_device.cuh"

namespace wg3 {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;
constexpr double kFourPi = 4.0 * kPi;
constexpr double kKappaMin = 1e-6, kKappaMax = 1e4;
constexpr int kMaxProposals = 4096;  // rejection-loop cap (NaN safety, as in 2D)

template <int K>
struct Mix3 {
  double mu[K][3];
  double kappa[K], lambda[K], log_a[K];
  double c;
};

__device__ __forceinline__ double sigmoid(double x) {
  return x >= 0.0 ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x));
}

__device__ __forceinline__ double comp_log_norm3(double kappa) {  // sphdist.cpp:162-167
  if (kappa == 0.0) return -log(kFourPi);
  return log(kappa) - kappa - log(kTwoPi * (1.0 - exp(-2.0 * kappa)));
}

// raw row [mu (3K) | kappa' (K) | lambda' (K) | c'] -> mixture
template <int K, class T>
__device__ __forceinline__ void normalize3(const T* raw, Mix3<K>& o) {
  o.c = sigmoid(static_cast<double>(raw[5 * K]));
  double mx = -dinf();
#pragma unroll
  for (int i = 0; i < K; ++i) mx = fmax(mx, static_cast<double>(raw[4 * K + i]));
  double z = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i) z += exp(static_cast<double>(raw[4 * K + i]) - mx);
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double mx0 = raw[3 * i], my0 = raw[3 * i + 1], mz0 = raw[3 * i + 2];
    double mn = sqrt(mx0 * mx0 + my0 * my0 + mz0 * mz0);
    if (mn < 1e-12) {
      double a = kTwoPi * i / WG_MAX_MIXTURE;
      o.mu[i][0] = cos(a);
      o.mu[i][1] = sin(a);
      o.mu[i][2] = 0.0;
    } else {
      o.mu[i][0] = mx0 / mn;
      o.mu[i][1] = my0 / mn;
      o.mu[i][2] = mz0 / mn;
    }
    o.kappa[i] = wg::sclamp(exp(static_cast<double>(raw[3 * K + i])), kKappaMin, kKappaMax);
    o.lambda[i] = exp(static_cast<double>(raw[4 * K + i]) - mx) / z;
  }
#pragma unroll
  for (int i = 0; i < K; ++i) o.log_a[i] = comp_log_norm3(o.kappa[i]);
}

template <int K>
__device__ __forceinline__ double dot_mu(const Mix3<K>& m, int i, D3 nu) {
  return nu.x * m.mu[i][0] + nu.y * m.mu[i][1] + nu.z * m.mu[i][2];
}

template <int K>
__device__ __forceinline__ double mixture_pdf(const Mix3<K>& m, D3 nu) {
  double sum = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i) sum += m.lambda[i] * exp(m.kappa[i] * dot_mu(m, i, nu) + m.log_a[i]);
  return sum;
}

__device__ __forceinline__ D3 reflect(D3 nu, D3 n) { return sub(nu, scl(n, 2.0 * dot(nu, n))); }

template <int K>
__device__ __forceinline__ double reflected_pdf(const Mix3<K>& m, D3 nu, D3 n) {
  if (dot(nu, n) <= 0.0) return 0.0;
  return mixture_pdf(m, nu) + mixture_pdf(m, reflect(nu, n));
}

__device__ __forceinline__ D3 vmf_sample(wg::Pcg& rng, const double* mu, double k) {
  double ct;
  if (k == 0.0) {
    ct = 1.0 - 2.0 * rng.uni();
  } else {
    double u = rng.uni_pos();
    ct = 1.0 + log(u + (1.0 - u) * exp(-2.0 * k)) / k;
    ct = wg::sclamp(ct, -1.0, 1.0);
  }
  double st = sqrt(fmax(0.0, 1.0 - ct * ct));
  double phi = kTwoPi * rng.uni();
  D3 w{mu[0], mu[1], mu[2]};
  double sg = copysign(1.0, w.z);
  double a = -1.0 / (sg + w.z);
  double b = w.x * w.y * a;
  D3 ua{1.0 + sg * w.x * w.x * a, sg * b, -sg * w.x};
  D3 va{b, sg + w.y * w.y * a, -w.y};
  return add(add(scl(ua, st * cos(phi)), scl(va, st * sin(phi))), scl(w, ct));
}

template <int K>
__device__ __forceinline__ D3 mixture_sample(wg::Pcg& rng, const Mix3<K>& m) {
  int pick = 0;
  if (K > 1) {
    double u = rng.uni(), acc = 0.0;
    pick = K - 1;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      acc += m.lambda[i];
      if (u < acc) {
        pick = i;
        break;
      }
    }
  }
  return vmf_sample(rng, m.mu[pick], m.kappa[pick]);
}

template <int K>
__device__ __forceinline__ D3 reflected_sample(wg::Pcg& rng, const Mix3<K>& m, D3 n) {
  D3 nu{0.0, 0.0, 0.0};
  for (int it = 0; it < kMaxProposals; ++it) {
    nu = mixture_sample(rng, m);
    double d = dot(nu, n);
    if (d < 0.0) return reflect(nu, n);
    if (d > 0.0) return nu;
  }
  return nu;
}

__device__ __forceinline__ double uniform_pdf(D3 nu, bool on_n, D3 n) {
  double inv = 1.0 / kFourPi;
  if (!on_n) return inv;
  return dot(nu, n) > 0.0 ? 2.0 * inv : 0.0;
}

__device__ __forceinline__ D3 uniform_sample(wg::Pcg& rng, bool on_n, D3 n) {
  D3 nu{0.0, 0.0, 1.0};
  for (int it = 0; it < kMaxProposals; ++it) {
    double z = 1.0 - 2.0 * rng.uni();
    double s = sqrt(fmax(0.0, 1.0 - z * z));
    double a = kTwoPi * rng.uni();
    nu = {s * cos(a), s * sin(a), z};
    if (!on_n) return nu;
    double d = dot(nu, n);
    if (d > 0.0) return nu;
    if (d < 0.0) return {-nu.x, -nu.y, -nu.z};
  }
  return nu;
}

struct Mis3 {
  D3 nu;
  double pmis, pg, pu;
};

template <int K>
__device__ __forceinline__ double guided_pdf(const Mix3<K>& m, D3 nu, bool on_n, D3 n, bool refl) {
  return on_n ? (refl ? reflected_pdf(m, nu, n) : mixture_pdf(m, nu)) : mixture_pdf(m, nu);
}

template <int K>
__device__ __forceinline__ Mis3 mis_sample(wg::Pcg& rng, const Mix3<K>& m, bool on_n, D3 n, bool refl) {
  Mis3 o;
  bool guided = rng.uni() < m.c;
  if (guided) o.nu = on_n && refl ? reflected_sample(rng, m, n) : mixture_sample(rng, m);
  else o.nu = uniform_sample(rng, on_n, n);
  o.pg = guided_pdf(m, o.nu, on_n, n, refl);
  o.pu = uniform_pdf(o.nu, on_n, n);
  o.pmis = m.c * o.pg + (1.0 - m.c) * o.pu;
  return o;
}

// ---------------------------------------------------------------- Green's
// greens_ball / sample_greens_radius for d = 3 (proj/src/wost.cpp:27-65)
__device__ __forceinline__ double greens_ball3(double r, double R) {
  if (r <= 0.0) return dinf();
  return (1.0 / r - 1.0 / R) / kFourPi;
}
__device__ __forceinline__ double greens_radius3(double u, double R) {
  if (u <= 0.0) return 0.0;
  if (u >= 1.0) return R;
  double lo = 0.0, hi = 1.0, s = sqrt(u);
  for (int it = 0; it < 100; ++it) {
    double f = s * s * (3.0 - 2.0 * s) - u;
    double df = 6.0 * s * (1.0 - s);
    if (f > 0.0) hi = s;
    else lo = s;
    if (fabs(f) < 1e-10) break;
    double step = df > 0.0 ? f / df : 0.0;
    double nx = s - step;
    if (!(nx > lo && nx < hi)) nx = 0.5 * (lo + hi);
    if (nx == s) break;
    s = nx;
  }
  return s * R;
}

// ---------------------------------------------------------------- gradient
__device__ __forceinline__ double dlogv_dkappa3(double t, double kappa) {  // sphdist.cpp:315-321
  double e = expm1(-2.0 * kappa);
  double coth = 1.0 - 2.0 * (e + 1.0) / e;
  return 1.0 / kappa + t - coth;
}

// dV/dTheta' of one direction (sphdist.cpp:324-366), accumulated into g laid
// out like the raw row; returns V
template <int K, class T>
__device__ __forceinline__ double mix_grad_one(const Mix3<K>& m, const T* raw, D3 nu, double* g) {
  double v[K];
  double val = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    v[i] = exp(m.kappa[i] * dot_mu(m, i, nu) + m.log_a[i]);
    val += m.lambda[i] * v[i];
  }
#pragma unroll
  for (int i = 0; i < K; ++i) g[4 * K + i] += m.lambda[i] * (v[i] - val);
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double t = dot_mu(m, i, nu);
    double lv = m.lambda[i] * v[i];
    double ku = exp(static_cast<double>(raw[3 * K + i]));
    if (ku > kKappaMin && ku < kKappaMax) g[3 * K + i] += lv * dlogv_dkappa3(t, m.kappa[i]) * m.kappa[i];
    double mx0 = raw[3 * i], my0 = raw[3 * i + 1], mz0 = raw[3 * i + 2];
    double mn = sqrt(mx0 * mx0 + my0 * my0 + mz0 * mz0);
    if (mn >= 1e-12) {
      double s = lv * m.kappa[i] / mn;
      g[3 * i] += (nu.x - m.mu[i][0] * t) * s;
      g[3 * i + 1] += (nu.y - m.mu[i][1] * t) * s;
      g[3 * i + 2] += (nu.z - m.mu[i][2] * t) * s;
    }
  }
  return val;
}

// kl_grad + selection_grad of one record at the raw outputs, times scale;
// false when the record is skipped (V below the floor) or not finite
template <int K, class T>
__device__ __forceinline__ bool record_dy3(const T* raw, D3 nu, D3 n, bool on_n, double target,
                                           double pdf_mis, double pdf_u, bool refl, bool learn_sel,
                                           double e_fraction, double v_floor, double scale, float* dy) {
  constexpr int OD = 5 * K + 1;
  double g[OD];
#pragma unroll
  for (int j = 0; j < OD; ++j) g[j] = 0.0;
  Mix3<K> m;
  normalize3<K>(raw, m);
  if (target != 0.0) {
    double dv[OD];
#pragma unroll
    for (int j = 0; j < OD; ++j) dv[j] = 0.0;
    double v = mix_grad_one<K>(m, raw, nu, dv);
    if (on_n && refl) v += mix_grad_one<K>(m, raw, reflect(nu, n), dv);
    if (!(v > v_floor)) return false;
    double s = -target / (pdf_mis * v);
#pragma unroll
    for (int j = 0; j < OD - 1; ++j) g[j] = s * dv[j];
  }
  if (learn_sel) {
    double pg = on_n && refl ? reflected_pdf(m, nu, n) : mixture_pdf(m, nu);
    double pnow = m.c * pg + (1.0 - m.c) * pdf_u;
    if (pnow > 0.0) {
      double dc = -e_fraction * target * (pg - pdf_u) / (pnow * pdf_mis);
      g[OD - 1] = dc * m.c * (1.0 - m.c);
    }
  }
  bool fin = true;
#pragma unroll
  for (int j = 0; j < OD; ++j) {
    dy[j] = static_cast<float>(g[j] * scale);
    fin = fin && isfinite(dy[j]);
  }
  return fin;
}

}  // namespace wg3
