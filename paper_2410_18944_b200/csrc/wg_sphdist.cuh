// Directional distributions on S^1 in fp64 (proj/src/sphdist.cpp): Bessel
// normalisers, vMF mixture density and sampling, Neumann reflection, one-
// sample MIS against uniform directions and the Table-1 normalisation.
// Operation order follows the reference so that decoded mixtures match it to
// the last bit wherever CUDA's libm agrees with the host's (exp/log/cos/...
// are within 1-2 ulp of glibc; the rest is IEEE-exact).
#pragma once

#include "wg_device.cuh"

namespace wg {

// I0 / I1 power series below 20 (sphdist.cpp:26-46)
WG_D double i0_series(double x) {
  double q = 0.25 * x * x, term = 1.0, sum = 1.0;
  for (int m = 1; m < 200; ++m) {
    term *= q * (1.0 / (static_cast<double>(m) * m));
    sum += term;
    if (term < 1e-17 * sum) break;
  }
  return sum;
}
WG_D double i1_series(double x) {
  double q = 0.25 * x * x, term = 0.5 * x, sum = term;
  for (int m = 1; m < 200; ++m) {
    term *= q * (1.0 / (static_cast<double>(m) * (m + 1)));
    sum += term;
    if (term < 1e-17 * sum) break;
  }
  return sum;
}
// Hankel asymptotic correction (sphdist.cpp:49-60)
WG_D double asym_corr(double x, double mu) {
  double sum = 1.0, term = 1.0, prev = dinf();
  for (int k = 1; k < 30; ++k) {
    term *= -(mu - (2.0 * k - 1.0) * (2.0 * k - 1.0)) / (8.0 * x * k);
    if (fabs(term) >= prev) break;
    sum += term;
    prev = fabs(term);
    if (fabs(term) < 1e-16 * fabs(sum)) break;
  }
  return sum;
}
WG_D double log_bessel_i0(double x) {  // sphdist.cpp:69-72
  if (x < 20.0) return log(i0_series(x));
  return x - 0.5 * log(kTwoPi * x) + log(asym_corr(x, 0.0));
}
WG_D double bessel_i1_over_i0(double x) {  // sphdist.cpp:74-78
  if (x == 0.0) return 0.0;
  if (x < 20.0) return i1_series(x) / i0_series(x);
  return asym_corr(x, 4.0) / asym_corr(x, 0.0);
}

// decoded mixture (MixtureParams, sphdist.hpp:29-39), 2D only on the walk path
struct Mix {
  double mux[kMaxK], muy[kMaxK];
  double kappa[kMaxK], lambda[kMaxK], log_a[kMaxK];
  double c;
  int k;
};

// vmf_pdf in 2D (sphdist.cpp:82-92)
WG_D double vmf_pdf2(double nx, double ny, double mux, double muy, double kappa) {
  if (kappa == 0.0) return 1.0 / kTwoPi;
  double t = nx * mux + ny * muy + 0.0 * 0.0;
  return exp(kappa * t - log_bessel_i0(kappa)) / kTwoPi;
}

// mixture_pdf (sphdist.cpp:176-185); dot is the reference's Vec3 dot with z=0
WG_D double mixture_pdf(const Mix& m, double nx, double ny) {
  double sum = 0.0;
  for (int i = 0; i < m.k; ++i) {
    double la = m.log_a[i];
    double dt = nx * m.mux[i] + ny * m.muy[i] + 0.0 * 0.0;
    sum += la != 0.0 ? m.lambda[i] * exp(m.kappa[i] * dt + la)
                     : m.lambda[i] * vmf_pdf2(nx, ny, m.mux[i], m.muy[i], m.kappa[i]);
  }
  return sum;
}

// reflect_off_plane (sphdist.hpp:129-131)
WG_D void reflect(double nx, double ny, double px, double py, double* rx, double* ry) {
  double d = 2.0 * (nx * px + ny * py + 0.0 * 0.0);
  *rx = nx - px * d;
  *ry = ny - py * d;
}

// reflected_pdf (sphdist.cpp:204-208)
WG_D double reflected_pdf(const Mix& m, double nx, double ny, double px, double py) {
  if (nx * px + ny * py + 0.0 * 0.0 <= 0.0) return 0.0;
  double rx, ry;
  reflect(nx, ny, px, py, &rx, &ry);
  return mixture_pdf(m, nx, ny) + mixture_pdf(m, rx, ry);
}

// Rejection loops on the device are capped at kMaxProposals: with
// acceptance >= 1/2 per proposal a legitimate draw never reaches it, and
// NaN parameters (which no comparison accepts) cannot hang a kernel; they
// yield a NaN direction and the walk escapes the bbox test.
constexpr int kMaxProposals = 4096;

// Best-Fisher rejection sampler (sphdist.cpp:111-128)
WG_D double vm_angle(Pcg& rng, double kappa) {
  double tau = 1.0 + sqrt(1.0 + 4.0 * kappa * kappa);
  double rho = (tau - sqrt(2.0 * tau)) / (2.0 * kappa);
  double r = (1.0 + rho * rho) / (2.0 * rho);
  for (int it = 0;; ++it) {
    if (it == kMaxProposals) return kappa * 0.0 / 0.0;  // NaN
    double u1 = rng.uni_pos();
    double z = cos(kPi * u1);
    double f = (1.0 + r * z) / (r + z);
    double cv = kappa * (r - f);
    double u2 = rng.uni_pos();
    if (cv * (2.0 - cv) - u2 > 0.0 || log(cv / u2) + 1.0 - cv >= 0.0) {
      double u3 = rng.uni();
      double th = acos(sclamp(f, -1.0, 1.0));
      return u3 < 0.5 ? -th : th;
    }
  }
}

// vmf_sample 2D (sphdist.cpp:132-140) with rotate_to_frame2 (:97-99)
WG_D void vmf_sample2(Pcg& rng, double mux, double muy, double kappa, double* ox, double* oy) {
  double c, s;
  if (kappa == 0.0) {
    double a = kTwoPi * rng.uni();
    c = cos(a);
    s = sin(a);
  } else {
    double th = vm_angle(rng, kappa);
    c = cos(th);
    s = sin(th);
  }
  *ox = c * mux - s * muy;
  *oy = c * muy + s * mux;
}

// mixture_sample (sphdist.cpp:187-202)
WG_D void mixture_sample(Pcg& rng, const Mix& m, double* ox, double* oy) {
  int pick = 0;
  if (m.k > 1) {
    double u = rng.uni(), acc = 0.0;
    pick = m.k - 1;
    for (int i = 0; i < m.k; ++i) {
      acc += m.lambda[i];
      if (u < acc) {
        pick = i;
        break;
      }
    }
  }
  vmf_sample2(rng, m.mux[pick], m.muy[pick], m.kappa[pick], ox, oy);
}

// reflected_sample (sphdist.cpp:210-218)
WG_D void reflected_sample(Pcg& rng, const Mix& m, double px, double py, double* ox, double* oy) {
  for (int it = 0;; ++it) {
    double nx, ny;
    mixture_sample(rng, m, &nx, &ny);
    double d = nx * px + ny * py + 0.0 * 0.0;
    if (d < 0.0) {
      reflect(nx, ny, px, py, ox, oy);
      return;
    }
    if (d > 0.0 || it + 1 == kMaxProposals) {
      *ox = nx;
      *oy = ny;
      return;
    }
  }
}

// uniform_dir_sample 2D (sphdist.cpp:226-243); on_n selects the hemisphere
WG_D void uniform_sample(Pcg& rng, bool on_n, double px, double py, double* ox, double* oy) {
  for (int it = 0;; ++it) {
    double a = kTwoPi * rng.uni();
    double nx = cos(a), ny = sin(a);
    if (!on_n) {
      *ox = nx;
      *oy = ny;
      return;
    }
    double d = nx * px + ny * py + 0.0 * 0.0;
    if (d > 0.0) {
      *ox = nx;
      *oy = ny;
      return;
    }
    if (d < 0.0 || it + 1 == kMaxProposals) {
      *ox = -nx;
      *oy = -ny;
      return;
    }
  }
}

// uniform_dir_pdf 2D (sphdist.cpp:220-224)
WG_D double uniform_pdf(bool on_n, double nx, double ny, double px, double py) {
  double inv = 1.0 / kTwoPi;
  if (!on_n) return inv;
  return nx * px + ny * py + 0.0 * 0.0 > 0.0 ? 2.0 * inv : 0.0;
}

struct MisOut {
  double nx, ny, pmis, pg, pu;
};

// mis_sample (sphdist.cpp:254-270)
WG_D MisOut mis_sample(Pcg& rng, const Mix& m, bool on_n, double px, double py, bool refl) {
  MisOut o;
  bool guided = rng.uni() < m.c;
  if (guided) {
    if (on_n && refl) reflected_sample(rng, m, px, py, &o.nx, &o.ny);
    else mixture_sample(rng, m, &o.nx, &o.ny);
  } else {
    uniform_sample(rng, on_n, px, py, &o.nx, &o.ny);
  }
  o.pg = on_n ? (refl ? reflected_pdf(m, o.nx, o.ny, px, py) : mixture_pdf(m, o.nx, o.ny))
              : mixture_pdf(m, o.nx, o.ny);
  o.pu = uniform_pdf(on_n, o.nx, o.ny, px, py);
  o.pmis = m.c * o.pg + (1.0 - m.c) * o.pu;
  return o;
}

WG_D double sigmoid(double x) {  // sphdist.cpp:280-283
  return x >= 0.0 ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x));
}

// normalize_params(unpack_params(raw)) for dim 2 (sphdist.cpp:287-310,
// guide_field.cpp:424-441); raw layout [mu (2k) | kappa (k) | lambda (k) | c]
template <int K, typename T>
WG_D void normalize2(const T* raw, int k_rt, Mix& o) {
  const int k = K ? K : k_rt;
  o.k = k;
  o.c = sigmoid(static_cast<double>(raw[4 * k]));
  double mx = -dinf();
#pragma unroll
  for (int i = 0; i < (K ? K : kMaxK); ++i)
    if (i < k) mx = smax(mx, static_cast<double>(raw[3 * k + i]));
  double z = 0.0;
#pragma unroll
  for (int i = 0; i < (K ? K : kMaxK); ++i)
    if (i < k) z += exp(static_cast<double>(raw[3 * k + i]) - mx);
#pragma unroll
  for (int i = 0; i < (K ? K : kMaxK); ++i) {
    if (i >= k) break;
    double mx_ = raw[2 * i], my_ = raw[2 * i + 1];
    double mn = sqrt(mx_ * mx_ + my_ * my_ + 0.0 * 0.0);
    if (mn < 1e-12) {  // fallback_mu (sphdist.cpp:274-278)
      double a = kTwoPi * i / kMaxK;
      o.mux[i] = cos(a);
      o.muy[i] = sin(a);
    } else {
      o.mux[i] = mx_ / mn;
      o.muy[i] = my_ / mn;
    }
    o.kappa[i] = sclamp(exp(static_cast<double>(raw[2 * k + i])), kKappaMin, kKappaMax);
    o.lambda[i] = exp(static_cast<double>(raw[3 * k + i]) - mx) / z;
  }
  // component_log_norm, d = 2 (sphdist.cpp:162-167)
#pragma unroll
  for (int i = 0; i < (K ? K : kMaxK); ++i)
    if (i < k) o.log_a[i] = -log_bessel_i0(o.kappa[i]) - log(kTwoPi);
}

}  // namespace wg
