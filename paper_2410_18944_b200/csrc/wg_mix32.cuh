// Fast mixture math for the tensor-core walk path: the Table-1 normalisation
// and the per-component mixture densities in fp32 (the MLP output is fp32
// anyway), with the two numerically delicate pieces kept exact:
//   * the exponent of each vMF term is formed as kappa * (nu.mu - 1) in fp64
//     and only then rounded, so high-kappa lobes keep full relative accuracy;
//   * the Best-Fisher sampler of the picked component runs in fp64 with the
//     cancellation-free rho = 2 kappa tau / ((s + 1)(tau + sqrt(2 tau))).
// The sampler and the density use the same decoded parameters, so the
// multiplier p_u / p_mis is consistent with the sampled direction to fp32
// rounding and the estimator stays unbiased. log I0 uses the
// Abramowitz-Stegun 9.8.1 / 9.8.2 rational forms (|rel err| < 2e-7) in the
// exponentially scaled form log(I0(k)) - k.
#pragma once

#include "wg_sphdist.cuh"

namespace wg {

struct Mix32 {
  // fp32 mean directions; a SAMPLED direction is renormalised in fp64 (a step
  // of length R along |nu| = 1 + 6e-8 would overshoot a Dirichlet wall on the
  // bbox edge by more than the 1e-9 diag escape pad, wost.cpp:259-263). The
  // density evaluates the same promoted mu, so sampler and pdf stay consistent.
  float mux[8], muy[8];
  float kappa[8], lambda[8];
  float lne[8];  // log normaliser + kappa: v_i = exp(kappa_i (t_i - 1) + lne_i)
  float c;
};

// log(I0(x)) - x for x >= 0 (A&S 9.8.1 below 3.75, 9.8.2 above)
WG_D float log_i0e(float x) {
  if (x < 3.75f) {
    float t = x * (1.0f / 3.75f);
    t *= t;
    float p = 1.0f + t * (3.5156229f + t * (3.0899424f + t * (1.2067492f + t * (0.2659732f +
              t * (0.0360768f + t * 0.0045813f)))));
    return __logf(p) - x;
  }
  float t = 3.75f / x;
  float p = 0.39894228f + t * (0.01328592f + t * (0.00225319f + t * (-0.00157565f + t * (0.00916281f +
            t * (-0.02057706f + t * (0.02635537f + t * (-0.01647633f + t * 0.00392377f)))))));
  return __logf(p) - 0.5f * __logf(x);
}

// I1(x) / I0(x) for x >= 0 (A&S 9.8.1-9.8.4; the e^x / sqrt(x) factors
// cancel above 3.75), relative error < 3e-7
WG_D float i1_over_i0_f(float x) {
  if (x < 3.75f) {
    float t = x * (1.0f / 3.75f);
    t *= t;
    float p0 = 1.0f + t * (3.5156229f + t * (3.0899424f + t * (1.2067492f + t * (0.2659732f +
               t * (0.0360768f + t * 0.0045813f)))));
    float p1 = 0.5f + t * (0.87890594f + t * (0.51498869f + t * (0.15084934f + t * (0.02658733f +
               t * (0.00301532f + t * 0.00032411f)))));
    return x * p1 / p0;
  }
  float t = 3.75f / x;
  float q0 = 0.39894228f + t * (0.01328592f + t * (0.00225319f + t * (-0.00157565f + t * (0.00916281f +
             t * (-0.02057706f + t * (0.02635537f + t * (-0.01647633f + t * 0.00392377f)))))));
  float q1 = 0.39894228f + t * (-0.03988024f + t * (-0.00362018f + t * (0.00163801f + t * (-0.01031555f +
             t * (0.02282967f + t * (-0.02895312f + t * (0.01787654f + t * -0.00420059f)))))));
  return q1 / q0;
}

// normalize_params (sphdist.cpp:287-310) for K = 8, dim 2, from fp32 MLP outputs
WG_D void normalize32(const float* raw, Mix32& m) {
  float cr = raw[32];
  m.c = cr >= 0.0f ? 1.0f / (1.0f + __expf(-cr)) : __expf(cr) / (1.0f + __expf(cr));
  float mx = raw[24];
#pragma unroll
  for (int i = 1; i < 8; ++i) mx = fmaxf(mx, raw[24 + i]);
  float e[8], z = 0.0f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    e[i] = __expf(raw[24 + i] - mx);
    z += e[i];
  }
  const float iz = 1.0f / z;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float x = raw[2 * i], y = raw[2 * i + 1];
    float n = sqrtf(x * x + y * y);
    if (n < 1e-12f) {  // fallback_mu, sphdist.cpp:274-278
      float a = static_cast<float>(kTwoPi * i / kMaxK);
      m.mux[i] = cosf(a);
      m.muy[i] = sinf(a);
    } else {
      m.mux[i] = x / n;
      m.muy[i] = y / n;
    }
    float k = fminf(fmaxf(__expf(raw[16 + i]), 1e-6f), 1e4f);
    m.kappa[i] = k;
    m.lambda[i] = e[i] * iz;
    m.lne[i] = -log_i0e(k) - 1.8378770664093453f;  // - log(2 pi)
  }
}

// mixture_pdf (sphdist.cpp:176-185)
WG_D double mixture_pdf32(const Mix32& m, double nx, double ny) {
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double t = nx * m.mux[i] + ny * m.muy[i];
    float arg = static_cast<float>(static_cast<double>(m.kappa[i]) * (t - 1.0)) + m.lne[i];
    s += m.lambda[i] * __expf(arg);
  }
  return s;
}

WG_D double reflected_pdf32(const Mix32& m, double nx, double ny, double px, double py) {
  if (nx * px + ny * py <= 0.0) return 0.0;
  double rx, ry;
  reflect(nx, ny, px, py, &rx, &ry);
  return mixture_pdf32(m, nx, ny) + mixture_pdf32(m, rx, ry);
}

// Best-Fisher with the cancellation-free rho (fp64)
WG_D double vm_angle_stable(Pcg& rng, double kappa) {
  double s = sqrt(1.0 + 4.0 * kappa * kappa);
  double tau = 1.0 + s;
  double rho = 2.0 * kappa * tau / ((s + 1.0) * (tau + sqrt(2.0 * tau)));
  double r = (1.0 + rho * rho) / (2.0 * rho);
  for (;;) {
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

WG_D void mixture_sample32(Pcg& rng, const Mix32& m, double* ox, double* oy) {
  double u = rng.uni();
  float acc = 0.0f;
  float mux = m.mux[7], muy = m.muy[7];
  float kap = m.kappa[7];
  bool found = false;
#pragma unroll
  for (int i = 0; i < 8; ++i) {  // register-resident select of the picked lobe
    acc += m.lambda[i];
    if (!found && u < acc) {
      found = true;
      mux = m.mux[i];
      muy = m.muy[i];
      kap = m.kappa[i];
    }
  }
  double th = vm_angle_stable(rng, kap);
  double c = cos(th), s = sin(th);
  double dx = c * mux - s * muy, dy = c * muy + s * mux;
  double inv = 1.0 / sqrt(dx * dx + dy * dy);  // exact unit length (see Mix32)
  *ox = dx * inv;
  *oy = dy * inv;
}

WG_D void reflected_sample32(Pcg& rng, const Mix32& m, double px, double py, double* ox, double* oy) {
  for (;;) {
    double nx, ny;
    mixture_sample32(rng, m, &nx, &ny);
    double d = nx * px + ny * py;
    if (d < 0.0) {
      reflect(nx, ny, px, py, ox, oy);
      return;
    }
    if (d > 0.0) {
      *ox = nx;
      *oy = ny;
      return;
    }
  }
}

// mis_sample (sphdist.cpp:254-270) on the fp32 mixture
WG_D MisOut mis_sample32(Pcg& rng, const Mix32& m, double c, bool on_n, double px, double py,
                         bool refl) {
  MisOut o;
  bool guided = rng.uni() < c;
  if (guided) {
    if (on_n && refl) reflected_sample32(rng, m, px, py, &o.nx, &o.ny);
    else mixture_sample32(rng, m, &o.nx, &o.ny);
  } else {
    uniform_sample(rng, on_n, px, py, &o.nx, &o.ny);
  }
  o.pg = on_n ? (refl ? reflected_pdf32(m, o.nx, o.ny, px, py) : mixture_pdf32(m, o.nx, o.ny))
              : mixture_pdf32(m, o.nx, o.ny);
  o.pu = uniform_pdf(on_n, o.nx, o.ny, px, py);
  o.pmis = c * o.pg + (1.0 - c) * o.pu;
  return o;
}

}  // namespace wg
