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
  float hk[8];   // kappa_i / (2 + |mu_i|^2 - 1): see mixture_pdf32
  float c;
};

// log(I0(k)) - k for k = exp(lk), without logarithms: below 3.75 a degree-10
// Chebyshev-economised polynomial of log I0 in t = (k / 3.75)^2, above it a
// degree-8 one of log(I0(k) e^-k sqrt(k)) in u = 3.75 / k (fitted to
// scipy.special.i0 / i0e; |error| < 2.5e-6 resp. 1.2e-7 in fp32). Both are
// evaluated and one is selected (branch-free, interleaves across lobes); the
// caller already knows log k, the MLP output the concentration comes from.
WG_D float log_i0e_k(float k, float lk, float ik) {
  const float t = k * k * (1.0f / 14.0625f);
  float ps = -5.958795547e-01f;
  ps = fmaf(ps, t, 3.533270836e+00f);
  ps = fmaf(ps, t, -9.344935417e+00f);
  ps = fmaf(ps, t, 1.470542622e+01f);
  ps = fmaf(ps, t, -1.564052677e+01f);
  ps = fmaf(ps, t, 1.233080673e+01f);
  ps = fmaf(ps, t, -7.950976849e+00f);
  ps = fmaf(ps, t, 4.742706299e+00f);
  ps = fmaf(ps, t, -3.085052967e+00f);
  ps = fmaf(ps, t, 3.515514374e+00f);
  ps = ps * t;  // log I0(0) = 0
  const float u = fminf(3.75f * ik, 1.0f);
  float pl = 7.403874304e-03f;
  pl = fmaf(pl, u, -3.077054955e-02f);
  pl = fmaf(pl, u, 4.749890044e-02f);
  pl = fmaf(pl, u, -3.451954946e-02f);
  pl = fmaf(pl, u, 1.407056209e-02f);
  pl = fmaf(pl, u, -1.557706157e-03f);
  pl = fmaf(pl, u, 4.722106736e-03f);
  pl = fmaf(pl, u, 3.332294524e-02f);
  pl = fmaf(pl, u, -9.189384580e-01f);
  return k < 3.75f ? ps - k : pl - 0.5f * lk;
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

// fallback_mu directions (cos, sin)(2 pi i / 8) (sphdist.cpp:274-278)
// (indexed with unrolled constants, so the tables fold into immediates)
WG_D float fallback_cos(int i) {
  const float t[8] = {1.0f, 0.707106769f, 6.12323426e-17f, -0.707106769f,
                      -1.0f, -0.707106769f, -1.83697015e-16f, 0.707106769f};
  return t[i];
}
WG_D float fallback_sin(int i) {
  const float t[8] = {0.0f, 0.707106769f, 1.0f, 0.707106769f,
                      1.22464685e-16f, -0.707106769f, -1.0f, -0.707106769f};
  return t[i];
}

// normalize_params (sphdist.cpp:287-310) for K = 8, dim 2, from fp32 MLP
// outputs. Branch-free so the eight lobes interleave: log I0 evaluates both
// A&S forms and selects, the unit vector uses rsqrt (|mu| = 1 to 1 ulp; the
// sampler renormalises its output in fp64 and the density uses |nu - mu|).
WG_D void normalize32(const float* raw, Mix32& m) {
  const float cr = raw[32];
  const float ec = __expf(-fabsf(cr));  // sigmoid without overflow
  const float sg = 1.0f / (1.0f + ec);
  m.c = cr >= 0.0f ? sg : ec * sg;
  float mx = raw[24];
#pragma unroll
  for (int i = 1; i < 8; ++i) mx = fmaxf(mx, raw[24 + i]);
  float e[8], z = 0.0f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    e[i] = __expf(raw[24 + i] - mx);
    z += e[i];
  }
  const float iz = __frcp_rn(z);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float x = raw[2 * i], y = raw[2 * i + 1];
    const float n2 = x * x + y * y;
    const float r = rsqrtf(n2);
    // fallback_mu (sphdist.cpp:274-278) for |mu| < 1e-12
    const bool fb = !(n2 >= 1e-24f);
    m.mux[i] = fb ? fallback_cos(i) : x * r;
    m.muy[i] = fb ? fallback_sin(i) : y * r;
    // kappa = clamp(exp(raw), 1e-6, 1e4) = exp(clamp(raw, ln 1e-6, ln 1e4))
    const float lk = fminf(fmaxf(raw[16 + i], -13.81551056f), 9.210340372f);
    const float k = __expf(lk);
    m.kappa[i] = k;
    // kappa / (2 + eps) to O(eps^2) = 1e-14
    const float eps = fmaf(m.mux[i], m.mux[i], fmaf(m.muy[i], m.muy[i], -1.0f));  // |mu|^2 - 1
    m.hk[i] = k * fmaf(-0.25f, eps, 0.5f);
    m.lambda[i] = e[i] * iz;
    m.lne[i] = -log_i0e_k(k, lk, __expf(-lk)) - 1.8378770664093453f;  // - log(2 pi)
  }
}

// mixture_pdf (sphdist.cpp:176-185) of the lobes around mu_i / |mu_i| (the
// directions the sampler draws around). For unit nu and |mu|^2 = 1 + eps,
// kappa (nu.mu^ - 1) = -kappa |nu - mu|^2 / (2 + eps) exactly: no
// cancellation near the mode, so the exponent is formed in fp32 with full
// relative accuracy; nu enters as an fp32 hi + lo pair, so nu - mu is exact
// to fp32 rounding even for concentrated lobes (fx - mu is Sterbenz-exact).
WG_D double mixture_pdf32(const Mix32& m, double nx, double ny) {
  const float fx = static_cast<float>(nx), fy = static_cast<float>(ny);
  const float lx = static_cast<float>(nx - static_cast<double>(fx));
  const float ly = static_cast<float>(ny - static_cast<double>(fy));
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float dx = (fx - m.mux[i]) + lx, dy = (fy - m.muy[i]) + ly;
    const float arg = fmaf(-m.hk[i], fmaf(dx, dx, dy * dy), m.lne[i]);
    s = fmaf(m.lambda[i], __expf(arg), s);
  }
  return s;
}

WG_D double reflected_pdf32(const Mix32& m, double nx, double ny, double px, double py) {
  if (nx * px + ny * py <= 0.0) return 0.0;
  double rx, ry;
  reflect(nx, ny, px, py, &rx, &ry);
  return mixture_pdf32(m, nx, ny) + mixture_pdf32(m, rx, ry);
}

// Uniforms on this path are fp32 draws from single PCG32 outputs (Pcg::unif).
// Best-Fisher (sphdist.cpp:120-140) in fp32, returning the sampled angle as
// (cos th, sin th) directly. Every quantity that the reference forms by
// cancellation is rewritten exactly:
//   r - 1 = (1 - rho)^2 / (2 rho),  1 -+ z = 2 sin^2 / cos^2(pi u1 / 2),
//   r - f = (r - 1)(r + 1) / (r + z),  1 - f = (r - 1)(1 - z) / (r + z),
// so cv = kappa (r - f) and sin th = sqrt((1 - f)(1 + f)) keep full fp32
// relative accuracy for concentrated lobes (kappa up to 1e4), and no acos /
// cos / sin is needed (cos(acos f) = f). The envelope test is exact for any
// r > 1, so fp32 rounding of rho only changes the acceptance rate. Same
// three uniforms per accepted proposal (u1, u2, u3) as the reference.
WG_D void vm_cos_sin(Pcg& rng, float kappa, float* oc, float* os) {
  const float s = sqrtf(fmaf(4.0f * kappa, kappa, 1.0f));
  const float tau = 1.0f + s;
  const float rho = __fdividef(2.0f * kappa * tau, (s + 1.0f) * (tau + sqrtf(2.0f * tau)));
  // r - 1 > 0; r itself is never rounded to fp32 (for kappa = 1e4, r - 1 =
  // 5e-5 would lose 3 digits in 1 + (r - 1)): every place r appears is
  // written in terms of rm1, so proposal and test use the same exact r
  const float rm1 = __fdividef((1.0f - rho) * (1.0f - rho), 2.0f * rho);
  for (int it = 0;; ++it) {
    if (it == kMaxProposals) {  // NaN parameters: see kMaxProposals
      *oc = *os = kappa * 0.0f / 0.0f;
      return;
    }
    const float u1 = rng.unif_pos();
    float hs, hc;
    sincospif(0.5f * u1, &hs, &hc);
    const float omz = 2.0f * hs * hs;                   // 1 - z, z = cos(pi u1)
    const float inv = __frcp_rn(fmaf(2.0f * hc, hc, rm1));  // 1 / (r + z), r + z = (1 + z) + rm1
    const float cv = kappa * rm1 * (2.0f + rm1) * inv;  // kappa (r - f)
    const float omf = rm1 * omz * inv;                   // 1 - f
    const float u2 = rng.unif_pos();
    if (cv * (2.0f - cv) - u2 > 0.0f || __logf(__fdividef(cv, u2)) + 1.0f - cv >= 0.0f) {
      const float u3 = rng.unif();
      const float sn = sqrtf(fmaxf(omf * (2.0f - omf), 0.0f));
      *oc = fminf(fmaxf(1.0f - omf, -1.0f), 1.0f);
      *os = u3 < 0.5f ? -sn : sn;
      return;
    }
  }
}

// unit fp32 direction -> fp64 with |nu| = 1 to ~1e-15 (see Mix32): |v|^2 =
// 1 + d with |d| < 1e-6, one Newton step of rsqrt about 1 (error 3d^2/8)
WG_D void unit64(float x, float y, double* ox, double* oy) {
  const double dx = x, dy = y;
  const double inv = fma(-0.5, fma(dx, dx, dy * dy), 1.5);
  *ox = dx * inv;
  *oy = dy * inv;
}

WG_D void mixture_sample32(Pcg& rng, const Mix32& m, double* ox, double* oy) {
  const float u = rng.unif();
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
  float c, sn;
  vm_cos_sin(rng, kap, &c, &sn);
  unit64(c * mux - sn * muy, c * muy + sn * mux, ox, oy);
}

WG_D void reflected_sample32(Pcg& rng, const Mix32& m, double px, double py, double* ox, double* oy) {
  for (int it = 0;; ++it) {
    double nx, ny;
    mixture_sample32(rng, m, &nx, &ny);
    double d = nx * px + ny * py;
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

// uniform_dir_sample (sphdist.cpp:226-243) with one fp32 sincospi per
// proposal: full circle, or the hemisphere around the Neumann normal by flipping
WG_D void uniform_sample32(Pcg& rng, bool on_n, double px, double py, double* ox, double* oy) {
  for (int it = 0;; ++it) {
    float sn, cs;
    sincospif(2.0f * rng.unif(), &sn, &cs);
    double nx, ny;
    unit64(cs, sn, &nx, &ny);
    const double d = on_n ? nx * px + ny * py : 1.0;
    if (d != 0.0 || it + 1 == kMaxProposals) {
      *ox = d > 0.0 ? nx : -nx;
      *oy = d > 0.0 ? ny : -ny;
      return;
    }
  }
}

// mis_sample (sphdist.cpp:254-270) on the fp32 mixture, in two halves so the
// walk kernel can time them: the direction draw and the densities at it
WG_D bool mis_draw32(Pcg& rng, const Mix32& m, double c, bool on_n, double px, double py, bool refl,
                     double* nx, double* ny) {
  const bool guided = rng.unif() < static_cast<float>(c);
  if (guided) {
    if (on_n && refl) reflected_sample32(rng, m, px, py, nx, ny);
    else mixture_sample32(rng, m, nx, ny);
  } else {
    uniform_sample32(rng, on_n, px, py, nx, ny);
  }
  return guided;
}

WG_D MisOut mis_eval32(const Mix32& m, double c, bool on_n, double px, double py, bool refl, double nx,
                       double ny) {
  MisOut o;
  o.nx = nx;
  o.ny = ny;
  o.pg = on_n && refl ? reflected_pdf32(m, nx, ny, px, py) : mixture_pdf32(m, nx, ny);
  o.pu = uniform_pdf(on_n, nx, ny, px, py);
  o.pmis = c * o.pg + (1.0 - c) * o.pu;
  return o;
}

WG_D MisOut mis_sample32(Pcg& rng, const Mix32& m, double c, bool on_n, double px, double py,
                         bool refl) {
  double nx, ny;
  mis_draw32(rng, m, c, on_n, px, py, refl, &nx, &ny);
  return mis_eval32(m, c, on_n, px, py, refl, nx, ny);
}

}  // namespace wg
