// d = 3 vMF mixtures in fp32 for the tensor-core 3D walk kernels (the
// direction epilogue of wave_dir_kernel / walk3_tc_kernel); the exact kernel
// keeps the fp64 forms of wg3_mix.cuh, which these follow
// (sphdist.cpp:132-310) with cancellation-free rewrites:
//   * density exp(lne - kappa |nu - mu|^2 / 2): for unit vectors
//     kappa (nu.mu - 1) = -kappa |nu - mu|^2 / 2 exactly, and nu - mu is
//     formed in fp64 before rounding, so concentrated lobes (kappa up to
//     1e4) keep their relative accuracy;
//   * log-normaliser lne = log kappa - log(2 pi (1 - e^{-2 kappa})) with
//     expm1f, accurate down to kappa = 1e-6;
//   * inverse-CDF sampling written in 1 - w = -log(u + (1 - u) e^{-2 kappa}) /
//     kappa and sin(theta) = sqrt((1 - w)(1 + w)), no cancellation near the
//     mode;
//   * sampled directions renormalised in fp64 (one Newton step) because the
//     walk moves in fp64 and escapes are tested against a 1e-9 diag pad.
// Random draws are the fp64 kernel's (same PCG32 calls in the same order).
#pragma once

#include "wg3_mix.cuh"

namespace wg3 {

struct Mix3f {
  float mu[8][3];
  float kappa[8], lambda[8], lne[8];
  float c;
};

__device__ __forceinline__ void normalize3f(const float* raw, Mix3f& o) {
  const float cr = raw[40];
  o.c = cr >= 0.0f ? 1.0f / (1.0f + __expf(-cr)) : __expf(cr) / (1.0f + __expf(cr));
  float mx = raw[32];
#pragma unroll
  for (int i = 1; i < 8; ++i) mx = fmaxf(mx, raw[32 + i]);
  float e[8], z = 0.0f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    e[i] = __expf(raw[32 + i] - mx);
    z += e[i];
  }
  const float iz = 1.0f / z;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float x = raw[3 * i], y = raw[3 * i + 1], w = raw[3 * i + 2];
    const float n2 = x * x + y * y + w * w;
    if (n2 < 1e-24f) {  // zero-norm fallback directions (sphdist.cpp:274-278)
      float s, c;
      sincospif(2.0f * i / WG_MAX_MIXTURE, &s, &c);
      o.mu[i][0] = c;
      o.mu[i][1] = s;
      o.mu[i][2] = 0.0f;
    } else {
      const float r = rsqrtf(n2);
      o.mu[i][0] = x * r;
      o.mu[i][1] = y * r;
      o.mu[i][2] = w * r;
    }
    const float k = fminf(fmaxf(__expf(raw[24 + i]), 1e-6f), 1e4f);
    o.kappa[i] = k;
    o.lambda[i] = e[i] * iz;
    o.lne[i] = __logf(k) - __logf(-expm1f(-2.0f * k)) - 1.8378770664f;  // log(2 pi)
  }
}

__device__ __forceinline__ double mixture_pdf3f(const Mix3f& m, D3 nu) {
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float dx = static_cast<float>(nu.x - static_cast<double>(m.mu[i][0]));
    const float dy = static_cast<float>(nu.y - static_cast<double>(m.mu[i][1]));
    const float dz = static_cast<float>(nu.z - static_cast<double>(m.mu[i][2]));
    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    s = fmaf(m.lambda[i], __expf(fmaf(-0.5f * m.kappa[i], d2, m.lne[i])), s);
  }
  return s;
}

__device__ __forceinline__ double reflected_pdf3f(const Mix3f& m, D3 nu, D3 n) {
  if (dot(nu, n) <= 0.0) return 0.0;
  return mixture_pdf3f(m, nu) + mixture_pdf3f(m, reflect(nu, n));
}

// unit fp64 vector from an fp32-accurate direction: one Newton step on |v|
__device__ __forceinline__ D3 unit3(D3 v) {
  const double q = dot(v, v);
  const double s = 1.5 - 0.5 * q;  // 1 / sqrt(q) to second order near q = 1
  return scl(v, s);
}

__device__ __forceinline__ D3 vmf_sample3f(wg::Pcg& rng, const float* mu, float k) {
  float om;  // 1 - w
  if (k == 0.0f) {
    om = static_cast<float>(2.0 * rng.uni());
  } else {
    const float u = static_cast<float>(rng.uni_pos());
    om = -__logf(fmaf(1.0f - u, __expf(-2.0f * k), u)) / k;
    om = fminf(fmaxf(om, 0.0f), 2.0f);
  }
  const float ct = 1.0f - om;
  const float st = sqrtf(om * (2.0f - om));
  float sp, cp;
  sincospif(static_cast<float>(2.0 * rng.uni()), &sp, &cp);
  const float wx = mu[0], wy = mu[1], wz = mu[2];
  const float sg = copysignf(1.0f, wz);
  const float a = -1.0f / (sg + wz);
  const float b = wx * wy * a;
  const float ux = 1.0f + sg * wx * wx * a, uy = sg * b, uz = -sg * wx;
  const float vx = b, vy = sg + wy * wy * a, vz = -wy;
  const float c1 = st * cp, c2 = st * sp;
  D3 v{fmaf(ux, c1, fmaf(vx, c2, wx * ct)), fmaf(uy, c1, fmaf(vy, c2, wy * ct)),
       fmaf(uz, c1, fmaf(vz, c2, wz * ct))};
  return unit3(v);
}

__device__ __forceinline__ D3 mixture_sample3f(wg::Pcg& rng, const Mix3f& m) {
  const float u = static_cast<float>(rng.uni());
  float acc = 0.0f;
  int pick = 7;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    acc += m.lambda[i];
    if (u < acc) {
      pick = i;
      break;
    }
  }
  return vmf_sample3f(rng, m.mu[pick], m.kappa[pick]);
}

__device__ __forceinline__ D3 reflected_sample3f(wg::Pcg& rng, const Mix3f& m, D3 n) {
  D3 nu{0.0, 0.0, 0.0};
  for (int it = 0; it < kMaxProposals; ++it) {
    nu = mixture_sample3f(rng, m);
    const double d = dot(nu, n);
    if (d < 0.0) return reflect(nu, n);
    if (d > 0.0) return nu;
  }
  return nu;
}

// uniform_sample (wg3_mix.cuh) with the same draws, the azimuth's sine and
// cosine in fp32 (sincospif) instead of fp64 sin / cos, renormalised in fp64
__device__ __forceinline__ D3 uniform_sample3f(wg::Pcg& rng, bool on_n, D3 n) {
  D3 nu{0.0, 0.0, 1.0};
  for (int it = 0; it < kMaxProposals; ++it) {
    const double z = 1.0 - 2.0 * rng.uni();
    const float s = sqrtf(fmaxf(0.0f, static_cast<float>((1.0 - z) * (1.0 + z))));
    float sp, cp;
    sincospif(static_cast<float>(2.0 * rng.uni()), &sp, &cp);
    nu = unit3(D3{static_cast<double>(s * cp), static_cast<double>(s * sp), z});
    if (!on_n) return nu;
    const double d = dot(nu, n);
    if (d > 0.0) return nu;
    if (d < 0.0) return {-nu.x, -nu.y, -nu.z};
  }
  return nu;
}

// mis_sample (sphdist.cpp:254-270) with the fp32 mixture; c is the (possibly
// mode-overridden) selection probability
__device__ __forceinline__ Mis3 mis_sample3f(wg::Pcg& rng, const Mix3f& m, double c, bool on_n, D3 n, bool refl) {
  Mis3 o;
  const bool guided = rng.uni() < c;
  if (guided) o.nu = on_n && refl ? reflected_sample3f(rng, m, n) : mixture_sample3f(rng, m);
  else o.nu = uniform_sample3f(rng, on_n, n);
  o.pg = on_n && refl ? reflected_pdf3f(m, o.nu, n) : mixture_pdf3f(m, o.nu);
  o.pu = uniform_pdf(o.nu, on_n, n);
  o.pmis = c * o.pg + (1.0 - c) * o.pu;
  return o;
}

}  // namespace wg3
