// Per-record training loss gradient at the MLP outputs (fp64):
//   kl_grad (proj/src/guide_train.cpp:25-42) with mixture_grad(_reflected)
//   (proj/src/sphdist.cpp:324-381) and selection_grad (guide_train.cpp:44-56).
// Shared by the CUDA-core and the tcgen05 training tiles.
#pragma once

#include "wg_mix32.cuh"
#include "wg_sphdist.cuh"
#include "wg_train.cuh"

namespace wg {

// ---------------------------------------------------------------- loss grad
// dV/dTheta' of one direction (sphdist.cpp:324-366); accumulates into g
template <int K>
WG_D double mix_grad_one(const Mix& m, const float* raw, double nx, double ny, double* g) {
  double v[K];
  double val = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double dt = nx * m.mux[i] + ny * m.muy[i] + 0.0 * 0.0;
    v[i] = exp(m.kappa[i] * dt + m.log_a[i]);
    val += m.lambda[i] * v[i];
  }
#pragma unroll
  for (int i = 0; i < K; ++i) g[3 * K + i] += m.lambda[i] * (v[i] - val);
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double t = nx * m.mux[i] + ny * m.muy[i] + 0.0 * 0.0;
    double lv = m.lambda[i] * v[i];
    double ku = exp(static_cast<double>(raw[2 * K + i]));
    if (ku > kKappaMin && ku < kKappaMax)
      g[2 * K + i] += lv * (t - bessel_i1_over_i0(m.kappa[i])) * m.kappa[i];
    double mx = raw[2 * i], my = raw[2 * i + 1];
    double mn = sqrt(mx * mx + my * my + 0.0 * 0.0);
    if (mn >= 1e-12) {
      double s = lv * m.kappa[i] / mn;
      g[2 * i] += (nx - m.mux[i] * t) * s;
      g[2 * i + 1] += (ny - m.muy[i] * t) * s;
    }
  }
  return val;
}

// kl_grad (guide_train.cpp:25-42) + selection_grad (:44-56) for one record;
// writes dL/d(raw output) scaled by inv_count into dy. Returns false when the
// record is skipped (V below the floor).
template <int K>
WG_D bool record_dy(const float* raw, const DevRecord& r, const TrainArgs& a, float* dy) {
  constexpr int OD = 4 * K + 1;
  double g[OD];
#pragma unroll
  for (int j = 0; j < OD; ++j) g[j] = 0.0;
  Mix m;
  normalize2<K>(raw, K, m);
  const bool on_n = (r.flags & REC_ON_NEUMANN) != 0;
  const double nx = r.nux, ny = r.nuy, px = r.nx, py = r.ny;
  const double target = r.target;
  if (target != 0.0) {
    double dv[OD];
#pragma unroll
    for (int j = 0; j < OD; ++j) dv[j] = 0.0;
    double v = mix_grad_one<K>(m, raw, nx, ny, dv);
    if (on_n && a.reflect) {
      double rx, ry;
      reflect(nx, ny, px, py, &rx, &ry);
      v += mix_grad_one<K>(m, raw, rx, ry, dv);
    }
    if (!(v > a.v_floor)) return false;
    double s = -target / (static_cast<double>(r.pdf_mis) * v);
#pragma unroll
    for (int j = 0; j < OD - 1; ++j) g[j] = s * dv[j];
  }
  if (a.learn_selection) {
    double pg = on_n ? (a.reflect ? reflected_pdf(m, nx, ny, px, py) : mixture_pdf(m, nx, ny))
                     : mixture_pdf(m, nx, ny);
    double pu = r.pdf_u;
    double pnow = m.c * pg + (1.0 - m.c) * pu;
    if (pnow > 0.0) {
      double dc = -a.e_fraction * target * (pg - pu) / (pnow * static_cast<double>(r.pdf_mis));
      g[OD - 1] = dc * m.c * (1.0 - m.c);
    }
  }
  bool fin = true;
#pragma unroll
  for (int j = 0; j < OD; ++j) {
    dy[j] = static_cast<float>(g[j] * a.inv_count);
    fin = fin && isfinite(dy[j]);
  }
  return fin;  // a gradient beyond fp32 range is dropped (counted as skipped)
}



// fp32 variant for the tensor-core training tile: same formulas, per-component
// math in fp32 with the vMF exponent formed as kappa (t - 1) + lne (Mix32) and
// I1/I0 by rational approximation; sampling-time quantities (target, pdf_mis,
// pdf_u) come from the record.
__device__ __forceinline__ float mix_grad_one32(const Mix32& m, const float* raw, const float* inv_mn,
                                                const bool* kap_free, const float* i10, float nx, float ny,
                                                float* g) {
  float v[8], t[8];
  float val = 0.0f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    t[i] = nx * m.mux[i] + ny * m.muy[i];
    v[i] = __expf(m.kappa[i] * (t[i] - 1.0f) + m.lne[i]);
    val += m.lambda[i] * v[i];
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float lv = m.lambda[i] * v[i];
    g[24 + i] += lv - m.lambda[i] * val;
    if (kap_free[i]) g[16 + i] += lv * (t[i] - i10[i]) * m.kappa[i];
    const float s = lv * m.kappa[i] * inv_mn[i];
    g[2 * i] += (nx - m.mux[i] * t[i]) * s;
    g[2 * i + 1] += (ny - m.muy[i] * t[i]) * s;
  }
  return val;
}

__device__ __forceinline__ bool record_dy32(const float* raw, const DevRecord& r, const TrainArgs& a,
                                            float* dy) {
  float g[33];
#pragma unroll
  for (int j = 0; j < 33; ++j) g[j] = 0.0f;
  Mix32 m;
  normalize32(raw, m);
  float inv_mn[8], i10[8];  // I1/I0(kappa) once per record (both directions share it)
  bool kap_free[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    i10[i] = i1_over_i0_f(m.kappa[i]);
    const float mx = raw[2 * i], my = raw[2 * i + 1];
    const float mn = sqrtf(mx * mx + my * my);
    inv_mn[i] = mn >= 1e-12f ? 1.0f / mn : 0.0f;  // zero-norm means get no mu gradient
    const float ku = __expf(raw[16 + i]);
    kap_free[i] = ku > static_cast<float>(kKappaMin) && ku < static_cast<float>(kKappaMax);
  }
  const bool on_n = (r.flags & REC_ON_NEUMANN) != 0;
  const float nx = r.nux, ny = r.nuy, px = r.nx, py = r.ny;
  const float target = r.target;
  if (target != 0.0f) {  // kl_grad, guide_train.cpp:25-42
    float dv[33];
#pragma unroll
    for (int j = 0; j < 33; ++j) dv[j] = 0.0f;
    // the direction and, on a Neumann record with reflection, its mirror
    // image: one copy of the (large) per-direction code, run once or twice
    // (the training tile's time is mostly instruction fetch; same sums in the
    // same order as two inline calls)
    float v = 0.0f;
    const int ndir = on_n && a.reflect ? 2 : 1;
    const float d = 2.0f * (nx * px + ny * py);
#pragma unroll 1
    for (int k = 0; k < ndir; ++k) {
      const float ux = k == 0 ? nx : nx - px * d, uy = k == 0 ? ny : ny - py * d;
      const float vk = mix_grad_one32(m, raw, inv_mn, kap_free, i10, ux, uy, dv);
      v = k == 0 ? vk : v + vk;
    }
    if (!(static_cast<double>(v) > a.v_floor)) return false;
    const float s = -target / (r.pdf_mis * v);
#pragma unroll
    for (int j = 0; j < 32; ++j) g[j] = s * dv[j];  // scaled by inv_count below
  }
  if (a.learn_selection) {  // selection_grad, guide_train.cpp:44-56
    double pg = on_n ? (a.reflect ? reflected_pdf32(m, nx, ny, px, py) : mixture_pdf32(m, nx, ny))
                     : mixture_pdf32(m, nx, ny);
    const double c = m.c, pu = r.pdf_u;
    const double pnow = c * pg + (1.0 - c) * pu;
    if (pnow > 0.0) {
      const double dc = -a.e_fraction * target * (pg - pu) / (pnow * static_cast<double>(r.pdf_mis));
      g[32] = static_cast<float>(dc * c * (1.0 - c));
    }
  }
  const float ic = static_cast<float>(a.inv_count);
  bool fin = true;
#pragma unroll
  for (int j = 0; j < 33; ++j) {
    dy[j] = g[j] * ic;
    fin = fin && isfinite(dy[j]);
  }
  return fin;  // a gradient beyond fp32 range is dropped (counted as skipped)
}

}  // namespace wg
