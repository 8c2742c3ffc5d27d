// Per-record training loss gradient at the MLP outputs (fp64):
//   kl_grad (proj/src/guide_train.cpp:25-42) with mixture_grad(_reflected)
//   (proj/src/sphdist.cpp:324-381) and selection_grad (guide_train.cpp:44-56).
// Shared by the CUDA-core and the tcgen05 training tiles.
#pragma once

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
#pragma unroll
  for (int j = 0; j < OD; ++j) dy[j] = static_cast<float>(g[j] * a.inv_count);
  return true;
}


}  // namespace wg
