// 3D guiding field on device: dense D^3 x F grids per level, trilinear
// gather, then the same 3-layer ReLU MLP as the 2D field (no reference
// counterpart; 2D analogue proj/src/guide_field.cpp:80-123, 178-221). The
// exact evaluation keeps oracle/wost3d.inc Field3::eval's fp32 operation
// order (corner weights ((1-fx)(1-fy))(1-fz); corners summed as
// ((c000 + c100) + (c010 + c110)) + ((c001 + c101) + (c011 + c111))) and
// the 2D field's 4-way unrolled MLP accumulation (wg_field.cuh).
#pragma once

#include "wg_field.cuh"

namespace wg3 {

struct Field3View {
  const float* p;
  int32_t levels, F, in, hid, od, k;
  int32_t res[WG_MAX_LEVELS];
  int32_t lvl_off[WG_MAX_LEVELS];
  int32_t w1, b1, w2, b2, w3, b3;
  int32_t mlp_count;
  double bbox[6];
  double inv_ext[3];  // 1 / (bbox max - min) per axis (tensor-core gather)
};

__device__ __forceinline__ void field3_gather(const Field3View& f, double x, double y, double z,
                                              float* input) {
  float u = static_cast<float>(wg::sclamp((x - f.bbox[0]) / (f.bbox[3] - f.bbox[0]), 0.0, 1.0));
  float v = static_cast<float>(wg::sclamp((y - f.bbox[1]) / (f.bbox[4] - f.bbox[1]), 0.0, 1.0));
  float w = static_cast<float>(wg::sclamp((z - f.bbox[2]) / (f.bbox[5] - f.bbox[2]), 0.0, 1.0));
  const int F = f.F;
  for (int l = 0; l < f.levels; ++l) {
    const int res = f.res[l];
    const float rm = static_cast<float>(res - 1);
    float px = __fmul_rn(u, rm), py = __fmul_rn(v, rm), pz = __fmul_rn(w, rm);
    int ix = wg::imin(static_cast<int>(px), res - 2);
    int iy = wg::imin(static_cast<int>(py), res - 2);
    int iz = wg::imin(static_cast<int>(pz), res - 2);
    float fx = __fsub_rn(px, static_cast<float>(ix));
    float fy = __fsub_rn(py, static_cast<float>(iy));
    float fz = __fsub_rn(pz, static_cast<float>(iz));
    const size_t sy = static_cast<size_t>(res) * F, sz = static_cast<size_t>(res) * res * F;
    const float* c000 = f.p + f.lvl_off[l] + ((static_cast<size_t>(iz) * res + iy) * res + ix) * F;
    const float* c010 = c000 + sy;
    const float* c001 = c000 + sz;
    const float* c011 = c001 + sy;
    float gx = __fsub_rn(1.0f, fx), gy = __fsub_rn(1.0f, fy), gz = __fsub_rn(1.0f, fz);
    float w00 = __fmul_rn(gx, gy), w10 = __fmul_rn(fx, gy), w01 = __fmul_rn(gx, fy), w11 = __fmul_rn(fx, fy);
    float a000 = __fmul_rn(w00, gz), a100 = __fmul_rn(w10, gz), a010 = __fmul_rn(w01, gz),
          a110 = __fmul_rn(w11, gz);
    float a001 = __fmul_rn(w00, fz), a101 = __fmul_rn(w10, fz), a011 = __fmul_rn(w01, fz),
          a111 = __fmul_rn(w11, fz);
    for (int i = 0; i < F; ++i) {
      float lo = __fadd_rn(__fadd_rn(__fmul_rn(a000, __ldg(c000 + i)), __fmul_rn(a100, __ldg(c000 + F + i))),
                           __fadd_rn(__fmul_rn(a010, __ldg(c010 + i)), __fmul_rn(a110, __ldg(c010 + F + i))));
      float hi = __fadd_rn(__fadd_rn(__fmul_rn(a001, __ldg(c001 + i)), __fmul_rn(a101, __ldg(c001 + F + i))),
                           __fadd_rn(__fmul_rn(a011, __ldg(c011 + i)), __fmul_rn(a111, __ldg(c011 + F + i))));
      input[l * F + i] = __fadd_rn(lo, hi);
    }
  }
}

// Field3::eval: `mlp` is the w1..b3 block (shared memory staged by the caller)
template <int IN, int HID, int OD>
__device__ __forceinline__ void field3_eval_exact(const Field3View& f, const float* mlp, double x,
                                                  double y, double z, float* out) {
  float input[IN ? IN : 256];
  float h1[HID ? HID : 256];
  float h2[HID ? HID : 256];
  field3_gather(f, x, y, z, input);
  const int b1 = f.b1 - f.w1, w2 = f.w2 - f.w1, b2 = f.b2 - f.w1, w3 = f.w3 - f.w1, b3 = f.b3 - f.w1;
  wg::affine_exact<IN, HID>(input, f.in, mlp, mlp + b1, f.hid, h1, true);
  wg::affine_exact<HID, HID>(h1, f.hid, mlp + w2, mlp + b2, f.hid, h2, true);
  wg::affine_exact<HID, OD>(h2, f.hid, mlp + w3, mlp + b3, f.od, out, false);
}

}  // namespace wg3
