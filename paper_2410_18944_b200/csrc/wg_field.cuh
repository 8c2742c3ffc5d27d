// Guiding field on device: dense multi-resolution grid gather + 3-layer ReLU
// MLP (proj/src/guide_field.cpp). This header holds the CUDA-core "exact"
// evaluation, which reproduces GuidingField::eval's fp32 arithmetic bit for
// bit (same gather expression, same 4-way unrolled accumulation order, no FMA
// contraction). The tensor-core path lives in wg_mlp_tc.cuh.
#pragma once

#include "wg_device.cuh"

namespace wg {

struct FieldView {
  const float* p;  // all parameters (device global), GuidingField layout
  int32_t levels, F, in, hid, od, k, dim;
  int32_t res[WG_MAX_LEVELS];
  int32_t lvl_off[WG_MAX_LEVELS];
  int32_t w1, b1, w2, b2, w3, b3;  // absolute offsets into p
  int32_t mlp_count;               // w1 .. end
  double bbox[4];
};

// single-precision gather, guide_field.cpp:184-212
WG_D void field_gather(const FieldView& f, double x, double y, float* input) {
  double ex = f.bbox[2] - f.bbox[0], ey = f.bbox[3] - f.bbox[1];
  float u = static_cast<float>(sclamp((x - f.bbox[0]) / ex, 0.0, 1.0));
  float v = static_cast<float>(sclamp((y - f.bbox[1]) / ey, 0.0, 1.0));
  const int F = f.F;
  for (int l = 0; l < f.levels; ++l) {
    int res = f.res[l];
    float px = __fmul_rn(u, static_cast<float>(res - 1));
    float py = __fmul_rn(v, static_cast<float>(res - 1));
    int ix = imin(static_cast<int>(px), res - 2);
    int iy = imin(static_cast<int>(py), res - 2);
    float fx = __fsub_rn(px, static_cast<float>(ix));
    float fy = __fsub_rn(py, static_cast<float>(iy));
    const float* base = f.p + f.lvl_off[l] + (static_cast<size_t>(iy) * res + ix) * F;
    const float* up = base + static_cast<size_t>(res) * F;
    float w00 = __fmul_rn(__fsub_rn(1.0f, fx), __fsub_rn(1.0f, fy));
    float w10 = __fmul_rn(fx, __fsub_rn(1.0f, fy));
    float w01 = __fmul_rn(__fsub_rn(1.0f, fx), fy);
    float w11 = __fmul_rn(fx, fy);
    for (int i = 0; i < F; ++i) {
      float a = __fadd_rn(__fmul_rn(w00, __ldg(base + i)), __fmul_rn(w10, __ldg(base + F + i)));
      float b = __fadd_rn(__fmul_rn(w01, __ldg(up + i)), __fmul_rn(w11, __ldg(up + F + i)));
      input[l * F + i] = __fadd_rn(a, b);
    }
  }
}

// affine_forward_f (guide_field.cpp:149-170): y = b; rows in blocks of 4
// accumulated as (x0 w0 + x1 w1) + (x2 w2 + x3 w3); remainder rows singly.
template <int ROWS, int COLS>
WG_D void affine_exact(const float* x, int rows_rt, const float* w, const float* b, int cols_rt,
                       float* y, bool relu) {
  const int rows = ROWS ? ROWS : rows_rt;
  const int cols = COLS ? COLS : cols_rt;
#pragma unroll
  for (int j = 0; j < (COLS ? COLS : 256); ++j)
    if (j < cols) y[j] = b[j];
  int i = 0;
#pragma unroll 1
  for (; i + 4 <= rows; i += 4) {
    float x0 = x[i], x1 = x[i + 1], x2 = x[i + 2], x3 = x[i + 3];
    const float* w0 = w + static_cast<size_t>(i) * cols;
    const float* w1 = w0 + cols;
    const float* w2 = w1 + cols;
    const float* w3 = w2 + cols;
#pragma unroll
    for (int j = 0; j < (COLS ? COLS : 256); ++j) {
      if (j >= cols) break;
      float p = __fadd_rn(__fmul_rn(x0, w0[j]), __fmul_rn(x1, w1[j]));
      float q = __fadd_rn(__fmul_rn(x2, w2[j]), __fmul_rn(x3, w3[j]));
      y[j] = __fadd_rn(y[j], __fadd_rn(p, q));
    }
  }
#pragma unroll 1
  for (; i < rows; ++i) {
    float xi = x[i];
    const float* wr = w + static_cast<size_t>(i) * cols;
#pragma unroll
    for (int j = 0; j < (COLS ? COLS : 256); ++j) {
      if (j >= cols) break;
      y[j] = __fadd_rn(y[j], __fmul_rn(xi, wr[j]));
    }
  }
  if (relu) {
#pragma unroll
    for (int j = 0; j < (COLS ? COLS : 256); ++j)
      if (j < cols) y[j] = y[j] > 0.0f ? y[j] : 0.0f;
  }
}

// GuidingField::eval (guide_field.cpp:178-221). `mlp` points at the MLP block
// (w1..b3) — staged in shared memory by the caller — laid out as in params.
template <int IN, int HID, int OD>
WG_D void field_eval_exact(const FieldView& f, const float* mlp, double x, double y, float* out) {
  float input[IN ? IN : 256];
  float h1[HID ? HID : 256];
  float h2[HID ? HID : 256];
  field_gather(f, x, y, input);
  const int w1 = 0, b1 = f.b1 - f.w1, w2 = f.w2 - f.w1, b2 = f.b2 - f.w1, w3 = f.w3 - f.w1,
            b3 = f.b3 - f.w1;
  affine_exact<IN, HID>(input, f.in, mlp + w1, mlp + b1, f.hid, h1, true);
  affine_exact<HID, HID>(h1, f.hid, mlp + w2, mlp + b2, f.hid, h2, true);
  affine_exact<HID, OD>(h2, f.hid, mlp + w3, mlp + b3, f.od, out, false);
}

}  // namespace wg
