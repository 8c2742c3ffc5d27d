// Guiding-field MLP (16 -> 64 -> 64 -> 33, ReLU) on the 5th-generation
// tensor cores for one tile of 128 rows (one row per thread of a 128-thread
// CTA; thread t <-> TMEM lane t <-> MMA row t).
//
//   layer l:  D[tmem] = A_l (128 x K, smem) * B_l^T (N x K, smem), fp32 accum
//   A/B are fp32 values split into fp16 hi + lo; three MMAs per K-block
//   (hi*hi, lo*hi, hi*lo) give ~22 significant bits per product, so the
//   result tracks the fp32 reference MLP to ~1e-6 relative. Activations are
//   scaled by powers of two before the split (exact) to stay in fp16's
//   normal range; the epilogue undoes the scale, adds the bias and applies
//   ReLU, then writes the next layer's A tile. TMEM: 128 columns
//   (layer 1 -> cols 0-63, layer 2 -> 64-127, layer 3 -> 0-47).
#pragma once

#include "wg_field.cuh"
#include "wg_umma.cuh"
#include "wg_wpack.cuh"

namespace wg {

struct TcLayout {
  static constexpr int M = 128, NIN = 16, NH = 64, NO = 33, NO_PAD = 48;
  static constexpr uint32_t A_HI = 0;                      // 128 x 64 fp16
  static constexpr uint32_t A_LO = A_HI + M * NH * 2;      // 16 KB each
  static constexpr uint32_t B1_HI = A_LO + M * NH * 2;     // 64 x 16
  static constexpr uint32_t B1_LO = B1_HI + NH * NIN * 2;
  static constexpr uint32_t B2_HI = B1_LO + NH * NIN * 2;  // 64 x 64
  static constexpr uint32_t B2_LO = B2_HI + NH * NH * 2;
  static constexpr uint32_t B3_HI = B2_LO + NH * NH * 2;   // 48 x 64
  static constexpr uint32_t B3_LO = B3_HI + NO_PAD * NH * 2;
  static constexpr uint32_t BIAS = B3_LO + NO_PAD * NH * 2;  // 64 + 64 + 48 fp32
  static constexpr uint32_t BAR = BIAS + (NH + NH + NO_PAD) * 4;
  static constexpr uint32_t BAR_W = BAR + 8;  // weight bulk copy
  static constexpr uint32_t TMEM_SLOT = BAR + 16;
  static constexpr uint32_t BYTES = TMEM_SLOT + 8;
  static constexpr uint32_t TMEM_COLS = 128;
};
// [B1_HI, BAR) is byte-for-byte the forward prefix of the packed blob
static_assert(TcLayout::B1_HI % 16 == 0 && TcLayout::BAR - TcLayout::B1_HI == wpack::FWD_BYTES,
              "TcLayout weights must match the packed blob (wg_wpack.cuh)");

// Weights from the field's packed blob: one TMA bulk copy issued by thread 0;
// every thread waits with tc_wait_weights after the CTA barrier.
__device__ __forceinline__ void tc_fetch_weights(unsigned char* sm, const unsigned char* blob) {
  using L = TcLayout;
  if (threadIdx.x == 0) {
    uint64_t* wb = reinterpret_cast<uint64_t*>(sm + L::BAR_W);
    umma::mbar_init(wb, 1);
    umma::fence_async_smem();
    umma::mbar_expect_tx(wb, wpack::FWD_BYTES);
    umma::bulk_g2s(sm + L::B1_HI, blob, wpack::FWD_BYTES, wb);
  }
}
__device__ __forceinline__ void tc_wait_weights(unsigned char* sm) {
  umma::mbar_wait(reinterpret_cast<uint64_t*>(sm + TcLayout::BAR_W), 0);
}


// Stage B_l = W_l^T as split fp16 in the K-major layout, plus the biases,
// from fp32 parameters at absolute offsets (w1..b3) with `no` outputs
// (<= NO_PAD: 33 for the 2D field, 41 for the 3D one). Called by all threads
// of the CTA; caller syncs afterwards.
__device__ __forceinline__ void tc_stage_weights_raw(unsigned char* sm, const float* p, int w1, int b1,
                                                     int w2, int b2, int w3, int b3, int no) {
  using L = TcLayout;
  auto put = [&](uint32_t hi_off, uint32_t lo_off, int n, int k, int K, float v) {
    __half h, l;
    umma::split_f16(v, h, l);
    uint32_t o = umma::kmajor_off(n, k, K);
    *reinterpret_cast<__half*>(sm + hi_off + o) = h;
    *reinterpret_cast<__half*>(sm + lo_off + o) = l;
  };
  for (int e = threadIdx.x; e < L::NH * L::NIN; e += blockDim.x) {  // W1[k][n], k < 16
    int n = e % L::NH, k = e / L::NH;
    put(L::B1_HI, L::B1_LO, n, k, L::NIN, p[w1 + k * L::NH + n]);
  }
  for (int e = threadIdx.x; e < L::NH * L::NH; e += blockDim.x) {
    int n = e % L::NH, k = e / L::NH;
    put(L::B2_HI, L::B2_LO, n, k, L::NH, p[w2 + k * L::NH + n]);
  }
  for (int e = threadIdx.x; e < L::NO_PAD * L::NH; e += blockDim.x) {
    int n = e % L::NO_PAD, k = e / L::NO_PAD;
    put(L::B3_HI, L::B3_LO, n, k, L::NH, n < no ? p[w3 + k * no + n] : 0.0f);
  }
  float* bias = reinterpret_cast<float*>(sm + L::BIAS);
  for (int i = threadIdx.x; i < L::NH; i += blockDim.x) {
    bias[i] = p[b1 + i];
    bias[L::NH + i] = p[b2 + i];
  }
  for (int i = threadIdx.x; i < L::NO_PAD; i += blockDim.x) bias[2 * L::NH + i] = i < no ? p[b3 + i] : 0.0f;
  umma::fence_async_smem();
}
__device__ __forceinline__ void tc_stage_weights(unsigned char* sm, const FieldView& f) {
  tc_stage_weights_raw(sm, f.p, f.w1, f.b1, f.w2, f.b2, f.w3, f.b3, TcLayout::NO);
}

// One-time TMEM allocation (warp 0) and mbarrier init; caller syncs after.
__device__ __forceinline__ void tc_setup(unsigned char* sm) {
  using L = TcLayout;
  if (threadIdx.x < 32) umma::tmem_alloc(reinterpret_cast<uint32_t*>(sm + L::TMEM_SLOT), L::TMEM_COLS);
  if (threadIdx.x == 0) umma::mbar_init(reinterpret_cast<uint64_t*>(sm + L::BAR), 1);
}

__device__ __forceinline__ void tc_teardown(unsigned char* sm) {
  using L = TcLayout;
  __syncthreads();
  if (threadIdx.x < 32) {
    umma::fence_after();
    umma::tmem_dealloc(*reinterpret_cast<uint32_t*>(sm + L::TMEM_SLOT), L::TMEM_COLS);
  }
}

// Per-row power-of-two scale: brings the row's largest magnitude to [2^9, 2^10)
// so the fp16 hi/lo split keeps ~22 bits relative to the row; the MMA output
// row is multiplied back by `inv` in the epilogue (exact).
template <int K>
__device__ __forceinline__ void tc_row_scale(float* v, float& inv) {
  float m[8];  // tree max: 8 independent chains, then 3 levels
#pragma unroll
  for (int j = 0; j < 8; ++j) m[j] = fabsf(v[j]);
#pragma unroll
  for (int i = 8; i < K; ++i) m[i & 7] = fmaxf(m[i & 7], fabsf(v[i]));
#pragma unroll
  for (int w = 4; w > 0; w >>= 1)
#pragma unroll
    for (int j = 0; j < w; ++j) m[j] = fmaxf(m[j], m[j + w]);
  // frexp exponent e = eb - 126 of the max; s = 2^(10 - e), inv = 2^(e - 10),
  // built from the biased exponent eb (clamped so s and inv stay normal)
  int eb = (__float_as_int(m[0]) >> 23) & 0xff;
  eb = eb < 10 ? 10 : eb;
  const float s = __int_as_float((263 - eb) << 23);
  inv = __int_as_float((eb - 9) << 23);
#pragma unroll
  for (int i = 0; i < K; ++i) v[i] *= s;
}

// write this thread's A row: K values (already scaled), split hi/lo
template <int K>
__device__ __forceinline__ void tc_put_row(unsigned char* sm, int row, const float* v) {
  using L = TcLayout;
#pragma unroll
  for (int c = 0; c < K / 8; ++c) {
    __half2 hi[4], lo[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // packed F2FP conversions, two values at a time
      float2 x = make_float2(v[8 * c + 2 * i], v[8 * c + 2 * i + 1]);
      hi[i] = __float22half2_rn(x);
      float2 b = __half22float2(hi[i]);
      lo[i] = __float22half2_rn(make_float2(x.x - b.x, x.y - b.y));
    }
    uint32_t o = umma::kmajor_off(row, 8 * c, K);
    *reinterpret_cast<uint4*>(sm + L::A_HI + o) = *reinterpret_cast<uint4*>(hi);
    *reinterpret_cast<uint4*>(sm + L::A_LO + o) = *reinterpret_cast<uint4*>(lo);
  }
}

// issue one layer (thread 0 only): K/16 K-blocks x 3 split terms
template <int K, int N>
__device__ __forceinline__ void tc_issue(unsigned char* sm, uint32_t tmem_d, uint32_t b_hi,
                                         uint32_t b_lo) {
  using L = TcLayout;
  const uint32_t base = umma::smem_u32(sm);
  constexpr uint32_t idesc = umma::idesc_f16(L::M, N);
#pragma unroll
  for (int kb = 0; kb < K / 16; ++kb) {
    const uint32_t ko = kb * 256;
    uint64_t ahi = umma::desc_kmajor(base + L::A_HI + ko, K);
    uint64_t alo = umma::desc_kmajor(base + L::A_LO + ko, K);
    uint64_t bhi = umma::desc_kmajor(base + b_hi + ko, K);
    uint64_t blo = umma::desc_kmajor(base + b_lo + ko, K);
    umma::mma_f16(tmem_d, ahi, bhi, idesc, kb > 0 ? 1u : 0u);
    umma::mma_f16(tmem_d, alo, bhi, idesc, 1u);
    umma::mma_f16(tmem_d, ahi, blo, idesc, 1u);
  }
  umma::commit(reinterpret_cast<uint64_t*>(sm + L::BAR));
}

// Bilinear multi-resolution gather (guide_field.cpp:80-123) for the default
// shape (4 levels x 4 features): one 16-byte load per lattice corner.
__device__ __forceinline__ void tc_gather(const FieldView& f, double x, double y, float* in) {
  double ex = f.bbox[2] - f.bbox[0], ey = f.bbox[3] - f.bbox[1];
  float u = static_cast<float>(sclamp((x - f.bbox[0]) / ex, 0.0, 1.0));
  float v = static_cast<float>(sclamp((y - f.bbox[1]) / ey, 0.0, 1.0));
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const int res = f.res[l];
    float px = u * static_cast<float>(res - 1), py = v * static_cast<float>(res - 1);
    int ix = imin(static_cast<int>(px), res - 2), iy = imin(static_cast<int>(py), res - 2);
    float fx = px - ix, fy = py - iy;
    const float4* base = reinterpret_cast<const float4*>(f.p + f.lvl_off[l] + (iy * res + ix) * 4);
    float4 a = __ldg(base), b = __ldg(base + 1), c = __ldg(base + res), d = __ldg(base + res + 1);
    float w00 = (1.0f - fx) * (1.0f - fy), w10 = fx * (1.0f - fy);
    float w01 = (1.0f - fx) * fy, w11 = fx * fy;
    in[4 * l + 0] = (w00 * a.x + w10 * b.x) + (w01 * c.x + w11 * d.x);
    in[4 * l + 1] = (w00 * a.y + w10 * b.y) + (w01 * c.y + w11 * d.y);
    in[4 * l + 2] = (w00 * a.z + w10 * b.z) + (w01 * c.z + w11 * d.z);
    in[4 * l + 3] = (w00 * a.w + w10 * b.w) + (w01 * c.w + w11 * d.w);
  }
}

// Forward pass of the whole 128-row tile. Every thread of the CTA calls it
// with its row's 16 inputs (zeros for idle rows); out[0..NO) = raw outputs
// (NO = 33 for the 2D field, 41 for the 3D one; both fit the N = 48 layer).
template <int NO = TcLayout::NO>
__device__ __forceinline__ void tc_forward(unsigned char* sm, uint32_t& phase, const float* x,
                                           float* out, long long* bp = nullptr) {
  static_assert(NO <= TcLayout::NO_PAD, "output width exceeds the padded layer");
  long long* mma_cyc = bp;
  long long tq = bp ? clock64() : 0;
  using L = TcLayout;
  const int row = threadIdx.x;
  const int warp = threadIdx.x >> 5;
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sm + L::TMEM_SLOT);
  const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  const float* bias = reinterpret_cast<const float*>(sm + L::BIAS);
  float v[L::NH];
  float inv;
  // ---- layer 1
#pragma unroll
  for (int i = 0; i < L::NIN; ++i) v[i] = x[i];
  tc_row_scale<L::NIN>(v, inv);
  tc_put_row<L::NIN>(sm, row, v);
  umma::fence_async_smem();
  umma::fence_before();
  __syncthreads();
  if (bp) bp[1] += clock64() - tq;
  long long t0_634 = mma_cyc ? clock64() : 0;
  if (threadIdx.x == 0) {
    umma::fence_after();
    tc_issue<L::NIN, L::NH>(sm, tmem + 0, L::B1_HI, L::B1_LO);
  }
  umma::mbar_wait(bar, phase);
  phase ^= 1u;
  umma::fence_after();
  if (bp) tq = clock64();
  if (mma_cyc) *mma_cyc += clock64() - t0_634;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float a[32];
    umma::ld_x32(trow + 32 * c, a);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      float h = a[i] * inv + bias[32 * c + i];
      v[32 * c + i] = h > 0.0f ? h : 0.0f;
    }
  }
  tc_row_scale<L::NH>(v, inv);
  tc_put_row<L::NH>(sm, row, v);
  umma::fence_async_smem();
  umma::fence_before();
  __syncthreads();
  // ---- layer 2
  if (bp) bp[1] += clock64() - tq;
  long long t0_178 = mma_cyc ? clock64() : 0;
  if (threadIdx.x == 0) {
    umma::fence_after();
    tc_issue<L::NH, L::NH>(sm, tmem + 64, L::B2_HI, L::B2_LO);
  }
  umma::mbar_wait(bar, phase);
  phase ^= 1u;
  umma::fence_after();
  if (bp) tq = clock64();
  if (mma_cyc) *mma_cyc += clock64() - t0_178;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float a[32];
    umma::ld_x32(trow + 64 + 32 * c, a);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      float h = a[i] * inv + bias[L::NH + 32 * c + i];
      v[32 * c + i] = h > 0.0f ? h : 0.0f;
    }
  }
  tc_row_scale<L::NH>(v, inv);
  tc_put_row<L::NH>(sm, row, v);
  umma::fence_async_smem();
  umma::fence_before();
  __syncthreads();
  // ---- layer 3
  if (bp) bp[1] += clock64() - tq;
  long long t0_92 = mma_cyc ? clock64() : 0;
  if (threadIdx.x == 0) {
    umma::fence_after();
    tc_issue<L::NH, L::NO_PAD>(sm, tmem + 0, L::B3_HI, L::B3_LO);
  }
  umma::mbar_wait(bar, phase);
  phase ^= 1u;
  umma::fence_after();
  if (bp) tq = clock64();
  if (mma_cyc) *mma_cyc += clock64() - t0_92;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float a[16];
    umma::ld_x16(trow + 16 * c, a);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      int j = 16 * c + i;
      if (j < NO) out[j] = a[i] * inv + bias[2 * L::NH + j];
    }
  }
  // TMEM columns are rewritten by the next tile's MMAs: order these loads first
  umma::fence_before();
}

}  // namespace wg
