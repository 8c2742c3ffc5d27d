// Training tile on the 5th-generation tensor cores: forward, KL / selection
// loss gradient, backward and weight gradients for 128 records per tile
// (eval_with_tape + kl_grad + selection_grad + backward,
// proj/src/guide_field.cpp:223-315, proj/src/guide_train.cpp:25-56).
//
// One CTA = 128 threads = 128 records = one M = 128 UMMA tile; persistent over
// the minibatch's tiles. Per tile (all operands split fp16 hi/lo, three MMAs
// per K-block, fp32 accumulation in TMEM):
//   F1  H1 = relu(X W1 + b1)            A = X  (K-major)      -> TMEM c0
//   F2  H2 = relu(H1 W2 + b2)           A = H1                -> c64
//   F3  Y  = H2 W3 + b3                 A = H2                -> c128
//       dY = dL/dY per record (fp64 mixture / selection gradient, CUDA cores)
//   G3  dH2 = dY W3^T . [H2 > 0]        A = dY, B = W3        -> c0
//       dW3|db3 += [H2|1]^T dY          A = H2 tile read MN-major, B = dY MN-major -> cW3
//   G2  dH1 = dH2 W2^T . [H1 > 0]                             -> c64
//       dW2|db2 += [H1|1]^T dH2                               -> cW2
//   G1  dX  = dH1 W1^T                                        -> c128
//       dW1|db1 += [X|1]^T dH1                                -> cW1
// The activation tiles written K-major for the forward are read again,
// MN-major, as the A / B operands of the weight-gradient GEMMs (the UMMA
// descriptor only swaps LBO / SBO); a column of ones appended to X, H1 and H2
// makes row 16 / 64 of each weight-gradient product the bias gradient. Each
// tensor gets a tile-wide power-of-two scale (exact, undone in the epilogue)
// so the fp16 split keeps ~22 bits. Weight / bias gradients leave TMEM once per
// tile by atomics; dX goes to the grid corners by atomics. The split weight
// tiles arrive as the field's packed blob (wg_wpack.cuh) in one bulk copy.
#include "wg3_walk_common.cuh"
#include "wg_loss.cuh"
#include "wg_mlp_tc.cuh"
#include "wg_train.cuh"
#include "wg_wpack.cuh"

namespace wg {

namespace {

constexpr int TM = 128;
constexpr int KX = 24, KH = 72, KY = 48;  // padded K extents of X|1, H|1, dY
constexpr uint32_t AX = KX * TM * 2, AH = KH * TM * 2, AY = KY * TM * 2;
// shared-memory carve-up (bytes)
constexpr uint32_t S_XH = 0, S_XL = S_XH + AX;
constexpr uint32_t S_H1H = S_XL + AX, S_H1L = S_H1H + AH;  // H1, later dH1
constexpr uint32_t S_H2H = S_H1L + AH, S_H2L = S_H2H + AH;  // H2, later dH2
constexpr uint32_t S_YH = S_H2L + AH, S_YL = S_YH + AY;     // dY
// the field's packed weight blob (wg_wpack.cuh), one bulk copy
constexpr uint32_t S_W = S_YL + AY;
constexpr uint32_t S_B1H = S_W + wpack::B1H, S_B1L = S_W + wpack::B1L;  // forward weights
constexpr uint32_t S_B2H = S_W + wpack::B2H, S_B2L = S_W + wpack::B2L;
constexpr uint32_t S_B3H = S_W + wpack::B3H, S_B3L = S_W + wpack::B3L;
constexpr uint32_t S_BIAS = S_W + wpack::BIAS;                          // b1 64, b2 64, b3 48
constexpr uint32_t S_C3H = S_W + wpack::C3H, S_C3L = S_W + wpack::C3L;  // backward weights
constexpr uint32_t S_C2H = S_W + wpack::C2H, S_C2L = S_W + wpack::C2L;
constexpr uint32_t S_C1H = S_W + wpack::C1H, S_C1L = S_W + wpack::C1L;
constexpr uint32_t S_MAX = S_W + wpack::BYTES;  // 8 x u32 tile maxima
constexpr int STG = 65;                                    // staging row stride (floats)
constexpr uint32_t S_STAGE = S_MAX + 32;                   // 65 x 65 fp32 dW staging
constexpr uint32_t S_BAR = S_STAGE + (STG * STG * 4 + 15) / 16 * 16;  // mbarrier: 8-B aligned
constexpr uint32_t S_BAR_W = S_BAR + 8;                     // weight bulk-copy barrier
constexpr uint32_t S_TMEM = S_BAR_W + 8;
static_assert(S_W % 16 == 0, "bulk copy destination alignment");
constexpr uint32_t SMEM_BYTES = S_TMEM + 8;
static_assert(S_BAR % 8 == 0 && S_STAGE % 16 == 0, "shared-memory carve-up alignment");
// TMEM columns
constexpr uint32_t C0 = 0, C64 = 64, C128 = 128, CW3 = 192, CW2 = 256, CW1 = 320;

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | ((static_cast<uint64_t>(lbo >> 4) & 0x3FFFull) << 16) |
         ((static_cast<uint64_t>(sbo >> 4) & 0x3FFFull) << 32) | (1ull << 46);
}

// kind::f16, fp32 accumulate; a_mn / b_mn select MN-major operands
__device__ __forceinline__ uint32_t idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (static_cast<uint32_t>(a_mn) << 15) | (static_cast<uint32_t>(b_mn) << 16) |
         (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

// split fp16 store of K values into row `row` of a K-major tile (K multiple of 8)
template <int K>
__device__ __forceinline__ void put_row(unsigned char* sm, uint32_t hi_off, uint32_t lo_off, int row,
                                        const float* v) {
#pragma unroll
  for (int c = 0; c < K / 8; ++c) {
    __half2 hi[4], lo[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 x = make_float2(v[8 * c + 2 * i], v[8 * c + 2 * i + 1]);
      hi[i] = __float22half2_rn(x);
      float2 b = __half22float2(hi[i]);
      lo[i] = __float22half2_rn(make_float2(x.x - b.x, x.y - b.y));
    }
    uint32_t o = umma::kmajor_off(row, 8 * c, K);
    *reinterpret_cast<uint4*>(sm + hi_off + o) = *reinterpret_cast<uint4*>(hi);
    *reinterpret_cast<uint4*>(sm + lo_off + o) = *reinterpret_cast<uint4*>(lo);
  }
}

// tile-wide max |v| -> power-of-two scale bringing it to [2^9, 2^10)
__device__ __forceinline__ float tile_scale(unsigned char* sm, int slot, const float* v, int n,
                                            float& inv) {
  float m = 0.0f;
  for (int i = 0; i < n; ++i) m = fmaxf(m, fabsf(v[i]));
  // positive floats order like their bit patterns
  atomicMax(reinterpret_cast<unsigned*>(sm + S_MAX) + slot, __float_as_uint(m));
  __syncthreads();
  float tm = __uint_as_float(reinterpret_cast<volatile unsigned*>(sm + S_MAX)[slot]);
  int e = 0;
  frexpf(tm, &e);
  if (tm == 0.0f) e = 0;
  inv = ldexpf(1.0f, e - 10);
  return ldexpf(1.0f, 10 - e);
}

// one A x B^T product into TMEM: K/16 K-steps x 3 split terms
__device__ __forceinline__ void gemm(uint32_t tmem_d, uint32_t a_hi, uint32_t a_lo, uint32_t a_lbo,
                                     uint32_t a_sbo, uint32_t a_step, uint32_t b_hi, uint32_t b_lo,
                                     uint32_t b_lbo, uint32_t b_sbo, uint32_t b_step, int ksteps,
                                     uint32_t id, bool accumulate) {
  // issued by one thread: kept rolled (unrolled, the nine call sites were
  // ~1.6k instructions of a kernel whose time is mostly instruction fetch)
#pragma unroll 1
  for (int k = 0; k < ksteps; ++k) {
    uint64_t ah = desc(a_hi + k * a_step, a_lbo, a_sbo), al = desc(a_lo + k * a_step, a_lbo, a_sbo);
    uint64_t bh = desc(b_hi + k * b_step, b_lbo, b_sbo), bl = desc(b_lo + k * b_step, b_lbo, b_sbo);
    umma::mma_f16(tmem_d, ah, bh, id, (accumulate || k > 0) ? 1u : 0u);
    umma::mma_f16(tmem_d, al, bh, id, 1u);
    umma::mma_f16(tmem_d, ah, bl, id, 1u);
  }
}

__device__ __forceinline__ void wait_mma(unsigned char* sm, uint32_t& phase) {
  umma::mbar_wait(reinterpret_cast<uint64_t*>(sm + S_BAR), phase);
  phase ^= 1u;
  umma::fence_after();
}

__device__ __forceinline__ void publish_smem() {
  umma::fence_async_smem();
  umma::fence_before();
  __syncthreads();
}

template <int NC>
__device__ __forceinline__ void ld_row(uint32_t taddr, float* v) {
#pragma unroll
  for (int c = 0; c < NC / 16; ++c) {
    float a[16];
    umma::ld_x16(taddr + 16 * c, a);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[16 * c + i] = a[i];
  }
}

// weight-gradient rows leave TMEM through a shared-memory stage (row stride
// 65: conflict-free row writes) and then go out as flat, coalesced atomics:
// the nrow x ncol block is dense in the gradient vector at grad[w], the bias
// row (TMEM lane `bias_row`) dense at grad[b]. Only warps holding lanes of
// interest load TMEM (warp-uniform test: tcgen05.ld is warp-collective).
template <int NC>
__device__ __forceinline__ void flush_dw(unsigned char* sm, uint32_t trow, int row, int nrow, int bias_row,
                                         int ncol, float inv_w, float inv_b, float* grad, int w, int b) {
  float* st = reinterpret_cast<float*>(sm + S_STAGE);
  const int warp = threadIdx.x >> 5;
  if (warp * 32 <= bias_row) {
    float v[NC];
    ld_row<NC>(trow, v);
    if (row <= bias_row) {
      const float sc = row < nrow ? inv_w : inv_b;
      for (int j = 0; j < ncol; ++j) st[row * STG + j] = v[j] * sc;
    }
  }
  __syncthreads();
  const int nw = nrow * ncol;
  for (int e = threadIdx.x; e < nw; e += blockDim.x) {
    const int r = e / ncol;
    atomicAdd(grad + w + e, st[r * STG + (e - r * ncol)]);
  }
  for (int e = threadIdx.x; e < ncol; e += blockDim.x) atomicAdd(grad + b + e, st[bias_row * STG + e]);
}

// 16-byte vector reduction (the 4 features of one grid corner)
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

}  // namespace

// ---- the two field dimensions: gather / corner scatter / loss gradient
// (2D: bilinear 4 corners per level, 33 outputs, fp32 loss record_dy32;
// 3D: trilinear 8 corners per level, 41 outputs, fp64 loss record_dy3).
// The scatter recomputes the corners from the record's position instead of
// keeping them in registers through the tile.
struct Tc2 {
  using Args = TrainArgs;
  using Rec = DevRecord;
  static constexpr int OD = 33;
  __device__ static void gather(const FieldView& f, const Rec& r, float* x) {
    const double ex = f.bbox[2] - f.bbox[0], ey = f.bbox[3] - f.bbox[1];
    const float u = static_cast<float>(sclamp((static_cast<double>(r.x) - f.bbox[0]) / ex, 0.0, 1.0));
    const float v = static_cast<float>(sclamp((static_cast<double>(r.y) - f.bbox[1]) / ey, 0.0, 1.0));
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int res = f.res[l];
      const float px = u * static_cast<float>(res - 1), py = v * static_cast<float>(res - 1);
      const int ix = imin(static_cast<int>(px), res - 2), iy = imin(static_cast<int>(py), res - 2);
      const float fx = px - ix, fy = py - iy;
      const int c00 = f.lvl_off[l] + (iy * res + ix) * 4;
      const float w0 = (1.0f - fx) * (1.0f - fy), w1 = fx * (1.0f - fy), w2 = (1.0f - fx) * fy, w3 = fx * fy;
      const float4 e0 = __ldg(reinterpret_cast<const float4*>(f.p + c00));
      const float4 e1 = __ldg(reinterpret_cast<const float4*>(f.p + c00 + 4));
      const float4 e2 = __ldg(reinterpret_cast<const float4*>(f.p + c00 + res * 4));
      const float4 e3 = __ldg(reinterpret_cast<const float4*>(f.p + c00 + res * 4 + 4));
      x[4 * l + 0] = w0 * e0.x + w1 * e1.x + w2 * e2.x + w3 * e3.x;
      x[4 * l + 1] = w0 * e0.y + w1 * e1.y + w2 * e2.y + w3 * e3.y;
      x[4 * l + 2] = w0 * e0.z + w1 * e1.z + w2 * e2.z + w3 * e3.z;
      x[4 * l + 3] = w0 * e0.w + w1 * e1.w + w2 * e2.w + w3 * e3.w;
    }
  }
  __device__ static void scatter(const FieldView& f, const Rec& r, const float* dx, float sc, float* grad) {
    const double ex = f.bbox[2] - f.bbox[0], ey = f.bbox[3] - f.bbox[1];
    const float u = static_cast<float>(sclamp((static_cast<double>(r.x) - f.bbox[0]) / ex, 0.0, 1.0));
    const float v = static_cast<float>(sclamp((static_cast<double>(r.y) - f.bbox[1]) / ey, 0.0, 1.0));
#pragma unroll
    for (int l = 0; l < 4; ++l) {  // guide_field.cpp:305-314
      const int res = f.res[l];
      const float px = u * static_cast<float>(res - 1), py = v * static_cast<float>(res - 1);
      const int ix = imin(static_cast<int>(px), res - 2), iy = imin(static_cast<int>(py), res - 2);
      const float fx = px - ix, fy = py - iy;
      const int c00 = f.lvl_off[l] + (iy * res + ix) * 4;
      const int ci[4] = {c00, c00 + 4, c00 + res * 4, c00 + res * 4 + 4};
      const float wc[4] = {(1.0f - fx) * (1.0f - fy), fx * (1.0f - fy), (1.0f - fx) * fy, fx * fy};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float w = wc[c] * sc;
        red_add_v4(grad + ci[c], w * dx[4 * l], w * dx[4 * l + 1], w * dx[4 * l + 2], w * dx[4 * l + 3]);
      }
    }
  }
  __device__ static bool dy(const float* y, const Rec& r, const Args& a, float* d) {
    return record_dy32(y, r, a, d);
  }
};

struct Tc3 {
  using Args = TrainArgs3;
  using Rec = wg3::DevRecord3;
  static constexpr int OD = wg3::OD;  // 41
  __device__ static void cell(const wg3::Field3View& f, const Rec& r, float& u, float& v, float& q) {
    u = static_cast<float>(sclamp((static_cast<double>(r.x) - f.bbox[0]) * f.inv_ext[0], 0.0, 1.0));
    v = static_cast<float>(sclamp((static_cast<double>(r.y) - f.bbox[1]) * f.inv_ext[1], 0.0, 1.0));
    q = static_cast<float>(sclamp((static_cast<double>(r.z) - f.bbox[2]) * f.inv_ext[2], 0.0, 1.0));
  }
  __device__ static void gather(const wg3::Field3View& f, const Rec& r, float* x) {
    float u, v, q;
    cell(f, r, u, v, q);
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int res = f.res[l];
      const float rm = static_cast<float>(res - 1);
      const float px = u * rm, py = v * rm, pz = q * rm;
      const int ix = imin(static_cast<int>(px), res - 2), iy = imin(static_cast<int>(py), res - 2),
                iz = imin(static_cast<int>(pz), res - 2);
      const float fx = px - ix, fy = py - iy, fz = pz - iz, gx = 1.0f - fx, gy = 1.0f - fy, gz = 1.0f - fz;
      const int c0 = f.lvl_off[l] + ((iz * res + iy) * res + ix) * 4, sy = res * 4, sz = res * res * 4;
      const int ci[8] = {c0, c0 + 4, c0 + sy, c0 + sy + 4, c0 + sz, c0 + sz + 4, c0 + sz + sy, c0 + sz + sy + 4};
      const float w8[8] = {gx * gy * gz, fx * gy * gz, gx * fy * gz, fx * fy * gz,
                           gx * gy * fz, fx * gy * fz, gx * fy * fz, fx * fy * fz};
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 e = __ldg(reinterpret_cast<const float4*>(f.p + ci[c]));
        acc[0] = fmaf(w8[c], e.x, acc[0]);
        acc[1] = fmaf(w8[c], e.y, acc[1]);
        acc[2] = fmaf(w8[c], e.z, acc[2]);
        acc[3] = fmaf(w8[c], e.w, acc[3]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) x[4 * l + i] = acc[i];
    }
  }
  __device__ static void scatter(const wg3::Field3View& f, const Rec& r, const float* dx, float sc, float* grad) {
    float u, v, q;
    cell(f, r, u, v, q);
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int res = f.res[l];
      const float rm = static_cast<float>(res - 1);
      const float px = u * rm, py = v * rm, pz = q * rm;
      const int ix = imin(static_cast<int>(px), res - 2), iy = imin(static_cast<int>(py), res - 2),
                iz = imin(static_cast<int>(pz), res - 2);
      const float fx = px - ix, fy = py - iy, fz = pz - iz, gx = 1.0f - fx, gy = 1.0f - fy, gz = 1.0f - fz;
      const int c0 = f.lvl_off[l] + ((iz * res + iy) * res + ix) * 4, sy = res * 4, sz = res * res * 4;
      const int ci[8] = {c0, c0 + 4, c0 + sy, c0 + sy + 4, c0 + sz, c0 + sz + 4, c0 + sz + sy, c0 + sz + sy + 4};
      const float w8[8] = {gx * gy * gz, fx * gy * gz, gx * fy * gz, fx * fy * gz,
                           gx * gy * fz, fx * gy * fz, gx * fy * fz, fx * fy * fz};
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float w = w8[c] * sc;
        red_add_v4(grad + ci[c], w * dx[4 * l], w * dx[4 * l + 1], w * dx[4 * l + 2], w * dx[4 * l + 3]);
      }
    }
  }
  __device__ static bool dy(const float* y, const Rec& r, const Args& a, float* d) {
    const bool on_n = (r.flags & REC_ON_NEUMANN) != 0;
    return wg3::record_dy3<wg3::K8>(y, wg3::D3{r.nux, r.nuy, r.nuz}, wg3::D3{r.nx, r.ny, r.nz}, on_n, r.target,
                                    r.pdf_mis, r.pdf_u, a.reflect != 0, a.learn_selection != 0, a.e_fraction,
                                    a.v_floor, a.inv_count, d);
  }
};

template <class P>
__device__ __forceinline__ void grad_tc_body(const typename P::Args& a) {
  extern __shared__ __align__(128) unsigned char sm[];
  const auto& f = a.f;
  constexpr int OD = P::OD;
  static_assert(OD <= 48, "outputs fit the N = 48 tile");
  const int t = threadIdx.x, warp = t >> 5;
  const int64_t count = static_cast<int64_t>(min(*a.count, static_cast<unsigned long long>(a.list_cap)));
  const int64_t tiles = (count + TM - 1) / TM;
  if (static_cast<int64_t>(blockIdx.x) >= tiles) return;
  if (blockIdx.x == 0 && t == 0) a.grad[a.n_params] = static_cast<float>(count);

  // ---- split fp16 weight tiles + biases: one TMA bulk copy of the packed blob
  if (t == 0) {
    uint64_t* wb = reinterpret_cast<uint64_t*>(sm + S_BAR_W);
    umma::mbar_init(wb, 1);
    umma::fence_async_smem();
    umma::mbar_expect_tx(wb, wpack::BYTES);
    umma::bulk_g2s(sm + S_W, a.packed, wpack::BYTES, wb);
  }
  if (warp == 0) umma::tmem_alloc(reinterpret_cast<uint32_t*>(sm + S_TMEM), 512);
  if (t == 0) umma::mbar_init(reinterpret_cast<uint64_t*>(sm + S_BAR), 1);
  publish_smem();
  umma::fence_after();
  umma::mbar_wait(reinterpret_cast<uint64_t*>(sm + S_BAR_W), 0);  // weights landed
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sm + S_TMEM);
  const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  const uint32_t base = umma::smem_u32(sm);
  const float* bias = reinterpret_cast<const float*>(sm + S_BIAS);
  uint32_t phase = 0;
  unsigned consumed = 0, skipped = 0;

  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    if (t < 8) reinterpret_cast<unsigned*>(sm + S_MAX)[t] = 0u;
    __syncthreads();
    const int64_t ri = tile * TM + t;
    const bool live = ri < count;
    typename P::Rec r{};
    if (live) r = a.recs[a.list[ri]];
    // ---- gather (guide_field.cpp:80-123)
    float x[16];
    P::gather(f, r, x);
    if (!live)
      for (int i = 0; i < 16; ++i) x[i] = 0.0f;
    float inv_x, inv_h1, inv_h2, inv_dy, inv_d2, inv_d1;
    float row[KH];
    // ---- X | 1
    {
      float s = tile_scale(sm, 0, x, 16, inv_x);
#pragma unroll
      for (int i = 0; i < 16; ++i) row[i] = x[i] * s;
      row[16] = live ? 1.0f : 0.0f;
#pragma unroll
      for (int i = 17; i < KX; ++i) row[i] = 0.0f;
      put_row<KX>(sm, S_XH, S_XL, t, row);
    }
    publish_smem();
    if (t == 0) {  // F1: [128 x 24(16 used)] x W1 -> c0
      umma::fence_after();
      gemm(tmem + C0, base + S_XH, base + S_XL, 128, (KX / 8) * 128, 256, base + S_B1H, base + S_B1L,
           128, 256, 256, 1, idesc(128, 64, 0, 0), false);
      umma::commit(reinterpret_cast<uint64_t*>(sm + S_BAR));
    }
    wait_mma(sm, phase);
    uint64_t mask1 = 0, mask2 = 0;
    {
      float h[64];
      ld_row<64>(trow + C0, h);
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        float z = h[i] * inv_x + bias[i];
        h[i] = z > 0.0f ? z : 0.0f;
        if (z > 0.0f) mask1 |= 1ull << i;
      }
      float s = tile_scale(sm, 1, h, 64, inv_h1);
#pragma unroll
      for (int i = 0; i < 64; ++i) row[i] = h[i] * s;
      row[64] = live ? 1.0f : 0.0f;
#pragma unroll
      for (int i = 65; i < KH; ++i) row[i] = 0.0f;
      put_row<KH>(sm, S_H1H, S_H1L, t, row);
    }
    publish_smem();
    if (t == 0) {  // F2 -> c64
      umma::fence_after();
      gemm(tmem + C64, base + S_H1H, base + S_H1L, 128, (KH / 8) * 128, 256, base + S_B2H, base + S_B2L,
           128, 1024, 256, 4, idesc(128, 64, 0, 0), false);
      umma::commit(reinterpret_cast<uint64_t*>(sm + S_BAR));
    }
    wait_mma(sm, phase);
    {
      float h[64];
      ld_row<64>(trow + C64, h);
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        float z = h[i] * inv_h1 + bias[64 + i];
        h[i] = z > 0.0f ? z : 0.0f;
        if (z > 0.0f) mask2 |= 1ull << i;
      }
      float s = tile_scale(sm, 2, h, 64, inv_h2);
#pragma unroll
      for (int i = 0; i < 64; ++i) row[i] = h[i] * s;
      row[64] = live ? 1.0f : 0.0f;
#pragma unroll
      for (int i = 65; i < KH; ++i) row[i] = 0.0f;
      put_row<KH>(sm, S_H2H, S_H2L, t, row);
    }
    publish_smem();
    if (t == 0) {  // F3 -> c128 (N = 48)
      umma::fence_after();
      gemm(tmem + C128, base + S_H2H, base + S_H2L, 128, (KH / 8) * 128, 256, base + S_B3H, base + S_B3L,
           128, 1024, 256, 4, idesc(128, 48, 0, 0), false);
      umma::commit(reinterpret_cast<uint64_t*>(sm + S_BAR));
    }
    wait_mma(sm, phase);
    // ---- loss gradient at the raw outputs (fp64)
    {
      float y[48];
      ld_row<48>(trow + C128, y);
#pragma unroll
      for (int j = 0; j < OD; ++j) y[j] = y[j] * inv_h2 + bias[128 + j];
      float dy[OD];
      bool used = live && P::dy(y, r, a, dy);
      if (used) ++consumed;
      else if (live) ++skipped;
#pragma unroll
      for (int j = 0; j < 48; ++j) row[j] = (used && j < OD) ? dy[j] : 0.0f;
      float s = tile_scale(sm, 3, row, OD, inv_dy);
#pragma unroll
      for (int j = 0; j < 48; ++j) row[j] *= s;
      put_row<KY>(sm, S_YH, S_YL, t, row);
    }
    publish_smem();
    if (t == 0) {  // G3: dH2 -> c0 ; dW3 | db3 -> cW3
      umma::fence_after();
      gemm(tmem + C0, base + S_YH, base + S_YL, 128, (KY / 8) * 128, 256, base + S_C3H, base + S_C3L,
           128, (KY / 8) * 128, 256, 3, idesc(128, 64, 0, 0), false);
      gemm(tmem + CW3, base + S_H2H, base + S_H2L, (KH / 8) * 128, 128, 2 * (KH / 8) * 128,
           base + S_YH, base + S_YL, (KY / 8) * 128, 128, 2 * (KY / 8) * 128, 8,
           idesc(128, 48, 1, 1), false);
      umma::commit(reinterpret_cast<uint64_t*>(sm + S_BAR));
    }
    wait_mma(sm, phase);
    flush_dw<48>(sm, trow + CW3, t, 64, 64, OD, inv_h2 * inv_dy, inv_dy, a.grad, f.w3, f.b3);
    {
      float d[64];
      ld_row<64>(trow + C0, d);
#pragma unroll
      for (int i = 0; i < 64; ++i) d[i] = (mask2 >> i & 1ull) ? d[i] * inv_dy : 0.0f;
      float s = tile_scale(sm, 4, d, 64, inv_d2);
#pragma unroll
      for (int i = 0; i < 64; ++i) row[i] = d[i] * s;
#pragma unroll
      for (int i = 64; i < KH; ++i) row[i] = 0.0f;
      put_row<KH>(sm, S_H2H, S_H2L, t, row);  // dH2 replaces H2
    }
    publish_smem();
    if (t == 0) {  // G2: dH1 -> c64 ; dW2 | db2 -> cW2
      umma::fence_after();
      gemm(tmem + C64, base + S_H2H, base + S_H2L, 128, (KH / 8) * 128, 256, base + S_C2H, base + S_C2L,
           128, 1024, 256, 4, idesc(128, 64, 0, 0), false);
      gemm(tmem + CW2, base + S_H1H, base + S_H1L, (KH / 8) * 128, 128, 2 * (KH / 8) * 128,
           base + S_H2H, base + S_H2L, (KH / 8) * 128, 128, 2 * (KH / 8) * 128, 8,
           idesc(128, 64, 1, 1), false);
      umma::commit(reinterpret_cast<uint64_t*>(sm + S_BAR));
    }
    wait_mma(sm, phase);
    flush_dw<64>(sm, trow + CW2, t, 64, 64, 64, inv_h1 * inv_d2, inv_d2, a.grad, f.w2, f.b2);
    {
      float d[64];
      ld_row<64>(trow + C64, d);
#pragma unroll
      for (int i = 0; i < 64; ++i) d[i] = (mask1 >> i & 1ull) ? d[i] * inv_d2 : 0.0f;
      float s = tile_scale(sm, 5, d, 64, inv_d1);
#pragma unroll
      for (int i = 0; i < 64; ++i) row[i] = d[i] * s;
#pragma unroll
      for (int i = 64; i < KH; ++i) row[i] = 0.0f;
      put_row<KH>(sm, S_H1H, S_H1L, t, row);  // dH1 replaces H1
    }
    publish_smem();
    if (t == 0) {  // G1: dX -> c128 (N = 16) ; dW1 | db1 -> cW1
      umma::fence_after();
      gemm(tmem + C128, base + S_H1H, base + S_H1L, 128, (KH / 8) * 128, 256, base + S_C1H, base + S_C1L,
           128, 1024, 256, 4, idesc(128, 16, 0, 0), false);
      gemm(tmem + CW1, base + S_XH, base + S_XL, (KX / 8) * 128, 128, 2 * (KX / 8) * 128,
           base + S_H1H, base + S_H1L, (KH / 8) * 128, 128, 2 * (KH / 8) * 128, 8,
           idesc(128, 64, 1, 1), false);
      umma::commit(reinterpret_cast<uint64_t*>(sm + S_BAR));
    }
    wait_mma(sm, phase);
    flush_dw<64>(sm, trow + CW1, t, 16, 16, 64, inv_x * inv_d1, inv_d1, a.grad, f.w1, f.b1);
    {
      float dx[16];
      ld_row<16>(trow + C128, dx);
      if (live) P::scatter(f, r, dx, inv_d1, a.grad);  // grid corners (guide_field.cpp:305-314)
    }
    umma::fence_before();
    __syncthreads();  // TMEM / smem reuse by the next tile
  }
  unsigned c = consumed, sk = skipped;
  for (int o = 16; o > 0; o >>= 1) {
    c += __shfl_down_sync(0xffffffffu, c, o);
    sk += __shfl_down_sync(0xffffffffu, sk, o);
  }
  if ((t & 31) == 0) {
    if (c) atomicAdd(&a.totals->consumed, static_cast<unsigned long long>(c));
    if (sk) atomicAdd(&a.totals->skipped_v, static_cast<unsigned long long>(sk));
  }
  __syncthreads();
  if (warp == 0) {
    umma::fence_after();
    umma::tmem_dealloc(tmem, 512);
  }
}

// named kernels for profiles / launch lists
__global__ void __launch_bounds__(128, 1) grad_tc_kernel(TrainArgs a);
__global__ void __launch_bounds__(128, 1) grad3_tc_kernel(TrainArgs3 a);

bool tc_grad_available() { return true; }

template <class P, class Args>
cudaError_t launch_tc_tile(void (*k)(Args), const Args& a, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(SMEM_BYTES));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (a.packed == nullptr) return cudaErrorInvalidValue;
  int64_t tiles = (a.list_cap + TM - 1) / TM;
  int blocks = static_cast<int>(tiles < sms ? tiles : sms);
  k<<<blocks, TM, SMEM_BYTES, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_grad_tc(const TrainArgs& a, cudaStream_t st) { return launch_tc_tile<Tc2>(grad_tc_kernel, a, st); }

// the 3D minibatch gradient on the tensor cores (the tcgen05 counterpart of
// wg3_walk.cu's CUDA-core grad3_tile_kernel)
cudaError_t launch_grad3_tc(const TrainArgs3& a, cudaStream_t st) { return launch_tc_tile<Tc3>(grad3_tc_kernel, a, st); }

// the whole split-fp16 blob (forward + backward tiles, wg_wpack.cuh layout)
// of a 3D field: W3 has 41 outputs (zero padding to N = 48 from the memset)
__global__ void pack3_full_kernel(wg3::Field3View f, unsigned char* blob) {
  tc_stage_weights_raw(blob - TcLayout::B1_HI, f.p, f.w1, f.b1, f.w2, f.b2, f.w3, f.b3, wg3::OD);
  for (int e = threadIdx.x; e < 16 * 64; e += blockDim.x) {  // C1[k][n] = W1[k][n]
    const int k = e / 64, n = e % 64;
    wpack::put(blob, wpack::C1H, wpack::C1L, k, n, 64, f.p[f.w1 + e]);
  }
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
    const int k = e / 64, n = e % 64;
    wpack::put(blob, wpack::C2H, wpack::C2L, k, n, 64, f.p[f.w2 + e]);
  }
  for (int e = threadIdx.x; e < 64 * wg3::OD; e += blockDim.x) {
    const int k = e / wg3::OD, n = e % wg3::OD;
    wpack::put(blob, wpack::C3H, wpack::C3L, k, n, 48, f.p[f.w3 + e]);
  }
}

cudaError_t launch_pack3_full(const wg3::Field3View& f, unsigned char* blob, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(blob, 0, wpack::BYTES, st);
  if (e != cudaSuccess) return e;
  pack3_full_kernel<<<1, 256, 0, st>>>(f, blob);
  return cudaGetLastError();
}

size_t grad_tc_pack_bytes() { return wpack::BYTES; }

__global__ void __launch_bounds__(128, 1) grad_tc_kernel(TrainArgs a) { grad_tc_body<Tc2>(a); }
__global__ void __launch_bounds__(128, 1) grad3_tc_kernel(TrainArgs3 a) { grad_tc_body<Tc3>(a); }

}  // namespace wg
