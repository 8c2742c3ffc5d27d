// Online training of the guiding field on device (proj/src/guide_train.cpp).
//
//   compact_kernel usable records (pdf_mis >= floor) thinned by their
//                  deterministic key to a random subset of expected size
//                  min(n, cap), split into random minibatches (guide_train.cpp:101-130)
//   grad kernel    one CTA per 128-record tile: gather + MLP forward, per-record
//                  KL / selection gradient (Eq. 13 / 16) in fp64, backward, and
//                  the tile's weight gradients reduced in shared memory; grid
//                  corners receive their share by atomics (wg_train_tc.cu holds
//                  the tcgen05 version of the three GEMMs)
//   adam_kernel    bias-corrected Adam with fp64 moments (guide_field.cpp:317-331)
#include <algorithm>

#include "wg_kernels.cuh"
#include "wg_sphdist.cuh"
#include "wg_train.cuh"
#include "wg_loss.cuh"
#include "wg_wpack.cuh"

namespace wg {

// ---------------------------------------------------------------- selection
// Training set of a round (train_batch, guide_train.cpp:101-130): usable
// records (valid, pdf_mis >= floor) are thinned with probability
// p = min(1, cap / usable) by their deterministic 64-bit key (a uniform
// u = key / 2^64) and assigned to minibatch floor(u / p * n_mb); i.e. a
// uniformly random subset of expected size min(usable, cap) in random
// minibatches, without a sort. Device-only: the host never waits.
// `usable` is the GLOBAL count (summed over the ranks before this launch)
// and keys depend only on (seed, round, global point, depth), so the union
// of the ranks' selections is exactly the single-GPU selection: the cap and
// the minibatch size are global, as in the reference's one-process loop.
__global__ void compact_kernel(const DevRecord* recs, const unsigned long long* rec_count,
                               int64_t capacity, TrainCtl* ctl, TrainTotals* totals,
                               uint32_t* lists, int64_t list_cap, int64_t max_records,
                               int32_t minibatch) {
  const int64_t n = static_cast<int64_t>(min(*rec_count, static_cast<unsigned long long>(capacity)));
  const double usable = static_cast<double>(ctl->usable_global);
  const double take = fmin(usable, static_cast<double>(max_records));
  const int n_mb = take > 0.0 ? min(kMaxMinibatches, static_cast<int>(ceil(take / minibatch))) : 0;
  const double p = usable > 0.0 ? fmin(1.0, static_cast<double>(max_records) / usable) : 0.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    atomicAdd(&totals->seen, ctl->seen);
    atomicAdd(&totals->low_pdf, ctl->low_pdf);
  }
  // warp-strided so every lane of a warp takes part in the aggregated slot
  // allocation; each record contributes one 8-B (walk, flags) and one 8-B key load
  const int lane = threadIdx.x & 31;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + (threadIdx.x & ~31); i0 < n; i0 += stride) {
    const int64_t i = i0 + lane;
    bool sel = false;
    int mb = 0;
    if (i < n && n_mb > 0) {
      const char* rp = reinterpret_cast<const char*>(recs + i);
      const uint32_t flags = reinterpret_cast<const uint2*>(rp + 56)->y;
      if ((flags & (REC_VALID | REC_USABLE)) == (REC_VALID | REC_USABLE)) {
        const uint64_t key = *reinterpret_cast<const uint64_t*>(rp + 64);
        const double u = static_cast<double>(key >> 11) * 0x1.0p-53;
        if (u < p) {
          sel = true;
          mb = static_cast<int>(u / p * n_mb);
          mb = mb < n_mb - 1 ? mb : n_mb - 1;
        }
      }
    }
    const unsigned act = __ballot_sync(0xffffffffu, sel);
    if (!sel) continue;
    // one atomic per (warp, minibatch): lanes with the same minibatch share it
    const unsigned peers = __match_any_sync(act, mb);
    const int leader = __ffs(peers) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(&ctl->mb_count[mb], static_cast<unsigned long long>(__popc(peers)));
    base = __shfl_sync(peers, base, leader);
    const unsigned long long slot = base + __popc(peers & ((1u << lane) - 1u));
    if (static_cast<int64_t>(slot) < list_cap) lists[mb * list_cap + static_cast<int64_t>(slot)] = static_cast<uint32_t>(i);
    else atomicAdd(&totals->overflow, 1ull);
  }
}

cudaError_t launch_compact(const DevRecord* recs, const unsigned long long* rec_count,
                           int64_t capacity, TrainCtl* ctl, TrainTotals* totals, uint32_t* lists,
                           int64_t list_cap, int64_t max_records, int32_t minibatch,
                           cudaStream_t st) {
  compact_kernel<<<148 * 4, 256, 0, st>>>(recs, rec_count, capacity, ctl, totals, lists, list_cap,
                                         max_records, minibatch);
  return cudaGetLastError();
}

// Finalise a round's records: validity (the reference only backfills
// non-escaped walks, wost.cpp:373-383), usable / low-pdf counts for the
// selection, and - for scenes without source or Neumann terms, where every
// dacc is 0 - the target |S_K / Q_k| directly (see DevRecord). Scenes with
// local terms take their targets from backfill_chains_kernel instead.
// Imported records (walk < 0) keep their target. Grid-stride over the
// device-side record count.
__global__ void finalize_records_kernel(DevRecord* recs, const unsigned long long* rec_count,
                                        int64_t capacity, const double* term, const int32_t* esc,
                                        double pdf_floor, TrainCtl* ctl, bool chain) {
  const int64_t n = static_cast<int64_t>(min(*rec_count, static_cast<unsigned long long>(capacity)));
  unsigned usable = 0, low = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    DevRecord& r = recs[i];
    uint32_t fl = r.flags;
    if (!(fl & REC_WRITTEN)) continue;  // unused slot of a lane's chunk
    fl &= REC_WRITTEN | REC_ON_NEUMANN;
    if (r.walk >= 0) {
      if (esc[r.walk]) {
        r.flags = fl;  // not valid
        continue;
      }
      if (!chain) {
        const double q = r.thr_q;
        r.target = q == 0.0 ? 0.0f : static_cast<float>(fabs(term[r.walk] / q));
      }
    }
    fl |= REC_VALID;
    if (static_cast<double>(r.pdf_mis) < pdf_floor) {
      ++low;
    } else {
      ++usable;
      fl |= REC_USABLE;
    }
    r.flags = fl;
  }
  for (int o = 16; o > 0; o >>= 1) {
    usable += __shfl_down_sync(0xffffffffu, usable, o);
    low += __shfl_down_sync(0xffffffffu, low, o);
  }
  if ((threadIdx.x & 31) == 0 && (usable | low)) {
    atomicAdd(&ctl->usable, static_cast<unsigned long long>(usable));
    atomicAdd(&ctl->low_pdf, static_cast<unsigned long long>(low));
    atomicAdd(&ctl->seen, static_cast<unsigned long long>(usable + low));
  }
}

// backfill_targets_append (guide_train.cpp:58-79) for scenes with source /
// Neumann terms: one thread per walk follows its record chain from the last
// record backwards with the suffix sum S in fp64 (target_k = |S_{k+1} / Q_k|,
// then S += dacc_k), like the reference's backward recursion.
__global__ void backfill_chains_kernel(DevRecord* recs, int64_t n_walks, const int32_t* tail,
                                       const double* term, const int32_t* esc) {
  for (int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < n_walks;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (esc[w]) continue;
    double s = term[w];
    for (int32_t i = tail[w]; i >= 0;) {
      DevRecord& r = recs[i];
      const double q = r.thr_q;
      r.target = q == 0.0 ? 0.0f : static_cast<float>(fabs(s / q));
      s += static_cast<double>(r.dacc);
      i = r.prev;
    }
  }
}

cudaError_t launch_finalize_records(DevRecord* recs, const unsigned long long* rec_count,
                                    int64_t capacity, int64_t n_walks, const int32_t* tail,
                                    const double* term, const int32_t* esc, double pdf_floor,
                                    TrainCtl* ctl, bool chain, cudaStream_t st) {
  if (chain) {
    const int blocks = static_cast<int>(std::min<int64_t>((n_walks + 127) / 128, 148 * 8));
    backfill_chains_kernel<<<std::max(blocks, 1), 128, 0, st>>>(recs, n_walks, tail, term, esc);
  }
  finalize_records_kernel<<<148 * 4, 256, 0, st>>>(recs, rec_count, capacity, term, esc, pdf_floor, ctl,
                                                   chain);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- tile kernel
// CUDA-core tile: 128 records per CTA, thread = record. Activations and the
// backward signals live in padded shared-memory tiles (row stride +1 float)
// so row-per-thread writes and column-per-thread reads are conflict-free.
namespace {
constexpr int TB = 128;
constexpr int IN = 16, HID = 64, K8 = 8, OD = 33;
constexpr int SX = IN + 1, SH = HID + 1, SY = OD + 1;
constexpr int MLPN = IN * HID + HID + HID * HID + HID + HID * OD + OD;  // 7393
constexpr size_t TILE_SMEM =
    sizeof(float) * (MLPN + TB * SX + 4 * TB * SH + TB * SY);
}  // namespace

__global__ void __launch_bounds__(TB) grad_tile_kernel(TrainArgs a) {
  extern __shared__ __align__(16) float sm[];
  float* W = sm;                    // MLP block, params layout
  float* X = W + MLPN;              // [TB][SX]
  float* H1 = X + TB * SX;          // [TB][SH] post-ReLU
  float* H2 = H1 + TB * SH;
  float* D2 = H2 + TB * SH;         // dL/dh2pre
  float* D1 = D2 + TB * SH;         // dL/dh1pre
  float* DY = D1 + TB * SH;         // [TB][SY]
  const FieldView& f = a.f;
  for (int i = threadIdx.x; i < MLPN; i += TB) W[i] = f.p[f.w1 + i];
  const float* W1 = W;
  const float* B1 = W1 + IN * HID;
  const float* W2 = B1 + HID;
  const float* B2 = W2 + HID * HID;
  const float* W3 = B2 + HID;
  const float* B3 = W3 + HID * OD;
  __syncthreads();

  const int t = threadIdx.x;
  const int64_t ri = static_cast<int64_t>(blockIdx.x) * TB + t;
  const int64_t count = static_cast<int64_t>(min(*a.count, static_cast<unsigned long long>(a.list_cap)));
  if (static_cast<int64_t>(blockIdx.x) * TB >= count) return;
  if (blockIdx.x == 0 && t == 0) a.grad[a.n_params] = static_cast<float>(count);
  const bool live = ri < count;
  DevRecord r{};
  if (live) r = a.recs[a.list[ri]];

  // gather (fp32, guide_field.cpp:80-123) keeping corner indices/weights
  float x[IN];
  int cidx[4 * 4];
  float cw[4 * 4];
  {
    double ex = f.bbox[2] - f.bbox[0], ey = f.bbox[3] - f.bbox[1];
    float u = static_cast<float>(sclamp((static_cast<double>(r.x) - f.bbox[0]) / ex, 0.0, 1.0));
    float v = static_cast<float>(sclamp((static_cast<double>(r.y) - f.bbox[1]) / ey, 0.0, 1.0));
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      int res = f.res[l];
      float px = u * static_cast<float>(res - 1), py = v * static_cast<float>(res - 1);
      int ix = imin(static_cast<int>(px), res - 2), iy = imin(static_cast<int>(py), res - 2);
      float fx = px - ix, fy = py - iy;
      int c00 = f.lvl_off[l] + (iy * res + ix) * 4;
      int c10 = c00 + 4, c01 = c00 + res * 4, c11 = c01 + 4;
      float w00 = (1.0f - fx) * (1.0f - fy), w10 = fx * (1.0f - fy);
      float w01 = (1.0f - fx) * fy, w11 = fx * fy;
      cidx[4 * l] = c00;
      cidx[4 * l + 1] = c10;
      cidx[4 * l + 2] = c01;
      cidx[4 * l + 3] = c11;
      cw[4 * l] = w00;
      cw[4 * l + 1] = w10;
      cw[4 * l + 2] = w01;
      cw[4 * l + 3] = w11;
      float4 e00 = __ldg(reinterpret_cast<const float4*>(f.p + c00));
      float4 e10 = __ldg(reinterpret_cast<const float4*>(f.p + c10));
      float4 e01 = __ldg(reinterpret_cast<const float4*>(f.p + c01));
      float4 e11 = __ldg(reinterpret_cast<const float4*>(f.p + c11));
      x[4 * l + 0] = w00 * e00.x + w10 * e10.x + w01 * e01.x + w11 * e11.x;
      x[4 * l + 1] = w00 * e00.y + w10 * e10.y + w01 * e01.y + w11 * e11.y;
      x[4 * l + 2] = w00 * e00.z + w10 * e10.z + w01 * e01.z + w11 * e11.z;
      x[4 * l + 3] = w00 * e00.w + w10 * e10.w + w01 * e01.w + w11 * e11.w;
    }
  }
  // forward; activations go straight to the thread's smem row
  float* xr = X + t * SX;
  float* h1r = H1 + t * SH;
  float* h2r = H2 + t * SH;
#pragma unroll
  for (int i = 0; i < IN; ++i) xr[i] = x[i];
  float y[OD];
  {
    float h[HID];
#pragma unroll
    for (int j = 0; j < HID; ++j) {
      float acc = B1[j];
#pragma unroll
      for (int i = 0; i < IN; ++i) acc = fmaf(x[i], W1[i * HID + j], acc);
      h[j] = acc > 0.0f ? acc : 0.0f;
      h1r[j] = h[j];
    }
#pragma unroll 4
    for (int j = 0; j < HID; ++j) {
      float acc = B2[j];
#pragma unroll
      for (int i = 0; i < HID; ++i) acc = fmaf(h[i], W2[i * HID + j], acc);
      h2r[j] = acc > 0.0f ? acc : 0.0f;
    }
#pragma unroll
    for (int i = 0; i < HID; ++i) h[i] = h2r[i];
#pragma unroll
    for (int j = 0; j < OD; ++j) {
      float acc = B3[j];
#pragma unroll
      for (int i = 0; i < HID; ++i) acc = fmaf(h[i], W3[i * OD + j], acc);
      y[j] = acc;
    }
  }
  // loss gradient at the raw outputs
  float dy[OD];
  bool used = false;
  if (live) used = record_dy<K8>(y, r, a, dy);
  if (!used) {
#pragma unroll
    for (int j = 0; j < OD; ++j) dy[j] = 0.0f;
  }
  {
    unsigned c = __popc(__ballot_sync(0xffffffffu, used));
    unsigned sk = __popc(__ballot_sync(0xffffffffu, live && !used));
    if ((t & 31) == 0) {
      if (c) atomicAdd(&a.totals->consumed, c);
      if (sk) atomicAdd(&a.totals->skipped_v, sk);
    }
  }
  // backward through the layers (guide_field.cpp:258-303), row in smem
  float* d2r = D2 + t * SH;
  float* d1r = D1 + t * SH;
  float* dyr = DY + t * SY;
#pragma unroll
  for (int j = 0; j < OD; ++j) dyr[j] = dy[j];
#pragma unroll 4
  for (int i = 0; i < HID; ++i) {
    float acc = 0.0f;
#pragma unroll
    for (int j = 0; j < OD; ++j) acc = fmaf(W3[i * OD + j], dy[j], acc);
    d2r[i] = h2r[i] > 0.0f ? acc : 0.0f;
  }
  float dx[IN];
  {
    float dv[HID];
#pragma unroll
    for (int j = 0; j < HID; ++j) dv[j] = d2r[j];
#pragma unroll 4
    for (int i = 0; i < HID; ++i) {
      float acc = 0.0f;
#pragma unroll
      for (int j = 0; j < HID; ++j) acc = fmaf(W2[i * HID + j], dv[j], acc);
      d1r[i] = h1r[i] > 0.0f ? acc : 0.0f;
    }
#pragma unroll
    for (int j = 0; j < HID; ++j) dv[j] = d1r[j];
#pragma unroll
    for (int i = 0; i < IN; ++i) {
      float acc = 0.0f;
#pragma unroll
      for (int j = 0; j < HID; ++j) acc = fmaf(W1[i * HID + j], dv[j], acc);
      dx[i] = acc;
    }
  }
  // grid corners (guide_field.cpp:305-314)
  if (used) {
#pragma unroll
    for (int l = 0; l < 4; ++l)
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int q = 0; q < 4; ++q) atomicAdd(a.grad + cidx[4 * l + c] + q, cw[4 * l + c] * dx[4 * l + q]);
  }
  __syncthreads();
  // dW3 = H2^T DY, dW2 = H1^T D2, dW1 = X^T D1, biases = column sums
  const int gw1 = f.w1, gb1 = f.b1, gw2 = f.w2, gb2 = f.b2, gw3 = f.w3, gb3 = f.b3;
  for (int e = t; e < HID * OD; e += TB) {
    int i = e / OD, j = e % OD;
    float acc = 0.0f;
    for (int q = 0; q < TB; ++q) acc = fmaf(H2[q * SH + i], DY[q * SY + j], acc);
    atomicAdd(a.grad + gw3 + e, acc);
  }
  for (int e = t; e < HID * HID; e += TB) {
    int i = e / HID, j = e % HID;
    float acc = 0.0f;
    for (int q = 0; q < TB; ++q) acc = fmaf(H1[q * SH + i], D2[q * SH + j], acc);
    atomicAdd(a.grad + gw2 + e, acc);
  }
  for (int e = t; e < IN * HID; e += TB) {
    int i = e / HID, j = e % HID;
    float acc = 0.0f;
    for (int q = 0; q < TB; ++q) acc = fmaf(X[q * SX + i], D1[q * SH + j], acc);
    atomicAdd(a.grad + gw1 + e, acc);
  }
  if (t < OD) {
    float acc = 0.0f;
    for (int q = 0; q < TB; ++q) acc += DY[q * SY + t];
    atomicAdd(a.grad + gb3 + t, acc);
  }
  if (t < HID) {
    float a1 = 0.0f, a2 = 0.0f;
    for (int q = 0; q < TB; ++q) {
      a1 += D1[q * SH + t];
      a2 += D2[q * SH + t];
    }
    atomicAdd(a.grad + gb1 + t, a1);
    atomicAdd(a.grad + gb2 + t, a2);
  }
}

size_t grad_tile_smem() { return TILE_SMEM; }

cudaError_t launch_grad_cuda_core(const TrainArgs& a, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(grad_tile_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(TILE_SMEM));
  if (e != cudaSuccess) return e;
  int blocks = static_cast<int>((a.list_cap + TB - 1) / TB);
  grad_tile_kernel<<<blocks, TB, TILE_SMEM, st>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- Adam
// adam_step (guide_field.cpp:317-331). The minibatch's (global) record count
// sits in g[n]; a step only happens when it is non-zero, exactly like the
// reference which never steps on an empty minibatch.
// Adam (GuidingField::adam_step, guide_field.cpp:317-331) with fp64 moments
// and the step control folded in: every block derives the bias corrections
// from `steps + 1` and the record count g[n]; the last block to finish
// publishes |g|^2 and advances `steps`.
__global__ void adam_kernel(float* p, double* m, double* v, const float* g, int64_t n, double lr,
                            double b1, double b2, double eps, double prescale, AdamCtl* c, FieldView f,
                            unsigned char* blob) {
  const double cnt = static_cast<double>(g[n]);
  if (!(cnt > 0.0)) return;  // no usable records: no optimizer step
  const long long step = c->steps + 1;
  const double bc1 = 1.0 - pow(b1, static_cast<double>(step));
  const double bc2 = 1.0 - pow(b2, static_cast<double>(step));
  const double scale = prescale / cnt;
  double local = 0.0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double gi = static_cast<double>(g[i]) * scale;
    local += gi * gi;
    // the reference's operation order, each product rounded on its own (this
    // translation unit may contract FMAs elsewhere): bit-equal moments and
    // updates to GuidingField::adam_step given the same gradient
    double mi = m[i] = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(1.0 - b1, gi));
    double vi = v[i] = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dmul_rn(1.0 - b2, gi), gi));
    double up = __dmul_rn(lr, mi / bc1) / __dadd_rn(sqrt(vi / bc2), eps);
    const float np = static_cast<float>(static_cast<double>(p[i]) - up);
    p[i] = np;
    if (blob != nullptr && i >= f.w1) wpack::pack_param(f, blob, i, np);
  }
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x < 32) {
    double x = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (threadIdx.x == 0) {
      atomicAdd(&c->norm_acc, x);
      __threadfence();
      if (atomicAdd(&c->done, 1u) == gridDim.x - 1) {  // last block: publish the step
        __threadfence();
        c->norm2[(step - 1) % kNormRing] = atomicAdd(&c->norm_acc, 0.0);  // coherent read
        c->norm_acc = 0.0;
        c->done = 0u;
        c->steps = step;
      }
    }
  }
}

cudaError_t launch_adam(float* p, double* m, double* v, const float* g, int64_t n, double lr, double b1,
                        double b2, double eps, double prescale, AdamCtl* ctl, const FieldView& f,
                        unsigned char* blob, cudaStream_t st) {
  int blocks = static_cast<int>((n + 255) / 256);
  if (blocks > 148 * 4) blocks = 148 * 4;
  adam_kernel<<<blocks, 256, 0, st>>>(p, m, v, g, n, lr, b1, b2, eps, prescale, ctl, f, blob);
  return cudaGetLastError();
}

// the whole packed weight blob (wg_wpack.cuh) from the parameters, including
// the zero padding of B3 (rows 33..47), C3 (columns 33..47) and b3
__global__ void pack_weights_kernel(FieldView f, unsigned char* blob) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int64_t i = f.w1 + t; i < static_cast<int64_t>(f.b3) + 33; i += nt) wpack::pack_param(f, blob, i, f.p[i]);
  for (int e = t; e < 15 * 64; e += nt) {
    const int n = 33 + e / 64, k = e % 64;
    wpack::put(blob, wpack::B3H, wpack::B3L, n, k, 64, 0.0f);
    wpack::put(blob, wpack::C3H, wpack::C3L, k, n, 48, 0.0f);
  }
  if (t < 15) reinterpret_cast<float*>(blob + wpack::BIAS)[128 + 33 + t] = 0.0f;
}

cudaError_t launch_pack_weights(const FieldView& f, unsigned char* blob, cudaStream_t st) {
  pack_weights_kernel<<<32, 256, 0, st>>>(f, blob);
  return cudaGetLastError();
}

// host records (wg_guide_record, fp64) -> device records
__global__ void import_records_kernel(const wg_guide_record* in, int64_t n, DevRecord* out) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const wg_guide_record g = in[i];
  DevRecord r{};
  r.x = static_cast<float>(g.x[0]);
  r.y = static_cast<float>(g.x[1]);
  r.nux = static_cast<float>(g.nu[0]);
  r.nuy = static_cast<float>(g.nu[1]);
  r.nx = static_cast<float>(g.normal[0]);
  r.ny = static_cast<float>(g.normal[1]);
  r.pdf_mis = static_cast<float>(g.pdf_mis);
  r.pdf_g = static_cast<float>(g.pdf_g);
  r.pdf_u = static_cast<float>(g.pdf_u);
  r.c = static_cast<float>(g.c);
  r.target = static_cast<float>(g.target);
  r.flags = REC_WRITTEN | (g.on_neumann ? REC_ON_NEUMANN : 0u);
  r.walk = -1;
  r.key = Pcg::mix(0x696d706f7274ULL ^ Pcg::mix(static_cast<uint64_t>(i)));
  out[i] = r;
}

__global__ void export_records_kernel(const DevRecord* in, int64_t n, wg_guide_record* out,
                                      unsigned long long* count) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const DevRecord r = in[i];
  if (!(r.flags & REC_VALID)) return;
  unsigned long long o = atomicAdd(count, 1ull);
  wg_guide_record g{};
  g.x[0] = r.x;
  g.x[1] = r.y;
  g.nu[0] = r.nux;
  g.nu[1] = r.nuy;
  g.nu[2] = 0.0;
  g.target = r.target;
  g.pdf_mis = r.pdf_mis;
  g.pdf_g = r.pdf_g;
  g.pdf_u = r.pdf_u;
  g.c = r.c;
  g.on_neumann = (r.flags & REC_ON_NEUMANN) ? 1 : 0;
  g.normal[0] = r.nx;
  g.normal[1] = r.ny;
  out[o] = g;
}

cudaError_t launch_import_records(const wg_guide_record* in, int64_t n, DevRecord* out,
                                  cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  import_records_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, st>>>(in, n, out);
  return cudaGetLastError();
}

cudaError_t launch_export_records(const DevRecord* in, int64_t n, wg_guide_record* out,
                                  unsigned long long* count, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  export_records_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, st>>>(in, n, out, count);
  return cudaGetLastError();
}

}  // namespace wg
