#include <algorithm>
#include <cstdio>
#include <cstdlib>
// 3D guided walks with the guiding-field MLP on the 5th-generation tensor
// cores (the WG_MLP_TENSOR path of the 3D solver; default for the default 3D
// field shape).
//
// Lockstep CTA of 128 threads = one M = 128 tcgen05 tile: every iteration
//   A  each thread advances its walk through step_begin (fp64 BVH queries);
//      a walk that ends there is replaced at once by the thread's next walk,
//      so a row stays busy while walks remain;
//   B  the rows that need a direction gather their trilinear features (fp32,
//      one 16-B load per lattice corner) and the CTA runs the 3-layer MLP
//      on the tensor cores (wg_mlp_tc.cuh: split-fp16 operands, fp32 TMEM
//      accumulation, ~1e-6 relative to the fp32 MLP; the 41 outputs fit the
//      N = 48 last layer);
//   C  fp64 normalisation, d = 3 MIS sampling, ray and move (step_finish).
// Weights are split into fp16 hi/lo once per CTA from the fp32 parameters.
// This translation unit may contract FMAs (Makefile FAST_TUS): its results
// are compared with the oracle statistically, the exact kernel bit for bit.
#define WG3_PIN_FP 1  // pinned geometry arithmetic (wg3_geom.cuh)
#include "wg3_mix32.cuh"
#include "wg3_walk_common.cuh"
#include "wg_mlp_tc.cuh"

namespace wg3 {

// decode_guiding (wost.cpp:111-122) + sample_next_direction with the fp32
// mixture (wg3_mix32.cuh)
__device__ __forceinline__ Dir3 sample_guided_f(Lane3& w, const Walk3Args& a, const float* raw) {
  Mix3f m;
  normalize3f(raw, m);
  double c = sigmoid(static_cast<double>(raw[40]));  // fp64: 1 - c must not round to 0 (see wg_walk_tc.cu)
  if (a.sp.mode == WG_MODE_GUIDING_ONLY) c = 1.0;
  else if (a.sp.mode == WG_MODE_FIXED_MIS) c = a.sp.fixed_c;
  const Mis3 o = mis_sample3f(w.rng, m, c, w.on_n, w.n, a.sp.reflect != 0);
  return Dir3{o.nu, o.pmis, o.pg, o.pu, c, o.pu / o.pmis};
}

__device__ __forceinline__ void gather3_tc(const Field3View& f, D3 x, float* in) {
  // reciprocal extents (no fp64 division on the direction kernel's path)
  const float u = static_cast<float>(wg::sclamp((x.x - f.bbox[0]) * f.inv_ext[0], 0.0, 1.0));
  const float v = static_cast<float>(wg::sclamp((x.y - f.bbox[1]) * f.inv_ext[1], 0.0, 1.0));
  const float q = static_cast<float>(wg::sclamp((x.z - f.bbox[2]) * f.inv_ext[2], 0.0, 1.0));
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const int res = f.res[l];
    const float rm = static_cast<float>(res - 1);
    const float px = u * rm, py = v * rm, pz = q * rm;
    const int ix = wg::imin(static_cast<int>(px), res - 2), iy = wg::imin(static_cast<int>(py), res - 2),
              iz = wg::imin(static_cast<int>(pz), res - 2);
    const float fx = px - ix, fy = py - iy, fz = pz - iz, gx = 1.0f - fx, gy = 1.0f - fy, gz = 1.0f - fz;
    const float4* b = reinterpret_cast<const float4*>(f.p + f.lvl_off[l]) + (iz * res + iy) * res + ix;
    const int sy = res, sz = res * res;
    const float4 c000 = __ldg(b), c100 = __ldg(b + 1), c010 = __ldg(b + sy), c110 = __ldg(b + sy + 1);
    const float4 c001 = __ldg(b + sz), c101 = __ldg(b + sz + 1), c011 = __ldg(b + sz + sy),
                 c111 = __ldg(b + sz + sy + 1);
    const float w00 = gx * gy, w10 = fx * gy, w01 = gx * fy, w11 = fx * fy;
    const float a0 = w00 * gz, a1 = w10 * gz, a2 = w01 * gz, a3 = w11 * gz;
    const float a4 = w00 * fz, a5 = w10 * fz, a6 = w01 * fz, a7 = w11 * fz;
#define WG3_MIX(C)                                                                                     \
  ((a0 * c000.C + a1 * c100.C) + (a2 * c010.C + a3 * c110.C)) +                                        \
      ((a4 * c001.C + a5 * c101.C) + (a6 * c011.C + a7 * c111.C))
    in[4 * l + 0] = WG3_MIX(x);
    in[4 * l + 1] = WG3_MIX(y);
    in[4 * l + 2] = WG3_MIX(z);
    in[4 * l + 3] = WG3_MIX(w);
#undef WG3_MIX
  }
}

__device__ __forceinline__ void tc3_prologue(unsigned char* smem, const Field3View& f) {
  wg::tc_stage_weights_raw(smem, f.p, f.w1, f.b1, f.w2, f.b2, f.w3, f.b3, OD);
  wg::tc_setup(smem);
  wg::umma::fence_before();
  __syncthreads();
  wg::umma::fence_after();
}

__global__ void __launch_bounds__(128, 1) walk3_tc_kernel(Walk3Args a) {
  extern __shared__ __align__(128) unsigned char smem[];
  tc3_prologue(smem, a.f);
  const bool collect = a.recs != nullptr;
  const int64_t total = a.n_points * static_cast<int64_t>(a.n_rounds);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t next = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t phase = 0;
  Lane3 w;
  w.alive = false;
  w.rec_base = 0;
  w.rec_left = 0;
  int64_t walks_done = 0;
  for (;;) {
    // ---- A: advance to a step that needs a direction (or run out of walks)
    bool need = false;
    int rec = -1;
    while (!need) {
      if (!w.alive) {
        if (next >= total) break;
        lane3_init(w, a, next);
        next += stride;
        ++walks_done;
      }
      need = step_begin(w, a, collect, rec);
    }
    if (__syncthreads_count(need) == 0) break;
    // ---- B: features + MLP on the tensor cores for the whole tile
    float in[IN], raw[OD];
    if (need) {
      gather3_tc(a.f, w.x, in);
    } else {
#pragma unroll
      for (int i = 0; i < IN; ++i) in[i] = 0.0f;
    }
    wg::tc_forward<OD>(smem, phase, in, raw);
    // ---- C: mixture, MIS direction, move
    if (need) step_move(w, a, collect, rec, sample_guided_f(w, a, raw), true);
  }
  if (collect)
    for (int i = 0; i < w.rec_left; ++i) a.recs[w.rec_base + (8 - w.rec_left) + i].flags = 0u;
  unsigned long long wd = static_cast<unsigned long long>(walks_done);
  for (int o = 16; o > 0; o >>= 1) wd += __shfl_down_sync(0xffffffffu, wd, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&a.counters[2], wd);
  wg::tc_teardown(smem);
}

// field evaluation on the tensor cores: persistent CTAs over 128-point tiles
__global__ void __launch_bounds__(128) field3_eval_tc_kernel(Field3View f, int64_t n, const double* x,
                                                             double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  tc3_prologue(smem, f);
  uint32_t phase = 0;
  const int64_t tiles = (n + 127) / 128;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t i = t * 128 + threadIdx.x;
    float in[IN], o[OD];
    if (i < n) {
      gather3_tc(f, D3{x[3 * i], x[3 * i + 1], x[3 * i + 2]}, in);
    } else {
#pragma unroll
      for (int k = 0; k < IN; ++k) in[k] = 0.0f;
    }
    wg::tc_forward<OD>(smem, phase, in, o);
    if (i < n)
      for (int j = 0; j < OD; ++j) out[i * OD + j] = o[j];
  }
  wg::tc_teardown(smem);
}

// ---------------------------------------------------------------- wavefront
// The guided 3D walk as two kernels per iteration over a pool of walk slots
// (lane state in HBM, ~200 B per slot):
//   wave_geom_kernel  one thread per slot (high occupancy for the latency-bound
//                     fp64 BVH traversals): finishes the slot's pending move
//                     (record, Neumann ray, move, escape), refills an empty
//                     slot with the next walk id, runs step_begin, and queues
//                     the slot when it needs a direction;
//   wave_dir_kernel   persistent tcgen05 tiles over the queue: trilinear
//                     gather, the MLP, then per row the fp64 decode and MIS
//                     sampling (no BVH work, so no lockstep divergence).
// The host re-launches the pair until a geometry pass queues nothing.
enum : uint8_t { SLOT_EMPTY = 0, SLOT_NEED_DIR = 1, SLOT_NEED_MOVE = 2 };
// walks left at the drain hand-off to wave_tail_kernel: cfg 4 shape, 32 training
// rounds 408-434 ms at 37,888-131,072 vs 553-563 ms without (and 534-544 ms
// with every walk in the tail kernel); frozen rounds unchanged
constexpr long kTailDefault = 65536;
// occupancy of the latency-bound geometry kernel: 5 CTAs/SM (<= 102
// registers, a few hundred bytes of spills) measured 144 vs 171 ms walk time
// at 512^2 x 8 wpp against the unconstrained 132-register build; the
// tensor-core direction kernel is best left at 2 CTAs/SM (3: 193 ms)
#ifndef WG3_GEOM_MINB
#define WG3_GEOM_MINB 6
#endif
#ifndef WG3_DIR_MINB
#define WG3_DIR_MINB 1
#endif

// Morton cell (kSortBits per axis) of a position: the sort key of the
// geometry pass's order
__device__ __forceinline__ uint32_t spread3(uint32_t v) {  // <= 10 bits -> every third bit
  v &= 0x3FFu;
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}
__device__ __forceinline__ int sort_cell(const Walk3Args& a, const D3& x) {
  const double* b = a.s.bbox;
  const double q = static_cast<double>(1 << kSortBits);
  auto cell = [&](double c, double lo, double hi) {
    const int i = static_cast<int>((c - lo) / (hi - lo) * q);
    return static_cast<uint32_t>(i < 0 ? 0 : i > (1 << kSortBits) - 1 ? (1 << kSortBits) - 1 : i);
  };
  return static_cast<int>(spread3(cell(x.x, b[0], b[3])) | (spread3(cell(x.y, b[1], b[4])) << 1) |
                          (spread3(cell(x.z, b[2], b[5])) << 2));
}

__global__ void __launch_bounds__(128, WG3_GEOM_MINB) wave_geom_kernel(Walk3Args a, Wave3 v, int parity) {
  const bool collect = a.recs != nullptr;
  const unsigned long long total = static_cast<unsigned long long>(a.n_points) * a.n_rounds;
  unsigned int* qlen = v.qlen + parity;
  unsigned long long started = 0;
  // every walk id handed out: empty slots stay empty without touching their
  // lane or the counter (the drain of a round; a stale read only costs work)
  const bool exhausted = *reinterpret_cast<volatile unsigned long long*>(v.next_walk) >= total;
  // perm's first n entries hold every slot that can have work (all slots
  // while walks remain to start; the live ones once every id is handed out)
  const int64_t n = v.bins[kSortBins + 1];
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // slots in spatial-cell order: neighbouring lanes walk near each other,
    // so their BVH traversals take the same branches and load the same nodes
    const int64_t slot = v.perm[t];
    const uint8_t st = v.state[slot];
    if (st != SLOT_NEED_MOVE && exhausted) continue;
    Lane3 w;
    // a collecting slot carries its record chunk (rec_base / rec_left) from
    // walk to walk, so the lane is loaded even when the slot is empty
    if (st == SLOT_NEED_MOVE || collect) w = v.lanes[slot];
    if (st != SLOT_NEED_MOVE) w.alive = false;
    if (st == SLOT_NEED_MOVE) step_move(w, a, collect, v.rec[slot], v.dirs[slot], true);
    bool need = false;
    int rec = -1;
    for (int tries = 0; tries < 4 && !need; ++tries) {
      if (!w.alive) {
        const unsigned long long id = claim_walk(v.next_walk);
        if (id >= total) break;
        lane3_init(w, a, static_cast<int64_t>(id));
        if (!collect) {
          w.rec_base = 0;
          w.rec_left = 0;
        }
        ++started;
      }
      need = step_begin(w, a, collect, rec);
    }
    if (need) {
      v.lanes[slot] = w;
      v.rec[slot] = rec;
      v.state[slot] = SLOT_NEED_DIR;
      v.queue[claim_queue(qlen)] = static_cast<int32_t>(slot);
      v.sbin[slot] = static_cast<uint16_t>(sort_cell(a, w.x));  // where its next move starts
    } else {
      if (collect) v.lanes[slot] = w;  // record-chunk bookkeeping
      v.state[slot] = SLOT_EMPTY;
      v.sbin[slot] = static_cast<uint16_t>(kSortBins);
    }
  }
  for (int o = 16; o > 0; o >>= 1) started += __shfl_down_sync(0xffffffffu, started, o);
  if ((threadIdx.x & 31) == 0 && started) atomicAdd(&a.counters[2], started);
}

// ---- spatial ordering of the geometry pass: a counting sort of the slots
// by the Morton cell (kSortBits per axis) of their walk's position; slots
// without a pending move go last. The order only changes which lanes run
// side by side: every slot is visited exactly once either way.
__device__ __forceinline__ int slot_bin(const Wave3& v, int64_t slot) {
  const int b = v.sbin[slot];
  return b < kSortBins ? b : kSortBins;
}
__device__ __forceinline__ bool walks_exhausted(const Walk3Args& a, const Wave3& v) {
  return *reinterpret_cast<volatile unsigned long long*>(v.next_walk) >=
         static_cast<unsigned long long>(a.n_points) * a.n_rounds;
}
__global__ void __launch_bounds__(256) sort_count_kernel(Walk3Args a, Wave3 v) {
  // the drain of a round: once every walk id is out and few slots remain
  // live, the previous order (which covers them) is kept
  const bool skip = walks_exhausted(a, v) && v.bins[kSortBins + 1] < v.slots / 16;
  if (blockIdx.x == 0 && threadIdx.x == 0) v.bins[kSortBins + 2] = skip ? 1u : 0u;
  if (skip) return;
  if constexpr (kSortBins <= 8192) {  // block histogram in shared memory
    __shared__ unsigned int h[kSortBins + 1];
    for (int i = threadIdx.x; i <= kSortBins; i += blockDim.x) h[i] = 0u;
    __syncthreads();
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < v.slots;
         s += static_cast<int64_t>(gridDim.x) * blockDim.x)
      atomicAdd(&h[slot_bin(v, s)], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i <= kSortBins; i += blockDim.x)
      if (h[i]) atomicAdd(&v.bins[i], h[i]);
  } else {
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < v.slots;
         s += static_cast<int64_t>(gridDim.x) * blockDim.x)
      atomicAdd(&v.bins[slot_bin(v, s)], 1u);
  }
}
__global__ void __launch_bounds__(1024) sort_scan_kernel(Walk3Args a, Wave3 v) {  // exclusive scan, one CTA
  if (v.bins[kSortBins + 2]) return;
  constexpr int kPer = (kSortBins + 1 + 1023) / 1024;
  __shared__ unsigned int part[1024];
  unsigned int loc[kPer], sum = 0;
  for (int j = 0; j < kPer; ++j) {
    const int i = threadIdx.x * kPer + j;
    loc[j] = i <= kSortBins ? v.bins[i] : 0u;
    sum += loc[j];
  }
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan of the partial sums
    const unsigned int add = threadIdx.x >= o ? part[threadIdx.x - o] : 0u;
    __syncthreads();
    part[threadIdx.x] += add;
    __syncthreads();
  }
  unsigned int run = part[threadIdx.x] - sum;
  for (int j = 0; j < kPer; ++j) {
    const int i = threadIdx.x * kPer + j;
    if (i <= kSortBins) v.bins[i] = run;
    // entries the geometry pass visits: without walks left to start, the
    // slots with no pending move (the last bin) are left out
    if (i == kSortBins) v.bins[kSortBins + 1] = walks_exhausted(a, v) ? run : static_cast<unsigned int>(v.slots);
    run += loc[j];
  }
}
// block-local ranking: each CTA ranks its chunk of slots per cell in shared
// memory, reserves one range per non-empty cell with a single global atomic,
// then writes perm (instead of one contended global atomic per slot)
constexpr int kScatterPer = 16;  // slots per thread
__global__ void __launch_bounds__(256) sort_scatter_kernel(Walk3Args a, Wave3 v) {
  if (v.bins[kSortBins + 2]) return;
  __shared__ unsigned int h[kSortBins + 1];
  const bool drop_idle = walks_exhausted(a, v);
  for (int i = threadIdx.x; i <= kSortBins; i += blockDim.x) h[i] = 0u;
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x * kScatterPer + threadIdx.x;
  unsigned int rank[kScatterPer];
  uint16_t bin[kScatterPer];
#pragma unroll
  for (int k = 0; k < kScatterPer; ++k) {
    const int64_t s = base + static_cast<int64_t>(k) * blockDim.x;
    int b = kSortBins + 1;  // none
    if (s < v.slots) {
      b = slot_bin(v, s);
      if (b == kSortBins && drop_idle) b = kSortBins + 1;
    }
    bin[k] = static_cast<uint16_t>(b);
    if (b <= kSortBins) rank[k] = atomicAdd(&h[b], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= kSortBins; i += blockDim.x)
    if (h[i]) h[i] = atomicAdd(&v.bins[i], h[i]);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kScatterPer; ++k)
    if (bin[k] <= kSortBins)
      v.perm[h[bin[k]] + rank[k]] = static_cast<int32_t>(base + static_cast<int64_t>(k) * blockDim.x);
}
__global__ void perm_identity_kernel(Wave3 v) {
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < v.slots;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x)
    v.perm[s] = static_cast<int32_t>(s);
  if (blockIdx.x == 0 && threadIdx.x == 0) v.bins[kSortBins + 1] = static_cast<unsigned int>(v.slots);
}

// the field's MLP weights as the split-fp16 blob the direction kernel
// fetches with one bulk copy (the wg_wpack.cuh forward layout; W3 has 41
// outputs here): once per wavefront call, the weights are fixed during it
__global__ void pack3_weights_kernel(Field3View f, unsigned char* blob) {
  // blob = shared-memory image of [B1_HI, BAR)
  wg::tc_stage_weights_raw(blob - wg::TcLayout::B1_HI, f.p, f.w1, f.b1, f.w2, f.b2, f.w3, f.b3, OD);
}

__global__ void __launch_bounds__(128, WG3_DIR_MINB) wave_dir_kernel(Walk3Args a, Wave3 v, int parity) {
  extern __shared__ __align__(128) unsigned char smem[];
  if (blockIdx.x == 0 && threadIdx.x == 0) v.qlen[parity ^ 1] = 0u;  // next geometry pass's queue
  const unsigned int n = v.qlen[parity];
  if (static_cast<unsigned int>(blockIdx.x) * 128u >= n) return;
  // weights: one TMA bulk copy of the packed blob, overlapped with the TMEM
  // allocation
  wg::tc_fetch_weights(smem, v.wblob);
  wg::tc_setup(smem);
  wg::umma::fence_before();
  __syncthreads();
  wg::umma::fence_after();
  wg::tc_wait_weights(smem);
  uint32_t phase = 0;
  // the next tile's slot and position are loaded while this tile works, so a
  // tile's gather does not wait on the queue -> lane -> grid load chain
  unsigned int t = blockIdx.x;
  int32_t nslot = t * 128u + threadIdx.x < n ? v.queue[t * 128u + threadIdx.x] : -1;
  D3 nx = nslot >= 0 ? v.lanes[nslot].x : D3{0.0, 0.0, 0.0};
  for (; t * 128u < n; t += gridDim.x) {
    const int32_t slot = nslot;
    const bool live = slot >= 0;
    const D3 x = nx;
    const unsigned int rn = (t + gridDim.x) * 128u + threadIdx.x;
    nslot = rn < n ? v.queue[rn] : -1;
    float in[IN], raw[OD];
    Lane3 w;
    if (live) {
      gather3_tc(a.f, x, in);
      w = v.lanes[slot];
    } else {
#pragma unroll
      for (int i = 0; i < IN; ++i) in[i] = 0.0f;
    }
    wg::tc_forward<OD>(smem, phase, in, raw);
    nx = nslot >= 0 ? v.lanes[nslot].x : D3{0.0, 0.0, 0.0};
    if (live) {
      v.dirs[slot] = sample_guided_f(w, a, raw);
      v.lanes[slot].rng = w.rng;
      v.state[slot] = SLOT_NEED_MOVE;
    }
  }
  wg::tc_teardown(smem);
}

// The drain of a call: once every walk id is out and at most tail_n walks
// remain, the device loop exits and this kernel finishes them in lockstep
// CTAs like walk3_tc_kernel: pending move, begin_step, gather + MLP on the
// tensor cores for the rows still walking, MIS draw, repeat. A row whose walk
// ends takes the next walk of the last queue (qlen[0], zeroed by the last
// direction pass, counts the hand-out). Same step functions and MLP as the
// wavefront pair, so every walk's result is unchanged; what goes is the
// per-iteration cost of the drain (sort, two launches, the direction
// kernel's weight fetch, a geometry grid over the whole pool) while the
// round's longest walks finish.
#ifdef WG3_TAIL_PROF
__device__ unsigned long long g_tail_prof[16];
#endif
__global__ void __launch_bounds__(128, 2) wave_tail_kernel(Walk3Args a, Wave3 v) {
  extern __shared__ __align__(128) unsigned char smem[];
  const unsigned int n = v.qlen[1];
  // first an even share of the queue per CTA (<= 128 rows), then one at a time
  const unsigned int per = min(128u, (n + gridDim.x - 1) / gridDim.x);
  const unsigned int spread = per * gridDim.x;
  if (static_cast<unsigned int>(blockIdx.x) * per >= n) return;
  wg::tc_fetch_weights(smem, v.wblob);
  wg::tc_setup(smem);
  wg::umma::fence_before();
  __syncthreads();
  wg::umma::fence_after();
  wg::tc_wait_weights(smem);
  const bool collect = a.recs != nullptr;
  int32_t slot = -1;
  Lane3 w;
  w.alive = false;
  Dir3 d{};
  int rec = -1;
  bool need = false, more = true, first = true;
  uint32_t phase = 0;
#ifdef WG3_TAIL_PROF
  long long pc[4][3] = {}, c_g = 0, c_f = 0, c_mma = 0;
#endif
  for (;;) {
#ifdef WG3_TAIL_PROF
    const long long c0 = clock64();
#endif
    if (need) {  // the geometry pass's work for this slot (no walk ids left to claim)
      step_move(w, a, collect, rec, d, true);
      need = w.alive && step_begin(w, a, collect, rec);
    }
    while (!need && more) {  // next walk of the queue, with its pending move
      if (slot >= 0) {
        if (collect) v.lanes[slot] = w;  // record-chunk bookkeeping for wave_close_kernel
        v.state[slot] = SLOT_EMPTY;
        slot = -1;
      }
      const unsigned int i = first ? blockIdx.x * per + threadIdx.x : spread + claim_queue(v.qlen);
      first = false;
      if (i >= n || (i < spread && threadIdx.x >= per)) {
        more = false;
        break;
      }
      slot = v.queue[i];
      w = v.lanes[slot];
      d = v.dirs[slot];
      rec = v.rec[slot];
      step_move(w, a, collect, rec, d, true);
      need = w.alive && step_begin(w, a, collect, rec);
    }
    const int live_rows = __syncthreads_count(need);
    if (live_rows == 0) break;
#ifdef WG3_TAIL_PROF
    const long long c1 = clock64();
#endif
    float in[IN], raw[OD];  // the direction pass's
    if (need) {
      gather3_tc(a.f, w.x, in);
    } else {
#pragma unroll
      for (int i = 0; i < IN; ++i) in[i] = 0.0f;
    }
#ifdef WG3_TAIL_PROF
    __syncthreads();
    const long long c2 = clock64();
#endif
#ifdef WG3_TAIL_PROF
    long long bp[2] = {0, 0};
    wg::tc_forward<OD>(smem, phase, in, raw, bp);
    __syncthreads();
    const long long c3 = clock64();
#else
    wg::tc_forward<OD>(smem, phase, in, raw);
#endif
    if (need) d = sample_guided_f(w, a, raw);
#ifdef WG3_TAIL_PROF
    __syncthreads();
    {
      const int bk = live_rows > 64 ? 0 : live_rows > 16 ? 1 : live_rows > 4 ? 2 : 3;
      pc[bk][0] += c1 - c0;
      pc[bk][1] += clock64() - c1;
      pc[bk][2] += 1;
      c_g += c2 - c1;
      c_f += c3 - c2;
      c_mma += bp[0];
    }
#endif
  }
#ifdef WG3_TAIL_PROF
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 3; ++j) atomicAdd(&g_tail_prof[3 * i + j], static_cast<unsigned long long>(pc[i][j]));
    atomicAdd(&g_tail_prof[12], 1ull);
    atomicAdd(&g_tail_prof[13], static_cast<unsigned long long>(c_g));
    atomicAdd(&g_tail_prof[14], static_cast<unsigned long long>(c_f));
    atomicAdd(&g_tail_prof[15], static_cast<unsigned long long>(c_mma));
  }
#endif
  if (slot >= 0) {
    if (collect) v.lanes[slot] = w;
    v.state[slot] = SLOT_EMPTY;
  }
  wg::tc_teardown(smem);
}

// trailing record slots of every lane's last chunk are marked unused
__global__ void wave_close_kernel(Walk3Args a, Wave3 v) {
  for (int64_t slot = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; slot < v.slots;
       slot += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const Lane3& w = v.lanes[slot];
    for (int i = 0; i < w.rec_left; ++i) a.recs[w.rec_base + (8 - w.rec_left) + i].flags = 0u;
  }
}

// end of a two-iteration body of the device-side loop: continue while walk
// ids remain or the last geometry pass queued more than tail_n slots (the
// rest go to wave_tail_kernel); count the kernels
__global__ void wave_continue_kernel(Wave3 v, unsigned long long total, unsigned int tail_n,
                                     cudaGraphConditionalHandle cond, unsigned long long* launches,
                                     unsigned body_kernels) {
  if (threadIdx.x != 0) return;
  const bool more = v.qlen[1] > tail_n || *v.next_walk < total;
  cudaGraphSetConditional(cond, more ? 1u : 0u);
  atomicAdd(launches, static_cast<unsigned long long>(body_kernels));
}

cudaError_t launch_walks3_wave(const Walk3Args& a, const Wave3& v, int sms, unsigned int* h_qlen,
                               int64_t* launches, cudaStream_t st) {
  *launches = 0;
  const unsigned long long total = static_cast<unsigned long long>(a.n_points) * a.n_rounds;
  const int smem = walk3_tc_smem();
  cudaError_t e = cudaFuncSetAttribute(wave_dir_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(v.state, 0, static_cast<size_t>(v.slots), st);
  cudaMemsetAsync(v.qlen, 0, 2 * sizeof(unsigned int), st);
  cudaMemsetAsync(v.next_walk, 0, sizeof(unsigned long long), st);
  if (a.recs) cudaMemsetAsync(v.lanes, 0, sizeof(Lane3) * static_cast<size_t>(v.slots), st);
  pack3_weights_kernel<<<1, 256, 0, st>>>(a.f, v.wblob);
  perm_identity_kernel<<<sms * 4, 256, 0, st>>>(v);
  *launches += 2;
  // spatial re-ordering of the geometry pass every iteration (every second
  // one on record-collecting rounds, whose drains dominate). cfg 4 shape,
  // 512^2 x 256 frozen rounds: 3.25 s (every iteration) / 3.34 s (every
  // second) vs 3.91 s unsorted; 32 training rounds 0.91 / 0.89 / 0.88 s.
  // 4 bits per axis: 5 bits measured no faster (3.27 s; training 0.99 s)
  const int sort_period = a.recs ? 2 : 1;  // (with wide BVHs: frozen rounds equal at 1 and 2)
  const int geom_blocks = static_cast<int>((v.slots + 127) / 128);
  const int scatter_blocks = static_cast<int>((v.slots + 256 * kScatterPer - 1) / (256 * kScatterPer));
  cudaMemsetAsync(v.sbin, 0xFF, sizeof(uint16_t) * static_cast<size_t>(v.slots), st);  // no pending moves
  // persistent direction CTAs, 2 per SM (197 registers; cfg 4 frozen rounds
  // 2.84 s vs 2.91 s at 3 per SM and 3.07 s at 1)
#ifndef WG3_DIR_PER_SM
#define WG3_DIR_PER_SM 2
#endif
  const int dir_blocks = sms * WG3_DIR_PER_SM;
  // the drain hand-off: 2 tail CTAs per SM of 128 rows
  // (WOSTGPU_WAVE3_TAIL = walks left when the device loop hands over; 0 = off)
  const int tail_blocks = sms * 2;
  const char* tail_pe = std::getenv("WOSTGPU_WAVE3_TAIL");  // read per call (tests switch it)
  const long tail_env = tail_pe ? std::atol(tail_pe) : -1L;
  const unsigned int tail_n = static_cast<unsigned int>(
      tail_env >= 0 ? tail_env : kTailDefault);
  if (tail_n) {
    if ((e = cudaFuncSetAttribute(wave_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) !=
        cudaSuccess)
      return e;
  }
  // The iteration loop runs on the device: a CUDA graph whose while node
  // repeats a body of two iterations (parities 0 and 1) until a geometry
  // pass queued nothing and every walk id is out; wave_continue_kernel sets
  // the condition and counts the body's kernels into counters[5]. No host
  // polling, no per-iteration launches from the host.
  // WOSTGPU_PROFILE_LOOP=1 (profiling only): the same iterations launched
  // from the host, so kernel profilers see every launch (ncu does not
  // profile the device-launched bodies of a conditional graph node)
  // WOSTGPU_PROFILE_LOOP=2: also times each pass with events and prints
  // (iteration, queued walks, sort / geometry / direction microseconds)
  static const int host_loop = [] {
    const char* pe = std::getenv("WOSTGPU_PROFILE_LOOP");
    return pe && (pe[0] == '1' || pe[0] == '2') ? pe[0] - '0' : 0;
  }();
  if (host_loop) {
    cudaEvent_t ev[4];
    for (auto& x : ev) cudaEventCreate(&x);
    for (int it = 0;; it += 2) {
      for (int par = 0; par < 2; ++par) {
        unsigned int q0 = 0;
        if (host_loop == 2) {
          cudaMemcpyAsync(&q0, v.qlen + (par ^ 1), sizeof(unsigned int), cudaMemcpyDeviceToHost, st);
          cudaEventRecord(ev[0], st);
        }
        if (par == 0 || sort_period == 1) {
          cudaMemsetAsync(v.bins, 0, sizeof(unsigned int) * (kSortBins + 1), st);
          sort_count_kernel<<<sms * 2, 256, 0, st>>>(a, v);
          sort_scan_kernel<<<1, 1024, 0, st>>>(a, v);
          sort_scatter_kernel<<<scatter_blocks, 256, 0, st>>>(a, v);
          *launches += 3;
        }
        if (host_loop == 2) cudaEventRecord(ev[1], st);
        wave_geom_kernel<<<geom_blocks, 128, 0, st>>>(a, v, par);
        if (host_loop == 2) cudaEventRecord(ev[2], st);
        wave_dir_kernel<<<dir_blocks, 128, smem, st>>>(a, v, par);
        if (host_loop == 2) {
          cudaEventRecord(ev[3], st);
          cudaEventSynchronize(ev[3]);
          float t[3];
          for (int i = 0; i < 3; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
          std::fprintf(stderr, "wave3 it %d live %u sort %.1f geom %.1f dir %.1f\n", it + par, q0, t[0] * 1e3f,
                       t[1] * 1e3f, t[2] * 1e3f);
        }
        *launches += 2;
      }
      unsigned long long h[2] = {0, 0};
      cudaMemcpyAsync(&h[0], v.qlen + 1, sizeof(unsigned int), cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(&h[1], v.next_walk, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
      if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
      if (static_cast<unsigned int>(h[0]) <= tail_n && h[1] >= total) break;
    }
    for (auto& x : ev) cudaEventDestroy(x);
  } else {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  auto fail = [&](cudaError_t err) {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    return err;
  };
  if ((e = cudaGraphCreate(&graph, 0)) != cudaSuccess) return fail(e);
  cudaGraphConditionalHandle cond;
  if ((e = cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault)) != cudaSuccess)
    return fail(e);
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = cond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  if ((e = cudaGraphAddNode(&node, graph, nullptr, 0, &cp)) != cudaSuccess) return fail(e);
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  if ((e = cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal)) !=
      cudaSuccess)
    return fail(e);
  unsigned body_kernels = 0;
  for (int par = 0; par < 2; ++par) {
    if (par == 0 || sort_period == 1) {
      cudaMemsetAsync(v.bins, 0, sizeof(unsigned int) * (kSortBins + 1), st);
      sort_count_kernel<<<sms * 2, 256, 0, st>>>(a, v);
      sort_scan_kernel<<<1, 1024, 0, st>>>(a, v);
      sort_scatter_kernel<<<scatter_blocks, 256, 0, st>>>(a, v);
      body_kernels += 3;
    }
    wave_geom_kernel<<<geom_blocks, 128, 0, st>>>(a, v, par);
    wave_dir_kernel<<<dir_blocks, 128, smem, st>>>(a, v, par);
    body_kernels += 2;
  }
  wave_continue_kernel<<<1, 32, 0, st>>>(v, total, tail_n, cond, a.counters + 5, body_kernels + 1);
  cudaGraph_t captured = nullptr;
  if ((e = cudaStreamEndCapture(st, &captured)) != cudaSuccess) return fail(e);
  if ((e = cudaGraphInstantiate(&exec, graph, 0)) != cudaSuccess) return fail(e);
  if ((e = cudaGraphLaunch(exec, st)) != cudaSuccess) return fail(e);
  cudaGraphExecDestroy(exec);  // released once the launch completes
  cudaGraphDestroy(graph);
  }
  (void)h_qlen;
  if (tail_n) {
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (host_loop == 2) {
      unsigned int q = 0;
      cudaMemcpyAsync(&q, v.qlen + 1, sizeof(unsigned int), cudaMemcpyDeviceToHost, st);
      cudaEventCreate(&t0);
      cudaEventCreate(&t1);
      cudaEventRecord(t0, st);
      wave_tail_kernel<<<tail_blocks, 128, smem, st>>>(a, v);
      cudaEventRecord(t1, st);
      cudaEventSynchronize(t1);
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, t0, t1);
      std::fprintf(stderr, "wave3 tail live %u us %.1f\n", q, ms * 1e3f);
#ifdef WG3_TAIL_PROF
      unsigned long long pr[16];
      cudaMemcpyFromSymbol(pr, g_tail_prof, sizeof(pr));
      const double ctas = pr[12] ? double(pr[12]) : 1.0;
      double its = 0;
      for (int i = 0; i < 4; ++i) {
        const double n = pr[3 * i + 2] ? double(pr[3 * i + 2]) : 1.0;
        its += pr[3 * i + 2];
        std::fprintf(stderr, "wave3 tail prof rows %s: %.1f its/CTA, geo %.0f mlp %.0f cycles/it\n",
                     i == 0 ? ">64" : i == 1 ? "17-64" : i == 2 ? "5-16" : "<=4", pr[3 * i + 2] / ctas,
                     pr[3 * i] / n, pr[3 * i + 1] / n);
      }
      std::fprintf(stderr, "wave3 tail prof all: gather %.0f forward %.0f mma %.0f cycles/it\n", pr[13] / its,
                   pr[14] / its, pr[15] / its);
      const unsigned long long z[16] = {};
      cudaMemcpyToSymbol(g_tail_prof, z, sizeof(z));
#endif
      cudaEventDestroy(t0);
      cudaEventDestroy(t1);
    } else {
      wave_tail_kernel<<<tail_blocks, 128, smem, st>>>(a, v);
    }
    *launches += 1;
  }
  if (a.recs) {
    wave_close_kernel<<<geom_blocks, 128, 0, st>>>(a, v);
    *launches += 1;
  }
  return cudaGetLastError();
}

// diagnostic: the direction kernel's fp32 decode + mixture density of raw
// rows (41 floats) at unit directions nu (tests compare it with the oracle)
__global__ void mix3f_pdf_kernel(int64_t n, const float* raw, const double* nu, double* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float r[OD];
  for (int j = 0; j < OD; ++j) r[j] = raw[i * OD + j];
  Mix3f m;
  normalize3f(r, m);
  out[2 * i] = mixture_pdf3f(m, D3{nu[3 * i], nu[3 * i + 1], nu[3 * i + 2]});
  out[2 * i + 1] = sigmoid(static_cast<double>(r[40]));  // c as sample_guided_f forms it
}

cudaError_t launch_mix3f_pdf(int64_t n, const float* raw, const double* nu, double* out, cudaStream_t st) {
  mix3f_pdf_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, st>>>(n, raw, nu, out);
  return cudaGetLastError();
}

int walk3_tc_smem() { return static_cast<int>((wg::TcLayout::BYTES + 127) / 128 * 128); }

int walk3_tc_blocks_per_sm() {
  static int n = [] {
    int b = 0;
    const int smem = walk3_tc_smem();
    cudaFuncSetAttribute(walk3_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, walk3_tc_kernel, 128, smem);
    return b < 1 ? 1 : b;
  }();
  return n;
}

cudaError_t launch_walks3_tc(const Walk3Args& a, int blocks, cudaStream_t st) {
  const int smem = walk3_tc_smem();
  cudaError_t e = cudaFuncSetAttribute(walk3_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  walk3_tc_kernel<<<blocks, 128, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_field3_eval_tc(const Field3View& f, int64_t n, const double* x, double* out,
                                  cudaStream_t st) {
  const int smem = walk3_tc_smem();
  cudaError_t e =
      cudaFuncSetAttribute(field3_eval_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t tiles = (n + 127) / 128;
  const int blocks = static_cast<int>(tiles < sms * 2 ? tiles : sms * 2);
  field3_eval_tc_kernel<<<blocks > 0 ? blocks : 1, 128, smem, st>>>(f, n, x, out);
  return cudaGetLastError();
}

}  // namespace wg3
