// 2D guided walks as a wavefront (the 3D design, wg3_walk_tc.cu, on 2D
// scenes): two kernels per iteration over a pool of walk slots, walk state in
// HBM between them.
//   wave2_geom_kernel  one thread per slot, no CTA barrier: finishes the
//                      slot's pending move (record, Neumann ray, move,
//                      escape), refills an empty slot with the next walk id,
//                      then begin_step (closest point, roulette, silhouette,
//                      star radius, source / Neumann terms; wost.cpp:148-216)
//                      and queues the slot when it needs a direction;
//   wave2_dir_kernel   persistent tcgen05 tiles over the queue: bilinear
//                      gather, the MLP (wg_mlp_tc.cuh), then per row the
//                      decode and MIS sampling (sphdist.cpp:254-270) with the
//                      tensor path's fp32 mixture math (wg_mix32.cuh).
// Used for the tensor-core path when enough walks are in flight to fill the
// GPU (cfg 3: a 256-segment disk, 512^2 points): the lockstep kernel's
// iteration waits for the slowest of 128 BVH traversals (phase A ~60k
// cycles per iteration on cfg 3) at 4 warps per SM. The step logic follows
// the exact kernel (wg_walk.cu) with fp64 geometry and mixture math; this
// translation unit may contract FMAs (statistical parity, like the tensor
// path).
#include <cooperative_groups.h>
#include <cstdlib>

#include "wg_kernels.cuh"
#include "wg_mix32.cuh"
#include "wg_mlp_tc.cuh"
#include "wg_sphdist.cuh"

namespace wg {
namespace {

struct Lane2 {
  double x, y, nx, ny, T, acc, dacc, R;
  int seg, depth, round, rec_left, last_rec;
  bool on_n, alive, rec_ok;
  Pcg rng;
  int64_t point, rec_base;
};

struct Dir2 {
  double nux, nuy, pmis, pg, pu, sel, mult;
};

enum : uint8_t { SLOT_EMPTY = 0, SLOT_NEED_DIR = 1, SLOT_NEED_MOVE = 2 };
// walks left at the drain hand-off to wave2_tail_kernel: cfg 3 (512^2), 32
// training rounds 417-419 ms at 131,072, 427-429 at 65,536, 486 at 16,384,
// 600 ms without, 485 ms with every walk in the tail kernel; frozen rounds
// unchanged (200-204 ms)
constexpr long kTail2Default = 131072;

// greens_ball / sample_greens_radius, d = 2 (wost.cpp:27-65)
__device__ __forceinline__ double greens_ball_2d(double r, double R) {
  if (r <= 0.0) return dinf();
  return log(R / r) / kTwoPi;
}
__device__ double greens_radius_2d(double u, double R) {
  if (u <= 0.0) return 0.0;
  if (u >= 1.0) return R;
  double lo = 0.0, hi = 1.0, s = sqrt(u);
  for (int it = 0; it < 100; ++it) {
    double ls = log(s);
    double f = s * s * (1.0 - 2.0 * ls) - u;
    double df = -4.0 * s * ls;
    if (f > 0.0) hi = s;
    else lo = s;
    if (fabs(f) < 1e-10) break;
    double step = df > 0.0 ? f / df : 0.0;
    double nx = s - step;
    if (!(nx > lo && nx < hi)) nx = 0.5 * (lo + hi);
    if (nx == s) break;
    s = nx;
  }
  return s * R;
}

__device__ __forceinline__ void lane2_init(Lane2& w, const WalkArgs& a, int64_t id) {
  w.round = static_cast<int>(id / a.n_points);
  w.point = id - static_cast<int64_t>(w.round) * a.n_points;
  w.x = a.points[2 * w.point];
  w.y = a.points[2 * w.point + 1];
  w.nx = w.ny = 0.0;
  w.on_n = false;
  w.seg = -1;
  w.T = 1.0;
  w.acc = 0.0;
  w.dacc = 0.0;
  w.R = 0.0;
  w.depth = 0;
  w.alive = true;
  w.rng = Pcg::walk(a.seed, static_cast<uint64_t>(a.point_offset + w.point),
                    a.wpp_first + static_cast<uint64_t>(w.round));
  w.last_rec = -1;
  w.rec_ok = true;
}

__device__ __forceinline__ void finish2(Lane2& w, const WalkArgs& a, bool escaped, double terminal,
                                        bool collect) {
  const int64_t slot = static_cast<int64_t>(w.round) * a.n_points + w.point;
  a.est[slot] = escaped ? 0.0 : w.acc;
  a.esc[slot] = escaped ? 1 : 0;
  if (a.steps) a.steps[slot] = w.depth;
  atomicAdd(&a.counters[0], static_cast<unsigned long long>(w.depth));
  if (escaped) atomicAdd(&a.counters[1], 1ull);
  if (collect && a.rec_tail) {
    a.rec_tail[slot] = w.last_rec;
    a.rec_term[slot] = escaped ? 0.0 : w.T * terminal + w.dacc;
  }
  w.alive = false;
}

// begin_step (wost.cpp:148-216): false when the walk ends here
__device__ __forceinline__ bool step2_begin(Lane2& w, const WalkArgs& a, bool collect, int& rec) {
  const SceneView& s = a.scene;
  rec = -1;
  CP cd = closest_point(s, w.x, w.y, WG_KIND_DIRICHLET);
  if (cd.seg >= 0 && cd.d <= a.sp.eps) {
    double g = eval_value(s.values[s.seg_value[cd.seg]], cd.px, cd.py);
    w.acc += w.T * g;
    finish2(w, a, false, g, collect);
    return false;
  }
  if (w.depth >= a.sp.max_steps) {
    finish2(w, a, true, 0.0, collect);
    return false;
  }
  if (w.depth > a.sp.rr_depth) {
    double q = smin(1.0, fabs(w.T));
    if (q <= 0.0 || w.rng.uni() >= q) {
      finish2(w, a, false, 0.0, collect);
      return false;
    }
    w.T /= q;
  }
  double dsil = closest_silhouette(s, w.x, w.y);
  double dd = cd.seg >= 0 ? cd.d : dinf();
  if (dd == dinf() && dsil == dinf()) {
    atomicOr(&a.counters[4], 1ull);
    finish2(w, a, true, 0.0, false);
    return false;
  }
  w.R = smin(dd, smax(dsil, a.sp.rmin));
  double contrib = 0.0;
  if (!s.source_zero) {  // sample_source_point, wost.cpp:67-87
    double dx, dy;
    uniform_sample(w.rng, w.on_n, w.nx, w.ny, &dx, &dy);
    double r = greens_radius_2d(w.rng.uni(), w.R);
    double yx = w.x + dx * r, yy = w.y + dy * r;
    Hit h = source_ray_needed(s, r, w.R) ? ray_first_hit(s, w.x, w.y, dx, dy, r, WG_KIND_ALL, -1) : no_hit();
    double wt = h.seg >= 0 ? 0.0 : w.R * w.R / 4.0;
    if (wt != 0.0) {
      double f = 0.0;
      if (bbox_contains(s, yx, yy, 0.0)) f = eval_value(s.source, yx, yy);
      contrib -= wt * f;
    }
  }
  if (s.has_flux) {  // sample_neumann_contrib, wost.cpp:89-109
    double dx, dy;
    uniform_sample(w.rng, w.on_n, w.nx, w.ny, &dx, &dy);
    Hit h = ray_first_hit(s, w.x, w.y, dx, dy, w.R, WG_KIND_NEUMANN, w.seg);
    double add = 0.0;
    if (h.seg >= 0) {
      double hv = eval_value(s.values[s.seg_value[h.seg]], h.px, h.py);
      if (hv != 0.0) {
        double cz = fabs(dx * h.nx + dy * h.ny);
        if (a.sp.clamp_grazing) cz = smax(cz, a.sp.grazing_floor);
        if (cz != 0.0) add = greens_ball_2d(h.t, w.R) * hv * h.t * kTwoPi / cz;
      }
    }
    contrib += add;
  }
  w.acc += w.T * contrib;
  w.dacc += w.T * contrib;
  if (collect && w.rec_ok) {  // trace push (wost.cpp:206-214), chunks of 8 slots
    if (w.rec_left == 0) {
      unsigned long long b = atomicAdd(a.rec_counter, 8ull);
      if (static_cast<int64_t>(b) + 8 > a.rec_capacity) {
        w.rec_ok = false;
        atomicAdd(&a.counters[3], 1ull);
      } else {
        w.rec_base = static_cast<int64_t>(b);
        w.rec_left = 8;
      }
    }
    if (w.rec_ok) {
      rec = static_cast<int>(w.rec_base + (8 - w.rec_left));
      --w.rec_left;
    }
  }
  return true;
}

// record + finish_step (wost.cpp:218-264) along a guided direction
__device__ __forceinline__ void step2_move(Lane2& w, const WalkArgs& a, bool collect, int rec, const Dir2& d) {
  const SceneView& s = a.scene;
  if (rec >= 0) {
    DevRecord r;
    r.x = static_cast<float>(w.x);
    r.y = static_cast<float>(w.y);
    r.nux = static_cast<float>(d.nux);
    r.nuy = static_cast<float>(d.nuy);
    r.nx = static_cast<float>(w.nx);
    r.ny = static_cast<float>(w.ny);
    r.pdf_mis = static_cast<float>(d.pmis);
    r.pdf_g = static_cast<float>(d.pg);
    r.pdf_u = static_cast<float>(d.pu);
    r.c = static_cast<float>(d.sel);
    r.target = 0.0f;
    r.dacc = static_cast<float>(w.dacc);
    w.dacc = 0.0;
    r.thr_q = static_cast<float>(w.T * d.mult);
    r.pad_ = 0.0f;
    r.walk = static_cast<int32_t>(static_cast<int64_t>(w.round) * a.n_points + w.point);
    r.flags = REC_WRITTEN | (w.on_n ? REC_ON_NEUMANN : 0u);
    r.key = Pcg::mix(a.key_seed ^ Pcg::mix((static_cast<uint64_t>(a.point_offset + w.point) << 20) ^
                                           static_cast<uint64_t>(w.depth)));
    r.prev = w.last_rec;
    r.pad2_ = 0;
    a.recs[rec] = r;
    w.last_rec = rec;
  }
  if (d.mult == 0.0) {
    finish2(w, a, false, 0.0, collect);
    return;
  }
  Hit h = ray_first_hit(s, w.x, w.y, d.nux, d.nuy, w.R, WG_KIND_NEUMANN, w.seg);
  if (h.seg >= 0) {
    w.x = h.px;
    w.y = h.py;
    w.on_n = true;
    w.nx = h.nx;
    w.ny = h.ny;
    w.seg = h.seg;
  } else {
    w.x = w.x + d.nux * w.R;
    w.y = w.y + d.nuy * w.R;
    w.on_n = false;
    w.seg = -1;
  }
  w.T *= d.mult;
  ++w.depth;
  if (!bbox_contains(s, w.x, w.y, 1e-9 * s.diag)) finish2(w, a, true, 0.0, collect);
}

struct Wave2 {
  Lane2* lanes;
  Dir2* dirs;
  int32_t* rec;
  uint8_t* state;
  int32_t* queue;
  unsigned int* qlen;
  unsigned long long* next_walk;
  int64_t slots;
};

__global__ void __launch_bounds__(128, 4) wave2_geom_kernel(WalkArgs a, Wave2 v, int parity) {
  const bool collect = a.recs != nullptr;
  const unsigned long long total = static_cast<unsigned long long>(a.n_points) * a.n_rounds;
  unsigned int* qlen = v.qlen + parity;
  unsigned long long started = 0;
  for (int64_t slot = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; slot < v.slots;
       slot += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint8_t st = v.state[slot];
    Lane2 w;
    if (st == SLOT_NEED_MOVE || collect) w = v.lanes[slot];  // record-chunk bookkeeping carries over
    if (st != SLOT_NEED_MOVE) w.alive = false;
    if (st == SLOT_NEED_MOVE) step2_move(w, a, collect, v.rec[slot], v.dirs[slot]);
    bool need = false;
    int rec = -1;
    for (int tries = 0; tries < 4 && !need; ++tries) {
      if (!w.alive) {
        const unsigned long long id = atomicAdd(v.next_walk, 1ull);
        if (id >= total) break;
        lane2_init(w, a, static_cast<int64_t>(id));
        if (!collect) {
          w.rec_base = 0;
          w.rec_left = 0;
        }
        ++started;
      }
      need = step2_begin(w, a, collect, rec);
    }
    if (need) {
      v.lanes[slot] = w;
      v.rec[slot] = rec;
      v.state[slot] = SLOT_NEED_DIR;
      v.queue[atomicAdd(qlen, 1u)] = static_cast<int32_t>(slot);
    } else {
      if (collect) v.lanes[slot] = w;
      v.state[slot] = SLOT_EMPTY;
    }
  }
  for (int o = 16; o > 0; o >>= 1) started += __shfl_down_sync(0xffffffffu, started, o);
  if ((threadIdx.x & 31) == 0 && started) atomicAdd(&a.counters[2], started);
}

// decode + MIS draw of one MLP output row with the tensor path's fp32
// mixture math (wg_mix32.cuh)
__device__ __forceinline__ Dir2 draw2(Lane2& w, const WalkArgs& a, const float* raw) {
  Mix32 m;
  normalize32(raw, m);
  // decode_guiding (wost.cpp:111-122); c in fp64 from the logit so that
  // 1 - c (the defensive uniform weight in p_mis) never rounds to 0
  double sel = sigmoid(static_cast<double>(raw[32]));
  if (a.sp.mode == WG_MODE_GUIDING_ONLY) sel = 1.0;
  else if (a.sp.mode == WG_MODE_FIXED_MIS) sel = a.sp.fixed_c;
  double dnx, dny;
  mis_draw32(w.rng, m, sel, w.on_n, w.nx, w.ny, a.sp.reflect != 0, &dnx, &dny);
  const MisOut o = mis_eval32(m, sel, w.on_n, w.nx, w.ny, a.sp.reflect != 0, dnx, dny);
  return Dir2{o.nx, o.ny, o.pmis, o.pg, o.pu, sel, o.pu / o.pmis};
}

__global__ void __launch_bounds__(128) wave2_dir_kernel(WalkArgs a, Wave2 v, int parity) {
  extern __shared__ __align__(128) unsigned char smem[];
  if (blockIdx.x == 0 && threadIdx.x == 0) v.qlen[parity ^ 1] = 0u;
  const unsigned int n = v.qlen[parity];
  if (static_cast<unsigned int>(blockIdx.x) * 128u >= n) return;
  tc_stage_weights(smem, a.field);
  tc_setup(smem);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  uint32_t phase = 0;
  for (unsigned int t = blockIdx.x; t * 128u < n; t += gridDim.x) {
    const unsigned int row = t * 128u + threadIdx.x;
    const bool live = row < n;
    const int32_t slot = live ? v.queue[row] : 0;
    float in[16], raw[TcLayout::NO];
    Lane2 w;
    if (live) {
      w = v.lanes[slot];
      tc_gather(a.field, w.x, w.y, in);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) in[i] = 0.0f;
    }
    tc_forward(smem, phase, in, raw);
    if (live) {
      v.dirs[slot] = draw2(w, a, raw);
      v.lanes[slot].rng = w.rng;
      v.state[slot] = SLOT_NEED_MOVE;
    }
  }
  tc_teardown(smem);
}

// the drain hand-off (as wave_tail_kernel, wg3_walk_tc.cu): once every walk
// id is out and at most tail_n walks remain, lockstep CTAs finish them (move,
// begin_step, MLP on the tensor cores, draw) with the same step functions,
// taking the next walk of the last queue as rows free up
__global__ void __launch_bounds__(128, 2) wave2_tail_kernel(WalkArgs a, Wave2 v) {
  extern __shared__ __align__(128) unsigned char smem[];
  const unsigned int n = v.qlen[1];
  const unsigned int per = min(128u, (n + gridDim.x - 1) / gridDim.x);
  const unsigned int spread = per * gridDim.x;
  if (static_cast<unsigned int>(blockIdx.x) * per >= n) return;
  tc_stage_weights(smem, a.field);
  tc_setup(smem);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const bool collect = a.recs != nullptr;
  int32_t slot = -1;
  Lane2 w;
  w.alive = false;
  Dir2 d{};
  int rec = -1;
  bool need = false, more = true, first = true;
  uint32_t phase = 0;
  for (;;) {
    if (need) {
      step2_move(w, a, collect, rec, d);
      need = w.alive && step2_begin(w, a, collect, rec);
    }
    while (!need && more) {
      if (slot >= 0) {
        if (collect) v.lanes[slot] = w;  // record-chunk bookkeeping for wave2_close_kernel
        v.state[slot] = SLOT_EMPTY;
        slot = -1;
      }
      unsigned int i;
      if (first) {
        i = blockIdx.x * per + threadIdx.x;
      } else {
        namespace cg = cooperative_groups;
        const cg::coalesced_group g = cg::coalesced_threads();
        unsigned int base = 0;
        if (g.thread_rank() == 0) base = atomicAdd(v.qlen, g.size());
        i = spread + g.shfl(base, 0) + g.thread_rank();
      }
      if (i >= n || (first && threadIdx.x >= per)) {
        more = false;
        break;
      }
      first = false;
      slot = v.queue[i];
      w = v.lanes[slot];
      d = v.dirs[slot];
      rec = v.rec[slot];
      step2_move(w, a, collect, rec, d);
      need = w.alive && step2_begin(w, a, collect, rec);
    }
    if (__syncthreads_count(need) == 0) break;
    float in[16], raw[TcLayout::NO];
    if (need) {
      tc_gather(a.field, w.x, w.y, in);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) in[i] = 0.0f;
    }
    tc_forward(smem, phase, in, raw);
    if (need) d = draw2(w, a, raw);
  }
  if (slot >= 0) {
    if (collect) v.lanes[slot] = w;
    v.state[slot] = SLOT_EMPTY;
  }
  tc_teardown(smem);
}

__global__ void wave2_close_kernel(WalkArgs a, Wave2 v) {
  for (int64_t slot = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; slot < v.slots;
       slot += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const Lane2& w = v.lanes[slot];
    for (int i = 0; i < w.rec_left; ++i) a.recs[w.rec_base + (8 - w.rec_left) + i].flags = 0u;
  }
}

}  // namespace

void wave2_sizes(size_t* lane, size_t* dir) {
  *lane = sizeof(Lane2);
  *dir = sizeof(Dir2);
}

__global__ void wave2_continue_kernel(Wave2 v, unsigned long long total, unsigned int tail_n,
                                      cudaGraphConditionalHandle cond, unsigned long long* launches,
                                      unsigned body_kernels) {
  if (threadIdx.x != 0) return;
  const bool more = v.qlen[1] > tail_n || *v.next_walk < total;
  cudaGraphSetConditional(cond, more ? 1u : 0u);
  atomicAdd(launches, static_cast<unsigned long long>(body_kernels));
}

cudaError_t launch_walks2_wave(const WalkArgs& a, void* lanes, void* dirs, int32_t* rec, uint8_t* state,
                               int32_t* queue, unsigned int* qlen, unsigned long long* next_walk,
                               int64_t slots, int sms, unsigned int* h_qlen, int64_t* launches,
                               cudaStream_t st) {
  Wave2 v{static_cast<Lane2*>(lanes), static_cast<Dir2*>(dirs), rec, state, queue, qlen, next_walk, slots};
  *launches = 0;
  const int smem = static_cast<int>((TcLayout::BYTES + 127) / 128 * 128);
  cudaError_t e = cudaFuncSetAttribute(wave2_dir_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const unsigned long long total = static_cast<unsigned long long>(a.n_points) * a.n_rounds;
  cudaMemsetAsync(v.state, 0, static_cast<size_t>(slots), st);
  cudaMemsetAsync(v.qlen, 0, 2 * sizeof(unsigned int), st);
  cudaMemsetAsync(v.next_walk, 0, sizeof(unsigned long long), st);
  if (a.recs) cudaMemsetAsync(v.lanes, 0, sizeof(Lane2) * static_cast<size_t>(slots), st);
  const int geom_blocks = static_cast<int>((slots + 127) / 128);
  const int dir_blocks = sms * 2;
  // drain hand-off to wave2_tail_kernel (WOSTGPU_WAVE2_TAIL walks left; 0 = off)
  const char* tail_pe = std::getenv("WOSTGPU_WAVE2_TAIL");
  const unsigned int tail_n = static_cast<unsigned int>(tail_pe ? std::atol(tail_pe) : kTail2Default);
  if (tail_n &&
      (e = cudaFuncSetAttribute(wave2_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess)
    return e;
  // device-side iteration loop (as the 3D wavefront, wg3_walk_tc.cu): a CUDA
  // graph while node over a two-iteration body; wave2_continue_kernel sets
  // the condition and counts the body's kernels into counters[8]
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
  if ((e = cudaStreamBeginCaptureToGraph(st, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                         cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
    return fail(e);
  for (int par = 0; par < 2; ++par) {
    wave2_geom_kernel<<<geom_blocks, 128, 0, st>>>(a, v, par);
    wave2_dir_kernel<<<dir_blocks, 128, smem, st>>>(a, v, par);
  }
  wave2_continue_kernel<<<1, 32, 0, st>>>(v, total, tail_n, cond, a.counters + 8, 5u);
  cudaGraph_t captured = nullptr;
  if ((e = cudaStreamEndCapture(st, &captured)) != cudaSuccess) return fail(e);
  if ((e = cudaGraphInstantiate(&exec, graph, 0)) != cudaSuccess) return fail(e);
  if ((e = cudaGraphLaunch(exec, st)) != cudaSuccess) return fail(e);
  cudaGraphExecDestroy(exec);  // released once the launch completes
  cudaGraphDestroy(graph);
  (void)h_qlen;
  if (tail_n) {
    wave2_tail_kernel<<<sms * 2, 128, smem, st>>>(a, v);
    *launches += 1;
  }
  if (a.recs) {
    wave2_close_kernel<<<geom_blocks, 128, 0, st>>>(a, v);
    *launches += 1;
  }
  return cudaGetLastError();
}

}  // namespace wg
