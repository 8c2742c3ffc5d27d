// Guided walk kernel with the guiding-field MLP on the tcgen05 tensor cores.
//
// One CTA = 128 threads = 128 walk slots = one M = 128 UMMA tile. Every step
// of the CTA's walks is split in three phases:
//   A. per thread: refill the slot if its walk ended, then begin_step
//      (epsilon shell, roulette, star radius, source / Neumann terms;
//      proj/src/wost.cpp:148-216) until the walk needs a direction;
//   B. CTA-wide: grid gather on CUDA cores, then the 3-layer MLP as 27
//      single-thread tcgen05.mma issues into TMEM (wg_mlp_tc.cuh);
//   C. per thread: Table-1 normalisation + one-sample MIS / vMF / reflected
//      sampling in fp32 (normalize32 / mis_draw32, wg_mix32.cuh; the
//      selection probability c stays fp64) and finish_step (wost.cpp:218-264).
// Walk state stays in registers; the scene and the split fp16 weights stay in
// shared memory for the whole launch. Statistics go through the same
// [round][point] estimate buffer + Welford pass as the other walk kernels.
#include <cstdio>
#include <cstdlib>

#include "wg_kernels.cuh"
#include "wg_train.cuh"
#include "wg_mix32.cuh"
#include "wg_mlp_tc.cuh"
#include "wg_walk_common.cuh"

// WG_SUBPROF (diagnostic builds only): per-thread clock64 totals of the
// sub-phases of a step, summed over all walks and printed by the last CTA.
#ifdef WG_SUBPROF
__device__ unsigned long long g_sub[16];
__device__ unsigned int g_sub_done;
#define SUB_T(v) long long v = clock64()
#define SUB_ADD(i, t0) (sub[i] += clock64() - (t0))
#define SUB_CNT(i) (++sub[i])
#else
#define SUB_T(v)
#define SUB_ADD(i, t0)
#define SUB_CNT(i)
#endif

namespace wg {

namespace {

struct TLane {
  double x, y, nx, ny, T, acc, R, contrib, rr;
  int seg, depth, rec;
  bool on_n, alive;
  Pcg rng;
  int64_t point;
  int round;
  int64_t rec_base;
  int rec_left, last_rec;
  double dacc;  // accumulator increments since the last record (DevRecord::dacc)
  bool rec_ok;
};

__host__ __device__ __forceinline__ size_t al16(size_t b) { return (b + 15) & ~size_t(15); }

// Tail iterations: once at most kSmallRows slots of a CTA still need a
// direction (the longest walks of a round; most of a round's iterations),
// the CTA evaluates their MLP rows on CUDA cores instead of an M = 128 tile:
// ~1-1.5k cycles against ~6.5k for the three tensor-core layer round trips.
// fp32 weights staged once per launch; layers 1-2 map thread t to hidden unit
// t % 64 for every second row (each weight load reused across rows).
constexpr int kSmallRows = 16;

struct SmallMlp {
  float w1[16][80], b1[64];  // row stride = 16 mod 32: lane pairs read rows k, k+1 conflict-free
  float w2[64][80], b2[64];
  float w3[64][33], b3[36];
  float x[kSmallRows][16];
  float h1[kSmallRows][64], h2[kSmallRows][64];
  float r[kSmallRows][33];
  int slot_count;
};

__device__ __forceinline__ void small_stage(SmallMlp& M, const FieldView& f) {
  for (int e = threadIdx.x; e < 16 * 64; e += blockDim.x) M.w1[e / 64][e % 64] = f.p[f.w1 + e];
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) M.w2[e / 64][e % 64] = f.p[f.w2 + e];
  for (int e = threadIdx.x; e < 64 * 33; e += blockDim.x) M.w3[e / 33][e % 33] = f.p[f.w3 + e];
  for (int e = threadIdx.x; e < 64; e += blockDim.x) {
    M.b1[e] = f.p[f.b1 + e];
    M.b2[e] = f.p[f.b2 + e];
  }
  for (int e = threadIdx.x; e < 33; e += blockDim.x) M.b3[e] = f.p[f.b3 + e];
}

// layers 1-2: thread t -> hidden unit t / 2 over K half t % 2 (interleaved,
// k = 2i + t % 2), halves combined by one shuffle: all 128 threads work on
// every live row with two accumulator chains
template <int K>
__device__ __forceinline__ void small_layer(const float (*w)[80], const float* b, const float* in, int in_stride,
                                            float* out, int n) {
  const int j = threadIdx.x >> 1, s = threadIdx.x & 1;
  for (int r = 0; r < n; ++r) {
    const float* x = in + r * in_stride;
    float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
    for (int i = 0; i < K; i += 4) {
      a0 = fmaf(w[i + s][j], x[i + s], a0);
      a1 = fmaf(w[i + 2 + s][j], x[i + 2 + s], a1);
    }
    float acc = a0 + a1;
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (s == 0) out[r * 64 + j] = fmaxf(acc + b[j], 0.0f);
  }
}

// layer 3: thread t -> output t / 4 (0..31) over K quarter t % 4 (shuffle
// reduced); output 32 by warp 0 with a warp reduction
__device__ __forceinline__ void small_layer3(SmallMlp& M, int n) {
  const int t = threadIdx.x, o = t >> 2, q = t & 3;
  for (int r = 0; r < n; ++r) {
    float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
    for (int kk = 0; kk < 16; kk += 2) {
      a0 = fmaf(M.w3[16 * q + kk][o], M.h2[r][16 * q + kk], a0);
      a1 = fmaf(M.w3[16 * q + kk + 1][o], M.h2[r][16 * q + kk + 1], a1);
    }
    float acc = a0 + a1;
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (q == 0) M.r[r][o] = acc + M.b3[o];
    if (t < 32) {
      float v = fmaf(M.w3[t][32], M.h2[r][t], M.w3[t + 32][32] * M.h2[r][t + 32]);
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o2);
      if (t == 0) M.r[r][32] = v + M.b3[32];
    }
  }
}

// MLP rows 0..n-1 of M.x -> M.r (raw outputs); all threads, barriers inside.
// Rows n..kSmallRows-1 of x / h1 / h2 may hold stale values: they are read
// by the unrolled row loops but never written back.
__device__ __forceinline__ void small_mlp(SmallMlp& M, int n) {
  small_layer<16>(M.w1, M.b1, &M.x[0][0], 16, &M.h1[0][0], n);
  __syncthreads();
  small_layer<64>(M.w2, M.b2, &M.h1[0][0], 64, &M.h2[0][0], n);
  __syncthreads();
  small_layer3(M, n);
  __syncthreads();
}

__device__ __forceinline__ void t_finish(TLane& w, const WalkArgs& a, bool escaped, double terminal,
                                         bool collect) {
  const int64_t slot = static_cast<int64_t>(w.round) * a.n_points + w.point;
  a.est[slot] = escaped ? 0.0 : w.acc;
  a.esc[slot] = escaped ? 1 : 0;
  if (a.steps) a.steps[slot] = w.depth;
  atomicAdd(&a.counters[0], static_cast<unsigned long long>(w.depth));
  if (escaped) atomicAdd(&a.counters[1], 1ull);
  if (collect && a.rec_tail) {  // the walk's end of the record chain (see DevRecord)
    a.rec_tail[slot] = w.last_rec;
    a.rec_term[slot] = escaped ? 0.0 : w.T * terminal + w.dacc;
  }
  w.alive = false;
}

// begin_step (wost.cpp:148-216); false when the walk terminated
__device__ __forceinline__ bool t_begin(TLane& w, const WalkArgs& a, const SceneView& s,
                                        const SmallSegs& ss, bool collect, long long* sub) {
  (void)sub;
  SUB_T(t0);
  CP cd = t_closest(s, ss, w.x, w.y, WG_KIND_DIRICHLET);
  SUB_ADD(0, t0);
  if (cd.seg >= 0 && cd.d <= a.sp.eps) {
    double g = eval_value(s.values[s.seg_value[cd.seg]], cd.px, cd.py);
    w.acc += w.T * g;
    t_finish(w, a, false, g, collect);
    return false;
  }
  if (w.depth >= a.sp.max_steps) {
    t_finish(w, a, true, 0.0, collect);
    return false;
  }
  w.rr = 1.0;
  if (w.depth > a.sp.rr_depth) {
    double q = smin(1.0, fabs(w.T));
    if (q <= 0.0 || w.rng.uni() >= q) {
      t_finish(w, a, false, 0.0, collect);
      return false;
    }
    w.T /= q;
    w.rr = 1.0 / q;
  }
  SUB_T(t1);
  double dsil = s.n_sil <= kSmallScene ? sil_small(s, w.x, w.y) : closest_silhouette(s, w.x, w.y);
  SUB_ADD(1, t1);
  SUB_T(t2);
  double dd = cd.seg >= 0 ? cd.d : dinf();
  if (dd == dinf() && dsil == dinf()) {
    atomicOr(&a.counters[4], 1ull);
    t_finish(w, a, true, 0.0, false);
    return false;
  }
  w.R = smin(dd, smax(dsil, a.sp.rmin));
  double contrib = 0.0;
  if (!s.source_zero) {
    double dx, dy;
    uniform_sample32(w.rng, w.on_n, w.nx, w.ny, &dx, &dy);
    double r = t_greens_radius(w.rng.uni(), w.R);
    double yx = w.x + dx * r, yy = w.y + dy * r;
    Hit h = source_ray_needed(s, r, w.R) ? t_ray(s, ss, w.x, w.y, dx, dy, r, WG_KIND_ALL, -1) : no_hit();
    double wt = h.seg >= 0 ? 0.0 : w.R * w.R / 4.0;
    if (wt != 0.0) {
      double f = 0.0;
      if (bbox_contains(s, yx, yy, 0.0)) f = eval_value(s.source, yx, yy);
      contrib -= wt * f;
    }
  }
  if (s.has_flux) {
    double dx, dy;
    uniform_sample32(w.rng, w.on_n, w.nx, w.ny, &dx, &dy);
    Hit h = t_ray(s, ss, w.x, w.y, dx, dy, w.R, WG_KIND_NEUMANN, w.seg);
    double add = 0.0;
    if (h.seg >= 0) {
      double hv = eval_value(s.values[s.seg_value[h.seg]], h.px, h.py);
      if (hv != 0.0) {
        double cz = fabs(dx * h.nx + dy * h.ny);
        if (a.sp.clamp_grazing) cz = smax(cz, a.sp.grazing_floor);
        if (cz != 0.0) add = (h.t <= 0.0 ? dinf() : log(w.R / h.t) / kTwoPi) * hv * h.t * kTwoPi / cz;
      }
    }
    contrib += add;
  }
  w.acc += w.T * contrib;
  w.dacc += w.T * contrib;
  w.contrib = contrib;
  SUB_ADD(2, t2);
  w.rec = -1;
  if (collect && w.rec_ok) {
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
      w.rec = static_cast<int>(w.rec_base + (8 - w.rec_left));
      --w.rec_left;
    }
  }
  return true;
}

}  // namespace

// The CTA's 128 walks share one M = 128 tile and step in lockstep (CTA
// barrier per step).
__device__ __forceinline__ void walk_tc_body(const WalkArgs& a, unsigned char* smem) {
  unsigned char* tc = smem;  // TcLayout block first (128-B aligned)
  SceneView s = a.scene;
  if (a.scene_smem_bytes > 0) {
    unsigned char* p =
        smem + al16(TcLayout::BYTES + (a.small_mlp ? sizeof(SmallMlp) : 0));
    size_t off = 0;
    auto carve = [&](size_t bytes) {
      unsigned char* q = p + off;
      off += al16(bytes);
      return q;
    };
    Node* nodes = reinterpret_cast<Node*>(carve(sizeof(Node) * s.n_nodes));
    Seg* segs = reinterpret_cast<Seg*>(carve(sizeof(Seg) * s.n_segs));
    SilVertex* sil = reinterpret_cast<SilVertex*>(carve(sizeof(SilVertex) * s.n_sil));
    double* sn = reinterpret_cast<double*>(carve(sizeof(double) * 2 * s.n_sil_normals));
    for (int i = threadIdx.x; i < s.n_nodes; i += blockDim.x) nodes[i] = a.scene.nodes[i];
    for (int i = threadIdx.x; i < s.n_segs; i += blockDim.x) segs[i] = a.scene.segs[i];
    for (int i = threadIdx.x; i < s.n_sil; i += blockDim.x) sil[i] = a.scene.sil[i];
    for (int i = threadIdx.x; i < 2 * s.n_sil_normals; i += blockDim.x) sn[i] = a.scene.sil_n[i];
    s.nodes = nodes;
    s.segs = segs;
    s.sil = sil;
    s.sil_n = sn;
  }
  // per-kind segment lists of small scenes (BVH leaf order)
  __shared__ Seg seg_lists[2 * kSmallScene];
  __shared__ int seg_counts[2];
  if (s.n_segs <= kSmallScene && threadIdx.x == 0) {
    int nd = 0, nn = 0;
    for (int i = 0; i < s.n_segs; ++i) {
      const Seg g = s.segs[i];
      if (g.kind == WG_DIRICHLET) seg_lists[nd++] = g;
      else seg_lists[kSmallScene + nn++] = g;
    }
    seg_counts[0] = nd;
    seg_counts[1] = nn;
  }
  SmallSegs ss{seg_lists, seg_lists + kSmallScene, 0, 0};
  SmallMlp& small = *reinterpret_cast<SmallMlp*>(smem + TcLayout::BYTES);
  tc_fetch_weights(tc, a.wblob);
  tc_setup(tc);
  if (a.small_mlp) small_stage(small, a.field);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  tc_wait_weights(tc);
  ss.nd = seg_counts[0];
  ss.nn = seg_counts[1];

  const bool collect = a.recs != nullptr;
  const int64_t total = a.n_points * static_cast<int64_t>(a.n_rounds);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  // walk ids interleaved over the CTAs (id = thread * grid + block): a round
  // with fewer walks than slots spreads evenly over every SM instead of
  // filling the first CTAs (a CTA lasts as long as its longest walk)
  int64_t next = static_cast<int64_t>(threadIdx.x) * gridDim.x + blockIdx.x;
  const double pad = 1e-9 * s.diag;
  const FieldView& fv = a.field;
  uint32_t phase = 0;
  TLane w;
  w.alive = false;
  w.rec_base = 0;
  w.rec_left = 0;
  int64_t walks_done = 0;

  long long t_iter = a.phase_prof ? clock64() : 0;
  long long bpa[3] = {0, 0, 0};
  long long sub[12] = {};
  for (;;) {
    if (a.phase_prof) {  // phase C of the previous iteration ends here
      long long t_top = clock64();
      if (threadIdx.x == 0) a.phase_prof[8 * blockIdx.x + 2] += static_cast<unsigned long long>(t_top - t_iter);
      t_iter = t_top;
    }
    if (a.small_mlp && threadIdx.x == 0) small.slot_count = 0;  // consumed after the phase-A barrier
    // ---- phase A: every slot advances to a walk that needs a direction
    bool need = false;
    for (;;) {
      if (!w.alive) {
        if (next >= total) break;
        w.round = static_cast<int>(next / a.n_points);
        w.point = next - static_cast<int64_t>(w.round) * a.n_points;
        w.x = a.points[2 * w.point];
        w.y = a.points[2 * w.point + 1];
        w.nx = w.ny = 0.0;
        w.on_n = false;
        w.seg = -1;
        w.T = 1.0;
        w.acc = 0.0;
        w.R = 0.0;
        w.depth = 0;
        w.alive = true;
        w.rng = Pcg::walk(a.seed, static_cast<uint64_t>(a.point_offset + w.point),
                          a.wpp_first + static_cast<uint64_t>(w.round));
        w.last_rec = -1;
        w.dacc = 0.0;
        w.rec_ok = true;
        next += stride;
        ++walks_done;
      }
      if (t_begin(w, a, s, ss, collect, sub)) {
        need = true;
        break;
      }
    }
    int active = 0;
    {
      active = __syncthreads_count(need);
      if (active == 0) break;
      // tail handoff (WalkArgs::spill): a few live walks left and no fresh
      // ones; a warp per walk finishes them with lower step latency
      if (a.spill_rows > 0 && active <= a.spill_rows && !__syncthreads_or(next < total)) {
        if (need) {
          SpillLane& o = a.spill[atomicAdd(&a.counters[7], 1ull)];
          o.x = w.x;
          o.y = w.y;
          o.nx = w.nx;
          o.ny = w.ny;
          o.T = w.T;
          o.acc = w.acc;
          o.dacc = w.dacc;
          o.R = w.R;
          o.point = w.point;
          o.rec_base = w.rec_base;
          o.rng = w.rng;
          o.seg = w.seg;
          o.depth = w.depth;
          o.rec = w.rec;
          o.round = w.round;
          o.rec_left = w.rec_left;
          o.last_rec = w.last_rec;
          o.on_n = w.on_n;
          o.rec_ok = w.rec_ok;
          w.rec_left = 0;  // the record block travels with the walk
        }
        break;
      }
    }
    long long t_b = a.phase_prof ? clock64() : 0;
    if (a.phase_prof && threadIdx.x == 0) {
      a.phase_prof[8 * blockIdx.x + 0] += static_cast<unsigned long long>(t_b - t_iter);
      a.phase_prof[8 * blockIdx.x + 3] += 1;
    }

    // ---- phase B: guiding-field MLP for the whole tile on the tensor cores
    SUB_T(tg);
    long long t_g = a.phase_prof ? clock64() : 0;
    float xin[TcLayout::NIN];
    if (need) {
      tc_gather(fv, w.x, w.y, xin);
    } else {
#pragma unroll
      for (int i = 0; i < TcLayout::NIN; ++i) xin[i] = 0.0f;
    }
    if (a.phase_prof) t_g = clock64() - t_g;
    SUB_ADD(3, tg);
    SUB_T(tb);
    float raw[TcLayout::NO];
    if (a.small_mlp && active <= kSmallRows) {  // tail iteration: CUDA-core rows (SmallMlp)
      int slot = -1;
      if (need) {
        slot = atomicAdd(&small.slot_count, 1);
#pragma unroll
        for (int i = 0; i < 16; ++i) small.x[slot][i] = xin[i];
      }
      __syncthreads();
      long long t_s = a.phase_prof ? clock64() : 0;
      small_mlp(small, active);
      if (a.phase_prof && threadIdx.x == 0) {
        a.phase_prof[8 * blockIdx.x + 7] += static_cast<unsigned long long>(clock64() - t_s);
        a.phase_prof[8 * blockIdx.x + 6] += 1ull << 40;  // small-path iteration count (high bits)
      }
      if (need)
#pragma unroll
        for (int i = 0; i < TcLayout::NO; ++i) raw[i] = small.r[slot][i];
    } else {
      tc_forward(tc, phase, xin, raw, a.phase_prof ? bpa : nullptr);
    }
    if (a.phase_prof && threadIdx.x == 0) {
      a.phase_prof[8 * blockIdx.x + 4] += static_cast<unsigned long long>(bpa[0]);
      a.phase_prof[8 * blockIdx.x + 6] += static_cast<unsigned long long>(bpa[1]);
      a.phase_prof[8 * blockIdx.x + 5] += static_cast<unsigned long long>(t_g);
    }
    bpa[0] = bpa[1] = bpa[2] = 0;
    if (a.phase_prof) {
      long long t_c = clock64();
      if (threadIdx.x == 0) a.phase_prof[8 * blockIdx.x + 1] += static_cast<unsigned long long>(t_c - t_b);
      t_iter = t_c;  // phase C is charged to the next iteration's phase A slot
    }
    SUB_ADD(4, tb);
    if (!need) continue;
    SUB_CNT(11);

    // ---- phase C: decode + sample + move (wost.cpp:111-146, 218-264)
    SUB_T(tn);
    Mix32 m;
    normalize32(raw, m);
    SUB_ADD(5, tn);
    SUB_T(ts);
    // the selection probability in fp64 from the logit (sphdist.cpp:280-283):
    // an fp32 sigmoid rounds to exactly 1 above ~16.6, which would drop the
    // defensive (1 - c) p_u term from p_mis and leave p_u / p_mis unbounded
    double sel = sigmoid(static_cast<double>(raw[32]));
    if (a.sp.mode == WG_MODE_GUIDING_ONLY) sel = 1.0;
    else if (a.sp.mode == WG_MODE_FIXED_MIS) sel = a.sp.fixed_c;
    double dnx, dny;
    mis_draw32(w.rng, m, sel, w.on_n, w.nx, w.ny, a.sp.reflect != 0, &dnx, &dny);
    SUB_ADD(9, ts);
    SUB_T(te);
    MisOut o = mis_eval32(m, sel, w.on_n, w.nx, w.ny, a.sp.reflect != 0, dnx, dny);
    SUB_ADD(10, te);
    double mult = o.pu / o.pmis;
    SUB_ADD(6, ts);
    SUB_T(tr);
    if (w.rec >= 0) {
      DevRecord r;
      r.x = static_cast<float>(w.x);
      r.y = static_cast<float>(w.y);
      r.nux = static_cast<float>(o.nx);
      r.nuy = static_cast<float>(o.ny);
      r.nx = static_cast<float>(w.nx);
      r.ny = static_cast<float>(w.ny);
      r.pdf_mis = static_cast<float>(o.pmis);
      r.pdf_g = static_cast<float>(o.pg);
      r.pdf_u = static_cast<float>(o.pu);
      r.c = static_cast<float>(sel);
      r.target = 0.0f;
      r.dacc = static_cast<float>(w.dacc);
      r.thr_q = static_cast<float>(w.T * mult);
      r.pad_ = 0.0f;
      r.walk = static_cast<int32_t>(static_cast<int64_t>(w.round) * a.n_points + w.point);
      r.flags = REC_WRITTEN | (w.on_n ? REC_ON_NEUMANN : 0u);
      r.key = Pcg::mix(a.key_seed ^ Pcg::mix((static_cast<uint64_t>(a.point_offset + w.point) << 20) ^
                                             static_cast<uint64_t>(w.depth)));
      r.prev = w.last_rec;
      r.pad2_ = 0;
      a.recs[w.rec] = r;
      w.last_rec = w.rec;
      w.dacc = 0.0;
    }
    SUB_ADD(7, tr);
    if (mult == 0.0) {
      t_finish(w, a, false, 0.0, collect);
      continue;
    }
    SUB_T(th);
    Hit h = t_ray(s, ss, w.x, w.y, o.nx, o.ny, w.R, WG_KIND_NEUMANN, w.seg);
    SUB_ADD(8, th);
    if (h.seg >= 0) {
      w.x = h.px;
      w.y = h.py;
      w.on_n = true;
      w.nx = h.nx;
      w.ny = h.ny;
      w.seg = h.seg;
    } else {
      w.x = w.x + o.nx * w.R;
      w.y = w.y + o.ny * w.R;
      w.on_n = false;
      w.seg = -1;
    }
    w.T *= mult;
    ++w.depth;
    if (!bbox_contains(s, w.x, w.y, pad)) t_finish(w, a, true, 0.0, collect);
  }
  if (collect)
    for (int i = 0; i < w.rec_left; ++i) a.recs[w.rec_base + (8 - w.rec_left) + i].flags = 0u;
  unsigned long long wd = static_cast<unsigned long long>(walks_done);
  for (int o = 16; o > 0; o >>= 1) wd += __shfl_down_sync(0xffffffffu, wd, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&a.counters[2], wd);
#ifdef WG_SUBPROF
  for (int i = 0; i < 12; ++i) atomicAdd(&g_sub[i], static_cast<unsigned long long>(sub[i]));
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&g_sub_done, 1u) == gridDim.x - 1) {
      __threadfence();
      double n = static_cast<double>(g_sub[11] > 0 ? g_sub[11] : 1);
      printf("[sub] steps %.0f cyc/step: cp %.0f sil %.0f begin_rest %.0f gather %.0f mlp %.0f norm %.0f "
             "sample %.0f (draw %.0f pdf %.0f) rec %.0f ray %.0f\n",
             n, g_sub[0] / n, g_sub[1] / n, g_sub[2] / n, g_sub[3] / n, g_sub[4] / n, g_sub[5] / n,
             g_sub[6] / n, g_sub[9] / n, g_sub[10] / n, g_sub[7] / n, g_sub[8] / n);
      for (int i = 0; i < 16; ++i) g_sub[i] = 0;
      g_sub_done = 0;
    }
  }
#endif
  tc_teardown(tc);
}

__global__ void __launch_bounds__(128, 1) walk_kernel_tc(WalkArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  walk_tc_body(a, smem);
}

// GuidingField::eval_batch on the tensor cores: persistent CTAs over 128-point tiles
__global__ void __launch_bounds__(128) field_eval_tc_kernel(FieldView f, int64_t n, const double* xy,
                                                            double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  tc_stage_weights(smem, f);
  tc_setup(smem);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  uint32_t phase = 0;
  const int64_t tiles = (n + 127) / 128;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    int64_t i = t * 128 + threadIdx.x;
    float xin[16], o[33];
    if (i < n) tc_gather(f, xy[2 * i], xy[2 * i + 1], xin);
    else
      for (int k = 0; k < 16; ++k) xin[k] = 0.0f;
    tc_forward(smem, phase, xin, o);
    if (i < n)
      for (int j = 0; j < 33; ++j) out[i * 33 + j] = o[j];
  }
  tc_teardown(smem);
}

// lockstep 128-walk CTAs (a warp-independent variant with per-warp M = 128
// MMAs measured slower on cfg 2, 0.85 vs 1.2 ms per round: 4x the tensor /
// smem traffic, and the waiting warps' mbarrier polling slows the running
// ones)
int walk_tc_block() { return 128; }

// ---- diagnostics of the fp32 mixture math (wostgpu_mixture32_*)
__global__ void mix32_pdf_kernel(const float* raw, int64_t n, const double* nu, double* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float r[33];
  for (int j = 0; j < 33; ++j) r[j] = raw[i * 33 + j];
  Mix32 m;
  normalize32(r, m);
  out[2 * i] = mixture_pdf32(m, nu[2 * i], nu[2 * i + 1]);
  out[2 * i + 1] = m.c;
}

__global__ void mix32_sample_kernel(const float* raw, int64_t n, uint64_t seed, double* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float r[33];
  for (int j = 0; j < 33; ++j) r[j] = raw[j];
  Mix32 m;
  normalize32(r, m);
  Pcg rng = Pcg::walk(seed, static_cast<uint64_t>(i), 0);
  mixture_sample32(rng, m, &out[2 * i], &out[2 * i + 1]);
}

cudaError_t launch_mix32_pdf(const float* raw, int64_t n, const double* nu, double* out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  mix32_pdf_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, st>>>(raw, n, nu, out);
  return cudaGetLastError();
}

cudaError_t launch_mix32_sample(const float* raw, int64_t n, uint64_t seed, double* out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  mix32_sample_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, st>>>(raw, n, seed, out);
  return cudaGetLastError();
}

int walk_tc_smem(const WalkArgs& a) {
  size_t tile = TcLayout::BYTES + (a.small_mlp ? sizeof(SmallMlp) : 0);
  return static_cast<int>(al16(tile) + (a.scene_smem_bytes > 0 ? al16(a.scene_smem_bytes) : 0));
}

int walk_tc_blocks_per_sm(int smem) {
  int n = 0;
  cudaFuncSetAttribute(walk_kernel_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, walk_kernel_tc, walk_tc_block(), smem);
  // 512 TMEM columns per SM: 128 per lockstep CTA
  const int tmem_cap = 4;
  return n < tmem_cap ? n : tmem_cap;
}

cudaError_t launch_walks_tc(const WalkArgs& a, int blocks, cudaStream_t st) {
  int smem = walk_tc_smem(a);
  cudaError_t e = cudaFuncSetAttribute(walk_kernel_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  walk_kernel_tc<<<blocks, walk_tc_block(), smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_field_eval_tc(const FieldView& f, int64_t n, const double* xy, double* out,
                                 int sm_count, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  int smem = static_cast<int>(al16(TcLayout::BYTES));
  cudaError_t e = cudaFuncSetAttribute(field_eval_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int64_t tiles = (n + 127) / 128;
  int blocks = static_cast<int>(tiles < sm_count * 2 ? tiles : sm_count * 2);
  field_eval_tc_kernel<<<blocks, 128, smem, st>>>(f, n, xy, out);
  return cudaGetLastError();
}

}  // namespace wg
