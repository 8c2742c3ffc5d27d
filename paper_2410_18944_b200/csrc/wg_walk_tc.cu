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
//      sampling in fp64 (wg_sphdist.cuh) and finish_step (wost.cpp:218-264).
// Walk state stays in registers; the scene and the split fp16 weights stay in
// shared memory for the whole launch. Statistics go through the same
// [round][point] estimate buffer + Welford pass as the other walk kernels.
#include "wg_kernels.cuh"
#include "wg_train.cuh"
#include "wg_mix32.cuh"
#include "wg_mlp_tc.cuh"

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
  bool rec_ok;
};

__host__ __device__ __forceinline__ size_t al16(size_t b) { return (b + 15) & ~size_t(15); }

__device__ __forceinline__ void t_finish(TLane& w, const WalkArgs& a, bool escaped, double terminal,
                                         bool collect) {
  const int64_t slot = static_cast<int64_t>(w.round) * a.n_points + w.point;
  a.est[slot] = escaped ? 0.0 : w.acc;
  a.esc[slot] = escaped ? 1 : 0;
  if (a.steps) a.steps[slot] = w.depth;
  atomicAdd(&a.counters[0], static_cast<unsigned long long>(w.depth));
  if (escaped) atomicAdd(&a.counters[1], 1ull);
  (void)terminal;  // targets are formed later from (est, P, Q): see DevRecord
  (void)collect;
  w.alive = false;
}

__device__ double t_greens_radius(double u, double R) {  // wost.cpp:37-65, d = 2
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

// begin_step (wost.cpp:148-216); false when the walk terminated
__device__ __forceinline__ bool t_begin(TLane& w, const WalkArgs& a, const SceneView& s, bool collect) {
  CP cd = closest_point(s, w.x, w.y, WG_KIND_DIRICHLET);
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
  double dsil = closest_silhouette(s, w.x, w.y);
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
    uniform_sample(w.rng, w.on_n, w.nx, w.ny, &dx, &dy);
    double r = t_greens_radius(w.rng.uni(), w.R);
    double yx = w.x + dx * r, yy = w.y + dy * r;
    Hit h = ray_first_hit(s, w.x, w.y, dx, dy, r, WG_KIND_ALL, -1);
    double wt = h.seg >= 0 ? 0.0 : w.R * w.R / 4.0;
    if (wt != 0.0) {
      double f = 0.0;
      if (bbox_contains(s, yx, yy, 0.0)) f = eval_value(s.source, yx, yy);
      contrib -= wt * f;
    }
  }
  if (s.has_flux) {
    double dx, dy;
    uniform_sample(w.rng, w.on_n, w.nx, w.ny, &dx, &dy);
    Hit h = ray_first_hit(s, w.x, w.y, dx, dy, w.R, WG_KIND_NEUMANN, w.seg);
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
  w.contrib = contrib;
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

__global__ void __launch_bounds__(128) walk_kernel_tc(WalkArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* tc = smem;  // TcLayout block first (128-B aligned)
  SceneView s = a.scene;
  if (a.scene_smem_bytes > 0) {
    unsigned char* p = smem + al16(TcLayout::BYTES);
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
  tc_stage_weights(tc, a.field);
  tc_setup(tc);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();

  const bool collect = a.recs != nullptr;
  const int64_t total = a.n_points * static_cast<int64_t>(a.n_rounds);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t next = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const double pad = 1e-9 * s.diag;
  const FieldView& fv = a.field;
  uint32_t phase = 0;
  TLane w;
  w.alive = false;
  w.rec_base = 0;
  w.rec_left = 0;
  int64_t walks_done = 0;

  long long t_iter = a.phase_prof ? clock64() : 0;
  for (;;) {
    if (a.phase_prof) {  // phase C of the previous iteration ends here
      long long t_top = clock64();
      if (threadIdx.x == 0) a.phase_prof[4 * blockIdx.x + 2] += static_cast<unsigned long long>(t_top - t_iter);
      t_iter = t_top;
    }
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
        w.rec_ok = true;
        next += stride;
        ++walks_done;
      }
      if (t_begin(w, a, s, collect)) {
        need = true;
        break;
      }
    }
    if (!__syncthreads_or(need)) break;
    long long t_b = a.phase_prof ? clock64() : 0;
    if (a.phase_prof && threadIdx.x == 0) {
      a.phase_prof[4 * blockIdx.x + 0] += static_cast<unsigned long long>(t_b - t_iter);
      a.phase_prof[4 * blockIdx.x + 3] += 1;
    }

    // ---- phase B: guiding-field MLP for the whole tile on the tensor cores
    float xin[TcLayout::NIN];
    if (need) {
      tc_gather(fv, w.x, w.y, xin);
    } else {
#pragma unroll
      for (int i = 0; i < TcLayout::NIN; ++i) xin[i] = 0.0f;
    }
    float raw[TcLayout::NO];
    tc_forward(tc, phase, xin, raw);
    if (a.phase_prof) {
      long long t_c = clock64();
      if (threadIdx.x == 0) a.phase_prof[4 * blockIdx.x + 1] += static_cast<unsigned long long>(t_c - t_b);
      t_iter = t_c;  // phase C is charged to the next iteration's phase A slot
    }
    if (!need) continue;

    // ---- phase C: decode + sample + move (wost.cpp:111-146, 218-264)
    Mix32 m;
    normalize32(raw, m);
    double sel = m.c;
    if (a.sp.mode == WG_MODE_GUIDING_ONLY) sel = 1.0;
    else if (a.sp.mode == WG_MODE_FIXED_MIS) sel = a.sp.fixed_c;
    MisOut o = mis_sample32(w.rng, m, sel, w.on_n, w.nx, w.ny, a.sp.reflect != 0);
    double mult = o.pu / o.pmis;
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
      r.acc_p = static_cast<float>(w.acc);
      r.thr_q = static_cast<float>(w.T * mult);
      r.pad_ = 0.0f;
      r.walk = static_cast<int32_t>(static_cast<int64_t>(w.round) * a.n_points + w.point);
      r.flags = REC_WRITTEN | (w.on_n ? REC_ON_NEUMANN : 0u);
      r.key = Pcg::mix(a.key_seed ^ Pcg::mix((static_cast<uint64_t>(a.point_offset + w.point) << 20) ^
                                             static_cast<uint64_t>(w.depth)));
      a.recs[w.rec] = r;
      w.last_rec = w.rec;
    }
    if (mult == 0.0) {
      t_finish(w, a, false, 0.0, collect);
      continue;
    }
    Hit h = ray_first_hit(s, w.x, w.y, o.nx, o.ny, w.R, WG_KIND_NEUMANN, w.seg);
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
  tc_teardown(tc);
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

int walk_tc_smem(const WalkArgs& a) {
  return static_cast<int>(al16(TcLayout::BYTES) + (a.scene_smem_bytes > 0 ? al16(a.scene_smem_bytes) : 0));
}

int walk_tc_blocks_per_sm(int smem) {
  int n = 0;
  cudaFuncSetAttribute(walk_kernel_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, walk_kernel_tc, 128, smem);
  // 4 x 128 TMEM columns per SM
  return n < 4 ? n : 4;
}

cudaError_t launch_walks_tc(const WalkArgs& a, int blocks, cudaStream_t st) {
  int smem = walk_tc_smem(a);
  cudaError_t e = cudaFuncSetAttribute(walk_kernel_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  walk_kernel_tc<<<blocks, 128, smem, st>>>(a);
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
