// Walk-on-stars walk kernel and the batched geometry / field query kernels.
//
// One CUDA thread owns one walk slot and refills it from a grid-strided walk
// index space (round-major: id = r * n_points + point) as soon as its walk
// terminates, so lanes of a warp stay busy across walks of different length.
// Per-walk state lives in registers for the whole walk; the scene (BVH nodes,
// segments, silhouette vertices) and the MLP weights are staged once per CTA
// in shared memory. Estimates go to an [n_rounds][n_points] buffer and a
// second kernel pushes them into the Welford accumulators in wpp order, so
// statistics are bit-identical to n_rounds sequential solve_batch calls
// (proj/src/wost.cpp:290-384).
#include <cstdio>

#include "wg_kernels.cuh"
#include "wg_train.cuh"
#include "wg_sphdist.cuh"

namespace wg {

// ---------------------------------------------------------------- staging
__device__ __forceinline__ SceneView stage_scene(const SceneView& g, int smem_bytes,
                                                 unsigned char* smem) {
  if (smem_bytes <= 0) return g;
  SceneView s = g;
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    unsigned char* p = smem + off;
    off += (bytes + 15) & ~size_t(15);
    return p;
  };
  Node* nodes = reinterpret_cast<Node*>(carve(sizeof(Node) * g.n_nodes));
  Seg* segs = reinterpret_cast<Seg*>(carve(sizeof(Seg) * g.n_segs));
  SilVertex* sil = reinterpret_cast<SilVertex*>(carve(sizeof(SilVertex) * g.n_sil));
  double* sn = reinterpret_cast<double*>(carve(sizeof(double) * 2 * g.n_sil_normals));
  for (int i = threadIdx.x; i < g.n_nodes; i += blockDim.x) nodes[i] = g.nodes[i];
  for (int i = threadIdx.x; i < g.n_segs; i += blockDim.x) segs[i] = g.segs[i];
  for (int i = threadIdx.x; i < g.n_sil; i += blockDim.x) sil[i] = g.sil[i];
  for (int i = threadIdx.x; i < 2 * g.n_sil_normals; i += blockDim.x) sn[i] = g.sil_n[i];
  s.nodes = nodes;
  s.segs = segs;
  s.sil = sil;
  s.sil_n = sn;
  return s;
}

__host__ __device__ inline size_t align16(size_t b) { return (b + 15) & ~size_t(15); }

// ---------------------------------------------------------------- walks
struct Lane {
  double x, y, nx, ny, T, acc, R;
  int seg, depth;
  bool on_n, alive;
  Pcg rng;
  int64_t point;  // local point index
  int round;
  // records
  int64_t rec_base;
  int rec_left;
  int last_rec;
  double dacc;  // accumulator increments since the last record (DevRecord::dacc)
  bool rec_ok;
};

__device__ __forceinline__ void lane_init(Lane& w, const WalkArgs& a, int64_t id) {
  w.round = static_cast<int>(id / a.n_points);
  w.point = id - static_cast<int64_t>(w.round) * a.n_points;
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
  // Rng::for_walk(seed, global point index, wpp index), rng.hpp:28-32
  w.rng = Pcg::walk(a.seed, static_cast<uint64_t>(a.point_offset + w.point),
                    a.wpp_first + static_cast<uint64_t>(w.round));
  w.last_rec = -1;
  w.dacc = 0.0;
  w.rec_ok = true;
}

// greens ball (wost.cpp:27-35) and the radial inverse CDF (wost.cpp:37-65)
__device__ __forceinline__ double greens_ball2(double r, double R) {
  if (r <= 0.0) return dinf();
  return log(R / r) / kTwoPi;
}
__device__ double greens_radius2(double u, double R) {
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

__device__ __forceinline__ void finish_walk(Lane& w, const WalkArgs& a, bool escaped,
                                            double terminal, bool collect) {
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

template <bool GUIDED, int IN, int HID, int OD, int K>
__global__ void __launch_bounds__(128) walk_kernel(WalkArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SceneView s = stage_scene(a.scene, a.scene_smem_bytes, smem);
  const float* mlp = nullptr;
  if (GUIDED) {
    float* m = reinterpret_cast<float*>(smem + align16(a.scene_smem_bytes > 0 ? a.scene_smem_bytes : 0));
    for (int i = threadIdx.x; i < a.field.mlp_count; i += blockDim.x) m[i] = a.field.p[a.field.w1 + i];
    mlp = m;
  }
  __syncthreads();

  const bool collect = a.recs != nullptr;
  const int64_t total = a.n_points * static_cast<int64_t>(a.n_rounds);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t next = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const double eps = a.sp.eps, rmin = a.sp.rmin;
  const double pad = 1e-9 * s.diag;
  Lane w;
  w.alive = false;
  w.rec_base = 0;
  w.rec_left = 0;
  int64_t walks_done = 0;

  for (;;) {
    if (!w.alive) {
      if (next >= total) break;
      lane_init(w, a, next);
      next += stride;
      ++walks_done;
    }
    // ---------------- begin_step (wost.cpp:148-216)
    CP cd = closest_point(s, w.x, w.y, WG_KIND_DIRICHLET);
    if (cd.seg >= 0 && cd.d <= eps) {
      double g = eval_value(s.values[s.seg_value[cd.seg]], cd.px, cd.py);
      w.acc += w.T * g;
      finish_walk(w, a, false, g, collect);
      continue;
    }
    if (w.depth >= a.sp.max_steps) {
      finish_walk(w, a, true, 0.0, collect);
      continue;
    }
    double rr = 1.0;
    if (w.depth > a.sp.rr_depth) {  // Russian roulette, wost.cpp:169-180
      double q = smin(1.0, fabs(w.T));
      if (q <= 0.0 || w.rng.uni() >= q) {
        finish_walk(w, a, false, 0.0, collect);
        continue;
      }
      w.T /= q;
      rr = 1.0 / q;
    }
    double dsil = closest_silhouette(s, w.x, w.y);
    double dd = cd.seg >= 0 ? cd.d : dinf();
    if (dd == dinf() && dsil == dinf()) {  // SceneError, wost.cpp:184-186
      atomicOr(&a.counters[4], 1ull);
      finish_walk(w, a, true, 0.0, false);
      continue;
    }
    w.R = smin(dd, smax(dsil, rmin));
    double contrib = 0.0;
    if (!s.source_zero) {  // sample_source_point, wost.cpp:67-87
      double dx, dy;
      uniform_sample(w.rng, w.on_n, w.nx, w.ny, &dx, &dy);
      double r = greens_radius2(w.rng.uni(), w.R);
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
          if (cz != 0.0) add = greens_ball2(h.t, w.R) * hv * h.t * kTwoPi / cz;
        }
      }
      contrib += add;
    }
    w.acc += w.T * contrib;
    w.dacc += w.T * contrib;

    int rec = -1;
    if (collect && w.rec_ok) {  // trace push (wost.cpp:206-214)
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

    // ---------------- decode_guiding + finish_step (wost.cpp:111-146, 218-264)
    double nux, nuy, pmis, pg, pu, sel, mult;
    if (GUIDED) {
      Mix m;
      {
        float out[OD ? OD : 256];
        field_eval_exact<IN, HID, OD>(a.field, mlp, w.x, w.y, out);
        normalize2<K>(out, a.field.k, m);
      }
      if (a.sp.mode == WG_MODE_GUIDING_ONLY) m.c = 1.0;
      else if (a.sp.mode == WG_MODE_FIXED_MIS) m.c = a.sp.fixed_c;
      MisOut o = mis_sample(w.rng, m, w.on_n, w.nx, w.ny, a.sp.reflect != 0);
      nux = o.nx;
      nuy = o.ny;
      pmis = o.pmis;
      pg = o.pg;
      pu = o.pu;
      sel = m.c;
      mult = pu / pmis;
    } else {
      uniform_sample(w.rng, w.on_n, w.nx, w.ny, &nux, &nuy);
      pu = uniform_pdf(w.on_n, nux, nuy, w.nx, w.ny);
      pmis = pu;
      pg = 0.0;
      sel = 0.0;
      mult = 1.0;
    }
    if (rec >= 0) {
      DevRecord r;
      r.x = static_cast<float>(w.x);
      r.y = static_cast<float>(w.y);
      r.nux = static_cast<float>(nux);
      r.nuy = static_cast<float>(nuy);
      r.nx = static_cast<float>(w.nx);
      r.ny = static_cast<float>(w.ny);
      r.pdf_mis = static_cast<float>(pmis);
      r.pdf_g = static_cast<float>(pg);
      r.pdf_u = static_cast<float>(pu);
      r.c = static_cast<float>(sel);
      r.target = 0.0f;
      r.dacc = static_cast<float>(w.dacc);
      w.dacc = 0.0;
      r.thr_q = static_cast<float>(GUIDED ? w.T * mult : w.T);
      r.pad_ = 0.0f;
      r.walk = static_cast<int32_t>(static_cast<int64_t>(w.round) * a.n_points + w.point);
      r.flags = REC_WRITTEN | (w.on_n ? REC_ON_NEUMANN : 0u);
      (void)rr;
      r.key = Pcg::mix(a.key_seed ^ Pcg::mix((static_cast<uint64_t>(a.point_offset + w.point) << 20) ^
                                             static_cast<uint64_t>(w.depth)));
      r.prev = w.last_rec;
      r.pad2_ = 0;
      a.recs[rec] = r;
      w.last_rec = rec;
    }
    if (mult == 0.0) {  // sampled into the invalid half space
      finish_walk(w, a, false, 0.0, collect);
      continue;
    }
    Hit h = ray_first_hit(s, w.x, w.y, nux, nuy, w.R, WG_KIND_NEUMANN, w.seg);
    if (h.seg >= 0) {
      w.x = h.px;
      w.y = h.py;
      w.on_n = true;
      w.nx = h.nx;
      w.ny = h.ny;
      w.seg = h.seg;
    } else {
      w.x = w.x + nux * w.R;
      w.y = w.y + nuy * w.R;
      w.on_n = false;
      w.seg = -1;
    }
    if (GUIDED) w.T *= mult;
    ++w.depth;
    if (!bbox_contains(s, w.x, w.y, pad)) finish_walk(w, a, true, 0.0, collect);
  }
  // unused slots of this lane's record chunk are marked invalid
  if (collect)
    for (int i = 0; i < w.rec_left; ++i) a.recs[w.rec_base + (8 - w.rec_left) + i].flags = 0u;
  // warp-aggregated walk counter
  unsigned long long wd = static_cast<unsigned long long>(walks_done);
  for (int o = 16; o > 0; o >>= 1) wd += __shfl_down_sync(0xffffffffu, wd, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&a.counters[2], wd);
}

// Welford pushes in wpp order, PointStats::push (proj/include/wost/wost.hpp:133-138)
__global__ void welford_kernel(const double* est, const int32_t* esc, int64_t n, int32_t rounds,
                               wg_point_stats* st) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  wg_point_stats p = st[i];
  for (int r = 0; r < rounds; ++r) {
    double v = est[static_cast<int64_t>(r) * n + i];
    ++p.count;
    double d = v - p.mean;
    p.mean += d / static_cast<double>(p.count);
    p.m2 += d * (v - p.mean);
    if (esc[static_cast<int64_t>(r) * n + i]) ++p.escaped;
  }
  st[i] = p;
}

// ---------------------------------------------------------------- queries
__global__ void __launch_bounds__(128) query_kernel(QueryArgs a) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const SceneView& s = a.scene;
  double x = a.xy[2 * i], y = a.xy[2 * i + 1];
  switch (a.op) {
    case 0: {
      CP c = closest_point(s, x, y, a.kinds);
      a.out_pt[2 * i] = c.px;
      a.out_pt[2 * i + 1] = c.py;
      a.out_d[i] = c.d;
      a.out_seg[i] = c.seg;
      if (c.seg < 0) a.out_pt[2 * i] = a.out_pt[2 * i + 1] = 0.0;
      break;
    }
    case 1: a.out_d[i] = closest_silhouette(s, x, y); break;
    case 2: {
      Hit h = ray_first_hit(s, x, y, a.dir[2 * i], a.dir[2 * i + 1], a.t_max[i], a.kinds,
                            a.exclude ? a.exclude[i] : -1);
      a.out_d[i] = h.t;
      a.out_pt[2 * i] = h.px;
      a.out_pt[2 * i + 1] = h.py;
      a.out_n[2 * i] = h.nx;
      a.out_n[2 * i + 1] = h.ny;
      a.out_seg[i] = h.seg;
      a.out_kind[i] = h.kind;
      break;
    }
    case 3: {  // Accel::star_radius, geom2d.cpp:248-255
      double dd = closest_point(s, x, y, WG_KIND_DIRICHLET).d;
      double ds = closest_silhouette(s, x, y);
      if (dd == dinf() && ds == dinf()) atomicOr(a.err, 1ull);
      a.out_d[i] = smin(dd, smax(ds, a.r_min));
      break;
    }
  }
}

__global__ void __launch_bounds__(128) field_eval_kernel(FieldView f, int64_t n, const double* xy,
                                                         double* out) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float o[256];
  field_eval_exact<0, 0, 0>(f, f.p + f.w1, xy[2 * i], xy[2 * i + 1], o);
  for (int j = 0; j < f.od; ++j) out[i * f.od + j] = o[j];
}

__global__ void __launch_bounds__(128) field_eval_kernel_default(FieldView f, int64_t n,
                                                                 const double* xy, double* out) {
  __shared__ float mlp[16 * 64 + 64 + 64 * 64 + 64 + 64 * 33 + 33];
  for (int i = threadIdx.x; i < f.mlp_count; i += blockDim.x) mlp[i] = f.p[f.w1 + i];
  __syncthreads();
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float o[33];
  field_eval_exact<16, 64, 33>(f, mlp, xy[2 * i], xy[2 * i + 1], o);
#pragma unroll
  for (int j = 0; j < 33; ++j) out[i * 33 + j] = o[j];
}

__global__ void normalize_kernel(int64_t n, const double* raw, int k, int dim, wg_mixture* out) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int od = (2 + dim) * k + 1;
  Mix m;
  normalize2<0>(raw + i * od, k, m);
  wg_mixture o;
  for (int c = 0; c < kMaxK; ++c) {
    o.mu[c][0] = c < k ? m.mux[c] : 0.0;
    o.mu[c][1] = c < k ? m.muy[c] : 0.0;
    o.mu[c][2] = 0.0;
    o.kappa[c] = c < k ? m.kappa[c] : 0.0;
    o.lambda[c] = c < k ? m.lambda[c] : 0.0;
    o.log_a[c] = c < k ? m.log_a[c] : 0.0;
  }
  o.c = m.c;
  o.k = k;
  o.dim = dim;
  out[i] = o;
}

// ---------------------------------------------------------------- launchers

cudaError_t launch_queries(const QueryArgs& a, cudaStream_t st) {
  if (a.n == 0) return cudaSuccess;
  int blocks = static_cast<int>((a.n + 127) / 128);
  query_kernel<<<blocks, 128, 0, st>>>(a);
  return cudaGetLastError();
}

template <bool G, int IN, int HID, int OD, int K>
static cudaError_t launch_walk_t(const WalkArgs& a, int blocks, cudaStream_t st) {
  size_t smem = a.scene_smem_bytes > 0 ? align16(a.scene_smem_bytes) : 0;
  if (G) smem += align16(sizeof(float) * a.field.mlp_count);
  auto k = walk_kernel<G, IN, HID, OD, K>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  k<<<blocks, 128, smem, st>>>(a);
  return cudaGetLastError();
}

template <bool G, int IN, int HID, int OD, int K>
static int occupancy_t(int smem_bytes) {
  int n = 0;
  auto k = walk_kernel<G, IN, HID, OD, K>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, 128, smem_bytes);
  return n;
}

int walk_blocks_per_sm(bool guided_default, bool guided_generic, int smem) {
  if (guided_default) return occupancy_t<true, 16, 64, 33, 8>(smem);
  if (guided_generic) return occupancy_t<true, 0, 0, 0, 0>(smem);
  return occupancy_t<false, 0, 0, 0, 0>(smem);
}

cudaError_t launch_walks(const WalkArgs& a, bool guided_default, bool guided_generic, int blocks,
                         cudaStream_t st) {
  if (guided_default) return launch_walk_t<true, 16, 64, 33, 8>(a, blocks, st);
  if (guided_generic) return launch_walk_t<true, 0, 0, 0, 0>(a, blocks, st);
  return launch_walk_t<false, 0, 0, 0, 0>(a, blocks, st);
}

cudaError_t launch_welford(const double* est, const int32_t* esc, int64_t n, int32_t rounds,
                           wg_point_stats* stats, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  welford_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, st>>>(est, esc, n, rounds, stats);
  return cudaGetLastError();
}

cudaError_t launch_field_eval(const FieldView& f, int64_t n, const double* xy, double* out,
                              cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  int blocks = static_cast<int>((n + 127) / 128);
  if (f.in == 16 && f.hid == 64 && f.od == 33)
    field_eval_kernel_default<<<blocks, 128, 0, st>>>(f, n, xy, out);
  else
    field_eval_kernel<<<blocks, 128, 0, st>>>(f, n, xy, out);
  return cudaGetLastError();
}

cudaError_t launch_normalize(int64_t n, const double* raw, int k, int dim, wg_mixture* out,
                             cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  normalize_kernel<<<static_cast<int>((n + 127) / 128), 128, 0, st>>>(n, raw, k, dim, out);
  return cudaGetLastError();
}

}  // namespace wg
