// Host runtime behind the C-ABI (include/wostgpu.h): scene / BVH build and
// upload, field initialisation and state, the solver (walk queues, record
// arena, training buffers, NCCL communicator) and every extern "C" entry.
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/wostgpu.h"
#include "wg_kernels.cuh"
#include "wg_train.cuh"

namespace wg {
cudaError_t launch_grad_tc(const TrainArgs& a, cudaStream_t st);  // wg_train_tc.cu
bool tc_grad_available();
}  // namespace wg

using namespace wg;

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

struct WgError : std::runtime_error {
  int code;
  WgError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(expr)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw WgError(WG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));    \
  } while (0)
#define CKL(expr)     \
  do {                \
    CK(expr);         \
    g_launches += 1;  \
  } while (0)
#define NCK(expr)                                                                     \
  do {                                                                                \
    ncclResult_t r_ = (expr);                                                         \
    if (r_ != ncclSuccess)                                                            \
      throw WgError(WG_ERR_CUDA, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
  } while (0)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return WG_OK;
  } catch (const WgError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return WG_ERR_RUNTIME;
  }
}

void need(bool ok, int code, const std::string& msg) {
  if (!ok) throw WgError(code, msg);
}

// owning device buffer
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  void alloc(size_t b) {
    if (b <= bytes && p) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    CK(cudaMalloc(&p, b ? b : 16));
    bytes = b;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
  template <class T>
  void upload(const T* h, size_t n) {
    alloc(sizeof(T) * n);
    if (n) CK(cudaMemcpy(p, h, sizeof(T) * n, cudaMemcpyHostToDevice));
  }
};

void check_device() {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  need(prop.major == 10, WG_ERR_CUDA,
       "wostgpu needs an sm_100 (B200) device; found sm_" + std::to_string(prop.major) +
           std::to_string(prop.minor));
}

// ---------------------------------------------------------------- host PCG32
// proj/include/wost/rng.hpp (host side, for the field's initial parameters)
struct HostPcg {
  Pcg r;
  HostPcg(uint64_t seed, uint64_t stream) { r.seed(seed, stream); }
  double uni(double lo, double hi) { return lo + (hi - lo) * r.uni(); }
};

}  // namespace

// ================================================================ scene
struct wg_scene_s {
  int device = 0;
  double bbox[4];
  double eps = 0, t_eps = 0, diag = 0;
  int32_t has_flux = 0, source_zero = 1;
  std::vector<Node> h_nodes;
  std::vector<Seg> h_segs;
  std::vector<SilVertex> h_sil;
  std::vector<double> h_sil_n;
  DBuf nodes, segs, sil, sil_n, seg_kind, seg_value, values;
  std::vector<std::unique_ptr<DBuf>> rasters;
  DevValue source{};
  SceneView view{};
  int smem_bytes = 0;  // bytes to stage nodes+segs+silhouettes, 0 if too big
};

namespace {

DevValue upload_value(const wg_value_spec& v, wg_scene_s* s) {
  DevValue d{};
  d.type = v.type;
  d.analytic_id = v.analytic_id;
  d.c0 = v.c0;
  d.cx = v.cx;
  d.cy = v.cy;
  d.rw = v.raster_w;
  d.rh = v.raster_h;
  for (int i = 0; i < 4; ++i) d.rb[i] = v.raster_bbox[i];
  d.raster = nullptr;
  if (v.type == WG_VALUE_RASTER) {
    need(v.raster_w >= 1 && v.raster_h >= 1 && v.raster_data, WG_ERR_SCENE,
         "raster resolution must be at least 1x1");
    for (int64_t i = 0; i < (int64_t)v.raster_w * v.raster_h; ++i)
      need(std::isfinite(v.raster_data[i]), WG_ERR_SCENE, "raster carries a non-finite cell value");
    auto b = std::make_unique<DBuf>();
    b->upload(v.raster_data, (size_t)v.raster_w * v.raster_h);
    d.raster = b->as<double>();
    s->rasters.push_back(std::move(b));
  }
  return d;
}

// median-split BVH identical to Accel::build (proj/src/geom2d.cpp:109-140):
// same nth_element comparator (centroid along the longer axis, tie by id),
// same leaf size 4, same DFS preorder => the same traversal order and ties
int build_bvh(std::vector<Seg>& segs, std::vector<Node>& nodes, int begin, int end) {
  Node nd;
  nd.lox = nd.loy = dinf();
  nd.hix = nd.hiy = -dinf();
  auto grow = [&](double x, double y) {
    nd.lox = std::min(nd.lox, x);
    nd.loy = std::min(nd.loy, y);
    nd.hix = std::max(nd.hix, x);
    nd.hiy = std::max(nd.hiy, y);
  };
  for (int i = begin; i < end; ++i) {
    grow(segs[i].ax, segs[i].ay);
    grow(segs[i].bx, segs[i].by);
  }
  nd.left = nd.right = -1;
  nd.begin = nd.end = 0;
  int idx = static_cast<int>(nodes.size());
  nodes.push_back(nd);
  if (end - begin <= 4) {
    nodes[idx].begin = begin;
    nodes[idx].end = end;
    return idx;
  }
  double ex = nd.hix - nd.lox, ey = nd.hiy - nd.loy;
  bool sx = ex >= ey;
  int mid = (begin + end) / 2;
  std::nth_element(segs.begin() + begin, segs.begin() + mid, segs.begin() + end,
                   [sx](const Seg& p, const Seg& q) {
                     double cp = sx ? p.ax + p.bx : p.ay + p.by;
                     double cq = sx ? q.ax + q.bx : q.ay + q.by;
                     if (cp != cq) return cp < cq;
                     return p.id < q.id;
                   });
  int l = build_bvh(segs, nodes, begin, mid);
  int r = build_bvh(segs, nodes, mid, end);
  nodes[idx].left = l;
  nodes[idx].right = r;
  return idx;
}

}  // namespace

// ================================================================ field
struct wg_field_s {
  wg_field_config cfg{};
  double bbox[4];
  int64_t n_params = 0;
  int64_t adam_steps = 0;
  DBuf p, m, v;
  FieldView view{};
};

namespace {

void field_layout(wg_field_s* f) {
  const wg_field_config& c = f->cfg;
  FieldView& v = f->view;
  v.levels = c.n_levels;
  v.F = c.features;
  v.in = c.n_levels * c.features;
  v.hid = c.hidden;
  v.k = c.mixture_k;
  v.dim = c.mixture_dim;
  v.od = (2 + c.mixture_dim) * c.mixture_k + 1;
  int64_t off = 0;
  for (int l = 0; l < c.n_levels; ++l) {
    v.res[l] = c.level_res[l];
    v.lvl_off[l] = static_cast<int32_t>(off);
    off += (int64_t)c.level_res[l] * c.level_res[l] * c.features;
  }
  v.w1 = (int32_t)off;
  off += (int64_t)v.in * v.hid;
  v.b1 = (int32_t)off;
  off += v.hid;
  v.w2 = (int32_t)off;
  off += (int64_t)v.hid * v.hid;
  v.b2 = (int32_t)off;
  off += v.hid;
  v.w3 = (int32_t)off;
  off += (int64_t)v.hid * v.od;
  v.b3 = (int32_t)off;
  off += v.od;
  v.mlp_count = (int32_t)(off - v.w1);
  f->n_params = off;
  for (int i = 0; i < 4; ++i) v.bbox[i] = f->bbox[i];
}

bool default_shape(const FieldView& v) {
  return v.levels == 4 && v.F == 4 && v.in == 16 && v.hid == 64 && v.od == 33 && v.k == 8 &&
         v.dim == 2;
}

}  // namespace

// ================================================================ solver
struct wg_solver_s {
  wg_scene_s* scene = nullptr;
  wg_field_s* field = nullptr;
  wg_solver_config cfg{};
  int mlp = WG_MLP_EXACT;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
  double last_walk_ms = 0, last_train_ms = 0;
  int sm_count = 148;
  // points and statistics
  int64_t n_points = 0, point_offset = 0;
  DBuf points, stats;
  // per-round results
  DBuf est, esc, steps;
  int32_t est_rounds = 0;
  int32_t last_rounds = 0;
  // records of the last collecting round
  DBuf recs;
  int64_t rec_capacity = 0;
  int64_t last_rec_count = 0;
  bool have_records = false;
  // counters
  DBuf counters;  // 8 x u64
  unsigned long long last_counters[8] = {};
  // training
  DBuf keys, keys_sorted, idx, idx_sorted, sort_temp, grad, tcount, norm2;
  size_t sort_temp_bytes = 0;
  // NCCL
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  // accumulated over wostgpu_run
  double run_walk_ms = 0, run_train_ms = 0;
  int64_t run_walks = 0, run_steps = 0, run_escaped = 0, run_train_steps = 0;
  cudaEvent_t ev_run0 = nullptr, ev_run1 = nullptr;
};

namespace {

SolverParams solver_params(const wg_solver_s* s) {
  SolverParams p{};
  p.eps = s->cfg.epsilon_shell > 0.0 ? s->cfg.epsilon_shell : s->scene->eps;
  p.rmin = s->cfg.r_min > 0.0 ? s->cfg.r_min : p.eps;
  p.fixed_c = s->cfg.fixed_c;
  p.grazing_floor = s->cfg.grazing_floor;
  p.rr_depth = s->cfg.rr_depth;
  p.max_steps = s->cfg.max_steps;
  p.mode = s->cfg.mode;
  p.reflect = s->cfg.reflect_at_neumann;
  p.clamp_grazing = s->cfg.clamp_grazing;
  return p;
}

void run_rounds(wg_solver_s* s, uint64_t seed, uint64_t wpp_first, int32_t rounds, bool collect,
                uint64_t key_seed) {
  need(s->n_points > 0, WG_ERR_INVALID, "solver has no evaluation points");
  const bool guided = s->cfg.mode != WG_MODE_UNIFORM;
  need(!guided || s->field, WG_ERR_INVALID, "guided sampler modes need a guiding field");
  need(!collect || rounds == 1, WG_ERR_INVALID, "record collection runs one round at a time");
  const bool dflt = guided && default_shape(s->field->view);
  // chunk rounds so the estimate buffer stays below ~1 GiB
  int32_t chunk = static_cast<int32_t>(std::max<int64_t>(1, (int64_t(1) << 30) / (s->n_points * 16)));
  chunk = std::min(chunk, rounds);
  if (s->est_rounds < chunk) {
    s->est.alloc(sizeof(double) * s->n_points * chunk);
    s->esc.alloc(sizeof(int32_t) * s->n_points * chunk);
    s->steps.alloc(sizeof(int32_t) * s->n_points * chunk);
    s->est_rounds = chunk;
  }
  if (collect) {
    int64_t cap = std::max<int64_t>(s->n_points * 96, 1 << 16);
    if (s->rec_capacity < cap) {
      s->recs.alloc(sizeof(DevRecord) * cap);
      s->rec_capacity = cap;
    }
  }
  s->counters.alloc(sizeof(unsigned long long) * 8);
  CK(cudaMemsetAsync(s->counters.p, 0, sizeof(unsigned long long) * 8, s->stream));

  WalkArgs a{};
  a.scene = s->scene->view;
  a.scene_smem_bytes = s->scene->smem_bytes;
  if (guided) a.field = s->field->view;
  a.sp = solver_params(s);
  a.points = s->points.as<double>();
  a.n_points = s->n_points;
  a.point_offset = s->point_offset;
  a.seed = seed;
  a.est = s->est.as<double>();
  a.esc = s->esc.as<int32_t>();
  a.steps = s->steps.as<int32_t>();
  a.counters = s->counters.as<unsigned long long>();
  a.recs = collect ? s->recs.as<DevRecord>() : nullptr;
  a.rec_counter = a.counters + 5;
  a.rec_capacity = s->rec_capacity;
  a.key_seed = key_seed;

  // guided walks on the default field shape: tcgen05 MLP tile kernel, or the
  // bit-faithful CUDA-core MLP with 8 lanes per walk
  const bool tc = dflt && s->mlp == WG_MLP_TENSOR;
  const bool g8 = dflt && !tc;
  int smem = (s->scene->smem_bytes > 0 ? ((s->scene->smem_bytes + 15) & ~15) : 0) +
             (guided ? ((int)sizeof(float) * s->field->view.mlp_count + 15) / 16 * 16 : 0);
  if (g8) smem = walk_g8_smem(a);
  if (tc) smem = walk_tc_smem(a);
  const int lanes_per_walk = g8 ? 8 : 1;
  const int block = g8 ? 256 : 128;
  int per_sm = std::max(1, tc ? walk_tc_blocks_per_sm(smem)
                              : g8 ? walk_g8_blocks_per_sm(smem)
                                   : walk_blocks_per_sm(dflt, guided && !dflt, smem));
  CK(cudaEventRecord(s->ev0, s->stream));
  for (int32_t r0 = 0; r0 < rounds; r0 += chunk) {
    int32_t n = std::min(chunk, rounds - r0);
    a.wpp_first = wpp_first + r0;
    a.n_rounds = n;
    int64_t total = s->n_points * n;
    int64_t want = (total * lanes_per_walk + block - 1) / block;
    int blocks = static_cast<int>(std::min<int64_t>(want, (int64_t)per_sm * s->sm_count));
    if (tc) CKL(launch_walks_tc(a, std::max(1, blocks), s->stream));
    else if (g8) CKL(launch_walks_g8(a, std::max(1, blocks), s->stream));
    else CKL(launch_walks(a, dflt, guided && !dflt, std::max(1, blocks), s->stream));
    CKL(launch_welford(a.est, a.esc, s->n_points, n, s->stats.as<wg_point_stats>(), s->stream));
  }
  CK(cudaEventRecord(s->ev1, s->stream));
  CK(cudaMemcpyAsync(s->last_counters, s->counters.p, sizeof(unsigned long long) * 8,
                     cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
  s->last_walk_ms = ms;
  s->last_rounds = std::min(chunk, rounds);
  need(s->last_counters[4] == 0, WG_ERR_SCENE,
       "walk: unbounded star region (no Dirichlet boundary and no Neumann silhouette)");
  if (collect) {
    s->last_rec_count = std::min<int64_t>((int64_t)s->last_counters[5], s->rec_capacity);
    s->have_records = true;
  }
}

void ensure_train_buffers(wg_solver_s* s, int64_t n) {
  s->keys.alloc(sizeof(uint64_t) * n);
  s->keys_sorted.alloc(sizeof(uint64_t) * n);
  s->idx.alloc(sizeof(uint32_t) * n);
  s->idx_sorted.alloc(sizeof(uint32_t) * n);
  size_t tb = sort_temp_bytes(n);
  if (tb > s->sort_temp_bytes) {
    s->sort_temp.alloc(tb);
    s->sort_temp_bytes = tb;
  }
  s->grad.alloc(sizeof(float) * (s->field->n_params + 1));
  s->norm2.alloc(sizeof(double) * 8);
}

// train_batch over the device records [0, n_recs) (guide_train.cpp:94-198)
wg_train_stats train_records(wg_solver_s* s, int64_t n_recs, const wg_train_config& tc,
                             uint64_t round, bool keep_order) {
  wg_field_s* f = s->field;
  need(f != nullptr, WG_ERR_INVALID, "training needs a guiding field");
  need(default_shape(f->view), WG_ERR_NOT_BUILT,
       "device training is built for the default field shape (L=4, F=4, hidden 64, K=8, 2D)");
  wg_train_stats st{};
  CK(cudaEventRecord(s->ev2, s->stream));
  // size once for the whole record arena: no allocation churn between rounds
  ensure_train_buffers(s, std::max<int64_t>(std::max(n_recs, s->rec_capacity), 1));
  unsigned long long* cnt = s->counters.as<unsigned long long>();
  CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * 8, s->stream));
  const uint32_t* order;
  if (!keep_order) {
    CKL(launch_select(s->recs.as<DevRecord>(), n_recs, tc.pdf_floor, s->keys.as<uint64_t>(),
                      s->keys_sorted.as<uint64_t>(), s->idx.as<uint32_t>(),
                      s->idx_sorted.as<uint32_t>(), s->sort_temp.p, s->sort_temp_bytes, cnt,
                      s->stream));
    order = s->idx_sorted.as<uint32_t>();
  } else {
    CKL(launch_select(s->recs.as<DevRecord>(), n_recs, tc.pdf_floor, s->keys.as<uint64_t>(),
                      s->keys_sorted.as<uint64_t>(), s->idx.as<uint32_t>(),
                      s->idx_sorted.as<uint32_t>(), s->sort_temp.p, s->sort_temp_bytes, cnt,
                      s->stream));
    order = s->idx_sorted.as<uint32_t>();
  }
  unsigned long long h[3];
  CK(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  int64_t usable = (int64_t)h[1];
  st.records_seen = (int64_t)h[0];
  st.skipped_low_pdf = (int64_t)h[2];
  int64_t take = std::min<int64_t>(usable, tc.max_records_per_round);
  // all ranks must run the same number of Adam steps: agree on the largest
  int64_t n_steps = (take + tc.minibatch - 1) / tc.minibatch;
  if (s->comm) {
    int64_t* d = reinterpret_cast<int64_t*>(s->norm2.as<double>() + 4);
    CK(cudaMemcpyAsync(d, &n_steps, sizeof(int64_t), cudaMemcpyHostToDevice, s->stream));
    NCK(ncclAllReduce(d, d, 1, ncclInt64, ncclMax, s->comm, s->stream));
    CK(cudaMemcpyAsync(&n_steps, d, sizeof(int64_t), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
  }
  if (n_steps == 0) {
    CK(cudaEventRecord(s->ev3, s->stream));
    return st;
  }
  const bool use_tc = s->mlp == WG_MLP_TENSOR && tc_grad_available();
  double norm_sum = 0.0;
  for (int64_t b = 0; b < n_steps; ++b) {
    int64_t begin = b * tc.minibatch;
    int64_t count = std::max<int64_t>(0, std::min<int64_t>(tc.minibatch, take - begin));
    CK(cudaMemsetAsync(s->grad.p, 0, sizeof(float) * (f->n_params + 1), s->stream));
    TrainArgs ta{};
    ta.f = f->view;
    ta.recs = s->recs.as<DevRecord>();
    ta.order = order;
    ta.begin = begin;
    ta.count = count;
    ta.grad = s->grad.as<float>();
    ta.inv_count = 1.0;  // mean taken in the Adam kernel (after the allreduce)
    ta.reflect = tc.reflect;
    ta.learn_selection = tc.learn_selection;
    ta.e_fraction = tc.e_fraction;
    ta.v_floor = tc.v_floor;
    ta.counters = cnt + 3;
    if (count > 0) {
      if (use_tc) CKL(launch_grad_tc(ta, s->stream));
      else CKL(launch_grad_cuda_core(ta, s->stream));
    }
    float fc = static_cast<float>(count);
    CK(cudaMemcpyAsync(s->grad.as<float>() + f->n_params, &fc, sizeof(float),
                       cudaMemcpyHostToDevice, s->stream));
    if (s->comm)
      NCK(ncclAllReduce(s->grad.p, s->grad.p, f->n_params + 1, ncclFloat, ncclSum, s->comm,
                        s->stream));
    CK(cudaMemsetAsync(s->norm2.p, 0, sizeof(double), s->stream));
    f->adam_steps += 1;
    CKL(launch_adam(f->p.as<float>(), f->m.as<double>(), f->v.as<double>(), s->grad.as<float>(),
                    f->n_params, tc.lr, tc.beta1, tc.beta2, tc.eps, f->adam_steps,
                    s->grad.as<float>() + f->n_params, s->norm2.as<double>(), s->stream));
    double n2 = 0;
    CK(cudaMemcpyAsync(&n2, s->norm2.p, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    norm_sum += std::sqrt(n2);
    st.steps += 1;
  }
  st.mean_grad_norm = norm_sum / static_cast<double>(st.steps);
  CK(cudaMemcpyAsync(h, cnt + 3, sizeof(unsigned long long) * 2, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaEventRecord(s->ev3, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  st.records_consumed = (int64_t)h[0];
  st.skipped_low_v = (int64_t)h[1];
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, s->ev2, s->ev3));
  s->last_train_ms = ms;
  st.seconds = ms * 1e-3;
  return st;
}

}  // namespace

// ================================================================ C-ABI
extern "C" {

const char* wostgpu_last_error(void) { return g_err.c_str(); }

int wostgpu_init(int device) {
  return guarded([&] {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    need(device >= 0 && device < n, WG_ERR_CUDA, "no such CUDA device");
    CK(cudaSetDevice(device));
    check_device();
  });
}

int wostgpu_device_info(int* sm_count, int* major, int* minor) {
  return guarded([&] {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, dev));
    *sm_count = p.multiProcessorCount;
    *major = p.major;
    *minor = p.minor;
  });
}

int64_t wostgpu_kernel_launches(void) { return g_launches.load(); }

int wostgpu_scene_create(const double* seg, const int32_t* kind, const int32_t* value_index,
                         int32_t n_seg, const wg_value_spec* values, int32_t n_values,
                         const wg_value_spec* source, const double bbox[4], double eps,
                         wg_scene* out) {
  return guarded([&] {
    check_device();
    auto s = std::make_unique<wg_scene_s>();
    for (int i = 0; i < 4; ++i) s->bbox[i] = bbox[i];
    const bool validate = eps > 0.0;
    s->eps = validate ? eps : 1e-3;
    if (validate) {  // Scene::validate, proj/src/scene.cpp:119-143
      need(bbox[0] <= bbox[2] && bbox[1] <= bbox[3], WG_ERR_SCENE, "scene bbox is empty");
      need(n_seg > 0, WG_ERR_SCENE, "scene has no boundary segments");
    }
    need(n_seg > 0, WG_ERR_SCENE, "build_accel: scene has no segments");
    std::vector<int32_t> hk(n_seg), hv(n_seg);
    s->h_segs.resize(n_seg);
    for (int i = 0; i < n_seg; ++i) {
      Seg g;
      g.ax = seg[4 * i];
      g.ay = seg[4 * i + 1];
      g.bx = seg[4 * i + 2];
      g.by = seg[4 * i + 3];
      g.kind = kind[i];
      g.id = i;
      if (validate) {
        std::string w = "segment " + std::to_string(i);
        need(!(g.ax == g.bx && g.ay == g.by), WG_ERR_SCENE, w + ": a == b (zero-length segment)");
        auto in = [&](double x, double y) {
          return x >= bbox[0] && x <= bbox[2] && y >= bbox[1] && y <= bbox[3];
        };
        need(in(g.ax, g.ay) && in(g.bx, g.by), WG_ERR_SCENE, w + ": endpoint outside scene bbox");
        need(value_index[i] >= 0 && value_index[i] < n_values, WG_ERR_SCENE,
             w + ": value is not defined");
      }
      s->h_segs[i] = g;
      hk[i] = kind[i];
      hv[i] = value_index[i];
    }
    // BVH (geom2d.cpp:80-140)
    std::vector<Seg> order = s->h_segs;
    build_bvh(order, s->h_nodes, 0, n_seg);
    {
      double ex = s->h_nodes[0].hix - s->h_nodes[0].lox, ey = s->h_nodes[0].hiy - s->h_nodes[0].loy;
      s->t_eps = 1e-6 * std::sqrt(ex * ex + ey * ey);
    }
    {
      double ex = bbox[2] - bbox[0], ey = bbox[3] - bbox[1];
      s->diag = std::sqrt(ex * ex + ey * ey);
    }
    // Neumann vertex adjacency keyed by exact bits (geom2d.cpp:93-106)
    std::map<std::pair<uint64_t, uint64_t>, int> keymap;
    std::vector<std::vector<double>> normals;
    std::vector<std::pair<double, double>> pos;
    for (const Seg& g : order) {
      if (g.kind != WG_NEUMANN) continue;
      double ux = g.bx - g.ax, uy = g.by - g.ay;
      double px = -uy, py = ux;
      double l = std::sqrt(px * px + py * py);
      double nx = px / l, ny = py / l;
      for (int e = 0; e < 2; ++e) {
        double x = e ? g.bx : g.ax, y = e ? g.by : g.ay;
        uint64_t kx, ky;
        std::memcpy(&kx, &x, 8);
        std::memcpy(&ky, &y, 8);
        auto it = keymap.find({kx, ky});
        int vi;
        if (it == keymap.end()) {
          vi = (int)pos.size();
          keymap[{kx, ky}] = vi;
          pos.push_back({x, y});
          normals.emplace_back();
        } else {
          vi = it->second;
        }
        normals[vi].push_back(nx);
        normals[vi].push_back(ny);
      }
    }
    for (size_t v = 0; v < pos.size(); ++v) {
      SilVertex sv;
      sv.px = pos[v].first;
      sv.py = pos[v].second;
      sv.n_begin = (int32_t)(s->h_sil_n.size() / 2);
      sv.n_count = (int32_t)(normals[v].size() / 2);
      s->h_sil.push_back(sv);
      s->h_sil_n.insert(s->h_sil_n.end(), normals[v].begin(), normals[v].end());
    }
    // values and flux flag (Scene::has_neumann_flux, scene.cpp:83-91)
    std::vector<DevValue> dv;
    for (int i = 0; i < n_values; ++i) dv.push_back(upload_value(values[i], s.get()));
    s->has_flux = 0;
    for (int i = 0; i < n_seg; ++i) {
      if (kind[i] != WG_NEUMANN) continue;
      const wg_value_spec& v = values[value_index[i]];
      if (v.type != WG_VALUE_CONSTANT || v.c0 != 0.0) s->has_flux = 1;
    }
    if (source && source->type != WG_VALUE_ZERO) {
      s->source = upload_value(*source, s.get());
      s->source_zero = 0;
    } else {
      s->source.type = WG_VALUE_ZERO;
      s->source_zero = 1;
    }
    // upload
    s->nodes.upload(s->h_nodes.data(), s->h_nodes.size());
    s->segs.upload(order.data(), order.size());
    s->sil.upload(s->h_sil.data(), s->h_sil.size());
    s->sil_n.upload(s->h_sil_n.data(), s->h_sil_n.size());
    s->seg_kind.upload(hk.data(), hk.size());
    s->seg_value.upload(hv.data(), hv.size());
    s->values.upload(dv.data(), dv.size());
    SceneView& v = s->view;
    v.nodes = s->nodes.as<Node>();
    v.segs = s->segs.as<Seg>();
    v.sil = s->sil.as<SilVertex>();
    v.sil_n = s->sil_n.as<double>();
    v.n_nodes = (int32_t)s->h_nodes.size();
    v.n_segs = n_seg;
    v.n_sil = (int32_t)s->h_sil.size();
    v.n_sil_normals = (int32_t)(s->h_sil_n.size() / 2);
    v.seg_kind = s->seg_kind.as<int32_t>();
    v.seg_value = s->seg_value.as<int32_t>();
    v.values = s->values.as<DevValue>();
    v.source = s->source;
    for (int i = 0; i < 4; ++i) v.bbox[i] = bbox[i];
    v.eps = s->eps;
    v.t_eps = s->t_eps;
    v.diag = s->diag;
    v.has_flux = s->has_flux;
    v.source_zero = s->source_zero;
    auto a16 = [](size_t b) { return (b + 15) & ~size_t(15); };
    size_t bytes = a16(sizeof(Node) * v.n_nodes) + a16(sizeof(Seg) * v.n_segs) +
                   a16(sizeof(SilVertex) * v.n_sil) + a16(sizeof(double) * 2 * v.n_sil_normals);
    s->smem_bytes = bytes <= 96 * 1024 ? (int)bytes : 0;
    *out = s.release();
  });
}

int wostgpu_scene_destroy(wg_scene s) {
  return guarded([&] { delete s; });
}

int wostgpu_scene_info(wg_scene s, double* t_eps, int32_t* flux, double root_box[4]) {
  return guarded([&] {
    if (t_eps) *t_eps = s->t_eps;
    if (flux) *flux = s->has_flux;
    if (root_box) {
      root_box[0] = s->h_nodes[0].lox;
      root_box[1] = s->h_nodes[0].loy;
      root_box[2] = s->h_nodes[0].hix;
      root_box[3] = s->h_nodes[0].hiy;
    }
  });
}

static int run_query(wg_scene s, int op, int64_t n, const double* xy, const double* dir,
                     const double* tmax, uint32_t kinds, const int32_t* exclude, double r_min,
                     double* out_d, double* out_pt, double* out_n, int32_t* out_seg,
                     int32_t* out_kind) {
  return guarded([&] {
    if (n == 0) return;
    DBuf dxy, ddir, dtm, dex, od, opt, on, oseg, okind, err;
    dxy.upload(xy, 2 * n);
    if (dir) ddir.upload(dir, 2 * n);
    if (tmax) dtm.upload(tmax, n);
    if (exclude) dex.upload(exclude, n);
    od.alloc(sizeof(double) * n);
    opt.alloc(sizeof(double) * 2 * n);
    on.alloc(sizeof(double) * 2 * n);
    oseg.alloc(sizeof(int32_t) * n);
    okind.alloc(sizeof(int32_t) * n);
    err.alloc(8);
    CK(cudaMemset(err.p, 0, 8));
    QueryArgs a{};
    a.scene = s->view;
    a.n = n;
    a.op = op;
    a.kinds = kinds;
    a.r_min = r_min;
    a.xy = dxy.as<double>();
    a.dir = dir ? ddir.as<double>() : nullptr;
    a.t_max = tmax ? dtm.as<double>() : nullptr;
    a.exclude = exclude ? dex.as<int32_t>() : nullptr;
    a.out_d = od.as<double>();
    a.out_pt = opt.as<double>();
    a.out_n = on.as<double>();
    a.out_seg = oseg.as<int32_t>();
    a.out_kind = okind.as<int32_t>();
    a.err = err.as<unsigned long long>();
    CKL(launch_queries(a, 0));
    CK(cudaDeviceSynchronize());
    unsigned long long e = 0;
    CK(cudaMemcpy(&e, err.p, 8, cudaMemcpyDeviceToHost));
    need(e == 0, WG_ERR_SCENE,
         "star_radius: both Dirichlet and silhouette distances are infinite (unbounded star region)");
    if (out_d) CK(cudaMemcpy(out_d, od.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
    if (out_pt) CK(cudaMemcpy(out_pt, opt.p, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost));
    if (out_n) CK(cudaMemcpy(out_n, on.p, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost));
    if (out_seg) CK(cudaMemcpy(out_seg, oseg.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    if (out_kind) CK(cudaMemcpy(out_kind, okind.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  });
}

int wostgpu_closest_point(wg_scene s, int64_t n, const double* xy, uint32_t kinds, double* point,
                          double* dist, int32_t* segment) {
  return run_query(s, 0, n, xy, nullptr, nullptr, kinds, nullptr, 0.0, dist, point, nullptr,
                   segment, nullptr);
}
int wostgpu_closest_silhouette(wg_scene s, int64_t n, const double* xy, double* dist) {
  return run_query(s, 1, n, xy, nullptr, nullptr, 0, nullptr, 0.0, dist, nullptr, nullptr,
                   nullptr, nullptr);
}
int wostgpu_ray_first_hit(wg_scene s, int64_t n, const double* o, const double* d,
                          const double* tmax, uint32_t kinds, const int32_t* exclude, double* t,
                          double* point, double* normal, int32_t* segment, int32_t* kind) {
  return run_query(s, 2, n, o, d, tmax, kinds, exclude, 0.0, t, point, normal, segment, kind);
}
int wostgpu_star_radius(wg_scene s, int64_t n, const double* xy, double r_min, double* r) {
  return run_query(s, 3, n, xy, nullptr, nullptr, 0, nullptr, r_min, r, nullptr, nullptr,
                   nullptr, nullptr);
}

int wostgpu_field_create(const wg_field_config* cfg, const double bbox[4], uint64_t seed,
                         wg_field* out) {
  return guarded([&] {
    check_device();
    const wg_field_config& c = *cfg;
    // GuidingField validation, guide_field.cpp:16-32
    need(c.n_levels >= 1 && c.n_levels <= WG_MAX_LEVELS && c.features >= 1 && c.mixture_k >= 1,
         WG_ERR_INVALID, "guiding field: L, F and K must be >= 1");
    need(c.mixture_k <= WG_MAX_MIXTURE, WG_ERR_INVALID, "guiding field: K exceeds the component cap");
    need(c.mixture_dim == 2 || c.mixture_dim == 3, WG_ERR_INVALID,
         "guiding field: mixture dim must be 2 or 3");
    need(c.hidden >= 1, WG_ERR_INVALID, "guiding field: hidden width must be >= 1");
    for (int l = 0; l < c.n_levels; ++l)
      need(c.level_res[l] >= 2, WG_ERR_INVALID,
           "guiding field: grid resolution must be >= 2 per axis");
    need(c.n_levels * c.features <= 256 && c.hidden <= 256, WG_ERR_INVALID,
         "guiding field: L*F and hidden width are capped at 256");
    need(bbox[0] <= bbox[2] && bbox[1] <= bbox[3] && bbox[2] - bbox[0] > 0.0 &&
             bbox[3] - bbox[1] > 0.0,
         WG_ERR_INVALID, "guiding field: bbox is empty");
    auto f = std::make_unique<wg_field_s>();
    f->cfg = c;
    for (int i = 0; i < 4; ++i) f->bbox[i] = bbox[i];
    field_layout(f.get());
    // initial parameters: the reference's init stream (guide_field.cpp:36-51)
    std::vector<float> p(f->n_params, 0.0f);
    HostPcg rng(Pcg::mix(seed), 0x67e5504410b1426fULL);
    const FieldView& v = f->view;
    for (int64_t i = 0; i < v.w1; ++i) p[i] = static_cast<float>(rng.uni(-1e-4, 1e-4));
    auto layer = [&](int64_t wo, int64_t wc, int64_t bo, int64_t bc, int fan_in) {
      double sc = 1.0 / std::sqrt(static_cast<double>(fan_in));
      for (int64_t i = 0; i < wc; ++i) p[wo + i] = static_cast<float>(rng.uni(-sc, sc));
      for (int64_t i = 0; i < bc; ++i) p[bo + i] = 0.0f;
    };
    layer(v.w1, (int64_t)v.in * v.hid, v.b1, v.hid, v.in);
    layer(v.w2, (int64_t)v.hid * v.hid, v.b2, v.hid, v.hid);
    layer(v.w3, (int64_t)v.hid * v.od, v.b3, v.od, v.hid);
    f->p.upload(p.data(), p.size());
    f->m.alloc(sizeof(double) * f->n_params);
    f->v.alloc(sizeof(double) * f->n_params);
    CK(cudaMemset(f->m.p, 0, sizeof(double) * f->n_params));
    CK(cudaMemset(f->v.p, 0, sizeof(double) * f->n_params));
    f->view.p = f->p.as<float>();
    *out = f.release();
  });
}

int wostgpu_field_destroy(wg_field f) {
  return guarded([&] { delete f; });
}

int wostgpu_field_param_count(wg_field f, int64_t* n) {
  return guarded([&] { *n = f->n_params; });
}

int wostgpu_field_get_state(wg_field f, float* p, double* m, double* v, int64_t* steps) {
  return guarded([&] {
    CK(cudaDeviceSynchronize());
    if (p) CK(cudaMemcpy(p, f->p.p, sizeof(float) * f->n_params, cudaMemcpyDeviceToHost));
    if (m) CK(cudaMemcpy(m, f->m.p, sizeof(double) * f->n_params, cudaMemcpyDeviceToHost));
    if (v) CK(cudaMemcpy(v, f->v.p, sizeof(double) * f->n_params, cudaMemcpyDeviceToHost));
    if (steps) *steps = f->adam_steps;
  });
}

int wostgpu_field_set_state(wg_field f, const float* p, const double* m, const double* v,
                            int64_t steps) {
  return guarded([&] {
    CK(cudaDeviceSynchronize());
    if (p) CK(cudaMemcpy(f->p.p, p, sizeof(float) * f->n_params, cudaMemcpyHostToDevice));
    if (m) CK(cudaMemcpy(f->m.p, m, sizeof(double) * f->n_params, cudaMemcpyHostToDevice));
    if (v) CK(cudaMemcpy(f->v.p, v, sizeof(double) * f->n_params, cudaMemcpyHostToDevice));
    if (steps >= 0) f->adam_steps = steps;
  });
}

int wostgpu_field_eval_batch(wg_field f, int64_t n, const double* xy, double* out, int mlp) {
  return guarded([&] {
    need(mlp == WG_MLP_EXACT || default_shape(f->view), WG_ERR_NOT_BUILT,
         "tensor-core field evaluation is built for the default field shape");
    if (n == 0) return;
    DBuf dxy, dout;
    dxy.upload(xy, 2 * n);
    dout.alloc(sizeof(double) * n * f->view.od);
    if (mlp == WG_MLP_TENSOR) {
      int dev = 0, sms = 148;
      CK(cudaGetDevice(&dev));
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      CKL(launch_field_eval_tc(f->view, n, dxy.as<double>(), dout.as<double>(), sms, 0));
    } else {
      CKL(launch_field_eval(f->view, n, dxy.as<double>(), dout.as<double>(), 0));
    }
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out, dout.p, sizeof(double) * n * f->view.od, cudaMemcpyDeviceToHost));
  });
}

int wostgpu_normalize_params(int64_t n, const double* raw, int32_t k, int32_t dim, wg_mixture* out) {
  return guarded([&] {
    need(dim == 2, WG_ERR_NOT_BUILT, "device normalisation is built for dim 2");
    need(k >= 1 && k <= WG_MAX_MIXTURE, WG_ERR_INVALID, "mixture size out of range");
    if (n == 0) return;
    const int od = (2 + dim) * k + 1;
    DBuf draw, dout;
    draw.upload(raw, (size_t)n * od);
    dout.alloc(sizeof(wg_mixture) * n);
    CKL(launch_normalize(n, draw.as<double>(), k, dim, dout.as<wg_mixture>(), 0));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out, dout.p, sizeof(wg_mixture) * n, cudaMemcpyDeviceToHost));
  });
}

int wostgpu_solver_create(wg_scene scene, wg_field field, const wg_solver_config* cfg,
                          wg_solver* out) {
  return guarded([&] {
    check_device();
    need(scene != nullptr, WG_ERR_INVALID, "solver needs a scene");
    bool has_dirichlet = false;
    for (const Seg& g : scene->h_segs) has_dirichlet |= g.kind == WG_DIRICHLET;
    need(has_dirichlet, WG_ERR_SCENE, "solver: scene has no Dirichlet boundary; walks cannot terminate");
    need(cfg->mode == WG_MODE_UNIFORM || field != nullptr, WG_ERR_INVALID,
         "guided sampler modes need a guiding field");
    if (field) need(field->view.dim == 2, WG_ERR_NOT_BUILT, "2D walks need a 2D guiding field");
    auto s = std::make_unique<wg_solver_s>();
    s->scene = scene;
    s->field = field;
    s->cfg = *cfg;
    s->mlp = WG_MLP_EXACT;
    CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&s->ev0));
    CK(cudaEventCreate(&s->ev1));
    CK(cudaEventCreate(&s->ev2));
    CK(cudaEventCreate(&s->ev3));
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&s->sm_count, cudaDevAttrMultiProcessorCount, dev));
    *out = s.release();
  });
}

int wostgpu_solver_destroy(wg_solver s) {
  return guarded([&] {
    if (!s) return;
    if (s->comm) ncclCommDestroy(s->comm);
    cudaStreamSynchronize(s->stream);
    cudaEventDestroy(s->ev0);
    cudaEventDestroy(s->ev1);
    cudaEventDestroy(s->ev2);
    cudaEventDestroy(s->ev3);
    cudaStreamDestroy(s->stream);
    delete s;
  });
}

int wostgpu_solver_set_mlp(wg_solver s, int mlp) {
  return guarded([&] {
    need(mlp == WG_MLP_EXACT || mlp == WG_MLP_TENSOR, WG_ERR_INVALID, "unknown MLP path");
    s->mlp = mlp;
  });
}

int wostgpu_solver_set_points(wg_solver s, int64_t n, const double* xy, int64_t offset) {
  return guarded([&] {
    s->n_points = n;
    s->point_offset = offset;
    s->points.alloc(sizeof(double) * 2 * std::max<int64_t>(n, 1));
    s->stats.alloc(sizeof(wg_point_stats) * std::max<int64_t>(n, 1));
    if (n) {
      CK(cudaMemcpyAsync(s->points.p, xy, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, s->stream));
      CK(cudaMemsetAsync(s->stats.p, 0, sizeof(wg_point_stats) * n, s->stream));
    }
    CK(cudaStreamSynchronize(s->stream));
  });
}

int wostgpu_solver_get_stats(wg_solver s, wg_point_stats* st) {
  return guarded([&] {
    CK(cudaMemcpyAsync(st, s->stats.p, sizeof(wg_point_stats) * s->n_points,
                       cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
  });
}

int wostgpu_solver_set_stats(wg_solver s, const wg_point_stats* st) {
  return guarded([&] {
    CK(cudaMemcpyAsync(s->stats.p, st, sizeof(wg_point_stats) * s->n_points,
                       cudaMemcpyHostToDevice, s->stream));
    CK(cudaStreamSynchronize(s->stream));
  });
}

int wostgpu_solve_rounds(wg_solver s, uint64_t seed, uint64_t wpp_first, int32_t n_rounds,
                         int32_t collect) {
  return guarded([&] {
    need(n_rounds >= 1, WG_ERR_INVALID, "n_rounds must be >= 1");
    uint64_t key_seed = Pcg::mix(seed ^ 0x7261696e5f6b6579ULL) ^ Pcg::mix(wpp_first + 1);
    run_rounds(s, seed, wpp_first, n_rounds, collect != 0, key_seed);
  });
}

int wostgpu_solve_batch(wg_solver s, int64_t n, const double* xy, wg_point_stats* st,
                        uint64_t seed, uint64_t wpp, int32_t collect) {
  int rc = wostgpu_solver_set_points(s, n, xy, 0);
  if (rc) return rc;
  rc = wostgpu_solver_set_stats(s, st);
  if (rc) return rc;
  rc = wostgpu_solve_rounds(s, seed, wpp, 1, collect);
  if (rc) return rc;
  return wostgpu_solver_get_stats(s, st);
}

int wostgpu_fetch_records(wg_solver s, wg_guide_record* out, int64_t capacity, int64_t* n) {
  return guarded([&] {
    need(s->have_records, WG_ERR_INVALID, "no collecting round has run");
    DBuf d, c;
    d.alloc(sizeof(wg_guide_record) * std::max<int64_t>(s->last_rec_count, 1));
    c.alloc(8);
    CK(cudaMemsetAsync(c.p, 0, 8, s->stream));
    CKL(launch_export_records(s->recs.as<DevRecord>(), s->last_rec_count,
                              d.as<wg_guide_record>(), c.as<unsigned long long>(), s->stream));
    unsigned long long cnt = 0;
    CK(cudaMemcpyAsync(&cnt, c.p, 8, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    *n = (int64_t)cnt;
    if (out) {
      int64_t m = std::min<int64_t>((int64_t)cnt, capacity);
      CK(cudaMemcpy(out, d.p, sizeof(wg_guide_record) * m, cudaMemcpyDeviceToHost));
    }
  });
}

int wostgpu_fetch_walks(wg_solver s, double* est, int32_t* esc, int32_t* steps) {
  return guarded([&] {
    CK(cudaStreamSynchronize(s->stream));
    int64_t n = s->n_points;
    if (est) CK(cudaMemcpy(est, s->est.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
    if (esc) CK(cudaMemcpy(esc, s->esc.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    if (steps) CK(cudaMemcpy(steps, s->steps.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  });
}

int wostgpu_solver_counters(wg_solver s, int64_t* walks, int64_t* steps, int64_t* escaped,
                            int64_t* records) {
  return guarded([&] {
    if (walks) *walks = (int64_t)s->last_counters[2];
    if (steps) *steps = (int64_t)s->last_counters[0];
    if (escaped) *escaped = (int64_t)s->last_counters[1];
    if (records) *records = (int64_t)s->last_counters[5];
  });
}

int wostgpu_train_round(wg_solver s, const wg_train_config* cfg, uint64_t round,
                        wg_train_stats* stats) {
  return guarded([&] {
    need(s->have_records, WG_ERR_INVALID, "no collecting round has run");
    wg_train_stats st = train_records(s, s->last_rec_count, *cfg, round, false);
    if (stats) *stats = st;
  });
}

int wostgpu_train_batch(wg_solver s, const wg_guide_record* recs, int64_t n,
                        const wg_train_config* cfg, uint64_t round, wg_train_stats* stats) {
  return guarded([&] {
    need(s->field != nullptr, WG_ERR_INVALID, "training needs a guiding field");
    int64_t cap = std::max<int64_t>(n, 1);
    if (s->rec_capacity < cap) {
      s->recs.alloc(sizeof(DevRecord) * cap);
      s->rec_capacity = cap;
    }
    DBuf hrec;
    hrec.upload(recs, (size_t)n);
    CKL(launch_import_records(hrec.as<wg_guide_record>(), n, s->recs.as<DevRecord>(), s->stream));
    // the selection key of an imported record is its index mixed with the round
    wg_train_stats st = train_records(s, n, *cfg, round, false);
    st.records_seen = n;
    s->have_records = false;
    if (stats) *stats = st;
  });
}

int wostgpu_field_grad(wg_solver s, const wg_guide_record* recs, int64_t n,
                       const wg_train_config* cfg, double* grad) {
  return guarded([&] {
    wg_field_s* f = s->field;
    need(f != nullptr, WG_ERR_INVALID, "gradient needs a guiding field");
    need(default_shape(f->view), WG_ERR_NOT_BUILT,
         "device training is built for the default field shape");
    int64_t cap = std::max<int64_t>(n, 1);
    if (s->rec_capacity < cap) {
      s->recs.alloc(sizeof(DevRecord) * cap);
      s->rec_capacity = cap;
    }
    DBuf hrec;
    hrec.upload(recs, (size_t)n);
    CKL(launch_import_records(hrec.as<wg_guide_record>(), n, s->recs.as<DevRecord>(), s->stream));
    ensure_train_buffers(s, cap);
    // identity order, pdf floor applied by zero-weighting below the floor
    std::vector<uint32_t> ord;
    std::vector<wg_guide_record> keep;
    for (int64_t i = 0; i < n; ++i)
      if (recs[i].pdf_mis >= cfg->pdf_floor) ord.push_back((uint32_t)i);
    CK(cudaMemcpyAsync(s->idx_sorted.p, ord.data(), sizeof(uint32_t) * ord.size(),
                       cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemsetAsync(s->grad.p, 0, sizeof(float) * (f->n_params + 1), s->stream));
    s->counters.alloc(64);
    CK(cudaMemsetAsync(s->counters.p, 0, 64, s->stream));
    TrainArgs ta{};
    ta.f = f->view;
    ta.recs = s->recs.as<DevRecord>();
    ta.order = s->idx_sorted.as<uint32_t>();
    ta.begin = 0;
    ta.count = (int64_t)ord.size();
    ta.grad = s->grad.as<float>();
    ta.inv_count = 1.0 / static_cast<double>(n);
    ta.reflect = cfg->reflect;
    ta.learn_selection = cfg->learn_selection;
    ta.e_fraction = cfg->e_fraction;
    ta.v_floor = cfg->v_floor;
    ta.counters = s->counters.as<unsigned long long>();
    const bool use_tc = s->mlp == WG_MLP_TENSOR && tc_grad_available();
    if (ta.count > 0) {
      if (use_tc) CKL(launch_grad_tc(ta, s->stream));
      else CKL(launch_grad_cuda_core(ta, s->stream));
    }
    std::vector<float> g(f->n_params);
    CK(cudaMemcpyAsync(g.data(), s->grad.p, sizeof(float) * f->n_params, cudaMemcpyDeviceToHost,
                       s->stream));
    CK(cudaStreamSynchronize(s->stream));
    for (int64_t i = 0; i < f->n_params; ++i) grad[i] = g[i];
  });
}

int wostgpu_run(wg_solver s, uint64_t seed, int32_t wpp, int64_t train_until,
                const wg_train_config* tcfg, wg_train_stats* totals, double* device_ms) {
  return guarded([&] {
    need(wpp >= 1, WG_ERR_INVALID, "wpp must be >= 1");
    if (!s->ev_run0) {
      CK(cudaEventCreate(&s->ev_run0));
      CK(cudaEventCreate(&s->ev_run1));
    }
    s->run_walk_ms = s->run_train_ms = 0;
    s->run_walks = s->run_steps = s->run_escaped = s->run_train_steps = 0;
    wg_train_stats tot{};
    const bool guided = s->cfg.mode != WG_MODE_UNIFORM;
    CK(cudaEventRecord(s->ev_run0, s->stream));
    int32_t b = 0;
    auto account = [&]() {
      s->run_walk_ms += s->last_walk_ms;
      s->run_walks += (int64_t)s->last_counters[2];
      s->run_steps += (int64_t)s->last_counters[0];
      s->run_escaped += (int64_t)s->last_counters[1];
    };
    // Engine::run_batch while training is active (solver.cpp:92-104)
    for (; b < wpp && guided && tcfg && (int64_t)b < train_until; ++b) {
      uint64_t key_seed = Pcg::mix(seed ^ 0x7261696e5f6b6579ULL) ^ Pcg::mix((uint64_t)b + 1);
      run_rounds(s, seed, (uint64_t)b, 1, true, key_seed);
      account();
      s->run_train_steps += (int64_t)s->last_counters[0];
      wg_train_stats st = train_records(s, s->last_rec_count, *tcfg, (uint64_t)b, false);
      s->run_train_ms += s->last_train_ms;
      // TrainStats::merge (guide_train.cpp:12-23)
      double total = (double)(tot.steps + st.steps);
      if (total > 0)
        tot.mean_grad_norm = (tot.mean_grad_norm * tot.steps + st.mean_grad_norm * st.steps) / total;
      tot.records_seen += st.records_seen;
      tot.records_consumed += st.records_consumed;
      tot.skipped_low_pdf += st.skipped_low_pdf;
      tot.skipped_low_v += st.skipped_low_v;
      tot.steps += st.steps;
      tot.seconds += st.seconds;
    }
    // the remaining rounds share a frozen field: one multi-round launch
    if (b < wpp) {
      run_rounds(s, seed, (uint64_t)b, wpp - b, false, 0);
      account();
    }
    CK(cudaEventRecord(s->ev_run1, s->stream));
    CK(cudaEventSynchronize(s->ev_run1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, s->ev_run0, s->ev_run1));
    if (device_ms) *device_ms = ms;
    if (totals) *totals = tot;
  });
}

int wostgpu_run_profile(wg_solver s, double* walk_ms, double* train_ms, int64_t* walks,
                        int64_t* steps, int64_t* escaped, int64_t* train_steps) {
  return guarded([&] {
    if (walk_ms) *walk_ms = s->run_walk_ms;
    if (train_ms) *train_ms = s->run_train_ms;
    if (walks) *walks = s->run_walks;
    if (steps) *steps = s->run_steps;
    if (escaped) *escaped = s->run_escaped;
    if (train_steps) *train_steps = s->run_train_steps;
  });
}

int wostgpu_comm_unique_id(char id[128]) {
  return guarded([&] {
    ncclUniqueId u;
    NCK(ncclGetUniqueId(&u));
    static_assert(sizeof(u) == 128, "nccl id size");
    std::memcpy(id, &u, 128);
  });
}

int wostgpu_solver_attach_comm(wg_solver s, const char id[128], int32_t nranks, int32_t rank) {
  return guarded([&] {
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    NCK(ncclCommInitRank(&s->comm, nranks, u, rank));
    s->nranks = nranks;
    s->rank = rank;
  });
}

int wostgpu_solver_timing(wg_solver s, double* walk_ms, double* train_ms) {
  return guarded([&] {
    if (walk_ms) *walk_ms = s->last_walk_ms;
    if (train_ms) *train_ms = s->last_train_ms;
  });
}

}  // extern "C"
