// 3D walk-on-stars on device (SURVEY.md §8 a′, configs 4-5): the walk
// kernel, the 3D field's evaluation and training tile, and the solver3
// C-ABI (include/wostgpu3.h). Contract: oracle/wost3d.inc (the 3D analogue
// of begin_step / finish_step, proj/src/wost.cpp:148-264, and of
// train_batch, proj/src/guide_train.cpp:94-198).
//
// Walks: one CUDA thread per walk slot, refilled from a grid-strided walk
// index space (round-major) when its walk ends, like the 2D CUDA-core
// kernel (wg_walk.cu). Geometry, sampling and the walk state are fp64 in the
// oracle's operation order (this TU compiles with -fmad=false); the guided
// direction comes from the exact fp32 field evaluation with the MLP staged
// in shared memory, then fp64 normalisation and d = 3 MIS (wg3_mix.cuh).
//
// Records reuse the 2D arena and its device pipeline (finalize, compact,
// Adam; wg_train.cu): a DevRecord3 has DevRecord's size and the offsets the
// shared kernels read (flags, walk, key, thr_q, pdf_mis, target), and stores
// z, nu_z, n_z in the slots 3D never uses (dacc: 3D scenes have no local
// source / flux terms, so targets are |S_K / Q_k| without a chain walk).
#include <cstdio>
#include <cstdlib>
#include <string>
#include <map>

#include "wg3_runtime.hpp"
#include "wg3_walk_common.cuh"
#include "wg_wpack.cuh"

namespace wg3 {

// begin_step's first-step geometry at every start point (StartGeo3): the
// same calls, in the same order and arithmetic, as step_begin makes for a
// walk at depth 0 (so cached and queried answers are bit-identical)
__global__ void start_geo3_kernel(Scene3View s, const double* points, int64_t n, StartGeo3* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const D3 x{points[3 * i], points[3 * i + 1], points[3 * i + 2]};
  const CP3 cd = closest_dirichlet_seeded(s, x, -1);
  const double dd = cd.tri >= 0 ? sqrt(cd.d2) : dinf();
  const double bound2 = dd == dinf() ? dinf() : dd * dd;
  out[i] = StartGeo3{cd, closest_silhouette_d2(s, x, bound2)};
}

template <bool GUIDED>
__global__ void __launch_bounds__(128) walk3_kernel(Walk3Args a) {
  extern __shared__ __align__(16) float mlp_s[];
  if (GUIDED) {
    for (int i = threadIdx.x; i < a.f.mlp_count; i += blockDim.x) mlp_s[i] = a.f.p[a.f.w1 + i];
    __syncthreads();
  }
  const bool collect = a.recs != nullptr;
  const int64_t total = a.n_points * static_cast<int64_t>(a.n_rounds);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t next = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  Lane3 w;
  w.alive = false;
  w.rec_base = 0;
  w.rec_left = 0;
  int64_t walks_done = 0;
  for (;;) {
    if (!w.alive) {
      if (next >= total) break;
      lane3_init(w, a, next);
      next += stride;
      ++walks_done;
    }
    int rec;
    if (!step_begin(w, a, collect, rec)) continue;
    if (GUIDED) {
      Mix3<K8> m;
      {
        float raw[OD];
        field3_eval_exact<IN, HID, OD>(a.f, mlp_s, w.x.x, w.x.y, w.x.z, raw);
        decode3(raw, a.sp, m);
      }
      step_finish(w, a, collect, rec, &m);
    } else {
      step_finish(w, a, collect, rec, nullptr);
    }
  }
  // unused slots of this lane's record chunk are marked invalid
  if (collect)
    for (int i = 0; i < w.rec_left; ++i) a.recs[w.rec_base + (8 - w.rec_left) + i].flags = 0u;
  unsigned long long wd = static_cast<unsigned long long>(walks_done);
  for (int o = 16; o > 0; o >>= 1) wd += __shfl_down_sync(0xffffffffu, wd, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&a.counters[2], wd);
}

__global__ void __launch_bounds__(128) field3_eval_kernel(Field3View f, int64_t n, const double* x,
                                                          double* out) {
  extern __shared__ __align__(16) float mlp_s[];
  for (int i = threadIdx.x; i < f.mlp_count; i += blockDim.x) mlp_s[i] = f.p[f.w1 + i];
  __syncthreads();
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float o[OD];
    field3_eval_exact<IN, HID, OD>(f, mlp_s, x[3 * i], x[3 * i + 1], x[3 * i + 2], o);
    for (int j = 0; j < OD; ++j) out[i * OD + j] = o[j];
  }
}

// ---------------------------------------------------------------- training
// CUDA-core tile, 128 records per CTA, thread = record (the 3D counterpart of
// wg_train.cu's grad_tile_kernel): fp32 trilinear gather and MLP, the fp64
// loss gradient at the outputs (record_dy3), backward with activations in
// padded shared-memory rows, dW as tile GEMMs with one atomic per weight per
// CTA, grid corners by atomics.
struct Grad3Args {
  Field3View f;
  const DevRecord3* recs;
  const uint32_t* list;
  const unsigned long long* count;
  int64_t list_cap;
  float* grad;  // [n_params + 1]; grad[n_params] = record count
  int64_t n_params;
  double inv_count;
  int32_t reflect, learn_selection;
  double e_fraction, v_floor;
  wg::TrainTotals* totals;
};

constexpr int TB = 128;
constexpr int SX = IN + 1, SH = HID + 1, SY = OD + 1;
constexpr size_t GRAD3_SMEM = sizeof(float) * (MLPN + TB * SX + 4 * TB * SH + TB * SY);

__global__ void __launch_bounds__(TB) grad3_tile_kernel(Grad3Args a) {
  extern __shared__ __align__(16) float sm[];
  float* W = sm;
  float* X = W + MLPN;
  float* H1 = X + TB * SX;
  float* H2 = H1 + TB * SH;
  float* D2 = H2 + TB * SH;
  float* D1 = D2 + TB * SH;
  float* DY = D1 + TB * SH;
  const Field3View& f = a.f;
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
  DevRecord3 r{};
  if (live) r = a.recs[a.list[ri]];
  // trilinear gather keeping the 8 corners per level
  float x[IN];
  int cidx[8 * 4];
  float cw[8 * 4];
  {
    float u = static_cast<float>(wg::sclamp((static_cast<double>(r.x) - f.bbox[0]) / (f.bbox[3] - f.bbox[0]), 0.0, 1.0));
    float v = static_cast<float>(wg::sclamp((static_cast<double>(r.y) - f.bbox[1]) / (f.bbox[4] - f.bbox[1]), 0.0, 1.0));
    float q = static_cast<float>(wg::sclamp((static_cast<double>(r.z) - f.bbox[2]) / (f.bbox[5] - f.bbox[2]), 0.0, 1.0));
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int res = f.res[l];
      const float rm = static_cast<float>(res - 1);
      float px = u * rm, py = v * rm, pz = q * rm;
      int ix = wg::imin(static_cast<int>(px), res - 2), iy = wg::imin(static_cast<int>(py), res - 2),
          iz = wg::imin(static_cast<int>(pz), res - 2);
      float fx = px - ix, fy = py - iy, fz = pz - iz, gx = 1.0f - fx, gy = 1.0f - fy, gz = 1.0f - fz;
      const int sy = res * 4, sz = res * res * 4;
      const int c0 = f.lvl_off[l] + ((iz * res + iy) * res + ix) * 4;
      const int ci[8] = {c0, c0 + 4, c0 + sy, c0 + sy + 4, c0 + sz, c0 + sz + 4, c0 + sz + sy, c0 + sz + sy + 4};
      const float w8[8] = {gx * gy * gz, fx * gy * gz, gx * fy * gz, fx * fy * gz,
                           gx * gy * fz, fx * gy * fz, gx * fy * fz, fx * fy * fz};
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        cidx[8 * l + c] = ci[c];
        cw[8 * l + c] = w8[c];
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
  float dy[OD];
  bool used = false;
  if (live) {
    const bool on_n = (r.flags & REC_ON_NEUMANN) != 0;
    used = record_dy3<K8>(y, D3{r.nux, r.nuy, r.nuz}, D3{r.nx, r.ny, r.nz}, on_n, r.target, r.pdf_mis,
                          r.pdf_u, a.reflect != 0, a.learn_selection != 0, a.e_fraction, a.v_floor,
                          a.inv_count, dy);
  }
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
  if (used) {
#pragma unroll
    for (int l = 0; l < 4; ++l)
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int q = 0; q < 4; ++q) atomicAdd(a.grad + cidx[8 * l + c] + q, cw[8 * l + c] * dx[4 * l + q]);
  }
  __syncthreads();
  for (int e = t; e < HID * OD; e += TB) {
    int i = e / OD, j = e % OD;
    float acc = 0.0f;
    for (int q = 0; q < TB; ++q) acc = fmaf(H2[q * SH + i], DY[q * SY + j], acc);
    atomicAdd(a.grad + f.w3 + e, acc);
  }
  for (int e = t; e < HID * HID; e += TB) {
    int i = e / HID, j = e % HID;
    float acc = 0.0f;
    for (int q = 0; q < TB; ++q) acc = fmaf(H1[q * SH + i], D2[q * SH + j], acc);
    atomicAdd(a.grad + f.w2 + e, acc);
  }
  for (int e = t; e < IN * HID; e += TB) {
    int i = e / HID, j = e % HID;
    float acc = 0.0f;
    for (int q = 0; q < TB; ++q) acc = fmaf(X[q * SX + i], D1[q * SH + j], acc);
    atomicAdd(a.grad + f.w1 + e, acc);
  }
  if (t < OD) {
    float acc = 0.0f;
    for (int q = 0; q < TB; ++q) acc += DY[q * SY + t];
    atomicAdd(a.grad + f.b3 + t, acc);
  }
  if (t < HID) {
    float a1 = 0.0f, a2 = 0.0f;
    for (int q = 0; q < TB; ++q) {
      a1 += D1[q * SH + t];
      a2 += D2[q * SH + t];
    }
    atomicAdd(a.grad + f.b1 + t, a1);
    atomicAdd(a.grad + f.b2 + t, a2);
  }
}

__global__ void import3_kernel(const wg_guide_record3* in, int64_t n, DevRecord3* out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const wg_guide_record3& s = in[i];
    DevRecord3 r{};
    r.x = static_cast<float>(s.x[0]);
    r.y = static_cast<float>(s.x[1]);
    r.z = static_cast<float>(s.x[2]);
    r.nux = static_cast<float>(s.nu[0]);
    r.nuy = static_cast<float>(s.nu[1]);
    r.nuz = static_cast<float>(s.nu[2]);
    r.nx = static_cast<float>(s.normal[0]);
    r.ny = static_cast<float>(s.normal[1]);
    r.nz = static_cast<float>(s.normal[2]);
    r.pdf_mis = static_cast<float>(s.pdf_mis);
    r.pdf_g = static_cast<float>(s.pdf_g);
    r.pdf_u = static_cast<float>(s.pdf_u);
    r.c = static_cast<float>(s.c);
    r.target = static_cast<float>(s.target);
    r.thr_q = 1.0f;
    r.walk = -1;  // imported: keeps its target
    r.flags = REC_WRITTEN | (s.on_neumann ? REC_ON_NEUMANN : 0u);
    r.key = Pcg::mix(static_cast<uint64_t>(i) + 0x9e3779b97f4a7c15ULL);
    r.prev = -1;
    out[i] = r;
  }
}

__global__ void export3_kernel(const DevRecord3* in, int64_t n, wg_guide_record3* out,
                               unsigned long long* count) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const DevRecord3& r = in[i];
    if (!(r.flags & wg::REC_VALID)) continue;
    unsigned long long k = atomicAdd(count, 1ull);
    wg_guide_record3 o{};
    o.x[0] = r.x;
    o.x[1] = r.y;
    o.x[2] = r.z;
    o.nu[0] = r.nux;
    o.nu[1] = r.nuy;
    o.nu[2] = r.nuz;
    o.normal[0] = r.nx;
    o.normal[1] = r.ny;
    o.normal[2] = r.nz;
    o.target = r.target;
    o.pdf_mis = r.pdf_mis;
    o.pdf_g = r.pdf_g;
    o.pdf_u = r.pdf_u;
    o.c = r.c;
    o.on_neumann = (r.flags & REC_ON_NEUMANN) ? 1 : 0;
    out[k] = o;
  }
}

}  // namespace wg3

// ================================================================ host
using namespace wgrt;
using namespace wg3;

namespace {

enum { C_STEPS = 0, C_ESCAPED = 1, C_WALKS = 2, C_REC_OVERFLOW = 3, C_SCENE_ERR = 4, C_WAVE_LAUNCHES = 5, C_N = 8 };

void field3_layout(wg_field_s* f) {
  const wg_field_config& c = f->cfg;
  Field3View& v = f->view3;
  v = Field3View{};
  int64_t off = 0;
  v.levels = c.n_levels;
  v.F = c.features;
  for (int l = 0; l < c.n_levels; ++l) {
    v.res[l] = c.level_res[l];
    v.lvl_off[l] = static_cast<int32_t>(off);
    off += static_cast<int64_t>(c.level_res[l]) * c.level_res[l] * c.level_res[l] * c.features;
  }
  v.in = c.n_levels * c.features;
  v.hid = c.hidden;
  v.k = c.mixture_k;
  v.od = 5 * c.mixture_k + 1;
  v.w1 = static_cast<int32_t>(off);
  off += static_cast<int64_t>(v.in) * v.hid;
  v.b1 = static_cast<int32_t>(off);
  off += v.hid;
  v.w2 = static_cast<int32_t>(off);
  off += static_cast<int64_t>(v.hid) * v.hid;
  v.b2 = static_cast<int32_t>(off);
  off += v.hid;
  v.w3 = static_cast<int32_t>(off);
  off += static_cast<int64_t>(v.hid) * v.od;
  v.b3 = static_cast<int32_t>(off);
  off += v.od;
  v.mlp_count = static_cast<int32_t>(off - v.w1);
  need(off < (int64_t(1) << 31), WG_ERR_INVALID, "3D field: parameter count exceeds int32");
  f->n_params = off;
  for (int i = 0; i < 6; ++i) v.bbox[i] = f->bbox3[i];
  for (int i = 0; i < 3; ++i) v.inv_ext[i] = 1.0 / (f->bbox3[i + 3] - f->bbox3[i]);
}

wg::SolverParams params3(const wg_solver3_s* s) {
  wg::SolverParams p{};
  p.eps = s->cfg.epsilon_shell > 0.0 ? s->cfg.epsilon_shell : s->scene->eps;
  p.rmin = s->cfg.r_min > 0.0 ? s->cfg.r_min : p.eps;
  p.fixed_c = s->cfg.fixed_c;
  p.clamp_grazing = s->cfg.clamp_grazing;
  p.grazing_floor = s->cfg.grazing_floor;
  p.rr_depth = s->cfg.rr_depth;
  p.max_steps = s->cfg.max_steps;
  p.mode = s->cfg.mode;
  p.reflect = s->cfg.reflect_at_neumann;
  return p;
}

struct Ev3 {  // event pairs around walk launches / training rounds of one call
  std::vector<cudaEvent_t> walk, train;
  int nw = 0, nt = 0;
};
std::map<const wg_solver3_s*, Ev3>& events() {
  static std::map<const wg_solver3_s*, Ev3> m;
  return m;
}
cudaEvent_t ev_next(std::vector<cudaEvent_t>& pool, int& used) {
  if (used == static_cast<int>(pool.size())) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    pool.push_back(e);
  }
  return pool[used++];
}
double ev_ms(const std::vector<cudaEvent_t>& pool, int used) {
  double ms = 0.0;
  for (int i = 0; i + 1 < used; i += 2) {
    float t = 0.0f;
    CK(cudaEventElapsedTime(&t, pool[i], pool[i + 1]));
    ms += t;
  }
  return ms;
}

void reset3(wg_solver3_s* s) {
  s->counters.alloc(sizeof(unsigned long long) * C_N);
  CK(cudaMemsetAsync(s->counters.p, 0, sizeof(unsigned long long) * C_N, s->st));
  s->totals.alloc(sizeof(wg::TrainTotals));
  CK(cudaMemsetAsync(s->totals.p, 0, sizeof(wg::TrainTotals), s->st));
  Ev3& e = events()[s];
  e.nw = e.nt = 0;
}

int walk3_blocks_per_sm(bool guided, int smem) {
  int n = 0;
  if (guided)
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, walk3_kernel<true>, 128, smem));
  else
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, walk3_kernel<false>, 128, smem));
  return std::max(n, 1);
}

void enqueue3_rounds(wg_solver3_s* s, uint64_t seed, uint64_t wpp_first, int32_t rounds, bool collect,
                     uint64_t key_seed) {
  need(s->n_points > 0, WG_ERR_INVALID, "solver has no evaluation points");
  const bool guided = s->cfg.mode != WG_MODE_UNIFORM;
  need(!guided || s->field, WG_ERR_INVALID, "guided sampler modes need a guiding field");
  need(!collect || rounds == 1, WG_ERR_INVALID, "record collection runs one round at a time");
  int32_t chunk = static_cast<int32_t>(std::max<int64_t>(1, (int64_t(1) << 30) / (s->n_points * 16)));
  chunk = std::min(chunk, rounds);
  if (s->last_rounds < chunk) {
    s->est.alloc(sizeof(double) * s->n_points * chunk);
    s->esc.alloc(sizeof(int32_t) * s->n_points * chunk);
    s->steps.alloc(sizeof(int32_t) * s->n_points * chunk);
    s->last_rounds = chunk;
  }
  if (collect) {
    // 3D walks average ~20 steps (cfg 4): 48 records per point, doubled for
    // the next call after any overflow (as in 2D); 80 + 4 B per record
    int64_t cap = std::max<int64_t>({s->n_points * 48, int64_t(1) << 16, s->rec_cap_min});
    if (s->rec_cap < cap) {
      s->recs.alloc(sizeof(DevRecord3) * cap);
      s->rec_dacc.alloc(sizeof(float) * cap);
      s->rec_cap = cap;
    }
    s->rec_counter.alloc(sizeof(unsigned long long));
    CK(cudaMemsetAsync(s->rec_counter.p, 0, sizeof(unsigned long long), s->st));
    s->rec_tail.alloc(sizeof(int32_t) * s->n_points);
    s->rec_term.alloc(sizeof(double) * s->n_points);
    CK(cudaMemsetAsync(s->rec_tail.p, 0xFF, sizeof(int32_t) * s->n_points, s->st));
    s->have_records = true;
  }
  Walk3Args a{};
  a.s = s->scene->view;
  if (guided) a.f = s->field->view3;
  a.sp = params3(s);
  a.points = s->points.as<double>();
  a.n_points = s->n_points;
  a.point_offset = s->point_offset;
  a.seed = seed;
  a.est = s->est.as<double>();
  a.esc = s->esc.as<int32_t>();
  a.steps = s->steps.as<int32_t>();
  a.counters = s->counters.as<unsigned long long>();
  a.recs = collect ? s->recs.as<DevRecord3>() : nullptr;
  a.rec_counter = collect ? s->rec_counter.as<unsigned long long>() : nullptr;
  a.rec_capacity = s->rec_cap;
  a.key_seed = key_seed;
  a.rec_tail = collect ? s->rec_tail.as<int32_t>() : nullptr;
  a.rec_term = collect ? s->rec_term.as<double>() : nullptr;
  a.rec_dacc = collect ? s->rec_dacc.as<float>() : nullptr;
  if (!s->start_ok) {  // once per point set (the scene is fixed per solver)
    s->start_geo.alloc(sizeof(StartGeo3) * s->n_points);
    start_geo3_kernel<<<static_cast<unsigned>((s->n_points + 127) / 128), 128, 0, s->st>>>(
        s->scene->view, s->points.as<double>(), s->n_points, s->start_geo.as<StartGeo3>());
    CKL(cudaGetLastError());
    s->start_ok = true;
  }
  a.start = s->start_geo.as<StartGeo3>();
  const bool tc = guided && s->mlp == WG_MLP_TENSOR;
  const int smem = guided ? static_cast<int>(sizeof(float) * s->field->view3.mlp_count) : 0;
  if (guided && !tc)
    CK(cudaFuncSetAttribute(walk3_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  static int per_sm[2] = {0, 0};
  if (!tc && !per_sm[guided]) per_sm[guided] = walk3_blocks_per_sm(guided, smem);
  const int sm_blocks = tc ? walk3_tc_blocks_per_sm() : per_sm[guided];
  const int sms = sm_count();
  Ev3& e = events()[s];
  for (int32_t r0 = 0; r0 < rounds; r0 += chunk) {
    const int32_t n = std::min(chunk, rounds - r0);
    a.wpp_first = wpp_first + r0;
    a.n_rounds = n;
    const int64_t want = (s->n_points * n + 127) / 128;
    const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_blocks * sms)));
    CK(cudaEventRecord(ev_next(e.walk, e.nw), s->st));
    // wavefront pair once enough walks are in flight to fill the GPU (measured
    // on cfg 4, 512^2 points: 9.0M vs 3.0M walks/s multi-round, 4.4M vs 2.5M
    // per training round); lockstep tiles below that (128^2 training rounds:
    // the wavefront's per-iteration launches dominate). WOSTGPU_WALK3 =
    // wave / lockstep forces one.
    const char* fe = std::getenv("WOSTGPU_WALK3");
    const int force = !fe ? 0 : std::string(fe) == "wave" ? 1 : std::string(fe) == "lockstep" ? 2 : 0;
    const bool wave = force == 1 || (force == 0 && s->n_points * n >= 65536);
    if (tc && wave) {
      // walk slots in flight: 96 x 128 per SM (1.8M on B200, ~220 B each).
      // More walks in flight keep the spatially sorted geometry pass
      // coherent and hide its latency: cfg 4 frozen rounds (512^2 x 256)
      // 1.93 / 1.75 / 1.66 / 1.61 / 1.61 s at 16 / 32 / 64 / 96 / 128
      const int64_t slots = std::min<int64_t>(s->n_points * n, (int64_t)sms * 96 * 128);
      if (s->w_slots < slots) {
        s->w_lanes.alloc(sizeof(Lane3) * slots);
        s->w_dirs.alloc(sizeof(Dir3) * slots);
        s->w_rec.alloc(sizeof(int32_t) * slots);
        s->w_state.alloc(slots);
        s->w_queue.alloc(sizeof(int32_t) * slots);
        s->w_perm.alloc(sizeof(int32_t) * slots);
        s->w_sbin.alloc(sizeof(uint16_t) * slots);
        s->w_slots = slots;
      }
      s->w_qlen.alloc(2 * sizeof(unsigned int));
      s->w_next.alloc(sizeof(unsigned long long));
      if (!s->h_qlen) CK(cudaMallocHost(&s->h_qlen, 4 * sizeof(unsigned int)));
      Wave3 v{s->w_lanes.as<Lane3>(), s->w_dirs.as<Dir3>(), s->w_rec.as<int32_t>(), s->w_state.as<uint8_t>(),
              s->w_queue.as<int32_t>(), s->w_qlen.as<unsigned int>(), s->w_next.as<unsigned long long>(),
              slots, nullptr};
      s->w_blob.alloc(wg::wpack::FWD_BYTES);
      v.wblob = s->w_blob.as<unsigned char>();
      s->w_bins.alloc(sizeof(unsigned int) * (kSortBins + 3));
      v.perm = s->w_perm.as<int32_t>();
      v.bins = s->w_bins.as<unsigned int>();
      v.sbin = s->w_sbin.as<uint16_t>();
      int64_t launched = 0;
      CK(launch_walks3_wave(a, v, sms, s->h_qlen, &launched, s->st));
      g_launches += launched;
    } else if (tc) CKL(launch_walks3_tc(a, blocks, s->st));
    else if (guided) walk3_kernel<true><<<blocks, 128, smem, s->st>>>(a);
    else walk3_kernel<false><<<blocks, 128, 0, s->st>>>(a);
    CKL(cudaGetLastError());
    CK(cudaEventRecord(ev_next(e.walk, e.nw), s->st));
    CKL(wg::launch_welford(a.est, a.esc, s->n_points, n, s->stats.as<wg_point_stats>(), s->st));
  }
}

// backfill_targets_append (guide_train.cpp:58-79) for 3D scenes with source /
// flux terms: per walk, backward over its record chain with the fp64 suffix
// sum S (target_k = |S / Q_k|, then S += dacc_k), dacc from the side array
__global__ void backfill3_chains_kernel(DevRecord3* recs, const float* dacc, int64_t n_walks,
                                        const int32_t* tail, const double* term, const int32_t* esc) {
  for (int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < n_walks;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (esc[w]) continue;
    double s = term[w];
    for (int32_t i = tail[w]; i >= 0;) {
      DevRecord3& r = recs[i];
      const double q = r.thr_q;
      r.target = q == 0.0 ? 0.0f : static_cast<float>(fabs(s / q));
      s += static_cast<double>(dacc[i]);
      i = r.prev;
    }
  }
}

void enqueue3_finalize(wg_solver3_s* s, double pdf_floor, bool from_walks) {
  s->ctl.alloc(sizeof(wg::TrainCtl));
  CK(cudaMemsetAsync(s->ctl.p, 0, sizeof(wg::TrainCtl), s->st));
  // scenes with local terms: chain targets here; the shared finalize then
  // keeps them (chain = true, no walks for its 2D chain pass)
  const Scene3View& v = s->scene->view;
  const bool chain = from_walks && (v.source.type != WG_VALUE_ZERO || v.has_flux);
  if (chain) {
    const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((s->n_points + 127) / 128, 148 * 8)));
    backfill3_chains_kernel<<<blocks, 128, 0, s->st>>>(s->recs.as<DevRecord3>(), s->rec_dacc.as<float>(),
                                                       s->n_points, s->rec_tail.as<int32_t>(),
                                                       s->rec_term.as<double>(), s->esc.as<int32_t>());
    CKL(cudaGetLastError());
  }
  CKL(wg::launch_finalize_records(reinterpret_cast<DevRecord*>(s->recs.p),
                                  s->rec_counter.as<unsigned long long>(), s->rec_cap,
                                  from_walks && !chain ? s->n_points : 0, s->rec_tail.as<int32_t>(),
                                  s->rec_term.as<double>(), s->esc.as<int32_t>(), pdf_floor,
                                  s->ctl.as<wg::TrainCtl>(), chain, s->st));
}

void ensure3_train(wg_solver3_s* s, const wg_train_config& tc) {
  need(tc.minibatch >= 1, WG_ERR_INVALID, "minibatch must be >= 1");
  const int n_mb = static_cast<int>((tc.max_records_per_round + tc.minibatch - 1) / tc.minibatch);
  need(n_mb <= wg::kMaxMinibatches, WG_ERR_INVALID, "max_records / minibatch exceeds the device limit");
  int64_t cap = tc.minibatch + tc.minibatch / 4 + 1024;
  if (s->list_cap < cap) {
    s->lists.alloc(sizeof(uint32_t) * wg::kMaxMinibatches * cap);
    s->list_cap = cap;
  }
  s->grad.alloc(sizeof(float) * (s->field->n_params + 1));
}

void enqueue3_minibatch(wg_solver3_s* s, const wg_train_config& tc, int b, double inv_count) {
  wg_field_s* f = s->field;
  CK(cudaMemsetAsync(s->grad.p, 0, sizeof(float) * (f->n_params + 1), s->st));
  if (s->mlp == WG_MLP_TENSOR) {
    // tcgen05 training tile (wg_train_tc.cu): forward, loss gradient and
    // backward of 128 records per tile on the tensor cores; the split-fp16
    // weight blob is packed from the current parameters (Adam moved them
    // since the previous minibatch)
    s->g_blob.alloc(wg::wpack::BYTES);
    CKL(wg::launch_pack3_full(f->view3, s->g_blob.as<unsigned char>(), s->st));
    wg::TrainArgs3 g{};
    g.f = f->view3;
    g.recs = s->recs.as<DevRecord3>();
    g.list = s->lists.as<uint32_t>() + static_cast<int64_t>(b) * s->list_cap;
    g.count = &s->ctl.as<wg::TrainCtl>()->mb_count[b];
    g.list_cap = s->list_cap;
    g.grad = s->grad.as<float>();
    g.n_params = f->n_params;
    g.inv_count = inv_count;
    g.reflect = tc.reflect;
    g.learn_selection = tc.learn_selection;
    g.e_fraction = tc.e_fraction;
    g.v_floor = tc.v_floor;
    g.totals = s->totals.as<wg::TrainTotals>();
    g.packed = s->g_blob.as<unsigned char>();
    CKL(wg::launch_grad3_tc(g, s->st));
    return;
  }
  Grad3Args g{};
  g.f = f->view3;
  g.recs = s->recs.as<DevRecord3>();
  g.list = s->lists.as<uint32_t>() + static_cast<int64_t>(b) * s->list_cap;
  g.count = &s->ctl.as<wg::TrainCtl>()->mb_count[b];
  g.list_cap = s->list_cap;
  g.grad = s->grad.as<float>();
  g.n_params = f->n_params;
  g.inv_count = inv_count;
  g.reflect = tc.reflect;
  g.learn_selection = tc.learn_selection;
  g.e_fraction = tc.e_fraction;
  g.v_floor = tc.v_floor;
  g.totals = s->totals.as<wg::TrainTotals>();
  CK(cudaFuncSetAttribute(grad3_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(GRAD3_SMEM)));
  const int blocks = static_cast<int>((s->list_cap + TB - 1) / TB);
  grad3_tile_kernel<<<blocks, TB, GRAD3_SMEM, s->st>>>(g);
  CKL(cudaGetLastError());
}

void enqueue3_train(wg_solver3_s* s, const wg_train_config& tc, bool from_walks) {
  wg_field_s* f = s->field;
  need(f != nullptr, WG_ERR_INVALID, "training needs a guiding field");
  need(default_shape3(f->view3), WG_ERR_NOT_BUILT,
       "3D training is built for the default 3D field shape (L=4, F=4, hidden 64, K=8)");
  ensure3_train(s, tc);
  Ev3& e = events()[s];
  CK(cudaEventRecord(ev_next(e.train, e.nt), s->st));
  enqueue3_finalize(s, tc.pdf_floor, from_walks);
  // selection rate from the usable count summed over the ranks (wg_train.cu
  // compact_kernel): the cap and minibatch size are global
  wg::TrainCtl* c = s->ctl.as<wg::TrainCtl>();
  if (s->comm)
    NCK(nccl().allReduce(&c->usable, &c->usable_global, 1, ncclUint64, ncclSum, s->comm, s->st));
  else
    CK(cudaMemcpyAsync(&c->usable_global, &c->usable, sizeof(unsigned long long), cudaMemcpyDeviceToDevice,
                       s->st));
  CKL(wg::launch_compact(reinterpret_cast<const DevRecord*>(s->recs.p),
                         s->rec_counter.as<unsigned long long>(), s->rec_cap,
                         s->ctl.as<wg::TrainCtl>(), s->totals.as<wg::TrainTotals>(),
                         s->lists.as<uint32_t>(), s->list_cap, tc.max_records_per_round, tc.minibatch,
                         s->st));
  const int n_mb = static_cast<int>((tc.max_records_per_round + tc.minibatch - 1) / tc.minibatch);
  for (int b = 0; b < n_mb; ++b) {
    enqueue3_minibatch(s, tc, b, 1.0 / static_cast<double>(tc.minibatch));
    if (s->comm)
      NCK(nccl().allReduce(s->grad.p, s->grad.p, f->n_params + 1, ncclFloat, ncclSum, s->comm, s->st));
    CKL(wg::launch_adam(f->p.as<float>(), f->m.as<double>(), f->v.as<double>(), s->grad.as<float>(),
                        f->n_params, tc.lr, tc.beta1, tc.beta2, tc.eps, static_cast<double>(tc.minibatch),
                        f->adam.as<wg::AdamCtl>(), f->view, nullptr, s->st));
  }
  CK(cudaEventRecord(ev_next(e.train, e.nt), s->st));
}

wg_train_stats sync3(wg_solver3_s* s, long long steps_before) {
  CK(cudaStreamSynchronize(s->st));
  unsigned long long c[C_N];
  CK(cudaMemcpy(c, s->counters.p, sizeof(c), cudaMemcpyDeviceToHost));
  // kernels the device-side wavefront loops launched (counted on the device)
  g_launches += static_cast<int64_t>(c[C_WAVE_LAUNCHES]);
  CK(cudaMemset(s->counters.as<unsigned long long>() + C_WAVE_LAUNCHES, 0, sizeof(unsigned long long)));
  if (c[C_REC_OVERFLOW] > 0) {  // as in 2D (wg_solver.cu sync_collect): fail, grow for the next call
    s->rec_cap_min = std::max<int64_t>(s->rec_cap_min, 2 * s->rec_cap);
    char msg[256];
    std::snprintf(msg, sizeof(msg),
                  "3D record arena overflow in a training round (%llu record chunks dropped, capacity %lld "
                  "records); the arena now holds %lld records: rerun, or reserve more with "
                  "wostgpu_solver3_reserve_records",
                  c[C_REC_OVERFLOW], static_cast<long long>(s->rec_cap), static_cast<long long>(s->rec_cap_min));
    throw wgrt::WgError(WG_ERR_RUNTIME, msg);
  }
  Ev3& e = events()[s];
  s->last_walk_ms = static_cast<float>(ev_ms(e.walk, e.nw));
  s->last_train_ms = static_cast<float>(ev_ms(e.train, e.nt));
  need(c[C_SCENE_ERR] == 0, WG_ERR_SCENE, "walk: unbounded star region");
  wg_train_stats st{};
  if (s->field && steps_before >= 0) {
    wg::TrainTotals t{};
    CK(cudaMemcpy(&t, s->totals.p, sizeof(t), cudaMemcpyDeviceToHost));
    long long after = 0;
    CK(cudaMemcpy(&after, s->field->adam.p, sizeof(long long), cudaMemcpyDeviceToHost));
    st.records_seen = (int64_t)t.seen;
    st.records_consumed = (int64_t)t.consumed;
    st.skipped_low_pdf = (int64_t)t.low_pdf;
    st.skipped_low_v = (int64_t)t.skipped_v;
    st.steps = after - steps_before;
    if (st.steps > 0) {
      std::vector<double> n2(wg::kNormRing);
      CK(cudaMemcpy(n2.data(), s->field->adam.as<wg::AdamCtl>()->norm2, sizeof(double) * wg::kNormRing,
                    cudaMemcpyDeviceToHost));
      double acc = 0.0;
      for (long long k = steps_before; k < after; ++k) acc += std::sqrt(n2[k % wg::kNormRing]);
      st.mean_grad_norm = acc / static_cast<double>(st.steps);
    }
    st.seconds = s->last_train_ms * 1e-3;
  }
  return st;
}

long long adam_steps3(wg_solver3_s* s) {
  long long v = 0;
  CK(cudaMemcpyAsync(&v, s->field->adam.p, sizeof(long long), cudaMemcpyDeviceToHost, s->st));
  CK(cudaStreamSynchronize(s->st));
  return v;
}

uint64_t key_seed3(uint64_t seed, uint64_t wpp) {
  return Pcg::mix(seed ^ 0x7261696e5f6b6579ULL) ^ Pcg::mix(wpp + 1);
}

}  // namespace

wg_solver3_s::~wg_solver3_s() {
  if (comm) nccl().commDestroy(comm);
  if (h_qlen) cudaFreeHost(h_qlen);
  if (st) cudaStreamDestroy(st);
  auto it = events().find(this);
  if (it != events().end()) {
    for (cudaEvent_t e : it->second.walk) cudaEventDestroy(e);
    for (cudaEvent_t e : it->second.train) cudaEventDestroy(e);
    events().erase(it);
  }
}

extern "C" {

int wostgpu_field3_create(const wg_field_config* cfg, const double bbox[6], uint64_t seed, wg_field* out) {
  return guarded([&] {
    check_device();
    const wg_field_config& c = *cfg;
    need(c.n_levels >= 1 && c.n_levels <= WG_MAX_LEVELS && c.features >= 1 && c.mixture_k >= 1,
         WG_ERR_INVALID, "guiding field: L, F and K must be >= 1");
    need(c.mixture_k <= WG_MAX_MIXTURE, WG_ERR_INVALID, "guiding field: K exceeds the component cap");
    need(c.mixture_dim == 3, WG_ERR_INVALID, "3D guiding field: mixture dim must be 3");
    need(c.hidden >= 1, WG_ERR_INVALID, "guiding field: hidden width must be >= 1");
    for (int l = 0; l < c.n_levels; ++l)
      need(c.level_res[l] >= 2, WG_ERR_INVALID, "guiding field: grid resolution must be >= 2 per axis");
    need(c.n_levels * c.features <= 256 && c.hidden <= 256, WG_ERR_INVALID,
         "guiding field: L*F and hidden width are capped at 256");
    need(bbox[3] - bbox[0] > 0.0 && bbox[4] - bbox[1] > 0.0 && bbox[5] - bbox[2] > 0.0, WG_ERR_INVALID,
         "guiding field: bbox is empty");
    auto f = std::make_unique<wg_field_s>();
    f->cfg = c;
    f->sdim = 3;
    for (int i = 0; i < 6; ++i) f->bbox3[i] = bbox[i];
    f->bbox[0] = bbox[0];
    f->bbox[1] = bbox[1];
    f->bbox[2] = bbox[3];
    f->bbox[3] = bbox[4];
    field3_layout(f.get());
    // the GuidingField initialisation stream (guide_field.cpp:36-51) over the 3D layout
    std::vector<float> p(static_cast<size_t>(f->n_params), 0.0f);
    Pcg rng;
    rng.seed(Pcg::mix(seed), 0x67e5504410b1426fULL);
    auto uni = [&](double lo, double hi) { return lo + (hi - lo) * rng.uni(); };
    const Field3View& v = f->view3;
    for (int64_t i = 0; i < v.w1; ++i) p[i] = static_cast<float>(uni(-1e-4, 1e-4));
    auto layer = [&](int64_t wo, int64_t wc, int64_t bo, int64_t bc, int fan_in) {
      double sc = 1.0 / std::sqrt(static_cast<double>(fan_in));
      for (int64_t i = 0; i < wc; ++i) p[wo + i] = static_cast<float>(uni(-sc, sc));
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
    f->adam.alloc(sizeof(wg::AdamCtl));
    CK(cudaMemset(f->adam.p, 0, sizeof(wg::AdamCtl)));
    f->view3.p = f->p.as<float>();
    f->view = wg::FieldView{};
    f->view.p = f->p.as<float>();
    f->view.w1 = v.w1;  // unused by the 3D path (no packed blob)
    *out = f.release();
  });
}

int wostgpu_mixture3f_pdf(int64_t n, const float* raw, const double* nu, double* out) {
  return guarded([&] {
    need(n >= 0 && (n == 0 || (raw && nu && out)), WG_ERR_INVALID, "mixture3f_pdf: bad arguments");
    if (n == 0) return;
    DBuf draw, dnu, dout;
    draw.upload(raw, static_cast<size_t>(n) * OD);
    dnu.upload(nu, static_cast<size_t>(n) * 3);
    dout.alloc(sizeof(double) * 2 * n);
    CKL(launch_mix3f_pdf(n, draw.as<float>(), dnu.as<double>(), dout.as<double>(), 0));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out, dout.p, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost));
  });
}

int wostgpu_field3_eval_batch(wg_field f, int64_t n, const double* x, double* out, int mlp) {
  return guarded([&] {
    need(f->sdim == 3, WG_ERR_INVALID, "field3_eval_batch: 2D field");
    need(default_shape3(f->view3), WG_ERR_NOT_BUILT, "3D field evaluation is built for the default 3D shape");
    if (n <= 0) return;
    DBuf dx, dout;
    dx.upload(x, static_cast<size_t>(3 * n));
    dout.alloc(sizeof(double) * n * OD);
    if (mlp == WG_MLP_TENSOR) {
      CKL(launch_field3_eval_tc(f->view3, n, dx.as<double>(), dout.as<double>(), nullptr));
      CK(cudaMemcpy(out, dout.p, sizeof(double) * n * OD, cudaMemcpyDeviceToHost));
      return;
    }
    const int smem = static_cast<int>(sizeof(float) * f->view3.mlp_count);
    CK(cudaFuncSetAttribute(field3_eval_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int blocks = static_cast<int>(std::min<int64_t>((n + 127) / 128, 148 * 8));
    field3_eval_kernel<<<blocks, 128, smem>>>(f->view3, n, dx.as<double>(), dout.as<double>());
    CKL(cudaGetLastError());
    CK(cudaMemcpy(out, dout.p, sizeof(double) * n * OD, cudaMemcpyDeviceToHost));
  });
}

int wostgpu_solver3_create(wg_scene3 scene, wg_field field, const wg_solver_config* cfg, wg_solver3* out) {
  return guarded([&] {
    check_device();
    need(scene != nullptr, WG_ERR_INVALID, "solver needs a scene");
    need(field == nullptr || field->sdim == 3, WG_ERR_INVALID, "3D solver needs a 3D field");
    need(cfg->mode == WG_MODE_UNIFORM || field != nullptr, WG_ERR_INVALID,
         "guided sampler modes need a guiding field");
    if (field) need(default_shape3(field->view3), WG_ERR_NOT_BUILT, "3D walks are built for the default 3D field shape");
    auto s = std::make_unique<wg_solver3_s>();
    s->scene = scene;
    s->field = field;
    s->cfg = *cfg;
    s->mlp = WG_MLP_TENSOR;  // the tensor-core walk kernel for guided modes (exact: set_mlp)
    CK(cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking));
    s->counters.alloc(sizeof(unsigned long long) * C_N);
    CK(cudaMemset(s->counters.p, 0, sizeof(unsigned long long) * C_N));
    *out = s.release();
  });
}

int wostgpu_solver3_set_mlp(wg_solver3 s, int mlp) {
  return guarded([&] {
    need(mlp == WG_MLP_EXACT || mlp == WG_MLP_TENSOR, WG_ERR_INVALID, "mlp must be WG_MLP_EXACT or WG_MLP_TENSOR");
    s->mlp = mlp;
  });
}

int wostgpu_solver3_destroy(wg_solver3 s) {
  return guarded([&] { delete s; });
}

int wostgpu_solver3_set_points(wg_solver3 s, int64_t n, const double* x, int64_t offset) {
  return guarded([&] {
    need(n > 0, WG_ERR_INVALID, "no evaluation points");
    s->points.upload(x, static_cast<size_t>(3 * n));
    s->stats.alloc(sizeof(wg_point_stats) * n);
    CK(cudaMemset(s->stats.p, 0, sizeof(wg_point_stats) * n));
    s->n_points = n;
    s->point_offset = offset;
    s->last_rounds = 0;
    s->have_records = false;
    s->start_ok = false;
  });
}

int wostgpu_solver3_get_stats(wg_solver3 s, wg_point_stats* st) {
  return guarded([&] {
    CK(cudaStreamSynchronize(s->st));
    CK(cudaMemcpy(st, s->stats.p, sizeof(wg_point_stats) * s->n_points, cudaMemcpyDeviceToHost));
  });
}

int wostgpu_solver3_solve_rounds(wg_solver3 s, uint64_t seed, uint64_t wpp_first, int32_t n_rounds,
                                 int32_t collect) {
  return guarded([&] {
    reset3(s);
    enqueue3_rounds(s, seed, wpp_first, n_rounds, collect != 0, key_seed3(seed, wpp_first));
    sync3(s, -1);
  });
}

int wostgpu_solver3_fetch_walks(wg_solver3 s, double* est, int32_t* esc, int32_t* steps) {
  return guarded([&] {
    CK(cudaStreamSynchronize(s->st));
    const size_t n = static_cast<size_t>(s->n_points);
    if (est) CK(cudaMemcpy(est, s->est.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
    if (esc) CK(cudaMemcpy(esc, s->esc.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    if (steps) CK(cudaMemcpy(steps, s->steps.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  });
}

int wostgpu_solver3_fetch_records(wg_solver3 s, wg_guide_record3* out, int64_t capacity, int64_t* n) {
  return guarded([&] {
    need(s->have_records, WG_ERR_INVALID, "no collecting round to fetch records from");
    enqueue3_finalize(s, 1e-8, true);
    unsigned long long used = 0;
    CK(cudaMemcpyAsync(&used, s->rec_counter.p, sizeof(used), cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    const int64_t m = std::min<int64_t>(static_cast<int64_t>(used), s->rec_cap);
    DBuf dout, dcount;
    dout.alloc(sizeof(wg_guide_record3) * std::max<int64_t>(m, 1));
    dcount.alloc(sizeof(unsigned long long));
    CK(cudaMemsetAsync(dcount.p, 0, sizeof(unsigned long long), s->st));
    const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, 148 * 4)));
    export3_kernel<<<blocks, 256, 0, s->st>>>(s->recs.as<DevRecord3>(), m, dout.as<wg_guide_record3>(),
                                               dcount.as<unsigned long long>());
    CKL(cudaGetLastError());
    unsigned long long k = 0;
    CK(cudaMemcpyAsync(&k, dcount.p, sizeof(k), cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    *n = static_cast<int64_t>(k);
    if (out) CK(cudaMemcpy(out, dout.p, sizeof(wg_guide_record3) * std::min<int64_t>(k, capacity),
                           cudaMemcpyDeviceToHost));
  });
}

int wostgpu_solver3_counters(wg_solver3 s, int64_t* walks, int64_t* steps, int64_t* escaped, int64_t* records) {
  return guarded([&] {
    CK(cudaStreamSynchronize(s->st));
    unsigned long long c[C_N];
    CK(cudaMemcpy(c, s->counters.p, sizeof(c), cudaMemcpyDeviceToHost));
    if (walks) *walks = (int64_t)c[C_WALKS];
    if (steps) *steps = (int64_t)c[C_STEPS];
    if (escaped) *escaped = (int64_t)c[C_ESCAPED];
    if (records) {
      unsigned long long r = 0;
      if (s->have_records) CK(cudaMemcpy(&r, s->rec_counter.p, sizeof(r), cudaMemcpyDeviceToHost));
      *records = (int64_t)std::min<unsigned long long>(r, (unsigned long long)s->rec_cap);
    }
  });
}

int wostgpu_solver3_train_round(wg_solver3 s, const wg_train_config* cfg, uint64_t round, wg_train_stats* st) {
  return guarded([&] {
    (void)round;
    need(s->have_records, WG_ERR_INVALID, "train_round needs a collecting round");
    need(s->field != nullptr, WG_ERR_INVALID, "training needs a guiding field");
    const long long before = adam_steps3(s);
    reset3(s);
    enqueue3_train(s, *cfg, true);
    wg_train_stats r = sync3(s, before);
    if (st) *st = r;
  });
}

int wostgpu_solver3_field_grad(wg_solver3 s, const wg_guide_record3* recs, int64_t n,
                               const wg_train_config* cfg, double* grad) {
  return guarded([&] {
    need(s->field != nullptr, WG_ERR_INVALID, "field_grad needs a guiding field");
    need(n > 0, WG_ERR_INVALID, "field_grad needs records");
    wg_train_config tc = *cfg;
    tc.minibatch = static_cast<int32_t>(n);
    tc.max_records_per_round = n;
    reset3(s);
    ensure3_train(s, tc);
    if (s->rec_cap < n) {
      s->recs.alloc(sizeof(DevRecord3) * n);
      s->rec_dacc.alloc(sizeof(float) * n);
      s->rec_cap = n;
    }
    DBuf h;
    h.upload(recs, static_cast<size_t>(n));
    const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 4));
    import3_kernel<<<blocks, 256, 0, s->st>>>(h.as<wg_guide_record3>(), n, s->recs.as<DevRecord3>());
    CKL(cudaGetLastError());
    s->rec_counter.alloc(sizeof(unsigned long long));
    unsigned long long nn = static_cast<unsigned long long>(n);
    CK(cudaMemcpyAsync(s->rec_counter.p, &nn, sizeof(nn), cudaMemcpyHostToDevice, s->st));
    enqueue3_finalize(s, -1.0, false);  // every record usable, in order
    // the minibatch list is the records in order (no selection)
    std::vector<uint32_t> order(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) order[i] = static_cast<uint32_t>(i);
    CK(cudaMemcpyAsync(s->lists.p, order.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice, s->st));
    CK(cudaMemcpyAsync(&s->ctl.as<wg::TrainCtl>()->mb_count[0], &nn, sizeof(nn), cudaMemcpyHostToDevice, s->st));
    enqueue3_minibatch(s, tc, 0, 1.0 / static_cast<double>(n));
    std::vector<float> g(static_cast<size_t>(s->field->n_params));
    CK(cudaMemcpyAsync(g.data(), s->grad.p, sizeof(float) * g.size(), cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    for (size_t i = 0; i < g.size(); ++i) grad[i] = g[i];
    s->have_records = false;
  });
}

int wostgpu_solver3_run(wg_solver3 s, uint64_t seed, int32_t wpp, int64_t train_until,
                        const wg_train_config* tcfg, wg_train_stats* totals, double* device_ms) {
  return guarded([&] {
    need(wpp >= 0, WG_ERR_INVALID, "wpp must be >= 0");
    const bool guided = s->cfg.mode != WG_MODE_UNIFORM;
    const bool train = guided && tcfg != nullptr && s->field != nullptr;
    const long long before = train ? adam_steps3(s) : -1;
    reset3(s);
    CK(cudaMemsetAsync(s->stats.p, 0, sizeof(wg_point_stats) * s->n_points, s->st));
    if (!s->ev[0]) {
      CK(cudaEventCreate(&s->ev[0]));
      CK(cudaEventCreate(&s->ev[1]));
    }
    CK(cudaEventRecord(s->ev[0], s->st));
    int32_t b = 0;
    const int64_t tu = train ? std::min<int64_t>(train_until, wpp) : 0;
    for (; b < tu; ++b) {
      enqueue3_rounds(s, seed, (uint64_t)b, 1, true, key_seed3(seed, (uint64_t)b));
      enqueue3_train(s, *tcfg, true);
    }
    // training-round walk steps = steps counted so far
    DBuf snap;
    snap.alloc(sizeof(unsigned long long));
    CK(cudaMemcpyAsync(snap.p, s->counters.as<unsigned long long>() + C_STEPS, sizeof(unsigned long long),
                       cudaMemcpyDeviceToDevice, s->st));
    if (b < wpp) enqueue3_rounds(s, seed, (uint64_t)b, wpp - b, false, 0);
    CK(cudaEventRecord(s->ev[1], s->st));
    wg_train_stats st = sync3(s, before);
    float ms = 0.0f;
    CK(cudaEventElapsedTime(&ms, s->ev[0], s->ev[1]));
    if (device_ms) *device_ms = ms;
    if (totals) *totals = st;
    unsigned long long c[C_N], ts = 0;
    CK(cudaMemcpy(c, s->counters.p, sizeof(c), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&ts, snap.p, sizeof(ts), cudaMemcpyDeviceToHost));
    s->prof_walk_ms = s->last_walk_ms;
    s->prof_train_ms = s->last_train_ms;
    s->prof_walks = (int64_t)c[C_WALKS];
    s->prof_steps = (int64_t)c[C_STEPS];
    s->prof_escaped = (int64_t)c[C_ESCAPED];
    s->prof_train_steps = (int64_t)ts;
  });
}

int wostgpu_solver3_run_profile(wg_solver3 s, double* walk_ms, double* train_ms, int64_t* walks,
                                int64_t* steps, int64_t* escaped, int64_t* train_steps) {
  return guarded([&] {
    if (walk_ms) *walk_ms = s->prof_walk_ms;
    if (train_ms) *train_ms = s->prof_train_ms;
    if (walks) *walks = s->prof_walks;
    if (steps) *steps = s->prof_steps;
    if (escaped) *escaped = s->prof_escaped;
    if (train_steps) *train_steps = s->prof_train_steps;
  });
}

int wostgpu_solver3_reserve_records(wg_solver3 s, int64_t n) {
  return guarded([&] {
    need(n >= 0, WG_ERR_INVALID, "record count must be >= 0");
    s->rec_cap_min = std::max<int64_t>(s->rec_cap_min, n);
  });
}

int wostgpu_solver3_attach_comm(wg_solver3 s, const char id[128], int32_t nranks, int32_t rank) {
  return guarded([&] {
    need(nranks >= 1 && rank >= 0 && rank < nranks, WG_ERR_INVALID, "bad rank / nranks");
    if (s->comm) {
      nccl().commDestroy(s->comm);
      s->comm = nullptr;
    }
    // a single-rank communicator is created too: it runs the multi-GPU
    // pipeline (allreduce on the solver stream before Adam) on one GPU
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    NCK(nccl().commInitRank(&s->comm, nranks, uid, rank));
    s->nranks = nranks;
    s->rank = rank;
  });
}

}  // extern "C"
