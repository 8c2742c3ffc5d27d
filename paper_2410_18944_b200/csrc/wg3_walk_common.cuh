// One 3D walk step split in the two halves every 3D walk kernel shares
// (the exact CUDA-core kernel in wg3_walk.cu, the tcgen05 kernel in
// wg3_walk_tc.cu), around the guiding-field evaluation that differs:
//   step_begin  = begin_step  (proj/src/wost.cpp:148-216, d = 3, f = h = 0)
//   step_finish = sample_next_direction + finish_step (wost.cpp:124-146, 218-264)
// plus the record layout and the walk-lane state. Contract: oracle/wost3d.inc.
#pragma once

#include <cooperative_groups.h>
#include <cooperative_groups/reduce.h>

#include "wg3_field.cuh"
#include "wg3_mix.cuh"
#include "wg_kernels.cuh"
#include "wg_train.cuh"

namespace wg3 {

using wg::DevRecord;
using wg::Pcg;
using wg::REC_ON_NEUMANN;
using wg::REC_WRITTEN;

// A 3D record has DevRecord's size and the offsets the shared record kernels
// (finalize, compact; wg_train.cu) read; z, nu_z, n_z live in the slots 3D
// never uses (dacc: 3D scenes have no local source / flux terms, so targets
// are |S_K / Q_k| without a chain walk).
struct __align__(16) DevRecord3 {
  float x, y, nux, nuy, nx, ny;
  float pdf_mis, pdf_g, pdf_u, c;
  float target;
  float z;  // DevRecord::dacc
  float thr_q;
  float nuz;  // DevRecord::pad_
  int32_t walk;
  uint32_t flags;
  uint64_t key;
  int32_t prev;
  float nz;  // DevRecord::pad2_
};
static_assert(sizeof(DevRecord3) == sizeof(DevRecord), "DevRecord3 aliases DevRecord");
static_assert(offsetof(DevRecord3, pdf_mis) == offsetof(DevRecord, pdf_mis) &&
                  offsetof(DevRecord3, target) == offsetof(DevRecord, target) &&
                  offsetof(DevRecord3, thr_q) == offsetof(DevRecord, thr_q) &&
                  offsetof(DevRecord3, walk) == offsetof(DevRecord, walk) &&
                  offsetof(DevRecord3, flags) == offsetof(DevRecord, flags) &&
                  offsetof(DevRecord3, key) == offsetof(DevRecord, key) &&
                  offsetof(DevRecord3, prev) == offsetof(DevRecord, prev),
              "fields the shared record kernels read");

// default 3D field shape: 4 levels x 4 features -> 64 -> 64 -> 41 (K = 8)
constexpr int IN = 16, HID = 64, K8 = 8, OD = 5 * K8 + 1;
constexpr int MLPN = IN * HID + HID + HID * HID + HID + HID * OD + OD;  // 7913

inline bool default_shape3(const Field3View& v) {
  return v.levels == 4 && v.F == 4 && v.in == IN && v.hid == HID && v.od == OD && v.k == K8;
}

// begin_step's geometry at a start point: every walk of a point begins
// there, so its first closest-point / silhouette queries (the unseeded,
// costliest ones) are answered once per point (start_geo3_kernel)
struct StartGeo3 {
  CP3 cd;      // closest Dirichlet point (closest_dirichlet_seeded, no seed)
  double ds2;  // closest_silhouette_d2 bounded by cd's distance squared
};

struct Walk3Args {
  Scene3View s;
  Field3View f;
  wg::SolverParams sp;
  const double* points;  // [n_points][3]
  int64_t n_points, point_offset;
  uint64_t seed, wpp_first;
  int32_t n_rounds;
  double* est;
  int32_t* esc;
  int32_t* steps;
  DevRecord3* recs;
  unsigned long long* rec_counter;
  int64_t rec_capacity;
  uint64_t key_seed;
  unsigned long long* counters;  // [0] steps [1] escaped [2] walks [3] rec overflow [4] scene error
  int32_t* rec_tail;
  double* rec_term;
  float* rec_dacc;  // per record slot: accumulator increments since the walk's
                    // previous record (DevRecord::dacc, held aside in 3D)
  const StartGeo3* start;  // [n_points] cached first-step geometry (nullptr: query)
};

struct Lane3 {
  D3 x, n;
  double T, acc, R;
  double dacc;  // source / flux increments since the walk's last record
  int tri, depth, round, rec_left, last_rec;
  int cp_seed;  // leaf-order index of the previous step's closest Dirichlet triangle (-1: none)
  bool on_n, alive, rec_ok;
  Pcg rng;
  int64_t point, rec_base;
};

// next walk id from the hand-out counter, one atomic per group of lanes
// claiming together
__device__ __forceinline__ unsigned long long claim_walk(unsigned long long* counter) {
  namespace cg = cooperative_groups;
  const cg::coalesced_group g = cg::coalesced_threads();
  unsigned long long base = 0;
  if (g.thread_rank() == 0) base = atomicAdd(counter, static_cast<unsigned long long>(g.size()));
  return g.shfl(base, 0) + g.thread_rank();
}

// slot of a queue with a shared length counter, one atomic per group of
// lanes appending together
__device__ __forceinline__ unsigned int claim_queue(unsigned int* len) {
  namespace cg = cooperative_groups;
  const cg::coalesced_group g = cg::coalesced_threads();
  unsigned int base = 0;
  if (g.thread_rank() == 0) base = atomicAdd(len, g.size());
  return g.shfl(base, 0) + g.thread_rank();
}

__device__ __forceinline__ void lane3_init(Lane3& w, const Walk3Args& a, int64_t id) {
  w.round = static_cast<int>(id / a.n_points);
  w.point = id - static_cast<int64_t>(w.round) * a.n_points;
  w.x = {a.points[3 * w.point], a.points[3 * w.point + 1], a.points[3 * w.point + 2]};
  w.n = {0.0, 0.0, 0.0};
  w.on_n = false;
  w.tri = -1;
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
  w.cp_seed = -1;
}

__device__ __forceinline__ void finish3(Lane3& w, const Walk3Args& a, bool escaped, double terminal,
                                        bool collect) {
  const int64_t slot = static_cast<int64_t>(w.round) * a.n_points + w.point;
  a.est[slot] = escaped ? 0.0 : w.acc;
  a.esc[slot] = escaped ? 1 : 0;
  if (a.steps) a.steps[slot] = w.depth;
  // step / escape totals: one atomic per group of lanes finishing together
  // (a same-address atomic per walk serialises at L2)
  namespace cg = cooperative_groups;
  const cg::coalesced_group g = cg::coalesced_threads();
  const unsigned long long steps = cg::reduce(g, static_cast<unsigned long long>(w.depth),
                                              cg::plus<unsigned long long>());
  const unsigned long long esc = cg::reduce(g, escaped ? 1ull : 0ull, cg::plus<unsigned long long>());
  if (g.thread_rank() == 0) {
    atomicAdd(&a.counters[0], steps);
    if (esc) atomicAdd(&a.counters[1], esc);
  }
  if (collect) {
    a.rec_tail[slot] = w.last_rec;
    a.rec_term[slot] = escaped ? 0.0 : pa(pm(w.T, terminal), w.dacc);
  }
  w.alive = false;
}

// begin_step: terminates the walk (returns false) or sets its star radius,
// reserves its record slot (rec, -1 when not collecting) and returns true:
// the walk needs a direction this step
__device__ __forceinline__ bool step_begin(Lane3& w, const Walk3Args& a, bool collect, int& rec) {
  const Scene3View& s = a.s;
  rec = -1;
  // the start point's answers are the same for every walk of the point
  const bool at_start = w.depth == 0 && a.start != nullptr;
  const CP3 cd = at_start ? a.start[w.point].cd : closest_dirichlet_seeded(s, w.x, w.cp_seed);
  w.cp_seed = cd.local;
  const double dd = cd.tri >= 0 ? sqrt(cd.d2) : dinf();
  if (cd.tri >= 0 && dd <= a.sp.eps) {
    const double g = value_at(s.values[s.tri[0][cd.local].value], cd.p);
    w.acc = pa(w.acc, pm(w.T, g));
    finish3(w, a, false, g, collect);
    return false;
  }
  if (w.depth >= a.sp.max_steps) {
    finish3(w, a, true, 0.0, collect);
    return false;
  }
  if (w.depth > a.sp.rr_depth) {  // Russian roulette, wost.cpp:169-180
    const double q = fmin(1.0, fabs(w.T));
    if (q <= 0.0 || w.rng.uni() >= q) {
      finish3(w, a, false, 0.0, collect);
      return false;
    }
    w.T /= q;
  }
  // R = min(dD, max(d_sil, r_min)) needs d_sil only when it is below dD: the
  // silhouette search starts bounded by dD^2 and reports inf when nothing
  // is closer, which leaves R = dD exactly as the unbounded query would
  const double bound2 = dd == dinf() ? dinf() : dd * dd;
  const double ds2 = at_start ? a.start[w.point].ds2 : closest_silhouette_d2(s, w.x, bound2);
  const double dsil = ds2 < bound2 ? sqrt(ds2) : dinf();
  if (dd == dinf() && dsil == dinf()) {  // SceneError, wost.cpp:184-186
    atomicOr(&a.counters[4], 1ull);
    finish3(w, a, true, 0.0, false);
    return false;
  }
  const double R = fmin(dd, fmax(dsil, a.sp.rmin));
  w.R = R;
  if (s.source.type != WG_VALUE_ZERO || s.has_flux) {
    double contrib = 0.0;
    if (s.source.type != WG_VALUE_ZERO) {  // sample_source_point (wost.cpp:67-87), d = 3
      const D3 dir = uniform_sample(w.rng, w.on_n, w.n);
      const double r = greens_radius3(w.rng.uni(), R);
      const D3 y = add(w.x, scl(dir, r));
      const Hit3 h = ray_first_hit(s, w.x, dir, r, WG_KIND_ALL, -1);
      const double wt = h.tri >= 0 ? 0.0 : R * R / 6.0;
      if (wt != 0.0) contrib = ps(contrib, pm(wt, bbox_contains(s, y, 0.0) ? value_at(s.source, y) : 0.0));
    }
    if (s.has_flux) {  // sample_neumann_contrib (wost.cpp:89-109), d = 3
      const D3 dir = uniform_sample(w.rng, w.on_n, w.n);
      const Hit3 h = ray_first_hit(s, w.x, dir, R, WG_KIND_NEUMANN, w.tri);
      double add_ = 0.0;
      if (h.tri >= 0) {
        const D3 hp = add(w.x, scl(dir, h.t));
        const double hv = value_at(s.values[s.tri[1][h.local].value], hp);
        if (hv != 0.0) {
          double cz = fabs(dot(dir, hit_normal(s, h, dir)));
          if (a.sp.clamp_grazing) cz = fmax(cz, a.sp.grazing_floor);
          if (cz != 0.0) add_ = greens_ball3(h.t, R) * hv * h.t * h.t * kFourPi / cz;
        }
      }
      contrib += add_;
    }
    w.acc = pa(w.acc, pm(w.T, contrib));
    w.dacc = pa(w.dacc, pm(w.T, contrib));
  }
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

// a sampled direction with its densities (mult = p_u / p_mis; 1 when uniform)
struct Dir3 {
  D3 nu;
  double pmis, pg, pu, sel, mult;
};

// direction: guided MIS from m, or uniform when m == nullptr
// (sample_next_direction, wost.cpp:124-146)
__device__ __forceinline__ Dir3 step_sample(Lane3& w, const Walk3Args& a, const Mix3<K8>* m) {
  Dir3 d;
  if (m) {
    Mis3 o = mis_sample(w.rng, *m, w.on_n, w.n, a.sp.reflect != 0);
    d.nu = o.nu;
    d.pmis = o.pmis;
    d.pg = o.pg;
    d.pu = o.pu;
    d.sel = m->c;
    d.mult = o.pu / o.pmis;
  } else {
    d.nu = uniform_sample(w.rng, w.on_n, w.n);
    d.pu = uniform_pdf(d.nu, w.on_n, w.n);
    d.pmis = d.pu;
    d.pg = 0.0;
    d.sel = 0.0;
    d.mult = 1.0;
  }
  return d;
}

// record + move along d (finish_step, wost.cpp:218-264); guided walks carry
// the MIS multiplier in their throughput
__device__ __forceinline__ void step_move(Lane3& w, const Walk3Args& a, bool collect, int rec, const Dir3& d,
                                          bool guided) {
  const Scene3View& s = a.s;
  if (rec >= 0) {
    DevRecord3 r;
    r.x = static_cast<float>(w.x.x);
    r.y = static_cast<float>(w.x.y);
    r.z = static_cast<float>(w.x.z);
    r.nux = static_cast<float>(d.nu.x);
    r.nuy = static_cast<float>(d.nu.y);
    r.nuz = static_cast<float>(d.nu.z);
    r.nx = static_cast<float>(w.n.x);
    r.ny = static_cast<float>(w.n.y);
    r.nz = static_cast<float>(w.n.z);
    r.pdf_mis = static_cast<float>(d.pmis);
    r.pdf_g = static_cast<float>(d.pg);
    r.pdf_u = static_cast<float>(d.pu);
    r.c = static_cast<float>(d.sel);
    r.target = 0.0f;
    r.thr_q = static_cast<float>(guided ? w.T * d.mult : w.T);
    r.walk = static_cast<int32_t>(static_cast<int64_t>(w.round) * a.n_points + w.point);
    r.flags = REC_WRITTEN | (w.on_n ? REC_ON_NEUMANN : 0u);
    r.key = Pcg::mix(a.key_seed ^ Pcg::mix((static_cast<uint64_t>(a.point_offset + w.point) << 20) ^
                                           static_cast<uint64_t>(w.depth)));
    r.prev = w.last_rec;
    a.recs[rec] = r;
    a.rec_dacc[rec] = static_cast<float>(w.dacc);
    w.dacc = 0.0;
    w.last_rec = rec;
  }
  if (d.mult == 0.0) {  // sampled into the invalid half space
    finish3(w, a, false, 0.0, collect);
    return;
  }
  Hit3 h = ray_first_hit(s, w.x, d.nu, w.R, WG_KIND_NEUMANN, w.tri);
  if (h.tri >= 0) {
    w.x = add(w.x, scl(d.nu, h.t));
    w.n = hit_normal(s, h, d.nu);
    w.on_n = true;
    w.tri = h.tri;
  } else {
    w.x = add(w.x, scl(d.nu, w.R));
    w.on_n = false;
    w.tri = -1;
  }
  if (guided) w.T *= d.mult;
  ++w.depth;
  if (!bbox_contains(s, w.x, 1e-9 * s.diag)) finish3(w, a, true, 0.0, collect);
}

__device__ __forceinline__ void step_finish(Lane3& w, const Walk3Args& a, bool collect, int rec,
                                            const Mix3<K8>* m) {
  const Dir3 d = step_sample(w, a, m);
  step_move(w, a, collect, rec, d, m != nullptr);
}

// mixture of one raw output row with the sampler-mode override (decode_guiding, wost.cpp:111-122)
template <class T>
__device__ __forceinline__ void decode3(const T* raw, const wg::SolverParams& sp, Mix3<K8>& m) {
  normalize3<K8>(raw, m);
  if (sp.mode == WG_MODE_GUIDING_ONLY) m.c = 1.0;
  else if (sp.mode == WG_MODE_FIXED_MIS) m.c = sp.fixed_c;
}

// tensor-core walk kernels (wg3_walk_tc.cu): lockstep tiles, and the
// wavefront pair (geometry kernel + tensor-core direction kernel)
struct Wave3 {
  Lane3* lanes;          // [slots]
  Dir3* dirs;            // [slots]
  int32_t* rec;          // [slots] record slot reserved by step_begin
  uint8_t* state;        // [slots] 0 empty, 1 needs a direction, 2 needs a move
  int32_t* queue;        // [slots] slots needing a direction this iteration
  unsigned int* qlen;    // [2] queue lengths (double-buffered by iteration parity)
  unsigned long long* next_walk;  // walk-id hand-out counter
  int64_t slots;
  unsigned char* wblob;  // [wg::wpack::FWD_BYTES] split-fp16 MLP weights, packed per call
  int32_t* perm;         // [slots] geometry-pass order: slots grouped by spatial cell
  unsigned int* bins;    // [kSortBins + 3] cell histogram / offsets, [+1] entries in perm, [+2] skip
  uint16_t* sbin;        // [slots] sort cell of the slot's pending move (>= kSortBins: none), set by the geometry pass
};
#ifndef WG3_SORT_BITS
#define WG3_SORT_BITS 4
#endif
constexpr int kSortBits = WG3_SORT_BITS;              // per axis
constexpr int kSortBins = 1 << (3 * kSortBits);       // + 1 bin for slots without a pending move
}  // namespace wg3

namespace wg {
// 3D minibatch gradient on the tensor cores (wg_train_tc.cu grad3_tc_kernel;
// the fields of TrainArgs with the 3D field and records)
struct TrainArgs3 {
  wg3::Field3View f;
  const wg3::DevRecord3* recs;
  const uint32_t* list;
  const unsigned long long* count;
  int64_t list_cap;
  float* grad;  // [n_params + 1]; grad[n_params] = record count
  int64_t n_params;
  double inv_count;
  int32_t reflect, learn_selection;
  double e_fraction, v_floor;
  TrainTotals* totals;
  const unsigned char* packed;  // split-fp16 blob of the 3D field (launch_pack3_full)
};
cudaError_t launch_grad3_tc(const TrainArgs3& a, cudaStream_t st);
cudaError_t launch_pack3_full(const wg3::Field3View& f, unsigned char* blob, cudaStream_t st);
}  // namespace wg

namespace wg3 {
// returns the number of kernels launched in *launches
cudaError_t launch_walks3_wave(const Walk3Args& a, const Wave3& w, int sms, unsigned int* h_qlen,
                               int64_t* launches, cudaStream_t st);
int walk3_tc_smem();
int walk3_tc_blocks_per_sm();
cudaError_t launch_walks3_tc(const Walk3Args& a, int blocks, cudaStream_t st);
cudaError_t launch_mix3f_pdf(int64_t n, const float* raw, const double* nu, double* out, cudaStream_t st);
cudaError_t launch_field3_eval_tc(const Field3View& f, int64_t n, const double* x, double* out,
                                  cudaStream_t st);

}  // namespace wg3
