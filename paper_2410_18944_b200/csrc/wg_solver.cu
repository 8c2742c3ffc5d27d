// Host runtime behind the C-ABI, part 2: the solver — StepContext +
// SolveScratch + the Engine's record arena and training state
// (proj/include/wost/wost.hpp:33-51, proj/src/solver.cpp:53-105).
//
// Everything a round does is enqueued on the solver's stream with no host
// synchronisation: walk kernel -> Welford -> [compaction -> per minibatch:
// gradient tile -> NCCL allreduce -> Adam prep -> Adam]. The host only waits
// when a caller asks for results (statistics, records, TrainStats, timings).
#include <cstdio>
#include <cstdlib>
#include <string>

#include "wg_runtime.hpp"
#include "wg_wpack.cuh"

using namespace wg;
using namespace wgrt;

namespace wg {
cudaError_t launch_grad_tc(const TrainArgs& a, cudaStream_t st);  // wg_train_tc.cu
bool tc_grad_available();
}  // namespace wg

// counters[] slots (run-cumulative): walk kernels atomically add into them
enum {
  C_STEPS = 0,
  C_ESCAPED = 1,
  C_WALKS = 2,
  C_REC_OVERFLOW = 3,
  C_SCENE_ERR = 4,
  C_TRAIN_STEPS = 5,
  C_WAVE_LAUNCHES = 8,  // kernels of the device-side 2D wavefront loop
  C_N = 9
};

struct wg_solver_s {
  wg_scene_s* scene = nullptr;
  wg_field_s* field = nullptr;
  wg_solver_config cfg{};
  int mlp = WG_MLP_EXACT;
  cudaStream_t stream = nullptr;
  int sms = 148;
  // points and statistics
  int64_t n_points = 0, point_offset = 0;
  DBuf points, stats;
  // per-round results ([round][point])
  DBuf est, esc, steps;
  int32_t est_rounds = 0;
  // records of the current / last collecting round
  DBuf recs, rec_counter;  // rec_counter: u64 bump allocator of the arena
  DBuf rec_tail, rec_term;  // per walk of the collecting round: chain end, terminal term
  bool recs_from_walks = false;
  int64_t rec_capacity = 0;
  int64_t rec_capacity_min = 0;  // grown after an arena overflow
  bool have_records = false;
  // device control
  DBuf counters;  // C_N x u64
  DBuf ctl;       // TrainCtl (per round)
  DBuf totals;    // TrainTotals (per run / train call)
  DBuf lists, grad;
  int64_t list_cap = 0;
  DBuf phase_prof;  // WOSTGPU_PHASE_PROF diagnostics
  DBuf spill;       // lockstep-kernel tail handoff (SpillLane per slot)
  // timing: event pairs around walk launches and training rounds
  std::vector<cudaEvent_t> ev_walk, ev_train;
  int n_walk_ev = 0, n_train_ev = 0;
  cudaEvent_t ev_run0 = nullptr, ev_run1 = nullptr;
  // results of the last synchronised call
  unsigned long long last_counters[C_N] = {};
  double last_walk_ms = 0, last_train_ms = 0;
  // NCCL
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  // wavefront walk pool (wg_wave2.cu)
  DBuf w_lanes, w_dirs, w_rec, w_state, w_queue, w_qlen, w_next;
  int64_t w_slots = 0;
  unsigned int* h_qlen = nullptr;  // pinned
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

cudaEvent_t pool_event(std::vector<cudaEvent_t>& pool, int& used) {
  if (used == static_cast<int>(pool.size())) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    pool.push_back(e);
  }
  return pool[used++];
}

double pool_ms(const std::vector<cudaEvent_t>& pool, int used) {
  double ms = 0.0;
  for (int i = 0; i + 1 < used; i += 2) {
    float t = 0.0f;
    CK(cudaEventElapsedTime(&t, pool[i], pool[i + 1]));
    ms += t;
  }
  return ms;
}

void reset_run(wg_solver_s* s) {
  s->counters.alloc(sizeof(unsigned long long) * C_N);
  CK(cudaMemsetAsync(s->counters.p, 0, sizeof(unsigned long long) * C_N, s->stream));
  s->totals.alloc(sizeof(TrainTotals));
  CK(cudaMemsetAsync(s->totals.p, 0, sizeof(TrainTotals), s->stream));
  s->n_walk_ev = s->n_train_ev = 0;
}

// the field's packed weight blob, repacked on the stream if the host changed
// the parameters since it was last written
unsigned char* field_blob(wg_field_s* f, cudaStream_t st) {
  f->wpack.alloc(wpack::BYTES);
  if (f->pack_dirty) {
    CKL(launch_pack_weights(f->view, f->wpack.as<unsigned char>(), st));
    f->pack_dirty = false;
  }
  return f->wpack.as<unsigned char>();
}

// enqueue solve_batch for `rounds` consecutive wpp indices (no host sync)
void enqueue_rounds(wg_solver_s* s, uint64_t seed, uint64_t wpp_first, int32_t rounds, bool collect,
                    uint64_t key_seed, double pdf_floor) {
  need(s->n_points > 0, WG_ERR_INVALID, "solver has no evaluation points");
  const bool guided = s->cfg.mode != WG_MODE_UNIFORM;
  need(!guided || s->field, WG_ERR_INVALID, "guided sampler modes need a guiding field");
  need(!collect || rounds == 1, WG_ERR_INVALID, "record collection runs one round at a time");
  const bool dflt = guided && default_shape(s->field->view);
  int32_t chunk = static_cast<int32_t>(std::max<int64_t>(1, (int64_t(1) << 30) / (s->n_points * 16)));
  chunk = std::min(chunk, rounds);
  if (s->est_rounds < chunk) {
    s->est.alloc(sizeof(double) * s->n_points * chunk);
    s->esc.alloc(sizeof(int32_t) * s->n_points * chunk);
    s->steps.alloc(sizeof(int32_t) * s->n_points * chunk);
    s->est_rounds = chunk;
  }
  if (collect) {
    // Record arena: every step of every walk in the round may write one
    // record (the reference keeps them all, guide_train.cpp:58-79). 256 per
    // point covers long-walk scenes (const-source-disk reaches ~120 records
    // per point once guiding is trained); a walk that finds the arena full
    // stops recording, which would bias the training set towards early,
    // short walks, so any overflow doubles the arena for the next call.
    int64_t cap = std::max<int64_t>({s->n_points * 256, int64_t(1) << 16, s->rec_capacity_min});
    if (s->rec_capacity < cap) {
      s->recs.alloc(sizeof(DevRecord) * cap);
      s->rec_capacity = cap;
    }
    s->rec_counter.alloc(sizeof(unsigned long long));
    CK(cudaMemsetAsync(s->rec_counter.p, 0, sizeof(unsigned long long), s->stream));
    s->rec_tail.alloc(sizeof(int32_t) * s->n_points);
    s->rec_term.alloc(sizeof(double) * s->n_points);
    CK(cudaMemsetAsync(s->rec_tail.p, 0xFF, sizeof(int32_t) * s->n_points, s->stream));  // -1
    s->ctl.alloc(sizeof(TrainCtl));
    CK(cudaMemsetAsync(s->ctl.p, 0, sizeof(TrainCtl), s->stream));
    s->have_records = true;
    s->recs_from_walks = true;
  }
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
  a.rec_counter = collect ? s->rec_counter.as<unsigned long long>() : nullptr;
  a.rec_capacity = s->rec_capacity;
  a.key_seed = key_seed;
  a.pdf_floor = pdf_floor;
  a.ctl = collect ? s->ctl.as<TrainCtl>() : nullptr;
  a.rec_tail = collect ? s->rec_tail.as<int32_t>() : nullptr;
  a.rec_term = collect ? s->rec_term.as<double>() : nullptr;

  // guided walks on the default field shape: tcgen05 MLP tile kernel, or the
  // bit-faithful CUDA-core MLP with 8 lanes per walk; otherwise generic
  const bool tc = dflt && s->mlp == WG_MLP_TENSOR;
  const bool g8 = dflt && !tc;
  int smem = (s->scene->smem_bytes > 0 ? ((s->scene->smem_bytes + 15) & ~15) : 0) +
             (guided ? ((int)sizeof(float) * s->field->view.mlp_count + 15) / 16 * 16 : 0);
  if (g8) smem = walk_g8_smem(a);
  if (tc) {
    // CUDA-core tail MLP on; WOSTGPU_SMALL_MLP=0 drops it (and its 46 KB of
    // shared memory). Measured on cfg 3 at 512^2, where that lets a second
    // CTA onto each SM: 2.70 vs 2.73M walks/s, so the default keeps it.
    static const int small_env = [] {
      const char* e = std::getenv("WOSTGPU_SMALL_MLP");
      return e ? std::atoi(e) : 1;
    }();
    a.small_mlp = small_env != 0;
    smem = walk_tc_smem(a);
    a.wblob = field_blob(s->field, s->stream);
  }
  const int lanes_per_walk = g8 ? 8 : 1;
  const int block = g8 ? 256 : tc ? walk_tc_block() : 128;
  const int per_sm = std::max(1, tc   ? walk_tc_blocks_per_sm(smem)
                                 : g8 ? walk_g8_blocks_per_sm(smem)
                                      : walk_blocks_per_sm(dflt, guided && !dflt, smem));
  for (int32_t r0 = 0; r0 < rounds; r0 += chunk) {
    int32_t n = std::min(chunk, rounds - r0);
    a.wpp_first = wpp_first + r0;
    a.n_rounds = n;
    int64_t want = (s->n_points * n * lanes_per_walk + block - 1) / block;
    // tensor-core lockstep kernel: at least one CTA per SM (walk ids are
    // interleaved over CTAs, so a small round spreads over every SM)
    if (tc) want = std::max<int64_t>(want, s->sms);
    int blocks = static_cast<int>(std::min<int64_t>(want, (int64_t)per_sm * s->sms));
    static const bool phase_prof = std::getenv("WOSTGPU_PHASE_PROF") != nullptr;
    if (phase_prof && tc) {
      s->phase_prof.alloc(sizeof(unsigned long long) * 8 * blocks);
      CK(cudaMemsetAsync(s->phase_prof.p, 0, sizeof(unsigned long long) * 8 * blocks, s->stream));
      a.phase_prof = s->phase_prof.as<unsigned long long>();
    }
    CK(cudaEventRecord(pool_event(s->ev_walk, s->n_walk_ev), s->stream));
    // tensor-core walks as a wavefront pair when geometry dominates and
    // enough walks are in flight to fill the GPU (cfg 3, 256 segments at
    // 512^2: 3.28 vs 2.72M walks/s); lockstep tiles otherwise: small scenes
    // (<= 16 segments, shared-memory segment lists; cfg 2 multi-round: 99 vs
    // 41M walks/s) and 16,384-walk training rounds. WOSTGPU_WALK2 = wave /
    // lockstep forces one.
    const char* w2 = std::getenv("WOSTGPU_WALK2");
    const int force2 = !w2 ? 0 : std::string(w2) == "wave" ? 1 : std::string(w2) == "lockstep" ? 2 : 0;
    const bool wave = tc && (force2 == 1 || (force2 == 0 && s->scene->view.n_segs > 16 &&
                                              s->n_points * n >= 65536));
    if (wave) {
      const int64_t slots = std::min<int64_t>(s->n_points * n, (int64_t)s->sms * 16 * 128);
      if (s->w_slots < slots) {
        size_t lb = 0, db = 0;
        wave2_sizes(&lb, &db);
        s->w_lanes.alloc(lb * slots);
        s->w_dirs.alloc(db * slots);
        s->w_rec.alloc(sizeof(int32_t) * slots);
        s->w_state.alloc(slots);
        s->w_queue.alloc(sizeof(int32_t) * slots);
        s->w_slots = slots;
      }
      s->w_qlen.alloc(2 * sizeof(unsigned int));
      s->w_next.alloc(sizeof(unsigned long long));
      if (!s->h_qlen) CK(cudaMallocHost(&s->h_qlen, 4 * sizeof(unsigned int)));
      int64_t launched = 0;
      CK(launch_walks2_wave(a, s->w_lanes.p, s->w_dirs.p, s->w_rec.as<int32_t>(), s->w_state.as<uint8_t>(),
                            s->w_queue.as<int32_t>(), s->w_qlen.as<unsigned int>(),
                            s->w_next.as<unsigned long long>(), slots, s->sms, s->h_qlen, &launched, s->stream));
      g_launches += launched;
    } else if (tc) {
      // tail handoff to the warp-per-walk kernel (WalkArgs::spill) once a
      // CTA has <= 24 live walks: small scenes only, where both kernels scan
      // shared-memory segment lists. cfg 2 walk time per round 0.566 -> 0.478
      // ms (T = 16 / 32 / 48 / 64: 0.485 / 0.481 / 0.493 / 0.519); cfg 3's
      // 256-gon: 1.55 vs 1.59 ms, off. WOSTGPU_SPILL_ROWS overrides (0 = off)
      static const int spill_env = [] {
        const char* e = std::getenv("WOSTGPU_SPILL_ROWS");
        return e ? std::atoi(e) : -1;
      }();
      const int nb = std::max(1, blocks);
      const int spill_want = spill_env >= 0 ? spill_env : s->scene->view.n_segs <= 16 ? 24 : 0;
      const int spill_rows = a.small_mlp ? std::max(0, std::min(spill_want, 128)) : 0;
      a.spill_rows = spill_rows;
      if (spill_rows > 0) {
        s->spill.alloc(sizeof(SpillLane) * nb * spill_rows);
        a.spill = s->spill.as<SpillLane>();
        CK(cudaMemsetAsync(a.counters + 7, 0, sizeof(unsigned long long), s->stream));
      }
      CKL(launch_walks_tc(a, nb, s->stream));
      if (spill_rows > 0) CKL(launch_walks_coop_resume(a, nb * spill_rows, s->sms, s->stream));
    }
    if (phase_prof && tc) {  // diagnostics: cycles per CTA iteration of the slowest CTA
      std::vector<unsigned long long> h(8 * blocks);
      CK(cudaMemcpyAsync(h.data(), s->phase_prof.p, sizeof(unsigned long long) * 8 * blocks,
                         cudaMemcpyDeviceToHost, s->stream));
      CK(cudaStreamSynchronize(s->stream));
      int worst = 0;
      auto tot = [&](int b) { return h[8 * b] + h[8 * b + 1] + h[8 * b + 2]; };
      for (int b = 0; b < blocks; ++b)
        if (tot(b) > tot(worst)) worst = b;
      const unsigned long long* q = &h[8 * worst];
      double it = static_cast<double>(std::max<unsigned long long>(q[3], 1));
      const double small_it = static_cast<double>(q[6] >> 40);
      const double prep = static_cast<double>(q[6] & ((1ull << 40) - 1));
      std::fprintf(stderr,
                   "[phase] cta %d iters %.0f cycles/iter A %.0f B %.0f (gather %.0f prep %.0f mma %.0f) C %.0f; "
                   "small-MLP iters %.0f at %.0f cycles\n",
                   worst, it, q[0] / it, q[1] / it, q[5] / it, prep / it, q[4] / it, q[2] / it, small_it,
                   small_it > 0 ? q[7] / small_it : 0.0);
    }
    if (tc || wave) {
    } else if (g8) CKL(launch_walks_g8(a, std::max(1, blocks), s->stream));
    else CKL(launch_walks(a, dflt, guided && !dflt, std::max(1, blocks), s->stream));
    CK(cudaEventRecord(pool_event(s->ev_walk, s->n_walk_ev), s->stream));
    CKL(launch_welford(a.est, a.esc, s->n_points, n, s->stats.as<wg_point_stats>(), s->stream));
  }
}

// targets + validity + usable counts of the arena's records (see DevRecord)
void enqueue_finalize(wg_solver_s* s, double pdf_floor) {
  s->ctl.alloc(sizeof(TrainCtl));
  CK(cudaMemsetAsync(s->ctl.p, 0, sizeof(TrainCtl), s->stream));
  // walk-collected records of scenes with source / Neumann terms take their
  // targets from the per-walk backward suffix sums (DevRecord)
  const SceneView& v = s->scene->view;
  const bool walks = s->recs_from_walks;
  const bool chain = walks && (!v.source_zero || v.has_flux);
  CKL(launch_finalize_records(s->recs.as<DevRecord>(), s->rec_counter.as<unsigned long long>(),
                              s->rec_capacity, walks ? s->n_points : 0, s->rec_tail.as<int32_t>(),
                              s->rec_term.as<double>(), s->esc.as<int32_t>(), pdf_floor,
                              s->ctl.as<TrainCtl>(), chain, s->stream));
}

void ensure_train_buffers(wg_solver_s* s, const wg_train_config& tc) {
  need(tc.minibatch >= 1, WG_ERR_INVALID, "minibatch must be >= 1");
  const int n_mb = static_cast<int>((tc.max_records_per_round + tc.minibatch - 1) / tc.minibatch);
  need(n_mb <= kMaxMinibatches, WG_ERR_INVALID, "max_records / minibatch exceeds the device limit");
  int64_t cap = tc.minibatch + tc.minibatch / 4 + 1024;
  if (s->list_cap < cap) {
    s->lists.alloc(sizeof(uint32_t) * kMaxMinibatches * cap);
    s->list_cap = cap;
  }
  s->grad.alloc(sizeof(float) * (s->field->n_params + 1));
}

void enqueue_minibatch(wg_solver_s* s, const wg_train_config& tc, int b, double inv_count) {
  wg_field_s* f = s->field;
  CK(cudaMemsetAsync(s->grad.p, 0, sizeof(float) * (f->n_params + 1), s->stream));
  TrainArgs ta{};
  ta.f = f->view;
  ta.recs = s->recs.as<DevRecord>();
  ta.list = s->lists.as<uint32_t>() + static_cast<int64_t>(b) * s->list_cap;
  ta.count = &s->ctl.as<TrainCtl>()->mb_count[b];
  ta.list_cap = s->list_cap;
  ta.grad = s->grad.as<float>();
  ta.n_params = f->n_params;
  ta.inv_count = inv_count;
  ta.reflect = tc.reflect;
  ta.learn_selection = tc.learn_selection;
  ta.e_fraction = tc.e_fraction;
  ta.v_floor = tc.v_floor;
  ta.totals = s->totals.as<TrainTotals>();
  // tensor-core walks train on the tcgen05 gradient tile; the bit-faithful
  // (MLP_EXACT) path on the CUDA-core fp64-loss tile
  if (s->mlp == WG_MLP_TENSOR && tc_grad_available()) {
    ta.packed = field_blob(f, s->stream);
    CKL(launch_grad_tc(ta, s->stream));
  }
  else CKL(launch_grad_cuda_core(ta, s->stream));
}

void check_trainable(wg_solver_s* s) {
  need(s->field != nullptr, WG_ERR_INVALID, "training needs a guiding field");
  need(default_shape(s->field->view), WG_ERR_NOT_BUILT,
       "device training is built for the default field shape (L=4, F=4, hidden 64, K=8, 2D)");
}

// The selection rate of a round comes from the usable-record count summed
// over the ranks: one 8-byte NCCL allreduce on the solver
// stream, or the host-supplied global count of the split-phase API.
void enqueue_usable_global(wg_solver_s* s, const int64_t* host_global) {
  TrainCtl* c = s->ctl.as<TrainCtl>();
  if (host_global) {
    static_assert(sizeof(unsigned long long) == sizeof(int64_t), "count width");
    CK(cudaMemcpyAsync(&c->usable_global, host_global, sizeof(int64_t), cudaMemcpyHostToDevice,
                       s->stream));
    CK(cudaStreamSynchronize(s->stream));  // the host value is borrowed for the call only
  } else if (s->comm) {
    NCK(nccl().allReduce(&c->usable, &c->usable_global, 1, ncclUint64, ncclSum, s->comm, s->stream));
  } else {
    CK(cudaMemcpyAsync(&c->usable_global, &c->usable, sizeof(unsigned long long),
                       cudaMemcpyDeviceToDevice, s->stream));
  }
}

void enqueue_select(wg_solver_s* s, const wg_train_config& tc) {
  CKL(launch_compact(s->recs.as<DevRecord>(), s->rec_counter.as<unsigned long long>(),
                     s->rec_capacity, s->ctl.as<TrainCtl>(), s->totals.as<TrainTotals>(),
                     s->lists.as<uint32_t>(), s->list_cap, tc.max_records_per_round, tc.minibatch,
                     s->stream));
}

int n_minibatches(const wg_train_config& tc) {
  return static_cast<int>((tc.max_records_per_round + tc.minibatch - 1) / tc.minibatch);
}

// Adam on the (globally reduced) gradient buffer; no step when its record
// count slot is 0
void enqueue_adam(wg_solver_s* s, const wg_train_config& tc) {
  wg_field_s* f = s->field;
  CKL(launch_adam(f->p.as<float>(), f->m.as<double>(), f->v.as<double>(), s->grad.as<float>(),
                  f->n_params, tc.lr, tc.beta1, tc.beta2, tc.eps,
                  static_cast<double>(tc.minibatch), f->adam.as<AdamCtl>(), f->view,
                  f->wpack.p && !f->pack_dirty ? f->wpack.as<unsigned char>() : nullptr, s->stream));
}

// train_batch on the arena's records (guide_train.cpp:94-198), enqueued only
void enqueue_train(wg_solver_s* s, const wg_train_config& tc) {
  check_trainable(s);
  wg_field_s* f = s->field;
  ensure_train_buffers(s, tc);
  CK(cudaEventRecord(pool_event(s->ev_train, s->n_train_ev), s->stream));
  enqueue_finalize(s, tc.pdf_floor);
  enqueue_usable_global(s, nullptr);
  enqueue_select(s, tc);
  const int n_mb = n_minibatches(tc);
  for (int b = 0; b < n_mb; ++b) {
    // records enter the fp32 gradient sum pre-scaled by 1 / minibatch (the
    // same constant on every rank); Adam divides by count / minibatch
    enqueue_minibatch(s, tc, b, 1.0 / static_cast<double>(tc.minibatch));
    if (s->comm)
      NCK(nccl().allReduce(s->grad.p, s->grad.p, f->n_params + 1, ncclFloat, ncclSum, s->comm,
                        s->stream));
    enqueue_adam(s, tc);
  }
  CK(cudaEventRecord(pool_event(s->ev_train, s->n_train_ev), s->stream));
}

long long adam_steps(wg_solver_s* s) {
  long long st = 0;
  CK(cudaMemcpyAsync(&st, s->field->adam.p, sizeof(long long), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return st;
}

// synchronise and collect counters, timings and TrainStats
wg_train_stats sync_collect(wg_solver_s* s, long long steps_before) {
  CK(cudaStreamSynchronize(s->stream));
  CK(cudaMemcpy(s->last_counters, s->counters.p, sizeof(s->last_counters), cudaMemcpyDeviceToHost));
  g_launches += static_cast<int64_t>(s->last_counters[C_WAVE_LAUNCHES]);
  CK(cudaMemset(s->counters.as<unsigned long long>() + C_WAVE_LAUNCHES, 0, sizeof(unsigned long long)));
  if (s->last_counters[C_REC_OVERFLOW] > 0) {
    // a collecting round filled the record arena: its walks stopped recording,
    // which would have trained on a short-walk-biased set. Fail the call (the
    // arena is doubled for the next one; wostgpu_solver_reserve_records
    // pre-sizes it) instead of returning a silently biased field.
    s->rec_capacity_min = std::max<int64_t>(s->rec_capacity_min, 2 * s->rec_capacity);
    char msg[256];
    std::snprintf(msg, sizeof(msg),
                  "record arena overflow in a training round (%llu record chunks dropped, capacity %lld "
                  "records); the arena now holds %lld records: rerun, or reserve more with "
                  "wostgpu_solver_reserve_records",
                  s->last_counters[C_REC_OVERFLOW], static_cast<long long>(s->rec_capacity),
                  static_cast<long long>(s->rec_capacity_min));
    throw wgrt::WgError(WG_ERR_RUNTIME, msg);
  }
  s->last_walk_ms = pool_ms(s->ev_walk, s->n_walk_ev);
  s->last_train_ms = pool_ms(s->ev_train, s->n_train_ev);
  need(s->last_counters[C_SCENE_ERR] == 0, WG_ERR_SCENE,
       "walk: unbounded star region (no Dirichlet boundary and no Neumann silhouette)");
  wg_train_stats st{};
  if (s->field && steps_before >= 0) {
    TrainTotals t{};
    CK(cudaMemcpy(&t, s->totals.p, sizeof(t), cudaMemcpyDeviceToHost));
    AdamCtl* a = s->field->adam.as<AdamCtl>();
    long long steps_after = 0;
    CK(cudaMemcpy(&steps_after, a, sizeof(long long), cudaMemcpyDeviceToHost));
    st.records_seen = (int64_t)t.seen;
    st.records_consumed = (int64_t)t.consumed;
    st.skipped_low_pdf = (int64_t)t.low_pdf;
    st.skipped_low_v = (int64_t)t.skipped_v;
    st.steps = steps_after - steps_before;
    if (st.steps > 0) {
      std::vector<double> n2(kNormRing);
      CK(cudaMemcpy(n2.data(), a->norm2, sizeof(double) * kNormRing, cudaMemcpyDeviceToHost));
      double acc = 0.0;
      for (long long k = steps_before; k < steps_after; ++k) acc += std::sqrt(n2[k % kNormRing]);
      st.mean_grad_norm = acc / static_cast<double>(st.steps);
    }
    st.seconds = s->last_train_ms * 1e-3;
  }
  return st;
}

uint64_t round_key_seed(uint64_t seed, uint64_t wpp) {
  return Pcg::mix(seed ^ 0x7261696e5f6b6579ULL) ^ Pcg::mix(wpp + 1);
}

void import_records(wg_solver_s* s, const wg_guide_record* recs, int64_t n, double pdf_floor) {
  int64_t cap = std::max<int64_t>(n, 1);
  if (s->rec_capacity < cap) {
    s->recs.alloc(sizeof(DevRecord) * cap);
    s->rec_capacity = cap;
  }
  DBuf h;
  h.upload(recs, (size_t)n);
  CKL(launch_import_records(h.as<wg_guide_record>(), n, s->recs.as<DevRecord>(), s->stream));
  s->rec_counter.alloc(sizeof(unsigned long long));
  unsigned long long nn = static_cast<unsigned long long>(n);
  CK(cudaMemcpyAsync(s->rec_counter.p, &nn, sizeof(nn), cudaMemcpyHostToDevice, s->stream));
  s->recs_from_walks = false;
  enqueue_finalize(s, pdf_floor);
  CK(cudaStreamSynchronize(s->stream));  // h goes out of scope
}

}  // namespace

extern "C" {

int wostgpu_solver_create(wg_scene scene, wg_field field, const wg_solver_config* cfg,
                          wg_solver* out) {
  return guarded([&] {
    check_device();
    need(scene != nullptr, WG_ERR_INVALID, "solver needs a scene");
    need(field == nullptr || field->sdim == 2, WG_ERR_INVALID,
         "2D solver: the field is 3D (use wostgpu_solver3_create)");
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
    s->mlp = WG_MLP_TENSOR;  // fast path; WG_MLP_EXACT = bit-faithful reference arithmetic
    CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&s->ev_run0));
    CK(cudaEventCreate(&s->ev_run1));
    s->sms = sm_count();
    reset_run(s.get());
    *out = s.release();
  });
}

int wostgpu_solver_destroy(wg_solver s) {
  return guarded([&] {
    if (!s) return;
    cudaStreamSynchronize(s->stream);
    if (s->comm) nccl().commDestroy(s->comm);
    for (cudaEvent_t e : s->ev_walk) cudaEventDestroy(e);
    for (cudaEvent_t e : s->ev_train) cudaEventDestroy(e);
    cudaEventDestroy(s->ev_run0);
    cudaEventDestroy(s->ev_run1);
    cudaStreamDestroy(s->stream);
    if (s->h_qlen) cudaFreeHost(s->h_qlen);
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
    reset_run(s);
    enqueue_rounds(s, seed, wpp_first, n_rounds, collect != 0, round_key_seed(seed, wpp_first),
                   1e-8);
    sync_collect(s, -1);
  });
}

int wostgpu_solve_batch(wg_solver s, int64_t n, const double* xy, wg_point_stats* st,
                        uint64_t seed, uint64_t wpp, int32_t collect_records) {
  int rc = wostgpu_solver_set_points(s, n, xy, 0);
  if (rc) return rc;
  rc = wostgpu_solver_set_stats(s, st);
  if (rc) return rc;
  rc = wostgpu_solve_rounds(s, seed, wpp, 1, collect_records);
  if (rc) return rc;
  return wostgpu_solver_get_stats(s, st);
}

int wostgpu_fetch_records(wg_solver s, wg_guide_record* out, int64_t capacity, int64_t* n) {
  return guarded([&] {
    need(s->have_records, WG_ERR_INVALID, "no collecting round has run");
    enqueue_finalize(s, 1e-8);  // targets from the walks' final estimates
    unsigned long long total = 0;
    CK(cudaMemcpyAsync(&total, s->rec_counter.p, 8, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    int64_t m = std::min<int64_t>((int64_t)total, s->rec_capacity);
    DBuf d, c;
    d.alloc(sizeof(wg_guide_record) * std::max<int64_t>(m, 1));
    c.alloc(8);
    CK(cudaMemsetAsync(c.p, 0, 8, s->stream));
    CKL(launch_export_records(s->recs.as<DevRecord>(), m, d.as<wg_guide_record>(),
                              c.as<unsigned long long>(), s->stream));
    unsigned long long cnt = 0;
    CK(cudaMemcpyAsync(&cnt, c.p, 8, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    *n = (int64_t)cnt;
    if (out) {
      int64_t k = std::min<int64_t>((int64_t)cnt, capacity);
      CK(cudaMemcpy(out, d.p, sizeof(wg_guide_record) * k, cudaMemcpyDeviceToHost));
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
    if (walks) *walks = (int64_t)s->last_counters[C_WALKS];
    if (steps) *steps = (int64_t)s->last_counters[C_STEPS];
    if (escaped) *escaped = (int64_t)s->last_counters[C_ESCAPED];
    if (records) {
      unsigned long long r = 0;
      if (s->have_records) {
        CK(cudaMemcpyAsync(&r, s->rec_counter.p, 8, cudaMemcpyDeviceToHost, s->stream));
        CK(cudaStreamSynchronize(s->stream));
      }
      *records = (int64_t)r;
    }
  });
}

int wostgpu_train_round(wg_solver s, const wg_train_config* cfg, uint64_t round,
                        wg_train_stats* stats) {
  (void)round;
  return guarded([&] {
    need(s->have_records, WG_ERR_INVALID, "no collecting round has run");
    reset_run(s);
    long long before = adam_steps(s);
    enqueue_train(s, *cfg);
    wg_train_stats st = sync_collect(s, before);
    if (stats) *stats = st;
  });
}

// train_batch (guide_train.cpp:94-198) on host records with the reference's
// own selection: usable records (pdf_mis >= floor) in a Fisher-Yates order
// from Rng(mix(seed) ^ mix(round + 1), round), truncated to the cap, cut
// into consecutive minibatches; one device gradient + Adam step per
// minibatch over exactly the records the reference uses. (The device-side
// rounds select by key thinning instead, wg_train.cu compact_kernel: the
// host never waits there.)
int wostgpu_train_batch(wg_solver s, const wg_guide_record* recs, int64_t n,
                        const wg_train_config* cfg, uint64_t round, wg_train_stats* stats) {
  return guarded([&] {
    check_trainable(s);
    need(n >= 0 && (n == 0 || recs != nullptr), WG_ERR_INVALID, "records: null pointer");
    need(n <= static_cast<int64_t>(UINT32_MAX), WG_ERR_INVALID, "too many records");
    need(cfg->minibatch >= 1, WG_ERR_INVALID, "minibatch must be >= 1");
    wg_train_stats st{};
    st.records_seen = n;
    std::vector<uint32_t> order;
    order.reserve(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      if (recs[i].pdf_mis < cfg->pdf_floor) ++st.skipped_low_pdf;
      else order.push_back(static_cast<uint32_t>(i));
    }
    Pcg rng;
    rng.seed(Pcg::mix(cfg->seed) ^ Pcg::mix(round + 1), round);
    for (size_t i = order.size(); i > 1; --i) {
      // Rng::uniform_index (rng.hpp:61-73): Lemire's bounded draw
      const uint32_t m_n = static_cast<uint32_t>(i);
      uint64_t m = static_cast<uint64_t>(rng.u32()) * m_n;
      uint32_t lo = static_cast<uint32_t>(m);
      if (lo < m_n) {
        const uint32_t t = (0u - m_n) % m_n;
        while (lo < t) {
          m = static_cast<uint64_t>(rng.u32()) * m_n;
          lo = static_cast<uint32_t>(m);
        }
      }
      std::swap(order[i - 1], order[static_cast<size_t>(m >> 32)]);
    }
    if (static_cast<int64_t>(order.size()) > cfg->max_records_per_round)
      order.resize(static_cast<size_t>(cfg->max_records_per_round));
    if (order.empty()) {
      s->have_records = false;
      if (stats) *stats = st;
      return;
    }
    reset_run(s);
    const long long before = adam_steps(s);
    import_records(s, recs, n, cfg->pdf_floor);
    ensure_train_buffers(s, *cfg);
    CK(cudaEventRecord(pool_event(s->ev_train, s->n_train_ev), s->stream));
    const int64_t mb = cfg->minibatch;
    for (int64_t b0 = 0; b0 < static_cast<int64_t>(order.size()); b0 += mb) {
      const unsigned long long cnt = static_cast<unsigned long long>(
          std::min<int64_t>(mb, static_cast<int64_t>(order.size()) - b0));
      // pageable sources: the copies are staged before the calls return
      CK(cudaMemcpyAsync(s->lists.p, order.data() + b0, sizeof(uint32_t) * cnt, cudaMemcpyHostToDevice,
                         s->stream));
      CK(cudaMemcpyAsync(&s->ctl.as<TrainCtl>()->mb_count[0], &cnt, sizeof(cnt), cudaMemcpyHostToDevice,
                         s->stream));
      enqueue_minibatch(s, *cfg, 0, 1.0 / static_cast<double>(cfg->minibatch));
      enqueue_adam(s, *cfg);
    }
    CK(cudaEventRecord(pool_event(s->ev_train, s->n_train_ev), s->stream));
    const wg_train_stats d = sync_collect(s, before);
    st.records_consumed = d.records_consumed;
    st.skipped_low_v = d.skipped_low_v;
    st.steps = d.steps;
    st.mean_grad_norm = d.mean_grad_norm;
    st.seconds = d.seconds;
    s->have_records = false;
    if (stats) *stats = st;
  });
}

int wostgpu_field_check_pack(wg_field f, int64_t* mismatched_bytes) {
  return guarded([&] {
    need(f != nullptr && mismatched_bytes != nullptr, WG_ERR_INVALID, "null argument");
    *mismatched_bytes = -1;
    if (!f->wpack.p || f->pack_dirty) return;  // no maintained blob to check
    DBuf fresh;
    fresh.alloc(wpack::BYTES);
    CK(cudaMemset(fresh.p, 0, wpack::BYTES));
    CKL(launch_pack_weights(f->view, fresh.as<unsigned char>(), 0));
    CK(cudaDeviceSynchronize());
    std::vector<unsigned char> a(wpack::BYTES), b(wpack::BYTES);
    CK(cudaMemcpy(a.data(), f->wpack.p, wpack::BYTES, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), fresh.p, wpack::BYTES, cudaMemcpyDeviceToHost));
    int64_t m = 0;
    for (size_t i = 0; i < a.size(); ++i) m += a[i] != b[i];
    *mismatched_bytes = m;
  });
}

int wostgpu_field_grad(wg_solver s, const wg_guide_record* recs, int64_t n,
                       const wg_train_config* cfg, double* grad) {
  return guarded([&] {
    wg_field_s* f = s->field;
    need(f != nullptr, WG_ERR_INVALID, "gradient needs a guiding field");
    need(default_shape(f->view), WG_ERR_NOT_BUILT, "device training is built for the default field shape");
    reset_run(s);
    import_records(s, recs, n, cfg->pdf_floor);
    wg_train_config tc = *cfg;
    tc.minibatch = static_cast<int32_t>(std::max<int64_t>(n, 1));
    tc.max_records_per_round = tc.minibatch;
    ensure_train_buffers(s, tc);
    // the given order, low-pdf records dropped (the reference skips them)
    std::vector<uint32_t> ord;
    for (int64_t i = 0; i < n; ++i)
      if (recs[i].pdf_mis >= cfg->pdf_floor) ord.push_back((uint32_t)i);
    CK(cudaMemcpyAsync(s->lists.p, ord.data(), sizeof(uint32_t) * ord.size(), cudaMemcpyHostToDevice,
                       s->stream));
    unsigned long long cnt = ord.size();
    CK(cudaMemcpyAsync(&s->ctl.as<TrainCtl>()->mb_count[0], &cnt, sizeof(cnt), cudaMemcpyHostToDevice,
                       s->stream));
    enqueue_minibatch(s, tc, 0, 1.0 / static_cast<double>(n));
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
    const bool guided = s->cfg.mode != WG_MODE_UNIFORM;
    const bool train = guided && tcfg != nullptr;
    reset_run(s);
    long long before = train ? adam_steps(s) : -1;
    const double pdf_floor = tcfg ? tcfg->pdf_floor : 1e-8;
    CK(cudaEventRecord(s->ev_run0, s->stream));
    int32_t b = 0;
    // Engine::run_batch while training is active (solver.cpp:92-104)
    for (; train && b < wpp && (int64_t)b < train_until; ++b) {
      enqueue_rounds(s, seed, (uint64_t)b, 1, true, round_key_seed(seed, (uint64_t)b), pdf_floor);
      enqueue_train(s, *tcfg);
    }
    // walk steps taken on training rounds (they also write trace records)
    unsigned long long* c = s->counters.as<unsigned long long>();
    CK(cudaMemcpyAsync(c + C_TRAIN_STEPS, c + C_STEPS, sizeof(unsigned long long),
                       cudaMemcpyDeviceToDevice, s->stream));
    // the remaining rounds share a frozen field: one multi-round launch
    if (b < wpp) enqueue_rounds(s, seed, (uint64_t)b, wpp - b, false, 0, pdf_floor);
    CK(cudaEventRecord(s->ev_run1, s->stream));
    wg_train_stats st = sync_collect(s, before);
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, s->ev_run0, s->ev_run1));
    if (device_ms) *device_ms = ms;
    if (totals) *totals = st;
  });
}

int wostgpu_run_profile(wg_solver s, double* walk_ms, double* train_ms, int64_t* walks,
                        int64_t* steps, int64_t* escaped, int64_t* train_steps) {
  return guarded([&] {
    if (walk_ms) *walk_ms = s->last_walk_ms;
    if (train_ms) *train_ms = s->last_train_ms;
    if (walks) *walks = (int64_t)s->last_counters[C_WALKS];
    if (steps) *steps = (int64_t)s->last_counters[C_STEPS];
    if (escaped) *escaped = (int64_t)s->last_counters[C_ESCAPED];
    if (train_steps) *train_steps = (int64_t)s->last_counters[C_TRAIN_STEPS];
  });
}

int wostgpu_comm_unique_id(char id[128]) {
  return guarded([&] {
    ncclUniqueId u;
    NCK(nccl().getUniqueId(&u));
    static_assert(sizeof(u) == 128, "nccl id size");
    std::memcpy(id, &u, 128);
  });
}

int wostgpu_solver_reserve_records(wg_solver s, int64_t n) {
  return guarded([&] {
    need(n >= 0, WG_ERR_INVALID, "record count must be >= 0");
    s->rec_capacity_min = std::max<int64_t>(s->rec_capacity_min, n);
  });
}

int wostgpu_solver_attach_comm(wg_solver s, const char id[128], int32_t nranks, int32_t rank) {
  return guarded([&] {
    need(nranks >= 1 && rank >= 0 && rank < nranks, WG_ERR_INVALID, "bad rank / nranks");
    if (s->comm) {  // re-attach: release the previous communicator
      CK(cudaStreamSynchronize(s->stream));
      nccl().commDestroy(s->comm);
      s->comm = nullptr;
    }
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    NCK(nccl().commInitRank(&s->comm, nranks, u, rank));
    s->nranks = nranks;
    s->rank = rank;
  });
}

int wostgpu_train_prepare(wg_solver s, const wg_train_config* cfg, int64_t* usable_local) {
  return guarded([&] {
    need(s->have_records && s->recs_from_walks, WG_ERR_INVALID, "train_prepare needs a collecting round");
    check_trainable(s);
    reset_run(s);
    ensure_train_buffers(s, *cfg);
    enqueue_finalize(s, cfg->pdf_floor);
    unsigned long long u = 0;
    CK(cudaMemcpyAsync(&u, &s->ctl.as<TrainCtl>()->usable, sizeof(u), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    if (usable_local) *usable_local = static_cast<int64_t>(u);
  });
}

int wostgpu_train_select(wg_solver s, const wg_train_config* cfg, int64_t usable_global,
                         int32_t* n_mb) {
  return guarded([&] {
    need(s->have_records, WG_ERR_INVALID, "train_select needs prepared records");
    need(usable_global >= 0, WG_ERR_INVALID, "usable_global must be >= 0");
    check_trainable(s);
    ensure_train_buffers(s, *cfg);
    enqueue_usable_global(s, &usable_global);
    enqueue_select(s, *cfg);
    CK(cudaStreamSynchronize(s->stream));
    if (n_mb) *n_mb = n_minibatches(*cfg);
  });
}

int wostgpu_train_minibatch_grad(wg_solver s, const wg_train_config* cfg, int32_t b, float* grad_sum) {
  return guarded([&] {
    need(s->have_records, WG_ERR_INVALID, "train_minibatch_grad needs selected records");
    need(b >= 0 && b < n_minibatches(*cfg), WG_ERR_INVALID, "minibatch index out of range");
    check_trainable(s);
    ensure_train_buffers(s, *cfg);
    enqueue_minibatch(s, *cfg, b, 1.0 / static_cast<double>(cfg->minibatch));
    CK(cudaMemcpyAsync(grad_sum, s->grad.p, sizeof(float) * (s->field->n_params + 1),
                       cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
  });
}

int wostgpu_train_apply(wg_solver s, const wg_train_config* cfg, const float* grad_sum) {
  return guarded([&] {
    check_trainable(s);
    ensure_train_buffers(s, *cfg);
    CK(cudaMemcpyAsync(s->grad.p, grad_sum, sizeof(float) * (s->field->n_params + 1),
                       cudaMemcpyHostToDevice, s->stream));
    enqueue_adam(s, *cfg);
    CK(cudaStreamSynchronize(s->stream));
  });
}

int wostgpu_solver_timing(wg_solver s, double* walk_ms, double* train_ms) {
  return guarded([&] {
    if (walk_ms) *walk_ms = s->last_walk_ms;
    if (train_ms) *train_ms = s->last_train_ms;
  });
}

}  // extern "C"
