// Kernel argument blocks and launch wrappers shared by the kernel TUs and the
// host runtime (wg_runtime.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "wg_device.cuh"
#include "wg_field.cuh"

namespace wg {

// Guide record as kept in HBM during a collecting round (80 B), one per walk
// step, appended by the walk kernel.
//
// Target without a backward pass: backfill_targets_append
// (proj/src/guide_train.cpp:58-79) runs u_k = rr_k (local_k + mult_k u_{k+1})
// backwards from the terminal value. Unrolled, u_0 = P_{k+1} + Q_{k+1} u_{k+1}
// with P_{k+1} = the walk's accumulated estimate after step k's local term and
// Q_{k+1} = its throughput after step k's multiplier, and u_0 is the walk's
// final estimate. So each record stores (P, Q) when it is written and the
// target |u_{k+1}| = |(u_0 - P) / Q| is formed later, in one parallel pass,
// from the walk's final estimate — no per-walk serial chain in the walk kernel.
struct __align__(16) DevRecord {
  float x, y;
  float nux, nuy;
  float nx, ny;
  float pdf_mis, pdf_g, pdf_u, c;
  float target;  // |u(x_{k+1})|, filled by the finalise pass
  float dacc;    // accumulator increments since the walk's previous record
                 // (this step's source / Neumann term included)
  float thr_q;   // Q: throughput after this step's multiplier (0 = walk died)
  float pad_;
  int32_t walk;  // estimate-buffer slot of the walk (round * n_points + point); -1 imported
  uint32_t flags;
  uint64_t key;  // deterministic selection key (seed, round, point, depth)
  int32_t prev;  // arena slot of the walk's previous record, -1 for its first
  int32_t pad2_;
};
// Targets (backfill_targets_append, guide_train.cpp:58-79): with the walk's
// terminal term S_K = T_K g (0 when killed), S_{k+1} = S_K + sum_{j>k} dacc_j
// and target_k = |S_{k+1} / Q_k|. A backward suffix sum like the reference's
// recursion, so no cancellation against the walk total when throughputs
// decay; scenes without source / Neumann terms have dacc = 0 and need no
// chain walk (target = |S_K / Q_k|, one record per thread).
static_assert(sizeof(DevRecord) == 80 && offsetof(DevRecord, walk) == 56 && offsetof(DevRecord, key) == 64,
              "record layout (compact_kernel loads walk|flags and key by offset)");
enum : uint32_t { REC_ON_NEUMANN = 1u, REC_VALID = 2u, REC_USABLE = 4u, REC_WRITTEN = 8u };

struct TrainCtl;  // wg_train.cuh

struct SolverParams {
  double eps, rmin, fixed_c, grazing_floor;
  int32_t rr_depth, max_steps, mode, reflect, clamp_grazing;
};

struct WalkArgs {
  SceneView scene;         // global-memory view
  int32_t scene_smem_bytes;  // > 0: stage nodes/segs/silhouettes in smem
  FieldView field;
  SolverParams sp;
  const double* points;  // [n_points][2]
  int64_t n_points;
  int64_t point_offset;  // global index of points[0]
  uint64_t seed;
  uint64_t wpp_first;
  int32_t n_rounds;
  double* est;      // [n_rounds][n_points]
  int32_t* esc;     // [n_rounds][n_points]
  int32_t* steps;   // [n_rounds][n_points] (may be null)
  // records (collecting rounds)
  DevRecord* recs;
  unsigned long long* rec_counter;
  int64_t rec_capacity;
  uint64_t key_seed;
  double pdf_floor;  // TrainConfig::pdf_floor, for the usable-record count
  TrainCtl* ctl;     // round's record counts (collecting rounds)
  // counters: [0] steps, [1] escaped, [2] walks, [3] record overflow, [4] scene error
  unsigned long long* counters;
  // per walk (collecting rounds): arena slot of the walk's last record (-1:
  // none) and its terminal term T_K g plus increments after the last record
  int32_t* rec_tail;
  double* rec_term;
  // tensor-core kernel: the field's packed split-fp16 weights (wg_wpack.cuh)
  const unsigned char* wblob;
  // tensor-core lockstep kernel: CUDA-core MLP for tail iterations (<= 16
  // live rows). Off when its shared memory would cost the launch its second
  // CTA per SM (large staged scenes with many walks in flight)
  int32_t small_mlp;
  // optional per-CTA phase timing [gridDim][8]: cycles in phase A (begin
  // step + barrier), B (MLP), C (sample + move), iterations, MMA windows,
  // gather, MLP prep (WOSTGPU_PHASE_PROF)
  unsigned long long* phase_prof;
  // lockstep-kernel tail handoff: once at most spill_rows walks of a CTA are
  // live and it has no fresh walks left, the CTA writes them here (count in
  // counters[7]) and exits; the warp-per-walk kernel finishes them
  // (walk_kernel_coop_resume). 0 = off
  struct SpillLane* spill;
  int32_t spill_rows;
};

// a walk handed from the lockstep kernel's tail to the warp-per-walk kernel:
// its state after begin_step, direction still to draw (TLane / CLane fields)
struct SpillLane {
  double x, y, nx, ny, T, acc, dacc, R;
  int64_t point, rec_base;
  Pcg rng;
  int32_t seg, depth, rec, round, rec_left, last_rec, on_n, rec_ok;
};

struct QueryArgs {
  SceneView scene;
  int64_t n;
  int32_t op;  // 0 closest_point, 1 silhouette, 2 ray, 3 star radius
  uint32_t kinds;
  double r_min;
  const double* xy;
  const double* dir;
  const double* t_max;
  const int32_t* exclude;
  double* out_d;     // dist / t / r
  double* out_pt;    // [n][2]
  double* out_n;     // [n][2]
  int32_t* out_seg;
  int32_t* out_kind;
  unsigned long long* err;
};

// launchers (defined in wg_walk.cu)
cudaError_t launch_queries(const QueryArgs& a, cudaStream_t st);
cudaError_t launch_walks(const WalkArgs& a, bool guided_exact_default, bool guided_generic,
                         int blocks, cudaStream_t st);
int walk_blocks_per_sm(bool guided_exact_default, bool guided_generic, int smem_bytes);
// 8-lanes-per-walk guided kernel for the default field shape (wg_walk_g8.cu)
int walk_g8_smem(const WalkArgs& a);
int walk_g8_blocks_per_sm(int smem);
cudaError_t launch_walks_g8(const WalkArgs& a, int blocks, cudaStream_t st);
// tcgen05 MLP walk kernel / field evaluation (wg_walk_tc.cu)
int walk_tc_smem(const WalkArgs& a);
int walk_tc_blocks_per_sm(int smem);
int walk_tc_block();
cudaError_t launch_walks_tc(const WalkArgs& a, int blocks, cudaStream_t st);
// warp-per-walk guided kernel for the default field shape (wg_walk_coop.cu)
int walk_coop_smem(const WalkArgs& a);
cudaError_t launch_walks_coop_resume(const WalkArgs& a, int max_walks, int sms, cudaStream_t st);
// wavefront pair for guided 2D walks on the tensor cores (wg_wave2.cu)
void wave2_sizes(size_t* lane_bytes, size_t* dir_bytes);
cudaError_t launch_walks2_wave(const WalkArgs& a, void* lanes, void* dirs, int32_t* rec, uint8_t* state,
                               int32_t* queue, unsigned int* qlen, unsigned long long* next_walk,
                               int64_t slots, int sms, unsigned int* h_qlen, int64_t* launches,
                               cudaStream_t st);
cudaError_t launch_mix32_pdf(const float* raw, int64_t n, const double* nu, double* out, cudaStream_t st);
cudaError_t launch_mix32_sample(const float* raw, int64_t n, uint64_t seed, double* out, cudaStream_t st);
cudaError_t launch_field_eval_tc(const FieldView& f, int64_t n, const double* xy, double* out,
                                 int sm_count, cudaStream_t st);
cudaError_t launch_welford(const double* est, const int32_t* esc, int64_t n_points,
                           int32_t n_rounds, wg_point_stats* stats, cudaStream_t st);
cudaError_t launch_field_eval(const FieldView& f, int64_t n, const double* xy, double* out,
                              cudaStream_t st);
cudaError_t launch_normalize(int64_t n, const double* raw, int k, int dim, wg_mixture* out,
                             cudaStream_t st);

}  // namespace wg
