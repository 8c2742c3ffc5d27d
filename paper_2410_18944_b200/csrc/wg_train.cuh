// Training kernels' argument blocks and launchers (wg_train.cu, wg_train_tc.cu).
//
// A training round runs entirely on the device with no host synchronisation:
//   walk kernels count valid / usable records at backfill (TrainCtl),
//   compact_kernel thins the usable records to the round's training set and
//     splits it into minibatch index lists,
//   per minibatch: grad tile kernel -> [NCCL allreduce] -> adam_prep -> adam,
//   where the record count travels in the gradient buffer's last slot, so the
//   (global) minibatch size and "is there a step at all" are decided on device.
#pragma once

#include "wg_kernels.cuh"

namespace wg {

constexpr int kMaxMinibatches = 8;
constexpr int kNormRing = 4096;

// per-solver, reset at the start of every collecting round
struct TrainCtl {
  unsigned long long seen, usable, low_pdf;  // this rank's records, filled at backfill
  unsigned long long usable_global;          // usable summed over the ranks (selection rate)
  unsigned long long mb_count[kMaxMinibatches];
  unsigned long long overflow;
};

// per-run totals (TrainStats, proj/include/wost/guide_train.hpp:48-58)
struct TrainTotals {
  unsigned long long seen, low_pdf, consumed, skipped_v, overflow;
};

// per-field optimizer control (device truth of GuidingField::adam_steps_).
// adam_kernel reads `steps` when it starts and the last of its blocks to
// finish advances it, so no separate control launch sits between the
// gradient and the update.
struct AdamCtl {
  long long steps;
  double norm_acc;     // |g|^2 block partials of the running step
  unsigned int done;   // blocks of the running step that have finished
  int pad;
  double norm2[kNormRing];  // |g|^2 of every step (ring)
};

struct TrainArgs {
  FieldView f;
  const DevRecord* recs;
  const uint32_t* list;                // record indices of this minibatch
  const unsigned long long* count;     // device: number of valid entries in list
  int64_t list_cap;                    // grid covers list_cap records
  float* grad;                         // [n_params + 1]; grad[n_params] = record count
  int64_t n_params;
  double inv_count;                    // per-record scale: 1 / minibatch in training
                                       // (keeps the fp32 sums in range; Adam rescales
                                       // by minibatch / count), 1 / n in field_grad
  int32_t reflect, learn_selection;
  double e_fraction, v_floor;
  TrainTotals* totals;
  const unsigned char* packed;         // tensor-core tile: split-fp16 weight blob (pack kernel)
};

cudaError_t launch_compact(const DevRecord* recs, const unsigned long long* rec_count,
                           int64_t capacity, TrainCtl* ctl, TrainTotals* totals, uint32_t* lists,
                           int64_t list_cap, int64_t max_records, int32_t minibatch,
                           cudaStream_t st);
// targets (DevRecord), validity and usable counts of the arena's records;
// chain = the scene has source / Neumann terms (per-walk backward suffix sums)
cudaError_t launch_finalize_records(DevRecord* recs, const unsigned long long* rec_count,
                                    int64_t capacity, int64_t n_walks, const int32_t* tail,
                                    const double* term, const int32_t* esc, double pdf_floor,
                                    TrainCtl* ctl, bool chain, cudaStream_t st);
size_t grad_tile_smem();
size_t grad_tc_pack_bytes();
cudaError_t launch_grad_cuda_core(const TrainArgs& a, cudaStream_t st);
// Adam step on all n parameters with the mean gradient prescale * g[0..n) /
// g[n] (g holds sum_i grad_i / prescale, g[n] the record count); no step when
// g[n] == 0. blob != nullptr: the packed weight
// blob (wg_wpack.cuh) is updated for every MLP parameter written.
cudaError_t launch_adam(float* p, double* m, double* v, const float* g, int64_t n, double lr, double b1,
                        double b2, double eps, double prescale, AdamCtl* ctl, const FieldView& f,
                        unsigned char* blob, cudaStream_t st);
cudaError_t launch_import_records(const wg_guide_record* in, int64_t n, DevRecord* out,
                                  cudaStream_t st);
cudaError_t launch_export_records(const DevRecord* in, int64_t n, wg_guide_record* out,
                                  unsigned long long* count, cudaStream_t st);

}  // namespace wg
