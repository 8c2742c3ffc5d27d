// Training kernels' argument block and launchers (wg_train.cu, wg_train_tc.cu).
#pragma once

#include "wg_kernels.cuh"

namespace wg {

struct TrainArgs {
  FieldView f;
  const DevRecord* recs;
  const uint32_t* order;  // sorted record indices
  int64_t begin, count;   // minibatch slice of `order`
  float* grad;            // [n_params], accumulated
  double inv_count;
  int32_t reflect, learn_selection;
  double e_fraction, v_floor;
  unsigned long long* counters;  // [0] consumed, [1] skipped_low_v
};

size_t sort_temp_bytes(int64_t n);
cudaError_t launch_select(const DevRecord* recs, int64_t n, double pdf_floor, uint64_t* keys,
                          uint64_t* keys_sorted, uint32_t* idx, uint32_t* idx_sorted, void* temp,
                          size_t temp_bytes, unsigned long long* cnt, cudaStream_t st);
size_t grad_tile_smem();
cudaError_t launch_grad_cuda_core(const TrainArgs& a, cudaStream_t st);
cudaError_t launch_adam(float* p, double* m, double* v, float* g, int64_t n, double lr, double b1,
                        double b2, double eps, int64_t step, const float* count, double* norm2,
                        cudaStream_t st);
cudaError_t launch_import_records(const wg_guide_record* in, int64_t n, DevRecord* out,
                                  cudaStream_t st);
cudaError_t launch_export_records(const DevRecord* in, int64_t n, wg_guide_record* out,
                                  unsigned long long* count, cudaStream_t st);

}  // namespace wg
