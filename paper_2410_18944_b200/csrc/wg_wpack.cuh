// Packed split-fp16 weight blob of the default guiding-field MLP
// (16 -> 64 -> 64 -> 33), laid out exactly as the tensor-core kernels keep
// the weights in shared memory, so a kernel fetches them with one TMA bulk
// copy instead of re-splitting ~8k fp32 weights in every CTA:
//
//   [B1 hi|lo][B2 hi|lo][B3 hi|lo][bias b1|b2|b3]   forward tiles (walk kernel prefix)
//   [C3 hi|lo][C2 hi|lo][C1 hi|lo]                  backward tiles (training tile)
//
// B_l[n][k] = W_l[k][n] (K-major B operand of the forward GEMM, N x K) and
// C_l[n][k] = W_l[n][k] (K-major B operand of the backward GEMM); every value
// v is stored as hi = fp16(v), lo = fp16(v - hi). The blob lives with the
// field (wg_field_s::wpack): pack_weights_kernel writes all of it whenever
// the parameters change from the host, and adam_kernel rewrites the entries
// of each MLP parameter it updates.
#pragma once

#include <cuda_fp16.h>

#include "wg_field.cuh"
#include "wg_umma.cuh"

namespace wg {
namespace wpack {

constexpr uint32_t BW1 = 64 * 16 * 2, BW2 = 64 * 64 * 2, BW3F = 48 * 64 * 2, BW3B = 64 * 48 * 2,
                   BW1B = 16 * 64 * 2;
constexpr uint32_t B1H = 0, B1L = B1H + BW1;
constexpr uint32_t B2H = B1L + BW1, B2L = B2H + BW2;
constexpr uint32_t B3H = B2L + BW2, B3L = B3H + BW3F;
constexpr uint32_t BIAS = B3L + BW3F;  // fp32: b1 [64], b2 [64], b3 [48] (33 used)
constexpr uint32_t C3H = BIAS + (64 + 64 + 48) * 4, C3L = C3H + BW3B;
constexpr uint32_t C2H = C3L + BW3B, C2L = C2H + BW2;
constexpr uint32_t C1H = C2L + BW2, C1L = C1H + BW1B;
constexpr uint32_t BYTES = C1L + BW1B;
constexpr uint32_t FWD_BYTES = C3H;  // forward tiles + biases
static_assert(BIAS % 16 == 0 && C3H % 16 == 0 && BYTES % 16 == 0, "bulk-copy granularity");

__device__ __forceinline__ void put(unsigned char* blob, uint32_t hi, uint32_t lo, int n, int k, int K,
                                    float v) {
  const __half h = __float2half_rn(v), l = __float2half_rn(v - __half2float(h));
  const uint32_t o = umma::kmajor_off(n, k, K);
  *reinterpret_cast<__half*>(blob + hi + o) = h;
  *reinterpret_cast<__half*>(blob + lo + o) = l;
}

// the blob entries of parameter i (absolute index into the field's params,
// i >= f.w1) with value v
__device__ __forceinline__ void pack_param(const FieldView& f, unsigned char* blob, int64_t i, float v) {
  float* bias = reinterpret_cast<float*>(blob + BIAS);
  if (i < f.b1) {  // W1 [16][64]
    const int j = static_cast<int>(i - f.w1), k = j / 64, n = j % 64;
    put(blob, B1H, B1L, n, k, 16, v);
    put(blob, C1H, C1L, k, n, 64, v);
  } else if (i < f.w2) {
    bias[i - f.b1] = v;
  } else if (i < f.b2) {  // W2 [64][64]
    const int j = static_cast<int>(i - f.w2), k = j / 64, n = j % 64;
    put(blob, B2H, B2L, n, k, 64, v);
    put(blob, C2H, C2L, k, n, 64, v);
  } else if (i < f.w3) {
    bias[64 + (i - f.b2)] = v;
  } else if (i < f.b3) {  // W3 [64][33]
    const int j = static_cast<int>(i - f.w3), k = j / 33, n = j % 33;
    put(blob, B3H, B3L, n, k, 64, v);
    put(blob, C3H, C3L, k, n, 48, v);
  } else if (i < f.b3 + 33) {
    bias[128 + (i - f.b3)] = v;
  }
}

}  // namespace wpack

// whole blob from the field parameters, zero padding included (wg_train.cu)
cudaError_t launch_pack_weights(const FieldView& f, unsigned char* blob, cudaStream_t st);

}  // namespace wg
