// Host runtime internals shared by wg_runtime.cu (scene, queries, field) and
// wg_solver.cu (walk rounds, training, Engine loop): status/exception
// plumbing behind the C-ABI, an owning device buffer, and the scene / field
// handle structs.
#pragma once

#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/wostgpu.h"
#include "wg3_field.cuh"
#include "wg_kernels.cuh"
#include "wg_train.cuh"

namespace wgrt {

using namespace wg;

inline thread_local std::string g_err;
inline std::atomic<int64_t> g_launches{0};

struct WgError : std::runtime_error {
  int code;
  WgError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(expr)                                                                                 \
  do {                                                                                           \
    cudaError_t e_ = (expr);                                                                     \
    if (e_ != cudaSuccess)                                                                       \
      throw ::wgrt::WgError(WG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));    \
  } while (0)
#define CKL(expr)              \
  do {                         \
    CK(expr);                  \
    ::wgrt::g_launches += 1;   \
  } while (0)
// NCCL is resolved at run time (dlopen) instead of linked: the process may
// already hold torch's bundled libnccl.so.2, and linking the system copy would
// shadow it. Only the five entry points below are used.
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};
const NcclApi& nccl();  // wg_core.cu

#define NCK(expr)                                                                    \
  do {                                                                               \
    ncclResult_t r_ = (expr);                                                        \
    if (r_ != ncclSuccess)                                                           \
      throw ::wgrt::WgError(WG_ERR_CUDA,                                             \
                            std::string(#expr) + ": " + ::wgrt::nccl().getErrorString(r_)); \
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

inline void need(bool ok, int code, const std::string& msg) {
  if (!ok) throw WgError(code, msg);
}

// owning device buffer (grows, never shrinks)
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

inline void check_device() {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  need(prop.major == 10, WG_ERR_CUDA,
       "wostgpu needs an sm_100 (B200) device; found sm_" + std::to_string(prop.major) +
           std::to_string(prop.minor));
}

inline int sm_count() {
  int dev = 0, n = 148;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

inline bool default_shape(const FieldView& v) {
  return v.levels == 4 && v.F == 4 && v.in == 16 && v.hid == 64 && v.od == 33 && v.k == 8 &&
         v.dim == 2;
}

}  // namespace wgrt

// ================================================================ handles
struct wg_scene_s {
  int device = 0;
  double bbox[4];
  double eps = 0, t_eps = 0, diag = 0;
  int32_t has_flux = 0, source_zero = 1;
  std::vector<wg::Node> h_nodes;
  std::vector<wg::Seg> h_segs;
  std::vector<wg::SilVertex> h_sil;
  std::vector<double> h_sil_n;
  std::vector<wg::Node> h_sil_nodes;  // point BVH over the silhouette candidates (> 32)
  wgrt::DBuf nodes, segs, sil, sil_n, seg_kind, seg_value, values, sil_nodes;
  std::vector<std::unique_ptr<wgrt::DBuf>> rasters;
  wg::DevValue source{};
  wg::SceneView view{};
  int smem_bytes = 0;  // bytes to stage nodes+segs+silhouettes, 0 if too big
};

struct wg_field_s {
  wg_field_config cfg{};
  double bbox[4];
  int64_t n_params = 0;
  wgrt::DBuf p, m, v;
  wgrt::DBuf adam;  // wg::AdamCtl: step count + per-step control, device truth
  wg::FieldView view{};
  // packed split-fp16 MLP weights (wg_wpack.cuh) for the tensor-core kernels;
  // dirty after any host write of the parameters, kept current by Adam
  wgrt::DBuf wpack;
  bool pack_dirty = true;
  // spatial dimension: 2 (GuidingField) or 3 (wostgpu_field3_create; view3
  // and bbox3 describe it, view is unused)
  int sdim = 2;
  wg3::Field3View view3{};
  double bbox3[6] = {0, 0, 0, 0, 0, 0};
};
