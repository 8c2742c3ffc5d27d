// Host-side handles of the 3D path (include/wostgpu3.h): scene (triangle
// BVHs + silhouette-edge index on device) and solver (walk queues, record
// arena, training buffers). The 3D field reuses wg_field_s (wg_runtime.hpp)
// with sdim = 3.
#pragma once

#include "../../include/wostgpu3.h"
#include "wg3_field.cuh"
#include "wg3_geom.cuh"
#include "wg_runtime.hpp"

struct wg_scene3_s {
  int device = 0;
  double bbox[6];
  double eps = 0, t_eps = 0, diag = 0;
  int64_t n_tri = 0, n_always = 0, n_crease = 0;
  int64_t n_node[3] = {0, 0, 0};
  wgrt::DBuf node[3], tri[2], edge, values, tbox, node4k[3];
  wg3::Scene3View view{};
};

struct wg_solver3_s {
  wg_scene3 scene = nullptr;
  wg_field field = nullptr;
  wg_solver_config cfg{};
  int mlp = WG_MLP_EXACT;
  cudaStream_t st = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t n_points = 0, point_offset = 0;
  wgrt::DBuf points, stats, est, esc, steps, counters;
  int32_t last_rounds = 0;
  // records of the last collecting round (wg3::DevRecord3 in a wg::DevRecord arena)
  wgrt::DBuf recs, rec_counter, rec_tail, rec_term, rec_dacc;
  int64_t rec_cap = 0;
  int64_t rec_cap_min = 0;  // grown after an arena overflow
  bool have_records = false;
  // wavefront walk pool (WG_MLP_TENSOR guided walks, wg3_walk_tc.cu)
  wgrt::DBuf w_lanes, w_dirs, w_rec, w_state, w_queue, w_qlen, w_next, w_blob, w_perm, w_bins, w_sbin, g_blob;
  int64_t w_slots = 0;
  // first-step geometry per start point (StartGeo3), valid for the current points
  wgrt::DBuf start_geo;
  bool start_ok = false;
  unsigned int* h_qlen = nullptr;  // pinned
  // training
  wgrt::DBuf grad, lists, ctl, totals;
  int64_t list_cap = 0;
  // NCCL
  ncclComm_t comm = nullptr;
  int32_t nranks = 1, rank = 0;
  // timing / profile
  float last_walk_ms = 0.0f, last_train_ms = 0.0f;
  double prof_walk_ms = 0, prof_train_ms = 0;
  int64_t prof_walks = 0, prof_steps = 0, prof_escaped = 0, prof_train_steps = 0;
  ~wg_solver3_s();
};
