/* wostgpu3 — the 3D walk-on-stars path (SURVEY.md §8 a′, configs 4-5),
 * C-ABI boundary.
 *
 * The reference has no 3D code (proj/src/wost.cpp hardcodes dim 2 at :75-76,
 * :99, :108; GuidingField takes Vec2 positions), so these entry points are
 * the 3D analogues of the 2D ones in include/wostgpu.h, with the same
 * conventions: plain pointers and sizes, WG_* status codes,
 * wostgpu_last_error() for the message, no CPU fallback. The contract the
 * GPU path is tested against is the CPU restatement oracle/wost3d.inc
 * ("parity unpinned" for geometry and walks: there is no reference output;
 * the d = 3 vMF formulas it uses are pinned against the reference).
 *
 * Scenes are triangle meshes: tri = n x {a.xyz, b.xyz, c.xyz} (fp64), kind
 * WG_DIRICHLET / WG_NEUMANN, value_index into wg_value3_spec values
 * (Dirichlet g / Neumann flux h, constant or linear), an optional source f
 * (constant or linear, 0 outside the scene bbox; NULL or WG_VALUE_ZERO: none).
 */
#ifndef WOSTGPU3_H
#define WOSTGPU3_H

#include "wostgpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct wg_scene3_s* wg_scene3;
typedef struct wg_solver3_s* wg_solver3;

/* ---- scene ---------------------------------------------------------------
 * Accel::Accel analogue (proj/src/geom2d.cpp:80-140): per-kind triangle BVHs
 * and the silhouette-edge index of the Neumann set. epsilon_shell <= 0 skips
 * the bbox containment check and uses 1e-3. WG_ERR_SCENE on an empty scene,
 * degenerate triangles, undefined values. */
int wostgpu_scene3_create(const double* tri, const int32_t* kind, const int32_t* value_index,
                          int32_t n_tri, const wg_value3_spec* values, int32_t n_values,
                          const wg_value3_spec* source, const double bbox[6], double epsilon_shell,
                          wg_scene3* out);
int wostgpu_scene3_destroy(wg_scene3 scene);
/* t_epsilon (1e-6 x root-box diagonal, geom2d.hpp:61 analogue), BVH node
 * counts (Dirichlet, Neumann, edges) and silhouette-edge counts (always /
 * crease) */
int wostgpu_scene3_info(wg_scene3 scene, double* t_epsilon, int64_t n_nodes[3],
                        int64_t* n_sil_always, int64_t* n_sil_crease);

/* batched queries, one CUDA thread per query (analogues of
 * geom2d.cpp:142-255; selection is order-independent: minimum of
 * (distance^2, triangle id) / (t, triangle id)) */
int wostgpu_closest_point3(wg_scene3 scene, int64_t n, const double* xyz, uint32_t kinds,
                           double* point, double* dist, int32_t* tri);
int wostgpu_closest_silhouette3(wg_scene3 scene, int64_t n, const double* xyz, double* dist);
int wostgpu_ray_first_hit3(wg_scene3 scene, int64_t n, const double* origin, const double* dir,
                           const double* t_max, uint32_t kinds, const int32_t* exclude, double* t,
                           double* point, double* normal, int32_t* tri, int32_t* kind);
int wostgpu_star_radius3(wg_scene3 scene, int64_t n, const double* xyz, double r_min, double* r);

/* ---- field -----------------------------------------------------------------
 * 3D guiding field: levels of dense res^3 x F grids (trilinear), the 2D
 * field's MLP, output (2 + 3) K + 1 (cfg->mixture_dim must be 3). Same
 * initialisation stream as GuidingField (guide_field.cpp:36-51) over the 3D
 * layout. The handle is a wg_field: wostgpu_field_param_count / get_state /
 * set_state / destroy apply; the 2D-only calls reject it. */
int wostgpu_field3_create(const wg_field_config* cfg, const double bbox[6], uint64_t seed,
                          wg_field* out);
/* mlp = WG_MLP_EXACT: fp32 CUDA cores in the oracle's operation order (bit
 * for bit); WG_MLP_TENSOR: tcgen05 split-fp16 MMAs (~1e-6 relative) */
int wostgpu_field3_eval_batch(wg_field field, int64_t n, const double* xyz, double* out, int mlp);
/* diagnostic (the tensor-core 3D direction kernel's fp32 mixture math): decode
 * raw row i (41 floats, K = 8) and evaluate the d = 3 mixture pdf at the unit
 * direction nu[i] (normalize_params + mixture_pdf, sphdist.cpp:176-185,
 * 287-310); out[2i] = pdf, out[2i+1] = c */
int wostgpu_mixture3f_pdf(int64_t n, const float* raw, const double* nu, double* out);

/* ---- solver ------------------------------------------------------------------
 * solve_batch / Engine analogues over 3D points (include/wostgpu.h for the
 * 2D versions; same semantics, xyz instead of xy) */
int wostgpu_solver3_create(wg_scene3 scene, wg_field field, const wg_solver_config* cfg,
                           wg_solver3* out);
int wostgpu_solver3_destroy(wg_solver3 solver);
/* MLP path inside guided walks: WG_MLP_TENSOR (default; lockstep 128-walk
 * CTAs with the tcgen05 MLP) or WG_MLP_EXACT (per-thread fp32 MLP in the
 * oracle's operation order: per-walk parity with oracle/wost3d.inc) */
int wostgpu_solver3_set_mlp(wg_solver3 solver, int mlp);
int wostgpu_solver3_set_points(wg_solver3 solver, int64_t n, const double* xyz,
                               int64_t global_offset);
int wostgpu_solver3_get_stats(wg_solver3 solver, wg_point_stats* stats);
int wostgpu_solver3_solve_rounds(wg_solver3 solver, uint64_t seed, uint64_t wpp_first,
                                 int32_t n_rounds, int32_t collect_records);
int wostgpu_solver3_fetch_walks(wg_solver3 solver, double* estimate, int32_t* escaped,
                                int32_t* steps);
int wostgpu_solver3_fetch_records(wg_solver3 solver, wg_guide_record3* out, int64_t capacity,
                                  int64_t* n);
int wostgpu_solver3_counters(wg_solver3 solver, int64_t* walks, int64_t* steps, int64_t* escaped,
                             int64_t* records);
/* train_batch on the last collecting round's records (guide_train.cpp:94-198) */
int wostgpu_solver3_train_round(wg_solver3 solver, const wg_train_config* cfg, uint64_t round,
                                wg_train_stats* stats);
/* mean gradient of one minibatch made of `records` in order (fp64 out) */
int wostgpu_solver3_field_grad(wg_solver3 solver, const wg_guide_record3* records, int64_t n,
                               const wg_train_config* cfg, double* grad);
/* the Engine loop (solver.cpp:92-104): wpp rounds, training while
 * round < train_until, device time of the whole loop in device_ms */
int wostgpu_solver3_run(wg_solver3 solver, uint64_t seed, int32_t wpp, int64_t train_until,
                        const wg_train_config* train_cfg, wg_train_stats* totals,
                        double* device_ms);
int wostgpu_solver3_run_profile(wg_solver3 solver, double* walk_ms, double* train_ms,
                                int64_t* walks, int64_t* steps, int64_t* escaped,
                                int64_t* train_steps);
/* as wostgpu_solver_reserve_records (default: 48 records per point) */
int wostgpu_solver3_reserve_records(wg_solver3 solver, int64_t n);
int wostgpu_solver3_attach_comm(wg_solver3 solver, const char id[128], int32_t nranks,
                                int32_t rank);

#ifdef __cplusplus
}
#endif

#endif /* WOSTGPU3_H */
