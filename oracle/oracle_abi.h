/* TEST INFRASTRUCTURE ONLY — never linked or called by the product path.
 *
 * One C-ABI shape, two implementations:
 *   ref_*  oracle/ref_shim.cpp   : thin extern "C" wrappers around the real
 *                                  reference library compiled from
 *                                  /root/reference/proj/src (oracle/_ref/)
 *   orc_*  oracle/wost_oracle.cpp: an independent CPU restatement of the
 *                                  reference algorithm (the checker the GPU
 *                                  parity tests use)
 * Tests call both through ctypes with identical arguments; the restatement is
 * pinned against the reference (tests/test_oracle_vs_ref.py) and against the
 * committed golden vectors (tests/golden/).
 */
#ifndef WOST_ORACLE_ABI_H
#define WOST_ORACLE_ABI_H

#include "../include/wostgpu_types.h"

#ifdef __cplusplus
extern "C" {
#endif

#define WG_ORACLE_DECLS(P)                                                     \
  const char* P##_last_error(void);                                            \
  /* scenes */                                                                 \
  void* P##_scene_create(const double* seg, const int32_t* kind,               \
                         const int32_t* value_index, int32_t n_seg,            \
                         const wg_value_spec* values, int32_t n_values,        \
                         const wg_value_spec* source, const double* bbox,      \
                         double epsilon_shell);                                \
  void P##_scene_destroy(void* scene);                                         \
  double P##_t_epsilon(void* scene);                                           \
  int32_t P##_has_neumann_flux(void* scene);                                   \
  /* geometry, proj/src/geom2d.cpp */                                          \
  int P##_closest_point(void* scene, int64_t n, const double* xy,              \
                        uint32_t kinds, double* pt, double* dist,              \
                        int32_t* seg);                                         \
  int P##_closest_silhouette(void* scene, int64_t n, const double* xy,         \
                             double* dist);                                    \
  int P##_ray_first_hit(void* scene, int64_t n, const double* origin,          \
                        const double* dir, const double* t_max,                \
                        uint32_t kinds, const int32_t* exclude, double* t,     \
                        double* pt, double* normal, int32_t* seg,              \
                        int32_t* kind);                                        \
  int P##_star_radius(void* scene, int64_t n, const double* xy, double r_min,  \
                      double* r);                                              \
  /* directional distributions, proj/src/sphdist.cpp */                        \
  double P##_bessel_i0(double x);                                              \
  double P##_log_bessel_i0(double x);                                          \
  double P##_bessel_i1_over_i0(double x);                                      \
  void P##_normalize_params(int64_t n, const double* raw, int32_t k,           \
                            int32_t dim, wg_mixture* out);                     \
  double P##_mixture_pdf(const wg_mixture* m, const double* nu);               \
  double P##_mis_pdf(const wg_mixture* m, const double* nu,                    \
                     const double* normal, int32_t reflect);                   \
  /* guiding field, proj/src/guide_field.cpp */                                \
  void* P##_field_create(const wg_field_config* cfg, const double* bbox,       \
                         uint64_t seed);                                       \
  void P##_field_destroy(void* field);                                         \
  int64_t P##_field_param_count(void* field);                                  \
  void P##_field_get_params(void* field, float* out);                          \
  void P##_field_set_params(void* field, const float* in);                     \
  void P##_field_eval_batch(void* field, int64_t n, const double* xy,          \
                            double* out);                                      \
  /* walks, proj/src/wost.cpp */                                               \
  int P##_walks(void* scene, void* field, const wg_solver_config* cfg,         \
                int64_t n, const double* xy, const int64_t* point_index,       \
                uint64_t seed, uint64_t wpp_index, double* estimate,           \
                int32_t* escaped, int32_t* n_records);                         \
  int P##_solve_batch(void* scene, void* field, const wg_solver_config* cfg,   \
                      int64_t n, const double* xy, wg_point_stats* stats,      \
                      uint64_t seed, uint64_t wpp_index, int32_t collect,      \
                      wg_guide_record** records, int64_t* n_records);          \
  void P##_free(void* p);                                                      \
  /* training, proj/src/guide_train.cpp */                                     \
  int P##_train_batch(void* field, const wg_guide_record* recs, int64_t n,     \
                      const wg_train_config* cfg, uint64_t round,              \
                      wg_train_stats* stats);                                  \
  int P##_field_grad(void* field, const wg_guide_record* recs, int64_t n,      \
                     const wg_train_config* cfg, double* grad_out);

WG_ORACLE_DECLS(ref)
WG_ORACLE_DECLS(orc)

/* 3D contract (oracle/wost3d.inc): restatement only, no reference code */
void* orc3_scene_create(const double* tri, const int32_t* kind, const int32_t* value_index,
                        int32_t n_tri, const wg_value3_spec* values, int32_t n_values,
                        const wg_value3_spec* source, const double* bbox, double epsilon_shell);
void orc3_scene_destroy(void* scene);
double orc3_t_epsilon(void* scene);
void orc3_silhouette_info(void* scene, int64_t* n_always, int64_t* n_crease);
int orc3_closest_point(void* scene, int64_t n, const double* xyz, uint32_t kinds, double* pt,
                       double* dist, int32_t* tri);
int orc3_closest_silhouette(void* scene, int64_t n, const double* xyz, double* dist);
int orc3_ray_first_hit(void* scene, int64_t n, const double* origin, const double* dir,
                       const double* t_max, uint32_t kinds, const int32_t* exclude, double* t,
                       double* pt, double* normal, int32_t* tri, int32_t* kind);
int orc3_star_radius(void* scene, int64_t n, const double* xyz, double r_min, double* r);
void* orc3_field_create(const wg_field_config* cfg, const double* bbox, uint64_t seed);
void orc3_field_destroy(void* field);
int64_t orc3_field_param_count(void* field);
void orc3_field_get_params(void* field, float* out);
void orc3_field_set_params(void* field, const float* in);
void orc3_field_eval_batch(void* field, int64_t n, const double* xyz, double* out);
int orc3_walks(void* scene, void* field, const wg_solver_config* cfg, int64_t n, const double* xyz,
               const int64_t* point_index, uint64_t seed, uint64_t wpp_index, double* estimate,
               int32_t* escaped, int32_t* steps);
int orc3_walk_records(void* scene, void* field, const wg_solver_config* cfg, int64_t n,
                      const double* xyz, const int64_t* point_index, uint64_t seed,
                      uint64_t wpp_index, wg_guide_record3** records, int64_t* n_records);
int orc3_field_grad(void* field, const wg_guide_record3* recs, int64_t n,
                    const wg_train_config* cfg, double* grad_out);
int orc3_train_batch(void* field, const wg_guide_record3* recs, int64_t n,
                     const wg_train_config* cfg, uint64_t round, wg_train_stats* stats);
int orc3_run(void* scene, void* field, const wg_solver_config* cfg, int64_t n, const double* xyz,
             int64_t point_offset, uint64_t seed, int32_t wpp, int64_t train_until,
             const wg_train_config* train_cfg, wg_point_stats* stats);

#ifdef __cplusplus
}
#endif

#endif
