/* Plain-C data types shared by the wostgpu C-ABI (include/wostgpu.h), the CPU
 * oracle (oracle/) and the reference shim (oracle/ref_shim.cpp).
 *
 * Every struct mirrors a reference C++ type field for field, so arrays of them
 * can be handed across the boundary with no repacking. Reference citations are
 * relative to the arXiv 2410.18944 C++ artifact (proj/...).
 */
#ifndef WOSTGPU_TYPES_H
#define WOSTGPU_TYPES_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes returned by every C-ABI entry point */
enum {
  WG_OK = 0,
  WG_ERR_INVALID = 1,   /* std::invalid_argument in the reference */
  WG_ERR_SCENE = 2,     /* wost::SceneError (proj/include/wost/scene.hpp:12) */
  WG_ERR_RUNTIME = 3,   /* std::runtime_error (IO, checkpoints) */
  WG_ERR_CUDA = 4,      /* CUDA / NCCL failure */
  WG_ERR_NOT_BUILT = 5  /* kernel for this configuration not compiled in */
};

/* BoundaryKind (proj/include/wost/scene.hpp:16) */
enum { WG_DIRICHLET = 0, WG_NEUMANN = 1 };

/* KindMask (proj/include/wost/geom2d.hpp:11-15) */
enum { WG_KIND_DIRICHLET = 1u, WG_KIND_NEUMANN = 2u, WG_KIND_ALL = 3u };

/* SamplerMode (proj/include/wost/wost.hpp:15) */
enum {
  WG_MODE_UNIFORM = 0,
  WG_MODE_GUIDING_ONLY = 1,
  WG_MODE_FIXED_MIS = 2,
  WG_MODE_LEARNABLE_MIS = 3
};

/* ValueSpec / SourceField variants (proj/include/wost/scene.hpp:31-67).
 * Analytic std::function values exist only in presets
 * (proj/src/presets.cpp:190-208); they are carried as functor ids. */
enum {
  WG_VALUE_ZERO = -1, /* SourceField::Zero */
  WG_VALUE_CONSTANT = 0,
  WG_VALUE_LINEAR = 1,
  WG_VALUE_RASTER = 2,
  WG_VALUE_ANALYTIC = 3
};
enum {
  WG_ANALYTIC_X2_MINUS_Y2 = 1, /* harmonic-disk g, presets.cpp:191-192 */
  WG_ANALYTIC_R2_MINUS_1 = 2   /* const-source-disk g, presets.cpp:202-203 */
};

typedef struct wg_value_spec {
  int32_t type;        /* WG_VALUE_* */
  int32_t analytic_id; /* WG_ANALYTIC_* when type == WG_VALUE_ANALYTIC */
  double c0, cx, cy;   /* Constant: c0; Linear: c0 + cx*x + cy*y */
  /* RasterGrid (scene.hpp:20-28): row-major, row 0 at bbox.min.y,
   * nearest-cell lookup clamped to the edge cell */
  int32_t raster_w, raster_h;
  double raster_bbox[4]; /* min.x, min.y, max.x, max.y */
  const double* raster_data;
} wg_value_spec;

/* SolverConfig (proj/include/wost/wost.hpp:20-31) */
typedef struct wg_solver_config {
  double epsilon_shell; /* 0 -> scene value */
  double r_min;         /* 0 -> epsilon */
  int32_t rr_depth;
  int32_t mode; /* WG_MODE_* */
  double fixed_c;
  int32_t reflect_at_neumann;
  int32_t clamp_grazing;
  double grazing_floor;
  int32_t max_steps;
  int32_t pad_;
} wg_solver_config;

/* PointStats (proj/include/wost/wost.hpp:127-143): Welford accumulator */
typedef struct wg_point_stats {
  double mean;
  double m2;
  int64_t count;
  int64_t escaped;
} wg_point_stats;

/* FieldConfig (proj/include/wost/guide_field.hpp:13-25) */
#define WG_MAX_LEVELS 8
typedef struct wg_field_config {
  int32_t n_levels;
  int32_t level_res[WG_MAX_LEVELS];
  int32_t features;
  int32_t hidden;
  int32_t mixture_k;
  int32_t mixture_dim;
} wg_field_config;

/* TrainConfig (proj/include/wost/guide_train.hpp:60-75) */
typedef struct wg_train_config {
  int32_t minibatch;
  int32_t learn_selection;
  int64_t max_records_per_round;
  double lr, beta1, beta2, eps;
  double e_fraction;
  int32_t reflect;
  int32_t pad_;
  double pdf_floor;
  double v_floor;
  uint64_t seed;
} wg_train_config;

/* TrainStats (proj/include/wost/guide_train.hpp:48-58) */
typedef struct wg_train_stats {
  int64_t records_seen;
  int64_t records_consumed;
  int64_t skipped_low_pdf;
  int64_t skipped_low_v;
  int64_t steps;
  double mean_grad_norm;
  double seconds;
} wg_train_stats;

/* GuideRecord (proj/include/wost/guide_train.hpp:14-25) */
typedef struct wg_guide_record {
  double x[2];
  double nu[3];
  double target;
  double pdf_mis, pdf_g, pdf_u, c;
  int32_t on_neumann;
  int32_t pad_;
  double normal[2];
} wg_guide_record;

/* MixtureParams (proj/include/wost/sphdist.hpp:29-39), K <= 16 */
#define WG_MAX_MIXTURE 16
typedef struct wg_mixture {
  double mu[WG_MAX_MIXTURE][3];
  double kappa[WG_MAX_MIXTURE];
  double lambda[WG_MAX_MIXTURE];
  double log_a[WG_MAX_MIXTURE];
  double c;
  int32_t k;
  int32_t dim;
} wg_mixture;

/* ---- 3D (no reference counterpart; SURVEY.md §8 a', configs 4-5) ------ */
/* value of a 3D triangle (Dirichlet g or Neumann flux h) or of the 3D
 * source f: Constant c0 or Linear c0 + cx x + cy y + cz z (the 3D analogue of
 * ValueSpec, scene.hpp:31-67); type WG_VALUE_ZERO marks "no source" */
typedef struct wg_value3_spec {
  int32_t type; /* WG_VALUE_CONSTANT or WG_VALUE_LINEAR */
  int32_t pad_;
  double c0, cx, cy, cz;
} wg_value3_spec;

/* GuideRecord with 3D position and normal */
typedef struct wg_guide_record3 {
  double x[3];
  double nu[3];
  double target;
  double pdf_mis, pdf_g, pdf_u, c;
  int32_t on_neumann;
  int32_t pad_;
  double normal[3];
} wg_guide_record3;

#ifdef __cplusplus
}
#endif

#endif /* WOSTGPU_TYPES_H */
