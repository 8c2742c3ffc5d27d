/* wostgpu — B200 (sm_100a) guided walk-on-stars, C-ABI boundary.
 *
 * This is the drop-in boundary for the reference's hot path
 * (arXiv 2410.18944 artifact, proj/include/wost/*.hpp). Every entry point
 * names the reference interface it replaces. Arrays are plain host pointers
 * with explicit sizes; no C++ or torch types cross the boundary. Device
 * state lives behind opaque handles. Every function returns a WG_* status
 * (include/wostgpu_types.h); the message of the last failure on the calling
 * thread is wostgpu_last_error(). Reference C++ exceptions map to codes:
 * SceneError -> WG_ERR_SCENE, std::invalid_argument -> WG_ERR_INVALID,
 * std::runtime_error -> WG_ERR_RUNTIME. The C++ facade include/wostgpu.hpp
 * rethrows them as the same exception types.
 *
 * There is no CPU fallback: every compute entry point runs CUDA kernels and
 * fails with WG_ERR_CUDA when no sm_100 device is usable.
 */
#ifndef WOSTGPU_H
#define WOSTGPU_H

#include "wostgpu_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct wg_scene_s* wg_scene;   /* Scene + Accel on one device */
typedef struct wg_field_s* wg_field;   /* GuidingField on one device */
typedef struct wg_solver_s* wg_solver; /* StepContext + SolveScratch + Engine state */

/* ---- runtime ----------------------------------------------------------- */
const char* wostgpu_last_error(void);
/* binds the calling thread to `device` (one process per GPU) */
int wostgpu_init(int device);
int wostgpu_device_info(int* sm_count, int* cc_major, int* cc_minor);
/* waits for all device work of the library and reports a pending device
 * error; handles must be destroyed by the caller before (the CUDA context
 * is shared with the host process, so it is not reset) */
int wostgpu_shutdown(void);
/* number of kernels this library launched since load (bench evidence) */
int64_t wostgpu_kernel_launches(void);

/* ---- scene + acceleration structure ------------------------------------ */
/* Scene (proj/include/wost/scene.hpp:70-96) + Accel::Accel
 * (proj/src/geom2d.cpp:80-107, proj/include/wost/geom2d.hpp:38-40).
 * seg: n_seg x {ax, ay, bx, by}; kind: WG_DIRICHLET/WG_NEUMANN;
 * value_index: index into values. source may be NULL (SourceField::Zero).
 * epsilon_shell <= 0 skips Scene::validate (the reference's in-code test
 * scenes do not validate) and uses 1e-3. Throws SceneError on an empty scene
 * (geom2d.cpp:81-82) and on validate() failures (scene.cpp:119-143). */
int wostgpu_scene_create(const double* seg, const int32_t* kind, const int32_t* value_index,
                         int32_t n_seg, const wg_value_spec* values, int32_t n_values,
                         const wg_value_spec* source, const double bbox[4],
                         double epsilon_shell, wg_scene* out);
int wostgpu_scene_destroy(wg_scene scene);
/* Accel::t_epsilon (geom2d.hpp:61), Scene::has_neumann_flux (scene.cpp:83) */
int wostgpu_scene_info(wg_scene scene, double* t_epsilon, int32_t* has_neumann_flux,
                       double root_box[4]);

/* Batched Accel queries (one CUDA thread per query):
 * Accel::closest_point      proj/src/geom2d.cpp:142-180
 * Accel::closest_silhouette proj/src/geom2d.cpp:182-200
 * Accel::ray_first_hit      proj/src/geom2d.cpp:202-246 (t = +inf, seg = -1 on miss)
 * Accel::star_radius        proj/src/geom2d.cpp:248-255 (WG_ERR_SCENE if unbounded) */
int wostgpu_closest_point(wg_scene scene, int64_t n, const double* xy, uint32_t kinds,
                          double* point, double* dist, int32_t* segment);
int wostgpu_closest_silhouette(wg_scene scene, int64_t n, const double* xy, double* dist);
int wostgpu_ray_first_hit(wg_scene scene, int64_t n, const double* origin, const double* dir,
                          const double* t_max, uint32_t kinds, const int32_t* exclude,
                          double* t, double* point, double* normal, int32_t* segment,
                          int32_t* kind);
int wostgpu_star_radius(wg_scene scene, int64_t n, const double* xy, double r_min, double* r);

/* ---- guiding field ------------------------------------------------------ */
/* GuidingField(FieldConfig, Bbox, seed): proj/src/guide_field.cpp:13-55
 * (same initialisation stream: parameters are bit-identical) */
int wostgpu_field_create(const wg_field_config* cfg, const double bbox[4], uint64_t seed,
                         wg_field* out);
int wostgpu_field_destroy(wg_field field);
int wostgpu_field_param_count(wg_field field, int64_t* n);
/* params()/set_param (guide_field.hpp:73-77) and the Adam state saved by
 * GuidingField::save (guide_field.cpp:351-372); m, v may be NULL */
int wostgpu_field_get_state(wg_field field, float* params, double* adam_m, double* adam_v,
                            int64_t* adam_steps);
int wostgpu_field_set_state(wg_field field, const float* params, const double* adam_m,
                            const double* adam_v, int64_t adam_steps);
/* get_param / set_param (guide_field.hpp:73-77) over a contiguous range */
int wostgpu_field_get_params(wg_field field, int64_t offset, int64_t count, float* out);
int wostgpu_field_set_params(wg_field field, int64_t offset, int64_t count, const float* in);
/* GuidingField::eval_with_tape + backward (guide_field.cpp:223-243,
 * 258-315) for n points: grad[n_params] += sum_i J(x_i)^T d_out[i x od], in
 * fp64 as the reference (summation order across points differs: fp64
 * atomics) */
int wostgpu_field_backward(wg_field field, int64_t n, const double* xy, const double* d_out,
                           double* grad);
/* GuidingField::adam_step (guide_field.cpp:317-331) on an fp64 gradient,
 * which is zeroed on return as in the reference */
int wostgpu_field_adam_step(wg_field field, double* grad, double lr, double beta1, double beta2,
                            double eps);
/* GuidingField::eval_batch (guide_field.cpp:178-221, 251-256): row-major
 * [n x output_dim]. mlp = WG_MLP_EXACT reproduces the reference's fp32
 * accumulation order bit for bit (CUDA cores); WG_MLP_TENSOR runs the
 * tcgen05 tensor-core kernel (fp32 operands split into fp16 hi + lo, three
 * MMAs per K-step, fp32 accumulation in TMEM: ~1e-6 relative). */
enum { WG_MLP_EXACT = 0, WG_MLP_TENSOR = 1 };
int wostgpu_field_eval_batch(wg_field field, int64_t n, const double* xy, double* out, int mlp);
/* normalize_params(unpack_params(...)) (sphdist.cpp:287-310,
 * guide_field.cpp:424-441) on device for n raw rows */
int wostgpu_normalize_params(int64_t n, const double* raw, int32_t k, int32_t dim,
                             wg_mixture* out);
/* Diagnostics of the tensor-core walk path's fp32 mixture math (default
 * shape: K = 8, dim 2; no reference counterpart, used by the parity tests):
 * mixture32_pdf decodes raw row i (33 floats) and evaluates the mixture pdf
 * at nu[i] (unit, fp64): out[2i] = pdf, out[2i+1] = selection probability c;
 * mixture32_sample draws n directions from the single mixture `raw`, sample
 * i with its own PCG32 stream (seed, i). */
/* diagnostic: bytes in which the field's Adam-maintained split-fp16 weight
 * blob (tensor-core kernels) differs from a fresh pack of its parameters;
 * -1 when no maintained blob exists yet */
int wostgpu_field_check_pack(wg_field field, int64_t* mismatched_bytes);
int wostgpu_mixture32_pdf(int64_t n, const float* raw, const double* nu, double* out);
int wostgpu_mixture32_sample(const float* raw, int64_t n, uint64_t seed, double* nu_out);

/* ---- solver (solve_batch / Engine) --------------------------------------- */
/* StepContext{scene, accel, field, cfg} (proj/include/wost/wost.hpp:33-51)
 * plus the device walk queues and record arena. field may be NULL in
 * uniform mode. */
int wostgpu_solver_create(wg_scene scene, wg_field field, const wg_solver_config* cfg,
                          wg_solver* out);
int wostgpu_solver_destroy(wg_solver solver);
/* selects the MLP path used inside guided walks (default WG_MLP_TENSOR when
 * the field shape is the default 16->64->64->33, else WG_MLP_EXACT) */
int wostgpu_solver_set_mlp(wg_solver solver, int mlp);
/* Evaluation points, kept resident in HBM. global_offset is the global index
 * of points[0]: walk streams are Rng::for_walk(seed, global index, wpp)
 * (proj/include/wost/rng.hpp:28-32), so sharding points over ranks leaves
 * every walk's random stream unchanged. Resets the per-point statistics. */
int wostgpu_solver_set_points(wg_solver solver, int64_t n, const double* xy,
                              int64_t global_offset);
int wostgpu_solver_get_stats(wg_solver solver, wg_point_stats* stats);
int wostgpu_solver_set_stats(wg_solver solver, const wg_point_stats* stats);

/* solve_batch for n_rounds consecutive wpp indices [wpp_first, wpp_first +
 * n_rounds) (proj/src/wost.cpp:290-384): one walk per point per round,
 * Welford statistics pushed in wpp order exactly as n_rounds sequential
 * solve_batch calls would. collect_records != 0 (n_rounds must be 1) keeps
 * the round's GuideRecords on device (backfill_targets_append,
 * guide_train.cpp:58-79) for wostgpu_train_round / wostgpu_fetch_records. */
int wostgpu_solve_rounds(wg_solver solver, uint64_t seed, uint64_t wpp_first, int32_t n_rounds,
                         int32_t collect_records);
/* drop-in solve_batch(ctx, points, stats, seed, wpp_index, collect, records)
 * with host arrays: stats are read, updated in place and written back */
int wostgpu_solve_batch(wg_solver solver, int64_t n, const double* xy, wg_point_stats* stats,
                        uint64_t seed, uint64_t wpp_index, int32_t collect_records);
/* the records of the last collecting round (point order is not preserved) */
int wostgpu_fetch_records(wg_solver solver, wg_guide_record* out, int64_t capacity,
                          int64_t* n);
/* per-walk results of the last round (estimate, escaped flag, steps) for
 * wost_walk parity (proj/src/wost.cpp:274-288) */
int wostgpu_fetch_walks(wg_solver solver, double* estimate, int32_t* escaped, int32_t* steps);
/* device-side counters of the last solve call: walks, steps, escaped */
int wostgpu_solver_counters(wg_solver solver, int64_t* walks, int64_t* steps, int64_t* escaped,
                            int64_t* records);

/* train_batch on the records of the last collecting round
 * (proj/src/guide_train.cpp:94-198): filter pdf_mis < floor, random subset
 * of at most max_records_per_round, minibatch Adam. With a communicator
 * attached the round is the single-GPU round over the union of the ranks'
 * records: the usable count is allreduced before the selection (so the cap
 * and the minibatch size are GLOBAL, guide_train.cpp:111-116,128) and the
 * gradient sums before every Adam step; every rank takes the same step. */
int wostgpu_train_round(wg_solver solver, const wg_train_config* cfg, uint64_t round,
                        wg_train_stats* stats);
/* drop-in train_batch(field, records, cfg, round) with host records
 * (proj/src/guide_train.cpp:94-198, declared proj/include/wost/guide_train.hpp:104-105):
 * the reference's own selection (Fisher-Yates order from the round's PCG32
 * stream, cap, consecutive minibatches), so seen / consumed / skipped / steps
 * equal the reference's on the same records; gradients on the device */
int wostgpu_train_batch(wg_solver solver, const wg_guide_record* records, int64_t n,
                        const wg_train_config* cfg, uint64_t round, wg_train_stats* stats);
/* mean gradient of one minibatch made of `records` in order, fp64 out
 * (the inner loop of train_batch, guide_train.cpp:146-171) */
int wostgpu_field_grad(wg_solver solver, const wg_guide_record* records, int64_t n,
                       const wg_train_config* cfg, double* grad);

/* Split-phase training round for callers that reduce across ranks with
 * their own collectives (MPI, gloo, ...). Steps and semantics are those of
 * wostgpu_train_round's device pipeline with the two NCCL allreduces
 * replaced by the caller's sums:
 *   train_prepare        targets, validity; this rank's usable record count
 *                        (records with pdf_mis >= cfg->pdf_floor)
 *   train_select         the training set from the GLOBAL usable count (sum
 *                        over ranks); *n_minibatches = ceil(cap / minibatch)
 *   train_minibatch_grad this rank's gradient sum of minibatch b:
 *                        grad_sum[n_params + 1], each record pre-scaled by
 *                        1 / cfg->minibatch, grad_sum[n_params] = record count
 *   train_apply          one Adam step (guide_field.cpp:317-331) on the
 *                        summed buffer: mean = sum * minibatch / count; no step
 *                        when the count is 0 */
int wostgpu_train_prepare(wg_solver solver, const wg_train_config* cfg, int64_t* usable_local);
int wostgpu_train_select(wg_solver solver, const wg_train_config* cfg, int64_t usable_global,
                         int32_t* n_minibatches);
int wostgpu_train_minibatch_grad(wg_solver solver, const wg_train_config* cfg, int32_t b,
                                 float* grad_sum);
int wostgpu_train_apply(wg_solver solver, const wg_train_config* cfg, const float* grad_sum);

/* The Engine loop (proj/src/solver.cpp:92-104, 136-146) natively: for b in
 * [0, wpp): solve round b over the solver's points (collecting records while
 * training_active(b, train_until), guide_train.cpp:200-202) and then
 * train_round(b). Rounds after training stops are independent and run as
 * one multi-round launch. device_ms is the CUDA-event time of the whole loop
 * on the solver's stream; stats accumulate on device (fetch with
 * wostgpu_solver_get_stats). totals receives the merged TrainStats. */
int wostgpu_run(wg_solver solver, uint64_t seed, int32_t wpp, int64_t train_until,
                const wg_train_config* train_cfg, wg_train_stats* totals, double* device_ms);
/* accumulated over the last wostgpu_run: walk-kernel ms, training ms, walks,
 * walk steps, escaped walks, training-round walk steps */
int wostgpu_run_profile(wg_solver solver, double* walk_ms, double* train_ms, int64_t* walks,
                        int64_t* steps, int64_t* escaped, int64_t* train_steps);

/* ---- multi-GPU ------------------------------------------------------------ */
/* NCCL communicator for gradient allreduce (one rank per GPU). Rank 0 calls
 * wostgpu_comm_unique_id and broadcasts the 128 bytes out of band. */
int wostgpu_comm_unique_id(char id[128]);
/* Record arena capacity (records per collecting round) of the following
 * calls, at least n. A training round whose records overflow the arena
 * fails its call with WG_ERR_RUNTIME (and doubles the arena) instead of
 * training on a short-walk-biased subset; the default holds 256 records per
 * point. */
int wostgpu_solver_reserve_records(wg_solver solver, int64_t n);
int wostgpu_solver_attach_comm(wg_solver solver, const char id[128], int32_t nranks,
                               int32_t rank);

/* ---- timing ---------------------------------------------------------------- */
/* device time (ms) of the walk kernel(s) and training kernels of the last
 * solve / train call, from CUDA events on the solver's stream */
int wostgpu_solver_timing(wg_solver solver, double* walk_ms, double* train_ms);

#ifdef __cplusplus
}
#endif

#endif /* WOSTGPU_H */
