// wostgpu C++ facade: the reference's wost:: solver / scene / estimator API
// (arXiv 2410.18944 artifact, proj/include/wost/*.hpp) on top of the C-ABI in
// wostgpu.h. Header-only; link with -lwostgpu (paper_2410_18944_b200/).
//
// Type and function names, argument meaning and exceptions follow the
// reference so a caller such as Engine::run_batch (proj/src/solver.cpp:92-104)
// switches by changing the namespace:
//   wost::Accel          -> wostgpu::Accel          (geom2d.hpp:38)
//   wost::GuidingField   -> wostgpu::GuidingField   (guide_field.hpp:37)
//   wost::solve_batch    -> wostgpu::solve_batch    (wost.hpp:160)
//   wost::train_batch    -> wostgpu::train_batch    (guide_train.hpp:104)
// Status codes are rethrown as the reference's exception types: SceneError,
// std::invalid_argument, std::runtime_error.
#pragma once

#include <cstdint>
#include <cstring>
#include <istream>
#include <ostream>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>
#include <algorithm>

#include "wostgpu.h"

namespace wostgpu {

struct SceneError : std::runtime_error {  // wost::SceneError (scene.hpp:12)
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == WG_OK) return;
  std::string msg = wostgpu_last_error();
  if (rc == WG_ERR_SCENE) throw SceneError(msg);
  if (rc == WG_ERR_INVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// wostgpu_shutdown: waits for the library's device work (call after the
// last handle is destroyed)
inline void shutdown() { check(wostgpu_shutdown()); }

struct Vec2 {
  double x = 0.0, y = 0.0;
};
struct Bbox {
  Vec2 min, max;
};

enum class BoundaryKind { Dirichlet = WG_DIRICHLET, Neumann = WG_NEUMANN };
enum KindMask : unsigned { kDirichletMask = 1u, kNeumannMask = 2u, kAllKinds = 3u };
enum class SamplerMode {
  Uniform = WG_MODE_UNIFORM,
  GuidingOnly = WG_MODE_GUIDING_ONLY,
  FixedMis = WG_MODE_FIXED_MIS,
  LearnableMis = WG_MODE_LEARNABLE_MIS
};

// Scene description in the reference's shape (scene.hpp:17-96): named
// values (Constant / Linear / Raster / Analytic), a source field, segments
// that refer to values by name, validate() resolving value_index.
//
// Analytic values are std::function in the reference; a device cannot call
// host code, so here they name one of the device's built-in analytic
// functions (the preset ones, wostgpu_types.h): WG_ANALYTIC_X2_MINUS_Y2
// (x^2 - y^2, harmonic-disk g, presets.cpp:191-192) and
// WG_ANALYTIC_R2_MINUS_1 (|x|^2 - 1, const-source-disk g, presets.cpp:202-203).
// An Analytic value with id 0 (an arbitrary host function) is rejected with
// std::invalid_argument when the scene is uploaded.
struct RasterGrid {  // scene.hpp:20-28
  int width = 0, height = 0;
  Bbox bbox;
  std::vector<double> data;  // row-major, row 0 at bbox.min.y
  double at(Vec2 p) const {  // scene.cpp:13-20, nearest cell, clamped
    double u = (p.x - bbox.min.x) / (bbox.max.x - bbox.min.x);
    double v = (p.y - bbox.min.y) / (bbox.max.y - bbox.min.y);
    int i = std::clamp(static_cast<int>(u * width), 0, width - 1);
    int j = std::clamp(static_cast<int>(v * height), 0, height - 1);
    return data[static_cast<size_t>(j) * width + i];
  }
};

struct ValueSpec {  // scene.hpp:31-54
  struct Constant {
    double v;
  };
  struct Linear {
    double c0, cx, cy;
  };
  struct Raster {
    RasterGrid grid;
  };
  struct Analytic {
    int id = 0;  // WG_ANALYTIC_*
    std::string name;
  };
  std::variant<Constant, Linear, Raster, Analytic> spec = Constant{0.0};
  bool is_analytic() const { return std::holds_alternative<Analytic>(spec); }
  double eval(Vec2 p) const {  // scene.cpp:22-37
    if (auto* c = std::get_if<Constant>(&spec)) return c->v;
    if (auto* l = std::get_if<Linear>(&spec)) return l->c0 + l->cx * p.x + l->cy * p.y;
    if (auto* r = std::get_if<Raster>(&spec)) return r->grid.at(p);
    const int id = std::get<Analytic>(spec).id;
    if (id == WG_ANALYTIC_X2_MINUS_Y2) return p.x * p.x - p.y * p.y;
    if (id == WG_ANALYTIC_R2_MINUS_1) return p.x * p.x + p.y * p.y - 1.0;
    throw std::invalid_argument("analytic value without a device function id");
  }
  // the C-ABI spec; raster data is borrowed from this object
  wg_value_spec c() const {
    wg_value_spec o{};
    o.type = WG_VALUE_CONSTANT;
    if (auto* c = std::get_if<Constant>(&spec)) {
      o.c0 = c->v;
    } else if (auto* l = std::get_if<Linear>(&spec)) {
      o.type = WG_VALUE_LINEAR;
      o.c0 = l->c0;
      o.cx = l->cx;
      o.cy = l->cy;
    } else if (auto* r = std::get_if<Raster>(&spec)) {
      o.type = WG_VALUE_RASTER;
      raster_c(r->grid, o);
    } else {
      const Analytic& a = std::get<Analytic>(spec);
      if (a.id != WG_ANALYTIC_X2_MINUS_Y2 && a.id != WG_ANALYTIC_R2_MINUS_1)
        throw std::invalid_argument("value '" + a.name + "': analytic values need a device function id");
      o.type = WG_VALUE_ANALYTIC;
      o.analytic_id = a.id;
    }
    return o;
  }
  static void raster_c(const RasterGrid& g, wg_value_spec& o) {
    o.raster_w = g.width;
    o.raster_h = g.height;
    o.raster_bbox[0] = g.bbox.min.x;
    o.raster_bbox[1] = g.bbox.min.y;
    o.raster_bbox[2] = g.bbox.max.x;
    o.raster_bbox[3] = g.bbox.max.y;
    o.raster_data = g.data.data();
  }
};

struct SourceField {  // scene.hpp:56-67
  struct Zero {};
  struct Constant {
    double v;
  };
  struct Raster {
    RasterGrid grid;
  };
  std::variant<Zero, Constant, Raster> spec;
  bool is_zero() const { return std::holds_alternative<Zero>(spec); }
  wg_value_spec c() const {
    wg_value_spec o{};
    o.type = WG_VALUE_ZERO;
    if (auto* c = std::get_if<Constant>(&spec)) {
      o.type = WG_VALUE_CONSTANT;
      o.c0 = c->v;
    } else if (auto* r = std::get_if<Raster>(&spec)) {
      o.type = WG_VALUE_RASTER;
      ValueSpec::raster_c(r->grid, o);
    }
    return o;
  }
};

struct BoundarySegment {  // scene.hpp:69-74
  Vec2 a, b;
  BoundaryKind kind = BoundaryKind::Dirichlet;
  std::string value_ref;
  int value_index = -1;  // resolved by Scene::validate
};

struct Scene {  // scene.hpp:76-96
  Bbox bbox;
  double epsilon_shell = 0.0;
  std::vector<std::pair<std::string, ValueSpec>> values;
  SourceField source;
  std::vector<BoundarySegment> segments;

  int find_value(const std::string& name) const {
    for (size_t i = 0; i < values.size(); ++i)
      if (values[i].first == name) return static_cast<int>(i);
    return -1;
  }
  bool has_dirichlet() const {
    for (const auto& g : segments)
      if (g.kind == BoundaryKind::Dirichlet) return true;
    return false;
  }
  // Scene::validate (scene.cpp:119-143): value references resolved here; the
  // geometric and raster invariants are checked again by the device upload
  // (wostgpu_scene_create) with the reference's messages
  void validate() {
    if (!(bbox.min.x < bbox.max.x && bbox.min.y < bbox.max.y)) throw SceneError("scene bbox is empty");
    if (epsilon_shell <= 0.0)
      throw SceneError("epsilon_shell must be > 0 (got " + std::to_string(epsilon_shell) + ")");
    if (segments.empty()) throw SceneError("scene has no boundary segments");
    for (size_t i = 0; i < segments.size(); ++i) {
      BoundarySegment& g = segments[i];
      g.value_index = find_value(g.value_ref);
      if (g.value_index < 0)
        throw SceneError("segment " + std::to_string(i) + ": value '" + g.value_ref + "' is not defined");
    }
  }
};

struct ClosestPoint {  // geom2d.hpp:30-34
  Vec2 point;
  double dist = 0.0;
  int segment = -1;
};
struct HitInfo {  // geom2d.hpp:22-28
  double t = 0.0;
  Vec2 point, normal;
  int segment = -1;
  BoundaryKind kind = BoundaryKind::Dirichlet;
};

using PointStats = wg_point_stats;   // wost.hpp:127-143 (same layout)
using GuideRecord = wg_guide_record; // guide_train.hpp:14-25 (same fields)
using TrainStats = wg_train_stats;
using TrainConfig = wg_train_config;

inline TrainConfig default_train_config() {  // guide_train.hpp:60-75
  TrainConfig t{};
  t.minibatch = 1 << 14;
  t.learn_selection = 1;
  t.max_records_per_round = 1 << 15;
  t.lr = 1e-2;
  t.beta1 = 0.9;
  t.beta2 = 0.99;
  t.eps = 1e-8;
  t.e_fraction = 0.2;
  t.reflect = 1;
  t.pdf_floor = 1e-8;
  t.v_floor = 1e-12;
  t.seed = 0;
  return t;
}

struct SolverConfig {  // wost.hpp:20-31
  double epsilon_shell = 0.0, r_min = 0.0;
  int rr_depth = 128;
  SamplerMode mode = SamplerMode::Uniform;
  double fixed_c = 0.5;
  bool reflect_at_neumann = true, clamp_grazing = false;
  double grazing_floor = 1e-3;
  int max_steps = 1 << 16;
  wg_solver_config c() const {
    wg_solver_config o{};
    o.epsilon_shell = epsilon_shell;
    o.r_min = r_min;
    o.rr_depth = rr_depth;
    o.mode = static_cast<int32_t>(mode);
    o.fixed_c = fixed_c;
    o.reflect_at_neumann = reflect_at_neumann;
    o.clamp_grazing = clamp_grazing;
    o.grazing_floor = grazing_floor;
    o.max_steps = max_steps;
    return o;
  }
};

struct FieldConfig {  // guide_field.hpp:13-25
  std::vector<int> level_res = {16, 32, 64, 128};
  int features = 4, hidden = 64, mixture_k = 8, mixture_dim = 2;
  int output_dim() const { return (2 + mixture_dim) * mixture_k + 1; }
  wg_field_config c() const {
    wg_field_config o{};
    o.n_levels = static_cast<int32_t>(level_res.size());
    for (size_t i = 0; i < level_res.size() && i < WG_MAX_LEVELS; ++i) o.level_res[i] = level_res[i];
    o.features = features;
    o.hidden = hidden;
    o.mixture_k = mixture_k;
    o.mixture_dim = mixture_dim;
    return o;
  }
};

class Accel {  // geom2d.hpp:38-91, batched on the device
 public:
  // Accel(const Scene&) (geom2d.cpp:80-107): the scene is uploaded with its
  // values; segments whose value_index is unresolved are resolved by name
  explicit Accel(const Scene& s) {
    std::vector<double> seg;
    std::vector<int32_t> kind, vi;
    for (const auto& g : s.segments) {
      seg.insert(seg.end(), {g.a.x, g.a.y, g.b.x, g.b.y});
      kind.push_back(static_cast<int32_t>(g.kind));
      const int idx = g.value_index >= 0 ? g.value_index : s.find_value(g.value_ref);
      if (idx < 0) throw SceneError("value '" + g.value_ref + "' is not defined");
      vi.push_back(idx);
    }
    std::vector<wg_value_spec> vals;
    for (const auto& nv : s.values) vals.push_back(nv.second.c());
    const wg_value_spec src = s.source.c();
    double bb[4] = {s.bbox.min.x, s.bbox.min.y, s.bbox.max.x, s.bbox.max.y};
    check(wostgpu_scene_create(seg.data(), kind.data(), vi.data(), static_cast<int32_t>(kind.size()),
                               vals.data(), static_cast<int32_t>(vals.size()), &src, bb, s.epsilon_shell,
                               &h_));
  }
  // batched queries (the C-ABI entries; one CUDA thread per query)
  void closest_point_batch(std::span<const Vec2> xs, unsigned kinds, std::span<ClosestPoint> out) const {
    const size_t n = xs.size();
    std::vector<double> pt(2 * n), d(n);
    std::vector<int32_t> sg(n);
    check(wostgpu_closest_point(h_, static_cast<int64_t>(n), &xs.data()->x, kinds, pt.data(), d.data(),
                                sg.data()));
    for (size_t i = 0; i < n; ++i) out[i] = {{pt[2 * i], pt[2 * i + 1]}, d[i], sg[i]};
  }
  void star_radius_batch(std::span<const Vec2> xs, double r_min, double* r) const {
    check(wostgpu_star_radius(h_, static_cast<int64_t>(xs.size()), &xs.data()->x, r_min, r));
  }
  ~Accel() { wostgpu_scene_destroy(h_); }
  Accel(const Accel&) = delete;
  Accel& operator=(const Accel&) = delete;

  ClosestPoint closest_point(Vec2 x, unsigned kinds) const {
    ClosestPoint c;
    check(wostgpu_closest_point(h_, 1, &x.x, kinds, &c.point.x, &c.dist, &c.segment));
    return c;
  }
  double closest_silhouette(Vec2 x) const {
    double d = 0;
    check(wostgpu_closest_silhouette(h_, 1, &x.x, &d));
    return d;
  }
  std::optional<HitInfo> ray_first_hit(Vec2 o, Vec2 d, double t_max, unsigned kinds,
                                       int exclude_segment = -1) const {
    HitInfo h;
    int32_t kind = -1;
    check(wostgpu_ray_first_hit(h_, 1, &o.x, &d.x, &t_max, kinds, &exclude_segment, &h.t, &h.point.x,
                                &h.normal.x, &h.segment, &kind));
    if (h.segment < 0) return std::nullopt;
    h.kind = static_cast<BoundaryKind>(kind);
    return h;
  }
  double star_radius(Vec2 x, double r_min) const {
    double r = 0;
    check(wostgpu_star_radius(h_, 1, &x.x, r_min, &r));
    return r;
  }
  double t_epsilon() const {
    double t = 0;
    check(wostgpu_scene_info(h_, &t, nullptr, nullptr));
    return t;
  }
  wg_scene handle() const { return h_; }

 private:
  wg_scene h_ = nullptr;
};

class GuidingField {  // guide_field.hpp:37-96
 public:
  GuidingField(const FieldConfig& cfg, const Bbox& bbox, uint64_t seed) : cfg_(cfg), bbox_(bbox) {
    wg_field_config c = cfg.c();
    double bb[4] = {bbox.min.x, bbox.min.y, bbox.max.x, bbox.max.y};
    check(wostgpu_field_create(&c, bb, seed, &h_));
    check(wostgpu_field_param_count(h_, &n_));
  }
  ~GuidingField() {
    if (h_) wostgpu_field_destroy(h_);
  }
  GuidingField(const GuidingField&) = delete;
  GuidingField& operator=(const GuidingField&) = delete;
  GuidingField(GuidingField&& o) noexcept : cfg_(o.cfg_), bbox_(o.bbox_), h_(o.h_), n_(o.n_) {
    o.h_ = nullptr;
  }
  const FieldConfig& config() const { return cfg_; }
  const Bbox& bbox() const { return bbox_; }
  size_t param_count() const { return static_cast<size_t>(n_); }
  std::vector<float> params() const {
    std::vector<float> p(n_);
    check(wostgpu_field_get_state(h_, p.data(), nullptr, nullptr, nullptr));
    return p;
  }
  int64_t adam_steps() const {
    int64_t s = 0;
    check(wostgpu_field_get_state(h_, nullptr, nullptr, nullptr, &s));
    return s;
  }
  // GuidingField::eval (guide_field.cpp:178-221): the reference's fp32 MLP
  // arithmetic bit for bit (one point; batch with eval_batch)
  void eval(Vec2 x, double* out) const { check(wostgpu_field_eval_batch(h_, 1, &x.x, out, WG_MLP_EXACT)); }
  // eval_with_tape / backward (guide_field.cpp:223-243, 258-315): the tape
  // keeps the point; backward re-runs the fp64 forward on the device and
  // accumulates J^T d_out into grad
  struct Tape {
    Vec2 x;
  };
  void eval_with_tape(Vec2 x, double* out, Tape& tape) const {
    tape.x = x;
    eval(x, out);
  }
  void backward(const Tape& tape, const double* d_out, std::vector<double>& grad) const {
    if (grad.size() != param_count()) throw std::invalid_argument("backward: gradient size mismatch");
    check(wostgpu_field_backward(h_, 1, &tape.x.x, d_out, grad.data()));
  }
  // GuidingField::adam_step (guide_field.cpp:317-331); zeroes grad
  void adam_step(std::vector<double>& grad, double lr, double beta1, double beta2, double eps) {
    if (grad.size() != param_count()) throw std::invalid_argument("adam_step: gradient size mismatch");
    check(wostgpu_field_adam_step(h_, grad.data(), lr, beta1, beta2, eps));
  }
  float get_param(size_t i) const {
    float v = 0.0f;
    check(wostgpu_field_get_params(h_, static_cast<int64_t>(i), 1, &v));
    return v;
  }
  void set_param(size_t i, float v) { check(wostgpu_field_set_params(h_, static_cast<int64_t>(i), 1, &v)); }
  // row-major [points x output_dim] (guide_field.cpp:251-256)
  void eval_batch(std::span<const Vec2> xs, double* out, int mlp = WG_MLP_EXACT) const {
    check(wostgpu_field_eval_batch(h_, static_cast<int64_t>(xs.size()), &xs.data()->x, out, mlp));
  }
  wg_field handle() const { return h_; }

  // WGF1 checkpoint, byte-compatible with GuidingField::save / load
  // (guide_field.cpp:333-411): magic, version 1, level count + resolutions,
  // features, hidden, K, dim (u32), bbox (4 f64), Adam steps (i64), parameter
  // count (u64), fp32 params, fp64 Adam m, fp64 Adam v
  void save(std::ostream& out) const {
    std::vector<float> p(n_);
    std::vector<double> m(n_), v(n_);
    int64_t steps = 0;
    check(wostgpu_field_get_state(h_, p.data(), m.data(), v.data(), &steps));
    out.write("WGF1", 4);
    put<uint32_t>(out, 1);
    put<uint32_t>(out, static_cast<uint32_t>(cfg_.level_res.size()));
    for (int r : cfg_.level_res) put<uint32_t>(out, static_cast<uint32_t>(r));
    for (int x : {cfg_.features, cfg_.hidden, cfg_.mixture_k, cfg_.mixture_dim})
      put<uint32_t>(out, static_cast<uint32_t>(x));
    for (double x : {bbox_.min.x, bbox_.min.y, bbox_.max.x, bbox_.max.y}) put<double>(out, x);
    put<int64_t>(out, steps);
    put<uint64_t>(out, static_cast<uint64_t>(n_));
    out.write(reinterpret_cast<const char*>(p.data()), static_cast<std::streamsize>(p.size() * 4));
    out.write(reinterpret_cast<const char*>(m.data()), static_cast<std::streamsize>(m.size() * 8));
    out.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * 8));
  }
  static GuidingField load(std::istream& in) {
    char magic[4];
    in.read(magic, 4);
    if (!in || std::memcmp(magic, "WGF1", 4) != 0)
      throw std::runtime_error("guiding field checkpoint: bad magic");
    if (get<uint32_t>(in) != 1) throw std::runtime_error("guiding field checkpoint: unknown version");
    FieldConfig cfg;
    cfg.level_res.resize(get<uint32_t>(in));
    for (auto& r : cfg.level_res) r = static_cast<int>(get<uint32_t>(in));
    cfg.features = static_cast<int>(get<uint32_t>(in));
    cfg.hidden = static_cast<int>(get<uint32_t>(in));
    cfg.mixture_k = static_cast<int>(get<uint32_t>(in));
    cfg.mixture_dim = static_cast<int>(get<uint32_t>(in));
    Bbox bb;
    bb.min.x = get<double>(in);
    bb.min.y = get<double>(in);
    bb.max.x = get<double>(in);
    bb.max.y = get<double>(in);
    const int64_t steps = get<int64_t>(in);
    GuidingField f(cfg, bb, 0);
    if (get<uint64_t>(in) != static_cast<uint64_t>(f.n_))
      throw std::runtime_error("guiding field checkpoint: size mismatch");
    std::vector<float> p(f.n_);
    std::vector<double> m(f.n_), v(f.n_);
    in.read(reinterpret_cast<char*>(p.data()), static_cast<std::streamsize>(p.size() * 4));
    in.read(reinterpret_cast<char*>(m.data()), static_cast<std::streamsize>(m.size() * 8));
    in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(v.size() * 8));
    if (!in) throw std::runtime_error("guiding field checkpoint: truncated");
    check(wostgpu_field_set_state(f.h_, p.data(), m.data(), v.data(), steps));
    return f;
  }

 private:
  template <typename T>
  static void put(std::ostream& out, T v) {
    out.write(reinterpret_cast<const char*>(&v), sizeof(T));
  }
  template <typename T>
  static T get(std::istream& in) {
    T v{};
    in.read(reinterpret_cast<char*>(&v), sizeof(T));
    return v;
  }
  FieldConfig cfg_;
  Bbox bbox_;
  wg_field h_ = nullptr;
  int64_t n_ = 0;
};

// StepContext + SolveScratch (wost.hpp:33-51, 147-154): the device solver
class StepContext {
 public:
  StepContext(const Accel& accel, const GuidingField* field, const SolverConfig& cfg) {
    wg_solver_config c = cfg.c();
    check(wostgpu_solver_create(accel.handle(), field ? field->handle() : nullptr, &c, &h_));
  }
  ~StepContext() { wostgpu_solver_destroy(h_); }
  StepContext(const StepContext&) = delete;
  StepContext& operator=(const StepContext&) = delete;
  wg_solver handle() const { return h_; }

 private:
  wg_solver h_ = nullptr;
};

// SolveScratch (wost.hpp:147-154): the reference reuses its host wavefront
// buffers across rounds; the device solver (StepContext) owns its walk
// queues and record arena, so the scratch object carries nothing and the
// parameter is accepted for source compatibility
struct SolveScratch {};

// solve_batch (wost.hpp:160-163): one walk per point for wpp round
// `wpp_index`, Welford statistics updated in place, records appended
inline void solve_batch(const StepContext& ctx, std::span<const Vec2> points,
                        std::span<PointStats> stats, uint64_t seed, uint64_t wpp_index,
                        bool collect_records, std::vector<GuideRecord>* records,
                        SolveScratch* scratch = nullptr) {
  (void)scratch;
  if (points.size() != stats.size()) throw std::invalid_argument("points and stats differ in size");
  check(wostgpu_solve_batch(ctx.handle(), static_cast<int64_t>(points.size()), &points.data()->x,
                            stats.data(), seed, wpp_index, collect_records ? 1 : 0));
  if (collect_records && records) {
    int64_t n = 0;
    check(wostgpu_fetch_records(ctx.handle(), nullptr, 0, &n));
    size_t base = records->size();
    records->resize(base + static_cast<size_t>(n));
    check(wostgpu_fetch_records(ctx.handle(), records->data() + base, n, &n));
  }
}

// train_batch (guide_train.hpp:104-105) on host records
inline TrainStats train_batch(const StepContext& ctx, std::span<const GuideRecord> records,
                              const TrainConfig& cfg, uint64_t round) {
  TrainStats st{};
  check(wostgpu_train_batch(ctx.handle(), records.data(), static_cast<int64_t>(records.size()), &cfg,
                            round, &st));
  return st;
}

// Engine::run_batch loop of run_solve (solver.cpp:92-104, 136-146) natively
inline TrainStats run(const StepContext& ctx, std::span<const Vec2> points,
                      std::span<PointStats> stats, uint64_t seed, int wpp, int64_t train_until,
                      const TrainConfig* train_cfg, double* device_ms = nullptr) {
  check(wostgpu_solver_set_points(ctx.handle(), static_cast<int64_t>(points.size()),
                                  &points.data()->x, 0));
  check(wostgpu_solver_set_stats(ctx.handle(), stats.data()));
  TrainStats st{};
  double ms = 0;
  check(wostgpu_run(ctx.handle(), seed, wpp, train_until, train_cfg, &st, &ms));
  check(wostgpu_solver_get_stats(ctx.handle(), stats.data()));
  if (device_ms) *device_ms = ms;
  return st;
}

}  // namespace wostgpu
