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
#include <vector>

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

// Scene description in the reference's shape (scene.hpp:70-96): values are
// wg_value_spec (constant / linear / raster / preset analytic)
struct BoundarySegment {
  Vec2 a, b;
  BoundaryKind kind = BoundaryKind::Dirichlet;
  int value_index = 0;
};
struct Scene {
  Bbox bbox;
  double epsilon_shell = 0.0;
  std::vector<wg_value_spec> values;
  wg_value_spec source{WG_VALUE_ZERO, 0, 0, 0, 0, 0, 0, {0, 0, 0, 0}, nullptr};
  std::vector<BoundarySegment> segments;
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
  explicit Accel(const Scene& s) {
    std::vector<double> seg;
    std::vector<int32_t> kind, vi;
    for (const auto& g : s.segments) {
      seg.insert(seg.end(), {g.a.x, g.a.y, g.b.x, g.b.y});
      kind.push_back(static_cast<int32_t>(g.kind));
      vi.push_back(g.value_index);
    }
    double bb[4] = {s.bbox.min.x, s.bbox.min.y, s.bbox.max.x, s.bbox.max.y};
    check(wostgpu_scene_create(seg.data(), kind.data(), vi.data(), static_cast<int32_t>(kind.size()),
                               s.values.data(), static_cast<int32_t>(s.values.size()), &s.source, bb,
                               s.epsilon_shell, &h_));
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

// solve_batch (wost.hpp:160-163): one walk per point for wpp round
// `wpp_index`, Welford statistics updated in place, records appended
inline void solve_batch(const StepContext& ctx, std::span<const Vec2> points,
                        std::span<PointStats> stats, uint64_t seed, uint64_t wpp_index,
                        bool collect_records, std::vector<GuideRecord>* records) {
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
