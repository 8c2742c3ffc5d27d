// TEST INFRASTRUCTURE ONLY. extern "C" wrappers around the UNMODIFIED reference
// library (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/). Used to pin the CPU restatement (oracle/wost_oracle.cpp), to
// generate golden fixtures (tests/golden/make_golden.py) and as the CPU
// baseline arm of bench.py. Nothing here re-implements reference arithmetic;
// every function forwards to the reference API named in its comment.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "oracle_abi.h"
#include "wost/geom2d.hpp"
#include "wost/guide_field.hpp"
#include "wost/guide_train.hpp"
#include "wost/image.hpp"
#include "wost/presets.hpp"
#include "wost/solver.hpp"
#include "wost/sphdist.hpp"
#include "wost/wost.hpp"

using namespace wost;

namespace {

thread_local std::string g_err;

struct RefScene {
  Scene scene;
  std::optional<Accel> accel;
};

ValueSpec to_value(const wg_value_spec& v) {
  ValueSpec out;
  switch (v.type) {
    case WG_VALUE_CONSTANT: out.spec = ValueSpec::Constant{v.c0}; break;
    case WG_VALUE_LINEAR: out.spec = ValueSpec::Linear{v.c0, v.cx, v.cy}; break;
    case WG_VALUE_RASTER: {
      RasterGrid g;
      g.width = v.raster_w;
      g.height = v.raster_h;
      g.bbox = Bbox{{v.raster_bbox[0], v.raster_bbox[1]},
                    {v.raster_bbox[2], v.raster_bbox[3]}};
      g.data.assign(v.raster_data, v.raster_data + (size_t)v.raster_w * v.raster_h);
      out.spec = ValueSpec::Raster{std::move(g)};
      break;
    }
    case WG_VALUE_ANALYTIC:
      // the two preset closed forms (proj/src/presets.cpp:191, :202)
      if (v.analytic_id == WG_ANALYTIC_X2_MINUS_Y2)
        out.spec = ValueSpec::Analytic{[](Vec2 q) { return q.x * q.x - q.y * q.y; }, "x^2-y^2"};
      else
        out.spec = ValueSpec::Analytic{[](Vec2 q) { return q.x * q.x + q.y * q.y - 1.0; }, "r^2-1"};
      break;
    default: throw std::invalid_argument("bad value spec type");
  }
  return out;
}

SolverConfig to_solver(const wg_solver_config* c) {
  SolverConfig s;
  s.epsilon_shell = c->epsilon_shell;
  s.r_min = c->r_min;
  s.rr_depth = c->rr_depth;
  s.mode = static_cast<SamplerMode>(c->mode);
  s.fixed_c = c->fixed_c;
  s.reflect_at_neumann = c->reflect_at_neumann != 0;
  s.clamp_grazing = c->clamp_grazing != 0;
  s.grazing_floor = c->grazing_floor;
  s.max_steps = c->max_steps;
  return s;
}

FieldConfig to_field(const wg_field_config* c) {
  FieldConfig f;
  f.level_res.assign(c->level_res, c->level_res + c->n_levels);
  f.features = c->features;
  f.hidden = c->hidden;
  f.mixture_k = c->mixture_k;
  f.mixture_dim = c->mixture_dim;
  return f;
}

TrainConfig to_train(const wg_train_config* c) {
  TrainConfig t;
  t.minibatch = c->minibatch;
  t.max_records_per_round = static_cast<size_t>(c->max_records_per_round);
  t.lr = c->lr;
  t.beta1 = c->beta1;
  t.beta2 = c->beta2;
  t.eps = c->eps;
  t.e_fraction = c->e_fraction;
  t.learn_selection = c->learn_selection != 0;
  t.reflect = c->reflect != 0;
  t.pdf_floor = c->pdf_floor;
  t.v_floor = c->v_floor;
  t.seed = c->seed;
  return t;
}

GuideRecord to_record(const wg_guide_record& r) {
  GuideRecord g;
  g.x = {r.x[0], r.x[1]};
  g.nu = {r.nu[0], r.nu[1], r.nu[2]};
  g.target = r.target;
  g.pdf_mis = r.pdf_mis;
  g.pdf_g = r.pdf_g;
  g.pdf_u = r.pdf_u;
  g.c = r.c;
  g.on_neumann = r.on_neumann != 0;
  g.normal = {r.normal[0], r.normal[1]};
  return g;
}

wg_guide_record from_record(const GuideRecord& g) {
  wg_guide_record r{};
  r.x[0] = g.x.x;
  r.x[1] = g.x.y;
  r.nu[0] = g.nu.x;
  r.nu[1] = g.nu.y;
  r.nu[2] = g.nu.z;
  r.target = g.target;
  r.pdf_mis = g.pdf_mis;
  r.pdf_g = g.pdf_g;
  r.pdf_u = g.pdf_u;
  r.c = g.c;
  r.on_neumann = g.on_neumann ? 1 : 0;
  r.normal[0] = g.normal.x;
  r.normal[1] = g.normal.y;
  return r;
}

void to_mixture(const MixtureParams& m, wg_mixture* out) {
  std::memset(out, 0, sizeof(*out));
  for (int i = 0; i < m.k; ++i) {
    out->mu[i][0] = m.comps[i].mu.x;
    out->mu[i][1] = m.comps[i].mu.y;
    out->mu[i][2] = m.comps[i].mu.z;
    out->kappa[i] = m.comps[i].kappa;
    out->lambda[i] = m.comps[i].lambda;
    out->log_a[i] = m.log_a[i];
  }
  out->c = m.c;
  out->k = m.k;
  out->dim = m.dim;
}

MixtureParams from_mixture(const wg_mixture* m) {
  MixtureParams p;
  p.k = m->k;
  p.dim = m->dim;
  p.c = m->c;
  for (int i = 0; i < m->k; ++i) {
    p.comps[i].mu = {m->mu[i][0], m->mu[i][1], m->mu[i][2]};
    p.comps[i].kappa = m->kappa[i];
    p.comps[i].lambda = m->lambda[i];
    p.log_a[i] = m->log_a[i];
  }
  return p;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return WG_OK;
  } catch (const SceneError& e) {
    g_err = e.what();
    return WG_ERR_SCENE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return WG_ERR_INVALID;
  } catch (const std::exception& e) {
    g_err = e.what();
    return WG_ERR_RUNTIME;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void* ref_scene_create(const double* seg, const int32_t* kind, const int32_t* value_index,
                       int32_t n_seg, const wg_value_spec* values, int32_t n_values,
                       const wg_value_spec* source, const double* bbox, double eps) {
  RefScene* out = nullptr;
  int rc = guarded([&] {
    auto rs = std::make_unique<RefScene>();
    Scene& s = rs->scene;
    s.bbox = Bbox{{bbox[0], bbox[1]}, {bbox[2], bbox[3]}};
    s.epsilon_shell = eps;
    for (int i = 0; i < n_values; ++i)
      s.values.emplace_back("v" + std::to_string(i), to_value(values[i]));
    if (!source || source->type == WG_VALUE_ZERO) s.source.spec = SourceField::Zero{};
    else if (source->type == WG_VALUE_CONSTANT) s.source.spec = SourceField::Constant{source->c0};
    else {
      ValueSpec v = to_value(*source);
      s.source.spec = SourceField::Raster{std::get<ValueSpec::Raster>(v.spec).grid};
    }
    for (int i = 0; i < n_seg; ++i) {
      BoundarySegment b;
      b.a = {seg[4 * i + 0], seg[4 * i + 1]};
      b.b = {seg[4 * i + 2], seg[4 * i + 3]};
      b.kind = kind[i] == WG_NEUMANN ? BoundaryKind::Neumann : BoundaryKind::Dirichlet;
      b.value_ref = "v" + std::to_string(value_index[i]);
      s.segments.push_back(b);
    }
    // test scenes (proj/tests/test_geom2d.cpp:11-20) skip validate(); so do
    // we when eps <= 0 is passed deliberately (it is then forced to 1e-3)
    if (eps > 0.0) s.validate();
    else {
      s.epsilon_shell = 1e-3;
      for (auto& b : s.segments) b.value_index = s.find_value(b.value_ref);
    }
    rs->accel.emplace(s);  // Accel::Accel, proj/src/geom2d.cpp:80
    out = rs.release();
  });
  return rc == WG_OK ? out : nullptr;
}

void ref_scene_destroy(void* s) { delete static_cast<RefScene*>(s); }
double ref_t_epsilon(void* s) { return static_cast<RefScene*>(s)->accel->t_epsilon(); }
int32_t ref_has_neumann_flux(void* s) { return static_cast<RefScene*>(s)->scene.has_neumann_flux(); }

int ref_closest_point(void* sp, int64_t n, const double* xy, uint32_t kinds, double* pt,
                      double* dist, int32_t* seg) {
  auto* s = static_cast<RefScene*>(sp);
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) {
      ClosestPoint c = s->accel->closest_point({xy[2 * i], xy[2 * i + 1]}, kinds);
      pt[2 * i] = c.point.x;
      pt[2 * i + 1] = c.point.y;
      dist[i] = c.dist;
      seg[i] = c.segment;
    }
  });
}

int ref_closest_silhouette(void* sp, int64_t n, const double* xy, double* dist) {
  auto* s = static_cast<RefScene*>(sp);
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i)
      dist[i] = s->accel->closest_silhouette({xy[2 * i], xy[2 * i + 1]});
  });
}

int ref_ray_first_hit(void* sp, int64_t n, const double* o, const double* d,
                      const double* t_max, uint32_t kinds, const int32_t* exclude, double* t,
                      double* pt, double* normal, int32_t* seg, int32_t* kind) {
  auto* s = static_cast<RefScene*>(sp);
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) {
      auto h = s->accel->ray_first_hit({o[2 * i], o[2 * i + 1]}, {d[2 * i], d[2 * i + 1]},
                                       t_max[i], kinds, exclude ? exclude[i] : -1);
      if (h) {
        t[i] = h->t;
        pt[2 * i] = h->point.x;
        pt[2 * i + 1] = h->point.y;
        normal[2 * i] = h->normal.x;
        normal[2 * i + 1] = h->normal.y;
        seg[i] = h->segment;
        kind[i] = h->kind == BoundaryKind::Neumann ? WG_NEUMANN : WG_DIRICHLET;
      } else {
        t[i] = kInf;
        pt[2 * i] = pt[2 * i + 1] = 0.0;
        normal[2 * i] = normal[2 * i + 1] = 0.0;
        seg[i] = -1;
        kind[i] = -1;
      }
    }
  });
}

int ref_star_radius(void* sp, int64_t n, const double* xy, double r_min, double* r) {
  auto* s = static_cast<RefScene*>(sp);
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) r[i] = s->accel->star_radius({xy[2 * i], xy[2 * i + 1]}, r_min);
  });
}

double ref_bessel_i0(double x) { return bessel_i0(x); }
double ref_log_bessel_i0(double x) { return log_bessel_i0(x); }
double ref_bessel_i1_over_i0(double x) { return bessel_i1_over_i0(x); }

void ref_normalize_params(int64_t n, const double* raw, int32_t k, int32_t dim, wg_mixture* out) {
  const int od = UnnormParams::param_count(k, dim);
  for (int64_t i = 0; i < n; ++i)
    to_mixture(normalize_params(unpack_params(raw + i * od, k, dim)), &out[i]);
}

double ref_mixture_pdf(const wg_mixture* m, const double* nu) {
  return mixture_pdf({nu[0], nu[1], nu[2]}, from_mixture(m));
}

double ref_mis_pdf(const wg_mixture* m, const double* nu, const double* normal, int32_t reflect) {
  Vec3 n3;
  if (normal) n3 = {normal[0], normal[1], normal[2]};
  return mis_pdf({nu[0], nu[1], nu[2]}, from_mixture(m), normal ? &n3 : nullptr, reflect != 0);
}

void* ref_field_create(const wg_field_config* cfg, const double* bbox, uint64_t seed) {
  GuidingField* f = nullptr;
  int rc = guarded([&] {
    f = new GuidingField(to_field(cfg), Bbox{{bbox[0], bbox[1]}, {bbox[2], bbox[3]}}, seed);
  });
  return rc == WG_OK ? f : nullptr;
}
void ref_field_destroy(void* f) { delete static_cast<GuidingField*>(f); }
int64_t ref_field_param_count(void* f) { return static_cast<GuidingField*>(f)->param_count(); }
void ref_field_get_params(void* fp, float* out) {
  auto* f = static_cast<GuidingField*>(fp);
  for (size_t i = 0; i < f->param_count(); ++i) out[i] = f->get_param(i);
}
void ref_field_set_params(void* fp, const float* in) {
  auto* f = static_cast<GuidingField*>(fp);
  for (size_t i = 0; i < f->param_count(); ++i) f->set_param(i, in[i]);
}
// WGF1 checkpoints through the reference's own GuidingField::save / load
// (proj/src/guide_field.cpp:351-411)
int ref_field_save(void* fp, const char* path) {
  return guarded([&] {
    std::ofstream out(path, std::ios::binary);
    static_cast<GuidingField*>(fp)->save(out);
    if (!out) throw std::runtime_error("write failed");
  });
}
void* ref_field_load(const char* path) {
  GuidingField* f = nullptr;
  int rc = guarded([&] {
    std::ifstream in(path, std::ios::binary);
    f = new GuidingField(GuidingField::load(in));
  });
  return rc == WG_OK ? f : nullptr;
}
int64_t ref_field_adam_steps(void* fp) { return static_cast<GuidingField*>(fp)->adam_steps(); }
// GuidingField::eval_with_tape + backward (proj/src/guide_field.cpp:223-243,
// 258-315) summed over n points, in point order
void ref_field_backward(void* fp, int64_t n, const double* xy, const double* d_out, double* grad) {
  auto* f = static_cast<GuidingField*>(fp);
  const int od = f->config().output_dim();
  std::vector<double> g(grad, grad + f->param_count());
  std::vector<double> out(od);
  GuidingField::Tape tape;
  for (int64_t i = 0; i < n; ++i) {
    f->eval_with_tape({xy[2 * i], xy[2 * i + 1]}, out.data(), tape);
    f->backward(tape, d_out + i * od, g);
  }
  std::copy(g.begin(), g.end(), grad);
}

// GuidingField::adam_step (proj/src/guide_field.cpp:317-331) on a given
// gradient (which the reference zeroes on return)
void ref_field_adam_step(void* fp, const double* grad, double lr, double beta1, double beta2, double eps) {
  auto* f = static_cast<GuidingField*>(fp);
  std::vector<double> g(grad, grad + f->param_count());
  f->adam_step(g, lr, beta1, beta2, eps);
}

// result formats through the reference's own writers (proj/src/image.cpp,
// solver.cpp:317-327) for byte-level comparison with the Python harness
int ref_write_image(int32_t w, int32_t h, const double* bbox, const wg_point_stats* cells,
                    const char* csv, const char* pfm, const char* png) {
  return guarded([&] {
    SolutionImage img = make_image(w, h, Bbox{{bbox[0], bbox[1]}, {bbox[2], bbox[3]}});
    for (size_t i = 0; i < img.cells.size(); ++i) {
      img.cells[i].mean = cells[i].mean;
      img.cells[i].m2 = cells[i].m2;
      img.cells[i].count = cells[i].count;
      img.cells[i].escaped = cells[i].escaped;
    }
    if (csv && *csv) write_csv(img, csv);
    if (pfm && *pfm) write_pfm(img, pfm);
    if (png && *png) write_png(img, png);
  });
}
double ref_compute_relmse(int32_t w, int32_t h, const double* est, const double* refv) {
  SolutionImage a = make_image(w, h, Bbox{{0, 0}, {1, 1}}), b = a;
  for (size_t i = 0; i < a.cells.size(); ++i) {
    a.cells[i].mean = est[i];
    b.cells[i].mean = refv[i];
  }
  return compute_relmse(a, b);
}
int ref_write_convergence_log(int32_t n, const int32_t* wpp, const double* relmse, const double* sec,
                              const char* path) {
  return guarded([&] {
    std::vector<LogRow> rows(n);
    for (int32_t i = 0; i < n; ++i) rows[i] = LogRow{wpp[i], relmse[i], sec[i]};
    write_convergence_log(rows, path);
  });
}
// write_scene(make_preset(name).scene) into buf (NUL-terminated); returns
// the JSON length, or -1 (error text in ref_last_error)
int64_t ref_preset_scene_json(const char* name, char* buf, int64_t cap) {
  int64_t n = -1;
  guarded([&] {
    std::string js = write_scene(make_preset(name).scene);
    n = static_cast<int64_t>(js.size());
    if (buf && cap > n) std::memcpy(buf, js.c_str(), js.size() + 1);
  });
  return n;
}
// load_scene(json) -> geometry back out, for loader parity
int64_t ref_load_scene_json(const char* text, double* seg, int32_t* kind, int32_t* value_index,
                            int64_t cap, double* bbox, double* eps) {
  int64_t n = -1;
  guarded([&] {
    Scene sc = load_scene(text);
    n = static_cast<int64_t>(sc.segments.size());
    for (int64_t i = 0; i < n && i < cap; ++i) {
      const auto& s = sc.segments[i];
      seg[4 * i] = s.a.x;
      seg[4 * i + 1] = s.a.y;
      seg[4 * i + 2] = s.b.x;
      seg[4 * i + 3] = s.b.y;
      kind[i] = s.kind == BoundaryKind::Dirichlet ? 0 : 1;
      value_index[i] = s.value_index;
    }
    bbox[0] = sc.bbox.min.x;
    bbox[1] = sc.bbox.min.y;
    bbox[2] = sc.bbox.max.x;
    bbox[3] = sc.bbox.max.y;
    *eps = sc.epsilon_shell;
  });
  return n;
}
void ref_field_eval_batch(void* fp, int64_t n, const double* xy, double* out) {
  auto* f = static_cast<GuidingField*>(fp);
  std::vector<Vec2> xs(n);
  for (int64_t i = 0; i < n; ++i) xs[i] = {xy[2 * i], xy[2 * i + 1]};
  f->eval_batch(xs, out);  // proj/src/guide_field.cpp:251
}

int ref_walks(void* sp, void* fp, const wg_solver_config* cfg, int64_t n, const double* xy,
              const int64_t* point_index, uint64_t seed, uint64_t wpp_index, double* estimate,
              int32_t* escaped, int32_t* n_records) {
  auto* s = static_cast<RefScene*>(sp);
  return guarded([&] {
    StepContext ctx{&s->scene, &*s->accel, static_cast<GuidingField*>(fp), to_solver(cfg)};
    std::vector<GuideRecord> recs;
    for (int64_t i = 0; i < n; ++i) {
      recs.clear();
      // proj/src/wost.cpp:274 with the stream of proj/include/wost/rng.hpp:28
      WalkResult r = wost_walk(ctx, {xy[2 * i], xy[2 * i + 1]},
                               Rng::for_walk(seed, point_index ? point_index[i] : i, wpp_index),
                               n_records ? &recs : nullptr);
      estimate[i] = r.estimate;
      escaped[i] = r.escaped ? 1 : 0;
      if (n_records) n_records[i] = static_cast<int32_t>(recs.size());
    }
  });
}

int ref_solve_batch(void* sp, void* fp, const wg_solver_config* cfg, int64_t n, const double* xy,
                    wg_point_stats* stats, uint64_t seed, uint64_t wpp_index, int32_t collect,
                    wg_guide_record** records, int64_t* n_records) {
  auto* s = static_cast<RefScene*>(sp);
  return guarded([&] {
    StepContext ctx{&s->scene, &*s->accel, static_cast<GuidingField*>(fp), to_solver(cfg)};
    std::vector<Vec2> pts(n);
    for (int64_t i = 0; i < n; ++i) pts[i] = {xy[2 * i], xy[2 * i + 1]};
    std::vector<PointStats> st(n);
    for (int64_t i = 0; i < n; ++i) {
      st[i].mean = stats[i].mean;
      st[i].m2 = stats[i].m2;
      st[i].count = stats[i].count;
      st[i].escaped = stats[i].escaped;
    }
    std::vector<GuideRecord> recs;
    solve_batch(ctx, pts, st, seed, wpp_index, collect != 0, collect ? &recs : nullptr);
    for (int64_t i = 0; i < n; ++i) {
      stats[i].mean = st[i].mean;
      stats[i].m2 = st[i].m2;
      stats[i].count = st[i].count;
      stats[i].escaped = st[i].escaped;
    }
    if (records) {
      auto* out = static_cast<wg_guide_record*>(std::malloc(sizeof(wg_guide_record) * (recs.size() + 1)));
      for (size_t i = 0; i < recs.size(); ++i) out[i] = from_record(recs[i]);
      *records = out;
      *n_records = static_cast<int64_t>(recs.size());
    }
  });
}

void ref_free(void* p) { std::free(p); }

int ref_train_batch(void* fp, const wg_guide_record* recs, int64_t n, const wg_train_config* cfg,
                    uint64_t round, wg_train_stats* stats) {
  auto* f = static_cast<GuidingField*>(fp);
  return guarded([&] {
    std::vector<GuideRecord> rv(n);
    for (int64_t i = 0; i < n; ++i) rv[i] = to_record(recs[i]);
    TrainStats ts = train_batch(*f, rv, to_train(cfg), round);  // guide_train.cpp:94
    stats->records_seen = ts.records_seen;
    stats->records_consumed = ts.records_consumed;
    stats->skipped_low_pdf = ts.skipped_low_pdf;
    stats->skipped_low_v = ts.skipped_low_v;
    stats->steps = ts.steps;
    stats->mean_grad_norm = ts.mean_grad_norm;
    stats->seconds = ts.seconds;
  });
}

// Mean gradient of one minibatch made of `recs` in the given order: the inner
// loop of train_batch (proj/src/guide_train.cpp:146-171) without the shuffle,
// cap and Adam step, composed from the reference's own eval_with_tape,
// kl_grad, selection_grad and backward.
int ref_field_grad(void* fp, const wg_guide_record* recs, int64_t n, const wg_train_config* cfg,
                   double* grad_out) {
  auto* f = static_cast<GuidingField*>(fp);
  return guarded([&] {
    TrainConfig tc = to_train(cfg);
    const int k = f->config().mixture_k, dim = f->config().mixture_dim;
    const int od = f->config().output_dim();
    std::vector<double> grad(f->param_count(), 0.0);
    GuidingField::Tape tape;
    std::vector<double> out(od), d_out(od);
    double inv_count = 1.0 / static_cast<double>(n);
    for (int64_t r = 0; r < n; ++r) {
      GuideRecord rec = to_record(recs[r]);
      if (rec.pdf_mis < tc.pdf_floor) continue;
      f->eval_with_tape(rec.x, out.data(), tape);
      UnnormParams raw = unpack_params(out.data(), k, dim);
      ParamGrad pg;
      if (!kl_grad(rec, raw, tc.reflect, tc.v_floor, pg, nullptr)) continue;
      pg.c_raw = tc.learn_selection
                     ? selection_grad(rec, normalize_params(raw), tc.reflect, tc.e_fraction)
                     : 0.0;
      double* m = d_out.data();
      for (int i = 0; i < k; ++i)
        for (int a = 0; a < dim; ++a) *m++ = pg.mu_raw[i][a] * inv_count;
      for (int i = 0; i < k; ++i) *m++ = pg.kappa_raw[i] * inv_count;
      for (int i = 0; i < k; ++i) *m++ = pg.lambda_raw[i] * inv_count;
      *m = pg.c_raw * inv_count;
      f->backward(tape, d_out.data(), grad);
    }
    std::memcpy(grad_out, grad.data(), grad.size() * sizeof(double));
  });
}

// ---- harness entry points (bench.py CPU baseline; not part of the oracle ABI)

// run_solve (proj/src/solver.cpp:124) on a preset at the given grid/wpp/mode;
// relMSE against generate_reference (analytic presets; solver.cpp:169-181).
int ref_run_solve(const char* preset, int32_t width, int32_t height, int32_t wpp, int32_t mode,
                  int64_t train_until, uint64_t seed, wg_point_stats* stats_out,
                  double* seconds, double* relmse, double* train_seconds) {
  return guarded([&] {
    RunConfig cfg;
    cfg.preset = preset;
    cfg.grid.width = width;
    cfg.grid.height = height;
    cfg.wpp = wpp;
    cfg.mode = static_cast<SamplerMode>(mode);
    cfg.train_until = static_cast<uint64_t>(train_until);
    cfg.seed = seed;
    RunResult res = run_solve(cfg);
    *seconds = res.seconds;
    *train_seconds = res.train_stats.seconds;
    if (stats_out)
      for (size_t i = 0; i < res.image.cells.size(); ++i) {
        stats_out[i].mean = res.image.cells[i].mean;
        stats_out[i].m2 = res.image.cells[i].m2;
        stats_out[i].count = res.image.cells[i].count;
        stats_out[i].escaped = res.image.cells[i].escaped;
      }
    SolutionImage ref = generate_reference(cfg, 1);
    *relmse = compute_relmse(res.image, ref);
  });
}

// run_solve writing the trained field as a WGF1 checkpoint (cfg.field_out)
int ref_run_solve_field(const char* preset, int32_t width, int32_t height, int32_t wpp, int32_t mode,
                        int64_t train_until, uint64_t seed, const char* field_out, double* relmse) {
  return guarded([&] {
    RunConfig cfg;
    cfg.preset = preset;
    cfg.grid.width = width;
    cfg.grid.height = height;
    cfg.wpp = wpp;
    cfg.mode = static_cast<SamplerMode>(mode);
    cfg.train_until = static_cast<uint64_t>(train_until);
    cfg.seed = seed;
    cfg.field_out = field_out;
    RunResult res = run_solve(cfg);
    SolutionImage ref = generate_reference(cfg, 1);
    *relmse = compute_relmse(res.image, ref);
  });
}

// preset scene geometry, for pinning the product's preset fixtures
int ref_preset(const char* name, double* seg_out, int32_t* kind_out, int32_t* n_seg,
               double* eval_bbox, double* scene_bbox, double* eps) {
  return guarded([&] {
    Preset p = make_preset(name);
    if (seg_out) {
      for (size_t i = 0; i < p.scene.segments.size(); ++i) {
        const auto& s = p.scene.segments[i];
        seg_out[4 * i + 0] = s.a.x;
        seg_out[4 * i + 1] = s.a.y;
        seg_out[4 * i + 2] = s.b.x;
        seg_out[4 * i + 3] = s.b.y;
        kind_out[i] = s.kind == BoundaryKind::Neumann ? WG_NEUMANN : WG_DIRICHLET;
      }
    }
    *n_seg = static_cast<int32_t>(p.scene.segments.size());
    eval_bbox[0] = p.eval_bbox.min.x;
    eval_bbox[1] = p.eval_bbox.min.y;
    eval_bbox[2] = p.eval_bbox.max.x;
    eval_bbox[3] = p.eval_bbox.max.y;
    scene_bbox[0] = p.scene.bbox.min.x;
    scene_bbox[1] = p.scene.bbox.min.y;
    scene_bbox[2] = p.scene.bbox.max.x;
    scene_bbox[3] = p.scene.bbox.max.y;
    *eps = p.scene.epsilon_shell;
  });
}

double ref_strip_vlin_solution(double x, double y) { return strip_vlin_solution({x, y}); }

}  // extern "C"
