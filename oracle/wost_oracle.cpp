// ============================================================================
// TEST INFRASTRUCTURE ONLY — the CPU oracle for the guided walk-on-stars path.
//
// An independent restatement of the reference algorithm (arXiv 2410.18944 C++
// artifact, paths relative to /root/reference/proj), written from the
// reference's behaviour, used ONLY by tests/, __graft_entry__.smoke() and the
// cpu_baseline leg of bench.py as the checker. The product (libwostgpu.so)
// never links, loads or calls it.
//
// Parity of this restatement is pinned two ways (tests/test_oracle.py):
//   * against the reference library itself, compiled from its own sources
//     into oracle/_ref/ (bit-exact for geometry, field eval, normalisation,
//     per-walk estimates; gradient/Adam to 1e-12),
//   * against golden vectors generated from oracle/_ref and the reference's
//     own unit-test known answers (tests/golden/).
//
// Floating point: compiled with -ffp-contract=off, and every expression keeps
// the reference's operation order, so results are bit-comparable with the
// strict build of the reference (oracle/_ref/libwost_ref.so).
// ============================================================================
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "oracle_abi.h"

namespace orc {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;
constexpr double kFourPi = 4.0 * kPi;
constexpr double kInf = std::numeric_limits<double>::infinity();
constexpr int kMaxK = WG_MAX_MIXTURE;
constexpr double kKappaMin = 1e-6, kKappaMax = 1e4;  // sphdist.hpp:17-18

struct SceneErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- vectors
// proj/include/wost/vec.hpp:14-96
struct V2 {
  double x = 0, y = 0;
};
struct V3 {
  double x = 0, y = 0, z = 0;
};
inline V2 add(V2 a, V2 b) { return {a.x + b.x, a.y + b.y}; }
inline V2 sub(V2 a, V2 b) { return {a.x - b.x, a.y - b.y}; }
inline V2 scl(V2 a, double s) { return {a.x * s, a.y * s}; }
inline double dot2(V2 a, V2 b) { return a.x * b.x + a.y * b.y; }
inline double cross2(V2 a, V2 b) { return a.x * b.y - a.y * b.x; }
inline double len2(V2 a) { return std::sqrt(dot2(a, a)); }
inline V3 add3(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 sub3(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 scl3(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double dot3(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline double len3(V3 a) { return std::sqrt(dot3(a, a)); }

struct Box {
  V2 lo{kInf, kInf}, hi{-kInf, -kInf};
  void grow(V2 p) {
    lo.x = std::min(lo.x, p.x);
    lo.y = std::min(lo.y, p.y);
    hi.x = std::max(hi.x, p.x);
    hi.y = std::max(hi.y, p.y);
  }
  bool contains(V2 p, double pad) const {
    return p.x >= lo.x - pad && p.x <= hi.x + pad && p.y >= lo.y - pad && p.y <= hi.y + pad;
  }
  double diag() const { return len2(sub(hi, lo)); }
};
// squared point-box distance, vec.hpp:92-96
inline double box_d2(const Box& b, V2 p) {
  double dx = std::max({b.lo.x - p.x, 0.0, p.x - b.hi.x});
  double dy = std::max({b.lo.y - p.y, 0.0, p.y - b.hi.y});
  return dx * dx + dy * dy;
}

// ---------------------------------------------------------------- PCG32
// proj/include/wost/rng.hpp:9-78: 64-bit LCG, xorshift-rotate output,
// per-walk stream from a splitmix64-style finaliser
struct Pcg {
  uint64_t s = 0, inc = 1;
  Pcg() : Pcg(0x853c49e6748fea9bULL, 0xda3e39cb94b95bdbULL) {}
  Pcg(uint64_t seed, uint64_t stream) {
    s = 0;
    inc = (stream << 1u) | 1u;
    u32();
    s += seed;
    u32();
  }
  static uint64_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  static Pcg walk(uint64_t seed, uint64_t point, uint64_t wpp) {
    uint64_t a = mix(seed ^ mix(point));
    uint64_t b = mix(a ^ mix(wpp + 0x632be59bd9b4e019ULL));
    return Pcg(a, b);
  }
  uint32_t u32() {
    uint64_t old = s;
    s = old * 6364136223846793005ULL + inc;
    uint32_t xs = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
    uint32_t rot = static_cast<uint32_t>(old >> 59u);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
  }
  uint64_t u64() {
    uint64_t hi = u32();
    return (hi << 32) | u32();
  }
  double uni() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
  double uni_pos() {
    double u;
    do u = uni();
    while (u == 0.0);
    return u;
  }
  double uni(double lo, double hi) { return lo + (hi - lo) * uni(); }
  uint32_t index(uint32_t n) {  // Lemire rejection, rng.hpp:61-73
    uint64_t m = static_cast<uint64_t>(u32()) * n;
    uint32_t lo = static_cast<uint32_t>(m);
    if (lo < n) {
      uint32_t t = (0u - n) % n;
      while (lo < t) {
        m = static_cast<uint64_t>(u32()) * n;
        lo = static_cast<uint32_t>(m);
      }
    }
    return static_cast<uint32_t>(m >> 32);
  }
};

// ---------------------------------------------------------------- scene
// proj/src/scene.cpp:13-101
struct Value {
  wg_value_spec spec{};
  std::vector<double> raster;
  double eval(V2 p) const {
    switch (spec.type) {
      case WG_VALUE_CONSTANT: return spec.c0;
      case WG_VALUE_LINEAR: return spec.c0 + spec.cx * p.x + spec.cy * p.y;
      case WG_VALUE_RASTER: {  // RasterGrid::at, scene.cpp:13-20
        double ex = spec.raster_bbox[2] - spec.raster_bbox[0];
        double ey = spec.raster_bbox[3] - spec.raster_bbox[1];
        double u = (p.x - spec.raster_bbox[0]) / ex;
        double v = (p.y - spec.raster_bbox[1]) / ey;
        int i = std::clamp(static_cast<int>(u * spec.raster_w), 0, spec.raster_w - 1);
        int j = std::clamp(static_cast<int>(v * spec.raster_h), 0, spec.raster_h - 1);
        return raster[static_cast<size_t>(j) * spec.raster_w + i];
      }
      case WG_VALUE_ANALYTIC:
        if (spec.analytic_id == WG_ANALYTIC_X2_MINUS_Y2) return p.x * p.x - p.y * p.y;
        return p.x * p.x + p.y * p.y - 1.0;
      default: return 0.0;
    }
  }
};

struct Seg {
  V2 a, b;
  int kind;  // WG_DIRICHLET / WG_NEUMANN
  int id;
};

struct Node {
  Box box;
  int left = -1, right = -1, begin = 0, end = 0;
};

struct SilVertex {
  V2 pos;
  std::vector<V2> normals;
};

struct Scene {
  Box bbox;
  double eps = 0;
  std::vector<Value> values;
  Value source;  // type WG_VALUE_ZERO for none
  std::vector<Seg> input;  // scene order
  std::vector<int> value_index;
  // Accel (proj/src/geom2d.cpp:80-140)
  std::vector<Seg> segs;  // BVH leaf order
  std::vector<Node> nodes;
  std::vector<SilVertex> sil;
  double t_eps = 0;

  double dirichlet(V2 p, int seg) const {
    if (input[seg].kind != WG_DIRICHLET) throw SceneErr("eval_dirichlet: not Dirichlet");
    return values[value_index[seg]].eval(p);
  }
  double neumann(V2 p, int seg) const {
    if (input[seg].kind != WG_NEUMANN) throw SceneErr("eval_neumann: not Neumann");
    return values[value_index[seg]].eval(p);
  }
  double source_at(V2 p) const {  // scene.cpp:55-69, zero outside bbox
    if (!bbox.contains(p, 0.0)) return 0.0;
    if (source.spec.type == WG_VALUE_ZERO) return 0.0;
    return source.eval(p);
  }
  bool source_zero() const { return source.spec.type == WG_VALUE_ZERO; }
  bool neumann_flux() const {  // scene.cpp:83-91
    for (size_t i = 0; i < input.size(); ++i) {
      if (input[i].kind != WG_NEUMANN) continue;
      const wg_value_spec& v = values[value_index[i]].spec;
      if (v.type != WG_VALUE_CONSTANT || v.c0 != 0.0) return true;
    }
    return false;
  }

  int build(int begin, int end) {  // median split, geom2d.cpp:109-140
    Node node;
    for (int i = begin; i < end; ++i) {
      node.box.grow(segs[i].a);
      node.box.grow(segs[i].b);
    }
    int idx = static_cast<int>(nodes.size());
    nodes.push_back(node);
    if (end - begin <= 4) {  // kLeafSize, geom2d.cpp:18
      nodes[idx].begin = begin;
      nodes[idx].end = end;
      return idx;
    }
    V2 ext = sub(node.box.hi, node.box.lo);
    bool sx = ext.x >= ext.y;
    int mid = (begin + end) / 2;
    std::nth_element(segs.begin() + begin, segs.begin() + mid, segs.begin() + end,
                     [sx](const Seg& p, const Seg& q) {
                       double cp = sx ? p.a.x + p.b.x : p.a.y + p.b.y;
                       double cq = sx ? q.a.x + q.b.x : q.a.y + q.b.y;
                       if (cp != cq) return cp < cq;
                       return p.id < q.id;
                     });
    int l = build(begin, mid);
    int r = build(mid, end);
    nodes[idx].left = l;
    nodes[idx].right = r;
    return idx;
  }

  void build_accel() {
    if (input.empty()) throw SceneErr("build_accel: scene has no segments");
    segs = input;
    nodes.clear();
    build(0, static_cast<int>(segs.size()));
    t_eps = 1e-6 * nodes[0].box.diag();
    // Neumann vertex adjacency keyed by exact coordinates, geom2d.cpp:93-106
    std::map<std::pair<uint64_t, uint64_t>, int> key;
    for (const Seg& s : segs) {
      if (s.kind != WG_NEUMANN) continue;
      V2 d = sub(s.b, s.a);
      V2 perp{-d.y, d.x};
      double l = len2(perp);
      V2 n{perp.x / l, perp.y / l};
      for (V2 p : {s.a, s.b}) {
        uint64_t kx, ky;
        std::memcpy(&kx, &p.x, 8);
        std::memcpy(&ky, &p.y, 8);
        auto it = key.find({kx, ky});
        int vi;
        if (it == key.end()) {
          vi = static_cast<int>(sil.size());
          key[{kx, ky}] = vi;
          sil.push_back({p, {}});
        } else {
          vi = it->second;
        }
        sil[vi].normals.push_back(n);
      }
    }
  }
};

// closest point on segment, geom2d.cpp:9-14
inline V2 closest_on_seg(V2 x, V2 a, V2 b) {
  V2 u = sub(b, a);
  double t = dot2(sub(x, a), u) / dot2(u, u);
  t = std::clamp(t, 0.0, 1.0);
  return add(a, scl(u, t));
}

struct CP {
  V2 p;
  double d = kInf;
  int seg = -1;
};

// stack DFS with box pruning, nearer child first, strict < (geom2d.cpp:142-180)
CP closest_point(const Scene& s, V2 x, unsigned kinds) {
  CP best;
  double bd2 = kInf;
  int st[64], top = 0;
  st[top++] = 0;
  while (top > 0) {
    const Node& nd = s.nodes[st[--top]];
    if (box_d2(nd.box, x) >= bd2) continue;
    if (nd.left < 0) {
      for (int i = nd.begin; i < nd.end; ++i) {
        const Seg& g = s.segs[i];
        if (!((g.kind == WG_DIRICHLET ? 1u : 2u) & kinds)) continue;
        V2 p = closest_on_seg(x, g.a, g.b);
        V2 dd = sub(p, x);
        double d2 = dot2(dd, dd);
        if (d2 < bd2) {
          bd2 = d2;
          best.p = p;
          best.seg = g.id;
        }
      }
    } else {
      double dl = box_d2(s.nodes[nd.left].box, x);
      double dr = box_d2(s.nodes[nd.right].box, x);
      if (dl <= dr) {
        if (dr < bd2) st[top++] = nd.right;
        if (dl < bd2) st[top++] = nd.left;
      } else {
        if (dl < bd2) st[top++] = nd.left;
        if (dr < bd2) st[top++] = nd.right;
      }
    }
  }
  if (best.seg >= 0) best.d = std::sqrt(bd2);
  return best;
}

// linear scan over Neumann vertices, facing flip test (geom2d.cpp:182-200)
double closest_silhouette(const Scene& s, V2 x) {
  double best = kInf;
  for (const SilVertex& v : s.sil) {
    double d = len2(sub(v.pos, x));
    if (d >= best) continue;
    bool cand = v.normals.size() < 2;
    if (!cand) {
      double lo = kInf, hi = -kInf;
      for (V2 n : v.normals) {
        double f = dot2(n, sub(v.pos, x));
        lo = std::min(lo, f);
        hi = std::max(hi, f);
      }
      cand = lo * hi <= 0.0;
    }
    if (cand) best = d;
  }
  return best;
}

// geom2d.cpp:41-51
inline double ray_seg(V2 o, V2 dir, V2 a, V2 b, double* s_out) {
  V2 u = sub(b, a);
  V2 w = sub(a, o);
  double den = cross2(dir, u);
  if (den == 0.0) return kInf;
  double t = cross2(w, u) / den;
  double sp = cross2(w, dir) / den;
  if (sp < 0.0 || sp > 1.0) return kInf;
  *s_out = sp;
  return t;
}

// slab test without NaNs on axis-parallel rays, geom2d.cpp:55-76
inline bool ray_box(V2 o, V2 dir, V2 inv, const Box& b, double t_max) {
  double t0 = 0.0, t1 = t_max;
  if (dir.x != 0.0) {
    double a = (b.lo.x - o.x) * inv.x, c = (b.hi.x - o.x) * inv.x;
    if (a > c) std::swap(a, c);
    t0 = std::max(t0, a);
    t1 = std::min(t1, c);
  } else if (o.x < b.lo.x || o.x > b.hi.x) {
    return false;
  }
  if (dir.y != 0.0) {
    double a = (b.lo.y - o.y) * inv.y, c = (b.hi.y - o.y) * inv.y;
    if (a > c) std::swap(a, c);
    t0 = std::max(t0, a);
    t1 = std::min(t1, c);
  } else if (o.y < b.lo.y || o.y > b.hi.y) {
    return false;
  }
  return t1 >= t0;
}

struct Hit {
  bool ok = false;
  double t = kInf;
  V2 p, n;
  int seg = -1, kind = -1;
};

// nearest hit in (t_eps, t_max], last equal t wins (geom2d.cpp:202-246)
Hit ray_first_hit(const Scene& s, V2 o, V2 dir, double t_max, unsigned kinds, int exclude) {
  V2 inv{1.0 / dir.x, 1.0 / dir.y};
  double bt = t_max;
  const Seg* bs = nullptr;
  double bsp = 0.0;
  int st[64], top = 0;
  st[top++] = 0;
  while (top > 0) {
    const Node& nd = s.nodes[st[--top]];
    if (!ray_box(o, dir, inv, nd.box, bt)) continue;
    if (nd.left < 0) {
      for (int i = nd.begin; i < nd.end; ++i) {
        const Seg& g = s.segs[i];
        if (!((g.kind == WG_DIRICHLET ? 1u : 2u) & kinds)) continue;
        if (g.id == exclude) continue;
        double sp;
        double t = ray_seg(o, dir, g.a, g.b, &sp);
        if (t > s.t_eps && t <= bt) {
          bt = t;
          bs = &g;
          bsp = sp;
        }
      }
    } else {
      st[top++] = nd.right;
      st[top++] = nd.left;
    }
  }
  Hit h;
  if (!bs) return h;
  h.ok = true;
  h.t = bt;
  h.p = add(bs->a, scl(sub(bs->b, bs->a), bsp));
  V2 d = sub(bs->b, bs->a);
  V2 perp{-d.y, d.x};
  double l = len2(perp);
  V2 n{perp.x / l, perp.y / l};
  if (dot2(n, dir) > 0.0) n = {-n.x, -n.y};
  h.n = n;
  h.seg = bs->id;
  h.kind = bs->kind;
  return h;
}

// geom2d.cpp:248-255
double star_radius(const Scene& s, V2 x, double r_min) {
  double dd = closest_point(s, x, WG_KIND_DIRICHLET).d;
  double ds = closest_silhouette(s, x);
  if (dd == kInf && ds == kInf) throw SceneErr("star_radius: unbounded star region");
  return std::min(dd, std::max(ds, r_min));
}

// ---------------------------------------------------------------- sphdist
// proj/src/sphdist.cpp:10-78: I0/I1 by power series below 20, Hankel
// asymptotic expansion above
double i0_series(double x) {
  double q = 0.25 * x * x, term = 1.0, sum = 1.0;
  for (int m = 1; m < 200; ++m) {
    term *= q * (1.0 / (static_cast<double>(m) * m));
    sum += term;
    if (term < 1e-17 * sum) break;
  }
  return sum;
}
double i1_series(double x) {
  double q = 0.25 * x * x, term = 0.5 * x, sum = term;
  for (int m = 1; m < 200; ++m) {
    term *= q * (1.0 / (static_cast<double>(m) * (m + 1)));
    sum += term;
    if (term < 1e-17 * sum) break;
  }
  return sum;
}
double asym_corr(double x, double mu) {
  double sum = 1.0, term = 1.0, prev = kInf;
  for (int k = 1; k < 30; ++k) {
    term *= -(mu - (2.0 * k - 1.0) * (2.0 * k - 1.0)) / (8.0 * x * k);
    if (std::abs(term) >= prev) break;
    sum += term;
    prev = std::abs(term);
    if (std::abs(term) < 1e-16 * std::abs(sum)) break;
  }
  return sum;
}
double bessel_i0(double x) {
  if (x < 20.0) return i0_series(x);
  return std::exp(x) / std::sqrt(kTwoPi * x) * asym_corr(x, 0.0);
}
double log_bessel_i0(double x) {
  if (x < 20.0) return std::log(i0_series(x));
  return x - 0.5 * std::log(kTwoPi * x) + std::log(asym_corr(x, 0.0));
}
double bessel_i1_over_i0(double x) {
  if (x == 0.0) return 0.0;
  if (x < 20.0) return i1_series(x) / i0_series(x);
  return asym_corr(x, 4.0) / asym_corr(x, 0.0);
}

struct Comp {
  V3 mu{1, 0, 0};
  double kappa = 0, lambda = 1;
};
struct Mix {
  Comp c[kMaxK];
  int k = 1, dim = 2;
  double sel = 0.5;
  double log_a[kMaxK] = {};
};

double sphere_area(int dim) { return dim == 2 ? kTwoPi : kFourPi; }

double vmf_pdf(V3 nu, const Comp& c, int dim) {  // sphdist.cpp:82-92
  if (c.kappa == 0.0) return 1.0 / sphere_area(dim);
  double t = dot3(nu, c.mu);
  if (dim == 2) return std::exp(c.kappa * t - log_bessel_i0(c.kappa)) / kTwoPi;
  double k = c.kappa;
  return k * std::exp(k * (t - 1.0)) / (kTwoPi * (1.0 - std::exp(-2.0 * k)));
}

// Best-Fisher rejection sampler, sphdist.cpp:111-128
double vm_angle(Pcg& rng, double kappa) {
  double tau = 1.0 + std::sqrt(1.0 + 4.0 * kappa * kappa);
  double rho = (tau - std::sqrt(2.0 * tau)) / (2.0 * kappa);
  double r = (1.0 + rho * rho) / (2.0 * rho);
  for (;;) {
    double u1 = rng.uni_pos();
    double z = std::cos(kPi * u1);
    double f = (1.0 + r * z) / (r + z);
    double cv = kappa * (r - f);
    double u2 = rng.uni_pos();
    if (cv * (2.0 - cv) - u2 > 0.0 || std::log(cv / u2) + 1.0 - cv >= 0.0) {
      double u3 = rng.uni();
      double th = std::acos(std::clamp(f, -1.0, 1.0));
      return u3 < 0.5 ? -th : th;
    }
  }
}

inline V3 rot2(double c, double s, V3 mu) {  // sphdist.cpp:97-99
  return {c * mu.x - s * mu.y, c * mu.y + s * mu.x, 0.0};
}

V3 vmf_sample(Pcg& rng, const Comp& c, int dim) {  // sphdist.cpp:132-158
  if (dim == 2) {
    if (c.kappa == 0.0) {
      double a = kTwoPi * rng.uni();
      return rot2(std::cos(a), std::sin(a), c.mu);
    }
    double th = vm_angle(rng, c.kappa);
    return rot2(std::cos(th), std::sin(th), c.mu);
  }
  double k = c.kappa, ct;
  if (k == 0.0) {
    ct = 1.0 - 2.0 * rng.uni();
  } else {
    double u = rng.uni_pos();
    ct = 1.0 + std::log(u + (1.0 - u) * std::exp(-2.0 * k)) / k;
    ct = std::clamp(ct, -1.0, 1.0);
  }
  double st = std::sqrt(std::max(0.0, 1.0 - ct * ct));
  double phi = kTwoPi * rng.uni();
  V3 w = c.mu;
  double sg = std::copysign(1.0, w.z);  // Duff et al. basis, sphdist.cpp:101-108
  double a = -1.0 / (sg + w.z);
  double b = w.x * w.y * a;
  V3 ua{1.0 + sg * w.x * w.x * a, sg * b, -sg * w.x};
  V3 va{b, sg + w.y * w.y * a, -w.y};
  return add3(add3(scl3(ua, st * std::cos(phi)), scl3(va, st * std::sin(phi))), scl3(w, ct));
}

double comp_log_norm(double kappa, int dim) {  // sphdist.cpp:162-167
  if (dim == 2) return -log_bessel_i0(kappa) - std::log(kTwoPi);
  if (kappa == 0.0) return -std::log(kFourPi);
  return std::log(kappa) - kappa - std::log(kTwoPi * (1.0 - std::exp(-2.0 * kappa)));
}

double mixture_pdf(V3 nu, const Mix& m) {  // sphdist.cpp:176-185
  double sum = 0.0;
  for (int i = 0; i < m.k; ++i) {
    const Comp& c = m.c[i];
    double la = m.log_a[i];
    sum += la != 0.0 ? c.lambda * std::exp(c.kappa * dot3(nu, c.mu) + la)
                     : c.lambda * vmf_pdf(nu, c, m.dim);
  }
  return sum;
}

V3 mixture_sample(Pcg& rng, const Mix& m) {  // sphdist.cpp:187-202
  int pick = 0;
  if (m.k > 1) {
    double u = rng.uni(), acc = 0.0;
    pick = m.k - 1;
    for (int i = 0; i < m.k; ++i) {
      acc += m.c[i].lambda;
      if (u < acc) {
        pick = i;
        break;
      }
    }
  }
  return vmf_sample(rng, m.c[pick], m.dim);
}

inline V3 reflect(V3 nu, V3 n) { return sub3(nu, scl3(n, 2.0 * dot3(nu, n))); }

double reflected_pdf(V3 nu, const Mix& m, V3 n) {  // sphdist.cpp:204-208
  if (dot3(nu, n) <= 0.0) return 0.0;
  return mixture_pdf(nu, m) + mixture_pdf(reflect(nu, n), m);
}

V3 reflected_sample(Pcg& rng, const Mix& m, V3 n) {  // sphdist.cpp:210-218
  for (;;) {
    V3 nu = mixture_sample(rng, m);
    double d = dot3(nu, n);
    if (d < 0.0) return reflect(nu, n);
    if (d > 0.0) return nu;
  }
}

double uniform_pdf(V3 nu, const V3* n, int dim) {  // sphdist.cpp:220-224
  double inv = 1.0 / sphere_area(dim);
  if (!n) return inv;
  return dot3(nu, *n) > 0.0 ? 2.0 * inv : 0.0;
}

V3 uniform_sample(Pcg& rng, const V3* n, int dim) {  // sphdist.cpp:226-243
  for (;;) {
    V3 nu;
    if (dim == 2) {
      double a = kTwoPi * rng.uni();
      nu = {std::cos(a), std::sin(a), 0.0};
    } else {
      double z = 1.0 - 2.0 * rng.uni();
      double s = std::sqrt(std::max(0.0, 1.0 - z * z));
      double a = kTwoPi * rng.uni();
      nu = {s * std::cos(a), s * std::sin(a), z};
    }
    if (!n) return nu;
    double d = dot3(nu, *n);
    if (d > 0.0) return nu;
    if (d < 0.0) return {-nu.x, -nu.y, -nu.z};
  }
}

double guided_pdf(V3 nu, const Mix& m, const V3* n, bool reflect_on) {
  return n ? (reflect_on ? reflected_pdf(nu, m, *n) : mixture_pdf(nu, m)) : mixture_pdf(nu, m);
}

double mis_pdf(V3 nu, const Mix& m, const V3* n, bool reflect_on) {  // :245-252
  double pg = guided_pdf(nu, m, n, reflect_on);
  double pu = uniform_pdf(nu, n, m.dim);
  return m.sel * pg + (1.0 - m.sel) * pu;
}

struct MisOut {
  V3 nu;
  double pmis = 0, pg = 0, pu = 0;
};

MisOut mis_sample(Pcg& rng, const Mix& m, const V3* n, bool reflect_on) {  // :254-270
  MisOut o;
  bool guided = rng.uni() < m.sel;
  if (guided)
    o.nu = n && reflect_on ? reflected_sample(rng, m, *n) : mixture_sample(rng, m);
  else
    o.nu = uniform_sample(rng, n, m.dim);
  o.pg = guided_pdf(o.nu, m, n, reflect_on);
  o.pu = uniform_pdf(o.nu, n, m.dim);
  o.pmis = m.sel * o.pg + (1.0 - m.sel) * o.pu;
  return o;
}

struct Raw {  // UnnormParams, sphdist.hpp:44-54
  double mu[kMaxK][3] = {};
  double kappa[kMaxK] = {};
  double lam[kMaxK] = {};
  double c = 0;
  int k = 1, dim = 2;
};

Raw unpack(const double* r, int k, int dim) {  // guide_field.cpp:424-441
  Raw p;
  p.k = k;
  p.dim = dim;
  const double* m = r;
  for (int i = 0; i < k; ++i) {
    p.mu[i][0] = m[0];
    p.mu[i][1] = m[1];
    p.mu[i][2] = dim == 3 ? m[2] : 0.0;
    m += dim;
  }
  for (int i = 0; i < k; ++i) p.kappa[i] = m[i];
  m += k;
  for (int i = 0; i < k; ++i) p.lam[i] = m[i];
  m += k;
  p.c = m[0];
  return p;
}

double sigmoid(double x) {
  return x >= 0.0 ? 1.0 / (1.0 + std::exp(-x)) : std::exp(x) / (1.0 + std::exp(x));
}

Mix normalize(const Raw& r) {  // Table-1 mappings, sphdist.cpp:287-310
  Mix o;
  o.k = r.k;
  o.dim = r.dim;
  o.sel = sigmoid(r.c);
  double mx = -kInf;
  for (int i = 0; i < r.k; ++i) mx = std::max(mx, r.lam[i]);
  double z = 0.0;
  for (int i = 0; i < r.k; ++i) z += std::exp(r.lam[i] - mx);
  for (int i = 0; i < r.k; ++i) {
    V3 m{r.mu[i][0], r.mu[i][1], r.dim == 3 ? r.mu[i][2] : 0.0};
    double mn = len3(m);
    if (mn < 1e-12) {
      double a = kTwoPi * i / kMaxK;
      o.c[i].mu = {std::cos(a), std::sin(a), 0.0};
    } else {
      o.c[i].mu = {m.x / mn, m.y / mn, m.z / mn};
    }
    o.c[i].kappa = std::clamp(std::exp(r.kappa[i]), kKappaMin, kKappaMax);
    o.c[i].lambda = std::exp(r.lam[i] - mx) / z;
  }
  for (int i = 0; i < o.k; ++i) o.log_a[i] = comp_log_norm(o.c[i].kappa, o.dim);
  return o;
}

struct Grad {  // ParamGrad, sphdist.hpp:57-80
  double mu[kMaxK][3] = {};
  double kappa[kMaxK] = {};
  double lam[kMaxK] = {};
  double c = 0;
};

double dlogv_dkappa(double t, double kappa, int dim) {  // sphdist.cpp:315-321
  if (dim == 2) return t - bessel_i1_over_i0(kappa);
  double e = std::expm1(-2.0 * kappa);
  double coth = 1.0 - 2.0 * (e + 1.0) / e;
  return 1.0 / kappa + t - coth;
}

// dV/dTheta' for one direction, sphdist.cpp:324-366
double mix_grad_one(V3 nu, const Raw& raw, const Mix& m, Grad& g) {
  const int k = raw.k;
  double v[kMaxK];
  double val = 0.0;
  for (int i = 0; i < k; ++i) {
    const Comp& c = m.c[i];
    double la = m.log_a[i];
    v[i] = la != 0.0 ? std::exp(c.kappa * dot3(nu, c.mu) + la) : vmf_pdf(nu, c, raw.dim);
    val += c.lambda * v[i];
  }
  for (int i = 0; i < k; ++i) g.lam[i] += m.c[i].lambda * (v[i] - val);
  for (int i = 0; i < k; ++i) {
    const Comp& c = m.c[i];
    double t = dot3(nu, c.mu);
    double lv = c.lambda * v[i];
    double ku = std::exp(raw.kappa[i]);
    if (ku > kKappaMin && ku < kKappaMax)
      g.kappa[i] += lv * dlogv_dkappa(t, c.kappa, raw.dim) * c.kappa;
    V3 mm{raw.mu[i][0], raw.mu[i][1], raw.dim == 3 ? raw.mu[i][2] : 0.0};
    double mn = len3(mm);
    if (mn >= 1e-12) {
      V3 dmu = scl3(sub3(nu, scl3(c.mu, t)), lv * c.kappa / mn);
      g.mu[i][0] += dmu.x;
      g.mu[i][1] += dmu.y;
      if (raw.dim == 3) g.mu[i][2] += dmu.z;
    }
  }
  return val;
}

// ---------------------------------------------------------------- field
// proj/src/guide_field.cpp: dense multiresolution grid + 3-layer ReLU MLP
struct Field {
  wg_field_config cfg{};
  Box bbox;
  std::vector<float> p;
  std::vector<double> m, v;
  int64_t steps = 0;
  std::vector<size_t> lvl_off;
  size_t w1 = 0, b1 = 0, w2 = 0, b2 = 0, w3 = 0, b3 = 0;

  int in_dim() const { return cfg.n_levels * cfg.features; }
  int out_dim() const { return (2 + cfg.mixture_dim) * cfg.mixture_k + 1; }

  void offsets() {  // guide_field.cpp:57-78
    size_t off = 0;
    lvl_off.clear();
    for (int l = 0; l < cfg.n_levels; ++l) {
      lvl_off.push_back(off);
      off += static_cast<size_t>(cfg.level_res[l]) * cfg.level_res[l] * cfg.features;
    }
    int in = in_dim(), hid = cfg.hidden, od = out_dim();
    w1 = off;
    off += static_cast<size_t>(in) * hid;
    b1 = off;
    off += hid;
    w2 = off;
    off += static_cast<size_t>(hid) * hid;
    b2 = off;
    off += hid;
    w3 = off;
    off += static_cast<size_t>(hid) * od;
    b3 = off;
    off += od;
    p.assign(off, 0.0f);
  }

  Field(const wg_field_config& c, const Box& b, uint64_t seed) : cfg(c), bbox(b) {
    // validation, guide_field.cpp:16-32
    if (cfg.n_levels < 1 || cfg.features < 1 || cfg.mixture_k < 1)
      throw std::invalid_argument("guiding field: L, F and K must be >= 1");
    if (cfg.mixture_k > kMaxK) throw std::invalid_argument("guiding field: K exceeds cap");
    if (cfg.mixture_dim != 2 && cfg.mixture_dim != 3)
      throw std::invalid_argument("guiding field: mixture dim must be 2 or 3");
    if (cfg.hidden < 1) throw std::invalid_argument("guiding field: hidden >= 1");
    for (int l = 0; l < cfg.n_levels; ++l)
      if (cfg.level_res[l] < 2) throw std::invalid_argument("guiding field: res >= 2");
    if (in_dim() > 256 || cfg.hidden > 256) throw std::invalid_argument("guiding field: cap 256");
    if (!(b.lo.x <= b.hi.x && b.lo.y <= b.hi.y) || b.hi.x - b.lo.x <= 0.0 || b.hi.y - b.lo.y <= 0.0)
      throw std::invalid_argument("guiding field: bbox is empty");
    offsets();
    // init stream, guide_field.cpp:36-51
    Pcg rng(Pcg::mix(seed), 0x67e5504410b1426fULL);
    for (size_t i = 0; i < w1; ++i) p[i] = static_cast<float>(rng.uni(-1e-4, 1e-4));
    auto layer = [&](size_t wo, size_t wc, size_t bo, size_t bc, int fan_in) {
      double sc = 1.0 / std::sqrt(static_cast<double>(fan_in));
      for (size_t i = 0; i < wc; ++i) p[wo + i] = static_cast<float>(rng.uni(-sc, sc));
      for (size_t i = 0; i < bc; ++i) p[bo + i] = 0.0f;
    };
    int in = in_dim(), hid = cfg.hidden, od = out_dim();
    layer(w1, static_cast<size_t>(in) * hid, b1, hid, in);
    layer(w2, static_cast<size_t>(hid) * hid, b2, hid, hid);
    layer(w3, static_cast<size_t>(hid) * od, b3, od, hid);
    m.assign(p.size(), 0.0);
    v.assign(p.size(), 0.0);
  }

  // fp32 sampling-path evaluation, guide_field.cpp:178-221
  void eval(V2 x, double* out) const {
    const int in = in_dim(), hid = cfg.hidden, od = out_dim(), f = cfg.features;
    float input[256], h1[256], h2[256], of[256];
    double ex = bbox.hi.x - bbox.lo.x, ey = bbox.hi.y - bbox.lo.y;
    float u = static_cast<float>(std::clamp((x.x - bbox.lo.x) / ex, 0.0, 1.0));
    float vv = static_cast<float>(std::clamp((x.y - bbox.lo.y) / ey, 0.0, 1.0));
    for (int l = 0; l < cfg.n_levels; ++l) {
      int res = cfg.level_res[l];
      float px = u * (res - 1), py = vv * (res - 1);
      int ix = std::min(static_cast<int>(px), res - 2);
      int iy = std::min(static_cast<int>(py), res - 2);
      float fx = px - ix, fy = py - iy;
      const float* base = p.data() + lvl_off[l] + (static_cast<size_t>(iy) * res + ix) * f;
      const float* up = base + static_cast<size_t>(res) * f;
      float w00 = (1.0f - fx) * (1.0f - fy), w10 = fx * (1.0f - fy);
      float w01 = (1.0f - fx) * fy, w11 = fx * fy;
      for (int i = 0; i < f; ++i)
        input[l * f + i] = (w00 * base[i] + w10 * base[f + i]) + (w01 * up[i] + w11 * up[f + i]);
    }
    affine_f(input, in, w1, b1, hid, h1, true);
    affine_f(h1, hid, w2, b2, hid, h2, true);
    affine_f(h2, hid, w3, b3, od, of, false);
    for (int j = 0; j < od; ++j) out[j] = of[j];
  }
  // 4-way unrolled fixed-order accumulation, guide_field.cpp:149-170
  void affine_f(const float* x, int rows, size_t wo, size_t bo, int cols, float* y, bool relu) const {
    const float* w = p.data() + wo;
    for (int j = 0; j < cols; ++j) y[j] = p[bo + j];
    int i = 0;
    for (; i + 4 <= rows; i += 4) {
      const float *r0 = w + static_cast<size_t>(i) * cols, *r1 = r0 + cols, *r2 = r1 + cols,
                  *r3 = r2 + cols;
      for (int j = 0; j < cols; ++j)
        y[j] += (x[i] * r0[j] + x[i + 1] * r1[j]) + (x[i + 2] * r2[j] + x[i + 3] * r3[j]);
    }
    for (; i < rows; ++i) {
      const float* r = w + static_cast<size_t>(i) * cols;
      for (int j = 0; j < cols; ++j) y[j] += x[i] * r[j];
    }
    if (relu)
      for (int j = 0; j < cols; ++j) y[j] = y[j] > 0.0f ? y[j] : 0.0f;
  }

  struct Tape {
    size_t ci[4 * WG_MAX_LEVELS];
    double cw[4 * WG_MAX_LEVELS];
    double in[256], h1p[256], h1[256], h2p[256], h2[256];
  };
  // fp64 forward keeping activations, guide_field.cpp:80-123, 223-243
  void eval_tape(V2 x, double* out, Tape& t) const {
    const int in = in_dim(), hid = cfg.hidden, od = out_dim(), f = cfg.features;
    double ex = bbox.hi.x - bbox.lo.x, ey = bbox.hi.y - bbox.lo.y;
    double u = std::clamp((x.x - bbox.lo.x) / ex, 0.0, 1.0);
    double vv = std::clamp((x.y - bbox.lo.y) / ey, 0.0, 1.0);
    for (int l = 0; l < cfg.n_levels; ++l) {
      int res = cfg.level_res[l];
      double px = u * (res - 1), py = vv * (res - 1);
      int ix = std::min(static_cast<int>(px), res - 2);
      int iy = std::min(static_cast<int>(py), res - 2);
      double fx = px - ix, fy = py - iy;
      size_t c00 = lvl_off[l] + (static_cast<size_t>(iy) * res + ix) * f;
      size_t c10 = c00 + f, c01 = c00 + static_cast<size_t>(res) * f, c11 = c01 + f;
      double w00 = (1.0 - fx) * (1.0 - fy), w10 = fx * (1.0 - fy), w01 = (1.0 - fx) * fy,
             w11 = fx * fy;
      t.ci[4 * l] = c00;
      t.ci[4 * l + 1] = c10;
      t.ci[4 * l + 2] = c01;
      t.ci[4 * l + 3] = c11;
      t.cw[4 * l] = w00;
      t.cw[4 * l + 1] = w10;
      t.cw[4 * l + 2] = w01;
      t.cw[4 * l + 3] = w11;
      for (int i = 0; i < f; ++i)
        t.in[l * f + i] = w00 * p[c00 + i] + w10 * p[c10 + i] + w01 * p[c01 + i] + w11 * p[c11 + i];
    }
    affine_d(t.in, in, w1, b1, hid, t.h1p);
    for (int i = 0; i < hid; ++i) t.h1[i] = t.h1p[i] > 0.0 ? t.h1p[i] : 0.0;
    affine_d(t.h1, hid, w2, b2, hid, t.h2p);
    for (int i = 0; i < hid; ++i) t.h2[i] = t.h2p[i] > 0.0 ? t.h2p[i] : 0.0;
    affine_d(t.h2, hid, w3, b3, od, out);
  }
  // 2-way unrolled fixed-order accumulation, guide_field.cpp:129-145
  void affine_d(const double* x, int rows, size_t wo, size_t bo, int cols, double* y) const {
    const float* w = p.data() + wo;
    for (int j = 0; j < cols; ++j) y[j] = p[bo + j];
    int i = 0;
    for (; i + 2 <= rows; i += 2) {
      const float* r0 = w + static_cast<size_t>(i) * cols;
      const float* r1 = r0 + cols;
      for (int j = 0; j < cols; ++j) y[j] += x[i] * r0[j] + x[i + 1] * r1[j];
    }
    for (; i < rows; ++i) {
      const float* r = w + static_cast<size_t>(i) * cols;
      for (int j = 0; j < cols; ++j) y[j] += x[i] * r[j];
    }
  }
  // reverse pass, guide_field.cpp:258-315
  void backward(const Tape& t, const double* dout, std::vector<double>& g) const {
    const int in = in_dim(), hid = cfg.hidden, od = out_dim(), f = cfg.features;
    double dh2[256], dh1[256], din[256];
    for (int j = 0; j < od; ++j) g[b3 + j] += dout[j];
    for (int i = 0; i < hid; ++i) {
      double acc = 0.0;
      for (int j = 0; j < od; ++j) {
        g[w3 + static_cast<size_t>(i) * od + j] += t.h2[i] * dout[j];
        acc += p[w3 + static_cast<size_t>(i) * od + j] * dout[j];
      }
      dh2[i] = t.h2p[i] > 0.0 ? acc : 0.0;
    }
    for (int j = 0; j < hid; ++j) g[b2 + j] += dh2[j];
    for (int i = 0; i < hid; ++i) {
      double acc = 0.0;
      for (int j = 0; j < hid; ++j) {
        g[w2 + static_cast<size_t>(i) * hid + j] += t.h1[i] * dh2[j];
        acc += p[w2 + static_cast<size_t>(i) * hid + j] * dh2[j];
      }
      dh1[i] = t.h1p[i] > 0.0 ? acc : 0.0;
    }
    for (int j = 0; j < hid; ++j) g[b1 + j] += dh1[j];
    for (int i = 0; i < in; ++i) {
      double acc = 0.0;
      for (int j = 0; j < hid; ++j) {
        g[w1 + static_cast<size_t>(i) * hid + j] += t.in[i] * dh1[j];
        acc += p[w1 + static_cast<size_t>(i) * hid + j] * dh1[j];
      }
      din[i] = acc;
    }
    for (int l = 0; l < cfg.n_levels; ++l)
      for (int c = 0; c < 4; ++c)
        for (int i = 0; i < f; ++i) g[t.ci[4 * l + c] + i] += t.cw[4 * l + c] * din[l * f + i];
  }
  // Adam with bias correction, fp64 moments, guide_field.cpp:317-331
  void adam(std::vector<double>& g, double lr, double b1_, double b2_, double eps) {
    ++steps;
    double bc1 = 1.0 - std::pow(b1_, static_cast<double>(steps));
    double bc2 = 1.0 - std::pow(b2_, static_cast<double>(steps));
    for (size_t i = 0; i < p.size(); ++i) {
      double gi = g[i];
      double mi = m[i] = b1_ * m[i] + (1.0 - b1_) * gi;
      double vi = v[i] = b2_ * v[i] + (1.0 - b2_) * gi * gi;
      double up = lr * (mi / bc1) / (std::sqrt(vi / bc2) + eps);
      p[i] = static_cast<float>(static_cast<double>(p[i]) - up);
      g[i] = 0.0;
    }
  }
};

// ---------------------------------------------------------------- training
struct Rec {  // GuideRecord, guide_train.hpp:14-25
  V2 x;
  V3 nu;
  double target = 0, pmis = 0, pg = 0, pu = 0, c = 0;
  bool on_n = false;
  V2 n;
};

// single-sample KL gradient (Eq. 13), guide_train.cpp:25-42
bool kl_grad(const Rec& r, const Raw& raw, bool refl, double v_floor, Grad& g, int64_t* skipped) {
  g = Grad{};
  if (r.target == 0.0) return true;
  Grad dv;
  Mix m = normalize(raw);
  double v;
  if (r.on_n && refl) {
    V3 n3{r.n.x, r.n.y, 0.0};
    v = mix_grad_one(r.nu, raw, m, dv);
    v += mix_grad_one(reflect(r.nu, n3), raw, m, dv);
  } else {
    v = mix_grad_one(r.nu, raw, m, dv);
  }
  if (!(v > v_floor)) {
    if (skipped) ++*skipped;
    return false;
  }
  double s = -r.target / (r.pmis * v);
  for (int i = 0; i < raw.k; ++i) {
    for (int a = 0; a < 3; ++a) g.mu[i][a] += s * dv.mu[i][a];
    g.kappa[i] += s * dv.kappa[i];
    g.lam[i] += s * dv.lam[i];
  }
  g.c += s * dv.c;
  return true;
}

// selection-probability gradient (Eq. 16), guide_train.cpp:44-56
double selection_grad(const Rec& r, const Mix& m, bool refl, double e) {
  V3 n3{r.n.x, r.n.y, 0.0};
  double pg = r.on_n ? (refl ? reflected_pdf(r.nu, m, n3) : mixture_pdf(r.nu, m)) : mixture_pdf(r.nu, m);
  double pu = r.pu;
  double pnow = m.sel * pg + (1.0 - m.sel) * pu;
  if (!(pnow > 0.0)) return 0.0;
  double dc = -e * r.target * (pg - pu) / (pnow * r.pmis);
  return dc * m.sel * (1.0 - m.sel);
}

// per-record gradient through the field into g (scaled by inv_count)
bool record_grad(const Field& f, const Rec& r, const wg_train_config& tc, double inv_count,
                 std::vector<double>& g, int64_t* skipped_v) {
  const int k = f.cfg.mixture_k, dim = f.cfg.mixture_dim, od = f.out_dim();
  Field::Tape t;
  double out[(2 + 3) * kMaxK + 1];
  f.eval_tape(r.x, out, t);
  Raw raw = unpack(out, k, dim);
  Grad pg;
  if (!kl_grad(r, raw, tc.reflect != 0, tc.v_floor, pg, skipped_v)) return false;
  pg.c = tc.learn_selection ? selection_grad(r, normalize(raw), tc.reflect != 0, tc.e_fraction) : 0.0;
  double dout[(2 + 3) * kMaxK + 1];
  double* m = dout;
  for (int i = 0; i < k; ++i)
    for (int a = 0; a < dim; ++a) *m++ = pg.mu[i][a] * inv_count;
  for (int i = 0; i < k; ++i) *m++ = pg.kappa[i] * inv_count;
  for (int i = 0; i < k; ++i) *m++ = pg.lam[i] * inv_count;
  *m = pg.c * inv_count;
  (void)od;
  f.backward(t, dout, g);
  return true;
}

// guide_train.cpp:94-198 (chunked reduction is summation-order bookkeeping;
// the oracle accumulates in record order, which is what one chunk does)
wg_train_stats train_batch(Field& f, const std::vector<Rec>& recs, const wg_train_config& tc,
                           uint64_t round) {
  wg_train_stats st{};
  st.records_seen = static_cast<int64_t>(recs.size());
  if (recs.empty()) return st;
  std::vector<uint32_t> order;
  for (uint32_t i = 0; i < recs.size(); ++i) {
    if (recs[i].pmis < tc.pdf_floor) {
      ++st.skipped_low_pdf;
      continue;
    }
    order.push_back(i);
  }
  Pcg rng(Pcg::mix(tc.seed) ^ Pcg::mix(round + 1), round);
  for (size_t i = order.size(); i > 1; --i)
    std::swap(order[i - 1], order[rng.index(static_cast<uint32_t>(i))]);
  if (order.size() > static_cast<size_t>(tc.max_records_per_round))
    order.resize(static_cast<size_t>(tc.max_records_per_round));
  if (order.empty()) return st;
  const size_t chunk = 2048;  // kGradChunk, guide_train.cpp:90
  std::vector<double> grad(f.p.size(), 0.0), cg(f.p.size(), 0.0);
  for (size_t b = 0; b < order.size(); b += tc.minibatch) {
    size_t e = std::min(b + static_cast<size_t>(tc.minibatch), order.size());
    double inv = 1.0 / static_cast<double>(e - b);
    for (size_t c0 = b; c0 < e; c0 += chunk) {
      size_t c1 = std::min(c0 + chunk, e);
      for (size_t r = c0; r < c1; ++r)
        if (record_grad(f, recs[order[r]], tc, inv, cg, &st.skipped_low_v)) ++st.records_consumed;
      for (size_t i = 0; i < grad.size(); ++i) {
        grad[i] += cg[i];
        cg[i] = 0.0;
      }
    }
    double n2 = 0.0;
    for (double g : grad) n2 += g * g;
    st.mean_grad_norm = (st.mean_grad_norm * st.steps + std::sqrt(n2)) / static_cast<double>(st.steps + 1);
    ++st.steps;
    f.adam(grad, tc.lr, tc.beta1, tc.beta2, tc.eps);
  }
  return st;
}

// ---------------------------------------------------------------- walks
// proj/src/wost.cpp
double greens_ball(double r, double R, int dim) {  // :27-31
  if (r <= 0.0) return kInf;
  if (dim == 2) return std::log(R / r) / kTwoPi;
  return (1.0 / r - 1.0 / R) / kFourPi;
}
double greens_mass(double R, int dim) { return dim == 2 ? R * R / 4.0 : R * R / 6.0; }

double greens_radius(double u, double R, int dim) {  // Newton + bisection, :37-65
  if (u <= 0.0) return 0.0;
  if (u >= 1.0) return R;
  double lo = 0.0, hi = 1.0, s = std::sqrt(u);
  for (int it = 0; it < 100; ++it) {
    double f, df;
    if (dim == 2) {
      f = s * s * (1.0 - 2.0 * std::log(s)) - u;
      df = -4.0 * s * std::log(s);
    } else {
      f = s * s * (3.0 - 2.0 * s) - u;
      df = 6.0 * s * (1.0 - s);
    }
    if (f > 0.0) hi = s;
    else lo = s;
    if (std::abs(f) < 1e-10) break;
    double step = df > 0.0 ? f / df : 0.0;
    double nx = s - step;
    if (!(nx > lo && nx < hi)) nx = 0.5 * (lo + hi);
    if (nx == s) break;
    s = nx;
  }
  return s * R;
}

struct Walk {
  V2 x;
  bool on_n = false;
  V2 n;
  int seg = -1;
  double T = 1.0, acc = 0.0, R = 0.0;
  int depth = 0;
  Pcg rng;
  bool alive = true, escaped = false;
  bool collect = false;
  double terminal = 0.0;
  struct Step {
    V2 x;
    V3 nu;
    double pmis = 0, pg = 0, pu = 0, c = 0;
    bool on_n = false;
    V2 n;
    double local = 0, mult = 0, rr = 1.0;
  };
  std::vector<Step> trace;
};

struct Ctx {
  const Scene* s = nullptr;
  const Field* f = nullptr;
  wg_solver_config cfg{};
  bool flux = false;
  double eps() const { return cfg.epsilon_shell > 0.0 ? cfg.epsilon_shell : s->eps; }
  double rmin() const { return cfg.r_min > 0.0 ? cfg.r_min : eps(); }
  bool guided() const { return cfg.mode != WG_MODE_UNIFORM; }
};

// begin_step, wost.cpp:148-216
bool begin_step(const Ctx& c, Walk& w) {
  if (!w.alive) return false;
  const Scene& s = *c.s;
  CP cd = closest_point(s, w.x, WG_KIND_DIRICHLET);
  if (cd.seg >= 0 && cd.d <= c.eps()) {
    double g = s.dirichlet(cd.p, cd.seg);
    w.acc += w.T * g;
    w.terminal = g;
    w.alive = false;
    return false;
  }
  if (w.depth >= c.cfg.max_steps) {
    w.alive = false;
    w.escaped = true;
    return false;
  }
  double rr = 1.0;
  if (w.depth > c.cfg.rr_depth) {
    double q = std::min(1.0, std::abs(w.T));
    if (q <= 0.0 || w.rng.uni() >= q) {
      w.terminal = 0.0;
      w.alive = false;
      return false;
    }
    w.T /= q;
    rr = 1.0 / q;
  }
  double dsil = closest_silhouette(s, w.x);
  double dd = cd.seg >= 0 ? cd.d : kInf;
  if (dd == kInf && dsil == kInf) throw SceneErr("walk: unbounded star region");
  double R = std::min(dd, std::max(dsil, c.rmin()));
  w.R = R;
  V3 n3{w.n.x, w.n.y, 0.0};
  const V3* np = w.on_n ? &n3 : nullptr;
  double contrib = 0.0;
  if (!s.source_zero()) {  // sample_source_point, wost.cpp:67-87
    V3 dir = uniform_sample(w.rng, np, 2);
    double r = greens_radius(w.rng.uni(), R, 2);
    V2 d2{dir.x, dir.y};
    V2 y = add(w.x, scl(d2, r));
    Hit h = ray_first_hit(s, w.x, d2, r, WG_KIND_ALL, -1);
    double wt = h.ok ? 0.0 : greens_mass(R, 2);
    if (wt != 0.0) contrib -= wt * s.source_at(y);
  }
  if (c.flux) {  // sample_neumann_contrib, wost.cpp:89-109
    V3 dir = uniform_sample(w.rng, np, 2);
    V2 d2{dir.x, dir.y};
    Hit h = ray_first_hit(s, w.x, d2, R, WG_KIND_NEUMANN, w.seg);
    double add_ = 0.0;
    if (h.ok) {
      double hv = s.neumann(h.p, h.seg);
      if (hv != 0.0) {
        double cz = std::abs(dot2(d2, h.n));
        if (c.cfg.clamp_grazing) cz = std::max(cz, c.cfg.grazing_floor);
        if (cz != 0.0) add_ = greens_ball(h.t, R, 2) * hv * h.t * kTwoPi / cz;
      }
    }
    contrib += add_;
  }
  w.acc += w.T * contrib;
  if (w.collect) {
    Walk::Step st;
    st.x = w.x;
    st.on_n = w.on_n;
    st.n = w.n;
    st.local = contrib;
    st.rr = rr;
    w.trace.push_back(st);
  }
  return true;
}

// decode + finish_step, wost.cpp:111-146, 218-264
void finish_step(const Ctx& c, Walk& w, const Mix* mp) {
  V3 n3{w.n.x, w.n.y, 0.0};
  const V3* np = w.on_n ? &n3 : nullptr;
  V3 nu;
  double pmis, pg, pu, sel;
  if (!mp) {
    nu = uniform_sample(w.rng, np, 2);
    pu = uniform_pdf(nu, np, 2);
    pmis = pu;
    pg = 0.0;
    sel = 0.0;
  } else {
    MisOut o = mis_sample(w.rng, *mp, np, c.cfg.reflect_at_neumann != 0);
    nu = o.nu;
    pmis = o.pmis;
    pg = o.pg;
    pu = o.pu;
    sel = mp->sel;
  }
  double mult = mp ? pu / pmis : 1.0;
  if (w.collect) {
    Walk::Step& st = w.trace.back();
    st.nu = nu;
    st.pmis = pmis;
    st.pg = pg;
    st.pu = pu;
    st.c = sel;
    st.mult = mult;
  }
  if (mult == 0.0) {
    w.terminal = 0.0;
    w.alive = false;
    return;
  }
  V2 d2{nu.x, nu.y};
  Hit h = ray_first_hit(*c.s, w.x, d2, w.R, WG_KIND_NEUMANN, w.seg);
  if (h.ok) {
    w.x = h.p;
    w.on_n = true;
    w.n = h.n;
    w.seg = h.seg;
  } else {
    w.x = add(w.x, scl(d2, w.R));
    w.on_n = false;
    w.seg = -1;
  }
  if (mp) w.T *= mult;
  ++w.depth;
  if (!c.s->bbox.contains(w.x, 1e-9 * c.s->bbox.diag())) {
    w.alive = false;
    w.escaped = true;
  }
}

Mix decode(const Ctx& c, V2 x) {  // decode_guiding, wost.cpp:111-122
  double out[(2 + 3) * kMaxK + 1];
  c.f->eval(x, out);
  Mix m = normalize(unpack(out, c.f->cfg.mixture_k, c.f->cfg.mixture_dim));
  if (c.cfg.mode == WG_MODE_GUIDING_ONLY) m.sel = 1.0;
  else if (c.cfg.mode == WG_MODE_FIXED_MIS) m.sel = c.cfg.fixed_c;
  return m;
}

// backfill_targets_append, guide_train.cpp:58-79
void backfill(const Walk& w, std::vector<Rec>& out) {
  size_t base = out.size();
  out.resize(base + w.trace.size());
  double un = w.terminal;
  for (size_t k = w.trace.size(); k-- > 0;) {
    const Walk::Step& s = w.trace[k];
    Rec& r = out[base + k];
    r.x = s.x;
    r.nu = s.nu;
    r.target = std::abs(un);
    r.pmis = s.pmis;
    r.pg = s.pg;
    r.pu = s.pu;
    r.c = s.c;
    r.on_n = s.on_n;
    r.n = s.n;
    un = s.rr * (s.local + s.mult * un);
  }
}

// wost_walk, wost.cpp:274-288 (solve_batch is bit-identical to it per walk,
// proj/tests/test_wost.cpp:436-482)
Walk run_walk(const Ctx& c, V2 x0, Pcg rng, bool collect) {
  Walk w;
  w.x = x0;
  w.rng = rng;
  w.collect = collect;
  while (w.alive) {
    if (!begin_step(c, w)) break;
    if (c.guided()) {
      Mix m = decode(c, w.x);
      finish_step(c, w, &m);
    } else {
      finish_step(c, w, nullptr);
    }
  }
  return w;
}

}  // namespace orc

// ============================================================== C-ABI
using namespace orc;

namespace {
thread_local std::string g_err;
template <class F>
int guarded(F&& f) {
  try {
    f();
    return WG_OK;
  } catch (const SceneErr& e) {
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
Mix from_wg(const wg_mixture* m) {
  Mix o;
  o.k = m->k;
  o.dim = m->dim;
  o.sel = m->c;
  for (int i = 0; i < m->k; ++i) {
    o.c[i].mu = {m->mu[i][0], m->mu[i][1], m->mu[i][2]};
    o.c[i].kappa = m->kappa[i];
    o.c[i].lambda = m->lambda[i];
    o.log_a[i] = m->log_a[i];
  }
  return o;
}
Rec from_wg(const wg_guide_record& r) {
  Rec o;
  o.x = {r.x[0], r.x[1]};
  o.nu = {r.nu[0], r.nu[1], r.nu[2]};
  o.target = r.target;
  o.pmis = r.pdf_mis;
  o.pg = r.pdf_g;
  o.pu = r.pdf_u;
  o.c = r.c;
  o.on_n = r.on_neumann != 0;
  o.n = {r.normal[0], r.normal[1]};
  return o;
}
}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

void* orc_scene_create(const double* seg, const int32_t* kind, const int32_t* value_index,
                       int32_t n_seg, const wg_value_spec* values, int32_t n_values,
                       const wg_value_spec* source, const double* bbox, double eps) {
  Scene* out = nullptr;
  int rc = guarded([&] {
    auto s = std::make_unique<Scene>();
    s->bbox.lo = {bbox[0], bbox[1]};
    s->bbox.hi = {bbox[2], bbox[3]};
    s->eps = eps > 0.0 ? eps : 1e-3;
    for (int i = 0; i < n_values; ++i) {
      Value v;
      v.spec = values[i];
      if (v.spec.type == WG_VALUE_RASTER)
        v.raster.assign(values[i].raster_data,
                        values[i].raster_data + (size_t)values[i].raster_w * values[i].raster_h);
      v.spec.raster_data = nullptr;
      s->values.push_back(std::move(v));
    }
    s->source.spec.type = WG_VALUE_ZERO;
    if (source && source->type != WG_VALUE_ZERO) {
      s->source.spec = *source;
      if (source->type == WG_VALUE_RASTER)
        s->source.raster.assign(source->raster_data,
                                source->raster_data + (size_t)source->raster_w * source->raster_h);
      s->source.spec.raster_data = nullptr;
    }
    for (int i = 0; i < n_seg; ++i) {
      Seg g{{seg[4 * i], seg[4 * i + 1]}, {seg[4 * i + 2], seg[4 * i + 3]}, kind[i], i};
      if (eps > 0.0) {  // Scene::validate, scene.cpp:119-143 (segment checks)
        if (g.a.x == g.b.x && g.a.y == g.b.y) throw SceneErr("a == b (zero-length segment)");
        if (!s->bbox.contains(g.a, 0.0) || !s->bbox.contains(g.b, 0.0))
          throw SceneErr("endpoint outside scene bbox");
        if (value_index[i] < 0 || value_index[i] >= n_values) throw SceneErr("value not defined");
      }
      s->input.push_back(g);
      s->value_index.push_back(value_index[i]);
    }
    s->build_accel();
    out = s.release();
  });
  return rc == WG_OK ? out : nullptr;
}

void orc_scene_destroy(void* s) { delete static_cast<Scene*>(s); }
double orc_t_epsilon(void* s) { return static_cast<Scene*>(s)->t_eps; }
int32_t orc_has_neumann_flux(void* s) { return static_cast<Scene*>(s)->neumann_flux(); }

int orc_closest_point(void* sp, int64_t n, const double* xy, uint32_t kinds, double* pt,
                      double* dist, int32_t* seg) {
  auto* s = static_cast<Scene*>(sp);
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) {
      CP c = closest_point(*s, {xy[2 * i], xy[2 * i + 1]}, kinds);
      pt[2 * i] = c.p.x;
      pt[2 * i + 1] = c.p.y;
      dist[i] = c.d;
      seg[i] = c.seg;
    }
  });
}

int orc_closest_silhouette(void* sp, int64_t n, const double* xy, double* dist) {
  auto* s = static_cast<Scene*>(sp);
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) dist[i] = closest_silhouette(*s, {xy[2 * i], xy[2 * i + 1]});
  });
}

int orc_ray_first_hit(void* sp, int64_t n, const double* o, const double* d, const double* t_max,
                      uint32_t kinds, const int32_t* exclude, double* t, double* pt,
                      double* normal, int32_t* seg, int32_t* kind) {
  auto* s = static_cast<Scene*>(sp);
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) {
      Hit h = ray_first_hit(*s, {o[2 * i], o[2 * i + 1]}, {d[2 * i], d[2 * i + 1]}, t_max[i],
                            kinds, exclude ? exclude[i] : -1);
      t[i] = h.ok ? h.t : kInf;
      pt[2 * i] = h.ok ? h.p.x : 0.0;
      pt[2 * i + 1] = h.ok ? h.p.y : 0.0;
      normal[2 * i] = h.ok ? h.n.x : 0.0;
      normal[2 * i + 1] = h.ok ? h.n.y : 0.0;
      seg[i] = h.seg;
      kind[i] = h.kind;
    }
  });
}

int orc_star_radius(void* sp, int64_t n, const double* xy, double r_min, double* r) {
  auto* s = static_cast<Scene*>(sp);
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) r[i] = star_radius(*s, {xy[2 * i], xy[2 * i + 1]}, r_min);
  });
}

double orc_bessel_i0(double x) { return bessel_i0(x); }
double orc_log_bessel_i0(double x) { return log_bessel_i0(x); }
double orc_bessel_i1_over_i0(double x) { return bessel_i1_over_i0(x); }

void orc_normalize_params(int64_t n, const double* raw, int32_t k, int32_t dim, wg_mixture* out) {
  const int od = (2 + dim) * k + 1;
  for (int64_t i = 0; i < n; ++i) {
    Mix m = normalize(unpack(raw + i * od, k, dim));
    wg_mixture& o = out[i];
    std::memset(&o, 0, sizeof(o));
    for (int c = 0; c < k; ++c) {
      o.mu[c][0] = m.c[c].mu.x;
      o.mu[c][1] = m.c[c].mu.y;
      o.mu[c][2] = m.c[c].mu.z;
      o.kappa[c] = m.c[c].kappa;
      o.lambda[c] = m.c[c].lambda;
      o.log_a[c] = m.log_a[c];
    }
    o.c = m.sel;
    o.k = k;
    o.dim = dim;
  }
}

double orc_mixture_pdf(const wg_mixture* m, const double* nu) {
  return mixture_pdf({nu[0], nu[1], nu[2]}, from_wg(m));
}

double orc_mis_pdf(const wg_mixture* m, const double* nu, const double* normal, int32_t refl) {
  V3 n3;
  if (normal) n3 = {normal[0], normal[1], normal[2]};
  return mis_pdf({nu[0], nu[1], nu[2]}, from_wg(m), normal ? &n3 : nullptr, refl != 0);
}

void* orc_field_create(const wg_field_config* cfg, const double* bbox, uint64_t seed) {
  Field* f = nullptr;
  int rc = guarded([&] {
    Box b;
    b.lo = {bbox[0], bbox[1]};
    b.hi = {bbox[2], bbox[3]};
    f = new Field(*cfg, b, seed);
  });
  return rc == WG_OK ? f : nullptr;
}
void orc_field_destroy(void* f) { delete static_cast<Field*>(f); }
int64_t orc_field_param_count(void* f) { return static_cast<int64_t>(static_cast<Field*>(f)->p.size()); }
void orc_field_get_params(void* fp, float* out) {
  auto* f = static_cast<Field*>(fp);
  std::memcpy(out, f->p.data(), f->p.size() * sizeof(float));
}
void orc_field_set_params(void* fp, const float* in) {
  auto* f = static_cast<Field*>(fp);
  std::memcpy(f->p.data(), in, f->p.size() * sizeof(float));
}
void orc_field_eval_batch(void* fp, int64_t n, const double* xy, double* out) {
  auto* f = static_cast<Field*>(fp);
  const int od = f->out_dim();
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) f->eval({xy[2 * i], xy[2 * i + 1]}, out + i * od);
}

int orc_walks(void* sp, void* fp, const wg_solver_config* cfg, int64_t n, const double* xy,
              const int64_t* point_index, uint64_t seed, uint64_t wpp_index, double* estimate,
              int32_t* escaped, int32_t* n_records) {
  auto* s = static_cast<Scene*>(sp);
  return guarded([&] {
    Ctx c;
    c.s = s;
    c.f = static_cast<Field*>(fp);
    c.cfg = *cfg;
    c.flux = s->neumann_flux();
    std::string err;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i) {
      try {
        Walk w = run_walk(c, {xy[2 * i], xy[2 * i + 1]},
                          Pcg::walk(seed, point_index ? point_index[i] : i, wpp_index),
                          n_records != nullptr);
        estimate[i] = w.escaped ? 0.0 : w.acc;
        escaped[i] = w.escaped ? 1 : 0;
        if (n_records) n_records[i] = w.escaped ? 0 : static_cast<int32_t>(w.trace.size());
      } catch (const std::exception& e) {
#pragma omp critical
        err = e.what();
      }
    }
    if (!err.empty()) throw SceneErr(err);
  });
}

int orc_solve_batch(void* sp, void* fp, const wg_solver_config* cfg, int64_t n, const double* xy,
                    wg_point_stats* stats, uint64_t seed, uint64_t wpp_index, int32_t collect,
                    wg_guide_record** records, int64_t* n_records) {
  auto* s = static_cast<Scene*>(sp);
  return guarded([&] {
    Ctx c;
    c.s = s;
    c.f = static_cast<Field*>(fp);
    c.cfg = *cfg;
    c.flux = s->neumann_flux();
    std::vector<Rec> recs;
    std::vector<Walk> ws(n);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i)
      ws[i] = run_walk(c, {xy[2 * i], xy[2 * i + 1]}, Pcg::walk(seed, i, wpp_index), collect != 0);
    for (int64_t i = 0; i < n; ++i) {  // Welford in point order, wost.cpp:373-383
      const Walk& w = ws[i];
      double v = w.escaped ? 0.0 : w.acc;
      wg_point_stats& p = stats[i];
      ++p.count;
      double d = v - p.mean;
      p.mean += d / static_cast<double>(p.count);
      p.m2 += d * (v - p.mean);
      if (w.escaped) {
        ++p.escaped;
        continue;
      }
      if (collect) backfill(w, recs);
    }
    if (records) {
      auto* out = static_cast<wg_guide_record*>(std::malloc(sizeof(wg_guide_record) * (recs.size() + 1)));
      for (size_t i = 0; i < recs.size(); ++i) {
        const Rec& r = recs[i];
        wg_guide_record& o = out[i];
        std::memset(&o, 0, sizeof(o));
        o.x[0] = r.x.x;
        o.x[1] = r.x.y;
        o.nu[0] = r.nu.x;
        o.nu[1] = r.nu.y;
        o.nu[2] = r.nu.z;
        o.target = r.target;
        o.pdf_mis = r.pmis;
        o.pdf_g = r.pg;
        o.pdf_u = r.pu;
        o.c = r.c;
        o.on_neumann = r.on_n ? 1 : 0;
        o.normal[0] = r.n.x;
        o.normal[1] = r.n.y;
      }
      *records = out;
      *n_records = static_cast<int64_t>(recs.size());
    }
  });
}

void orc_free(void* p) { std::free(p); }

int orc_train_batch(void* fp, const wg_guide_record* recs, int64_t n, const wg_train_config* cfg,
                    uint64_t round, wg_train_stats* stats) {
  auto* f = static_cast<Field*>(fp);
  return guarded([&] {
    std::vector<Rec> rv(n);
    for (int64_t i = 0; i < n; ++i) rv[i] = from_wg(recs[i]);
    *stats = train_batch(*f, rv, *cfg, round);
  });
}

int orc_field_grad(void* fp, const wg_guide_record* recs, int64_t n, const wg_train_config* cfg,
                   double* grad_out) {
  auto* f = static_cast<Field*>(fp);
  return guarded([&] {
    std::vector<double> g(f->p.size(), 0.0);
    double inv = 1.0 / static_cast<double>(n);
    for (int64_t r = 0; r < n; ++r) {
      Rec rec = from_wg(recs[r]);
      if (rec.pmis < cfg->pdf_floor) continue;
      record_grad(*f, rec, *cfg, inv, g, nullptr);
    }
    std::memcpy(grad_out, g.data(), g.size() * sizeof(double));
  });
}

}  // extern "C"

// 3D contract (SURVEY.md §8 a′): same translation unit, shares orc::
#include "wost3d.inc"
