// Device-side primitives of the walk-on-stars path: PCG32 streams, scene and
// BVH layout in device memory, and the fp64 geometry queries.
//
// Parity rule: every fp64 expression keeps the reference's operation order and
// the library is compiled with -fmad=false, so geometry results (indices AND
// distances) are bit-identical to the reference's strict build.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/wostgpu_types.h"

#define WG_HD __host__ __device__ __forceinline__
#define WG_D __device__ __forceinline__

namespace wg {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;
constexpr double kFourPi = 4.0 * kPi;
constexpr int kMaxK = WG_MAX_MIXTURE;
constexpr double kKappaMin = 1e-6, kKappaMax = 1e4;

WG_HD double dinf() { return __builtin_huge_val(); }

// std::min / std::max / std::clamp exactly (operand order matters for -0.0)
WG_HD double smin(double a, double b) { return b < a ? b : a; }
WG_HD double smax(double a, double b) { return a < b ? b : a; }
WG_HD double sclamp(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }
WG_HD int imin(int a, int b) { return b < a ? b : a; }

// ---------------------------------------------------------------- PCG32
// proj/include/wost/rng.hpp:9-78
struct Pcg {
  uint64_t s, inc;
  WG_HD uint32_t u32() {
    uint64_t old = s;
    s = old * 6364136223846793005ULL + inc;
    uint32_t xs = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
    uint32_t rot = static_cast<uint32_t>(old >> 59u);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
  }
  WG_HD void seed(uint64_t seed_, uint64_t stream) {
    s = 0;
    inc = (stream << 1u) | 1u;
    u32();
    s += seed_;
    u32();
  }
  WG_HD static uint64_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  WG_HD static Pcg walk(uint64_t seed_, uint64_t point, uint64_t wpp) {
    uint64_t a = mix(seed_ ^ mix(point));
    uint64_t b = mix(a ^ mix(wpp + 0x632be59bd9b4e019ULL));
    Pcg r;
    r.seed(a, b);
    return r;
  }
  WG_HD uint64_t u64() {
    uint64_t hi = u32();
    return (hi << 32) | u32();
  }
  WG_HD double uni() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
  WG_HD double uni_pos() {
    double u;
    do u = uni();
    while (u == 0.0);
    return u;
  }
  // fp32 uniforms from ONE 32-bit output (tensor-core walk path only):
  // [0, 1) and (0, 1] on the 2^-24 grid
  WG_HD float unif() { return static_cast<float>(u32() >> 8) * 0x1.0p-24f; }
  WG_HD float unif_pos() { return static_cast<float>((u32() >> 8) + 1u) * 0x1.0p-24f; }
};

// ---------------------------------------------------------------- scene
struct __align__(16) Node {  // 48 B: Bbox + children / leaf range
  double lox, loy, hix, hiy;
  int32_t left, right, begin, end;
};
struct __align__(8) Seg {  // 40 B, BVH leaf order
  double ax, ay, bx, by;
  int32_t kind;  // WG_DIRICHLET / WG_NEUMANN
  int32_t id;    // scene index
};
struct __align__(8) SilVertex {  // Neumann vertex + its incident normals
  double px, py;
  int32_t n_begin, n_count;
};
struct DevValue {
  int32_t type, analytic_id;
  double c0, cx, cy;
  int32_t rw, rh;
  double rb[4];
  const double* raster;  // device
};

struct SceneView {
  const Node* nodes;
  const Seg* segs;
  const SilVertex* sil;
  const double* sil_n;  // 2 doubles per normal
  int32_t n_nodes, n_segs, n_sil, n_sil_normals;
  // per scene segment (scene order): kind and value index
  const int32_t* seg_kind;
  const int32_t* seg_value;
  const DevValue* values;
  DevValue source;
  double bbox[4];
  double eps, t_eps, diag;
  int32_t has_flux, source_zero;
  int32_t n_neumann;  // Neumann segments: without any, Neumann-kind rays cannot hit
  int32_t pad_;
  const Node* sil_nodes;  // point BVH over the silhouette candidates (> 32 of them), else null
};

WG_D double eval_value(const DevValue& v, double x, double y) {
  switch (v.type) {
    case WG_VALUE_CONSTANT: return v.c0;
    case WG_VALUE_LINEAR: return v.c0 + v.cx * x + v.cy * y;
    case WG_VALUE_RASTER: {  // RasterGrid::at, proj/src/scene.cpp:13-20
      double ex = v.rb[2] - v.rb[0], ey = v.rb[3] - v.rb[1];
      double u = (x - v.rb[0]) / ex, w = (y - v.rb[1]) / ey;
      int i = static_cast<int>(u * v.rw), j = static_cast<int>(w * v.rh);
      i = i < 0 ? 0 : (v.rw - 1 < i ? v.rw - 1 : i);
      j = j < 0 ? 0 : (v.rh - 1 < j ? v.rh - 1 : j);
      return v.raster[static_cast<size_t>(j) * v.rw + i];
    }
    case WG_VALUE_ANALYTIC:
      if (v.analytic_id == WG_ANALYTIC_X2_MINUS_Y2) return x * x - y * y;
      return x * x + y * y - 1.0;
    default: return 0.0;
  }
}

// Occlusion test of a source sample at distance r inside the star ball of
// radius R (sample_source_point, wost.cpp:67-87). Without Neumann segments
// R is the Dirichlet distance, so for r < R every segment lies beyond the
// ray: ray_first_hit would return no hit, and the traversal is skipped.
WG_D bool source_ray_needed(const SceneView& s, double r, double R) { return s.n_neumann > 0 || !(r < R); }

WG_D bool bbox_contains(const SceneView& s, double x, double y, double pad) {
  return x >= s.bbox[0] - pad && x <= s.bbox[2] + pad && y >= s.bbox[1] - pad &&
         y <= s.bbox[3] + pad;
}

// squared point-box distance, proj/include/wost/vec.hpp:92-96
WG_D double box_d2(const Node& b, double px, double py) {
  double dx = smax(smax(b.lox - px, 0.0), px - b.hix);
  double dy = smax(smax(b.loy - py, 0.0), py - b.hiy);
  return dx * dx + dy * dy;
}

struct CP {
  double px, py, d;
  int seg;
};

// Accel::closest_point (proj/src/geom2d.cpp:142-180): stack DFS, box pruning,
// nearer child first, strict <; identical node order => identical ties.
WG_D CP closest_point(const SceneView& s, double x, double y, unsigned kinds) {
  CP best{0.0, 0.0, dinf(), -1};
  double bd2 = dinf();
  int st[64];
  int top = 0;
  st[top++] = 0;
  while (top > 0) {
    const Node nd = s.nodes[st[--top]];
    if (box_d2(nd, x, y) >= bd2) continue;
    if (nd.left < 0) {
      for (int i = nd.begin; i < nd.end; ++i) {
        const Seg g = s.segs[i];
        if (!((g.kind == WG_DIRICHLET ? 1u : 2u) & kinds)) continue;
        // closest_point_on_segment, geom2d.cpp:9-14
        double ux = g.bx - g.ax, uy = g.by - g.ay;
        double t = ((x - g.ax) * ux + (y - g.ay) * uy) / (ux * ux + uy * uy);
        t = sclamp(t, 0.0, 1.0);
        double px = g.ax + t * ux, py = g.ay + t * uy;
        double dx = px - x, dy = py - y;
        double d2 = dx * dx + dy * dy;
        if (d2 < bd2) {
          bd2 = d2;
          best.px = px;
          best.py = py;
          best.seg = g.id;
        }
      }
    } else {
      double dl = box_d2(s.nodes[nd.left], x, y);
      double dr = box_d2(s.nodes[nd.right], x, y);
      if (dl <= dr) {
        if (dr < bd2) st[top++] = nd.right;
        if (dl < bd2) st[top++] = nd.left;
      } else {
        if (dl < bd2) st[top++] = nd.left;
        if (dr < bd2) st[top++] = nd.right;
      }
    }
  }
  if (best.seg >= 0) best.d = sqrt(bd2);
  return best;
}

// Accel::closest_silhouette (geom2d.cpp:182-200). The result is the minimum
// over candidate vertices, so any visiting order gives the same value; the
// scan compares squared distances and takes one sqrt at the end, which is the
// same value (a correctly rounded sqrt is monotone, so min and sqrt commute).
WG_D void sil_vertex(const SceneView& s, int v, double x, double y, double& best) {
  const SilVertex sv = s.sil[v];
  double dx = sv.px - x, dy = sv.py - y;
  double d = dx * dx + dy * dy;
  if (d >= best) return;
  bool cand = sv.n_count < 2;
  if (!cand) {
    double lo = dinf(), hi = -dinf();
    for (int k = 0; k < sv.n_count; ++k) {
      double nx = s.sil_n[2 * (sv.n_begin + k)], ny = s.sil_n[2 * (sv.n_begin + k) + 1];
      double f = nx * dx + ny * dy;
      lo = smin(lo, f);
      hi = smax(hi, f);
    }
    cand = lo * hi <= 0.0;
  }
  if (cand) best = d;
}

WG_D double closest_silhouette(const SceneView& s, double x, double y) {
  double best = dinf();
  if (s.sil_nodes) {  // indexed: boxes at or beyond the best squared distance are skipped
    int st[64];
    int top = 0;
    st[top++] = 0;
    while (top > 0) {
      const Node nd = s.sil_nodes[st[--top]];
      if (box_d2(nd, x, y) >= best) continue;
      if (nd.left < 0) {
        for (int v = nd.begin; v < nd.end; ++v) sil_vertex(s, v, x, y, best);
      } else {
        const double dl = box_d2(s.sil_nodes[nd.left], x, y), dr = box_d2(s.sil_nodes[nd.right], x, y);
        if (dl <= dr) {
          st[top++] = nd.right;
          st[top++] = nd.left;
        } else {
          st[top++] = nd.left;
          st[top++] = nd.right;
        }
      }
    }
  } else {
#pragma unroll 2
    for (int v = 0; v < s.n_sil; ++v) sil_vertex(s, v, x, y, best);
  }
  return best == dinf() ? best : sqrt(best);
}

// slab test, geom2d.cpp:55-76
WG_D bool ray_box(double ox, double oy, double dx, double dy, double ix, double iy,
                  const Node& b, double t_max) {
  double t0 = 0.0, t1 = t_max;
  if (dx != 0.0) {
    double a = (b.lox - ox) * ix, c = (b.hix - ox) * ix;
    if (a > c) {
      double tmp = a;
      a = c;
      c = tmp;
    }
    t0 = smax(t0, a);
    t1 = smin(t1, c);
  } else if (ox < b.lox || ox > b.hix) {
    return false;
  }
  if (dy != 0.0) {
    double a = (b.loy - oy) * iy, c = (b.hiy - oy) * iy;
    if (a > c) {
      double tmp = a;
      a = c;
      c = tmp;
    }
    t0 = smax(t0, a);
    t1 = smin(t1, c);
  } else if (oy < b.loy || oy > b.hiy) {
    return false;
  }
  return t1 >= t0;
}

struct Hit {
  double t, px, py, nx, ny;
  int seg, kind;
};

WG_D Hit no_hit() {
  Hit h;
  h.seg = -1;
  h.kind = -1;
  h.t = dinf();
  h.px = h.py = h.nx = h.ny = 0.0;
  return h;
}

// Accel::ray_first_hit (geom2d.cpp:202-246): nearest t in (t_eps, t_max],
// the last equal t in traversal order wins; normal faces the ray.
WG_D Hit ray_first_hit(const SceneView& s, double ox, double oy, double dx, double dy,
                       double t_max, unsigned kinds, int exclude) {
  if (kinds == WG_KIND_NEUMANN && s.n_neumann == 0) return no_hit();  // nothing to hit
  double ix = 1.0 / dx, iy = 1.0 / dy;
  double bt = t_max;
  int bi = -1;
  double bsp = 0.0;
  int st[64];
  int top = 0;
  st[top++] = 0;
  while (top > 0) {
    const Node nd = s.nodes[st[--top]];
    if (!ray_box(ox, oy, dx, dy, ix, iy, nd, bt)) continue;
    if (nd.left < 0) {
      for (int i = nd.begin; i < nd.end; ++i) {
        const Seg g = s.segs[i];
        if (!((g.kind == WG_DIRICHLET ? 1u : 2u) & kinds)) continue;
        if (g.id == exclude) continue;
        // ray_segment, geom2d.cpp:41-51
        double ux = g.bx - g.ax, uy = g.by - g.ay;
        double wx = g.ax - ox, wy = g.ay - oy;
        double den = dx * uy - dy * ux;
        if (den == 0.0) continue;
        double t = (wx * uy - wy * ux) / den;
        double sp = (wx * dy - wy * dx) / den;
        if (sp < 0.0 || sp > 1.0) continue;
        if (t > s.t_eps && t <= bt) {
          bt = t;
          bi = i;
          bsp = sp;
        }
      }
    } else {
      st[top++] = nd.right;
      st[top++] = nd.left;
    }
  }
  Hit h;
  h.seg = -1;
  h.kind = -1;
  h.t = dinf();
  h.px = h.py = h.nx = h.ny = 0.0;
  if (bi < 0) return h;
  const Seg g = s.segs[bi];
  h.t = bt;
  double ux = g.bx - g.ax, uy = g.by - g.ay;
  h.px = g.ax + bsp * ux;
  h.py = g.ay + bsp * uy;
  double px = -uy, py = ux;
  double l = sqrt(px * px + py * py);
  double nx = px / l, ny = py / l;
  if (nx * dx + ny * dy > 0.0) {
    nx = -nx;
    ny = -ny;
  }
  h.nx = nx;
  h.ny = ny;
  h.seg = g.id;
  h.kind = g.kind;
  return h;
}

}  // namespace wg
