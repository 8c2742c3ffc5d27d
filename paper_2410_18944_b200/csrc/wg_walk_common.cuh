// Walk-kernel helpers shared by the tensor-core walk kernel (wg_walk_tc.cu)
// and the warp-per-walk kernel (wg_walk_coop.cu): small-scene geometry over
// per-kind shared-memory segment lists, and the 2D Green's-ball radius
// sampler of the source term.
#pragma once

#include "wg_kernels.cuh"

namespace wg {

// Small scenes (the benchmark square has 4 segments): no traversal stack.
// At launch the CTA copies the segments of each kind, in BVH leaf order, into
// shared-memory lists; a query scans only its kind's list, every segment
// evaluated with predicated updates so the fp64 divisions of consecutive
// segments overlap. Same per-segment arithmetic and the same strict-< / <=
// updates in visiting order as closest_point / ray_first_hit (wg_device.cuh):
// a one-leaf BVH visits segments in exactly this order, otherwise only
// exact-distance ties can resolve to a different (equidistant) segment.
constexpr int kSmallScene = 16;

struct SmallSegs {
  const Seg* d;  // Dirichlet segments
  const Seg* n;  // Neumann segments
  int nd, nn;
};

__device__ __forceinline__ CP cp_list(const Seg* segs, int n, double x, double y) {
  CP best{0.0, 0.0, dinf(), -1};
  double bd2 = dinf();
// the small-scene lists stay rolled: the walk kernel is instruction-fetch
// bound (14.3k SASS instructions unrolled 4x, 12.2k rolled; cfg 2 walk
// 0.598 -> 0.563 ms per round)
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    const Seg g = segs[i];
    double ux = g.bx - g.ax, uy = g.by - g.ay;
    double t = ((x - g.ax) * ux + (y - g.ay) * uy) / (ux * ux + uy * uy);
    t = sclamp(t, 0.0, 1.0);
    double px = g.ax + t * ux, py = g.ay + t * uy;
    double dx = px - x, dy = py - y;
    double d2 = dx * dx + dy * dy;
    const bool take = d2 < bd2;
    bd2 = take ? d2 : bd2;
    best.px = take ? px : best.px;
    best.py = take ? py : best.py;
    best.seg = take ? g.id : best.seg;
  }
  if (best.seg >= 0) best.d = sqrt(bd2);
  return best;
}

// the hit normal (normalised perp_left, flipped against the ray) is formed
// once, for the winner only
__device__ __forceinline__ Hit ray_list(const Seg* segs, int n, double t_eps, double ox, double oy,
                                        double dx, double dy, double t_max, int exclude) {
  double bt = t_max, bsp = 0.0;
  int bi = -1;
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    const Seg g = segs[i];
    double ux = g.bx - g.ax, uy = g.by - g.ay;
    double wx = g.ax - ox, wy = g.ay - oy;
    double den = dx * uy - dy * ux;
    const bool nz = den != 0.0;
    const double dd = nz ? den : 1.0;
    double t = (wx * uy - wy * ux) / dd;
    double sp = (wx * dy - wy * dx) / dd;
    const bool take = g.id != exclude && nz && !(sp < 0.0 || sp > 1.0) && t > t_eps && t <= bt;
    bt = take ? t : bt;
    bi = take ? i : bi;
    bsp = take ? sp : bsp;
  }
  Hit h;
  h.seg = -1;
  h.kind = -1;
  h.t = dinf();
  h.px = h.py = h.nx = h.ny = 0.0;
  if (bi < 0) return h;
  const Seg g = segs[bi];
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

// closest_silhouette for small vertex lists: squared distances of all
// vertices first (independent), then the candidate tests in order
__device__ __forceinline__ double sil_small(const SceneView& s, double x, double y) {
  double best = dinf();
#pragma unroll 1
  for (int v = 0; v < s.n_sil; ++v) {
    const SilVertex sv = s.sil[v];
    const double dx = sv.px - x, dy = sv.py - y;
    const double d = dx * dx + dy * dy;
    bool cand = sv.n_count < 2;
    if (!cand && d < best) {
      double lo = dinf(), hi = -dinf();
      for (int k = 0; k < sv.n_count; ++k) {
        double nx = s.sil_n[2 * (sv.n_begin + k)], ny = s.sil_n[2 * (sv.n_begin + k) + 1];
        double f = nx * dx + ny * dy;
        lo = smin(lo, f);
        hi = smax(hi, f);
      }
      cand = lo * hi <= 0.0;
    }
    best = (cand && d < best) ? d : best;
  }
  return best == dinf() ? best : sqrt(best);
}



__device__ __forceinline__ CP t_closest(const SceneView& s, const SmallSegs& ss, double x, double y,
                                        unsigned kinds) {
  if (s.n_segs > kSmallScene) return closest_point(s, x, y, kinds);
  return kinds == WG_KIND_DIRICHLET ? cp_list(ss.d, ss.nd, x, y) : closest_point(s, x, y, kinds);
}

__device__ __forceinline__ Hit t_ray(const SceneView& s, const SmallSegs& ss, double ox, double oy, double dx,
                                     double dy, double t_max, unsigned kinds, int exclude) {
  if (s.n_segs > kSmallScene || kinds != WG_KIND_NEUMANN)
    return ray_first_hit(s, ox, oy, dx, dy, t_max, kinds, exclude);
  return ray_list(ss.n, ss.nn, s.t_eps, ox, oy, dx, dy, t_max, exclude);
}

// sample_greens_radius (wost.cpp:37-65), d = 2: Newton + bisection on the
// radial CDF u = s^2 (1 - 2 ln s), s = r / R
__device__ __forceinline__ double t_greens_radius(double u, double R) {
  if (u <= 0.0) return 0.0;
  if (u >= 1.0) return R;
  double lo = 0.0, hi = 1.0, s = sqrt(u);
  for (int it = 0; it < 100; ++it) {
    double ls = log(s);
    double f = s * s * (1.0 - 2.0 * ls) - u;
    double df = -4.0 * s * ls;
    if (f > 0.0) hi = s;
    else lo = s;
    if (fabs(f) < 1e-10) break;
    double step = df > 0.0 ? f / df : 0.0;
    double nx = s - step;
    if (!(nx > lo && nx < hi)) nx = 0.5 * (lo + hi);
    if (nx == s) break;
    s = nx;
  }
  return s * R;
}

}  // namespace wg
