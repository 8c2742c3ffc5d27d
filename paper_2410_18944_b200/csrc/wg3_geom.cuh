// 3D scene queries on device (SURVEY.md §8 a′, configs 4-5): closest point
// on a triangle mesh, closest silhouette edge, first ray hit, star radius.
//
// The reference has no 3D code; the contract is oracle/wost3d.inc (the 3D
// analogue of proj/src/geom2d.cpp:142-255). Every selection rule is
// order-independent (minimum of (d^2, id) / (t, id)), so these BVH traversals
// return exactly what the oracle's own structure returns. Arithmetic is fp64
// in the oracle's operation order; translation units including this header
// compile with -fmad=false (Makefile), so results are bit-identical.
//
// HBM layout (per kind: Dirichlet, Neumann; plus the silhouette-edge index):
//   Node4 128 B  four children's fp32 boxes (SoA, rounded outward from fp64
//          so pruning is conservative) + child codes (interior node index, or
//          a leaf's first primitive and count); every device traversal uses
//          these 4-wide trees (SAH-built binary trees collapsed, wg3_scene.cu).
//   Node3  32 B  the binary tree they come from {lo.xyz f32, a i32 | hi.xyz
//          f32, b i32} (kept on the device as the per-kind presence flag).
//   Tri3   88 B  vertices (fp64), original id, value index, kind; stored in
//          leaf order so a leaf's triangles are contiguous.
//   Edge3 104 B  endpoints, the two incident Neumann normals, type.
// A 100k-triangle scene is ~10 MB: L2-resident (126 MB) on B200.
#pragma once

#include <cstdint>

#include "../../include/wostgpu_types.h"
#include "wg_device.cuh"

namespace wg3 {

using wg::dinf;

// Pinned fp64 arithmetic in translation units that contract FMAs (the
// tensor-core walk TU defines WG3_PIN_FP): every product and sum rounded on
// its own, in the oracle's order. Contraction would otherwise fuse these
// differently in different kernels (a product kept in a register in one,
// stored to a wavefront lane in another), so the wavefront and lockstep
// paths could part ways on a walk by one rounding. The -fmad=false TUs get
// the same roundings from plain operators (pinning them there measured 7.7%
// slower on uniform walks); pinning costs the wavefront 2.7% (cfg 4 shape).
#if defined(__CUDA_ARCH__) && defined(WG3_PIN_FP)
__device__ __forceinline__ double pm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double pa(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ps(double a, double b) { return __dsub_rn(a, b); }
#else
__host__ __device__ inline double pm(double a, double b) { return a * b; }
__host__ __device__ inline double pa(double a, double b) { return a + b; }
__host__ __device__ inline double ps(double a, double b) { return a - b; }
#endif

struct D3 {
  double x, y, z;
};
__host__ __device__ __forceinline__ D3 add(D3 a, D3 b) { return {pa(a.x, b.x), pa(a.y, b.y), pa(a.z, b.z)}; }
__host__ __device__ __forceinline__ D3 sub(D3 a, D3 b) { return {ps(a.x, b.x), ps(a.y, b.y), ps(a.z, b.z)}; }
__host__ __device__ __forceinline__ D3 scl(D3 a, double s) { return {pm(a.x, s), pm(a.y, s), pm(a.z, s)}; }
__host__ __device__ __forceinline__ double dot(D3 a, D3 b) {
  return pa(pa(pm(a.x, b.x), pm(a.y, b.y)), pm(a.z, b.z));
}
__host__ __device__ __forceinline__ D3 cross(D3 a, D3 b) {
  return {ps(pm(a.y, b.z), pm(a.z, b.y)), ps(pm(a.z, b.x), pm(a.x, b.z)), ps(pm(a.x, b.y), pm(a.y, b.x))};
}

struct __align__(16) Node3 {
  float lo[3];
  int32_t a;
  float hi[3];
  int32_t b;
};
struct __align__(8) Tri3 {
  double a[3], b[3], c[3];
  int32_t id, value, kind, pad_;
};
struct __align__(8) Edge3 {
  double a[3], b[3], n0[3], n1[3];
  int32_t type, pad_;  // 0: always a silhouette, 1: crease (facing test)
};
// 4-wide node (128 B, 8 x 16-B loads) of the closest-Dirichlet-point BVH:
// the binary tree collapsed so every node holds up to four children's fp32
// boxes (outward-rounded, as Node3's). child[i] >= 0: an interior Node4;
// child[i] < 0: a leaf, primitives [-(child[i]+1) >> 3, ... + (-(child[i]+1) & 7));
// an empty slot has an inverted box (never visited).
#ifndef WG3_BVH_W
#define WG3_BVH_W 4
#endif
constexpr int kBvhW = WG3_BVH_W;  // children per wide node (8-wide measured 15-25% slower on cfg 4)
struct __align__(16) Node4 {
  float lox[kBvhW], loy[kBvhW], loz[kBvhW], hix[kBvhW], hiy[kBvhW], hiz[kBvhW];
  int32_t child[kBvhW];
  int32_t pad_[kBvhW == 4 ? 4 : kBvhW];
};
static_assert(sizeof(Node4) % 16 == 0, "Node4 layout");
static_assert(sizeof(Node3) == 32, "Node3 layout");
static_assert(sizeof(Tri3) == 88, "Tri3 layout");
static_assert(sizeof(Edge3) == 104, "Edge3 layout");

struct Scene3View {
  const Node3* node[3];  // Dirichlet, Neumann, silhouette edges (nullptr if empty)
  const Tri3* tri[2];    // leaf-ordered triangles per kind
  const float4* tbox;    // [2 per Dirichlet triangle] fp32 box {lo, hi}, outward-rounded
  const Node4* node4;    // the Dirichlet BVH collapsed 4-wide (closest-point queries)
  const Node4* node4n;   // the Neumann BVH collapsed 4-wide (rays)
  const Node4* node4e;   // the silhouette-edge BVH collapsed 4-wide
  const Edge3* edge;     // leaf-ordered edges
  const wg_value3_spec* values;
  double bbox[6];
  double t_eps, diag, eps;
  double sil_tol;  // facings within this count as 0 (oracle/wost3d.inc)
  wg_value3_spec source;  // type WG_VALUE_ZERO: no source term
  int32_t has_flux;       // some Neumann triangle has h != 0
  int32_t pad_;
};

__device__ __forceinline__ D3 ld3(const double* p) { return {p[0], p[1], p[2]}; }


// fp32 lower bound of box_d2 for BVH pruning: the point as an fp32
// interval [lo, hi] (rounded outward), per-axis gaps and the sum rounded
// down, compared with the best distance rounded up. A box is skipped only if
// it is certainly farther than the best, so the search returns the same
// minimum as the fp64 test (it may visit a few more boxes); 4 fp32 ops per
// axis instead of two f32->f64 conversions and four fp64 ops.
struct PtBox {
  float xl, xu, yl, yu, zl, zu;
};
__device__ __forceinline__ PtBox pt_box(D3 p) {
  return {__double2float_rd(p.x), __double2float_ru(p.x), __double2float_rd(p.y),
          __double2float_ru(p.y), __double2float_rd(p.z), __double2float_ru(p.z)};
}
__device__ __forceinline__ float box_d2_lb(const float4& lo, const float4& hi, const PtBox& p) {
  const float dx = fmaxf(fmaxf(__fsub_rd(lo.x, p.xu), __fsub_rd(p.xl, hi.x)), 0.0f);
  const float dy = fmaxf(fmaxf(__fsub_rd(lo.y, p.yu), __fsub_rd(p.yl, hi.y)), 0.0f);
  const float dz = fmaxf(fmaxf(__fsub_rd(lo.z, p.zu), __fsub_rd(p.zl, hi.z)), 0.0f);
  return __fadd_rd(__fadd_rd(__fmul_rd(dx, dx), __fmul_rd(dy, dy)), __fmul_rd(dz, dz));
}

__device__ __forceinline__ double box_d2(const float4& lo, const float4& hi, D3 p) {
  double dx = fmax(fmax((double)lo.x - p.x, 0.0), p.x - (double)hi.x);
  double dy = fmax(fmax((double)lo.y - p.y, 0.0), p.y - (double)hi.y);
  double dz = fmax(fmax((double)lo.z - p.z, 0.0), p.z - (double)hi.z);
  return pa(pa(pm(dx, dx), pm(dy, dy)), pm(dz, dz));
}

// closest point on triangle abc (oracle/wost3d.inc closest_on_tri)
__device__ __forceinline__ D3 closest_on_tri(D3 p, D3 a, D3 b, D3 c) {
  D3 ab = sub(b, a), ac = sub(c, a), ap = sub(p, a);
  double d1 = dot(ab, ap), d2 = dot(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) return a;
  D3 bp = sub(p, b);
  double d3 = dot(ab, bp), d4 = dot(ac, bp);
  if (d3 >= 0.0 && d4 <= d3) return b;
  double vc = ps(pm(d1, d4), pm(d3, d2));
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    double v = d1 / (d1 - d3);
    return add(a, scl(ab, v));
  }
  D3 cp = sub(p, c);
  double d5 = dot(ab, cp), d6 = dot(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) return c;
  double vb = ps(pm(d5, d2), pm(d1, d6));
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    double w = d2 / (d2 - d6);
    return add(a, scl(ac, w));
  }
  double va = ps(pm(d3, d6), pm(d5, d4));
  if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
    double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    return add(b, scl(sub(c, b), w));
  }
  double den = 1.0 / (va + vb + vc);
  double v = pm(vb, den), w = pm(vc, den);
  return add(add(a, scl(ab, v)), scl(ac, w));
}

__device__ __forceinline__ D3 closest_on_seg(D3 p, D3 a, D3 b) {
  D3 ab = sub(b, a);
  double l2 = dot(ab, ab);
  double t = l2 > 0.0 ? wg::sclamp(dot(sub(p, a), ab) / l2, 0.0, 1.0) : 0.0;
  return add(a, scl(ab, t));
}

// Moller-Trumbore (oracle ray_tri); miss -> false
__device__ __forceinline__ bool ray_tri(D3 o, D3 d, D3 a, D3 b, D3 c, double* t) {
  D3 e1 = sub(b, a), e2 = sub(c, a);
  D3 p = cross(d, e2);
  double det = dot(e1, p);
  if (det == 0.0) return false;
  double inv = 1.0 / det;
  D3 s = sub(o, a);
  double u = dot(s, p) * inv;
  if (u < 0.0 || u > 1.0) return false;
  D3 q = cross(s, e1);
  double v = dot(d, q) * inv;
  if (v < 0.0 || u + v > 1.0) return false;
  *t = dot(e2, q) * inv;
  return true;
}


// traversal stack capacity: a 4-wide descent pushes at most 3 entries per
// interior node on its path; the scene build
// checks its trees' depths against these (wg3_scene.cu: an SAH tree that is
// too deep is rebuilt with median splits, and a median tree that is too deep
// fails the scene). The 4-wide stacks live in local memory: 40 entries
// (median 4-wide trees to depth 13, > 10^8 triangles) keep the geometry
// pass's per-thread footprint small (cfg 4 shape, 32 vs 64 entries: frozen
// rounds -1%, uniform -2%)
#ifndef WG3_STACK4
#define WG3_STACK4 40
#endif
constexpr int kStack4 = WG3_STACK4;

struct CP3 {
  D3 p;
  double d2;
  int tri;    // original id, -1 if none
  int local;  // leaf-order index within its kind's triangle array
};

// closest point over the 4-wide Dirichlet BVH: per node the four children's
// fp32 lower-bound distances, the nearest child descended into, the other
// candidates pushed with their bound (a popped entry whose bound exceeds the
// best is dropped without a load). Leaf children are tested when reached.
// The same minimum over (d^2, id) as cp_bvh.
__device__ __forceinline__ void cp_leaf(const Tri3* tris, const float4* tbox, D3 x, const PtBox& pb, int code,
                                        CP3& best, float& bf) {
  const int first = (-(code + 1)) >> 3, cnt = (-(code + 1)) & 7;
  for (int i = first; i < first + cnt; ++i) {
    if (tbox && box_d2_lb(tbox[2 * i], tbox[2 * i + 1], pb) > bf) continue;
    const Tri3& t = tris[i];
    D3 q = closest_on_tri(x, ld3(t.a), ld3(t.b), ld3(t.c));
    D3 dq = sub(x, q);
    double d2 = dot(dq, dq);
    int id = t.id;
    if (d2 < best.d2 || (d2 == best.d2 && id < best.tri)) {
      best.d2 = d2;
      best.p = q;
      best.tri = id;
      best.local = i;
      bf = __double2float_ru(d2);
    }
  }
}

struct Kids4 {
  float lx[kBvhW], ly[kBvhW], lz[kBvhW], hx[kBvhW], hy[kBvhW], hz[kBvhW];
  int c[kBvhW];
};
__device__ __forceinline__ void load4(const Node4* nodes, int node, Kids4& k) {
  const float4* q = reinterpret_cast<const float4*>(nodes + node);
  constexpr int V = kBvhW / 4;  // float4 per field
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const float4 lx = __ldg(q + 0 * V + v), ly = __ldg(q + 1 * V + v), lz = __ldg(q + 2 * V + v);
    const float4 hx = __ldg(q + 3 * V + v), hy = __ldg(q + 4 * V + v), hz = __ldg(q + 5 * V + v);
    const int4 ch = __ldg(reinterpret_cast<const int4*>(q + 6 * V + v));
    const float a0[4] = {lx.x, lx.y, lx.z, lx.w}, a1[4] = {ly.x, ly.y, ly.z, ly.w}, a2[4] = {lz.x, lz.y, lz.z, lz.w};
    const float b0[4] = {hx.x, hx.y, hx.z, hx.w}, b1[4] = {hy.x, hy.y, hy.z, hy.w}, b2[4] = {hz.x, hz.y, hz.z, hz.w};
    const int cc[4] = {ch.x, ch.y, ch.z, ch.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      k.lx[4 * v + j] = a0[j];
      k.ly[4 * v + j] = a1[j];
      k.lz[4 * v + j] = a2[j];
      k.hx[4 * v + j] = b0[j];
      k.hy[4 * v + j] = b1[j];
      k.hz[4 * v + j] = b2[j];
      k.c[4 * v + j] = cc[j];
    }
  }
}

__device__ __forceinline__ float kid_d2_lb(const Kids4& k, int i, const PtBox& pb) {
  const float dx = fmaxf(fmaxf(__fsub_rd(k.lx[i], pb.xu), __fsub_rd(pb.xl, k.hx[i])), 0.0f);
  const float dy = fmaxf(fmaxf(__fsub_rd(k.ly[i], pb.yu), __fsub_rd(pb.yl, k.hy[i])), 0.0f);
  const float dz = fmaxf(fmaxf(__fsub_rd(k.lz[i], pb.zu), __fsub_rd(pb.zl, k.hz[i])), 0.0f);
  return __fadd_rd(__fadd_rd(__fmul_rd(dx, dx), __fmul_rd(dy, dy)), __fmul_rd(dz, dz));
}

__device__ __forceinline__ void cp_bvh4(const Node4* nodes, const Tri3* tris, const float4* tbox, D3 x,
                                        CP3& best) {
  const PtBox pb = pt_box(x);
  float bf = __double2float_ru(best.d2);
  int st_code[kStack4];
  float st_key[kStack4];
  int sp = 0;
  int node = 0;
  // next: the most recently pushed entry still within the bound
  auto pop = [&]() {
    while (sp) {
      --sp;
      if (st_key[sp] <= bf) {
        node = st_code[sp];
        return true;
      }
    }
    return false;
  };
  for (;;) {
    if (node >= 0) {
      Kids4 k;
      load4(nodes, node, k);
      float km = __int_as_float(0x7f800000);
      int cm = 0;
      bool have = false;
#pragma unroll
      for (int i = 0; i < kBvhW; ++i) {
        const float d = kid_d2_lb(k, i, pb);
        if (d <= bf && k.lx[i] <= k.hx[i]) {  // (an empty slot has an inverted box)
          if (!have || d < km) {  // new nearest: the previous nearest goes on the stack
            if (have) {
              st_code[sp] = cm;
              st_key[sp] = km;
              ++sp;
            }
            km = d;
            cm = k.c[i];
            have = true;
          } else {
            st_code[sp] = k.c[i];
            st_key[sp] = d;
            ++sp;
          }
        }
      }
      if (have) {
        node = cm;
        continue;
      }
    } else {
      cp_leaf(tris, tbox, x, pb, node, best, bf);
    }
    if (!pop()) return;
  }
}

// closest Dirichlet point seeded with a candidate triangle (leaf-order index
// `seed`, -1 for none): the candidate's exact distance bounds the traversal
// from the start; the result is the same minimum over (d^2, id)
__device__ __forceinline__ CP3 closest_dirichlet_seeded(const Scene3View& s, D3 x, int seed) {
  CP3 best{{0.0, 0.0, 0.0}, dinf(), -1, -1};
  if (seed >= 0 && s.node[0]) {
    const Tri3& t = s.tri[0][seed];
    D3 q = closest_on_tri(x, ld3(t.a), ld3(t.b), ld3(t.c));
    D3 dq = sub(x, q);
    best = {q, dot(dq, dq), t.id, seed};
  }
  if (s.node4) cp_bvh4(s.node4, s.tri[0], s.tbox, x, best);
  return best;
}

// Accel::closest_point analogue: (point, distance, triangle id) or id -1, d = inf
__device__ __forceinline__ CP3 closest_point(const Scene3View& s, D3 x, unsigned kinds) {
  CP3 best{{0.0, 0.0, 0.0}, dinf(), -1, -1};
  if ((kinds & WG_KIND_DIRICHLET) && s.node4) cp_bvh4(s.node4, s.tri[0], s.tbox, x, best);
  if ((kinds & WG_KIND_NEUMANN) && s.node4n) cp_bvh4(s.node4n, s.tri[1], nullptr, x, best);
  return best;
}

__device__ __forceinline__ bool is_silhouette(const Edge3& e, D3 x, double tol) {
  if (e.type == 0) return true;
  D3 ax = sub(ld3(e.a), x);
  double f0 = dot(ld3(e.n0), ax), f1 = dot(ld3(e.n1), ax);
  if (fabs(f0) <= tol || fabs(f1) <= tol) return true;
  return f0 * f1 <= 0.0;
}

// the silhouette search over the 4-wide edge BVH (strict bound, as below)
__device__ __forceinline__ double sil_bvh4(const Scene3View& s, D3 x, double bound2) {
  double best = bound2;
  const PtBox pb = pt_box(x);
  float bf = __double2float_ru(best);
  int st_code[kStack4];
  float st_key[kStack4];
  int sp = 0;
  int node = 0;
  for (;;) {
    if (node >= 0) {
      Kids4 k;
      load4(s.node4e, node, k);
      float km = __int_as_float(0x7f800000);
      int cm = 0;
      bool have = false;
#pragma unroll
      for (int i = 0; i < kBvhW; ++i) {
        const float d = kid_d2_lb(k, i, pb);
        if (d < bf && k.lx[i] <= k.hx[i]) {
          if (!have || d < km) {
            if (have) {
              st_code[sp] = cm;
              st_key[sp] = km;
              ++sp;
            }
            km = d;
            cm = k.c[i];
            have = true;
          } else {
            st_code[sp] = k.c[i];
            st_key[sp] = d;
            ++sp;
          }
        }
      }
      if (have) {
        node = cm;
        continue;
      }
    } else {
      const int first = (-(node + 1)) >> 3, cnt = (-(node + 1)) & 7;
      for (int i = first; i < first + cnt; ++i) {
        const Edge3& e = s.edge[i];
        if (!is_silhouette(e, x, s.sil_tol)) continue;
        D3 dq = sub(x, closest_on_seg(x, ld3(e.a), ld3(e.b)));
        best = fmin(best, dot(dq, dq));
      }
      bf = __double2float_ru(best);
    }
    bool found = false;
    while (sp) {
      --sp;
      if (st_key[sp] < bf) {
        node = st_code[sp];
        found = true;
        break;
      }
    }
    if (!found) return best;
  }
}

// squared distance to the nearest silhouette edge (inf if none); with a
// bound, only edges strictly closer than sqrt(bound2) are searched for and
// bound2 comes back when there is none
__device__ __forceinline__ double closest_silhouette_d2(const Scene3View& s, D3 x, double bound2 = dinf()) {
  if (!s.node4e) return dinf();  // no silhouette edges at all
  return sil_bvh4(s, x, bound2);
}

__device__ __forceinline__ double closest_silhouette(const Scene3View& s, D3 x) {
  double b = closest_silhouette_d2(s, x);
  return b == dinf() ? dinf() : sqrt(b);
}

struct Hit3 {
  double t;
  int tri;    // original id, -1 on a miss
  int local;  // leaf-order index within its kind's array
  int kind;
};

// fp32 slab test against the box grown by `pad` on every side: with pad at
// least 2^-20 of the scene's coordinate scale it dominates the fp32
// rounding of (bound - origin) * (1 / d), so a box the segment [0, t_hi]
// truly meets is never rejected (the search visits a superset and the
// fp64 ray-triangle tests decide); 2 fp32 ops per slab instead of fp64
__device__ __forceinline__ bool ray_box_f(const float3& o, const float3& inv, const bool* dz, const float4& lo,
                                          const float4& hi, float t_hi, float pad) {
  float t0 = 0.0f, t1 = t_hi;
  const float oo[3] = {o.x, o.y, o.z}, iv[3] = {inv.x, inv.y, inv.z};
  const float l[3] = {lo.x - pad, lo.y - pad, lo.z - pad}, h[3] = {hi.x + pad, hi.y + pad, hi.z + pad};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (dz[a]) {
      if (oo[a] < l[a] || oo[a] > h[a]) return false;
      continue;
    }
    float ta = (l[a] - oo[a]) * iv[a], tb = (h[a] - oo[a]) * iv[a];
    if (ta > tb) {
      const float s = ta;
      ta = tb;
      tb = s;
    }
    t0 = fmaxf(t0, ta);
    t1 = fminf(t1, tb);
    if (t0 > t1) return false;
  }
  return true;
}

// first hit over a 4-wide BVH: children slab-tested in fp32 (ray_box_f's
// padded boxes), the nearest entry descended into, the others pushed with
// their entry t; the same minimum over (t, id) as ray_bvh
__device__ __forceinline__ void ray_bvh4(const Node4* nodes, const Tri3* tris, int kind, D3 o, D3 d,
                                         double t_max, double t_eps, int exclude, Hit3& h, float pad) {
  const bool dz[3] = {d.x == 0.0, d.y == 0.0, d.z == 0.0};
  const float3 of = make_float3(static_cast<float>(o.x), static_cast<float>(o.y), static_cast<float>(o.z));
  const float3 invf = make_float3(dz[0] ? 0.0f : static_cast<float>(1.0 / d.x),
                                  dz[1] ? 0.0f : static_cast<float>(1.0 / d.y),
                                  dz[2] ? 0.0f : static_cast<float>(1.0 / d.z));
  float tb_f = __double2float_ru(fmin(t_max, h.t)) * (1.0f + 0x1.0p-20f);
  int st_code[kStack4];
  float st_key[kStack4];
  int sp = 0;
  int node = 0;
  for (;;) {
    if (node >= 0) {
      Kids4 k;
      load4(nodes, node, k);
      float km = __int_as_float(0x7f800000);
      int cm = 0;
      bool have = false;
#pragma unroll
      for (int i = 0; i < kBvhW; ++i) {
        float t0 = 0.0f, t1 = tb_f;
        bool hit = true;
        const float lo[3] = {k.lx[i] - pad, k.ly[i] - pad, k.lz[i] - pad};
        const float hi[3] = {k.hx[i] + pad, k.hy[i] + pad, k.hz[i] + pad};
        const float oo[3] = {of.x, of.y, of.z}, iv[3] = {invf.x, invf.y, invf.z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (dz[a]) {
            hit = hit && !(oo[a] < lo[a] || oo[a] > hi[a]);
          } else {
            const float ta = (lo[a] - oo[a]) * iv[a], tb = (hi[a] - oo[a]) * iv[a];
            t0 = fmaxf(t0, fminf(ta, tb));
            t1 = fminf(t1, fmaxf(ta, tb));
          }
        }
        hit = hit && t0 <= t1 && k.lx[i] <= k.hx[i];
        if (hit) {
          if (!have || t0 < km) {
            if (have) {
              st_code[sp] = cm;
              st_key[sp] = km;
              ++sp;
            }
            km = t0;
            cm = k.c[i];
            have = true;
          } else {
            st_code[sp] = k.c[i];
            st_key[sp] = t0;
            ++sp;
          }
        }
      }
      if (have) {
        node = cm;
        continue;
      }
    } else {
      const int first = (-(node + 1)) >> 3, cnt = (-(node + 1)) & 7;
      for (int i = first; i < first + cnt; ++i) {
        const Tri3& t = tris[i];
        const int id = t.id;
        if (id == exclude) continue;
        double th;
        if (!ray_tri(o, d, ld3(t.a), ld3(t.b), ld3(t.c), &th)) continue;
        if (!(th > t_eps && th <= t_max)) continue;
        if (th < h.t || (th == h.t && id < h.tri)) {
          h.t = th;
          h.tri = id;
          h.local = i;
          h.kind = kind;
          tb_f = __double2float_ru(fmin(t_max, h.t)) * (1.0f + 0x1.0p-20f);
        }
      }
    }
    bool found = false;
    while (sp) {
      --sp;
      if (st_key[sp] <= tb_f) {
        node = st_code[sp];
        found = true;
        break;
      }
    }
    if (!found) return;
  }
}

// box growth of the fp32 slab test: 2^-20 of the scene's coordinate scale
__device__ __forceinline__ float ray_pad(const Scene3View& s) {
  double m = s.diag;
  for (int i = 0; i < 6; ++i) m = fmax(m, fabs(s.bbox[i]));
  return static_cast<float>(m * 0x1.0p-20);
}

__device__ __forceinline__ Hit3 ray_first_hit(const Scene3View& s, D3 o, D3 d, double t_max,
                                              unsigned kinds, int exclude) {
  Hit3 h{dinf(), -1, -1, -1};
  const float pad = ray_pad(s);
  if ((kinds & WG_KIND_DIRICHLET) && s.node4) ray_bvh4(s.node4, s.tri[0], 0, o, d, t_max, s.t_eps, exclude, h, pad);
  if ((kinds & WG_KIND_NEUMANN) && s.node4n) ray_bvh4(s.node4n, s.tri[1], 1, o, d, t_max, s.t_eps, exclude, h, pad);
  return h;
}

// unit geometric normal of the hit triangle, facing the incoming ray
__device__ __forceinline__ D3 hit_normal(const Scene3View& s, const Hit3& h, D3 d) {
  const Tri3& t = s.tri[h.kind][h.local];
  D3 a = ld3(t.a);
  D3 n = cross(sub(ld3(t.b), a), sub(ld3(t.c), a));
  n = scl(n, 1.0 / sqrt(dot(n, n)));
  if (dot(n, d) > 0.0) n = scl(n, -1.0);
  return n;
}

__device__ __forceinline__ double value_at(const wg_value3_spec& v, D3 p) {
  if (v.type == WG_VALUE_CONSTANT) return v.c0;
  return pa(pa(pa(v.c0, pm(v.cx, p.x)), pm(v.cy, p.y)), pm(v.cz, p.z));
}

__device__ __forceinline__ bool bbox_contains(const Scene3View& s, D3 p, double pad) {
  return p.x >= s.bbox[0] - pad && p.x <= s.bbox[3] + pad && p.y >= s.bbox[1] - pad &&
         p.y <= s.bbox[4] + pad && p.z >= s.bbox[2] - pad && p.z <= s.bbox[5] + pad;
}

}  // namespace wg3
