// 3D scenes: host BVH build (per-kind triangle BVHs + the silhouette-edge
// index of the Neumann set), batched query kernels and their C-ABI
// (include/wostgpu3.h). Contract: oracle/wost3d.inc (the 3D analogue of
// proj/src/geom2d.cpp:80-255).
//
// BVH: binary, binned surface-area-heuristic splits of the primitive
// centroids (16 bins per axis, the longest-axis median when no bin boundary
// beats it; ties by primitive index), leaves of <= 2, depth-first preorder so
// a node's first child follows it, then collapsed 4-wide. Built once per
// scene on the host (not hot); node boxes are fp32 rounded outward from the
// fp64 bounds. Every query is an order-independent minimum,
// so the tree shape changes speed only. cfg 4 shape (512^2, 256 frozen / 32
// training rounds): median splits with leaves of 4 1547-1549 / 401 ms, SAH
// leaves of 4 1501-1556 / 395-432, SAH leaves of 2 1464-1526 / 377-381, SAH
// leaves of 1 / 32 bins / 64 bins no better. WOSTGPU_BVH3 = median | sahN[B]
// (N = leaf size, B = bins) selects another rule for A/B runs.
#include <algorithm>
#include <array>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <functional>
#include <map>
#include <utility>

#include "wg3_runtime.hpp"

namespace wg3 {
namespace {

using wgrt::need;

float round_down(double d) {
  float f = static_cast<float>(d);
  if (static_cast<double>(f) > d) f = std::nextafter(f, -INFINITY);
  return f;
}
float round_up(double d) {
  float f = static_cast<float>(d);
  if (static_cast<double>(f) < d) f = std::nextafter(f, INFINITY);
  return f;
}

struct HBox {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  void grow(const double* p) {
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], p[a]);
      hi[a] = std::max(hi[a], p[a]);
    }
  }
  void grow(const HBox& b) {
    grow(b.lo);
    grow(b.hi);
  }
};

struct Builder {
  const std::vector<HBox>& box;
  double pad;  // node boxes grow by pad (conservative pruning under rounding)
  std::vector<double> cen;  // 3 per primitive
  std::vector<int> order;
  std::vector<Node3> nodes;
  bool sah;  // binned surface-area split instead of the median
  int leaf_max = 4;
  int sah_bins = 16;
  // binned SAH over the centroid bounds (16 bins per axis): the split minimising
  // area(left) x count(left) + area(right) x count(right), as a rank `mid` in
  // the (centroid, index) order along `ax`; the median when no split beats it
  void sah_split(int lo, int hi, const HBox& cb, int& ax, int& mid) {
    const int kB = sah_bins;
    auto area = [](const HBox& b) {
      if (b.lo[0] > b.hi[0]) return 0.0;
      const double e0 = b.hi[0] - b.lo[0], e1 = b.hi[1] - b.lo[1], e2 = b.hi[2] - b.lo[2];
      return e0 * e1 + e1 * e2 + e2 * e0;
    };
    double best = INFINITY;
    int best_ax = ax, best_cnt = (hi - lo) / 2;
    {  // the median's cost along the longest axis: the baseline to beat
      std::vector<int> tmp(order.begin() + lo, order.begin() + hi);
      const int m = (hi - lo) / 2;
      std::nth_element(tmp.begin(), tmp.begin() + m, tmp.end(), [&](int p, int q) {
        double kp = cen[3 * p + ax], kq = cen[3 * q + ax];
        return kp < kq || (kp == kq && p < q);
      });
      HBox l, r;
      for (int i = 0; i < m; ++i) l.grow(box[tmp[i]]);
      for (int i = m; i < hi - lo; ++i) r.grow(box[tmp[i]]);
      best = area(l) * m + area(r) * (hi - lo - m);
    }
    for (int a = 0; a < 3; ++a) {
      const double e = cb.hi[a] - cb.lo[a];
      if (!(e > 0.0)) continue;
      std::vector<HBox> bb(kB);
      std::vector<int> cnt(kB, 0);
      for (int i = lo; i < hi; ++i) {
        const int p = order[i];
        int k = static_cast<int>((cen[3 * p + a] - cb.lo[a]) / e * kB);
        k = k < 0 ? 0 : k >= kB ? kB - 1 : k;
        ++cnt[k];
        bb[k].grow(box[p]);
      }
      std::vector<double> rarea(kB);
      std::vector<int> rcnt(kB);
      HBox acc;
      int c = 0;
      for (int k = kB - 1; k >= 1; --k) {
        acc.grow(bb[k]);
        c += cnt[k];
        rarea[k] = area(acc);
        rcnt[k] = c;
      }
      HBox lacc;
      int lc = 0;
      for (int k = 0; k < kB - 1; ++k) {
        lacc.grow(bb[k]);
        lc += cnt[k];
        if (lc == 0 || rcnt[k + 1] == 0) continue;
        const double cost = area(lacc) * lc + rarea[k + 1] * rcnt[k + 1];
        if (cost < best) {
          best = cost;
          best_ax = a;
          best_cnt = lc;
        }
      }
    }
    ax = best_ax;
    mid = lo + best_cnt;
  }
  Builder(const std::vector<HBox>& b, double pad_, bool sah_ = false, int leaf_max_ = 4, int bins_ = 16)
      : box(b), pad(pad_), cen(3 * b.size()), order(b.size()), sah(sah_), leaf_max(leaf_max_), sah_bins(bins_) {
    for (size_t i = 0; i < b.size(); ++i) {
      order[i] = static_cast<int>(i);
      for (int a = 0; a < 3; ++a) cen[3 * i + a] = 0.5 * (b[i].lo[a] + b[i].hi[a]);
    }
    if (!b.empty()) build(0, static_cast<int>(b.size()));
  }
  int build(int lo, int hi) {
    const int id = static_cast<int>(nodes.size());
    nodes.emplace_back();
    HBox bb, cb;
    for (int i = lo; i < hi; ++i) {
      bb.grow(box[order[i]]);
      cb.grow(&cen[3 * order[i]]);
    }
    Node3 n;
    for (int a = 0; a < 3; ++a) {
      n.lo[a] = round_down(bb.lo[a] - pad);
      n.hi[a] = round_up(bb.hi[a] + pad);
    }
    if (hi - lo <= leaf_max) {
      n.a = lo;
      n.b = -(hi - lo);
      nodes[id] = n;
      return id;
    }
    double ext[3] = {cb.hi[0] - cb.lo[0], cb.hi[1] - cb.lo[1], cb.hi[2] - cb.lo[2]};
    int ax = ext[0] >= ext[1] && ext[0] >= ext[2] ? 0 : (ext[1] >= ext[2] ? 1 : 2);
    int mid = (lo + hi) / 2;
    if (sah) sah_split(lo, hi, cb, ax, mid);
    std::nth_element(order.begin() + lo, order.begin() + mid, order.begin() + hi, [&](int p, int q) {
      double kp = cen[3 * p + ax], kq = cen[3 * q + ax];
      return kp < kq || (kp == kq && p < q);
    });
    n.a = build(lo, mid);
    n.b = build(mid, hi);
    nodes[id] = n;
    return id;
  }
};

// the binary BVH collapsed 4-wide (Node4, wg3_geom.cuh): a node's children
// are its binary children with the internal one of largest surface area
// replaced by its own two children until there are four; boxes are the
// binary nodes' (outward-rounded) boxes
// interior nodes on the longest root-to-leaf path (binary / 4-wide): the
// device's 4-wide traversal stacks need 3 x depth entries
int depth2(const std::vector<Node3>& n, int i = 0) {
  if (n.empty() || n[i].b < 0) return 0;
  return 1 + std::max(depth2(n, n[i].a), depth2(n, n[i].b));
}
int depth4(const std::vector<Node4>& n, int i = 0) {
  if (n.empty()) return 0;
  int d = 0;
  for (int j = 0; j < kBvhW; ++j)
    if (n[i].lox[j] <= n[i].hix[j] && n[i].child[j] >= 0) d = std::max(d, depth4(n, n[i].child[j]));
  return 1 + d;
}
std::vector<Node4> collapse4(const std::vector<Node3>& n3);

bool depths_fit(const std::vector<Node3>& n3, const std::vector<Node4>& n4, const char* what) {
  const int d2 = depth2(n3), d4 = depth4(n4);
  if (std::getenv("WOSTGPU_BVH3_STATS"))
    std::fprintf(stderr, "bvh3 %s: %zu binary nodes depth %d, %zu 4-wide nodes depth %d\n", what, n3.size(), d2,
                 n4.size(), d4);
  // test hook: WOSTGPU_BVH3_STACK lowers the capacity the trees are checked
  // against (it cannot raise it above the device stacks' kStack4)
  int cap = kStack4;
  if (const char* e = std::getenv("WOSTGPU_BVH3_STACK")) cap = std::min(cap, std::max(1, std::atoi(e)));
  return 3 * d4 <= cap;
}

// the BVH of one primitive set: the configured split rule, median splits if
// that tree is too deep for the device stacks, an error if that one is too
struct Tree {
  std::vector<int> order;
  std::vector<Node3> n3;
  std::vector<Node4> n4;
};
Tree build_tree(const std::vector<HBox>& boxes, double pad, bool sah, int leaf_max, int bins, const char* what) {
  Tree t;
  {
    Builder b(boxes, pad, sah, leaf_max, bins);
    t.order = std::move(b.order);
    t.n3 = std::move(b.nodes);
  }
  t.n4 = collapse4(t.n3);
  if (depths_fit(t.n3, t.n4, what)) return t;
  need(sah, WG_ERR_INVALID, std::string("scene BVH too deep for the device traversal stacks: ") + what);
  return build_tree(boxes, pad, false, 4, bins, what);
}

std::vector<Node4> collapse4(const std::vector<Node3>& n3) {
  std::vector<Node4> out;
  if (n3.empty()) return out;
  auto internal = [&](int i) { return n3[i].b >= 0; };
  auto area = [&](int i) {
    const double e[3] = {static_cast<double>(n3[i].hi[0]) - n3[i].lo[0], static_cast<double>(n3[i].hi[1]) - n3[i].lo[1],
                         static_cast<double>(n3[i].hi[2]) - n3[i].lo[2]};
    return e[0] * e[1] + e[1] * e[2] + e[2] * e[0];
  };
  auto leaf_code = [&](int i) {
    const int first = n3[i].a, cnt = -n3[i].b;
    return -((first << 3) | cnt) - 1;
  };
  std::function<int(int)> build = [&](int i) -> int {
    const int id = static_cast<int>(out.size());
    out.emplace_back();
    std::vector<int> kids;
    if (internal(i)) kids = {n3[i].a, n3[i].b};
    else kids = {i};
    while (kids.size() < static_cast<size_t>(kBvhW)) {
      int best = -1;
      double ba = -1.0;
      for (size_t k = 0; k < kids.size(); ++k)
        if (internal(kids[k]) && area(kids[k]) > ba) {
          ba = area(kids[k]);
          best = static_cast<int>(k);
        }
      if (best < 0) break;
      const int c = kids[best];
      kids[best] = n3[c].a;
      kids.insert(kids.begin() + best + 1, n3[c].b);
    }
    Node4 n{};
    for (int j = 0; j < kBvhW; ++j) {
      if (j < static_cast<int>(kids.size())) {
        const Node3& c = n3[kids[j]];
        n.lox[j] = c.lo[0];
        n.loy[j] = c.lo[1];
        n.loz[j] = c.lo[2];
        n.hix[j] = c.hi[0];
        n.hiy[j] = c.hi[1];
        n.hiz[j] = c.hi[2];
        n.child[j] = internal(kids[j]) ? build(kids[j]) : leaf_code(kids[j]);
      } else {  // empty slot: an inverted box is never visited
        n.lox[j] = n.loy[j] = n.loz[j] = INFINITY;
        n.hix[j] = n.hiy[j] = n.hiz[j] = -INFINITY;
        n.child[j] = 0;
      }
    }
    out[id] = n;
    return id;
  };
  build(0);
  return out;
}

void cross3(const double* a, const double* b, double* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

// unit normal of triangle abc: cross(b - a, c - a) * (1 / |.|)
void tri_normal(const double* a, const double* b, const double* c, double* n) {
  double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  double e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  cross3(e1, e2, n);
  double inv = 1.0 / std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
  for (int i = 0; i < 3; ++i) n[i] = n[i] * inv;
}

// silhouette candidates: edges of Neumann triangles keyed by the exact bits
// of their endpoints; one (or > 2) incident triangles -> always, two
// non-coplanar -> crease (facing test at query time), coplanar or convex as
// seen from the domain (n0 . (v1 - a) < 0: never selected by the facing
// rule from inside) -> dropped (oracle/wost3d.inc)
std::vector<Edge3> silhouette_edges(const std::vector<Tri3>& tris, int64_t* n_always, int64_t* n_crease) {
  using VK = std::array<uint64_t, 3>;
  auto key = [](const double* p) {
    VK k;
    std::memcpy(k.data(), p, 24);
    return k;
  };
  struct E {
    double a[3], b[3];
    std::vector<std::array<double, 3>> n, opp;
  };
  std::map<std::pair<VK, VK>, E> m;
  for (const Tri3& t : tris) {
    if (t.kind != WG_NEUMANN) continue;
    std::array<double, 3> n;
    tri_normal(t.a, t.b, t.c, n.data());
    const double* v[3] = {t.a, t.b, t.c};
    for (int i = 0; i < 3; ++i) {
      const double* p = v[i];
      const double* q = v[(i + 1) % 3];
      VK kp = key(p), kq = key(q);
      if (kq < kp) {
        std::swap(kp, kq);
        std::swap(p, q);
      }
      E& e = m[{kp, kq}];
      std::memcpy(e.a, p, 24);
      std::memcpy(e.b, q, 24);
      e.n.push_back(n);
      std::array<double, 3> o;
      std::memcpy(o.data(), v[(i + 2) % 3], 24);
      e.opp.push_back(o);
    }
  }
  std::vector<Edge3> out;
  *n_always = *n_crease = 0;
  for (auto& kv : m) {
    const E& e = kv.second;
    Edge3 g{};
    std::memcpy(g.a, e.a, 24);
    std::memcpy(g.b, e.b, 24);
    if (e.n.size() == 2) {
      const auto &n0 = e.n[0], &n1 = e.n[1];
      if (n0[0] * n1[0] + n0[1] * n1[1] + n0[2] * n1[2] > 1.0 - 1e-9) continue;  // coplanar
      const auto& o1 = e.opp[1];
      if (n0[0] * (o1[0] - e.a[0]) + n0[1] * (o1[1] - e.a[1]) + n0[2] * (o1[2] - e.a[2]) < 0.0) continue;
      g.type = 1;
      std::memcpy(g.n0, n0.data(), 24);
      std::memcpy(g.n1, n1.data(), 24);
      ++*n_crease;
    } else {
      g.type = 0;
      ++*n_always;
    }
    out.push_back(g);
  }
  return out;
}

// ---------------------------------------------------------------- kernels
__global__ void cp3_kernel(Scene3View s, int64_t n, const double* x, uint32_t kinds, double* pt,
                           double* dist, int32_t* tri) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    CP3 c = closest_point(s, {x[3 * i], x[3 * i + 1], x[3 * i + 2]}, kinds);
    pt[3 * i] = c.p.x;
    pt[3 * i + 1] = c.p.y;
    pt[3 * i + 2] = c.p.z;
    dist[i] = c.tri >= 0 ? sqrt(c.d2) : dinf();
    tri[i] = c.tri;
  }
}

__global__ void sil3_kernel(Scene3View s, int64_t n, const double* x, double* dist) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dist[i] = closest_silhouette(s, {x[3 * i], x[3 * i + 1], x[3 * i + 2]});
}

__global__ void ray3_kernel(Scene3View s, int64_t n, const double* o, const double* d,
                            const double* t_max, uint32_t kinds, const int32_t* exclude, double* t,
                            double* pt, double* nrm, int32_t* tri, int32_t* kind) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    D3 oo{o[3 * i], o[3 * i + 1], o[3 * i + 2]}, dd{d[3 * i], d[3 * i + 1], d[3 * i + 2]};
    Hit3 h = ray_first_hit(s, oo, dd, t_max[i], kinds, exclude ? exclude[i] : -1);
    D3 p{0.0, 0.0, 0.0}, nn{0.0, 0.0, 0.0};
    if (h.tri >= 0) {
      p = add(oo, scl(dd, h.t));
      nn = hit_normal(s, h, dd);
    }
    t[i] = h.tri >= 0 ? h.t : dinf();
    pt[3 * i] = p.x;
    pt[3 * i + 1] = p.y;
    pt[3 * i + 2] = p.z;
    nrm[3 * i] = nn.x;
    nrm[3 * i + 1] = nn.y;
    nrm[3 * i + 2] = nn.z;
    tri[i] = h.tri;
    kind[i] = h.tri >= 0 ? h.kind : -1;
  }
}

__global__ void star3_kernel(Scene3View s, int64_t n, const double* x, double r_min, double* r,
                             int* unbounded) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    D3 p{x[3 * i], x[3 * i + 1], x[3 * i + 2]};
    CP3 c = closest_point(s, p, WG_KIND_DIRICHLET);
    double dd = c.tri >= 0 ? sqrt(c.d2) : dinf();
    double ds = closest_silhouette(s, p);
    if (dd == dinf() && ds == dinf()) {
      atomicOr(unbounded, 1);
      r[i] = dinf();
      continue;
    }
    r[i] = fmin(dd, fmax(ds, r_min));
  }
}

int grid_for(int64_t n) {
  int64_t b = (n + 127) / 128;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16)));
}

// device copies of host input arrays for one batched query
struct Staged {
  std::vector<std::unique_ptr<wgrt::DBuf>> bufs;
  template <class T>
  T* in(const T* h, size_t n) {
    if (!h) return nullptr;
    bufs.push_back(std::make_unique<wgrt::DBuf>());
    bufs.back()->upload(h, n);
    return bufs.back()->as<T>();
  }
  template <class T>
  T* out(size_t n) {
    bufs.push_back(std::make_unique<wgrt::DBuf>());
    bufs.back()->alloc(sizeof(T) * (n ? n : 1));
    return bufs.back()->as<T>();
  }
};

template <class T>
void down(T* h, const T* d, size_t n) {
  if (n) CK(cudaMemcpy(h, d, sizeof(T) * n, cudaMemcpyDeviceToHost));
}

}  // namespace
}  // namespace wg3

using namespace wgrt;
using namespace wg3;

extern "C" {

int wostgpu_scene3_create(const double* tri, const int32_t* kind, const int32_t* value_index,
                          int32_t n_tri, const wg_value3_spec* values, int32_t n_values,
                          const wg_value3_spec* source, const double bbox[6], double eps, wg_scene3* out) {
  return guarded([&] {
    check_device();
    need(n_tri > 0, WG_ERR_SCENE, "Accel: empty scene");
    auto s = std::make_unique<wg_scene3_s>();
    CK(cudaGetDevice(&s->device));
    for (int i = 0; i < 6; ++i) s->bbox[i] = bbox[i];
    s->eps = eps > 0.0 ? eps : 1e-3;
    for (int i = 0; i < n_values; ++i)
      need(values[i].type == WG_VALUE_CONSTANT || values[i].type == WG_VALUE_LINEAR, WG_ERR_INVALID,
           "3D scene: values must be constant or linear");
    std::vector<Tri3> tris(static_cast<size_t>(n_tri));
    int32_t has_flux = 0;
    HBox root;
    std::vector<HBox> boxes[2];
    std::vector<int> ids[2];
    for (int i = 0; i < n_tri; ++i) {
      Tri3& t = tris[i];
      std::memcpy(t.a, tri + 9 * i, 24);
      std::memcpy(t.b, tri + 9 * i + 3, 24);
      std::memcpy(t.c, tri + 9 * i + 6, 24);
      t.id = i;
      t.kind = kind[i];
      t.value = value_index[i];
      t.pad_ = 0;
      need(t.kind == WG_DIRICHLET || t.kind == WG_NEUMANN, WG_ERR_SCENE, "3D scene: bad kind");
      need(t.value >= 0 && t.value < n_values, WG_ERR_SCENE, "3D scene: value not defined");
      double nn[3], e1[3], e2[3];
      for (int a = 0; a < 3; ++a) {
        e1[a] = t.b[a] - t.a[a];
        e2[a] = t.c[a] - t.a[a];
      }
      cross3(e1, e2, nn);
      need(std::sqrt(nn[0] * nn[0] + nn[1] * nn[1] + nn[2] * nn[2]) != 0.0, WG_ERR_SCENE,
           "3D scene: degenerate triangle");
      if (eps > 0.0) {
        for (const double* p : {t.a, t.b, t.c})
          for (int a = 0; a < 3; ++a)
            need(p[a] >= bbox[a] && p[a] <= bbox[3 + a], WG_ERR_SCENE, "3D scene: vertex outside scene bbox");
      }
      if (t.kind == WG_NEUMANN && !(values[t.value].type == WG_VALUE_CONSTANT && values[t.value].c0 == 0.0))
        has_flux = 1;  // Scene::has_neumann_flux analogue (scene.cpp:83-91)
      HBox b;
      b.grow(t.a);
      b.grow(t.b);
      b.grow(t.c);
      root.grow(b);
      boxes[t.kind].push_back(b);
      ids[t.kind].push_back(i);
    }
    double rd = 0.0, sd = 0.0;
    for (int a = 0; a < 3; ++a) {
      rd += (root.hi[a] - root.lo[a]) * (root.hi[a] - root.lo[a]);
      sd += (bbox[3 + a] - bbox[a]) * (bbox[3 + a] - bbox[a]);
    }
    s->t_eps = 1e-6 * std::sqrt(rd);
    const double sil_tol = 1e-9 * std::sqrt(rd);
    const double box_pad = 1e-7 * std::sqrt(rd);  // oracle/wost3d.inc Bvh::pad
    s->diag = std::sqrt(sd);
    s->n_tri = n_tri;
    Scene3View& v = s->view;
    v = Scene3View{};
    const char* bvh_env = std::getenv("WOSTGPU_BVH3");  // median | sahN[B] (A/B of the split rule)
    const std::string rule = bvh_env ? bvh_env : "sah2";
    const bool sah = rule.rfind("sah", 0) == 0;
    const int leaf_max = sah && rule.size() >= 4 ? std::max(1, std::min(7, rule[3] - '0')) : (sah ? 2 : 4);
    const int sah_bins = sah && rule.size() > 4 ? std::max(2, std::atoi(rule.c_str() + 4)) : 16;
    for (int k = 0; k < 2; ++k) {
      Tree b = build_tree(boxes[k], box_pad, sah, leaf_max, sah_bins, k == 0 ? "dirichlet" : "neumann");
      std::vector<Tri3> leaf(b.order.size());
      for (size_t i = 0; i < b.order.size(); ++i) leaf[i] = tris[ids[k][b.order[i]]];
      s->n_node[k] = static_cast<int64_t>(b.n3.size());
      if (!b.n3.empty()) {
        s->node[k].upload(b.n3.data(), b.n3.size());
        s->tri[k].upload(leaf.data(), leaf.size());
        v.node[k] = s->node[k].as<Node3>();
        v.tri[k] = s->tri[k].as<Tri3>();
        {  // the 4-wide BVHs (closest point / rays)
          s->node4k[k].upload(b.n4.data(), b.n4.size());
          (k == 0 ? v.node4 : v.node4n) = s->node4k[k].as<Node4>();
        }
        if (k == 0) {  // fp32 boxes of the Dirichlet triangles, rounded outward (closest-point prefilter)
          std::vector<float> tb(8 * leaf.size());
          for (size_t i = 0; i < leaf.size(); ++i) {
            for (int a = 0; a < 3; ++a) {
              const double lo = std::min({leaf[i].a[a], leaf[i].b[a], leaf[i].c[a]});
              const double hi = std::max({leaf[i].a[a], leaf[i].b[a], leaf[i].c[a]});
              float fl = static_cast<float>(lo), fh = static_cast<float>(hi);
              if (static_cast<double>(fl) > lo) fl = std::nextafter(fl, -INFINITY);
              if (static_cast<double>(fh) < hi) fh = std::nextafter(fh, INFINITY);
              tb[8 * i + a] = fl;
              tb[8 * i + 4 + a] = fh;
            }
            tb[8 * i + 3] = tb[8 * i + 7] = 0.0f;
          }
          s->tbox.upload(tb.data(), tb.size());
          v.tbox = reinterpret_cast<const float4*>(s->tbox.as<float>());
        }
      }
    }
    std::vector<Edge3> edges = silhouette_edges(tris, &s->n_always, &s->n_crease);
    if (!edges.empty()) {
      std::vector<HBox> eb(edges.size());
      for (size_t i = 0; i < edges.size(); ++i) {
        eb[i].grow(edges[i].a);
        eb[i].grow(edges[i].b);
      }
      Tree b = build_tree(eb, box_pad, sah, leaf_max, sah_bins, "silhouette edges");
      std::vector<Edge3> leaf(edges.size());
      for (size_t i = 0; i < edges.size(); ++i) leaf[i] = edges[b.order[i]];
      s->n_node[2] = static_cast<int64_t>(b.n3.size());
      s->node[2].upload(b.n3.data(), b.n3.size());
      s->edge.upload(leaf.data(), leaf.size());
      v.node[2] = s->node[2].as<Node3>();
      v.edge = s->edge.as<Edge3>();
      s->node4k[2].upload(b.n4.data(), b.n4.size());
      v.node4e = s->node4k[2].as<Node4>();
    }
    s->values.upload(values, static_cast<size_t>(n_values));
    v.values = s->values.as<wg_value3_spec>();
    for (int i = 0; i < 6; ++i) v.bbox[i] = bbox[i];
    v.t_eps = s->t_eps;
    v.sil_tol = sil_tol;
    v.has_flux = has_flux;
    v.source = wg_value3_spec{};
    v.source.type = WG_VALUE_ZERO;
    if (source && source->type != WG_VALUE_ZERO) {
      need(source->type == WG_VALUE_CONSTANT || source->type == WG_VALUE_LINEAR, WG_ERR_INVALID,
           "3D scene: the source must be constant or linear");
      v.source = *source;
    }
    v.diag = s->diag;
    v.eps = s->eps;
    *out = s.release();
  });
}

int wostgpu_scene3_destroy(wg_scene3 s) {
  return guarded([&] { delete s; });
}

int wostgpu_scene3_info(wg_scene3 s, double* t_eps, int64_t n_nodes[3], int64_t* n_always,
                        int64_t* n_crease) {
  return guarded([&] {
    if (t_eps) *t_eps = s->t_eps;
    if (n_nodes)
      for (int k = 0; k < 3; ++k) n_nodes[k] = s->n_node[k];
    if (n_always) *n_always = s->n_always;
    if (n_crease) *n_crease = s->n_crease;
  });
}

int wostgpu_closest_point3(wg_scene3 s, int64_t n, const double* x, uint32_t kinds, double* pt,
                           double* dist, int32_t* tri) {
  return guarded([&] {
    if (n <= 0) return;
    Staged g;
    const double* dx = g.in(x, 3 * n);
    double* dp = g.out<double>(3 * n);
    double* dd = g.out<double>(n);
    int32_t* dt = g.out<int32_t>(n);
    cp3_kernel<<<grid_for(n), 128>>>(s->view, n, dx, kinds, dp, dd, dt);
    CKL(cudaGetLastError());
    down(pt, dp, 3 * n);
    down(dist, dd, n);
    down(tri, dt, n);
  });
}

int wostgpu_closest_silhouette3(wg_scene3 s, int64_t n, const double* x, double* dist) {
  return guarded([&] {
    if (n <= 0) return;
    Staged g;
    const double* dx = g.in(x, 3 * n);
    double* dd = g.out<double>(n);
    sil3_kernel<<<grid_for(n), 128>>>(s->view, n, dx, dd);
    CKL(cudaGetLastError());
    down(dist, dd, n);
  });
}

int wostgpu_ray_first_hit3(wg_scene3 s, int64_t n, const double* o, const double* d,
                           const double* t_max, uint32_t kinds, const int32_t* exclude, double* t,
                           double* pt, double* nrm, int32_t* tri, int32_t* kind) {
  return guarded([&] {
    if (n <= 0) return;
    Staged g;
    const double* dO = g.in(o, 3 * n);
    const double* dD = g.in(d, 3 * n);
    const double* dT = g.in(t_max, n);
    const int32_t* dE = g.in(exclude, n);
    double* ot = g.out<double>(n);
    double* op = g.out<double>(3 * n);
    double* on = g.out<double>(3 * n);
    int32_t* otri = g.out<int32_t>(n);
    int32_t* okind = g.out<int32_t>(n);
    ray3_kernel<<<grid_for(n), 128>>>(s->view, n, dO, dD, dT, kinds, dE, ot, op, on, otri, okind);
    CKL(cudaGetLastError());
    down(t, ot, n);
    down(pt, op, 3 * n);
    down(nrm, on, 3 * n);
    down(tri, otri, n);
    down(kind, okind, n);
  });
}

int wostgpu_star_radius3(wg_scene3 s, int64_t n, const double* x, double r_min, double* r) {
  return guarded([&] {
    if (n <= 0) return;
    Staged g;
    const double* dx = g.in(x, 3 * n);
    double* dr = g.out<double>(n);
    int* flag = g.out<int>(1);
    CK(cudaMemset(flag, 0, sizeof(int)));
    star3_kernel<<<grid_for(n), 128>>>(s->view, n, dx, r_min, dr, flag);
    CKL(cudaGetLastError());
    int h = 0;
    down(&h, flag, 1);
    need(h == 0, WG_ERR_SCENE, "star_radius: unbounded star region");
    down(r, dr, n);
  });
}

}  // extern "C"
