// Host runtime behind the C-ABI (include/wostgpu.h), part 1: device binding,
// scene + BVH build and upload, batched Accel queries, guiding-field state and
// evaluation. The solver (walk rounds, training, Engine loop) is wg_solver.cu.
#include <dlfcn.h>

#include <functional>
#include <map>

#include "wg_runtime.hpp"

using namespace wg;
using namespace wgrt;

namespace wgrt {
const NcclApi& nccl() {
  static NcclApi api;
  static bool loaded = false;
  if (!loaded) {
    // prefer a copy already mapped by the process (e.g. torch's), else the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    need(h != nullptr, WG_ERR_CUDA, "NCCL (libnccl.so.2) not found");
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.getErrorString = reinterpret_cast<decltype(api.getErrorString)>(dlsym(h, "ncclGetErrorString"));
    need(api.getUniqueId && api.commInitRank && api.allReduce && api.commDestroy && api.getErrorString,
         WG_ERR_CUDA, "NCCL symbols missing");
    loaded = true;
  }
  return api;
}
}  // namespace wgrt

namespace {

// host PCG32 for the field's initial parameters (proj/include/wost/rng.hpp)
struct HostPcg {
  Pcg r;
  HostPcg(uint64_t seed, uint64_t stream) { r.seed(seed, stream); }
  double uni(double lo, double hi) { return lo + (hi - lo) * r.uni(); }
};

DevValue upload_value(const wg_value_spec& v, wg_scene_s* s) {
  DevValue d{};
  d.type = v.type;
  d.analytic_id = v.analytic_id;
  d.c0 = v.c0;
  d.cx = v.cx;
  d.cy = v.cy;
  d.rw = v.raster_w;
  d.rh = v.raster_h;
  for (int i = 0; i < 4; ++i) d.rb[i] = v.raster_bbox[i];
  d.raster = nullptr;
  if (v.type == WG_VALUE_RASTER) {
    need(v.raster_w >= 1 && v.raster_h >= 1 && v.raster_data, WG_ERR_SCENE,
         "raster resolution must be at least 1x1");
    for (int64_t i = 0; i < (int64_t)v.raster_w * v.raster_h; ++i)
      need(std::isfinite(v.raster_data[i]), WG_ERR_SCENE, "raster carries a non-finite cell value");
    auto b = std::make_unique<DBuf>();
    b->upload(v.raster_data, (size_t)v.raster_w * v.raster_h);
    d.raster = b->as<double>();
    s->rasters.push_back(std::move(b));
  }
  return d;
}

// median-split BVH identical to Accel::build (proj/src/geom2d.cpp:109-140):
// same nth_element comparator (centroid along the longer axis, tie by id),
// same leaf size 4, same DFS preorder => the same traversal order and ties
int build_bvh(std::vector<Seg>& segs, std::vector<Node>& nodes, int begin, int end) {
  Node nd;
  nd.lox = nd.loy = dinf();
  nd.hix = nd.hiy = -dinf();
  auto grow = [&](double x, double y) {
    nd.lox = std::min(nd.lox, x);
    nd.loy = std::min(nd.loy, y);
    nd.hix = std::max(nd.hix, x);
    nd.hiy = std::max(nd.hiy, y);
  };
  for (int i = begin; i < end; ++i) {
    grow(segs[i].ax, segs[i].ay);
    grow(segs[i].bx, segs[i].by);
  }
  nd.left = nd.right = -1;
  nd.begin = nd.end = 0;
  int idx = static_cast<int>(nodes.size());
  nodes.push_back(nd);
  if (end - begin <= 4) {
    nodes[idx].begin = begin;
    nodes[idx].end = end;
    return idx;
  }
  double ex = nd.hix - nd.lox, ey = nd.hiy - nd.loy;
  bool sx = ex >= ey;
  int mid = (begin + end) / 2;
  std::nth_element(segs.begin() + begin, segs.begin() + mid, segs.begin() + end,
                   [sx](const Seg& p, const Seg& q) {
                     double cp = sx ? p.ax + p.bx : p.ay + p.by;
                     double cq = sx ? q.ax + q.bx : q.ay + q.by;
                     if (cp != cq) return cp < cq;
                     return p.id < q.id;
                   });
  int l = build_bvh(segs, nodes, begin, mid);
  int r = build_bvh(segs, nodes, mid, end);
  nodes[idx].left = l;
  nodes[idx].right = r;
  return idx;
}



void field_layout(wg_field_s* f) {
  const wg_field_config& c = f->cfg;
  FieldView& v = f->view;
  v.levels = c.n_levels;
  v.F = c.features;
  v.in = c.n_levels * c.features;
  v.hid = c.hidden;
  v.k = c.mixture_k;
  v.dim = c.mixture_dim;
  v.od = (2 + c.mixture_dim) * c.mixture_k + 1;
  int64_t off = 0;
  for (int l = 0; l < c.n_levels; ++l) {
    v.res[l] = c.level_res[l];
    v.lvl_off[l] = static_cast<int32_t>(off);
    off += (int64_t)c.level_res[l] * c.level_res[l] * c.features;
  }
  v.w1 = (int32_t)off;
  off += (int64_t)v.in * v.hid;
  v.b1 = (int32_t)off;
  off += v.hid;
  v.w2 = (int32_t)off;
  off += (int64_t)v.hid * v.hid;
  v.b2 = (int32_t)off;
  off += v.hid;
  v.w3 = (int32_t)off;
  off += (int64_t)v.hid * v.od;
  v.b3 = (int32_t)off;
  off += v.od;
  v.mlp_count = (int32_t)(off - v.w1);
  f->n_params = off;
  for (int i = 0; i < 4; ++i) v.bbox[i] = f->bbox[i];
}

// ---- GuidingField facade kernels (fp64, the reference's operation order;
// this translation unit compiles with -fmad=false)
constexpr int kTapeMax = 256;  // guide_field.cpp:260 (d_h2 / d_h1 / d_in of 256)

// y[j] = b[j] + sum_i x[i] w[i][j], rows in pairs (guide_field.cpp:129-145)
__device__ void affine64(const double* x, int rows, const float* w, const float* b, int cols, double* y) {
  for (int j = 0; j < cols; ++j) y[j] = b[j];
  int i = 0;
  for (; i + 2 <= rows; i += 2) {
    const double x0 = x[i], x1 = x[i + 1];
    const float* w0 = w + static_cast<size_t>(i) * cols;
    const float* w1 = w0 + cols;
    for (int j = 0; j < cols; ++j) y[j] += x0 * w0[j] + x1 * w1[j];
  }
  for (; i < rows; ++i) {
    const double xi = x[i];
    const float* wr = w + static_cast<size_t>(i) * cols;
    for (int j = 0; j < cols; ++j) y[j] += xi * wr[j];
  }
}

// GuidingField::eval_with_tape + backward (guide_field.cpp:223-243, 258-315)
// for one point per thread: grad += J(x)^T d_out, fp64 atomics
__global__ void field_backward_kernel(FieldView f, int64_t n, const double* xy, const double* d_out,
                                      double* grad) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const float* P = f.p;
  double input[kTapeMax], h1pre[kTapeMax], h2pre[kTapeMax], h1[kTapeMax], h2[kTapeMax];
  int64_t cidx[4 * WG_MAX_LEVELS];
  double cw[4 * WG_MAX_LEVELS];
  // gather_input (guide_field.cpp:80-123)
  const double u = sclamp((xy[2 * t] - f.bbox[0]) / (f.bbox[2] - f.bbox[0]), 0.0, 1.0);
  const double v = sclamp((xy[2 * t + 1] - f.bbox[1]) / (f.bbox[3] - f.bbox[1]), 0.0, 1.0);
  for (int l = 0; l < f.levels; ++l) {
    const int res = f.res[l];
    const double px = u * (res - 1), py = v * (res - 1);
    const int ix = imin(static_cast<int>(px), res - 2), iy = imin(static_cast<int>(py), res - 2);
    const double fx = px - ix, fy = py - iy;
    const int64_t c00 = f.lvl_off[l] + (static_cast<int64_t>(iy) * res + ix) * f.F;
    const int64_t c10 = c00 + f.F, c01 = c00 + static_cast<int64_t>(res) * f.F, c11 = c01 + f.F;
    const double w00 = (1.0 - fx) * (1.0 - fy), w10 = fx * (1.0 - fy), w01 = (1.0 - fx) * fy, w11 = fx * fy;
    cidx[4 * l + 0] = c00;
    cidx[4 * l + 1] = c10;
    cidx[4 * l + 2] = c01;
    cidx[4 * l + 3] = c11;
    cw[4 * l + 0] = w00;
    cw[4 * l + 1] = w10;
    cw[4 * l + 2] = w01;
    cw[4 * l + 3] = w11;
    for (int i = 0; i < f.F; ++i)
      input[l * f.F + i] = w00 * P[c00 + i] + w10 * P[c10 + i] + w01 * P[c01 + i] + w11 * P[c11 + i];
  }
  const int in = f.in, hid = f.hid, od = f.od;
  affine64(input, in, P + f.w1, P + f.b1, hid, h1pre);
  for (int i = 0; i < hid; ++i) h1[i] = h1pre[i] > 0.0 ? h1pre[i] : 0.0;
  affine64(h1, hid, P + f.w2, P + f.b2, hid, h2pre);
  for (int i = 0; i < hid; ++i) h2[i] = h2pre[i] > 0.0 ? h2pre[i] : 0.0;
  // backward: d_h2 reuses h1pre's storage after its mask is read, etc.
  const double* dout = d_out + t * od;
  double* d_h2 = h2pre;  // masked in place below
  for (int j = 0; j < od; ++j) atomicAdd(grad + f.b3 + j, dout[j]);
  for (int i = 0; i < hid; ++i) {
    const float* wr = P + f.w3 + static_cast<size_t>(i) * od;
    double* gw = grad + f.w3 + static_cast<size_t>(i) * od;
    double acc = 0.0;
    for (int j = 0; j < od; ++j) {
      atomicAdd(gw + j, h2[i] * dout[j]);
      acc += wr[j] * dout[j];
    }
    d_h2[i] = h2pre[i] > 0.0 ? acc : 0.0;
  }
  double* d_h1 = h2;  // h2 is no longer needed
  for (int j = 0; j < hid; ++j) atomicAdd(grad + f.b2 + j, d_h2[j]);
  for (int i = 0; i < hid; ++i) {
    const float* wr = P + f.w2 + static_cast<size_t>(i) * hid;
    double* gw = grad + f.w2 + static_cast<size_t>(i) * hid;
    double acc = 0.0;
    for (int j = 0; j < hid; ++j) {
      atomicAdd(gw + j, h1[i] * d_h2[j]);
      acc += wr[j] * d_h2[j];
    }
    d_h1[i] = h1pre[i] > 0.0 ? acc : 0.0;
  }
  double* d_in = h1pre;
  for (int j = 0; j < hid; ++j) atomicAdd(grad + f.b1 + j, d_h1[j]);
  for (int i = 0; i < in; ++i) {
    const float* wr = P + f.w1 + static_cast<size_t>(i) * hid;
    double* gw = grad + f.w1 + static_cast<size_t>(i) * hid;
    double acc = 0.0;
    for (int j = 0; j < hid; ++j) {
      atomicAdd(gw + j, input[i] * d_h1[j]);
      acc += wr[j] * d_h1[j];
    }
    d_in[i] = acc;
  }
  for (int l = 0; l < f.levels; ++l)
    for (int c = 0; c < 4; ++c)
      for (int i = 0; i < f.F; ++i) atomicAdd(grad + cidx[4 * l + c] + i, cw[4 * l + c] * d_in[l * f.F + i]);
}

// GuidingField::adam_step (guide_field.cpp:317-331) on an fp64 gradient
__global__ void field_adam64_kernel(float* p, double* m, double* v, const double* g, int64_t n, double lr,
                                    double b1, double b2, double eps, long long step) {
  const double bc1 = 1.0 - pow(b1, static_cast<double>(step));
  const double bc2 = 1.0 - pow(b2, static_cast<double>(step));
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double gi = g[i];
    const double mi = m[i] = b1 * m[i] + (1.0 - b1) * gi;
    const double vi = v[i] = b2 * v[i] + (1.0 - b2) * gi * gi;
    const double up = lr * (mi / bc1) / (sqrt(vi / bc2) + eps);
    p[i] = static_cast<float>(static_cast<double>(p[i]) - up);
  }
}

}  // namespace


extern "C" {

const char* wostgpu_last_error(void) { return g_err.c_str(); }

int wostgpu_init(int device) {
  return guarded([&] {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    need(device >= 0 && device < n, WG_ERR_CUDA, "no such CUDA device");
    CK(cudaSetDevice(device));
    check_device();
  });
}

int wostgpu_device_info(int* sm_count, int* major, int* minor) {
  return guarded([&] {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, dev));
    *sm_count = p.multiProcessorCount;
    *major = p.major;
    *minor = p.minor;
  });
}

int64_t wostgpu_kernel_launches(void) { return g_launches.load(); }

int wostgpu_scene_create(const double* seg, const int32_t* kind, const int32_t* value_index,
                         int32_t n_seg, const wg_value_spec* values, int32_t n_values,
                         const wg_value_spec* source, const double bbox[4], double eps,
                         wg_scene* out) {
  return guarded([&] {
    check_device();
    auto s = std::make_unique<wg_scene_s>();
    for (int i = 0; i < 4; ++i) s->bbox[i] = bbox[i];
    const bool validate = eps > 0.0;
    s->eps = validate ? eps : 1e-3;
    if (validate) {  // Scene::validate, proj/src/scene.cpp:119-143
      need(bbox[0] <= bbox[2] && bbox[1] <= bbox[3], WG_ERR_SCENE, "scene bbox is empty");
      need(n_seg > 0, WG_ERR_SCENE, "scene has no boundary segments");
    }
    need(n_seg > 0, WG_ERR_SCENE, "build_accel: scene has no segments");
    std::vector<int32_t> hk(n_seg), hv(n_seg);
    s->h_segs.resize(n_seg);
    for (int i = 0; i < n_seg; ++i) {
      Seg g;
      g.ax = seg[4 * i];
      g.ay = seg[4 * i + 1];
      g.bx = seg[4 * i + 2];
      g.by = seg[4 * i + 3];
      g.kind = kind[i];
      g.id = i;
      if (validate) {
        std::string w = "segment " + std::to_string(i);
        need(!(g.ax == g.bx && g.ay == g.by), WG_ERR_SCENE, w + ": a == b (zero-length segment)");
        auto in = [&](double x, double y) {
          return x >= bbox[0] && x <= bbox[2] && y >= bbox[1] && y <= bbox[3];
        };
        need(in(g.ax, g.ay) && in(g.bx, g.by), WG_ERR_SCENE, w + ": endpoint outside scene bbox");
        need(value_index[i] >= 0 && value_index[i] < n_values, WG_ERR_SCENE,
             w + ": value is not defined");
      }
      s->h_segs[i] = g;
      hk[i] = kind[i];
      hv[i] = value_index[i];
    }
    // BVH (geom2d.cpp:80-140)
    std::vector<Seg> order = s->h_segs;
    build_bvh(order, s->h_nodes, 0, n_seg);
    {
      double ex = s->h_nodes[0].hix - s->h_nodes[0].lox, ey = s->h_nodes[0].hiy - s->h_nodes[0].loy;
      s->t_eps = 1e-6 * std::sqrt(ex * ex + ey * ey);
    }
    {
      double ex = bbox[2] - bbox[0], ey = bbox[3] - bbox[1];
      s->diag = std::sqrt(ex * ex + ey * ey);
    }
    // Neumann vertex adjacency keyed by exact bits (geom2d.cpp:93-106)
    std::map<std::pair<uint64_t, uint64_t>, int> keymap;
    std::vector<std::vector<double>> normals;
    std::vector<std::pair<double, double>> pos;
    for (const Seg& g : order) {
      if (g.kind != WG_NEUMANN) continue;
      double ux = g.bx - g.ax, uy = g.by - g.ay;
      double px = -uy, py = ux;
      double l = std::sqrt(px * px + py * py);
      double nx = px / l, ny = py / l;
      for (int e = 0; e < 2; ++e) {
        double x = e ? g.bx : g.ax, y = e ? g.by : g.ay;
        uint64_t kx, ky;
        std::memcpy(&kx, &x, 8);
        std::memcpy(&ky, &y, 8);
        auto it = keymap.find({kx, ky});
        int vi;
        if (it == keymap.end()) {
          vi = (int)pos.size();
          keymap[{kx, ky}] = vi;
          pos.push_back({x, y});
          normals.emplace_back();
        } else {
          vi = it->second;
        }
        normals[vi].push_back(nx);
        normals[vi].push_back(ny);
      }
    }
    // silhouette candidates in index order, or (above 32 vertices) in the leaf
    // order of a point BVH (median split on the longer axis, leaves <= 4):
    // closest_silhouette is a minimum over vertices, so any order gives the
    // reference's value (geom2d.cpp:182-200 scans them linearly)
    std::vector<int> vorder(pos.size());
    for (size_t v = 0; v < pos.size(); ++v) vorder[v] = (int)v;
    if (pos.size() > 32) {
      std::function<int(int, int)> build = [&](int b0, int e0) -> int {
        const int id = (int)s->h_sil_nodes.size();
        s->h_sil_nodes.emplace_back();
        Node n{};
        n.lox = n.loy = INFINITY;
        n.hix = n.hiy = -INFINITY;
        for (int i = b0; i < e0; ++i) {
          const auto& p = pos[vorder[i]];
          n.lox = std::min(n.lox, p.first);
          n.loy = std::min(n.loy, p.second);
          n.hix = std::max(n.hix, p.first);
          n.hiy = std::max(n.hiy, p.second);
        }
        if (e0 - b0 <= 4) {
          n.left = n.right = -1;
          n.begin = b0;
          n.end = e0;
        } else {
          const bool ax = (n.hix - n.lox) >= (n.hiy - n.loy);
          const int mid = (b0 + e0) / 2;
          std::nth_element(vorder.begin() + b0, vorder.begin() + mid, vorder.begin() + e0, [&](int a_, int b_) {
            const double ka = ax ? pos[a_].first : pos[a_].second, kb = ax ? pos[b_].first : pos[b_].second;
            return ka < kb || (ka == kb && a_ < b_);
          });
          n.begin = n.end = 0;
          n.left = build(b0, mid);
          n.right = build(mid, e0);
        }
        s->h_sil_nodes[id] = n;
        return id;
      };
      build(0, (int)pos.size());
    }
    for (int v : vorder) {
      SilVertex sv;
      sv.px = pos[v].first;
      sv.py = pos[v].second;
      sv.n_begin = (int32_t)(s->h_sil_n.size() / 2);
      sv.n_count = (int32_t)(normals[v].size() / 2);
      s->h_sil.push_back(sv);
      s->h_sil_n.insert(s->h_sil_n.end(), normals[v].begin(), normals[v].end());
    }
    // values and flux flag (Scene::has_neumann_flux, scene.cpp:83-91)
    std::vector<DevValue> dv;
    for (int i = 0; i < n_values; ++i) dv.push_back(upload_value(values[i], s.get()));
    s->has_flux = 0;
    for (int i = 0; i < n_seg; ++i) {
      if (kind[i] != WG_NEUMANN) continue;
      const wg_value_spec& v = values[value_index[i]];
      if (v.type != WG_VALUE_CONSTANT || v.c0 != 0.0) s->has_flux = 1;
    }
    if (source && source->type != WG_VALUE_ZERO) {
      s->source = upload_value(*source, s.get());
      s->source_zero = 0;
    } else {
      s->source.type = WG_VALUE_ZERO;
      s->source_zero = 1;
    }
    // upload
    s->nodes.upload(s->h_nodes.data(), s->h_nodes.size());
    s->segs.upload(order.data(), order.size());
    s->sil.upload(s->h_sil.data(), s->h_sil.size());
    s->sil_n.upload(s->h_sil_n.data(), s->h_sil_n.size());
    if (!s->h_sil_nodes.empty()) s->sil_nodes.upload(s->h_sil_nodes.data(), s->h_sil_nodes.size());
    s->seg_kind.upload(hk.data(), hk.size());
    s->seg_value.upload(hv.data(), hv.size());
    s->values.upload(dv.data(), dv.size());
    SceneView& v = s->view;
    v.nodes = s->nodes.as<Node>();
    v.segs = s->segs.as<Seg>();
    v.sil = s->sil.as<SilVertex>();
    v.sil_n = s->sil_n.as<double>();
    v.n_nodes = (int32_t)s->h_nodes.size();
    v.n_segs = n_seg;
    v.n_sil = (int32_t)s->h_sil.size();
    v.n_sil_normals = (int32_t)(s->h_sil_n.size() / 2);
    v.sil_nodes = s->h_sil_nodes.empty() ? nullptr : s->sil_nodes.as<Node>();
    v.seg_kind = s->seg_kind.as<int32_t>();
    v.seg_value = s->seg_value.as<int32_t>();
    v.values = s->values.as<DevValue>();
    v.source = s->source;
    for (int i = 0; i < 4; ++i) v.bbox[i] = bbox[i];
    v.eps = s->eps;
    v.t_eps = s->t_eps;
    v.diag = s->diag;
    v.has_flux = s->has_flux;
    v.source_zero = s->source_zero;
    v.n_neumann = 0;
    for (int32_t i = 0; i < n_seg; ++i) v.n_neumann += hk[i] == WG_NEUMANN ? 1 : 0;
    auto a16 = [](size_t b) { return (b + 15) & ~size_t(15); };
    size_t bytes = a16(sizeof(Node) * v.n_nodes) + a16(sizeof(Seg) * v.n_segs) +
                   a16(sizeof(SilVertex) * v.n_sil) + a16(sizeof(double) * 2 * v.n_sil_normals);
    s->smem_bytes = bytes <= 96 * 1024 ? (int)bytes : 0;
    *out = s.release();
  });
}

int wostgpu_scene_destroy(wg_scene s) {
  return guarded([&] { delete s; });
}

int wostgpu_scene_info(wg_scene s, double* t_eps, int32_t* flux, double root_box[4]) {
  return guarded([&] {
    if (t_eps) *t_eps = s->t_eps;
    if (flux) *flux = s->has_flux;
    if (root_box) {
      root_box[0] = s->h_nodes[0].lox;
      root_box[1] = s->h_nodes[0].loy;
      root_box[2] = s->h_nodes[0].hix;
      root_box[3] = s->h_nodes[0].hiy;
    }
  });
}

static int run_query(wg_scene s, int op, int64_t n, const double* xy, const double* dir,
                     const double* tmax, uint32_t kinds, const int32_t* exclude, double r_min,
                     double* out_d, double* out_pt, double* out_n, int32_t* out_seg,
                     int32_t* out_kind) {
  return guarded([&] {
    if (n == 0) return;
    DBuf dxy, ddir, dtm, dex, od, opt, on, oseg, okind, err;
    dxy.upload(xy, 2 * n);
    if (dir) ddir.upload(dir, 2 * n);
    if (tmax) dtm.upload(tmax, n);
    if (exclude) dex.upload(exclude, n);
    od.alloc(sizeof(double) * n);
    opt.alloc(sizeof(double) * 2 * n);
    on.alloc(sizeof(double) * 2 * n);
    oseg.alloc(sizeof(int32_t) * n);
    okind.alloc(sizeof(int32_t) * n);
    err.alloc(8);
    CK(cudaMemset(err.p, 0, 8));
    QueryArgs a{};
    a.scene = s->view;
    a.n = n;
    a.op = op;
    a.kinds = kinds;
    a.r_min = r_min;
    a.xy = dxy.as<double>();
    a.dir = dir ? ddir.as<double>() : nullptr;
    a.t_max = tmax ? dtm.as<double>() : nullptr;
    a.exclude = exclude ? dex.as<int32_t>() : nullptr;
    a.out_d = od.as<double>();
    a.out_pt = opt.as<double>();
    a.out_n = on.as<double>();
    a.out_seg = oseg.as<int32_t>();
    a.out_kind = okind.as<int32_t>();
    a.err = err.as<unsigned long long>();
    CKL(launch_queries(a, 0));
    CK(cudaDeviceSynchronize());
    unsigned long long e = 0;
    CK(cudaMemcpy(&e, err.p, 8, cudaMemcpyDeviceToHost));
    need(e == 0, WG_ERR_SCENE,
         "star_radius: both Dirichlet and silhouette distances are infinite (unbounded star region)");
    if (out_d) CK(cudaMemcpy(out_d, od.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
    if (out_pt) CK(cudaMemcpy(out_pt, opt.p, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost));
    if (out_n) CK(cudaMemcpy(out_n, on.p, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost));
    if (out_seg) CK(cudaMemcpy(out_seg, oseg.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    if (out_kind) CK(cudaMemcpy(out_kind, okind.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  });
}

int wostgpu_closest_point(wg_scene s, int64_t n, const double* xy, uint32_t kinds, double* point,
                          double* dist, int32_t* segment) {
  return run_query(s, 0, n, xy, nullptr, nullptr, kinds, nullptr, 0.0, dist, point, nullptr,
                   segment, nullptr);
}
int wostgpu_closest_silhouette(wg_scene s, int64_t n, const double* xy, double* dist) {
  return run_query(s, 1, n, xy, nullptr, nullptr, 0, nullptr, 0.0, dist, nullptr, nullptr,
                   nullptr, nullptr);
}
int wostgpu_ray_first_hit(wg_scene s, int64_t n, const double* o, const double* d,
                          const double* tmax, uint32_t kinds, const int32_t* exclude, double* t,
                          double* point, double* normal, int32_t* segment, int32_t* kind) {
  return run_query(s, 2, n, o, d, tmax, kinds, exclude, 0.0, t, point, normal, segment, kind);
}
int wostgpu_star_radius(wg_scene s, int64_t n, const double* xy, double r_min, double* r) {
  return run_query(s, 3, n, xy, nullptr, nullptr, 0, nullptr, r_min, r, nullptr, nullptr,
                   nullptr, nullptr);
}

int wostgpu_field_create(const wg_field_config* cfg, const double bbox[4], uint64_t seed,
                         wg_field* out) {
  return guarded([&] {
    check_device();
    const wg_field_config& c = *cfg;
    // GuidingField validation, guide_field.cpp:16-32
    need(c.n_levels >= 1 && c.n_levels <= WG_MAX_LEVELS && c.features >= 1 && c.mixture_k >= 1,
         WG_ERR_INVALID, "guiding field: L, F and K must be >= 1");
    need(c.mixture_k <= WG_MAX_MIXTURE, WG_ERR_INVALID, "guiding field: K exceeds the component cap");
    need(c.mixture_dim == 2 || c.mixture_dim == 3, WG_ERR_INVALID,
         "guiding field: mixture dim must be 2 or 3");
    need(c.hidden >= 1, WG_ERR_INVALID, "guiding field: hidden width must be >= 1");
    for (int l = 0; l < c.n_levels; ++l)
      need(c.level_res[l] >= 2, WG_ERR_INVALID,
           "guiding field: grid resolution must be >= 2 per axis");
    need(c.n_levels * c.features <= 256 && c.hidden <= 256, WG_ERR_INVALID,
         "guiding field: L*F and hidden width are capped at 256");
    need(bbox[0] <= bbox[2] && bbox[1] <= bbox[3] && bbox[2] - bbox[0] > 0.0 &&
             bbox[3] - bbox[1] > 0.0,
         WG_ERR_INVALID, "guiding field: bbox is empty");
    auto f = std::make_unique<wg_field_s>();
    f->cfg = c;
    for (int i = 0; i < 4; ++i) f->bbox[i] = bbox[i];
    field_layout(f.get());
    // initial parameters: the reference's init stream (guide_field.cpp:36-51)
    std::vector<float> p(f->n_params, 0.0f);
    HostPcg rng(Pcg::mix(seed), 0x67e5504410b1426fULL);
    const FieldView& v = f->view;
    for (int64_t i = 0; i < v.w1; ++i) p[i] = static_cast<float>(rng.uni(-1e-4, 1e-4));
    auto layer = [&](int64_t wo, int64_t wc, int64_t bo, int64_t bc, int fan_in) {
      double sc = 1.0 / std::sqrt(static_cast<double>(fan_in));
      for (int64_t i = 0; i < wc; ++i) p[wo + i] = static_cast<float>(rng.uni(-sc, sc));
      for (int64_t i = 0; i < bc; ++i) p[bo + i] = 0.0f;
    };
    layer(v.w1, (int64_t)v.in * v.hid, v.b1, v.hid, v.in);
    layer(v.w2, (int64_t)v.hid * v.hid, v.b2, v.hid, v.hid);
    layer(v.w3, (int64_t)v.hid * v.od, v.b3, v.od, v.hid);
    f->p.upload(p.data(), p.size());
    f->m.alloc(sizeof(double) * f->n_params);
    f->v.alloc(sizeof(double) * f->n_params);
    CK(cudaMemset(f->m.p, 0, sizeof(double) * f->n_params));
    CK(cudaMemset(f->v.p, 0, sizeof(double) * f->n_params));
    f->adam.alloc(sizeof(AdamCtl));
    CK(cudaMemset(f->adam.p, 0, sizeof(AdamCtl)));
    f->view.p = f->p.as<float>();
    *out = f.release();
  });
}

int wostgpu_field_destroy(wg_field f) {
  return guarded([&] { delete f; });
}

int wostgpu_field_param_count(wg_field f, int64_t* n) {
  return guarded([&] { *n = f->n_params; });
}

int wostgpu_field_get_state(wg_field f, float* p, double* m, double* v, int64_t* steps) {
  return guarded([&] {
    CK(cudaDeviceSynchronize());
    if (p) CK(cudaMemcpy(p, f->p.p, sizeof(float) * f->n_params, cudaMemcpyDeviceToHost));
    if (m) CK(cudaMemcpy(m, f->m.p, sizeof(double) * f->n_params, cudaMemcpyDeviceToHost));
    if (v) CK(cudaMemcpy(v, f->v.p, sizeof(double) * f->n_params, cudaMemcpyDeviceToHost));
    if (steps) {
      long long st = 0;
      CK(cudaMemcpy(&st, f->adam.p, sizeof(long long), cudaMemcpyDeviceToHost));
      *steps = st;
    }
  });
}

int wostgpu_field_set_state(wg_field f, const float* p, const double* m, const double* v,
                            int64_t steps) {
  return guarded([&] {
    CK(cudaDeviceSynchronize());
    if (p) {
      CK(cudaMemcpy(f->p.p, p, sizeof(float) * f->n_params, cudaMemcpyHostToDevice));
      f->pack_dirty = true;
    }
    if (m) CK(cudaMemcpy(f->m.p, m, sizeof(double) * f->n_params, cudaMemcpyHostToDevice));
    if (v) CK(cudaMemcpy(f->v.p, v, sizeof(double) * f->n_params, cudaMemcpyHostToDevice));
    if (steps >= 0) {
      long long st = steps;
      CK(cudaMemcpy(f->adam.p, &st, sizeof(long long), cudaMemcpyHostToDevice));
    }
  });
}

int wostgpu_field_eval_batch(wg_field f, int64_t n, const double* xy, double* out, int mlp) {
  return guarded([&] {
    need(f->sdim == 2, WG_ERR_INVALID, "field_eval_batch: 3D field (use wostgpu_field3_eval_batch)");
    need(mlp == WG_MLP_EXACT || default_shape(f->view), WG_ERR_NOT_BUILT,
         "tensor-core field evaluation is built for the default field shape");
    if (n == 0) return;
    DBuf dxy, dout;
    dxy.upload(xy, 2 * n);
    dout.alloc(sizeof(double) * n * f->view.od);
    if (mlp == WG_MLP_TENSOR) {
      CKL(launch_field_eval_tc(f->view, n, dxy.as<double>(), dout.as<double>(), sm_count(), 0));
    } else {
      CKL(launch_field_eval(f->view, n, dxy.as<double>(), dout.as<double>(), 0));
    }
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out, dout.p, sizeof(double) * n * f->view.od, cudaMemcpyDeviceToHost));
  });
}

int wostgpu_field_get_params(wg_field f, int64_t offset, int64_t count, float* out) {
  return guarded([&] {
    need(f != nullptr && offset >= 0 && count >= 0 && offset + count <= f->n_params, WG_ERR_INVALID,
         "parameter range out of bounds");
    if (count == 0) return;
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out, f->p.as<float>() + offset, sizeof(float) * count, cudaMemcpyDeviceToHost));
  });
}

int wostgpu_field_set_params(wg_field f, int64_t offset, int64_t count, const float* in) {
  return guarded([&] {
    need(f != nullptr && offset >= 0 && count >= 0 && offset + count <= f->n_params, WG_ERR_INVALID,
         "parameter range out of bounds");
    if (count == 0) return;
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(f->p.as<float>() + offset, in, sizeof(float) * count, cudaMemcpyHostToDevice));
    f->pack_dirty = true;
  });
}

int wostgpu_field_backward(wg_field f, int64_t n, const double* xy, const double* d_out, double* grad) {
  return guarded([&] {
    need(f != nullptr && f->sdim == 2, WG_ERR_INVALID, "field_backward: 2D field expected");
    need(f->view.in <= kTapeMax && f->view.hid <= kTapeMax, WG_ERR_NOT_BUILT, "field too wide for the tape");
    if (n == 0) return;
    DBuf dxy, dd, dg;
    dxy.upload(xy, 2 * n);
    dd.upload(d_out, static_cast<size_t>(n) * f->view.od);
    dg.upload(grad, static_cast<size_t>(f->n_params));
    field_backward_kernel<<<static_cast<unsigned>((n + 63) / 64), 64>>>(f->view, n, dxy.as<double>(),
                                                                         dd.as<double>(), dg.as<double>());
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(grad, dg.p, sizeof(double) * f->n_params, cudaMemcpyDeviceToHost));
  });
}

int wostgpu_field_adam_step(wg_field f, double* grad, double lr, double beta1, double beta2, double eps) {
  return guarded([&] {
    need(f != nullptr && grad != nullptr, WG_ERR_INVALID, "null argument");
    CK(cudaDeviceSynchronize());
    long long steps = 0;
    CK(cudaMemcpy(&steps, f->adam.p, sizeof(long long), cudaMemcpyDeviceToHost));
    ++steps;
    DBuf dg;
    dg.upload(grad, static_cast<size_t>(f->n_params));
    field_adam64_kernel<<<sm_count() * 4, 256>>>(f->p.as<float>(), f->m.as<double>(), f->v.as<double>(),
                                                  dg.as<double>(), f->n_params, lr, beta1, beta2, eps, steps);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(f->adam.p, &steps, sizeof(long long), cudaMemcpyHostToDevice));
    f->pack_dirty = true;
    for (int64_t i = 0; i < f->n_params; ++i) grad[i] = 0.0;  // as adam_step leaves it
  });
}

int wostgpu_shutdown(void) {
  return guarded([&] { CK(cudaDeviceSynchronize()); });
}

int wostgpu_normalize_params(int64_t n, const double* raw, int32_t k, int32_t dim, wg_mixture* out) {
  return guarded([&] {
    need(dim == 2, WG_ERR_NOT_BUILT, "device normalisation is built for dim 2");
    need(k >= 1 && k <= WG_MAX_MIXTURE, WG_ERR_INVALID, "mixture size out of range");
    if (n == 0) return;
    const int od = (2 + dim) * k + 1;
    DBuf draw, dout;
    draw.upload(raw, (size_t)n * od);
    dout.alloc(sizeof(wg_mixture) * n);
    CKL(launch_normalize(n, draw.as<double>(), k, dim, dout.as<wg_mixture>(), 0));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out, dout.p, sizeof(wg_mixture) * n, cudaMemcpyDeviceToHost));
  });
}

int wostgpu_mixture32_pdf(int64_t n, const float* raw, const double* nu, double* out) {
  return guarded([&] {
    if (n == 0) return;
    DBuf draw, dnu, dout;
    draw.upload(raw, (size_t)n * 33);
    dnu.upload(nu, (size_t)n * 2);
    dout.alloc(sizeof(double) * 2 * n);
    CKL(launch_mix32_pdf(draw.as<float>(), n, dnu.as<double>(), dout.as<double>(), 0));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out, dout.p, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost));
  });
}

int wostgpu_mixture32_sample(const float* raw, int64_t n, uint64_t seed, double* nu_out) {
  return guarded([&] {
    if (n == 0) return;
    DBuf draw, dout;
    draw.upload(raw, 33);
    dout.alloc(sizeof(double) * 2 * n);
    CKL(launch_mix32_sample(draw.as<float>(), n, seed, dout.as<double>(), 0));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(nu_out, dout.p, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
