// Guided walk kernel, one warp per walk (default-shape field, fp32 MLP).
//
// The per-step chain of a guided walk (begin_step -> field eval -> decode ->
// sample -> move, proj/src/wost.cpp:111-264) is latency-bound: a round lasts
// as long as its longest walk. Here the 32 lanes of a warp carry ONE walk:
// the walk state is replicated in every lane (warp-uniform control flow, lane
// 0 performs all side effects), and the parallel parts of a step are split:
//   * MLP 16 -> 64 -> 64 -> 33: lane j owns hidden units j and j + 32 and
//     output j (lane 0 also output 32); weights in shared memory laid out so
//     each weight load is one conflict-free 32-lane access; activations are
//     exchanged through a 64-float per-warp buffer (broadcast reads);
//   * Table-1 decode and the mixture density: lanes 0-7 each own one lobe
//     (lanes 8-31 mirror them), softmax / density sums by xor shuffles;
//   * lobe selection: inclusive prefix scan of the weights over the lobe lanes.
// Geometry, Best-Fisher and the move run redundantly in all lanes on the
// same state and the same PCG32 stream, so every lane takes the same path.
// Walks are handed out dynamically (one atomic per walk), so long walks do
// not serialise behind a static slot. The mixture numerics are those of the
// tensor-core path (wg_mix32.cuh); the MLP is fp32 FMA with a
// different summation order than the reference (~1e-6 relative).
#include <cstdio>

#include "wg_kernels.cuh"
#include "wg_mix32.cuh"
#include "wg_train.cuh"
#include "wg_walk_common.cuh"

namespace wg {

namespace {

constexpr int kCoopWarps = 8;
constexpr int kCoopThreads = 32 * kCoopWarps;

// shared-memory weights: W1/W2 as (column j, column j + 32) float2 pairs per
// input row, W3 rows of 33 padded to 33 (lane j reads column j), biases
struct CoopW {
  float2 w1[16][32];
  float2 w2[64][32];
  float w3[64][33];
  float b1[64], b2[64], b3[33];
};

__host__ __device__ __forceinline__ size_t al16c(size_t b) { return (b + 15) & ~size_t(15); }

struct CLane {
  double x, y, nx, ny, T, acc, R;
  int seg, depth, rec;
  bool on_n;
  Pcg rng;
  int64_t point;
  int round;
  int64_t rec_base;
  int rec_left, last_rec;
  double dacc;  // accumulator increments since the last record (DevRecord::dacc)
  bool rec_ok;
};

// ---- lane-parallel small-scene geometry (<= 32 segments / vertices of a
// kind): lane i tests segment i, then an argmin over (distance, index). The
// smallest index among equal distances wins, which is exactly the winner of
// the sequential strict-< scan in visiting order (cp_list / ray_list /
// sil_small); ray hits keep the reference's "last equal t wins" with the
// largest index. Results are identical to the per-thread functions.
__device__ __forceinline__ CP w_cp_list(const Seg* segs, int n, double x, double y, int lane) {
  double d2 = dinf(), px = 0.0, py = 0.0;
  int id = -1;
  if (lane < n) {
    const Seg g = segs[lane];
    double ux = g.bx - g.ax, uy = g.by - g.ay;
    double t = ((x - g.ax) * ux + (y - g.ay) * uy) / (ux * ux + uy * uy);
    t = sclamp(t, 0.0, 1.0);
    px = g.ax + t * ux;
    py = g.ay + t * uy;
    double dx = px - x, dy = py - y;
    d2 = dx * dx + dy * dy;
    id = g.id;
  }
  int src = lane;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double od = __shfl_xor_sync(0xffffffffu, d2, o);
    const int os = __shfl_xor_sync(0xffffffffu, src, o);
    if (od < d2 || (od == d2 && os < src)) {
      d2 = od;
      src = os;
    }
  }
  CP best;
  best.px = __shfl_sync(0xffffffffu, px, src);
  best.py = __shfl_sync(0xffffffffu, py, src);
  best.seg = __shfl_sync(0xffffffffu, id, src);
  best.d = best.seg >= 0 && d2 < dinf() ? sqrt(d2) : dinf();
  if (!(d2 < dinf())) best.seg = -1;
  return best;
}

__device__ __forceinline__ Hit w_ray_list(const Seg* segs, int n, double t_eps, double ox, double oy, double dx,
                                          double dy, double t_max, int exclude, int lane) {
  double t = dinf(), sp = 0.0;
  bool ok = false;
  if (lane < n) {
    const Seg g = segs[lane];
    double ux = g.bx - g.ax, uy = g.by - g.ay;
    double wx = g.ax - ox, wy = g.ay - oy;
    double den = dx * uy - dy * ux;
    const bool nz = den != 0.0;
    const double dd = nz ? den : 1.0;
    t = (wx * uy - wy * ux) / dd;
    sp = (wx * dy - wy * dx) / dd;
    ok = g.id != exclude && nz && !(sp < 0.0 || sp > 1.0) && t > t_eps && t <= t_max;
  }
  if (!ok) t = dinf();
  int src = ok ? lane : -1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {  // min t, ties -> largest index (last equal wins)
    const double ot = __shfl_xor_sync(0xffffffffu, t, o);
    const int os = __shfl_xor_sync(0xffffffffu, src, o);
    if (ot < t || (ot == t && os > src)) {
      t = ot;
      src = os;
    }
  }
  Hit h;
  h.seg = -1;
  h.kind = -1;
  h.t = dinf();
  h.px = h.py = h.nx = h.ny = 0.0;
  if (src < 0) return h;
  const double bsp = __shfl_sync(0xffffffffu, sp, src);
  const Seg g = segs[src];
  h.t = t;
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

__device__ __forceinline__ double w_sil(const SceneView& s, double x, double y, int lane) {
  double d = dinf();
  if (lane < s.n_sil) {
    const SilVertex sv = s.sil[lane];
    const double dx = sv.px - x, dy = sv.py - y;
    const double dd = dx * dx + dy * dy;
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
    if (cand) d = dd;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d = fmin(d, __shfl_xor_sync(0xffffffffu, d, o));
  return d == dinf() ? d : sqrt(d);
}

__device__ __forceinline__ CP w_closest(const SceneView& s, const SmallSegs& ss, double x, double y, int lane) {
  if (s.n_segs > kSmallScene) return closest_point(s, x, y, WG_KIND_DIRICHLET);
  return w_cp_list(ss.d, ss.nd, x, y, lane);
}

__device__ __forceinline__ Hit w_ray_neumann(const SceneView& s, const SmallSegs& ss, double ox, double oy,
                                             double dx, double dy, double t_max, int exclude, int lane) {
  if (s.n_segs > kSmallScene) return ray_first_hit(s, ox, oy, dx, dy, t_max, WG_KIND_NEUMANN, exclude);
  return w_ray_list(ss.n, ss.nn, s.t_eps, ox, oy, dx, dy, t_max, exclude, lane);
}

__device__ __forceinline__ void c_finish(const CLane& w, const WalkArgs& a, bool escaped, int lane,
                                         double terminal = 0.0) {
  if (lane == 0) {
    const int64_t slot = static_cast<int64_t>(w.round) * a.n_points + w.point;
    if (a.rec_tail) {  // the walk's end of the record chain (see DevRecord)
      a.rec_tail[slot] = w.last_rec;
      a.rec_term[slot] = escaped ? 0.0 : w.T * terminal + w.dacc;
    }
    a.est[slot] = escaped ? 0.0 : w.acc;
    a.esc[slot] = escaped ? 1 : 0;
    if (a.steps) a.steps[slot] = w.depth;
    atomicAdd(&a.counters[0], static_cast<unsigned long long>(w.depth));
    if (escaped) atomicAdd(&a.counters[1], 1ull);
  }
}

// begin_step (wost.cpp:148-216), warp-uniform; false when the walk ended
__device__ __forceinline__ bool c_begin(CLane& w, const WalkArgs& a, const SceneView& s, const SmallSegs& ss,
                                        bool collect, int lane) {
  CP cd = w_closest(s, ss, w.x, w.y, lane);
  if (cd.seg >= 0 && cd.d <= a.sp.eps) {
    double g = eval_value(s.values[s.seg_value[cd.seg]], cd.px, cd.py);
    w.acc += w.T * g;
    c_finish(w, a, false, lane, g);
    return false;
  }
  if (w.depth >= a.sp.max_steps) {
    c_finish(w, a, true, lane);
    return false;
  }
  if (w.depth > a.sp.rr_depth) {
    double q = smin(1.0, fabs(w.T));
    if (q <= 0.0 || w.rng.uni() >= q) {
      c_finish(w, a, false, lane);
      return false;
    }
    w.T /= q;
  }
  double dsil = s.n_sil <= 32 ? w_sil(s, w.x, w.y, lane) : closest_silhouette(s, w.x, w.y);
  double dd = cd.seg >= 0 ? cd.d : dinf();
  if (dd == dinf() && dsil == dinf()) {
    if (lane == 0) atomicOr(&a.counters[4], 1ull);
    c_finish(w, a, true, lane);
    return false;
  }
  w.R = smin(dd, smax(dsil, a.sp.rmin));
  double contrib = 0.0;
  if (!s.source_zero) {
    double dx, dy;
    uniform_sample32(w.rng, w.on_n, w.nx, w.ny, &dx, &dy);
    double r = t_greens_radius(w.rng.uni(), w.R);
    double yx = w.x + dx * r, yy = w.y + dy * r;
    Hit h = source_ray_needed(s, r, w.R) ? t_ray(s, ss, w.x, w.y, dx, dy, r, WG_KIND_ALL, -1) : no_hit();
    double wt = h.seg >= 0 ? 0.0 : w.R * w.R / 4.0;
    if (wt != 0.0) {
      double f = 0.0;
      if (bbox_contains(s, yx, yy, 0.0)) f = eval_value(s.source, yx, yy);
      contrib -= wt * f;
    }
  }
  if (s.has_flux) {
    double dx, dy;
    uniform_sample32(w.rng, w.on_n, w.nx, w.ny, &dx, &dy);
    Hit h = w_ray_neumann(s, ss, w.x, w.y, dx, dy, w.R, w.seg, lane);
    double add = 0.0;
    if (h.seg >= 0) {
      double hv = eval_value(s.values[s.seg_value[h.seg]], h.px, h.py);
      if (hv != 0.0) {
        double cz = fabs(dx * h.nx + dy * h.ny);
        if (a.sp.clamp_grazing) cz = smax(cz, a.sp.grazing_floor);
        if (cz != 0.0) add = (h.t <= 0.0 ? dinf() : log(w.R / h.t) / kTwoPi) * hv * h.t * kTwoPi / cz;
      }
    }
    contrib += add;
  }
  w.acc += w.T * contrib;
  w.dacc += w.T * contrib;
  w.rec = -1;
  if (collect && w.rec_ok) {
    if (w.rec_left == 0) {
      unsigned long long b = 0;
      if (lane == 0) b = atomicAdd(a.rec_counter, 8ull);
      b = __shfl_sync(0xffffffffu, b, 0);
      if (static_cast<int64_t>(b) + 8 > a.rec_capacity) {
        w.rec_ok = false;
        if (lane == 0) atomicAdd(&a.counters[3], 1ull);
      } else {
        w.rec_base = static_cast<int64_t>(b);
        w.rec_left = 8;
      }
    }
    if (w.rec_ok) {
      w.rec = static_cast<int>(w.rec_base + (8 - w.rec_left));
      --w.rec_left;
    }
  }
  return true;
}

// the walk's 16 grid features (guide_field.cpp:80-123), every lane
__device__ __forceinline__ void c_gather(const FieldView& f, double x, double y, float* in) {
  double ex = f.bbox[2] - f.bbox[0], ey = f.bbox[3] - f.bbox[1];
  float u = static_cast<float>(sclamp((x - f.bbox[0]) / ex, 0.0, 1.0));
  float v = static_cast<float>(sclamp((y - f.bbox[1]) / ey, 0.0, 1.0));
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const int res = f.res[l];
    float px = u * static_cast<float>(res - 1), py = v * static_cast<float>(res - 1);
    int ix = imin(static_cast<int>(px), res - 2), iy = imin(static_cast<int>(py), res - 2);
    float fx = px - ix, fy = py - iy;
    const float4* base = reinterpret_cast<const float4*>(f.p + f.lvl_off[l] + (iy * res + ix) * 4);
    float4 p00 = __ldg(base), p10 = __ldg(base + 1), p01 = __ldg(base + res), p11 = __ldg(base + res + 1);
    float w00 = (1.0f - fx) * (1.0f - fy), w10 = fx * (1.0f - fy);
    float w01 = (1.0f - fx) * fy, w11 = fx * fy;
    in[4 * l + 0] = (w00 * p00.x + w10 * p10.x) + (w01 * p01.x + w11 * p11.x);
    in[4 * l + 1] = (w00 * p00.y + w10 * p10.y) + (w01 * p01.y + w11 * p11.y);
    in[4 * l + 2] = (w00 * p00.z + w10 * p10.z) + (w01 * p01.z + w11 * p11.z);
    in[4 * l + 3] = (w00 * p00.w + w10 * p10.w) + (w01 * p01.w + w11 * p11.w);
  }
}

// MLP for the warp's walk: returns output `lane` (and output 32 in *y32)
__device__ __forceinline__ float c_mlp(const CoopW& W, float* hb, const float* x, int lane, float* y32) {
  float a0 = W.b1[lane], a1 = W.b1[lane + 32], c0 = 0.0f, c1 = 0.0f;
#pragma unroll
  for (int k = 0; k < 16; k += 2) {
    const float2 u = W.w1[k][lane], v = W.w1[k + 1][lane];
    a0 = fmaf(u.x, x[k], a0);
    a1 = fmaf(u.y, x[k], a1);
    c0 = fmaf(v.x, x[k + 1], c0);
    c1 = fmaf(v.y, x[k + 1], c1);
  }
  hb[lane] = fmaxf(a0 + c0, 0.0f);
  hb[lane + 32] = fmaxf(a1 + c1, 0.0f);
  __syncwarp();
  a0 = W.b2[lane];
  a1 = W.b2[lane + 32];
  c0 = c1 = 0.0f;
  float e0 = 0.0f, e1 = 0.0f, f0 = 0.0f, f1 = 0.0f;
#pragma unroll
  for (int k = 0; k < 64; k += 4) {
    const float4 h = *reinterpret_cast<const float4*>(hb + k);
    const float2 p = W.w2[k][lane], q = W.w2[k + 1][lane], r = W.w2[k + 2][lane], t = W.w2[k + 3][lane];
    a0 = fmaf(p.x, h.x, a0);
    a1 = fmaf(p.y, h.x, a1);
    c0 = fmaf(q.x, h.y, c0);
    c1 = fmaf(q.y, h.y, c1);
    e0 = fmaf(r.x, h.z, e0);
    e1 = fmaf(r.y, h.z, e1);
    f0 = fmaf(t.x, h.w, f0);
    f1 = fmaf(t.y, h.w, f1);
  }
  __syncwarp();
  hb[lane] = fmaxf((a0 + c0) + (e0 + f0), 0.0f);
  hb[lane + 32] = fmaxf((a1 + c1) + (e1 + f1), 0.0f);
  __syncwarp();
  float o0 = W.b3[lane], o1 = 0.0f, o2 = 0.0f, o3 = 0.0f;
#pragma unroll
  for (int k = 0; k < 64; k += 4) {
    const float4 h = *reinterpret_cast<const float4*>(hb + k);
    o0 = fmaf(W.w3[k][lane], h.x, o0);
    o1 = fmaf(W.w3[k + 1][lane], h.y, o1);
    o2 = fmaf(W.w3[k + 2][lane], h.z, o2);
    o3 = fmaf(W.w3[k + 3][lane], h.w, o3);
  }
  // output 32 (selection logit): lane j takes hidden units j and j + 32
  float z = fmaf(W.w3[lane][32], hb[lane], W.w3[lane + 32][32] * hb[lane + 32]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  *y32 = W.b3[32] + z;
  __syncwarp();  // hb is rewritten by the next step
  return (o0 + o1) + (o2 + o3);
}

// one lobe per lane (lane & 7), fp32 Table-1 decode (wg_mix32.cuh numerics)
struct Lobe {
  float mux, muy, kappa, lambda, lne, hk;
};

__device__ __forceinline__ float sum8(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  return v;
}

__device__ __forceinline__ Lobe c_decode(float y, float y32, int lane, double* c_out) {
  const int i = lane & 7;
  const float mx = __shfl_sync(0xffffffffu, y, 2 * i), my = __shfl_sync(0xffffffffu, y, 2 * i + 1);
  const float kr = __shfl_sync(0xffffffffu, y, 16 + i), lr = __shfl_sync(0xffffffffu, y, 24 + i);
  const float cr = __shfl_sync(0xffffffffu, y32, 0);
  Lobe L;
  const float n2 = mx * mx + my * my;
  const float rn = rsqrtf(n2);
  if (n2 >= 1e-24f) {
    L.mux = mx * rn;
    L.muy = my * rn;
  } else {  // fallback_mu (sphdist.cpp:274-278)
    sincospif(0.25f * static_cast<float>(i), &L.muy, &L.mux);
  }
  const float lk = fminf(fmaxf(kr, -13.81551056f), 9.210340372f);
  L.kappa = __expf(lk);
  const float eps = fmaf(L.mux, L.mux, fmaf(L.muy, L.muy, -1.0f));
  L.hk = L.kappa * fmaf(-0.25f, eps, 0.5f);
  L.lne = -log_i0e_k(L.kappa, lk, __expf(-lk)) - 1.8378770664093453f;
  float mxl = lr;
  mxl = fmaxf(mxl, __shfl_xor_sync(0xffffffffu, mxl, 1));
  mxl = fmaxf(mxl, __shfl_xor_sync(0xffffffffu, mxl, 2));
  mxl = fmaxf(mxl, __shfl_xor_sync(0xffffffffu, mxl, 4));
  const float e = __expf(lr - mxl);
  L.lambda = e * __frcp_rn(sum8(e));
  const float ec = __expf(-fabsf(cr));
  const float sg = 1.0f / (1.0f + ec);
  // c in fp64 from the logit: an fp32 sigmoid rounds to 1 above ~16.6 and
  // would drop the defensive (1 - c) p_u term from p_mis
  (void)sg;
  (void)ec;
  *c_out = sigmoid(static_cast<double>(cr));
  return L;
}

// mixture density at unit nu: sum over the 8 lobe lanes (|nu - mu| form)
__device__ __forceinline__ double c_pdf(const Lobe& L, double nx, double ny) {
  const float fx = static_cast<float>(nx), fy = static_cast<float>(ny);
  const float lx = static_cast<float>(nx - static_cast<double>(fx));
  const float ly = static_cast<float>(ny - static_cast<double>(fy));
  const float dx = (fx - L.mux) + lx, dy = (fy - L.muy) + ly;
  return sum8(L.lambda * __expf(fmaf(-L.hk, fmaf(dx, dx, dy * dy), L.lne)));
}

// ancestral draw: lobe by prefix scan over the lobe lanes, Best-Fisher on it
__device__ __forceinline__ void c_mixture_sample(Pcg& rng, const Lobe& L, int lane, double* ox, double* oy) {
  const float u = rng.unif();
  const int i = lane & 7;
  float acc = L.lambda;
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
    const float t = __shfl_up_sync(0xffffffffu, acc, o, 8);
    if (i >= o) acc += t;
  }
  const unsigned hit = __ballot_sync(0xffffffffu, u < acc) & 0xFFu;
  const int pick = hit ? __ffs(hit) - 1 : 7;
  const float mux = __shfl_sync(0xffffffffu, L.mux, pick);
  const float muy = __shfl_sync(0xffffffffu, L.muy, pick);
  const float kap = __shfl_sync(0xffffffffu, L.kappa, pick);
  float c, sn;
  vm_cos_sin(rng, kap, &c, &sn);
  unit64(c * mux - sn * muy, c * muy + sn * mux, ox, oy);
}

}  // namespace

// finish the walks the lockstep kernel handed off (WalkArgs::spill), one
// warp per walk (a standalone warp-per-walk kernel that also started fresh
// walks measured slower than the lockstep tiles on cfg 2)
#ifdef WG_COOP_PROF
__device__ unsigned long long g_coop_prof[7];
void coop_prof_dump() {
  unsigned long long p[7];
  cudaMemcpyFromSymbol(p, g_coop_prof, sizeof(p));
  const double n = p[6] ? double(p[6]) : 1.0;
  std::fprintf(stderr, "coop prof steps %llu cycles/step: begin %.0f gather %.0f mlp %.0f decode %.0f sample+pdf %.0f record+ray %.0f\n",
               p[6], p[0] / n, p[1] / n, p[2] / n, p[3] / n, p[4] / n, p[5] / n);
  const unsigned long long z[7] = {};
  cudaMemcpyToSymbol(g_coop_prof, z, sizeof(z));
}
#endif
__device__ __forceinline__ void walk_coop_body(const WalkArgs& a, unsigned char* smem) {
  CoopW& W = *reinterpret_cast<CoopW*>(smem);
  float* hbuf = reinterpret_cast<float*>(smem + al16c(sizeof(CoopW))) + 64 * (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  SceneView s = a.scene;
  if (a.scene_smem_bytes > 0) {
    unsigned char* p = smem + al16c(sizeof(CoopW)) + sizeof(float) * 64 * kCoopWarps;
    size_t off = 0;
    auto carve = [&](size_t bytes) {
      unsigned char* q = p + off;
      off += al16c(bytes);
      return q;
    };
    Node* nodes = reinterpret_cast<Node*>(carve(sizeof(Node) * s.n_nodes));
    Seg* segs = reinterpret_cast<Seg*>(carve(sizeof(Seg) * s.n_segs));
    SilVertex* sil = reinterpret_cast<SilVertex*>(carve(sizeof(SilVertex) * s.n_sil));
    double* sn = reinterpret_cast<double*>(carve(sizeof(double) * 2 * s.n_sil_normals));
    for (int i = threadIdx.x; i < s.n_nodes; i += blockDim.x) nodes[i] = a.scene.nodes[i];
    for (int i = threadIdx.x; i < s.n_segs; i += blockDim.x) segs[i] = a.scene.segs[i];
    for (int i = threadIdx.x; i < s.n_sil; i += blockDim.x) sil[i] = a.scene.sil[i];
    for (int i = threadIdx.x; i < 2 * s.n_sil_normals; i += blockDim.x) sn[i] = a.scene.sil_n[i];
    s.nodes = nodes;
    s.segs = segs;
    s.sil = sil;
    s.sil_n = sn;
  }
  __shared__ Seg seg_lists[2 * kSmallScene];
  __shared__ int seg_counts[2];
  if (s.n_segs <= kSmallScene && threadIdx.x == 0) {
    int nd = 0, nn = 0;
    for (int i = 0; i < s.n_segs; ++i) {
      const Seg g = s.segs[i];
      if (g.kind == WG_DIRICHLET) seg_lists[nd++] = g;
      else seg_lists[kSmallScene + nn++] = g;
    }
    seg_counts[0] = nd;
    seg_counts[1] = nn;
  }
  // weights (row-major [in][out] params, guide_field.cpp layout)
  const FieldView& f = a.field;
  for (int e = threadIdx.x; e < 16 * 32; e += blockDim.x) {
    const int k = e / 32, j = e % 32;
    W.w1[k][j] = make_float2(f.p[f.w1 + k * 64 + j], f.p[f.w1 + k * 64 + j + 32]);
  }
  for (int e = threadIdx.x; e < 64 * 32; e += blockDim.x) {
    const int k = e / 32, j = e % 32;
    W.w2[k][j] = make_float2(f.p[f.w2 + k * 64 + j], f.p[f.w2 + k * 64 + j + 32]);
  }
  for (int e = threadIdx.x; e < 64 * 33; e += blockDim.x) W.w3[e / 33][e % 33] = f.p[f.w3 + e];
  for (int e = threadIdx.x; e < 64; e += blockDim.x) {
    W.b1[e] = f.p[f.b1 + e];
    W.b2[e] = f.p[f.b2 + e];
  }
  for (int e = threadIdx.x; e < 33; e += blockDim.x) W.b3[e] = f.p[f.b3 + e];
  __syncthreads();
  const SmallSegs ss{seg_lists, seg_lists + kSmallScene, seg_counts[0], seg_counts[1]};

  const bool collect = a.recs != nullptr;
  const int64_t total = a.n_points * static_cast<int64_t>(a.n_rounds);
  const double pad = 1e-9 * s.diag;
  const bool refl = a.sp.reflect != 0;
  CLane w;
  w.rec_base = 0;
  w.rec_left = 0;
  unsigned long long walks_done = 0;
#ifdef WG_COOP_PROF
  long long cprof[7] = {};
#endif

  for (;;) {
    unsigned long long idx = 0;
    if (lane == 0) idx = atomicAdd(&a.counters[6], 1ull);  // work queue head
    idx = __shfl_sync(0xffffffffu, idx, 0);
    {
      if (idx >= a.counters[7]) break;  // handed-off walks (written by the previous launch)
      if (collect && lane == 0)  // the previous walk's record block ends with it
        for (int i = 0; i < w.rec_left; ++i) a.recs[w.rec_base + (8 - w.rec_left) + i].flags = 0u;
      const SpillLane& o = a.spill[idx];
      w.x = o.x;
      w.y = o.y;
      w.nx = o.nx;
      w.ny = o.ny;
      w.T = o.T;
      w.acc = o.acc;
      w.dacc = o.dacc;
      w.R = o.R;
      w.point = o.point;
      w.rec_base = o.rec_base;
      w.rng = o.rng;
      w.seg = o.seg;
      w.depth = o.depth;
      w.rec = o.rec;
      w.round = o.round;
      w.rec_left = o.rec_left;
      w.last_rec = o.last_rec;
      w.on_n = o.on_n != 0;
      w.rec_ok = o.rec_ok != 0;
    }

    // a handed-off walk enters at its direction step (begin_step done)
#ifdef WG_COOP_PROF
    long long q0 = clock64(), q1, q2, q3, q4, q5, q6;
    for (bool go = true; go; go = (q0 = clock64(), c_begin(w, a, s, ss, collect, lane))) {
      q1 = clock64();
      cprof[0] += q1 - q0;
#else
    for (bool go = true; go; go = c_begin(w, a, s, ss, collect, lane)) {
#endif
      // field evaluation and Table-1 decode
      float xin[16];
      c_gather(f, w.x, w.y, xin);
#ifdef WG_COOP_PROF
      __syncwarp();
      q2 = clock64();
      cprof[1] += q2 - q1;
#endif
      float y32;
      const float y = c_mlp(W, hbuf, xin, lane, &y32);
#ifdef WG_COOP_PROF
      __syncwarp();
      q3 = clock64();
      cprof[2] += q3 - q2;
#endif
      double cdec;
      const Lobe L = c_decode(y, y32, lane, &cdec);
#ifdef WG_COOP_PROF
      __syncwarp();
      q4 = clock64();
      cprof[3] += q4 - q3;
#endif
      double sel = cdec;
      if (a.sp.mode == WG_MODE_GUIDING_ONLY) sel = 1.0;
      else if (a.sp.mode == WG_MODE_FIXED_MIS) sel = a.sp.fixed_c;
      // one-sample MIS draw (sphdist.cpp:254-270)
      double dnx, dny;
      if (w.rng.unif() < static_cast<float>(sel)) {
        if (w.on_n && refl) {
          for (int it = 0;; ++it) {  // reflected_sample (sphdist.cpp:210-218)
            double mx, my;
            c_mixture_sample(w.rng, L, lane, &mx, &my);
            const double d = mx * w.nx + my * w.ny;
            if (d < 0.0) {
              reflect(mx, my, w.nx, w.ny, &dnx, &dny);
              break;
            }
            if (d > 0.0 || it + 1 == kMaxProposals) {
              dnx = mx;
              dny = my;
              break;
            }
          }
        } else {
          c_mixture_sample(w.rng, L, lane, &dnx, &dny);
        }
      } else {
        uniform_sample32(w.rng, w.on_n, w.nx, w.ny, &dnx, &dny);
      }
      double pg;
      if (w.on_n && refl) {
        double rx, ry;
        reflect(dnx, dny, w.nx, w.ny, &rx, &ry);
        const double p1 = c_pdf(L, dnx, dny), p2 = c_pdf(L, rx, ry);
        pg = dnx * w.nx + dny * w.ny <= 0.0 ? 0.0 : p1 + p2;
      } else {
        pg = c_pdf(L, dnx, dny);
      }
      const double pu = uniform_pdf(w.on_n, dnx, dny, w.nx, w.ny);
      const double pmis = sel * pg + (1.0 - sel) * pu;
      const double mult = pu / pmis;
#ifdef WG_COOP_PROF
      __syncwarp();
      q5 = clock64();
      cprof[4] += q5 - q4;
#endif
      if (w.rec >= 0 && lane == 0) {
        DevRecord r;
        r.x = static_cast<float>(w.x);
        r.y = static_cast<float>(w.y);
        r.nux = static_cast<float>(dnx);
        r.nuy = static_cast<float>(dny);
        r.nx = static_cast<float>(w.nx);
        r.ny = static_cast<float>(w.ny);
        r.pdf_mis = static_cast<float>(pmis);
        r.pdf_g = static_cast<float>(pg);
        r.pdf_u = static_cast<float>(pu);
        r.c = static_cast<float>(sel);
        r.target = 0.0f;
        r.dacc = static_cast<float>(w.dacc);
        r.thr_q = static_cast<float>(w.T * mult);
        r.pad_ = 0.0f;
        r.walk = static_cast<int32_t>(static_cast<int64_t>(w.round) * a.n_points + w.point);
        r.flags = REC_WRITTEN | (w.on_n ? REC_ON_NEUMANN : 0u);
        r.key = Pcg::mix(a.key_seed ^ Pcg::mix((static_cast<uint64_t>(a.point_offset + w.point) << 20) ^
                                               static_cast<uint64_t>(w.depth)));
        r.prev = w.last_rec;
        r.pad2_ = 0;
        a.recs[w.rec] = r;
      }
      if (w.rec >= 0) {
        w.last_rec = w.rec;
        w.dacc = 0.0;
      }
      if (mult == 0.0) {
        c_finish(w, a, false, lane);
        break;
      }
      // finish_step (wost.cpp:218-264)
      Hit h = w_ray_neumann(s, ss, w.x, w.y, dnx, dny, w.R, w.seg, lane);
      if (h.seg >= 0) {
        w.x = h.px;
        w.y = h.py;
        w.on_n = true;
        w.nx = h.nx;
        w.ny = h.ny;
        w.seg = h.seg;
      } else {
        w.x = w.x + dnx * w.R;
        w.y = w.y + dny * w.R;
        w.on_n = false;
        w.seg = -1;
      }
      w.T *= mult;
      ++w.depth;
#ifdef WG_COOP_PROF
      __syncwarp();
      q6 = clock64();
      cprof[5] += q6 - q5;
      cprof[6] += 1;
#endif
      if (!bbox_contains(s, w.x, w.y, pad)) {
        c_finish(w, a, true, lane);
        break;
      }
    }
  }
#ifdef WG_COOP_PROF
  if (lane == 0)
    for (int i = 0; i < 7; ++i) atomicAdd(&g_coop_prof[i], static_cast<unsigned long long>(cprof[i]));
#endif
  if (collect && lane == 0)
    for (int i = 0; i < w.rec_left; ++i) a.recs[w.rec_base + (8 - w.rec_left) + i].flags = 0u;
  if (lane == 0 && walks_done) atomicAdd(&a.counters[2], walks_done);
}

__global__ void __launch_bounds__(kCoopThreads, 2) walk_kernel_coop_resume(WalkArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  walk_coop_body(a, smem);
}

int walk_coop_smem(const WalkArgs& a) {
  return static_cast<int>(al16c(sizeof(CoopW)) + sizeof(float) * 64 * kCoopWarps +
                          (a.scene_smem_bytes > 0 ? al16c(a.scene_smem_bytes) : 0));
}

// the lockstep kernel's handed-off tail walks (counters[7] of them, at most
// max_walks): one warp each
cudaError_t launch_walks_coop_resume(const WalkArgs& a, int max_walks, int sms, cudaStream_t st) {
  const int smem = walk_coop_smem(a);
  cudaError_t e = cudaFuncSetAttribute(walk_kernel_coop_resume, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(a.counters + 6, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, walk_kernel_coop_resume, kCoopThreads, smem);
  const int blocks = std::max(1, std::min((max_walks + kCoopWarps - 1) / kCoopWarps, sms * std::max(1, per_sm)));
  walk_kernel_coop_resume<<<blocks, kCoopThreads, smem, st>>>(a);
#ifdef WG_COOP_PROF
  static int calls = 0;
  if (++calls % 256 == 0) {
    cudaStreamSynchronize(st);
    coop_prof_dump();
  }
#endif
  return cudaGetLastError();
}

}  // namespace wg
