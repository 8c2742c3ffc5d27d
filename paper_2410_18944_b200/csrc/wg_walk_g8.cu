// Guided walk kernel, 8 lanes per walk (default field shape: 16 -> 64 -> 64 ->
// 33, K = 8 vMF components).
//
// Why: a training round of cfg 2 has only 16,384 walks, so the round time is
// the serial step chain of its longest walk; one thread per walk leaves the
// GPU latency-bound on the 7.2k-FMA MLP and the per-component fp64 math.
// Here a group of 8 consecutive lanes owns one walk:
//   * scalar walk state (position, throughput, PCG32 stream, ...) is
//     replicated in all 8 lanes, which execute the scalar code identically,
//     so control flow is uniform inside a group and every lane draws the same
//     random numbers;
//   * the MLP is split by output neuron (lane g owns outputs g, g+8, ...),
//     each output accumulated in exactly the reference's order, with the
//     previous layer's activations broadcast by 8-wide shuffles;
//   * lane g owns mixture component g for normalisation (Bessel series,
//     exp/log) and for the per-component terms of every mixture density;
//     sums over components are gathered and added in component order, so
//     every value is bit-identical to the sequential reference.
// Only lane 0 writes results, records and counters.
#include "wg_kernels.cuh"
#include "wg_train.cuh"
#include "wg_sphdist.cuh"

namespace wg {

namespace {
constexpr int GL = 8;        // lanes per walk
constexpr int NIN = 16, NH = 64, NO = 33, NK = 8;
constexpr int MLPN = NIN * NH + NH + NH * NH + NH + NH * NO + NO;  // 7393
constexpr int B1 = NIN * NH, W2 = B1 + NH, B2 = W2 + NH * NH, W3 = B2 + NH, B3 = W3 + NH * NO;

__host__ __device__ __forceinline__ size_t a16(size_t b) { return (b + 15) & ~size_t(15); }

struct Grp {
  unsigned mask;
  int g;  // lane within the group
};

template <class T>
__device__ __forceinline__ T gshfl(const Grp& gp, T v, int src) {
  return __shfl_sync(gp.mask, v, src, GL);
}

// per-group decoded mixture: lane g holds component g
struct MixL {
  double mux, muy, kappa, lambda, log_a;  // own component
  double lam_all[NK];                     // all weights (for sampling)
  double c;
};

// ordered sum over the 8 components of a per-lane term (component order, as
// the reference's sequential loops)
__device__ __forceinline__ double ordered_sum(const Grp& gp, double v) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NK; ++i) s += gshfl(gp, v, i);
  return s;
}

// mixture_pdf (sphdist.cpp:176-185) with one component per lane
__device__ __forceinline__ double mixture_pdf_g(const Grp& gp, const MixL& m, double nx, double ny) {
  double dt = nx * m.mux + ny * m.muy + 0.0 * 0.0;
  double term = m.lambda * exp(m.kappa * dt + m.log_a);
  return ordered_sum(gp, term);
}

__device__ __forceinline__ double reflected_pdf_g(const Grp& gp, const MixL& m, double nx, double ny,
                                                  double px, double py) {
  if (nx * px + ny * py + 0.0 * 0.0 <= 0.0) return 0.0;
  double rx, ry;
  reflect(nx, ny, px, py, &rx, &ry);
  double a = mixture_pdf_g(gp, m, nx, ny);
  double b = mixture_pdf_g(gp, m, rx, ry);
  return a + b;
}

// mixture_sample (sphdist.cpp:187-202): pick by cumulative weights, then the
// picked component's Best-Fisher / uniform draw (all lanes, same stream)
__device__ __forceinline__ void mixture_sample_g(const Grp& gp, Pcg& rng, const MixL& m,
                                                 double* ox, double* oy) {
  int pick = 0;
  double u = rng.uni(), acc = 0.0;
  pick = NK - 1;
#pragma unroll
  for (int i = 0; i < NK; ++i) {
    acc += m.lam_all[i];
    if (u < acc) {
      pick = i;
      break;
    }
  }
  double mux = gshfl(gp, m.mux, pick), muy = gshfl(gp, m.muy, pick);
  double kap = gshfl(gp, m.kappa, pick);
  vmf_sample2(rng, mux, muy, kap, ox, oy);
}

__device__ __forceinline__ void reflected_sample_g(const Grp& gp, Pcg& rng, const MixL& m, double px,
                                                   double py, double* ox, double* oy) {
  for (int it = 0;; ++it) {
    double nx, ny;
    mixture_sample_g(gp, rng, m, &nx, &ny);
    double d = nx * px + ny * py + 0.0 * 0.0;
    if (d < 0.0) {
      reflect(nx, ny, px, py, ox, oy);
      return;
    }
    if (d > 0.0 || it + 1 == kMaxProposals) {
      *ox = nx;
      *oy = ny;
      return;
    }
  }
}

// fp32 MLP, output-neuron split; exact accumulation order of affine_forward_f
// (guide_field.cpp:149-170). x: all 16 inputs (every lane).
__device__ __forceinline__ void mlp_g8(const Grp& gp, const float* __restrict__ W, const float* x,
                                       float* o /* o[q] = output gp.g + 8q, q < 5 */) {
  const int g = gp.g;
  float h[8];
  // layer 1: 16 -> 64
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int j = g + 8 * q;
    float y = W[B1 + j];
#pragma unroll
    for (int i = 0; i < NIN; i += 4) {
      float p = __fadd_rn(__fmul_rn(x[i], W[i * NH + j]), __fmul_rn(x[i + 1], W[(i + 1) * NH + j]));
      float r = __fadd_rn(__fmul_rn(x[i + 2], W[(i + 2) * NH + j]),
                          __fmul_rn(x[i + 3], W[(i + 3) * NH + j]));
      y = __fadd_rn(y, __fadd_rn(p, r));
    }
    h[q] = y > 0.0f ? y : 0.0f;
  }
  // layer 2: 64 -> 64 (inputs broadcast 4 at a time: input i lives in lane i%8, slot i/8)
  float h2[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) h2[q] = W[B2 + g + 8 * q];
#pragma unroll
  for (int i = 0; i < NH; i += 4) {
    float x0 = gshfl(gp, h[i / 8], i % 8), x1 = gshfl(gp, h[(i + 1) / 8], (i + 1) % 8);
    float x2 = gshfl(gp, h[(i + 2) / 8], (i + 2) % 8), x3 = gshfl(gp, h[(i + 3) / 8], (i + 3) % 8);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int j = g + 8 * q;
      float p = __fadd_rn(__fmul_rn(x0, W[W2 + i * NH + j]), __fmul_rn(x1, W[W2 + (i + 1) * NH + j]));
      float r = __fadd_rn(__fmul_rn(x2, W[W2 + (i + 2) * NH + j]),
                          __fmul_rn(x3, W[W2 + (i + 3) * NH + j]));
      h2[q] = __fadd_rn(h2[q], __fadd_rn(p, r));
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) h2[q] = h2[q] > 0.0f ? h2[q] : 0.0f;
  // layer 3: 64 -> 33 (lane g owns outputs g, g+8, g+16, g+24 and lane 0 also 32)
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const int j = g + 8 * q;
    o[q] = j < NO ? W[B3 + j] : 0.0f;
  }
#pragma unroll
  for (int i = 0; i < NH; i += 4) {
    float x0 = gshfl(gp, h2[i / 8], i % 8), x1 = gshfl(gp, h2[(i + 1) / 8], (i + 1) % 8);
    float x2 = gshfl(gp, h2[(i + 2) / 8], (i + 2) % 8), x3 = gshfl(gp, h2[(i + 3) / 8], (i + 3) % 8);
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const int j = g + 8 * q;
      if (q == 4 && g != 0) continue;
      float p = __fadd_rn(__fmul_rn(x0, W[W3 + i * NO + j]), __fmul_rn(x1, W[W3 + (i + 1) * NO + j]));
      float r = __fadd_rn(__fmul_rn(x2, W[W3 + (i + 2) * NO + j]),
                          __fmul_rn(x3, W[W3 + (i + 3) * NO + j]));
      o[q] = __fadd_rn(o[q], __fadd_rn(p, r));
    }
  }
}

// normalize_params (sphdist.cpp:287-310) with lane g = component g. Raw
// layout [mu (16) | kappa (8) | lambda (8) | c]; output j is in lane j%8 slot j/8.
__device__ __forceinline__ void normalize_g8(const Grp& gp, const float* o, MixL& m) {
  const int g = gp.g;
  const int s0 = (2 * g) % 8, s1 = (2 * g + 1) % 8;
  float a0 = gshfl(gp, o[0], s0), a1 = gshfl(gp, o[1], s0);
  float b0 = gshfl(gp, o[0], s1), b1 = gshfl(gp, o[1], s1);
  double mxr = g < 4 ? a0 : a1;
  double myr = g < 4 ? b0 : b1;
  double kr = o[2];
  double lr = o[3];
  double cr = gshfl(gp, o[4], 0);
  m.c = sigmoid(cr);
  // max logit (exact, order free) then the ordered partition sum
  double mx = lr;
#pragma unroll
  for (int d = 1; d < 8; d <<= 1) mx = smax(mx, __shfl_xor_sync(gp.mask, mx, d, GL));
  double e = exp(lr - mx);
  double z = 0.0;
#pragma unroll
  for (int i = 0; i < NK; ++i) {
    double ei = gshfl(gp, e, i);
    z += ei;
    (void)ei;
  }
  double mn = sqrt(mxr * mxr + myr * myr + 0.0 * 0.0);
  if (mn < 1e-12) {
    double a = kTwoPi * g / kMaxK;
    m.mux = cos(a);
    m.muy = sin(a);
  } else {
    m.mux = mxr / mn;
    m.muy = myr / mn;
  }
  m.kappa = sclamp(exp(kr), kKappaMin, kKappaMax);
  m.lambda = e / z;
#pragma unroll
  for (int i = 0; i < NK; ++i) m.lam_all[i] = gshfl(gp, m.lambda, i);
  m.log_a = -log_bessel_i0(m.kappa) - log(kTwoPi);
}

}  // namespace

struct GLane {
  double x, y, nx, ny, T, acc, R;
  int seg, depth;
  bool on_n, alive;
  Pcg rng;
  int64_t point;
  int round;
  int64_t rec_base;
  int rec_left, last_rec;
  double dacc;  // accumulator increments since the last record (DevRecord::dacc)
  bool rec_ok;
};

__global__ void __launch_bounds__(256) walk_kernel_g8(WalkArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  SceneView s = a.scene;
  size_t off = 0;
  if (a.scene_smem_bytes > 0) {
    auto carve = [&](size_t bytes) {
      unsigned char* p = smem + off;
      off += a16(bytes);
      return p;
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
    off = a16(a.scene_smem_bytes);
  }
  float* W = reinterpret_cast<float*>(smem + off);
  for (int i = threadIdx.x; i < MLPN; i += blockDim.x) W[i] = a.field.p[a.field.w1 + i];
  __syncthreads();

  const int lane = threadIdx.x & 31;
  Grp gp;
  gp.g = lane & (GL - 1);
  gp.mask = 0xffu << (lane & ~(GL - 1));
  const bool lead = gp.g == 0;
  const bool collect = a.recs != nullptr;
  const int64_t total = a.n_points * static_cast<int64_t>(a.n_rounds);
  const int64_t groups = (static_cast<int64_t>(gridDim.x) * blockDim.x) / GL;
  int64_t next = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / GL;
  const double eps = a.sp.eps, rmin = a.sp.rmin;
  const double pad = 1e-9 * s.diag;
  const FieldView& fv = a.field;
  GLane w;
  w.alive = false;
  w.rec_base = 0;
  w.rec_left = 0;
  int64_t walks_done = 0;

  auto finish = [&](bool escaped, double terminal) {
    if (lead) {
      const int64_t slot = static_cast<int64_t>(w.round) * a.n_points + w.point;
      a.est[slot] = escaped ? 0.0 : w.acc;
      a.esc[slot] = escaped ? 1 : 0;
      if (a.steps) a.steps[slot] = w.depth;
      atomicAdd(&a.counters[0], static_cast<unsigned long long>(w.depth));
      if (escaped) atomicAdd(&a.counters[1], 1ull);
      if (a.rec_tail) {  // the walk's end of the record chain (see DevRecord)
        a.rec_tail[slot] = w.last_rec;
        a.rec_term[slot] = escaped ? 0.0 : w.T * terminal + w.dacc;
      }
    }
    w.alive = false;
  };

  for (;;) {
    if (!w.alive) {
      if (next >= total) break;
      w.round = static_cast<int>(next / a.n_points);
      w.point = next - static_cast<int64_t>(w.round) * a.n_points;
      w.x = a.points[2 * w.point];
      w.y = a.points[2 * w.point + 1];
      w.nx = w.ny = 0.0;
      w.on_n = false;
      w.seg = -1;
      w.T = 1.0;
      w.acc = 0.0;
      w.R = 0.0;
      w.depth = 0;
      w.alive = true;
      w.rng = Pcg::walk(a.seed, static_cast<uint64_t>(a.point_offset + w.point),
                        a.wpp_first + static_cast<uint64_t>(w.round));
      w.last_rec = -1;
      w.dacc = 0.0;
      w.rec_ok = true;
      next += groups;
      ++walks_done;
    }
    // ---------------- begin_step (wost.cpp:148-216)
    CP cd = closest_point(s, w.x, w.y, WG_KIND_DIRICHLET);
    if (cd.seg >= 0 && cd.d <= eps) {
      double gv = eval_value(s.values[s.seg_value[cd.seg]], cd.px, cd.py);
      w.acc += w.T * gv;
      finish(false, gv);
      continue;
    }
    if (w.depth >= a.sp.max_steps) {
      finish(true, 0.0);
      continue;
    }
    double rr = 1.0;
    if (w.depth > a.sp.rr_depth) {
      double q = smin(1.0, fabs(w.T));
      if (q <= 0.0 || w.rng.uni() >= q) {
        finish(false, 0.0);
        continue;
      }
      w.T /= q;
      rr = 1.0 / q;
    }
    double dsil = closest_silhouette(s, w.x, w.y);
    double dd = cd.seg >= 0 ? cd.d : dinf();
    if (dd == dinf() && dsil == dinf()) {
      if (lead) atomicOr(&a.counters[4], 1ull);
      finish(true, 0.0);
      continue;
    }
    w.R = smin(dd, smax(dsil, rmin));
    double contrib = 0.0;
    if (!s.source_zero) {  // sample_source_point, wost.cpp:67-87
      double dx, dy;
      uniform_sample(w.rng, w.on_n, w.nx, w.ny, &dx, &dy);
      double r = 0.0;
      {
        double u = w.rng.uni();
        // greens radius (wost.cpp:37-65)
        if (u <= 0.0) r = 0.0;
        else if (u >= 1.0) r = w.R;
        else {
          double lo = 0.0, hi = 1.0, sv = sqrt(u);
          for (int it = 0; it < 100; ++it) {
            double ls = log(sv);
            double f = sv * sv * (1.0 - 2.0 * ls) - u;
            double df = -4.0 * sv * ls;
            if (f > 0.0) hi = sv;
            else lo = sv;
            if (fabs(f) < 1e-10) break;
            double step = df > 0.0 ? f / df : 0.0;
            double nxt = sv - step;
            if (!(nxt > lo && nxt < hi)) nxt = 0.5 * (lo + hi);
            if (nxt == sv) break;
            sv = nxt;
          }
          r = sv * w.R;
        }
      }
      double yx = w.x + dx * r, yy = w.y + dy * r;
      Hit h = source_ray_needed(s, r, w.R) ? ray_first_hit(s, w.x, w.y, dx, dy, r, WG_KIND_ALL, -1) : no_hit();
      double wt = h.seg >= 0 ? 0.0 : w.R * w.R / 4.0;
      if (wt != 0.0) {
        double f = 0.0;
        if (bbox_contains(s, yx, yy, 0.0)) f = eval_value(s.source, yx, yy);
        contrib -= wt * f;
      }
    }
    if (s.has_flux) {  // sample_neumann_contrib, wost.cpp:89-109
      double dx, dy;
      uniform_sample(w.rng, w.on_n, w.nx, w.ny, &dx, &dy);
      Hit h = ray_first_hit(s, w.x, w.y, dx, dy, w.R, WG_KIND_NEUMANN, w.seg);
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

    int rec = -1;
    if (collect && w.rec_ok) {
      if (w.rec_left == 0) {
        unsigned long long b = 0;
        if (lead) b = atomicAdd(a.rec_counter, 8ull);
        b = gshfl(gp, b, 0);
        if (static_cast<int64_t>(b) + 8 > a.rec_capacity) {
          w.rec_ok = false;
          if (lead) atomicAdd(&a.counters[3], 1ull);
        } else {
          w.rec_base = static_cast<int64_t>(b);
          w.rec_left = 8;
        }
      }
      if (w.rec_ok) {
        rec = static_cast<int>(w.rec_base + (8 - w.rec_left));
        --w.rec_left;
      }
    }

    // ---------------- decode + finish_step (wost.cpp:111-146, 218-264)
    MixL m;
    {
      float xin[NIN];
      field_gather(fv, w.x, w.y, xin);
      float o[5];
      mlp_g8(gp, W, xin, o);
      normalize_g8(gp, o, m);
    }
    if (a.sp.mode == WG_MODE_GUIDING_ONLY) m.c = 1.0;
    else if (a.sp.mode == WG_MODE_FIXED_MIS) m.c = a.sp.fixed_c;
    const bool refl = a.sp.reflect != 0;
    double nux, nuy;
    // mis_sample (sphdist.cpp:254-270)
    bool guided = w.rng.uni() < m.c;
    if (guided) {
      if (w.on_n && refl) reflected_sample_g(gp, w.rng, m, w.nx, w.ny, &nux, &nuy);
      else mixture_sample_g(gp, w.rng, m, &nux, &nuy);
    } else {
      uniform_sample(w.rng, w.on_n, w.nx, w.ny, &nux, &nuy);
    }
    double pg = w.on_n ? (refl ? reflected_pdf_g(gp, m, nux, nuy, w.nx, w.ny)
                               : mixture_pdf_g(gp, m, nux, nuy))
                       : mixture_pdf_g(gp, m, nux, nuy);
    double pu = uniform_pdf(w.on_n, nux, nuy, w.nx, w.ny);
    double pmis = m.c * pg + (1.0 - m.c) * pu;
    double mult = pu / pmis;
    if (rec >= 0 && lead) {
      DevRecord r;
      r.x = static_cast<float>(w.x);
      r.y = static_cast<float>(w.y);
      r.nux = static_cast<float>(nux);
      r.nuy = static_cast<float>(nuy);
      r.nx = static_cast<float>(w.nx);
      r.ny = static_cast<float>(w.ny);
      r.pdf_mis = static_cast<float>(pmis);
      r.pdf_g = static_cast<float>(pg);
      r.pdf_u = static_cast<float>(pu);
      r.c = static_cast<float>(m.c);
      r.target = 0.0f;
      r.dacc = static_cast<float>(w.dacc);
      r.thr_q = static_cast<float>(w.T * mult);
      r.pad_ = 0.0f;
      r.walk = static_cast<int32_t>(static_cast<int64_t>(w.round) * a.n_points + w.point);
      r.flags = REC_WRITTEN | (w.on_n ? REC_ON_NEUMANN : 0u);
      (void)rr;
      (void)contrib;
      r.key = Pcg::mix(a.key_seed ^ Pcg::mix((static_cast<uint64_t>(a.point_offset + w.point) << 20) ^
                                             static_cast<uint64_t>(w.depth)));
      r.prev = w.last_rec;
      r.pad2_ = 0;
      a.recs[rec] = r;
    }
    if (rec >= 0) {
      w.last_rec = rec;
      w.dacc = 0.0;
    }
    if (mult == 0.0) {
      finish(false, 0.0);
      continue;
    }
    Hit h = ray_first_hit(s, w.x, w.y, nux, nuy, w.R, WG_KIND_NEUMANN, w.seg);
    if (h.seg >= 0) {
      w.x = h.px;
      w.y = h.py;
      w.on_n = true;
      w.nx = h.nx;
      w.ny = h.ny;
      w.seg = h.seg;
    } else {
      w.x = w.x + nux * w.R;
      w.y = w.y + nuy * w.R;
      w.on_n = false;
      w.seg = -1;
    }
    w.T *= mult;
    ++w.depth;
    if (!bbox_contains(s, w.x, w.y, pad)) finish(true, 0.0);
  }
  if (collect && lead)
    for (int i = 0; i < w.rec_left; ++i) a.recs[w.rec_base + (8 - w.rec_left) + i].flags = 0u;
  unsigned long long wd = lead ? static_cast<unsigned long long>(walks_done) : 0ull;
  for (int o = 16; o > 0; o >>= 1) wd += __shfl_down_sync(0xffffffffu, wd, o);
  if (lane == 0) atomicAdd(&a.counters[2], wd);
}

int walk_g8_smem(const WalkArgs& a) {
  return static_cast<int>((a.scene_smem_bytes > 0 ? a16(a.scene_smem_bytes) : 0) +
                          a16(sizeof(float) * MLPN));
}

int walk_g8_blocks_per_sm(int smem) {
  int n = 0;
  cudaFuncSetAttribute(walk_kernel_g8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, walk_kernel_g8, 256, smem);
  return n;
}

cudaError_t launch_walks_g8(const WalkArgs& a, int blocks, cudaStream_t st) {
  int smem = walk_g8_smem(a);
  cudaError_t e = cudaFuncSetAttribute(walk_kernel_g8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  walk_kernel_g8<<<blocks, 256, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace wg
