// C++ caller of the batched Accel entries of the C-ABI (include/wostgpu.h:
// wostgpu_closest_point / _closest_silhouette / _ray_first_hit /
// _star_radius, the device versions of proj/src/geom2d.cpp:142-255), used by
// tests/test_gpu_parity.py: reads a scene + probes written by the test,
// writes every query's result for a bit-exact comparison with the oracle.
//
//   accel_queries IN OUT
//   IN : i32 n_seg, i32 n_probe, f64 seg[n_seg][4], i32 kind[n_seg],
//        f64 xy[n_probe][2], f64 dir[n_probe][2], f64 tmax[n_probe]
//   OUT: per kind mask 1..3: f64 pt[n][2], f64 dist[n], i32 seg[n];
//        f64 sil[n]; f64 t[n], f64 hit_pt[n][2], f64 normal[n][2], i32 hit_seg[n],
//        i32 hit_kind[n]; f64 star_r[n] (r_min 0; NaN where unbounded)
#include <cmath>
#include <cstdio>
#include <vector>

#include "wostgpu.hpp"

using namespace wostgpu;

template <class T>
static void rd(FILE* f, std::vector<T>& v) {
  if (std::fread(v.data(), sizeof(T), v.size(), f) != v.size()) throw std::runtime_error("short read");
}
template <class T>
static void wr(FILE* f, const std::vector<T>& v) {
  std::fwrite(v.data(), sizeof(T), v.size(), f);
}

int main(int argc, char** argv) {
  if (argc != 3) return 2;
  check(wostgpu_init(0));
  FILE* in = std::fopen(argv[1], "rb");
  int32_t ns = 0, np = 0;
  if (std::fread(&ns, 4, 1, in) != 1 || std::fread(&np, 4, 1, in) != 1) return 3;
  std::vector<double> seg(4 * ns), xy(2 * np), dir(2 * np), tmax(np);
  std::vector<int32_t> kind(ns);
  rd(in, seg);
  rd(in, kind);
  rd(in, xy);
  rd(in, dir);
  rd(in, tmax);
  std::fclose(in);

  Scene s;
  s.bbox = {{-1e3, -1e3}, {1e3, 1e3}};
  s.epsilon_shell = -1.0;  // an in-code test scene: no validate (geom2d tests)
  s.values = {{"v", ValueSpec{ValueSpec::Constant{0.0}}}};
  for (int i = 0; i < ns; ++i)
    s.segments.push_back({{seg[4 * i], seg[4 * i + 1]}, {seg[4 * i + 2], seg[4 * i + 3]},
                          kind[i] == WG_NEUMANN ? BoundaryKind::Neumann : BoundaryKind::Dirichlet, "v"});
  Accel accel(s);
  const wg_scene h = accel.handle();
  FILE* out = std::fopen(argv[2], "wb");
  for (unsigned kinds = 1; kinds <= 3; ++kinds) {
    std::vector<double> pt(2 * np), d(np);
    std::vector<int32_t> sg(np);
    check(wostgpu_closest_point(h, np, xy.data(), kinds, pt.data(), d.data(), sg.data()));
    wr(out, pt);
    wr(out, d);
    wr(out, sg);
  }
  std::vector<double> sil(np);
  check(wostgpu_closest_silhouette(h, np, xy.data(), sil.data()));
  wr(out, sil);
  std::vector<double> t(np), hp(2 * np), nrm(2 * np);
  std::vector<int32_t> hs(np), hk(np);
  check(wostgpu_ray_first_hit(h, np, xy.data(), dir.data(), tmax.data(), 3u, nullptr, t.data(), hp.data(),
                              nrm.data(), hs.data(), hk.data()));
  wr(out, t);
  wr(out, hp);
  wr(out, nrm);
  wr(out, hs);
  wr(out, hk);
  // the facade's batched star radius (SceneError for unbounded stars is a
  // whole-batch error in the C-ABI: report per point via single queries)
  std::vector<double> r(np);
  for (int i = 0; i < np; ++i) {
    try {
      r[i] = accel.star_radius({xy[2 * i], xy[2 * i + 1]}, 0.0);
    } catch (const SceneError&) {
      r[i] = std::nan("");
    }
  }
  wr(out, r);
  std::fclose(out);
  shutdown();
  return 0;
}
