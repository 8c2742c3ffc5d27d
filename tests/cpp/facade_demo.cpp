// Drop-in demo of the C++ facade (include/wostgpu.hpp): the reference's
// run_solve loop for the neumann-strip-vlin preset (proj/src/presets.cpp:55-85,
// 217-221) written against wostgpu:: instead of wost::. Prints one line:
//   relmse_uniform relmse_guided adam_steps
#include <cmath>
#include <cstdio>
#include <vector>

#include "wostgpu.hpp"

using namespace wostgpu;

static double strip_vlin(double x, double y) {  // presets.cpp:169-184
  const double pi = 3.14159265358979323846;
  double u = 0.5 * x;
  for (int n = 1; n < 2000; n += 2) {
    double cn = -4.0 / (n * n * pi * pi), a = n * pi * x, b = n * pi;
    double ratio = std::exp(a - b) * (1.0 - std::exp(-2.0 * a)) / (1.0 - std::exp(-2.0 * b));
    double term = cn * ratio * std::cos(n * pi * y);
    u += term;
    if (std::abs(term) < 1e-14 && n > 64) break;
  }
  return u;
}

int main(int argc, char** argv) {
  const int grid = argc > 1 ? std::atoi(argv[1]) : 32;
  const int wpp = argc > 2 ? std::atoi(argv[2]) : 64;
  check(wostgpu_init(0));
  Scene s;
  s.bbox = {{0, 0}, {1, 1}};
  s.epsilon_shell = 1e-3 * std::sqrt(2.0);
  s.values = {{"zero", ValueSpec{ValueSpec::Constant{0.0}}},
              {"y", ValueSpec{ValueSpec::Linear{0.0, 0.0, 1.0}}},
              {"insulated", ValueSpec{ValueSpec::Constant{0.0}}}};
  s.segments = {{{0, 0}, {0, 1}, BoundaryKind::Dirichlet, "zero"},
                {{1, 0}, {1, 1}, BoundaryKind::Dirichlet, "y"},
                {{0, 0}, {1, 0}, BoundaryKind::Neumann, "insulated"},
                {{0, 1}, {1, 1}, BoundaryKind::Neumann, "insulated"}};
  s.validate();
  Accel accel(s);
  std::vector<Vec2> pts;
  std::vector<double> ref;
  for (int j = 0; j < grid; ++j)
    for (int i = 0; i < grid; ++i) {
      Vec2 p{(i + 0.5) / grid, (j + 0.5) / grid};
      pts.push_back(p);
      ref.push_back(strip_vlin(p.x, p.y));
    }
  auto relmse = [&](const std::vector<PointStats>& st) {  // image.cpp:211-230
    double mx = 0, sum = 0;
    for (double r : ref) mx = std::max(mx, std::abs(r));
    double delta = 1e-4 * mx * mx;
    for (size_t i = 0; i < st.size(); ++i) {
      double d = st[i].mean - ref[i];
      sum += d * d / (ref[i] * ref[i] + delta);
    }
    return sum / st.size();
  };
  SolverConfig uc;
  StepContext uctx(accel, nullptr, uc);
  std::vector<PointStats> us(pts.size());
  SolveScratch scratch;
  for (int b = 0; b < wpp; ++b) solve_batch(uctx, pts, us, 1, b, false, nullptr, &scratch);

  FieldConfig fc;
  GuidingField field(fc, s.bbox, 1);
  SolverConfig gc;
  gc.mode = SamplerMode::LearnableMis;
  StepContext gctx(accel, &field, gc);
  std::vector<PointStats> gs(pts.size());
  TrainConfig tc = default_train_config();
  tc.seed = 1;
  run(gctx, pts, gs, 1, wpp, wpp, &tc);
  std::printf("%.9g %.9g %lld\n", relmse(us), relmse(gs), (long long)field.adam_steps());
  return 0;
}
