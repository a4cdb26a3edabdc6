// C++ caller of the drop-in boundary (include/diffmpm/mpm_batch.hpp over
// include/diffmpm.h).  Runs on a GPU box via tests/test_gpu_native.py:
//   * free fall of a fluid block: com_z drop and d com_z / d v0_z = t / N
//   * the reference's exception text for an out-of-interior particle
// Exit status 0 on success.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "diffmpm/mpm_batch.hpp"

int main() {
  using namespace diffmpm;
  Config cfg;
  cfg.num_envs = 2;
  cfg.dims = {16, 16, 16};
  cfg.dx = 1.0 / 16;
  cfg.dt = 1e-4;
  cfg.gravity = {0.0, 0.0, -9.8};
  cfg.substeps = 4;
  cfg.max_steps = 2;
  const int n1 = 8;
  cfg.particles_per_env = n1 * n1 * n1;
  Material fluid;
  fluid.kind = Law::kFluid;
  fluid.youngs = 1e4;
  fluid.density = 1000.0;
  fluid.volume = std::pow(0.2 / n1, 3);
  MpmBatch b(cfg, {fluid}, {});
  const int N = cfg.particles_per_env, E = cfg.num_envs;
  std::vector<float> x, v(3 * E * N, 0.f), F(9 * E * N, 0.f), C(9 * E * N, 0.f);
  std::vector<int> mat(E * N, 0);
  for (int e = 0; e < E; ++e)
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < n1; ++j)
        for (int k = 0; k < n1; ++k) {
          x.push_back(0.4f + 0.2f * (i + 0.5f) / n1);
          x.push_back(0.4f + 0.2f * (j + 0.5f) / n1);
          x.push_back(0.5f + 0.2f * (k + 0.5f) / n1);
        }
  for (int p = 0; p < E * N; ++p) F[9 * p] = F[9 * p + 4] = F[9 * p + 8] = 1.f;
  b.set_state(x, v, F, C, mat);
  std::vector<float> obs0, obs1;
  obs0 = b.step({});
  obs1 = b.step({});
  double z0 = 0;
  for (int p = 0; p < N; ++p) z0 += x[3 * p + 2] / N;
  const double t = 8 * cfg.dt;
  const double want = z0 - 0.5 * 9.8 * t * t;
  // symplectic Euler: v_{k+1} = v_k + g dt, x_{k+1} = x_k + v_{k+1} dt -> drop = g dt^2 n(n+1)/2
  const double want_se = z0 - 9.8 * cfg.dt * cfg.dt * 8 * 9 / 2.0;
  const double got = obs1[2];
  std::printf("com_z %.9f  analytic %.9f  symplectic %.9f\n", got, want, want_se);
  if (std::fabs(got - want_se) > 1e-6) return 1;
  std::vector<float> dobs(2 * E * DM_OBS_DIM, 0.f);
  for (int e = 0; e < E; ++e) dobs[(1 * E + e) * DM_OBS_DIM + 2] = 1.f;  // d L / d com_z at the last step
  Gradients g = b.backward(dobs);
  double gz = 0;
  for (int p = 0; p < N; ++p) gz += g.v[3 * p + 2];
  std::printf("sum dL/dv0_z %.6e  want t = %.6e\n", gz, t);
  if (std::fabs(gz - t) > 1e-3 * t) return 2;
  // reference error text (mpm.hpp:156-158)
  x[0] = 0.01f;
  b.set_state(x, v, F, C, mat);
  try {
    b.step({});
    return 3;
  } catch (const std::runtime_error& err) {
    std::printf("caught: %s\n", err.what());
    if (std::string(err.what()).find("particle 0") == std::string::npos) return 4;
  }
  std::printf("cpp adapter ok\n");
  return 0;
}
