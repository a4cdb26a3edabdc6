// diffmpm C++ adapter: EnvBatch<Task> (env.hpp:55-117) for the reference's
// MPM tasks (tasks.hpp:232-369 MiniRollFlat, 502-645 MiniFluidMove) on the
// GPU simulator, over the dm_task_* C ABI (include/diffmpm.h).
//
//   diffmpm::EnvBatch envs(diffmpm::TaskKind::kFluidMove, n, seed);
//   envs.step(actions, rewards, dones);          // EnvBatch::step, auto-reset
//   auto obs = envs.observe();                   // Task::observe per env
//   auto da = envs.backward(drewards, dobs);     // dL/dactions over the recorded steps
//
// Mirrors the reference: double actions / rewards / observations,
// per-env streams RngStream(seed, i), done at episode_len; errors rethrown
// as std::runtime_error / std::invalid_argument with the library's text.
// Header-only; link libdiffmpm.so.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../diffmpm.h"

namespace diffmpm {

enum class TaskKind : int { kFluidMove = DM_TASK_FLUID_MOVE, kRollFlat = DM_TASK_ROLL_FLAT };

class EnvBatch {
 public:
  // The task's reference Config{} (dm_task_default_config); horizon = the
  // tape capacity in control steps for backward.
  EnvBatch(TaskKind kind, int n, std::uint64_t seed, int horizon = 64, int device = 0, int env_offset = 0)
      : EnvBatch(default_config(kind), n, seed, horizon, device, env_offset) {}
  EnvBatch(const DmTaskConfig& cfg, int n, std::uint64_t seed, int horizon = 64, int device = 0, int env_offset = 0)
      : n_(n) {
    if (n < 1) throw std::invalid_argument("EnvBatch: need at least one env");
    t_ = dm_task_create(&cfg, n, env_offset, horizon, device);
    check(dm_task_last_error(t_, nullptr, 0));
    dm_task_dims(t_, &obs_dim_, &act_dim_, &particles_, &episode_len_);
    reset(seed);
  }
  ~EnvBatch() { dm_task_destroy(t_); }
  EnvBatch(const EnvBatch&) = delete;
  EnvBatch& operator=(const EnvBatch&) = delete;

  static DmTaskConfig default_config(TaskKind kind) {
    DmTaskConfig c;
    dm_task_default_config(static_cast<int>(kind), &c);
    return c;
  }

  void reset(std::uint64_t seed) { check(dm_task_reset(t_, seed)); }

  // EnvBatch::step (env.hpp:77-90): actions [n][act_dim]; recorded on the tape.
  void step(const std::vector<std::vector<double>>& actions, std::vector<double>& rewards, std::vector<bool>& dones,
            bool record = true) {
    if (static_cast<int>(actions.size()) != n_) throw std::invalid_argument("EnvBatch::step: action batch size");
    std::vector<double> a(static_cast<size_t>(n_) * act_dim_);
    for (int i = 0; i < n_; ++i) {
      if (static_cast<int>(actions[i].size()) != act_dim_) throw std::invalid_argument("EnvBatch::step: action size");
      for (int k = 0; k < act_dim_; ++k) a[static_cast<size_t>(i) * act_dim_ + k] = actions[i][k];
    }
    rewards.assign(n_, 0.0);
    std::vector<unsigned char> d(n_, 0);
    check(dm_task_step(t_, a.data(), rewards.data(), d.data(), record ? 1 : 0));
    dones.assign(n_, false);
    for (int i = 0; i < n_; ++i) dones[i] = d[i] != 0;
  }

  // Task::observe of every env: [n][obs_dim].
  std::vector<std::vector<double>> observe() {
    std::vector<double> o(static_cast<size_t>(n_) * obs_dim_);
    check(dm_task_observe(t_, o.data()));
    std::vector<std::vector<double>> out(n_);
    for (int i = 0; i < n_; ++i) out[i].assign(o.begin() + static_cast<size_t>(i) * obs_dim_, o.begin() + (i + 1) * obs_dim_);
    return out;
  }

  // dL/dactions [T][n][act_dim] of L = sum drewards * rewards + sum dobs * obs
  // over the recorded steps (drewards [T][n], dobs [T+1][n][obs_dim]; either
  // may be empty).  The tape restarts from the current state.
  std::vector<double> backward(const std::vector<double>& drewards, const std::vector<double>& dobs = {}) {
    const int T = dm_task_tape_steps(t_);
    std::vector<double> da(static_cast<size_t>(T) * n_ * act_dim_);
    check(dm_task_backward(t_, drewards.empty() ? nullptr : drewards.data(), dobs.empty() ? nullptr : dobs.data(),
                           da.data()));
    return da;
  }

  int size() const { return n_; }
  int obs_dim() const { return obs_dim_; }
  int act_dim() const { return act_dim_; }
  int episode_len() const { return episode_len_; }
  int particles_per_env() const { return particles_; }

 private:
  void check(int rc) const {
    if (rc == DM_OK) return;
    char buf[1024];
    dm_task_last_error(t_, buf, sizeof(buf));
    if (rc == DM_ERR_ARG) throw std::invalid_argument(buf);
    throw std::runtime_error(buf);
  }

  DmTask* t_ = nullptr;
  int n_ = 0, obs_dim_ = 0, act_dim_ = 0, particles_ = 0, episode_len_ = 0;
};

}  // namespace diffmpm
