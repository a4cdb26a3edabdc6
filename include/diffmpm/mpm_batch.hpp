// diffmpm C++ adapter: the reference's C++ simulator surface over the C ABI.
//
// The reference exposes its MPM path as C++ templates
// (/root/reference/proj/include/diffsim/mpm.hpp:23-367, env.hpp:55-117,
// tape.hpp:181-255).  This header gives C++ callers the same shape on the
// GPU: descriptors mirroring MpmMaterial / SdfCollider / CouplingParams, a
// batched state with lift/lower (set_state / get_state), a recorded control
// step (Task::step inside step_checkpointed) and a backward that returns the
// cotangents Tape::backward + Tape::grad would.  Errors are rethrown as the
// reference's exception types with its message text (std::runtime_error for
// "mpm: particle <p> outside grid interior (axis <a>)" etc.,
// std::invalid_argument for "mpm_step: substeps < 1").
//
// Header-only; link libdiffmpm.so (paper_2412_12089_b200/libdiffmpm.so).
#pragma once

#include <array>
#include <stdexcept>
#include <string>
#include <utility>
#include <cstdint>
#include <vector>

#include "../diffmpm.h"

namespace diffmpm {

enum class Law : int { kFixedCorotated = 0, kNeoHookean = 1, kElastoplastic = 2, kFluid = 3 };
enum class Shape : int { kPlane = 0, kSphere = 1, kBox = 2, kCylinder = 3, kHollowBox = 4 };

// MpmMaterial (mpm.hpp:23-41) + extensions; particle mass = density * volume.
struct Material {
  Law kind = Law::kElastoplastic;
  double youngs = 1e5, poisson = 0.3, density = 1000.0, volume = 1e-6, yield_stress = 1e3;
  bool wide_yield = false;
  double viscosity = 0.0, act_strength = 0.0, bulk = 0.0;
};

// SdfCollider geometry (mpm.hpp:76-84) + cylinder / hollow box.
struct Collider {
  Shape kind = Shape::kPlane;
  std::array<double, 3> normal{0.0, 0.0, 1.0};
  double radius = 0.1;
  std::array<double, 3> half{0.1, 0.1, 0.1};
  double length = 0.3, thickness = 0.02;
};

struct Config {
  int device = 0;
  int num_envs = 1, particles_per_env = 0;
  std::array<int, 3> dims{32, 32, 32};  // MpmGrid::dims (mpm.hpp:58)
  double dx = 1.0 / 32.0, dt = 1e-4;
  std::array<double, 3> gravity{0.0, 0.0, -9.81};
  bool sticky_boundary = false;          // false: slip (mpm.hpp:296-302)
  double alpha_c = 100.0, mu_b = 0.0;    // CouplingParams (mpm.hpp:134-137)
  int num_groups = 0;
  int substeps = 1;                      // mpm_step substeps per control step
  int max_steps = 1;                     // tape capacity (control steps)
  int checkpoint_every = 0;              // 0: one recompute segment per control step
  double spill_half = 0.0, spill_temp = 0.0;
  int obs_groups = 0;  // pooled per-group statistics appended to the observables
};

// Cotangents returned by backward (Tape::grad of every leaf, tape.hpp:166-170).
struct Gradients {
  std::vector<float> x, v, F, C;  // [E][N][3|9], original particle order
  std::vector<float> cvo;         // [T][E][K][9] collider center / velocity / omega
  std::vector<float> act;         // [T][E][G]
  std::vector<double> youngs;     // [E][num_materials]
};

class MpmBatch {
 public:
  MpmBatch(const Config& cfg, const std::vector<Material>& mats, const std::vector<Collider>& cols)
      : E_(cfg.num_envs), N_(cfg.particles_per_env), K_(static_cast<int>(cols.size())), G_(cfg.num_groups),
        M_(static_cast<int>(mats.size())) {
    DmConfig c{};
    c.device = cfg.device;
    c.num_envs = cfg.num_envs;
    c.particles_per_env = cfg.particles_per_env;
    for (int a = 0; a < 3; ++a) {
      c.dims[a] = cfg.dims[a];
      c.gravity[a] = cfg.gravity[a];
    }
    c.dx = cfg.dx;
    c.dt = cfg.dt;
    c.boundary = cfg.sticky_boundary ? 1 : 0;
    c.alpha_c = cfg.alpha_c;
    c.mu_b = cfg.mu_b;
    c.num_colliders = K_;
    c.num_groups = cfg.num_groups;
    c.substeps = cfg.substeps;
    c.max_steps = cfg.max_steps;
    c.checkpoint_every = cfg.checkpoint_every;
    c.spill_half = cfg.spill_half;
    c.spill_temp = cfg.spill_temp;
    c.obs_groups = cfg.obs_groups;
    std::vector<DmMaterial> dm(mats.size());
    for (std::size_t i = 0; i < mats.size(); ++i) {
      dm[i] = DmMaterial{static_cast<int>(mats[i].kind), mats[i].youngs,       mats[i].poisson,
                         mats[i].density,                 mats[i].volume,       mats[i].yield_stress,
                         mats[i].wide_yield ? 1 : 0,      mats[i].viscosity,    mats[i].act_strength,
                         mats[i].bulk};
    }
    std::vector<DmColliderShape> ds(cols.empty() ? 1 : cols.size());
    for (std::size_t i = 0; i < cols.size(); ++i) {
      DmColliderShape& s = ds[i];
      s.kind = static_cast<int>(cols[i].kind);
      for (int a = 0; a < 3; ++a) {
        s.normal[a] = cols[i].normal[a];
        s.half[a] = cols[i].half[a];
      }
      s.radius = cols[i].radius;
      s.length = cols[i].length;
      s.thickness = cols[i].thickness;
    }
    ctx_ = dm_create(&c, dm.data(), M_, ds.data());
    if (!ctx_) throw std::runtime_error("dm_create failed");
    char buf[512];
    if (dm_last_error(ctx_, buf, sizeof(buf)) != DM_OK) {
      std::string msg(buf);
      dm_destroy(ctx_);
      ctx_ = nullptr;
      if (msg.find("substeps") != std::string::npos) throw std::invalid_argument(msg);
      throw std::runtime_error(msg);
    }
  }
  ~MpmBatch() {
    if (ctx_) dm_destroy(ctx_);
  }
  MpmBatch(const MpmBatch&) = delete;
  MpmBatch& operator=(const MpmBatch&) = delete;

  int num_envs() const { return E_; }
  int particles_per_env() const { return N_; }
  int tape_steps() const { return dm_tape_steps(ctx_); }
  DmContext* handle() { return ctx_; }

  // lift_state (env.hpp:41-47): upload all envs' particles in visit order and
  // start a fresh tape.
  void set_state(const std::vector<float>& x, const std::vector<float>& v, const std::vector<float>& F,
                 const std::vector<float>& C, const std::vector<int>& material, const std::vector<int>& group = {}) {
    const std::size_t n = static_cast<std::size_t>(E_) * N_;
    if (x.size() != 3 * n || v.size() != 3 * n || F.size() != 9 * n || C.size() != 9 * n || material.size() != n ||
        (!group.empty() && group.size() != n))
      throw std::invalid_argument("set_state: array sizes do not match num_envs x particles_per_env");
    check(dm_set_state(ctx_, x.data(), v.data(), F.data(), C.data(), material.data(),
                       group.empty() ? nullptr : group.data()));
  }

  // EnvBatch::reset(seed) / reset_env(i) (env.hpp:66-96) on the device:
  // envs with a nonzero mask byte (all when `mask` is empty) get a fresh
  // seeded lattice state; returns the per-env origin offsets [E][3].
  std::vector<double> reset_lattice(const DmLatticeReset& spec, std::uint64_t seed, int env_offset = 0,
                                    const std::vector<unsigned char>& mask = {},
                                    const std::vector<int>& particle_group = {}) {
    if (!mask.empty() && mask.size() != static_cast<std::size_t>(E_))
      throw std::invalid_argument("reset_lattice: mask size must equal num_envs");
    std::vector<double> delta(static_cast<std::size_t>(E_) * 3);
    check(dm_reset_lattice(ctx_, &spec, seed, env_offset, mask.empty() ? nullptr : mask.data(),
                           particle_group.empty() ? nullptr : particle_group.data(), delta.data()));
    return delta;
  }

  // lower_state (env.hpp:49-53)
  void get_state(std::vector<float>& x, std::vector<float>& v, std::vector<float>& F, std::vector<float>& C) {
    const std::size_t n = static_cast<std::size_t>(E_) * N_;
    x.resize(3 * n);
    v.resize(3 * n);
    F.resize(9 * n);
    C.resize(9 * n);
    check(dm_get_state(ctx_, x.data(), v.data(), F.data(), C.data()));
  }

  // One recorded control step (Task::step + step_checkpointed).  cvo [E][K][9],
  // act [E][G]; returns the observables [E][7] (com, var, spill).
  std::vector<float> step(const std::vector<float>& cvo, const std::vector<float>& act = {}) {
    std::vector<float> obs(static_cast<std::size_t>(E_) * dm_obs_dim(ctx_));
    check(dm_step(ctx_, cvo.empty() ? nullptr : cvo.data(), act.empty() ? nullptr : act.data(), obs.data()));
    return obs;
  }

  // Tape::backward from observable cotangents dobs [T][E][7].
  Gradients backward(const std::vector<float>& dobs) {
    const int T = tape_steps();
    const std::size_t n = static_cast<std::size_t>(E_) * N_;
    Gradients g;
    g.x.resize(3 * n);
    g.v.resize(3 * n);
    g.F.resize(9 * n);
    g.C.resize(9 * n);
    g.cvo.resize(static_cast<std::size_t>(T) * E_ * (K_ > 0 ? K_ : 1) * 9);
    g.act.resize(static_cast<std::size_t>(T) * E_ * (G_ > 0 ? G_ : 1));
    g.youngs.resize(static_cast<std::size_t>(E_) * M_);
    check(dm_backward(ctx_, dobs.empty() ? nullptr : dobs.data(), nullptr, nullptr, nullptr, nullptr, g.x.data(),
                      g.v.data(), g.F.data(), g.C.data(), K_ ? g.cvo.data() : nullptr,
                      G_ ? g.act.data() : nullptr, g.youngs.data()));
    return g;
  }

 private:
  void check(int rc) {
    if (rc == DM_OK) return;
    char buf[1024];
    dm_last_error(ctx_, buf, sizeof(buf));
    if (rc == DM_ERR_ARG) throw std::invalid_argument(buf);
    throw std::runtime_error(buf);
  }

  DmContext* ctx_ = nullptr;
  int E_, N_, K_, G_, M_;
};

}  // namespace diffmpm
