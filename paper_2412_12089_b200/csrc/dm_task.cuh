// Task layer (included by dm_context.cu): EnvBatch<Task> (env.hpp:55-117)
// for the reference's MPM tasks MiniFluidMove (tasks.hpp:502-645) and
// MiniRollFlat (tasks.hpp:232-369) on the GPU simulator.  Host side, in
// double as the reference: per-env task state (container / roller position),
// the action -> collider maps with their clamps, rewards, observations,
// auto-reset from each env's RngStream, and the reverse sweep that chains
// the simulator's per-step cotangents (dm backward_step) through them to
// dL/dactions.  The particles live in the context's device state.

namespace {

// RngStream (rng.hpp:11-55), bit-identical.
struct TaskRng {
  uint64_t key = 0, ctr = 0;
  TaskRng() = default;
  TaskRng(uint64_t seed, uint64_t stream) : key(mix(seed ^ (0x9e3779b97f4a7c15ULL * (stream + 1)))), ctr(0) {}
  static uint64_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double next_double() { return static_cast<double>(mix(key ^ mix(++ctr)) >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * next_double(); }
};

// clamp (tape.hpp:380-384): derivative 1 strictly inside, 0 at and beyond the bounds
double task_clamp(double a, double lo, double hi) { return a < lo ? lo : (a > hi ? hi : a); }
double task_dclamp(double a, double lo, double hi) { return (a > lo && a < hi) ? 1.0 : 0.0; }
// reward_distance_tiered (env.hpp:33-39), tier gradient-blocked
double task_tiered(double d, double thr, double lo, double hi) {
  return (1.0 / ((1.0 + d) * (1.0 + d))) * (d > thr ? lo : hi);
}
double task_dtiered(double d, double thr, double lo, double hi) {
  return -2.0 * (d > thr ? lo : hi) / ((1.0 + d) * (1.0 + d) * (1.0 + d));
}

const double kWallN[4][3] = {{-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}};  // tasks.hpp:578-579

// Makes the current state the tape's initial state (tape restart).
int restart_tape(DmContext* ctx) {
  const int s = ctx->steps * ctx->cfg.substeps;
  if (s > 0) {
    const StateView S0 = store_view(ctx, 0), cur = fwd_state(ctx, s);
    if (cur.f != S0.f) {
      DM_CUDA(cudaMemcpyAsync(S0.f, cur.f, state_floats(ctx) * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
      DM_CUDA(cudaMemcpyAsync(S0.attr, cur.attr, ctx->Ntot * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx->stream));
    }
    if (ctx->law == kFluid) {  // a G2P output stores D(0,0) only; the initial state is general
      dm_launch(ctx->grid_tiles, 256, 0, ctx->stream, ctx->pdl, k_fiso_expand, ctx->Ntot, S0);
      ++ctx->launches;
    }
  }
  ctx->steps = 0;
  ctx->cfl_checked = 0;
  ctx->bwd_t = -1;
  ctx->kept_t = -1;
  ctx->kept_ok = false;
  DM_CUDA(cudaGetLastError());
  return DM_OK;
}

}  // namespace

struct DmTask {
  DmTaskConfig cfg{};
  DmContext* ctx = nullptr;
  std::string err;
  int E = 0, N = 0, A = 0, od = 0, env_offset = 0, horizon = 0, stride = 1, ncloud = 0, K = 0;
  double dx = 0.0, floor_z = 0.0;
  std::vector<float> tmpl;  // [N][3] sample_box template (visit order)
  float* d_tmpl = nullptr;
  unsigned char* d_mask = nullptr;
  float* d_cloud = nullptr;  // [E][ncloud][3]
  std::vector<TaskRng> rng;
  std::vector<int> cursor;
  std::vector<double> c;  // [E][3]: container center (cx, cy, 0) / roller position
  // tape: per recorded step
  int T = 0;
  bool tape_ok = true;  // every step on the context's tape was recorded
  std::vector<double> act_t, c_t, cpre_t;
  std::vector<float> obs_t;  // [horizon][E][7]
  std::vector<unsigned char> cut_t;

  bool fluid() const { return cfg.kind == DM_TASK_FLUID_MOVE; }
  double speed() const { return fluid() ? cfg.speed : cfg.roller_speed; }
  // clamp bounds of the task state after the move (tasks.hpp:326-328, 599-602)
  double lo(int a) const { return fluid() ? 4.0 * dx + cfg.container_half : 3.5 * dx; }
  double hi(int a) const { return fluid() ? 1.0 - 4.0 * dx - cfg.container_half : 1.0 - 3.5 * dx; }
  // Task::reset (tasks.hpp:281-285, 549-553): draws from the env's own stream
  void draw_reset(int e) {
    double* ce = &c[3 * (size_t)e];
    if (fluid()) {
      ce[0] = cfg.start_x + rng[e].uniform(-0.01, 0.01);
      ce[1] = cfg.start_y + rng[e].uniform(-0.01, 0.01);
      ce[2] = 0.0;
    } else {
      const double x = 0.5 + rng[e].uniform(-0.02, 0.02);
      const double y = 0.5 + rng[e].uniform(-0.02, 0.02);
      ce[0] = x;
      ce[1] = y;
      ce[2] = floor_z + cfg.block_height + cfg.roller_radius + 0.02;
    }
  }
};

namespace {
int task_fail(DmTask* t, const std::string& m, int rc = DM_ERR_ARG) {
  t->err = m;
  return rc;
}
int task_ctx_err(DmTask* t, int rc) {
  if (rc != DM_OK) t->err = t->ctx->err;
  return rc;
}
}  // namespace

extern "C" {

void dm_task_default_config(int kind, DmTaskConfig* o) {
  if (!o) return;
  *o = DmTaskConfig{};
  o->kind = kind;
  o->grid_n = 20;
  o->ppc = 8;
  o->dt = 0.02;
  o->cloud_k = 16;
  o->episode_len = 40;
  // MiniFluidMove::Config (tasks.hpp:511-525)
  o->container_half = 0.1;
  o->fill = 0.08;
  o->speed = 0.25;
  o->start_x = 0.35;
  o->start_y = 0.5;
  o->target_x = 0.65;
  o->target_y = 0.5;
  o->spill_temp = 0.01;
  // MiniRollFlat::Config (tasks.hpp:241-254)
  o->block_size = 0.2;
  o->block_height = 0.1;
  o->roller_radius = 0.07;
  o->roller_speed = 0.25;
  o->h_flat = 0.1;
  o->youngs = 1e5;
  o->yield_stress = 2e3;
  o->substeps = kind == DM_TASK_FLUID_MOVE ? 40 : 20;
}

DmTask* dm_task_create(const DmTaskConfig* cfg, int num_envs, int env_offset, int horizon, int device) {
  DmTask* t = new DmTask();
  if (!cfg) {
    t->err = "dm_task_create: no config";
    return t;
  }
  t->cfg = *cfg;
  const DmTaskConfig& c = t->cfg;
  if (c.kind != DM_TASK_FLUID_MOVE && c.kind != DM_TASK_ROLL_FLAT) {
    t->err = "dm_task_create: unknown task kind";
    return t;
  }
  if (num_envs < 1 || horizon < 1 || c.grid_n < 8 || c.ppc < 1 || c.substeps < 1 || c.episode_len < 1 ||
      c.cloud_k < 1 || !(c.dt > 0.0)) {
    t->err = "dm_task_create: num_envs, horizon, episode_len, cloud_k >= 1, grid_n >= 8, substeps >= 1, dt > 0";
    return t;
  }
  t->E = num_envs;
  t->env_offset = env_offset;
  t->horizon = horizon;
  t->dx = 1.0 / c.grid_n;
  t->floor_z = 3.0 * t->dx;
  // the particle template: sample_box (mpm.hpp:371-395) as the task's constructor
  double org[3], size[3];
  if (t->fluid()) {
    const double inner = c.container_half - 0.02;
    org[0] = c.start_x - inner;
    org[1] = c.start_y - inner;
    org[2] = t->floor_z + 0.25 * t->dx;
    size[0] = 2.0 * inner;
    size[1] = 2.0 * inner;
    size[2] = c.fill;
  } else {
    const double half = c.block_size / 2.0;
    org[0] = 0.5 - half;
    org[1] = 0.5 - half;
    org[2] = t->floor_z + 0.5 * t->dx;
    size[0] = c.block_size;
    size[1] = c.block_size;
    size[2] = c.block_height;
  }
  const double h = t->dx / std::cbrt(static_cast<double>(c.ppc));
  int n[3];
  for (int a = 0; a < 3; ++a) n[a] = std::max(1, static_cast<int>(std::round(size[a] / h)));
  const double vol = (size[0] / n[0]) * (size[1] / n[1]) * (size[2] / n[2]);
  for (int i = 0; i < n[0]; ++i)
    for (int j = 0; j < n[1]; ++j)
      for (int k = 0; k < n[2]; ++k) {
        t->tmpl.push_back(static_cast<float>(org[0] + size[0] * (i + 0.5) / n[0]));
        t->tmpl.push_back(static_cast<float>(org[1] + size[1] * (j + 0.5) / n[1]));
        t->tmpl.push_back(static_cast<float>(org[2] + size[2] * (k + 0.5) / n[2]));
      }
  t->N = n[0] * n[1] * n[2];
  t->stride = std::max(1, t->N / c.cloud_k);  // tasks.hpp:272, 539
  t->ncloud = (t->N + t->stride - 1) / t->stride;
  t->A = t->fluid() ? 2 : 3;
  t->od = (t->fluid() ? 7 : 5) + 3 * t->ncloud;
  t->K = t->fluid() ? 4 : 1;
  DmConfig dc{};
  dc.device = device;
  dc.num_envs = t->E;
  dc.particles_per_env = t->N;
  dc.dims[0] = dc.dims[1] = dc.dims[2] = c.grid_n;
  dc.dx = t->dx;
  dc.dt = c.dt / c.substeps;
  dc.gravity[2] = -9.81;  // tasks.hpp:323-324, 596-597
  dc.boundary = 0;
  dc.alpha_c = 100.0;  // CouplingParams defaults (mpm.hpp:134-137)
  dc.mu_b = 0.0;
  dc.num_colliders = t->K;
  dc.substeps = c.substeps;
  dc.max_steps = horizon;
  dc.spill_half = t->fluid() ? c.container_half : 0.0;
  dc.spill_temp = t->fluid() ? c.spill_temp : 0.0;
  DmMaterial m{};
  m.kind = t->fluid() ? kFluid : kElastoplastic;  // MpmMaterial defaults: rho 1000, nu 0.3 (mpm.hpp:23-30)
  m.youngs = t->fluid() ? 1e4 : c.youngs;
  m.poisson = 0.3;
  m.density = 1000.0;
  m.volume = vol;
  m.yield_stress = t->fluid() ? 1e3 : c.yield_stress;
  DmColliderShape sh[4]{};
  if (t->fluid()) {
    for (int w = 0; w < 4; ++w) {
      sh[w].kind = kPlane;
      for (int a = 0; a < 3; ++a) sh[w].normal[a] = kWallN[w][a];
    }
  } else {
    sh[0].kind = kSphere;
    sh[0].radius = c.roller_radius;
  }
  t->ctx = dm_create(&dc, &m, 1, sh);
  if (t->ctx->poisoned) {
    t->err = t->ctx->err;
    return t;
  }
  DmContext* ctx = t->ctx;
  const size_t E = t->E;
  bool ok = dalloc(ctx, &t->d_tmpl, (size_t)t->N * 3) && dalloc(ctx, &t->d_mask, E) &&
            dalloc(ctx, &t->d_cloud, E * t->ncloud * 3) && dalloc(ctx, &ctx->spc_tape, (size_t)horizon * E * 2) &&
            dalloc(ctx, &ctx->gspc, (size_t)horizon * E * 2) && dalloc(ctx, &ctx->cut_tape, (size_t)horizon * E) &&
            dalloc(ctx, &ctx->dcloud_buf, E * t->ncloud * 3);
  if (!ok) {
    t->err = "dm_task_create: device allocation failed";
    return t;
  }
  ctx->cut_any.assign(horizon, 0);
  ctx->cloud_n = t->ncloud;
  ctx->cloud_stride = t->stride;
  cudaMemcpy(t->d_tmpl, t->tmpl.data(), t->tmpl.size() * sizeof(float), cudaMemcpyHostToDevice);
  t->rng.resize(E);
  t->cursor.assign(E, 0);
  t->c.assign(3 * E, 0.0);
  t->act_t.assign((size_t)horizon * E * t->A, 0.0);
  t->c_t.assign((size_t)horizon * E * 3, 0.0);
  t->cpre_t.assign((size_t)horizon * E * 3, 0.0);
  t->obs_t.assign((size_t)horizon * E * DM_OBS_DIM, 0.f);
  t->cut_t.assign((size_t)horizon * E, 0);
  if (dm_task_reset(t, 0) != DM_OK) return t;
  return t;
}

void dm_task_destroy(DmTask* t) {
  if (!t) return;
  if (t->ctx) {
    void* ptrs[] = {t->d_tmpl, t->d_mask, t->d_cloud};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    dm_destroy(t->ctx);
  }
  delete t;
}

int dm_task_last_error(const DmTask* t, char* buf, int len) {
  if (!t) return DM_ERR_ARG;
  if (buf && len > 0) std::snprintf(buf, (size_t)len, "%s", t->err.c_str());
  return t->err.empty() ? DM_OK : DM_ERR_RUNTIME;
}

int dm_task_dims(const DmTask* t, int* obs_dim, int* act_dim, int* particles_per_env, int* episode_len) {
  if (!t) return DM_ERR_ARG;
  if (obs_dim) *obs_dim = t->od;
  if (act_dim) *act_dim = t->A;
  if (particles_per_env) *particles_per_env = t->N;
  if (episode_len) *episode_len = t->cfg.episode_len;
  return DM_OK;
}

int dm_task_tape_steps(const DmTask* t) { return t ? t->T : 0; }
DmContext* dm_task_context(DmTask* t) { return t ? t->ctx : nullptr; }

int dm_task_reset(DmTask* t, unsigned long long seed) {
  if (!t || !t->ctx) return DM_ERR_ARG;
  DmContext* ctx = t->ctx;
  if (ctx->poisoned && ctx->h_flags->err_key == ~0ull) ctx->poisoned = false;
  for (int e = 0; e < t->E; ++e) {
    t->rng[e] = TaskRng(seed, static_cast<uint64_t>(t->env_offset + e));  // env.hpp:66-73
    t->cursor[e] = 0;
    t->draw_reset(e);
  }
  DM_CUDA(cudaMemsetAsync(t->d_mask, 1, t->E, ctx->stream));
  dm_launch(ctx->grid_tiles, 256, 0, ctx->stream, ctx->pdl, k_task_reset, ctx->P, store_view(ctx, 0), t->d_tmpl, t->d_mask, 0);
  ++ctx->launches;
  ctx->steps = 0;
  ctx->cfl_checked = 0;
  ctx->bwd_t = -1;
  ctx->kept_t = -1;
  ctx->kept_ok = false;
  ctx->poisoned = false;
  t->T = 0;
  t->tape_ok = true;
  t->err.clear();
  const int rc = reset_flags(ctx);  // synchronises
  return task_ctx_err(t, rc);
}

int dm_task_observe(DmTask* t, double* obs) {
  if (!t || !t->ctx || !obs) return DM_ERR_ARG;
  DmContext* ctx = t->ctx;
  std::vector<float> o7((size_t)t->E * ctx->od), cl((size_t)t->E * t->ncloud * 3);
  int rc = observe_impl(ctx, nullptr, o7.data(), cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost);
  if (rc != DM_OK) return task_ctx_err(t, rc);
  dm_launch(ctx->grid_tiles, 256, 0, ctx->stream, ctx->pdl, k_cloud, ctx->P, fwd_state(ctx, ctx->steps * ctx->cfg.substeps), t->stride,
                                                    t->ncloud, t->d_cloud, t->ncloud * 3, 0);
  ++ctx->launches;
  DM_CUDA(cudaMemcpyAsync(cl.data(), t->d_cloud, cl.size() * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
  DM_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int e = 0; e < t->E; ++e) {
    double* o = obs + (size_t)e * t->od;
    const float* m = &o7[(size_t)e * ctx->od];
    const double* ce = &t->c[3 * (size_t)e];
    int k = 0;
    if (t->fluid()) {  // tasks.hpp:554-570
      o[k++] = ce[0];
      o[k++] = ce[1];
      o[k++] = t->cfg.target_x - ce[0];
      o[k++] = t->cfg.target_y - ce[1];
      for (int a = 0; a < 3; ++a) o[k++] = m[a];
    } else {  // tasks.hpp:286-304
      for (int a = 0; a < 3; ++a) o[k++] = ce[a];
      o[k++] = (double)m[2] - t->floor_z;
      o[k++] = m[5];
    }
    for (int q = 0; q < 3 * t->ncloud; ++q) o[k++] = cl[(size_t)e * t->ncloud * 3 + q];
  }
  return DM_OK;
}

int dm_task_step(DmTask* t, const double* actions, double* rewards, unsigned char* dones, int record) {
  if (!t || !t->ctx || !actions) return DM_ERR_ARG;
  DmContext* ctx = t->ctx;
  if (ctx->poisoned) return task_fail(t, ctx->err.empty() ? "context poisoned by an earlier error" : ctx->err,
                                      DM_ERR_RUNTIME);
  if (ctx->steps >= t->horizon) {
    if (record) return task_fail(t, "dm_task_step: tape capacity exceeded (horizon)", DM_ERR_CAPACITY);
    int rc = restart_tape(ctx);
    if (rc != DM_OK) return task_ctx_err(t, rc);
    t->T = 0;
  }
  if (!record) t->tape_ok = false;
  const int E = t->E, A = t->A, K = t->K, tt = ctx->steps;
  const double dt = t->cfg.dt, sp = t->speed();
  std::vector<float> cvo((size_t)E * K * 9, 0.f), spc((size_t)E * 2), o7((size_t)E * ctx->od);
  std::vector<double> cnew(3 * (size_t)E), cpre(3 * (size_t)E);
  for (int e = 0; e < E; ++e) {
    const double* a = actions + (size_t)e * A;
    const double* ce = &t->c[3 * (size_t)e];
    double vel[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < A; ++k) vel[k] = task_clamp(a[k], -1.0, 1.0) * sp;
    float* cv = &cvo[(size_t)e * K * 9];
    if (t->fluid()) {  // four inward walls, frozen at the start-of-step pose (tasks.hpp:577-589)
      const double half = t->cfg.container_half;
      for (int w = 0; w < 4; ++w) {
        cv[9 * w + 0] = static_cast<float>(ce[0] - kWallN[w][0] * half);
        cv[9 * w + 1] = static_cast<float>(ce[1] - kWallN[w][1] * half);
        cv[9 * w + 2] = 0.f;
        for (int q = 0; q < 3; ++q) cv[9 * w + 3 + q] = static_cast<float>(vel[q]);
      }
    } else {  // the roller sphere at the start-of-step pose (tasks.hpp:311-316)
      for (int q = 0; q < 3; ++q) {
        cv[q] = static_cast<float>(ce[q]);
        cv[3 + q] = static_cast<float>(vel[q]);
      }
    }
    const int na = t->fluid() ? 2 : 3;  // moved axes (tasks.hpp:326-328, 599-602)
    for (int q = 0; q < 3; ++q) {
      cpre[3 * e + q] = q < na ? ce[q] + vel[q] * dt : ce[q];
      cnew[3 * e + q] = q < na ? task_clamp(cpre[3 * e + q], t->lo(q), t->hi(q)) : ce[q];
    }
    spc[2 * e] = static_cast<float>(cnew[3 * e]);
    spc[2 * e + 1] = static_cast<float>(cnew[3 * e + 1]);
  }
  int rc = step_impl(ctx, cvo.data(), nullptr, o7.data(), cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost,
                     t->fluid() ? spc.data() : nullptr);
  if (rc != DM_OK) return task_ctx_err(t, rc);
  std::vector<unsigned char> done(E, 0);
  bool any = false;
  for (int e = 0; e < E; ++e) {
    const float* m = &o7[(size_t)e * ctx->od];
    double r;
    if (t->fluid()) {  // tasks.hpp:604-615
      const double ex = cnew[3 * e] - t->cfg.target_x, ey = cnew[3 * e + 1] - t->cfg.target_y;
      const double dist = std::sqrt(ex * ex + ey * ey + 1e-12);
      r = task_tiered(dist, 0.02, 1.0, 2.0) - (double)m[6];
    } else {  // tasks.hpp:330-338
      const double mean_z = (double)m[2] - t->floor_z;
      r = task_tiered(mean_z * (1.0 / t->cfg.h_flat), 0.33, 1.0, 2.0) - (double)m[5];
    }
    if (rewards) rewards[e] = r;
    const size_t te = (size_t)tt * E + e;
    for (int k = 0; k < A; ++k) t->act_t[te * A + k] = actions[(size_t)e * A + k];
    for (int q = 0; q < 3; ++q) {
      t->c_t[te * 3 + q] = t->c[3 * (size_t)e + q];
      t->cpre_t[te * 3 + q] = cpre[3 * e + q];
      t->c[3 * (size_t)e + q] = cnew[3 * e + q];
    }
    for (int q = 0; q < DM_OBS_DIM; ++q) t->obs_t[te * DM_OBS_DIM + q] = m[q];
    // EnvBatch::step: done at the episode length, auto-reset (env.hpp:80-90)
    if (++t->cursor[e] >= t->cfg.episode_len) {
      done[e] = 1;
      any = true;
      t->cursor[e] = 0;
      t->draw_reset(e);
    }
    t->cut_t[te] = done[e];
  }
  if (dones)
    for (int e = 0; e < E; ++e) dones[e] = done[e];
  if (any) {  // the done envs' particles take the template (Task::reset); the tape is cut there
    DM_CUDA(cudaMemcpyAsync(t->d_mask, done.data(), E, cudaMemcpyHostToDevice, ctx->stream));
    DM_CUDA(cudaMemcpyAsync(ctx->cut_tape + (size_t)tt * E, done.data(), E, cudaMemcpyHostToDevice, ctx->stream));
    dm_launch(ctx->grid_tiles, 256, 0, ctx->stream, ctx->pdl, k_task_reset, ctx->P, fwd_state(ctx, ctx->steps * ctx->cfg.substeps),
                                                           t->d_tmpl, t->d_mask, 0);
    ++ctx->launches;
    ctx->cut_any[tt] = 1;
    if (ctx->kept_t == tt) ctx->kept_ok = false;  // the kept segment's exit state was replaced
    DM_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  t->T = ctx->steps;
  return DM_OK;
}

int dm_task_backward(DmTask* t, const double* drewards, const double* dobs, double* dactions) {
  if (!t || !t->ctx) return DM_ERR_ARG;
  DmContext* ctx = t->ctx;
  const int T = t->T, E = t->E, A = t->A, K = t->K, od = t->od, nc = t->ncloud;
  if (T == 0) return task_fail(t, "dm_task_backward: no recorded steps");
  if (!t->tape_ok) return task_fail(t, "dm_task_backward: the tape holds unrecorded steps (record = 0)");
  int rc = backward_begin(ctx, nullptr, nullptr, nullptr, nullptr, cudaMemcpyHostToDevice);
  if (rc != DM_OK) return task_ctx_err(t, rc);
  std::vector<double> gc(3 * (size_t)E, 0.0), g(3 * (size_t)E), gspc(2 * (size_t)E);
  std::vector<float> dob((size_t)E * ctx->od), dcl((size_t)E * nc * 3), dcvo((size_t)E * K * 9);
  const double dt = t->cfg.dt, sp = t->speed();
  for (int tt = T - 1; tt >= 0; --tt) {
    std::fill(dob.begin(), dob.end(), 0.f);
    std::fill(dcl.begin(), dcl.end(), 0.f);
    bool any_cloud = false;
    for (int e = 0; e < E; ++e) {
      const size_t te = (size_t)tt * E + e;
      const bool cut = t->cut_t[te] != 0;
      double* ge = &g[3 * (size_t)e];
      for (int q = 0; q < 3; ++q) ge[q] = cut ? 0.0 : gc[3 * (size_t)e + q];  // from the later steps
      float* db = &dob[(size_t)e * ctx->od];
      // cotangent of obs_{t+1}: the observation of this step's end state (none across a reset)
      if (dobs && !cut) {
        const double* d = dobs + ((size_t)(tt + 1) * E + e) * od;
        int k;
        if (t->fluid()) {
          ge[0] += d[0] - d[2];
          ge[1] += d[1] - d[3];
          for (int a = 0; a < 3; ++a) db[a] += static_cast<float>(d[4 + a]);
          k = 7;
        } else {
          for (int a = 0; a < 3; ++a) ge[a] += d[a];
          db[2] += static_cast<float>(d[3]);  // mean_z = com_z - floor_z
          db[5] += static_cast<float>(d[4]);
          k = 5;
        }
        for (int q = 0; q < 3 * nc; ++q) {
          dcl[(size_t)e * nc * 3 + q] = static_cast<float>(d[k + q]);
          any_cloud = any_cloud || d[k + q] != 0.0;
        }
      }
      // the reward of this step
      const double dr = drewards ? drewards[te] : 0.0;
      if (dr != 0.0) {
        if (t->fluid()) {
          // c_{t+1} before any reset: clamp(c_pre) of this step
          double cx = task_clamp(t->cpre_t[te * 3 + 0], t->lo(0), t->hi(0));
          double cy = task_clamp(t->cpre_t[te * 3 + 1], t->lo(1), t->hi(1));
          const double ex = cx - t->cfg.target_x, ey = cy - t->cfg.target_y;
          const double dist = std::sqrt(ex * ex + ey * ey + 1e-12);
          const double gd = dr * task_dtiered(dist, 0.02, 1.0, 2.0) / dist;
          ge[0] += gd * ex;
          ge[1] += gd * ey;
          db[6] += static_cast<float>(-dr);
        } else {
          const double mean_z = (double)t->obs_t[te * DM_OBS_DIM + 2] - t->floor_z;
          const double ratio = mean_z * (1.0 / t->cfg.h_flat);
          db[2] += static_cast<float>(dr * task_dtiered(ratio, 0.33, 1.0, 2.0) * (1.0 / t->cfg.h_flat));
          db[5] += static_cast<float>(-dr);
        }
      }
    }
    rc = backward_step(ctx, dob.data(), dcvo.data(), nullptr, cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost,
                       any_cloud ? dcl.data() : nullptr, t->fluid() ? gspc.data() : nullptr);
    if (rc != DM_OK) return task_ctx_err(t, rc);
    for (int e = 0; e < E; ++e) {
      const size_t te = (size_t)tt * E + e;
      double* ge = &g[3 * (size_t)e];
      if (t->fluid()) {
        ge[0] += gspc[2 * (size_t)e];
        ge[1] += gspc[2 * (size_t)e + 1];
      }
      const int na = t->fluid() ? 2 : 3;
      double gcur[3] = {0.0, 0.0, 0.0}, gvel[3] = {0.0, 0.0, 0.0};
      for (int q = 0; q < na; ++q) {
        const double gp = ge[q] * task_dclamp(t->cpre_t[te * 3 + q], t->lo(q), t->hi(q));
        gcur[q] = gp;
        gvel[q] = gp * dt;
      }
      const float* dc = &dcvo[(size_t)e * K * 9];
      for (int w = 0; w < K; ++w)
        for (int q = 0; q < na; ++q) {
          gcur[q] += dc[9 * w + q];      // collider center (wall: c - n half)
          gvel[q] += dc[9 * w + 3 + q];  // collider velocity
        }
      double* da = dactions ? dactions + te * A : nullptr;
      for (int k = 0; k < A; ++k)
        if (da) da[k] = gvel[k] * sp * task_dclamp(t->act_t[te * A + k], -1.0, 1.0);
      for (int q = 0; q < 3; ++q) gc[3 * (size_t)e + q] = gcur[q];
    }
  }
  rc = backward_end(ctx, nullptr, nullptr, nullptr, nullptr, nullptr, cudaMemcpyDeviceToHost);
  if (rc != DM_OK) return task_ctx_err(t, rc);
  // the tape is consumed: later steps record a new rollout from the current state
  rc = restart_tape(ctx);
  if (rc != DM_OK) return task_ctx_err(t, rc);
  t->T = 0;
  t->tape_ok = true;
  return DM_OK;
}

}  // extern "C"
