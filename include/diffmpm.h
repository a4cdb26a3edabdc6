/* diffmpm: B200-native batched differentiable MLS-MPM (C ABI).
 *
 * Drop-in boundary for the reference's simulator path
 * (/root/reference/proj/include/diffsim).  The reference surface is C++
 * templates with no FFI; every entry point below names the reference symbol
 * it replaces (file:line).  Plain pointers and sizes only.  Host-pointer
 * entry points copy through pinned staging; *_device variants take device
 * pointers on the context's stream.
 *
 * Threading: one context per GPU, one CUDA stream per context; a context is
 * not thread-safe; separate contexts may be driven from separate threads or
 * processes.
 *
 * Errors: every call returns DM_OK or a DM_ERR_* code; dm_last_error()
 * returns the reference's exception text (mpm.hpp:156-158, 203-205, 338-339,
 * 354; tape.hpp:238-240) so adapters can rethrow it verbatim.
 */
#ifndef DIFFMPM_H
#define DIFFMPM_H

#ifdef __cplusplus
extern "C" {
#endif

#define DM_OK 0
#define DM_ERR_ARG 1       /* std::invalid_argument (mpm.hpp:354) */
#define DM_ERR_RUNTIME 2   /* std::runtime_error (mpm.hpp:156-158, 169, 205, 338-339) */
#define DM_ERR_CUDA 3
#define DM_ERR_CAPACITY 4  /* tape capacity (max_steps) exceeded */

#define DM_MAX_COLLIDERS 4
#define DM_MAX_GROUPS 16
#define DM_MAX_MATERIALS 4
#define DM_OBS_DIM 7 /* com(3), var(3), spill(1); + 8 per pooled group, see dm_obs_dim */

/* MpmMaterial (mpm.hpp:23-41) extended: kind 0 fixed-corotated,
 * 1 neo-Hookean (fem.hpp:124-142) + x-axis actuation, 2 elastoplastic
 * (Hencky / von Mises, mpm.hpp:165-198), 3 fluid (mpm.hpp:200-210) +
 * viscosity.  Particle mass = density * volume (sample_box, mpm.hpp:382-393). */
typedef struct {
  int kind;
  double youngs, poisson, density, volume, yield_stress;
  int wide_yield;
  double viscosity, act_strength, bulk;
} DmMaterial;

/* SdfCollider geometry (mpm.hpp:76-84) extended: kind 0 plane, 1 sphere,
 * 2 box, 3 capped cylinder, 4 open-top hollow box.  Center, velocity and
 * angular velocity are per control step (dm_step's cvo). */
typedef struct {
  int kind;
  double normal[3]; /* plane normal / cylinder axis (unit) */
  double radius;    /* sphere, cylinder */
  double half[3];   /* box; hollow-box cavity half extents */
  double length;    /* cylinder full length */
  double thickness; /* hollow-box wall thickness */
} DmColliderShape;

typedef struct {
  int device;
  int num_envs;          /* EnvBatch size (env.hpp:55-117) */
  int particles_per_env;
  int dims[3];           /* MpmGrid::dims (mpm.hpp:58) */
  double dx, dt;         /* MpmGrid::dx, mpm_step dt */
  double gravity[3];
  int boundary;          /* 0 slip (mpm.hpp:296-302), 1 sticky */
  double alpha_c, mu_b;  /* CouplingParams (mpm.hpp:134-137) */
  int num_colliders;     /* per env, <= DM_MAX_COLLIDERS */
  int num_groups;        /* actuation groups, <= DM_MAX_GROUPS */
  int substeps;          /* mpm_step substeps per control step (mpm.hpp:349-353) */
  int max_steps;         /* tape capacity in control steps */
  int checkpoint_every;  /* substeps per recompute segment; 0 = one per control step (algo.hpp:79-104) */
  double spill_half, spill_temp; /* spill observable footprint (tasks.hpp:606-614) */
  int obs_groups;        /* pooled per-group statistics appended to the observables (config 5):
                            per group mean x (3), mean v (3), var z (1), mean |v| (1) */
} DmConfig;

typedef struct DmContext DmContext;

/* Context owning every device buffer (SURVEY.md 8(b) "create/destroy"). */
DmContext* dm_create(const DmConfig* cfg, const DmMaterial* mats, int num_materials,
                     const DmColliderShape* shapes);
void dm_destroy(DmContext* ctx);
int dm_last_error(const DmContext* ctx, char* buf, int len);
/* cudaStream_t of the context, as void*. */
void* dm_stream(DmContext* ctx);
/* Bytes of device memory held by the context. */
unsigned long long dm_device_bytes(const DmContext* ctx);

/* Upload the state (lift_state/convert_state, env.hpp:41-47, mpm.hpp:425-444)
 * and reset the tape to step 0.  Host layout per env in the reference visit
 * order (tasks.hpp:203-219): x [E][N][3], v [E][N][3], F [E][N][9] row-major,
 * C [E][N][9]; material [E][N], group [E][N] (group may be NULL). */
int dm_set_state(DmContext* ctx, const float* x, const float* v, const float* F, const float* C,
                 const int* material, const int* group);
int dm_set_state_device(DmContext* ctx, const float* x, const float* v, const float* F, const float* C,
                        const int* material, const int* group);
/* Download the current state in the original particle order (lower_state, env.hpp:49-53). */
int dm_get_state(DmContext* ctx, float* x, float* v, float* F, float* C);
int dm_get_state_device(DmContext* ctx, float* x, float* v, float* F, float* C);

/* One control step = `substeps` MLS-MPM substeps (mpm_step, mpm.hpp:348-367)
 * with colliders frozen at the given pose (Task::step, tasks.hpp:306-339).
 * cvo [E][K][9]: center, velocity, angular velocity per collider;
 * act [E][G] actuation (may be NULL); obs [E][7] written after the step
 * (may be NULL).  The step is recorded on the tape (Tape::checkpoint,
 * tape.hpp:181-216). */
int dm_step(DmContext* ctx, const float* cvo, const float* act, float* obs);
int dm_step_device(DmContext* ctx, const float* cvo, const float* act, float* obs);

/* Backward through every recorded step (Tape::backward + backward_segment,
 * tape.hpp:124-164, 227-255).
 *   dobs      [T][E][7]  cotangents of the per-step observables (may be NULL)
 *   dfinal_x/v/F/C       cotangents of the final state, original order (may be NULL)
 * outputs (any may be NULL):
 *   dx0, dv0, dF0, dC0   cotangents of the initial state, original order
 *   dcvo  [T][E][K][9]   collider center / velocity / omega cotangents
 *   dact  [T][E][G]      actuation cotangents
 *   dE    [E][num_materials] Young's modulus cotangents (the reference tape
 *         cannot produce these, mpm.hpp:23-41) */
int dm_backward(DmContext* ctx, const float* dobs, const float* dfinal_x, const float* dfinal_v,
                const float* dfinal_F, const float* dfinal_C, float* dx0, float* dv0, float* dF0, float* dC0,
                float* dcvo, float* dact, double* dE);
int dm_backward_device(DmContext* ctx, const float* dobs, const float* dfinal_x, const float* dfinal_v,
                       const float* dfinal_F, const float* dfinal_C, float* dx0, float* dv0, float* dF0,
                       float* dC0, float* dcvo, float* dact, double* dE);

/* Incremental backward, one control step at a time in reverse order, for
 * callers whose per-step cotangents depend on the previous step's results
 * (a policy in the loop: action_t = pi(obs_t)).  begin: final-state
 * cotangent (any pointer may be NULL); step: cotangent of the observables of
 * the latest unprocessed step t (dobs_t [E][obs_dim], may be NULL), returns
 * that step's actuation / collider cotangents (dact_t [E][G], dcvo_t
 * [E][K][9], may be NULL); end: initial-state and Young's modulus cotangents.
 * dm_backward is begin + steps T-1..0 + end. */
int dm_backward_begin(DmContext* ctx, const float* dfinal_x, const float* dfinal_v, const float* dfinal_F,
                      const float* dfinal_C);
int dm_backward_begin_device(DmContext* ctx, const float* dfinal_x, const float* dfinal_v, const float* dfinal_F,
                             const float* dfinal_C);
int dm_backward_step(DmContext* ctx, const float* dobs_t, float* dcvo_t, float* dact_t);
int dm_backward_step_device(DmContext* ctx, const float* dobs_t, float* dcvo_t, float* dact_t);
int dm_backward_end(DmContext* ctx, float* dx0, float* dv0, float* dF0, float* dC0, double* dE);
int dm_backward_end_device(DmContext* ctx, float* dx0, float* dv0, float* dF0, float* dC0, double* dE);

/* Observables of the current state without stepping (the reset observation,
 * Task::observe, tasks.hpp:286-304).  cvo [E][K][9] may be NULL (no spill). */
int dm_observe(DmContext* ctx, const float* cvo, float* obs);
int dm_observe_device(DmContext* ctx, const float* cvo, float* obs);
/* Observable dimension per env: DM_OBS_DIM + 8 * obs_groups. */
int dm_obs_dim(const DmContext* ctx);
/* Number of control steps currently on the tape. */
int dm_tape_steps(const DmContext* ctx);

/* Device-side env reset: EnvBatch::reset / reset_env (env.hpp:66-96) with a
 * sample_box lattice (mpm.hpp:371-395) and per-env RngStream(seed, env)
 * draws (rng.hpp:11-55, env.hpp:71), generated on the GPU bit-identically to
 * the host generator (paper_2412_12089_b200/scenes.py lattice_reset_host) --
 * no host upload at reset.  Per env e (global index env_offset + e), in
 * double precision without contraction, then rounded to fp32:
 *   d_a   = origin_lo + (origin_hi - origin_lo) * u_{a+1}      a < origin_draws (else 0)
 *   x_p,a = (origin_a + d_a) + ((ijk_p,a + 0.5) * spacing_a)  lattice (i, j, k)-major, or with
 *         size_a > 0 sample_box's (origin_a + d_a) + (size_a * (ijk_p,a + 0.5)) / counts_a
 *   x_p,a += jitter_lo + (jitter_hi - jitter_lo) * u_{D + 3p + a + 1}      if jitter_hi > jitter_lo
 *   v_p,a  = velocity_sigma * normal (Box-Muller cosine, rng.hpp:35-43, draws after the jitter)
 *   F = I, C = 0
 * u_k = k-th double of the env's stream.  Envs whose mask byte is 0 keep
 * their current state; the tape restarts at step 0 (the state is a new
 * initial state, as dm_set_state).  origin_delta [E][3] receives d (may be
 * NULL); particle_group [N] gives every env's per-particle actuation group
 * (may be NULL: spec.group). */
typedef struct {
  double origin[3];
  double spacing[3];
  int counts[3]; /* nx * ny * nz == particles_per_env */
  int origin_draws;
  double origin_lo, origin_hi;
  double jitter_lo, jitter_hi;
  double velocity_sigma;
  int material, group;
  double size[3]; /* > 0: sample_box's expression origin_a + (size_a * (ijk_a + 0.5)) / counts_a
                     (mpm.hpp:386-388) instead of the spacing form */
} DmLatticeReset;
int dm_reset_lattice(DmContext* ctx, const DmLatticeReset* spec, unsigned long long seed, int env_offset,
                     const unsigned char* env_mask, const int* particle_group, double* origin_delta);
int dm_reset_lattice_device(DmContext* ctx, const DmLatticeReset* spec, unsigned long long seed, int env_offset,
                            const unsigned char* env_mask, const int* particle_group, double* origin_delta);

/* Synchronises the context stream and reports what the device recorded
 * since the last synchronising call: the first error in substep order
 * (mpm.hpp:156-158, 169, 205, 338-339) and one CFL warning per violating
 * control step (mpm.hpp:355-361, stderr).  Host-pointer entry points do this
 * after every control step; the *_device entry points do not synchronise, so
 * their device-detected errors surface at the next synchronising call
 * (dm_sync, dm_get_state*, dm_observe*, dm_backward*). */
int dm_sync(DmContext* ctx);

/* Test hook for the replay verification (Tape::backward_segment,
 * tape.hpp:234-241; test_tape.cpp:311-323): while replaying control step
 * `step` in the backward pass, flip the lowest mantissa bit of particle
 * `particle`'s x in env `env` -- a non-deterministic forward.  The backward
 * then fails with "checkpoint replay: non-deterministic forward (exit value
 * k changed)".  step = -1 disables it. */
int dm_debug_inject(DmContext* ctx, int step, int env, int particle);

/* Parity hooks: bin keys / stable permutation of the
 * current state (per env, local indices) and the current physical order's
 * original particle ids. */
int dm_debug_sort(DmContext* ctx, int* keys, int* perm);
/* Per-kernel-class CUDA-event timing on the context stream.  Classes:
 * 0 bin, 1 p2g, 2 g2p, 3 g2p_adj, 4 p2g_adj, 5 env_reduce, 6 obs, 7 obs_adj,
 * 8 layout, 9 grid, 10 grid_adj.  Returns (and clears) the accumulated ms /
 * launch counts and sets whether timing is recorded from now on.  ms, counts:
 * 11 entries or NULL. */
int dm_profile(DmContext* ctx, int enable, double* ms, long long* counts);
/* Kernel launches issued since the context was created. */
unsigned long long dm_launch_count(const DmContext* ctx);

/* ---------------- reference tasks (env.hpp, tasks.hpp) ----------------
 * EnvBatch<Task> (env.hpp:55-117) for the reference's MPM tasks on the GPU
 * simulator: MiniFluidMove (tasks.hpp:502-645: fluid in a container of four
 * inward plane walls moved by 2-D actions, reward = tiered distance of the
 * container to the target minus the smoothed spill) and MiniRollFlat
 * (tasks.hpp:232-369: an elastoplastic block flattened by a sphere roller
 * moved by 3-D actions, reward = tiered(mean_z / h_flat) - Var_z).  The
 * action -> collider maps with their clamps, the per-env task state
 * (container / roller position), the rewards, the observations (with the
 * stride-subsampled point cloud) and the auto-reset from each env's own
 * RngStream(seed, env_offset + i) run behind this ABI; dm_task_backward
 * returns dL/dactions for L = sum drewards * rewards + sum dobs * obs
 * through the recorded steps (recompute-on-backward per control step, the
 * role of step_checkpointed, algo.hpp:79-104).  Gradients do not flow across
 * an auto-reset (collect_rollout, algo.hpp:171-178).  Actions, rewards and
 * observations are double, as the reference's EnvBatch. */
#define DM_TASK_FLUID_MOVE 0
#define DM_TASK_ROLL_FLAT 1
typedef struct {
  int kind;
  int grid_n, ppc;        /* MPM grid resolution, particles per cell (sample_box) */
  double dt;              /* control step */
  int substeps, episode_len, cloud_k;
  /* MiniFluidMove::Config */
  double container_half, fill, speed, start_x, start_y, target_x, target_y, spill_temp;
  /* MiniRollFlat::Config */
  double block_size, block_height, roller_radius, roller_speed, h_flat, youngs, yield_stress;
} DmTaskConfig;
typedef struct DmTask DmTask;

/* The reference's Config{} defaults for a task kind. */
void dm_task_default_config(int kind, DmTaskConfig* out);
/* num_envs envs (global indices env_offset + i); horizon = tape capacity in
 * control steps (a full tape restarts itself when stepping with record = 0). */
DmTask* dm_task_create(const DmTaskConfig* cfg, int num_envs, int env_offset, int horizon, int device);
void dm_task_destroy(DmTask* task);
int dm_task_last_error(const DmTask* task, char* buf, int len);
/* obs_dim(), act_dim(), particles per env, episode_len() (tasks.hpp). */
int dm_task_dims(const DmTask* task, int* obs_dim, int* act_dim, int* particles_per_env, int* episode_len);
/* EnvBatch::reset(seed): every env re-drawn from RngStream(seed, env_offset + i); the tape restarts. */
int dm_task_reset(DmTask* task, unsigned long long seed);
/* Task::observe of every env: obs [E][obs_dim]. */
int dm_task_observe(DmTask* task, double* obs);
/* EnvBatch::step: actions [E][act_dim] -> rewards [E], dones [E] (either may
 * be NULL); done envs are reset from their own stream.  record != 0 records
 * the step on the tape for dm_task_backward. */
int dm_task_step(DmTask* task, const double* actions, double* rewards, unsigned char* dones, int record);
/* Backward through the recorded steps t = 0..T-1: drewards [T][E] (may be
 * NULL), dobs [T+1][E][obs_dim] cotangents of the observations before each
 * step and after the last (row 0, the reset observation, carries no
 * gradient; may be NULL) -> dactions [T][E][act_dim].  The tape restarts. */
int dm_task_backward(DmTask* task, const double* drewards, const double* dobs, double* dactions);
/* Recorded steps on the tape. */
int dm_task_tape_steps(const DmTask* task);
/* The underlying simulator context (device buffers, stream, profiling). */
DmContext* dm_task_context(DmTask* task);

#ifdef __cplusplus
}
#endif
#endif /* DIFFMPM_H */
