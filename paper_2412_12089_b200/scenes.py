"""Seeded synthetic scenes for the five BASELINE.json configurations.

Host-side task layer: builds initial particle states, material tables,
collider geometry, per-step actions, and the action -> collider / actuation
maps (with their vector-Jacobian products) that the reference tasks keep in
``Task::step`` (/root/reference/proj/include/diffsim/tasks.hpp:306-339,
572-616).  Every random draw comes from ``RngStream(seed, env_index)``
(env.hpp:71) so CPU oracle and GPU consume bit-identical inputs, and an env's
inputs do not depend on how envs are sharded over GPUs.

The BASELINE configs name no public dataset; all inputs are synthetic with
the shapes, sizes and parameter values the configs state (DESIGN.md lists the
choices the configs leave open).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .rng import RngStream

GRAVITY = (0.0, 0.0, -9.8)


@dataclass
class Scene:
    name: str
    n_envs: int
    n_per_env: int
    sim: dict
    materials: list
    colliders: list            # geometry per collider slot
    n_ctrl: int
    n_sub: int
    loss: dict
    x: np.ndarray              # [E, N, 3]
    v: np.ndarray              # [E, N, 3]
    F: np.ndarray              # [E, N, 9]
    C: np.ndarray              # [E, N, 9]
    material: np.ndarray       # [E, N] int32
    group: np.ndarray          # [E, N] int32
    actions: np.ndarray        # [E, T, A]
    task: "Task" = None
    checkpoint_every: int = 0  # substeps per recompute segment (0 = per control step)
    env_offset: int = 0        # global index of env 0 (sharding)
    extra: dict = field(default_factory=dict)

    @property
    def n_particles(self) -> int:
        return self.n_envs * self.n_per_env

    def cvo_act(self):
        """Per-env per-step collider (center, velocity, omega) [E,T,K,9] and
        actuation [E,T,G] from the actions."""
        return self.task.forward(self.actions)

    def env_state(self, e: int) -> dict:
        return {"x": self.x[e], "v": self.v[e], "F": self.F[e], "C": self.C[e],
                "material": self.material[e], "group": self.group[e]}

    def env_cols(self, e: int, cvo: np.ndarray) -> list:
        out = []
        for k, g in enumerate(self.colliders):
            d = dict(g)
            d["cvo"] = cvo[e, :, k, :]
            out.append(d)
        return out


class Task:
    """Maps actions to per-step collider kinematics / actuation (forward) and
    back (vjp).  Colliders are frozen at the start-of-step pose for all
    substeps and moved afterwards (tasks.hpp:311-316, 326-328)."""

    n_cols = 0
    n_act = 0

    def forward(self, actions):
        E, T, _ = actions.shape
        return np.zeros((E, T, max(1, self.n_cols), 9)), np.zeros((E, T, max(1, self.n_act)))

    def vjp(self, actions, g_cvo, g_act):
        return np.zeros_like(actions)


class MovingColliderTask(Task):
    """center_{t+1} = clip(center_t + v_t dt_ctrl, lo, hi); v_t = speed * clip(a_t)
    (MiniRollFlat/MiniFluidMove roller and container kinematics,
    tasks.hpp:326-328, 599-602), optional angular velocity omega_t."""

    def __init__(self, center0, speed, dt_ctrl, lo, hi, lin_axes, ang_axes=(), ang_speed=0.0):
        self.center0 = np.asarray(center0, dtype=np.float64)  # [E, 3]
        self.speed = float(speed)
        self.dt_ctrl = float(dt_ctrl)
        self.lo = np.asarray(lo, dtype=np.float64)
        self.hi = np.asarray(hi, dtype=np.float64)
        self.lin_axes = tuple(lin_axes)
        self.ang_axes = tuple(ang_axes)
        self.ang_speed = float(ang_speed)
        self.n_cols = 1
        self.n_act = 0

    def _vel(self, a):
        E, T, _ = a.shape
        ac = np.clip(a, -1.0, 1.0)
        vel = np.zeros((E, T, 3))
        om = np.zeros((E, T, 3))
        for i, ax in enumerate(self.lin_axes):
            vel[:, :, ax] = self.speed * ac[:, :, i]
        for j, ax in enumerate(self.ang_axes):
            om[:, :, ax] = self.ang_speed * ac[:, :, len(self.lin_axes) + j]
        return vel, om

    def forward(self, actions):
        E, T, _ = actions.shape
        vel, om = self._vel(actions)
        cvo = np.zeros((E, T, 1, 9))
        c = self.center0.copy()
        self._centers = []
        for t in range(T):
            cvo[:, t, 0, 0:3] = c
            cvo[:, t, 0, 3:6] = vel[:, t]
            cvo[:, t, 0, 6:9] = om[:, t]
            self._centers.append(c.copy())
            c = np.clip(c + vel[:, t] * self.dt_ctrl, self.lo, self.hi)
        return cvo, np.zeros((E, T, 1))

    def vjp(self, actions, g_cvo, g_act):
        E, T, A = actions.shape
        vel, om = self._vel(actions)
        self.forward(actions)
        g_vel = g_cvo[:, :, 0, 3:6].copy()
        g_om = g_cvo[:, :, 0, 6:9]
        gc = np.zeros((E, 3))  # adjoint of center_{t+1}
        for t in range(T - 1, -1, -1):
            pre = self._centers[t] + vel[:, t] * self.dt_ctrl
            inside = (pre > self.lo) & (pre < self.hi)
            gpre = gc * inside
            g_vel[:, t] += gpre * self.dt_ctrl
            gc = gpre + g_cvo[:, t, 0, 0:3]
        ga = np.zeros_like(actions)
        active = (actions > -1.0) & (actions < 1.0)
        for i, ax in enumerate(self.lin_axes):
            ga[:, :, i] = g_vel[:, :, ax] * self.speed
        for j, ax in enumerate(self.ang_axes):
            ga[:, :, len(self.lin_axes) + j] = g_om[:, :, ax] * self.ang_speed
        return ga * active


class ActuationTask(Task):
    """act_{t,g} = clip(a_{t,g}, -1, 1) (per-group muscle activation)."""

    def __init__(self, n_groups):
        self.n_act = n_groups
        self.n_cols = 0

    def forward(self, actions):
        E, T, _ = actions.shape
        return np.zeros((E, T, 1, 9)), np.clip(actions, -1.0, 1.0)

    def vjp(self, actions, g_cvo, g_act):
        return g_act * ((actions > -1.0) & (actions < 1.0))


# ---- samplers (mpm.hpp:371-423 style lattices) ----

def lattice(org, counts, spacing):
    """Cell-centred lattice: org + (i + 0.5) * spacing, particle-major in
    (i, j, k) order (sample_box, mpm.hpp:383-395)."""
    nx, ny, nz = counts
    i, j, k = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    pts = np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1).astype(np.float64) + 0.5
    return np.asarray(org, dtype=np.float64) + pts * np.asarray(spacing, dtype=np.float64)


def lattice_reset_spec(origin, counts, spacing, origin_draws=0, origin_range=(0.0, 0.0), jitter=(0.0, 0.0),
                       velocity_sigma=0.0, material=0, group=0, size=None):
    """Reset descriptor of a seeded lattice env (include/diffmpm.h DmLatticeReset).
    size: sample_box's box extent -- positions origin + (size (ijk + 0.5)) / counts
    (mpm.hpp:386-388) instead of origin + (ijk + 0.5) spacing."""
    return {"origin": tuple(float(a) for a in origin), "counts": tuple(int(c) for c in counts),
            "spacing": tuple(float(a) for a in spacing), "origin_draws": int(origin_draws),
            "origin_range": tuple(float(a) for a in origin_range), "jitter": tuple(float(a) for a in jitter),
            "velocity_sigma": float(velocity_sigma), "material": int(material), "group": int(group),
            "size": tuple(float(a) for a in size) if size is not None else (0.0, 0.0, 0.0)}


def sample_box(org, size, dx, ppc):
    """sample_box (mpm.hpp:371-395): lattice with spacing dx / cbrt(ppc),
    counts round(size / h) (>= 1), positions org + size (i + 0.5) / n in
    (i, j, k)-major order; returns (x [N, 3], particle volume)."""
    h = dx / np.cbrt(float(ppc))
    n = [max(1, int(np.round(s / h))) for s in size]
    vol = (size[0] / n[0]) * (size[1] / n[1]) * (size[2] / n[2])
    i, j, k = np.meshgrid(np.arange(n[0]), np.arange(n[1]), np.arange(n[2]), indexing="ij")
    ijk = np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1).astype(np.float64)
    x = np.asarray(org, np.float64) + (np.asarray(size, np.float64) * (ijk + 0.5)) / np.asarray(n, np.float64)
    return x, vol


def sample_cylinder(base_center, radius, height, dx, ppc):
    """sample_cylinder (mpm.hpp:397-423): the sample_box lattice of the
    cylinder's bounding box, keeping points with rx^2 + ry^2 <= r^2 (box
    order); returns (x [N, 3], particle volume of the box lattice)."""
    bc = np.asarray(base_center, np.float64)
    x, vol = sample_box((bc[0] - radius, bc[1] - radius, bc[2]), (2.0 * radius, 2.0 * radius, height), dx, ppc)
    rx, ry = x[:, 0] - bc[0], x[:, 1] - bc[1]
    return x[rx * rx + ry * ry <= radius * radius], vol


def lattice_reset_host(spec, seed, env_offset, n_envs):
    """Host generator of dm_reset_lattice (the device kernel restates it
    bit-for-bit): per env the stream RngStream(seed, env_offset + e) draws the
    origin offsets, then per-particle jitter (3 per particle), then Box-Muller
    velocities (env.hpp:66-96, mpm.hpp:371-395, rng.hpp:11-55).  Returns
    x [E,N,3] (float64), v [E,N,3], origin deltas [E,3]."""
    cnt = spec["counts"]
    N = cnt[0] * cnt[1] * cnt[2]
    i, j, k = np.meshgrid(np.arange(cnt[0]), np.arange(cnt[1]), np.arange(cnt[2]), indexing="ij")
    ijk = np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1).astype(np.float64)
    lo, hi = spec["origin_range"]
    jlo, jhi = spec["jitter"]
    xs, vs, ds = [], [], []
    size = np.asarray(spec.get("size", (0.0, 0.0, 0.0)), np.float64)
    for e in range(n_envs):
        r = RngStream(seed, env_offset + e)
        d = np.zeros(3)
        nd = spec["origin_draws"]
        if nd:
            d[:nd] = r.uniform(lo, hi, nd)
        off = np.where(size > 0.0, (size * (ijk + 0.5)) / np.asarray(cnt, np.float64),
                       (ijk + 0.5) * np.asarray(spec["spacing"]))
        x = (np.asarray(spec["origin"]) + d) + off
        if jhi > jlo:
            x = x + r.uniform(jlo, jhi, 3 * N).reshape(N, 3)
        v = np.zeros((N, 3))
        if spec["velocity_sigma"] != 0.0:
            v = spec["velocity_sigma"] * r.normals(3 * N).reshape(N, 3)
        xs.append(x)
        vs.append(v)
        ds.append(d)
    return np.stack(xs), np.stack(vs), np.stack(ds)


def kmeans_groups(pts, k, rng: RngStream, iters=20):
    """Seeded Lloyd k-means over rest positions; init = k distinct draws."""
    n = pts.shape[0]
    idx = []
    u = rng.doubles(4 * k)
    for val in u:
        cand = int(val * n)
        if cand not in idx:
            idx.append(cand)
        if len(idx) == k:
            break
    cent = pts[idx].copy()
    lab = np.zeros(n, dtype=np.int32)
    for _ in range(iters):
        d = ((pts[:, None, :] - cent[None, :, :]) ** 2).sum(-1)
        lab = np.argmin(d, axis=1).astype(np.int32)
        for g in range(k):
            m = lab == g
            if m.any():
                cent[g] = pts[m].mean(0)
    return lab


def _identity_F(E, N):
    F = np.zeros((E, N, 9))
    F[:, :, [0, 4, 8]] = 1.0
    return F


# ---- the five BASELINE configurations ----

def config1(seed=0, n_envs=1, env_offset=0, n_sub=50):
    """Single env elastic jelly cube: 16^3 lattice in [0.3,0.5]^3 with +-0.25
    cell jitter, 32^3 grid, fixed-corotated E=1e4 nu=0.3 rho=1, sticky box,
    dt=1e-4, 50 substeps, v0 ~ N(0, 0.5) per particle, loss |com - (0.5,0.4,0.5)|^2."""
    dx = 1.0 / 32
    spec = lattice_reset_spec((0.3, 0.3, 0.3), (16, 16, 16), (0.2 / 16,) * 3, jitter=(-0.25 * dx, 0.25 * dx),
                              velocity_sigma=0.5, size=(0.2, 0.2, 0.2))
    x, v, _ = lattice_reset_host(spec, seed, env_offset, n_envs)
    N = x.shape[1]
    mats = [{"kind": "fixed_corotated", "E": 1e4, "nu": 0.3, "rho": 1.0, "volume": 0.2 ** 3 / N}]
    sim = {"dims": (32, 32, 32), "dx": dx, "dt": 1e-4, "gravity": GRAVITY, "boundary": "sticky",
           "alpha_c": 100.0, "mu_b": 0.0}
    return Scene("cfg1_jelly", n_envs, N, sim, mats, [], 1, n_sub,
                 {"kind": "com_target", "target": (0.5, 0.4, 0.5)},
                 x, v, _identity_F(n_envs, N), np.zeros((n_envs, N, 9)),
                 np.zeros((n_envs, N), np.int32), np.zeros((n_envs, N), np.int32),
                 np.zeros((n_envs, 1, 1)), Task(), 0, env_offset, {"reset": spec, "seed": seed})


def config2(seed=0, n_envs=32, env_offset=0, n_ctrl=32, n_sub=16):
    """SoftJumper-like actuated neo-Hookean body: 40x16x32 lattice at 2
    particles per cell per axis (spacing dx/2), 48^3 grid, E=3e4 nu=0.3,
    8 k-means actuator groups, x-axis actuation, actions U[-1,1]^8 per step,
    dt=5e-5, 16 x 32 substeps, loss -sum_t mean_z."""
    dx = 1.0 / 48
    h = dx / 2
    cnt = (40, 16, 32)
    size = np.array(cnt) * h
    org = (0.5 - size[0] / 2, 0.5 - size[1] / 2, 3.5 * dx)
    base, _ = sample_box(org, tuple(size), dx, 8)  # 2 particles per cell per axis: counts = cnt
    N = base.shape[0]
    spec = lattice_reset_spec(org, cnt, (h, h, h), size=tuple(size))
    groups = kmeans_groups(base, 8, RngStream(seed, 1 << 40))
    acts = np.stack([RngStream(seed, env_offset + e).uniform(-1.0, 1.0, n_ctrl * 8).reshape(n_ctrl, 8)
                     for e in range(n_envs)])
    # rho = 1000 (the config leaves density open; with rho = 1 the sound speed
    # is 173 m/s and random x-actuation inverts elements within 3 steps)
    mats = [{"kind": "neo_hookean", "E": 3e4, "nu": 0.3, "rho": 1000.0, "volume": h ** 3, "act_strength": 1e4}]
    sim = {"dims": (48, 48, 48), "dx": dx, "dt": 5e-5, "gravity": GRAVITY, "boundary": "slip",
           "alpha_c": 100.0, "mu_b": 0.0}
    x = np.broadcast_to(base, (n_envs, N, 3)).copy()
    return Scene("cfg2_softjumper", n_envs, N, sim, mats, [], n_ctrl, n_sub, {"kind": "neg_mean_z"},
                 x, np.zeros((n_envs, N, 3)), _identity_F(n_envs, N), np.zeros((n_envs, N, 9)),
                 np.zeros((n_envs, N), np.int32), np.broadcast_to(groups, (n_envs, N)).astype(np.int32).copy(),
                 acts, ActuationTask(8), 0, env_offset, {"reset": spec, "seed": seed, "particle_group": groups})


def config3(seed=0, n_envs=256, env_offset=0, n_ctrl=24, n_sub=20, n_per_env=30000):
    """RollingFlat-like dough: 30k particles uniform in a seeded ellipsoid
    (semi-axes 0.12 * U(0.9,1.1)), 64^3 grid, Hencky/von Mises E=5e3 nu=0.2
    sigma_y=50, capped cylinder r=0.03 L=0.3 (axis y) with friction mu_b=0.5
    moved by (v_x, v_z, omega_y) actions, dt=5e-5, 20 x 24 substeps,
    checkpoint every 4 substeps, loss sum_t Var_z."""
    dx = 1.0 / 64
    xs = []
    cz = []
    acts = []
    for e in range(n_envs):
        r = RngStream(seed, env_offset + e)
        semi = 0.12 * r.uniform(0.9, 1.1, 3)
        pts = []
        need = n_per_env
        while need > 0:
            u = r.uniform(-1.0, 1.0, 3 * 2 * need).reshape(-1, 3)
            ok = u[(u ** 2).sum(1) <= 1.0]
            pts.append(ok[:need])
            need -= min(need, ok.shape[0])
        p = np.concatenate(pts)[:n_per_env] * semi
        center = np.array([0.5, 0.5, 3.5 * dx + semi[2]])
        xs.append(p + center)
        cz.append(center[2] + semi[2] + 0.03 + 0.005)
        acts.append(r.uniform(-1.0, 1.0, n_ctrl * 3).reshape(n_ctrl, 3))  # same stream, after geometry
    # particle volume from the nominal ellipsoid (radius 0.12): the same for
    # every env, so an env's inputs do not depend on which envs share the batch
    vol = 4.0 / 3.0 * np.pi * 0.12 ** 3 / n_per_env
    x = np.stack(xs)
    N = n_per_env
    acts = np.stack(acts)
    center0 = np.stack([np.array([0.5, 0.5, z]) for z in cz])
    dt = 5e-5
    task = MovingColliderTask(center0, 0.25, n_sub * dt, lo=(0.1, 0.1, 0.06), hi=(0.9, 0.9, 0.9),
                              lin_axes=(0, 2), ang_axes=(1,), ang_speed=10.0)
    mats = [{"kind": "elastoplastic", "E": 5e3, "nu": 0.2, "rho": 1.0, "volume": vol, "yield_stress": 50.0}]
    cols = [{"kind": "cylinder", "normal": (0.0, 1.0, 0.0), "radius": 0.03, "length": 0.3}]
    sim = {"dims": (64, 64, 64), "dx": dx, "dt": dt, "gravity": GRAVITY, "boundary": "slip",
           "alpha_c": 100.0, "mu_b": 0.5}
    return Scene("cfg3_rollingflat", n_envs, N, sim, mats, cols, n_ctrl, n_sub, {"kind": "var_z"},
                 x, np.zeros((n_envs, N, 3)), _identity_F(n_envs, N), np.zeros((n_envs, N, 9)),
                 np.zeros((n_envs, N), np.int32), np.zeros((n_envs, N), np.int32), acts, task, 4, env_offset)


def config4(seed=0, n_envs=1024, env_offset=0, n_ctrl=16, n_sub=32, lattice_counts=(32, 32, 16)):
    """FluidMove-like weakly compressible fluid in a moving open-top container:
    16,384 particles (32x32x16 lattice) filling the lower half of a 0.3^3
    cavity, 48^3 grid, bulk modulus 2e4, viscosity 0.01, rho=1000, container
    moved by 3-DoF actions U[-1,1]^3 * 0.25 m/s, 32 x 16 substeps, loss
    -sum_t [tiered(|com - p*|) - spill]."""
    dx = 1.0 / 48
    half = 0.15
    cnt = np.array(lattice_counts)
    spacing = np.array([2 * half, 2 * half, half]) / cnt
    # per env the lattice origin (and the container) is offset by two draws
    # U[-0.01, 0.01) from the env's stream; cavity floor at z = 0.15
    spec = lattice_reset_spec((0.5 - half, 0.5 - half, 0.15), cnt, spacing, origin_draws=2,
                              origin_range=(-0.01, 0.01), size=(2 * half, 2 * half, half))
    x, _, d = lattice_reset_host(spec, seed, env_offset, n_envs)
    org = np.asarray(spec["origin"]) + d
    c0 = [np.array([o[0] + half, o[1] + half, 0.15 + half]) for o in org]  # cavity center
    N = x.shape[1]
    acts = np.stack([RngStream(seed, env_offset + e).uniform(-1.0, 1.0, 2 + n_ctrl * 3)[2:].reshape(n_ctrl, 3)
                     for e in range(n_envs)])
    dt = 2.5e-4
    task = MovingColliderTask(np.stack(c0), 0.25, n_sub * dt, lo=(0.33, 0.33, 0.25), hi=(0.67, 0.67, 0.5),
                              lin_axes=(0, 1, 2))
    vol = (2 * half) * (2 * half) * half / N
    mats = [{"kind": "fluid", "E": 2e4, "nu": 0.3, "rho": 1000.0, "volume": vol, "bulk": 2e4, "viscosity": 0.01}]
    cols = [{"kind": "hollow_box", "half": (half, half, half), "thickness": 2 * dx}]
    sim = {"dims": (48, 48, 48), "dx": dx, "dt": dt, "gravity": GRAVITY, "boundary": "slip",
           "alpha_c": 100.0, "mu_b": 0.0}
    loss = {"kind": "fluid_move", "target": (0.55, 0.5, 0.2), "spill_half": half, "spill_temp": 0.01,
            "tier_threshold": 0.02, "tier_low": 1.0, "tier_high": 2.0}
    return Scene("cfg4_fluidmove", n_envs, N, sim, mats, cols, n_ctrl, n_sub, loss,
                 x, np.zeros((n_envs, N, 3)), _identity_F(n_envs, N), np.zeros((n_envs, N, 9)),
                 np.zeros((n_envs, N), np.int32), np.zeros((n_envs, N), np.int32), acts, task, 0, env_offset,
                 {"reset": spec, "seed": seed})


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4}
