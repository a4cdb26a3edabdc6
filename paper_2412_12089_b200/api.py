"""Python mirror of the reference simulator surface over the C ABI
(include/diffmpm.h).

``MpmBatch`` plays the role of the reference's batched MPM state plus tape:
``set_state`` ~ lift_state/convert_state (env.hpp:41-47, mpm.hpp:425-444),
``step`` ~ Task::step -> mpm_step over one control step recorded as a
checkpoint segment (tasks.hpp:306-339, tape.hpp:181-216), ``backward`` ~
Tape::backward (tape.hpp:124-164).  Errors raise the reference's exception
types with its message text (RuntimeError for std::runtime_error,
ValueError for std::invalid_argument).

Arrays may be numpy (host; copied through the ABI's host entry points) or
torch CUDA tensors (device pointers on the context's stream).  There is no
CPU fallback: without the CUDA library or a GPU the constructor raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

KIND_LAW = {"fixed_corotated": 0, "neo_hookean": 1, "elastoplastic": 2, "fluid": 3}
KIND_COL = {"plane": 0, "sphere": 1, "box": 2, "cylinder": 3, "hollow_box": 4}
OBS_DIM = 7


class DmMaterial(C.Structure):
    _fields_ = [("kind", C.c_int), ("youngs", C.c_double), ("poisson", C.c_double), ("density", C.c_double),
                ("volume", C.c_double), ("yield_stress", C.c_double), ("wide_yield", C.c_int),
                ("viscosity", C.c_double), ("act_strength", C.c_double), ("bulk", C.c_double)]


class DmColliderShape(C.Structure):
    _fields_ = [("kind", C.c_int), ("normal", C.c_double * 3), ("radius", C.c_double), ("half", C.c_double * 3),
                ("length", C.c_double), ("thickness", C.c_double)]


class DmConfig(C.Structure):
    _fields_ = [("device", C.c_int), ("num_envs", C.c_int), ("particles_per_env", C.c_int), ("dims", C.c_int * 3),
                ("dx", C.c_double), ("dt", C.c_double), ("gravity", C.c_double * 3), ("boundary", C.c_int),
                ("alpha_c", C.c_double), ("mu_b", C.c_double), ("num_colliders", C.c_int), ("num_groups", C.c_int),
                ("substeps", C.c_int), ("max_steps", C.c_int), ("checkpoint_every", C.c_int),
                ("spill_half", C.c_double), ("spill_temp", C.c_double), ("obs_groups", C.c_int)]


class DmLatticeReset(C.Structure):
    _fields_ = [("origin", C.c_double * 3), ("spacing", C.c_double * 3), ("counts", C.c_int * 3),
                ("origin_draws", C.c_int), ("origin_lo", C.c_double), ("origin_hi", C.c_double),
                ("jitter_lo", C.c_double), ("jitter_hi", C.c_double), ("velocity_sigma", C.c_double),
                ("material", C.c_int), ("group", C.c_int), ("size", C.c_double * 3)]


class DmTaskConfig(C.Structure):
    _fields_ = [("kind", C.c_int), ("grid_n", C.c_int), ("ppc", C.c_int), ("dt", C.c_double), ("substeps", C.c_int),
                ("episode_len", C.c_int), ("cloud_k", C.c_int), ("container_half", C.c_double), ("fill", C.c_double),
                ("speed", C.c_double), ("start_x", C.c_double), ("start_y", C.c_double), ("target_x", C.c_double),
                ("target_y", C.c_double), ("spill_temp", C.c_double), ("block_size", C.c_double),
                ("block_height", C.c_double), ("roller_radius", C.c_double), ("roller_speed", C.c_double),
                ("h_flat", C.c_double), ("youngs", C.c_double), ("yield_stress", C.c_double)]


_LIB = None

_P = C.c_void_p
_SIGS = {
    "dm_create": (_P, [C.POINTER(DmConfig), C.POINTER(DmMaterial), C.c_int, C.POINTER(DmColliderShape)]),
    "dm_destroy": (None, [_P]),
    "dm_last_error": (C.c_int, [_P, C.c_char_p, C.c_int]),
    "dm_stream": (_P, [_P]),
    "dm_device_bytes": (C.c_ulonglong, [_P]),
    "dm_set_state": (C.c_int, [_P] + [_P] * 6),
    "dm_set_state_device": (C.c_int, [_P] + [_P] * 6),
    "dm_get_state": (C.c_int, [_P] + [_P] * 4),
    "dm_get_state_device": (C.c_int, [_P] + [_P] * 4),
    "dm_step": (C.c_int, [_P] * 4),
    "dm_step_device": (C.c_int, [_P] * 4),
    "dm_backward": (C.c_int, [_P] * 13),
    "dm_backward_device": (C.c_int, [_P] * 13),
    "dm_tape_steps": (C.c_int, [_P]),
    "dm_debug_sort": (C.c_int, [_P, _P, _P]),
    "dm_launch_count": (C.c_ulonglong, [_P]),
    "dm_profile": (C.c_int, [_P, C.c_int, _P, _P]),
    "dm_backward_begin": (C.c_int, [_P] * 5),
    "dm_backward_begin_device": (C.c_int, [_P] * 5),
    "dm_backward_step": (C.c_int, [_P] * 4),
    "dm_backward_step_device": (C.c_int, [_P] * 4),
    "dm_backward_end": (C.c_int, [_P] * 6),
    "dm_backward_end_device": (C.c_int, [_P] * 6),
    "dm_obs_dim": (C.c_int, [_P]),
    "dm_observe": (C.c_int, [_P] * 3),
    "dm_observe_device": (C.c_int, [_P] * 3),
    "dm_reset_lattice": (C.c_int, [_P, C.POINTER(DmLatticeReset), C.c_ulonglong, C.c_int, _P, _P, _P]),
    "dm_reset_lattice_device": (C.c_int, [_P, C.POINTER(DmLatticeReset), C.c_ulonglong, C.c_int, _P, _P, _P]),
    "dm_sync": (C.c_int, [_P]),
    "dm_task_default_config": (None, [C.c_int, C.POINTER(DmTaskConfig)]),
    "dm_task_create": (_P, [C.POINTER(DmTaskConfig), C.c_int, C.c_int, C.c_int, C.c_int]),
    "dm_task_destroy": (None, [_P]),
    "dm_task_last_error": (C.c_int, [_P, C.c_char_p, C.c_int]),
    "dm_task_dims": (C.c_int, [_P, _P, _P, _P, _P]),
    "dm_task_reset": (C.c_int, [_P, C.c_ulonglong]),
    "dm_task_observe": (C.c_int, [_P, _P]),
    "dm_task_step": (C.c_int, [_P, _P, _P, _P, C.c_int]),
    "dm_task_backward": (C.c_int, [_P, _P, _P, _P]),
    "dm_task_tape_steps": (C.c_int, [_P]),
    "dm_task_context": (_P, [_P]),
    "dm_debug_inject": (C.c_int, [_P, C.c_int, C.c_int, C.c_int]),
}

PROF_CLASSES = ("bin", "p2g", "g2p", "g2p_adj", "p2g_adj", "env_reduce", "obs", "obs_adj", "layout", "grid",
                "grid_adj")


def lib():
    """Load the in-tree sm_100a library (building it if sources changed)."""
    global _LIB
    if _LIB is None:
        so = os.environ.get("DIFFMPM_SO") or _build.SO  # DIFFMPM_SO: A/B variants of the same ABI
        if so == _build.SO and (not os.path.exists(so) or _build.needs_build()):
            _build.build()
        L = C.CDLL(so)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):  # torch tensor
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)


def _is_dev(a):
    return a is not None and hasattr(a, "is_cuda") and a.is_cuda


def _f32(a, shape=None):
    if a is None or hasattr(a, "data_ptr"):
        return a
    out = np.ascontiguousarray(a, dtype=np.float32)
    return out.reshape(shape) if shape is not None else out


def _i32(a):
    if a is None or hasattr(a, "data_ptr"):
        return a
    return np.ascontiguousarray(a, dtype=np.int32)


class MpmBatch:
    """Batched differentiable MLS-MPM over ``num_envs`` independent envs."""

    def __init__(self, sim: dict, materials: list, colliders: list, num_envs: int, particles_per_env: int,
                 substeps: int, max_steps: int, num_groups: int = 0, checkpoint_every: int = 0,
                 spill_half: float = 0.0, spill_temp: float = 0.0, device: int = 0, obs_groups: int = 0):
        L = lib()
        cfg = DmConfig()
        cfg.device = device
        cfg.num_envs = num_envs
        cfg.particles_per_env = particles_per_env
        cfg.dims[:] = list(sim["dims"])
        cfg.dx = sim["dx"]
        cfg.dt = sim["dt"]
        cfg.gravity[:] = list(sim.get("gravity", (0.0, 0.0, -9.8)))
        cfg.boundary = {"slip": 0, "sticky": 1}[sim.get("boundary", "slip")]
        cfg.alpha_c = sim.get("alpha_c", 100.0)
        cfg.mu_b = sim.get("mu_b", 0.0)
        cfg.num_colliders = len(colliders)
        cfg.num_groups = num_groups
        cfg.substeps = substeps
        cfg.max_steps = max_steps
        cfg.checkpoint_every = checkpoint_every
        cfg.spill_half = spill_half
        cfg.spill_temp = spill_temp
        cfg.obs_groups = obs_groups
        mats = (DmMaterial * len(materials))()
        for i, m in enumerate(materials):
            mats[i].kind = KIND_LAW[m["kind"]]
            mats[i].youngs = m.get("E", 1e4)
            mats[i].poisson = m.get("nu", 0.3)
            mats[i].density = m.get("rho", 1.0)
            mats[i].volume = m["volume"]
            mats[i].yield_stress = m.get("yield_stress", 1e3)
            mats[i].wide_yield = int(m.get("wide_yield", 0))
            mats[i].viscosity = m.get("viscosity", 0.0)
            mats[i].act_strength = m.get("act_strength", 0.0)
            mats[i].bulk = m.get("bulk", 0.0)
        shapes = (DmColliderShape * max(1, len(colliders)))()
        for i, c in enumerate(colliders):
            shapes[i].kind = KIND_COL[c["kind"]]
            shapes[i].normal[:] = list(c.get("normal", (0.0, 0.0, 1.0)))
            shapes[i].radius = c.get("radius", 0.1)
            shapes[i].half[:] = list(c.get("half", (0.1, 0.1, 0.1)))
            shapes[i].length = c.get("length", 0.3)
            shapes[i].thickness = c.get("thickness", 0.02)
        self._L = L
        self.E, self.N, self.K, self.G = num_envs, particles_per_env, len(colliders), num_groups
        self.n_materials = len(materials)
        self.substeps = substeps
        self._h = L.dm_create(C.byref(cfg), mats, len(materials), shapes)
        if not self._h:
            raise MemoryError("dm_create failed")
        msg = C.create_string_buffer(512)
        if L.dm_last_error(self._h, msg, 512) != 0:
            text = msg.value.decode()
            L.dm_destroy(self._h)
            self._h = None
            raise (ValueError if "substeps" in text else RuntimeError)(text)
        self.obs_dim = int(L.dm_obs_dim(self._h))

    # ---- plumbing ----
    def close(self):
        if getattr(self, "_h", None):
            self._L.dm_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def _check(self, rc):
        if rc != 0:
            msg = C.create_string_buffer(1024)
            self._L.dm_last_error(self._h, msg, 1024)
            text = msg.value.decode()
            if rc == 1:
                raise ValueError(text)
            raise RuntimeError(text)

    @property
    def stream_ptr(self) -> int:
        return self._L.dm_stream(self._h) or 0

    @property
    def device_bytes(self) -> int:
        return int(self._L.dm_device_bytes(self._h))

    @property
    def launches(self) -> int:
        return int(self._L.dm_launch_count(self._h))

    @property
    def tape_steps(self) -> int:
        return int(self._L.dm_tape_steps(self._h))

    # ---- API ----
    def set_state(self, x, v, F, C_, material=None, group=None):
        """Upload [E,N,3]/[E,N,9] arrays (visit order) and reset the tape."""
        if _is_dev(x):
            self._check(self._L.dm_set_state_device(self._h, _ptr(x), _ptr(v), _ptr(F), _ptr(C_), _ptr(material),
                                                    _ptr(group)))
            return
        arrs = [_f32(x), _f32(v), _f32(F), _f32(C_), _i32(material), _i32(group)]
        if arrs[4] is not None and (arrs[4].min() < 0 or arrs[4].max() >= self.n_materials):
            raise ValueError("set_state: material id out of range")
        if arrs[5] is not None and self.G > 0 and (arrs[5].min() < 0 or arrs[5].max() >= self.G):
            raise ValueError("set_state: actuation group out of range")
        self._keep = arrs
        self._check(self._L.dm_set_state(self._h, *(_ptr(a) for a in arrs)))

    def reset_lattice(self, spec: dict, seed: int, env_offset: int = 0, env_mask=None, particle_group=None,
                      origin_delta=None):
        """Device-side reset (EnvBatch::reset / reset_env, env.hpp:66-96) of the
        envs whose mask byte is nonzero (all when env_mask is None) from a
        lattice spec (scenes.lattice_reset_spec): no host upload of the state;
        bit-identical to scenes.lattice_reset_host.  Restarts the tape.
        Returns the per-env origin offsets [E,3] (numpy) unless torch
        CUDA `env_mask` / `origin_delta` are given (device path)."""
        r = DmLatticeReset()
        r.origin[:] = list(spec["origin"])
        r.spacing[:] = list(spec["spacing"])
        r.counts[:] = list(spec["counts"])
        r.origin_draws = spec.get("origin_draws", 0)
        r.origin_lo, r.origin_hi = spec.get("origin_range", (0.0, 0.0))
        r.jitter_lo, r.jitter_hi = spec.get("jitter", (0.0, 0.0))
        r.velocity_sigma = spec.get("velocity_sigma", 0.0)
        r.material = spec.get("material", 0)
        r.group = spec.get("group", 0)
        r.size[:] = list(spec.get("size", (0.0, 0.0, 0.0)))
        if _is_dev(env_mask) or _is_dev(origin_delta) or _is_dev(particle_group):
            self._check(self._L.dm_reset_lattice_device(self._h, C.byref(r), seed, env_offset, _ptr(env_mask),
                                                        _ptr(particle_group), _ptr(origin_delta)))
            return origin_delta
        m = None if env_mask is None else np.ascontiguousarray(env_mask, dtype=np.uint8)
        g = None if particle_group is None else np.ascontiguousarray(particle_group, dtype=np.int32)
        d = np.zeros((self.E, 3), np.float64)
        self._check(self._L.dm_reset_lattice(self._h, C.byref(r), seed, env_offset, _ptr(m), _ptr(g), _ptr(d)))
        return d

    def get_state(self, out=None):
        """Current state in the original particle order (numpy, or into torch tensors `out`)."""
        if out is not None:
            self._check(self._L.dm_get_state_device(self._h, *(_ptr(o) for o in out)))
            return out
        n = self.E * self.N
        x = np.empty((self.E, self.N, 3), np.float32)
        v = np.empty((self.E, self.N, 3), np.float32)
        F = np.empty((self.E, self.N, 9), np.float32)
        Cm = np.empty((self.E, self.N, 9), np.float32)
        self._check(self._L.dm_get_state(self._h, _ptr(x), _ptr(v), _ptr(F), _ptr(Cm)))
        assert n == x.shape[0] * x.shape[1]
        return {"x": x, "v": v, "F": F, "C": Cm}

    def step(self, cvo=None, act=None, obs=None):
        """One control step.  cvo [E,K,9], act [E,G]; returns obs [E,7]."""
        if _is_dev(cvo) or _is_dev(act) or _is_dev(obs):
            self._check(self._L.dm_step_device(self._h, _ptr(cvo), _ptr(act), _ptr(obs)))
            return obs
        c = _f32(cvo) if cvo is not None else None
        a = _f32(act) if act is not None else None
        o = np.empty((self.E, self.obs_dim), np.float32) if obs is None else obs
        self._check(self._L.dm_step(self._h, _ptr(c), _ptr(a), _ptr(o)))
        return o

    def backward(self, dobs=None, dfinal=None, want=("x", "v", "F", "C", "cvo", "act", "E"), out=None):
        """Backward through the tape.  dobs [T,E,7]; dfinal dict of final-state
        cotangents.  Returns a dict of cotangents (numpy) or fills torch `out`."""
        T = self.tape_steps
        dfinal = dfinal or {}
        if out is not None and not any(_is_dev(a) for a in out.values()):
            # host path into caller-provided (e.g. pinned) numpy buffers
            d = _f32(dobs) if dobs is not None else None
            fin = [_f32(dfinal.get(k)) for k in ("x", "v", "F", "C")]
            self._check(self._L.dm_backward(self._h, _ptr(d), *(_ptr(a) for a in fin),
                                            *(_ptr(out.get(k)) for k in ("x", "v", "F", "C", "cvo", "act", "E"))))
            return out
        if out is not None:
            args = [out.get(k) for k in ("x", "v", "F", "C", "cvo", "act", "E")]
            self._check(self._L.dm_backward_device(self._h, _ptr(dobs), *(_ptr(dfinal.get(k)) for k in ("x", "v", "F", "C")),
                                                   *(_ptr(a) for a in args)))
            return out
        res = {}
        if "x" in want:
            res["x"] = np.zeros((self.E, self.N, 3), np.float32)
        if "v" in want:
            res["v"] = np.zeros((self.E, self.N, 3), np.float32)
        if "F" in want:
            res["F"] = np.zeros((self.E, self.N, 9), np.float32)
        if "C" in want:
            res["C"] = np.zeros((self.E, self.N, 9), np.float32)
        if "cvo" in want and self.K > 0:
            res["cvo"] = np.zeros((T, self.E, self.K, 9), np.float32)
        if "act" in want and self.G > 0:
            res["act"] = np.zeros((T, self.E, self.G), np.float32)
        if "E" in want:
            res["E"] = np.zeros((self.E, self.n_materials), np.float64)
        d = _f32(dobs) if dobs is not None else None
        fin = [_f32(dfinal.get(k)) for k in ("x", "v", "F", "C")]
        self._check(self._L.dm_backward(self._h, _ptr(d), *(_ptr(a) for a in fin),
                                        *(_ptr(res.get(k)) for k in ("x", "v", "F", "C", "cvo", "act", "E"))))
        return res

    def observe(self, cvo=None, obs=None):
        """Observables of the current state (reset observation) [E, obs_dim]."""
        if _is_dev(obs) or _is_dev(cvo):
            self._check(self._L.dm_observe_device(self._h, _ptr(cvo), _ptr(obs)))
            return obs
        o = np.empty((self.E, self.obs_dim), np.float32) if obs is None else obs
        self._check(self._L.dm_observe(self._h, _ptr(_f32(cvo) if cvo is not None else None), _ptr(o)))
        return o

    # ---- incremental backward (policy in the loop) ----
    def backward_begin(self, dfinal=None):
        dfinal = dfinal or {}
        vals = [dfinal.get(k) for k in ("x", "v", "F", "C")]
        if any(_is_dev(a) for a in vals):
            self._check(self._L.dm_backward_begin_device(self._h, *(_ptr(a) for a in vals)))
        else:
            vals = [_f32(a) for a in vals]
            self._check(self._L.dm_backward_begin(self._h, *(_ptr(a) for a in vals)))

    def backward_step(self, dobs_t=None, out_cvo=None, out_act=None):
        """Processes the latest unprocessed control step.  dobs_t [E, obs_dim]
        (torch CUDA tensors use the device path).  Returns (dcvo_t, dact_t)."""
        if _is_dev(dobs_t) or _is_dev(out_act) or _is_dev(out_cvo):
            self._check(self._L.dm_backward_step_device(self._h, _ptr(dobs_t), _ptr(out_cvo), _ptr(out_act)))
            return out_cvo, out_act
        d = _f32(dobs_t) if dobs_t is not None else None
        c = np.zeros((self.E, self.K, 9), np.float32) if self.K else None
        a = np.zeros((self.E, self.G), np.float32) if self.G else None
        self._check(self._L.dm_backward_step(self._h, _ptr(d), _ptr(c), _ptr(a)))
        return c, a

    def backward_end(self, out=None):
        if out is not None:
            self._check(self._L.dm_backward_end_device(self._h, *(_ptr(out.get(k)) for k in ("x", "v", "F", "C", "E"))))
            return out
        res = {"x": np.zeros((self.E, self.N, 3), np.float32), "v": np.zeros((self.E, self.N, 3), np.float32),
               "F": np.zeros((self.E, self.N, 9), np.float32), "C": np.zeros((self.E, self.N, 9), np.float32),
               "E": np.zeros((self.E, self.n_materials), np.float64)}
        self._check(self._L.dm_backward_end(self._h, *(_ptr(res[k]) for k in ("x", "v", "F", "C", "E"))))
        return res

    def sync(self):
        """Synchronise the context stream and raise what the device recorded
        since the last synchronising call (dm_sync): the *_device entry points
        report device-detected errors and CFL warnings lazily."""
        self._check(self._L.dm_sync(self._h))

    def debug_inject(self, step: int, env: int = 0, particle: int = 0):
        """Test hook (dm_debug_inject): make the backward's replay of control
        step `step` non-deterministic (one ulp of one particle's x)."""
        self._check(self._L.dm_debug_inject(self._h, step, env, particle))

    def torch_stream(self):
        """The context stream as a torch stream: run torch work that produces
        or consumes *_device buffers under ``with torch.cuda.stream(...)`` so
        it is ordered with the simulator's kernels (no host synchronisation)."""
        import torch
        if getattr(self, "_tstream", None) is None:
            self._tstream = torch.cuda.ExternalStream(self.stream_ptr)
        return self._tstream

    def profile(self, enable: bool = True):
        """Returns {class: (ms, launches)} accumulated since the last call and
        switches per-kernel CUDA-event timing on/off."""
        ms = np.zeros(len(PROF_CLASSES), np.float64)
        n = np.zeros(len(PROF_CLASSES), np.int64)
        self._check(self._L.dm_profile(self._h, int(enable), _ptr(ms), _ptr(n)))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(PROF_CLASSES)}

    def debug_sort(self):
        """(keys, perm) of the current state per env: bin key per particle (in
        physical order) and the stable sort permutation (local indices)."""
        n = self.E * self.N
        keys = np.empty(n, np.int32)
        perm = np.empty(n, np.int32)
        self._check(self._L.dm_debug_sort(self._h, _ptr(keys), _ptr(perm)))
        return keys.reshape(self.E, self.N), perm.reshape(self.E, self.N)


def from_scene(scene, max_steps=None, checkpoint_every=None, device=0) -> MpmBatch:
    """Context sized for a scenes.Scene."""
    ls = scene.loss
    return MpmBatch(scene.sim, scene.materials, scene.colliders, scene.n_envs, scene.n_per_env, scene.n_sub,
                    max_steps or scene.n_ctrl, num_groups=getattr(scene.task, "n_act", 0),
                    checkpoint_every=scene.checkpoint_every if checkpoint_every is None else checkpoint_every,
                    spill_half=ls.get("spill_half", 0.0), spill_temp=ls.get("spill_temp", 0.0), device=device,
                    obs_groups=scene.extra.get("obs_groups", 0))


def run_scene(sim_batch: MpmBatch, scene, want_grad=True):
    """Forward (+ backward) of a scene's full rollout.  Returns loss, obs and
    cotangents (host numpy)."""
    from .losses import loss_and_dobs
    cvo, act = scene.cvo_act()
    sim_batch.set_state(scene.x, scene.v, scene.F, scene.C, scene.material, scene.group)
    obs = np.zeros((scene.n_ctrl, scene.n_envs, sim_batch.obs_dim), np.float32)
    for t in range(scene.n_ctrl):
        obs[t] = sim_batch.step(cvo[:, t] if scene.colliders else None,
                                act[:, t] if getattr(scene.task, "n_act", 0) else None)
    loss, dobs = loss_and_dobs(scene.loss, np.transpose(obs[:, :, :OBS_DIM], (1, 0, 2)))
    if sim_batch.obs_dim > OBS_DIM:
        dobs = np.concatenate([dobs, np.zeros(dobs.shape[:2] + (sim_batch.obs_dim - OBS_DIM,))], axis=-1)
    out = {"loss": loss, "obs": obs}
    if want_grad:
        g = sim_batch.backward(dobs=np.ascontiguousarray(np.transpose(dobs, (1, 0, 2)), dtype=np.float32))
        out.update(g)
    return out


TASKS = {"fluid_move": 0, "roll_flat": 1}


def task_config(kind: str, **over) -> dict:
    """The reference task's Config{} defaults (tasks.hpp:241-254, 511-525),
    with overrides."""
    L = lib()
    c = DmTaskConfig()
    L.dm_task_default_config(TASKS[kind], C.byref(c))
    d = {f: getattr(c, f) for f, _ in DmTaskConfig._fields_}
    for k, v in over.items():
        if k not in d:
            raise KeyError(k)
        d[k] = v
    return d


class TaskBatch:
    """EnvBatch<Task> (env.hpp:55-117) for MiniFluidMove / MiniRollFlat
    (tasks.hpp) on the GPU simulator (dm_task_* ABI): reset / observe /
    step(actions) -> rewards, dones with auto-reset / backward(drewards,
    dobs) -> dL/dactions.  Double precision arrays, as the reference."""

    def __init__(self, cfg: dict, num_envs: int, seed: int = 0, horizon: int = 64, device: int = 0,
                 env_offset: int = 0):
        L = lib()
        c = DmTaskConfig()
        for f, _ in DmTaskConfig._fields_:
            setattr(c, f, cfg[f] if f != "kind" or not isinstance(cfg[f], str) else TASKS[cfg[f]])
        self._L = L
        self._h = L.dm_task_create(C.byref(c), num_envs, env_offset, horizon, device)
        if not self._h:
            raise MemoryError("dm_task_create failed")
        msg = C.create_string_buffer(1024)
        if L.dm_task_last_error(self._h, msg, 1024) != 0:
            text = msg.value.decode()
            L.dm_task_destroy(self._h)
            self._h = None
            raise ValueError(text)
        dims = [C.c_int(0) for _ in range(4)]
        L.dm_task_dims(self._h, *(C.byref(d) for d in dims))
        self.E = num_envs
        self.obs_dim, self.act_dim, self.particles_per_env, self.episode_len = (int(d.value) for d in dims)
        self.reset(seed)

    def close(self):
        if getattr(self, "_h", None):
            self._L.dm_task_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def _check(self, rc):
        if rc != 0:
            msg = C.create_string_buffer(1024)
            self._L.dm_task_last_error(self._h, msg, 1024)
            raise (ValueError if rc == 1 else RuntimeError)(msg.value.decode())

    def reset(self, seed: int):
        self._check(self._L.dm_task_reset(self._h, seed))

    def observe(self):
        o = np.zeros((self.E, self.obs_dim))
        self._check(self._L.dm_task_observe(self._h, _ptr(o)))
        return o

    def step(self, actions, record: bool = True):
        a = np.ascontiguousarray(actions, dtype=np.float64).reshape(self.E, self.act_dim)
        r = np.zeros(self.E)
        d = np.zeros(self.E, np.uint8)
        self._check(self._L.dm_task_step(self._h, _ptr(a), _ptr(r), _ptr(d), int(record)))
        return r, d.astype(bool)

    @property
    def tape_steps(self) -> int:
        return int(self._L.dm_task_tape_steps(self._h))

    def backward(self, drewards=None, dobs=None):
        T = self.tape_steps
        dr = None if drewards is None else np.ascontiguousarray(drewards, dtype=np.float64).reshape(T, self.E)
        do = None if dobs is None else np.ascontiguousarray(dobs, dtype=np.float64).reshape(T + 1, self.E,
                                                                                             self.obs_dim)
        da = np.zeros((T, self.E, self.act_dim))
        self._check(self._L.dm_task_backward(self._h, _ptr(dr), _ptr(do), _ptr(da)))
        return da
