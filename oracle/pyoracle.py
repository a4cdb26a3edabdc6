"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the CPU oracle.

* ``build/liboracle.so`` -- fp64 restatement of the reference MLS-MPM path
  (oracle/include/oracle/mpm.hpp), standalone.
* ``_ref/libref.so``     -- the reference headers (/root/reference/proj/include)
  compiled unchanged with the Eigen-free SVD shim, exposing the reference's
  own ``mpm_step<double>``/``mpm_step<Value>`` and the restatement on the
  reference tape (gradient oracle).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_ORACLE = os.path.join(HERE, "build", "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libref.so")

LAW = {"fixed_corotated": 0, "neo_hookean": 1, "elastoplastic": 2, "fluid": 3}
COLLIDER = {"plane": 0, "sphere": 1, "box": 2, "cylinder": 3, "hollow_box": 4}


class OrSim(C.Structure):
    _fields_ = [("dims", C.c_int * 3), ("dx", C.c_double), ("dt", C.c_double),
                ("gravity", C.c_double * 3), ("boundary", C.c_int),
                ("alpha_c", C.c_double), ("mu_b", C.c_double)]


class OrMat(C.Structure):
    _fields_ = [("kind", C.c_int), ("youngs", C.c_double), ("poisson", C.c_double),
                ("density", C.c_double), ("volume", C.c_double), ("yield_stress", C.c_double),
                ("wide_yield", C.c_int), ("viscosity", C.c_double), ("act_strength", C.c_double),
                ("bulk", C.c_double)]


class OrCol(C.Structure):
    _fields_ = [("kind", C.c_int), ("center", C.c_double * 3), ("velocity", C.c_double * 3),
                ("omega", C.c_double * 3), ("normal", C.c_double * 3), ("radius", C.c_double),
                ("half", C.c_double * 3), ("length", C.c_double), ("thickness", C.c_double)]


class OrLoss(C.Structure):
    _fields_ = [("kind", C.c_int), ("target", C.c_double * 3), ("spill_half", C.c_double),
                ("spill_temp", C.c_double), ("tier_threshold", C.c_double),
                ("tier_low", C.c_double), ("tier_high", C.c_double)]


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int)) if a is not None else None


def _fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


_libs: dict = {}


def lib(name: str = "oracle"):
    path = LIB_ORACLE if name == "oracle" else LIB_REF
    if name not in _libs:
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle all ref`)")
        _libs[name] = C.CDLL(path)
    return _libs[name]


def have_ref() -> bool:
    return os.path.exists(LIB_REF)


# ---- descriptor builders (plain dict specs -> ctypes) ----

def make_sim(spec) -> OrSim:
    s = OrSim()
    s.dims[:] = list(spec["dims"])
    s.dx = spec["dx"]
    s.dt = spec.get("dt", 1e-4)
    s.gravity[:] = list(spec.get("gravity", (0.0, 0.0, -9.8)))
    s.boundary = {"slip": 0, "sticky": 1}[spec.get("boundary", "slip")]
    s.alpha_c = spec.get("alpha_c", 100.0)
    s.mu_b = spec.get("mu_b", 0.0)
    return s


def make_mats(specs):
    arr = (OrMat * max(1, len(specs)))()
    for i, m in enumerate(specs):
        arr[i].kind = LAW[m["kind"]]
        arr[i].youngs = m.get("E", 1e4)
        arr[i].poisson = m.get("nu", 0.3)
        arr[i].density = m.get("rho", 1.0)
        arr[i].volume = m["volume"]
        arr[i].yield_stress = m.get("yield_stress", 1e3)
        arr[i].wide_yield = int(m.get("wide_yield", 0))
        arr[i].viscosity = m.get("viscosity", 0.0)
        arr[i].act_strength = m.get("act_strength", 0.0)
        arr[i].bulk = m.get("bulk", 0.0)
    return arr


def make_cols(specs):
    arr = (OrCol * max(1, len(specs)))()
    for i, c in enumerate(specs):
        arr[i].kind = COLLIDER[c["kind"]]
        arr[i].center[:] = list(c.get("center", (0.0, 0.0, 0.0)))
        arr[i].velocity[:] = list(c.get("velocity", (0.0, 0.0, 0.0)))
        arr[i].omega[:] = list(c.get("omega", (0.0, 0.0, 0.0)))
        arr[i].normal[:] = list(c.get("normal", (0.0, 0.0, 1.0)))
        arr[i].radius = c.get("radius", 0.1)
        arr[i].half[:] = list(c.get("half", (0.1, 0.1, 0.1)))
        arr[i].length = c.get("length", 0.3)
        arr[i].thickness = c.get("thickness", 0.02)
    return arr


def make_loss(spec) -> OrLoss:
    l = OrLoss()
    l.kind = {"com_target": 0, "neg_mean_z": 1, "var_z": 2, "fluid_move": 3}[spec["kind"]]
    l.target[:] = list(spec.get("target", (0.5, 0.4, 0.5)))
    l.spill_half = spec.get("spill_half", 0.0)
    l.spill_temp = spec.get("spill_temp", 0.0)
    l.tier_threshold = spec.get("tier_threshold", 0.02)
    l.tier_low = spec.get("tier_low", 1.0)
    l.tier_high = spec.get("tier_high", 2.0)
    return l


def cvo_from_cols(col_specs, n_ctrl):
    """[n_ctrl][ncol][9] center/velocity/omega per control step."""
    out = np.zeros((n_ctrl, max(1, len(col_specs)), 9))
    for t in range(n_ctrl):
        for c, cs in enumerate(col_specs):
            cvo = cs.get("cvo")
            if cvo is not None:
                out[t, c] = np.asarray(cvo)[t]
            else:
                out[t, c, 0:3] = cs.get("center", (0, 0, 0))
                out[t, c, 3:6] = cs.get("velocity", (0, 0, 0))
                out[t, c, 6:9] = cs.get("omega", (0, 0, 0))
    return np.ascontiguousarray(out)


class OracleError(RuntimeError):
    pass


def _state_arrays(state):
    x = np.ascontiguousarray(state["x"], dtype=np.float64).reshape(-1, 3).copy()
    n = x.shape[0]
    v = np.ascontiguousarray(state["v"], dtype=np.float64).reshape(n, 3).copy()
    F = np.ascontiguousarray(state["F"], dtype=np.float64).reshape(n, 9).copy()
    Cm = np.ascontiguousarray(state["C"], dtype=np.float64).reshape(n, 9).copy()
    mat = np.ascontiguousarray(state.get("material", np.zeros(n)), dtype=np.int32)
    grp = np.ascontiguousarray(state.get("group", np.zeros(n)), dtype=np.int32)
    return n, x, v, F, Cm, mat, grp


def rollout(sim, mats, cols, state, n_ctrl, n_sub, act=None, loss=None):
    """fp64 restatement forward.  Returns (state, obs[n_ctrl,7], loss)."""
    L = lib("oracle")
    n, x, v, F, Cm, mat, grp = _state_arrays(state)
    cvo = cvo_from_cols(cols, n_ctrl)
    nact = 0 if act is None else np.asarray(act).shape[-1]
    a = np.ascontiguousarray(np.zeros((n_ctrl, 1)) if act is None else np.asarray(act, dtype=np.float64).reshape(n_ctrl, nact))
    obs = np.zeros((n_ctrl, 7))
    lo = C.c_double(0.0)
    err = C.create_string_buffer(512)
    ls = make_loss(loss) if loss else None
    rc = L.or_rollout(C.byref(make_sim(sim)), make_mats(mats), len(mats), make_cols(cols), len(cols),
                      _dp(cvo), _dp(a), nact, n, _dp(x), _dp(v), _dp(F), _dp(Cm), _ip(mat), _ip(grp),
                      n_ctrl, n_sub, C.byref(ls) if ls else None, _dp(obs), C.byref(lo), err, 512)
    if rc != 0:
        raise OracleError(err.value.decode())
    return {"x": x, "v": v, "F": F, "C": Cm, "material": mat, "group": grp}, obs, lo.value


def p2g_grid(sim, mats, cols, state, act=None):
    L = lib("oracle")
    n, x, v, F, Cm, mat, grp = _state_arrays(state)
    nn = int(np.prod(sim["dims"]))
    mass = np.zeros(nn)
    mom = np.zeros((nn, 3))
    vel = np.zeros((nn, 3))
    cvo = cvo_from_cols(cols, 1)
    a = np.ascontiguousarray(np.zeros(8) if act is None else np.asarray(act, dtype=np.float64))
    err = C.create_string_buffer(512)
    rc = L.or_p2g_grid(C.byref(make_sim(sim)), make_mats(mats), len(mats), make_cols(cols), len(cols), _dp(cvo),
                       _dp(a), n, _dp(x), _dp(v), _dp(F), _dp(Cm), _ip(mat), _ip(grp), _dp(mass), _dp(mom), _dp(vel),
                       err, 512)
    if rc != 0:
        raise OracleError(err.value.decode())
    return mass, mom, vel


def stress(mat, F, act=0.0):
    L = lib("oracle")
    F = np.ascontiguousarray(F, dtype=np.float64).reshape(-1, 9)
    P = np.zeros_like(F)
    Fp = np.zeros_like(F)
    err = C.create_string_buffer(512)
    m = make_mats([mat])
    rc = L.or_stress(m, F.shape[0], _dp(F), C.c_double(act), _dp(P), _dp(Fp), err, 512)
    if rc != 0:
        raise OracleError(err.value.decode())
    return P, Fp


def collider_query(col, pts):
    L = lib("oracle")
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    d = np.zeros(pts.shape[0])
    nrm = np.zeros_like(pts)
    L.or_collider_query(make_cols([col]), pts.shape[0], _dp(pts), _dp(d), _dp(nrm))
    return d, nrm


def svd3(f):
    L = lib("oracle")
    f = np.ascontiguousarray(f, dtype=np.float64).reshape(9)
    u = np.zeros(9)
    s = np.zeros(3)
    vt = np.zeros(9)
    L.or_svd3(_dp(f), _dp(u), _dp(s), _dp(vt))
    return u.reshape(3, 3), s, vt.reshape(3, 3)


def bin_keys(sim, x32):
    L = lib("oracle")
    x32 = np.ascontiguousarray(x32, dtype=np.float32).reshape(-1, 3)
    keys = np.zeros(x32.shape[0], dtype=np.int32)
    L.or_bin_keys(C.byref(make_sim(sim)), _fp(x32), x32.shape[0], _ip(keys))
    return keys


def stable_sort(keys):
    L = lib("oracle")
    keys = np.ascontiguousarray(keys, dtype=np.int32)
    perm = np.zeros(keys.shape[0], dtype=np.int32)
    L.or_stable_sort(_ip(keys), keys.shape[0], _ip(perm))
    return perm


# ---- reference (oracle/_ref) ----

def ref_rollout(sim, mats, cols, state, n_sub):
    """The reference's own mpm_step<double> (elastoplastic/fluid; plane/sphere/box; slip)."""
    L = lib("ref")
    n, x, v, F, Cm, mat, grp = _state_arrays(state)
    secs = C.c_double(0.0)
    err = C.create_string_buffer(512)
    rc = L.ref_mpm_rollout(C.byref(make_sim(sim)), make_mats(mats), len(mats), make_cols(cols), len(cols), n,
                           _dp(x), _dp(v), _dp(F), _dp(Cm), _ip(mat), n_sub, C.byref(secs), err, 512)
    if rc != 0:
        raise OracleError(err.value.decode())
    return {"x": x, "v": v, "F": F, "C": Cm, "material": mat}, secs.value


def ref_grad(sim, mats, cols, state, n_sub, target, seg=0):
    """Reference tape gradient of |com(x_final) - target|^2 w.r.t. the initial state."""
    L = lib("ref")
    n, x, v, F, Cm, mat, grp = _state_arrays(state)
    g = [np.zeros((n, 3)), np.zeros((n, 3)), np.zeros((n, 9)), np.zeros((n, 9))]
    tgt = np.ascontiguousarray(target, dtype=np.float64)
    lo = C.c_double(0.0)
    secs = C.c_double(0.0)
    err = C.create_string_buffer(512)
    rc = L.ref_mpm_grad(C.byref(make_sim(sim)), make_mats(mats), len(mats), make_cols(cols), len(cols), n,
                        _dp(x), _dp(v), _dp(F), _dp(Cm), _ip(mat), n_sub, seg, _dp(tgt), C.byref(lo),
                        _dp(g[0]), _dp(g[1]), _dp(g[2]), _dp(g[3]), C.byref(secs), err, 512)
    if rc != 0:
        raise OracleError(err.value.decode())
    return lo.value, {"x": g[0], "v": g[1], "F": g[2], "C": g[3]}, secs.value


def set_svd_adjoint(mode: int) -> int:
    """SVD-law adjoint of the gradient oracle: 1 (default) records the
    fixed-corotated / Hencky maps as isotropic-map nodes with their exact
    derivative; 0 uses the reference's Tape::svd3x3 (svd3.hpp:27-63, clamped
    at repeated singular values).  Returns the previous mode."""
    L = lib("ref")
    L.ref_set_svd_adjoint.restype = C.c_int
    return int(L.ref_set_svd_adjoint(int(mode)))


def rollout_grad(sim, mats, cols, state, n_ctrl, n_sub, loss, act=None, seg=1):
    """Restatement on the reference tape: loss, obs and gradients w.r.t. the
    initial state, per-step collider (center, velocity, omega), per-step
    actuation and each material's E."""
    L = lib("ref")
    n, x, v, F, Cm, mat, grp = _state_arrays(state)
    cvo = cvo_from_cols(cols, n_ctrl)
    nact = 0 if act is None else np.asarray(act).shape[-1]
    a = np.ascontiguousarray(np.zeros((n_ctrl, 1)) if act is None else np.asarray(act, dtype=np.float64).reshape(n_ctrl, nact))
    g = [np.zeros((n, 3)), np.zeros((n, 3)), np.zeros((n, 9)), np.zeros((n, 9))]
    gcvo = np.zeros_like(cvo)
    gact = np.zeros_like(a)
    gE = np.zeros(max(1, len(mats)))
    obs = np.zeros((n_ctrl, 7))
    lo = C.c_double(0.0)
    secs = C.c_double(0.0)
    err = C.create_string_buffer(512)
    rc = L.ref_rollout_grad(C.byref(make_sim(sim)), make_mats(mats), len(mats), make_cols(cols), len(cols),
                            _dp(cvo), _dp(a), nact, n, _dp(x), _dp(v), _dp(F), _dp(Cm), _ip(mat), _ip(grp), n_ctrl,
                            n_sub, C.byref(make_loss(loss)), seg, C.byref(lo), _dp(obs), _dp(g[0]), _dp(g[1]),
                            _dp(g[2]), _dp(g[3]), _dp(gcvo), _dp(gact), _dp(gE), C.byref(secs), err, 512)
    if rc != 0:
        raise OracleError(err.value.decode())
    return {"loss": lo.value, "obs": obs, "x": g[0], "v": g[1], "F": g[2], "C": g[3], "cvo": gcvo[:, :len(cols)],
            "act": gact[:, :nact], "E": gE[:len(mats)], "seconds": secs.value}


# ---- reference tasks (tasks.hpp) ----

TASK_CFG_FIELDS = ("grid_n", "ppc", "dt", "substeps", "episode_len", "cloud_k", "container_half", "fill", "speed",
                   "start_x", "start_y", "target_x", "target_y", "spill_temp", "block_size", "block_height",
                   "roller_radius", "roller_speed", "h_flat", "youngs", "yield_stress")


def ref_task_dims(kind: int, cfg: dict):
    L = lib("ref")
    c = np.ascontiguousarray([float(cfg[k]) for k in TASK_CFG_FIELDS])
    dims = np.zeros(2, np.int32)
    err = C.create_string_buffer(512)
    rc = L.ref_task_rollout(C.c_int(kind), _dp(c), 1, C.c_ulonglong(0), 0, 0, None, None, None, None, None, None,
                            _ip(dims), err, 512)
    if rc != 0:
        raise OracleError(err.value.decode())
    return int(dims[0]), int(dims[1])


def ref_task_rollout(kind: int, cfg: dict, n_envs: int, seed: int, env_offset: int, actions, w_r=None, w_o=None):
    """The reference's MiniFluidMove (kind 0) / MiniRollFlat (1) stepped as
    EnvBatch does with the given actions [T, E, A]: rewards [T, E], obs
    [T+1, E, od]; with weights, dL/dactions of L = sum w_r r + sum w_o obs on
    the reference tape."""
    L = lib("ref")
    od, A = ref_task_dims(kind, cfg)
    a = np.ascontiguousarray(actions, dtype=np.float64)
    T = a.shape[0]
    assert a.shape == (T, n_envs, A)
    c = np.ascontiguousarray([float(cfg[k]) for k in TASK_CFG_FIELDS])
    rew = np.zeros((T, n_envs))
    obs = np.zeros((T + 1, n_envs, od))
    wr = None if w_r is None else np.ascontiguousarray(w_r, dtype=np.float64)
    wo = None if w_o is None else np.ascontiguousarray(w_o, dtype=np.float64)
    da = np.zeros_like(a)
    err = C.create_string_buffer(512)
    rc = L.ref_task_rollout(C.c_int(kind), _dp(c), n_envs, C.c_ulonglong(seed), env_offset, T, _dp(a), _dp(rew),
                            _dp(obs), _dp(wr), _dp(wo), _dp(da), None, err, 512)
    if rc != 0:
        raise OracleError(err.value.decode())
    return rew, obs, (da if wr is not None else None)


def ref_sample(kind: str, a, b, dx: float, ppc: int, cap: int = 1 << 20):
    """The reference's sample_box (kind "box": a = org, b = size) /
    sample_cylinder ("cylinder": a = base center, b = (radius, height))."""
    L = lib("ref")
    L.ref_sample.restype = C.c_int
    aa = np.ascontiguousarray(a, dtype=np.float64)
    bb = np.ascontiguousarray(list(b) + [0.0] * (3 - len(b)), dtype=np.float64)
    x = np.zeros((cap, 3))
    vol = C.c_double(0.0)
    n = L.ref_sample(0 if kind == "box" else 1, _dp(aa), _dp(bb), C.c_double(dx), ppc, _dp(x), cap, C.byref(vol))
    if n < 0:
        raise OracleError("ref_sample: capacity")
    return x[:n].copy(), vol.value
