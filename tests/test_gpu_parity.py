"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Gates:
  * bin keys and stable sort permutation bit-exact on identical fp32 positions
  * one substep from the oracle's (fp32-rounded) state: field rel <= 1e-5
  * free-running rollout end: field rel <= 1e-3
  * gradients vs the reference-tape oracle: cosine >= 0.999, rel L2 <= 1e-3
  * checkpointed backward == store-every-substep backward, bitwise
    (acceptance.cpp:198-209); replays deterministic run to run
"""
import zlib

import numpy as np
import pytest

import pyoracle as O
from helpers import cosine, field_rel, random_block, rel_l2, to_f32_state
from paper_2412_12089_b200 import api, scenes
from paper_2412_12089_b200.losses import loss_and_dobs

pytestmark = pytest.mark.gpu

SIM16 = {"dims": (16, 16, 16), "dx": 1 / 16, "dt": 1e-4, "gravity": (0, 0, -9.8), "boundary": "slip"}

LAWS = {
    "fixed_corotated": {"kind": "fixed_corotated", "E": 1e4, "nu": 0.3, "rho": 1, "volume": 1e-4},
    "neo_hookean": {"kind": "neo_hookean", "E": 3e4, "nu": 0.3, "rho": 1, "volume": 1e-4, "act_strength": 1e4},
    "elastoplastic": {"kind": "elastoplastic", "E": 5e3, "nu": 0.2, "rho": 1, "volume": 1e-4, "yield_stress": 20},
    "fluid": {"kind": "fluid", "E": 2e4, "nu": 0.3, "rho": 1000, "volume": 1e-4, "bulk": 2e4, "viscosity": 0.5},
}

COLS = {
    "none": [],
    "plane": [{"kind": "plane", "center": (0, 0, 0.42), "normal": (0, 0, 1), "velocity": (0, 0, 0.1)}],
    "sphere": [{"kind": "sphere", "center": (0.5, 0.5, 0.66), "radius": 0.08, "velocity": (0.1, 0, -0.3)}],
    "box": [{"kind": "box", "center": (0.3513, 0.5021, 0.4987), "half": (0.0511, 0.1013, 0.0493),
             "velocity": (0.3, 0, 0)}],
    # off-lattice geometry: no grid node sits on an SDF branch tie (the
    # inside-normal switch is discontinuous by design, mpm.hpp:114-122)
    "cylinder": [{"kind": "cylinder", "normal": (0, 1, 0), "radius": 0.0513, "length": 0.3107,
                  "center": (0.5031, 0.4987, 0.6029), "velocity": (0.1, 0, -0.3), "omega": (0, 5, 0)}],
    "hollow_box": [{"kind": "hollow_box", "half": (0.1013, 0.0987, 0.1021), "thickness": 0.0911,
                    "center": (0.5017, 0.4983, 0.4529), "velocity": (0.2, -0.1, 0.05)}],
}


def gpu_batch(sim, mats, cols, states, n_ctrl, n_sub, groups=0, ck=0, loss=None):
    E = len(states)
    N = states[0]["x"].shape[0]
    ls = loss or {}
    return api.MpmBatch(sim, mats, cols, E, N, n_sub, n_ctrl, num_groups=groups, checkpoint_every=ck,
                        spill_half=ls.get("spill_half", 0.0), spill_temp=ls.get("spill_temp", 0.0))


def stack(states, k):
    return np.stack([np.asarray(s[k]) for s in states])


def cvo_for(cols, n_ctrl, E=1):
    c = O.cvo_from_cols(cols, n_ctrl)[:, :len(cols)]  # [T, K, 9]
    return np.broadcast_to(c[:, None], (n_ctrl, E, len(cols), 9)).astype(np.float32) if cols else None


def gpu_rollout(sim, mats, cols, states, n_ctrl, n_sub, act=None, loss=None, grad=False, ck=0):
    E = len(states)
    G = 0 if act is None else act.shape[-1]
    b = gpu_batch(sim, mats, cols, states, n_ctrl, n_sub, groups=G, ck=ck, loss=loss)
    b.set_state(stack(states, "x"), stack(states, "v"), stack(states, "F"), stack(states, "C"),
                stack(states, "material"), stack(states, "group"))
    cvo = cvo_for(cols, n_ctrl, E)
    obs = np.zeros((n_ctrl, E, 7), np.float32)
    for t in range(n_ctrl):
        a = None if act is None else np.broadcast_to(np.asarray(act, np.float32)[t], (E, G))
        obs[t] = b.step(None if cvo is None else np.ascontiguousarray(cvo[t]), a)
    out = {"state": b.get_state(), "obs": obs, "batch": b}
    if grad:
        L, dobs = loss_and_dobs(loss, np.transpose(obs, (1, 0, 2)))
        out["loss"] = L
        out["grad"] = b.backward(dobs=np.ascontiguousarray(np.transpose(dobs, (1, 0, 2)), dtype=np.float32))
    return out


# ---------------- binning / sort ----------------

@pytest.mark.parametrize("seed,n,E,lo,hi", [(0, 3000, 3, 0.08, 0.92), (1, 3000, 3, 0.08, 0.92),
                                            (2, 4096, 1, 0.3, 0.5), (3, 20000, 2, 0.2, 0.5), (4, 700, 5, 0.1, 0.9)])
def test_sort_bit_exact(seed, n, E, lo, hi):
    """Several batch shapes (particles per warp from ~2 to ~600 chunks of the
    bin kernel's per-warp histograms): the permutation equals
    std::stable_sort by key."""
    rng = np.random.default_rng(seed)
    sim = dict(SIM16, dims=(48, 48, 48), dx=1 / 48)
    states = [random_block(rng, n, lo, hi) for _ in range(E)]
    b = gpu_batch(sim, [LAWS["fluid"]], [], states, 1, 1)
    b.set_state(stack(states, "x"), stack(states, "v"), stack(states, "F"), stack(states, "C"))
    keys, perm = b.debug_sort()
    for e, st in enumerate(states):
        k_ref = O.bin_keys(sim, st["x"].astype(np.float32))
        assert np.array_equal(keys[e], k_ref)
        assert np.array_equal(perm[e], O.stable_sort(k_ref))


def test_sort_bit_exact_wide_histograms():
    """More than 65535 particles per env: the bin kernel switches from 16-bit
    to 32-bit per-warp histograms / cursors; clustered positions put many
    particles in one tile (long runs, full cursors)."""
    rng = np.random.default_rng(11)
    sim = dict(SIM16, dims=(48, 48, 48), dx=1 / 48)
    n = 70000
    st = random_block(rng, n, 0.3, 0.36)
    b = gpu_batch(sim, [LAWS["fluid"]], [], [st], 1, 1)
    b.set_state(stack([st], "x"), stack([st], "v"), stack([st], "F"), stack([st], "C"))
    keys, perm = b.debug_sort()
    k_ref = O.bin_keys(sim, st["x"].astype(np.float32))
    assert np.array_equal(keys[0], k_ref)
    assert np.array_equal(perm[0], O.stable_sort(k_ref))


# ---------------- forward parity ----------------

@pytest.mark.parametrize("law", list(LAWS))
@pytest.mark.parametrize("col", list(COLS))
def test_single_substep_parity(law, col):
    rng = np.random.default_rng(zlib.crc32(f"{law}/{col}".encode()))
    st = to_f32_state(random_block(rng, 256, 0.4, 0.6, groups=2))
    sim = dict(SIM16, mu_b=0.3)
    act = np.array([[0.7, -0.4]]) if law == "neo_hookean" else None
    ref, _, _ = O.rollout(sim, [LAWS[law]], COLS[col], st, 1, 1, act=act)
    g = gpu_rollout(sim, [LAWS[law]], COLS[col], [st], 1, 1, act=act)["state"]
    for k in "xvFC":
        r = field_rel(g[k][0], ref[k], 256)
        assert r <= 1e-5, (k, r)


def test_rollout_end_cfg1():
    sc = scenes.config1(seed=3)
    st = sc.env_state(0)
    ref, obs_ref, _ = O.rollout(sc.sim, sc.materials, [], st, 1, sc.n_sub)
    g = gpu_rollout(sc.sim, sc.materials, [], [st], 1, sc.n_sub)
    for k in "xvFC":
        r = field_rel(g["state"][k][0], ref[k], sc.n_per_env)
        assert r <= 1e-3, (k, r)
    assert np.allclose(g["obs"][0, 0, :3], obs_ref[0, :3], rtol=1e-5, atol=1e-7)


def test_multi_env_independent():
    rng = np.random.default_rng(7)
    states = [to_f32_state(random_block(rng, 200, 0.4, 0.6)) for _ in range(4)]
    mats = [LAWS["fixed_corotated"]]
    g = gpu_rollout(SIM16, mats, [], states, 2, 3)
    for e in range(4):
        ref, _, _ = O.rollout(SIM16, mats, [], states[e], 2, 3)
        for k in "xvFC":
            assert field_rel(g["state"][k][e], ref[k], 200) <= 1e-4


# ---------------- errors ----------------

def test_out_of_interior_reports_particle():
    rng = np.random.default_rng(0)
    st = random_block(rng, 8, 0.4, 0.6)
    st["x"][0] = (0.01, 0.5, 0.5)
    with pytest.raises(RuntimeError, match="particle 0"):
        gpu_rollout(SIM16, [LAWS["fluid"]], [], [st], 1, 1)


@pytest.mark.parametrize("bad", ["nan", "inf", "fast"])
def test_blown_up_state_reports_not_faults(bad):
    """Non-finite or runaway particles are reported with the reference's text
    and leave the device usable (every index derived from particle data is
    range-checked before use)."""
    rng = np.random.default_rng(1)
    st = random_block(rng, 64, 0.4, 0.6)
    if bad == "nan":
        st["x"][5] = (np.nan, 0.5, 0.5)
    elif bad == "inf":
        st["x"][5] = (0.5, np.inf, 0.5)
    else:
        st["v"][5] = (0.0, 0.0, 1e30)
    # a runaway velocity spreads through the grid to its neighbours, so (as in
    # the reference's index-ordered g2p loop) the lowest failing index is named
    want = "advected outside grid interior" if bad == "fast" else "particle 5 outside grid interior"
    with pytest.raises(RuntimeError, match=want):
        gpu_rollout(SIM16, [LAWS["neo_hookean"]], [], [st], 2, 2)
    ok = gpu_rollout(SIM16, [LAWS["neo_hookean"]], [], [to_f32_state(random_block(rng, 64, 0.4, 0.6))], 1, 2)
    assert np.isfinite(ok["state"]["x"]).all()


# ---------------- gradients ----------------

GRAD_CASES = [
    ("fcr_var", LAWS["fixed_corotated"], "none", {"kind": "var_z"}, None, "sticky"),
    ("fcr_com", LAWS["fixed_corotated"], "sphere", {"kind": "com_target", "target": (0.5, 0.4, 0.5)}, None, "slip"),
    ("nh_act", LAWS["neo_hookean"], "none", {"kind": "var_z"}, True, "slip"),
    ("ep_cyl", LAWS["elastoplastic"], "cylinder", {"kind": "var_z"}, None, "slip"),
    ("ep_box", LAWS["elastoplastic"], "box", {"kind": "var_z"}, None, "slip"),
    ("nh_plane", LAWS["neo_hookean"], "plane", {"kind": "var_z"}, None, "slip"),
    ("fluid_hollow", LAWS["fluid"], "hollow_box",
     {"kind": "fluid_move", "target": (0.55, 0.5, 0.2), "spill_half": 0.1, "spill_temp": 0.01,
      "tier_threshold": 0.02, "tier_low": 1.0, "tier_high": 2.0}, None, "slip"),
]


@pytest.mark.parametrize("name,law,col,loss,use_act,boundary", GRAD_CASES, ids=[c[0] for c in GRAD_CASES])
def test_gradient_parity(name, law, col, loss, use_act, boundary):
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    st = to_f32_state(random_block(rng, 128, 0.42, 0.58, groups=2))
    sim = dict(SIM16, boundary=boundary, mu_b=0.3, dt=2e-4)
    act = rng.uniform(-1, 1, (2, 2)) if use_act else None
    ref = O.rollout_grad(sim, [law], COLS[col], st, 2, 4, loss, act=act, seg=1)
    g = gpu_rollout(sim, [law], COLS[col], [st], 2, 4, act=act, loss=loss, grad=True)
    assert abs(g["loss"][0] - ref["loss"]) <= 1e-4 * max(1.0, abs(ref["loss"]))
    for k in "xvFC":
        a, r = g["grad"][k][0], ref[k]
        if np.linalg.norm(r) < 1e-12:
            continue
        assert cosine(a, r) >= 0.999, (k, cosine(a, r))
        assert rel_l2(a, r) <= 1e-3, (k, rel_l2(a, r))
    if COLS[col]:
        a, r = g["grad"]["cvo"][:, 0], ref["cvo"]
        assert cosine(a, r) >= 0.999 and rel_l2(a, r) <= 1e-3
    if use_act:
        a, r = g["grad"]["act"][:, 0], ref["act"]
        assert cosine(a, r) >= 0.999 and rel_l2(a, r) <= 1e-3
    if np.abs(ref["E"]).max() > 0:
        # dL/dE is one scalar: a cancelling sum over every particle-substep of
        # fp32 terms (the vector gradients above carry the 1e-3 gate)
        assert abs(g["grad"]["E"][0, 0] - ref["E"][0]) <= 3e-3 * abs(ref["E"][0])


# ---------------- determinism / checkpointing ----------------

def test_checkpointed_equals_store_all_bitwise():
    rng = np.random.default_rng(11)
    states = [to_f32_state(random_block(rng, 300, 0.42, 0.58)) for _ in range(2)]
    loss = {"kind": "var_z"}
    a = gpu_rollout(SIM16, [LAWS["elastoplastic"]], COLS["sphere"], states, 3, 4, loss=loss, grad=True, ck=1)
    b = gpu_rollout(SIM16, [LAWS["elastoplastic"]], COLS["sphere"], states, 3, 4, loss=loss, grad=True, ck=4)
    c = gpu_rollout(SIM16, [LAWS["elastoplastic"]], COLS["sphere"], states, 3, 4, loss=loss, grad=True, ck=2)
    for k in ("x", "v", "F", "C", "cvo", "E"):
        assert np.array_equal(a["grad"][k], b["grad"][k]), k
        assert np.array_equal(a["grad"][k], c["grad"][k]), k
    for k in "xvFC":
        assert np.array_equal(a["state"][k], b["state"][k])


def test_run_to_run_bitwise_multi_env():
    """Whole rollouts (fwd + bwd) on 8 envs of config 4 are bit-identical run to
    run: deterministic sort, atomic-free fixed-order transfers."""
    sc = scenes.config4(seed=2, n_envs=8, n_ctrl=2, n_sub=8)
    b = api.from_scene(sc)
    r1 = api.run_scene(b, sc)
    r2 = api.run_scene(b, sc)
    for k in ("obs", "x", "v", "F", "C", "cvo", "E"):
        assert np.array_equal(r1[k], r2[k]), k
    assert np.isfinite(r1["x"]).all() and np.abs(r1["cvo"]).max() > 0


def test_cfg4_env_matches_oracle():
    """Config-4 physics (fluid + viscosity, moving hollow container) on the GPU
    against the fp64 oracle for one env: rollout-end observables within 1e-3."""
    sc = scenes.config4(seed=4, n_envs=2, n_ctrl=2, n_sub=8)
    b = api.from_scene(sc)
    out = api.run_scene(b, sc, want_grad=False)
    cvo, _ = sc.cvo_act()
    for e in range(2):
        _, obs_ref, _ = O.rollout(sc.sim, sc.materials, sc.env_cols(e, cvo), sc.env_state(e), sc.n_ctrl, sc.n_sub,
                                  loss=sc.loss)
        assert np.allclose(out["obs"][:, e, :3], obs_ref[:, :3], rtol=1e-5, atol=1e-6)
        assert np.allclose(out["obs"][:, e, 3:], obs_ref[:, 3:], rtol=1e-3, atol=1e-7)


def test_kept_last_segment_equals_replay_bitwise():
    """The step that fills the tape keeps its segment from the forward pass
    and the backward skips its replay; a context with spare tape capacity
    replays it.  Gradients and states are bit-identical (fluid: the one-word
    F storage is exercised too)."""
    sc = scenes.config4(seed=5, n_envs=3, n_ctrl=2, n_sub=6, lattice_counts=(8, 8, 4))
    out = []
    for spare in (0, 1):
        b = api.from_scene(sc, max_steps=sc.n_ctrl + spare)
        out.append(api.run_scene(b, sc))
        b.close()
    for k in ("obs", "x", "v", "F", "C", "cvo", "E"):
        assert np.array_equal(out[0][k], out[1][k]), k


def _grad_check(g, ref, keys="xvFC"):
    for k in keys:
        a, r = g["grad"][k][0], ref[k]
        if np.linalg.norm(r) < 1e-12:
            continue
        assert cosine(a, r) >= 0.999, (k, cosine(a, r))
        assert rel_l2(a, r) <= 1e-3, (k, rel_l2(a, r))


def test_gradient_parity_multi_collider():
    """Two colliders (plane floor + sphere): the generic multi-collider grid
    kernels (runtime kind switch, up to 4 colliders) and their adjoint."""
    rng = np.random.default_rng(21)
    st = to_f32_state(random_block(rng, 128, 0.42, 0.58))
    sim = dict(SIM16, mu_b=0.3, dt=2e-4)
    cols = COLS["plane"] + COLS["sphere"]
    loss = {"kind": "var_z"}
    ref = O.rollout_grad(sim, [LAWS["elastoplastic"]], cols, st, 2, 4, loss, seg=1)
    g = gpu_rollout(sim, [LAWS["elastoplastic"]], cols, [st], 2, 4, loss=loss, grad=True)
    assert abs(g["loss"][0] - ref["loss"]) <= 1e-4 * max(1.0, abs(ref["loss"]))
    _grad_check(g, ref)
    a, r = g["grad"]["cvo"][:, 0], np.asarray(ref["cvo"]).reshape(2, -1, 9)[:, :2]
    assert cosine(a.ravel(), r.ravel()) >= 0.999 and rel_l2(a.ravel(), r.ravel()) <= 1e-3


def test_gradient_parity_mixed_materials():
    """Two materials with different laws in one env (neo-Hookean + fluid): the
    runtime law dispatch kernels and per-material Young's-modulus cotangents."""
    rng = np.random.default_rng(22)
    st = to_f32_state(random_block(rng, 160, 0.42, 0.58))
    st["material"] = (np.arange(160) % 2).astype(np.int32)
    sim = dict(SIM16, dt=2e-4)
    mats = [LAWS["neo_hookean"], LAWS["fluid"]]
    loss = {"kind": "var_z"}
    ref = O.rollout_grad(sim, mats, [], st, 2, 4, loss, seg=1)
    g = gpu_rollout(sim, mats, [], [st], 2, 4, loss=loss, grad=True)
    assert abs(g["loss"][0] - ref["loss"]) <= 1e-4 * max(1.0, abs(ref["loss"]))
    _grad_check(g, ref)
    for m in range(2):
        if abs(ref["E"][m]) > 0:
            assert abs(g["grad"]["E"][0, m] - ref["E"][m]) <= 3e-3 * abs(ref["E"][m]), m


def test_gradient_parity_many_actuation_groups():
    """12 actuation groups (the 16-group adjoint instantiation)."""
    rng = np.random.default_rng(23)
    st = to_f32_state(random_block(rng, 160, 0.42, 0.58, groups=12))
    sim = dict(SIM16, dt=2e-4)
    act = rng.uniform(-1, 1, (2, 12))
    loss = {"kind": "var_z"}
    ref = O.rollout_grad(sim, [LAWS["neo_hookean"]], [], st, 2, 4, loss, act=act, seg=1)
    g = gpu_rollout(sim, [LAWS["neo_hookean"]], [], [st], 2, 4, act=act, loss=loss, grad=True)
    _grad_check(g, ref)
    a, r = g["grad"]["act"][:, 0], ref["act"]
    assert cosine(a.ravel(), r.ravel()) >= 0.999 and rel_l2(a.ravel(), r.ravel()) <= 1e-3


# ---------------- chunk boundaries inside one tile ----------------

@pytest.mark.parametrize("law", ["fluid", "elastoplastic", "fixed_corotated"])
@pytest.mark.parametrize("n", [1, 31, 32, 33, 64, 65, 97, 130])
def test_one_tile_chunk_counts(law, n):
    """Every particle in one 4^3-cell tile (base cells 4..7 per axis): the
    tile kernels walk it in 32-particle chunks with the perm index of chunk
    k + 1 in parity slot (k + 1) & 1 (two call sites per iteration for fluid,
    one parity-selected site for the SVD laws) -- counts around the chunk
    boundaries, forward and gradients against the oracle."""
    rng = np.random.default_rng(1000 + n)
    st = to_f32_state(random_block(rng, n, 0.29, 0.52))
    ref, _, _ = O.rollout(SIM16, [LAWS[law]], [], st, 1, 1)
    g = gpu_rollout(SIM16, [LAWS[law]], [], [st], 1, 1)["state"]
    for k in "xvFC":
        assert field_rel(g[k][0], ref[k], n) <= 1e-5, k
    loss = {"kind": "var_z"}
    refg = O.rollout_grad(SIM16, [LAWS[law]], [], st, 2, 3, loss, seg=1)
    gg = gpu_rollout(SIM16, [LAWS[law]], [], [st], 2, 3, loss=loss, grad=True)
    for k in "xvFC":
        a, r = gg["grad"][k][0], refg[k]
        if np.linalg.norm(r) < 1e-12:
            continue
        assert cosine(a, r) >= 0.999 and rel_l2(a, r) <= 1e-3, (k, cosine(a, r), rel_l2(a, r))
