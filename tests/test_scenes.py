"""CPU: seeded synthetic inputs, task action maps and losses."""
import numpy as np
import pytest

from paper_2412_12089_b200 import scenes
from paper_2412_12089_b200.losses import loss_and_dobs


def interior_ok(sc):
    dx = sc.sim["dx"]
    b = np.floor(sc.x / dx - 0.5)
    return (b >= 1).all() and (b + 2 <= np.array(sc.sim["dims"]) - 2).all()


@pytest.mark.parametrize("cfg,kw", [(1, {}), (2, {"n_envs": 2}), (3, {"n_envs": 2, "n_per_env": 3000}),
                                     (4, {"n_envs": 2})])
def test_configs_build(cfg, kw):
    sc = scenes.CONFIGS[cfg](seed=0, **kw)
    E, N = sc.n_envs, sc.n_per_env
    assert sc.x.shape == (E, N, 3) and sc.F.shape == (E, N, 9)
    assert interior_ok(sc)
    cvo, act = sc.cvo_act()
    assert cvo.shape[:2] == (E, sc.n_ctrl)
    assert np.isfinite(sc.x).all()


def test_config_sizes_match_baseline():
    assert scenes.config1().n_per_env == 4096
    assert scenes.config2(n_envs=1).n_per_env == 20480
    assert scenes.config4(n_envs=1).n_per_env == 16384
    sc = scenes.config4(n_envs=1)
    assert (sc.n_ctrl, sc.n_sub) == (16, 32) and tuple(sc.sim["dims"]) == (48, 48, 48)
    sc = scenes.config3(n_envs=1, n_per_env=30000)
    assert (sc.n_ctrl, sc.n_sub, sc.checkpoint_every) == (24, 20, 4)


@pytest.mark.parametrize("cfg", [1, 3, 4])
def test_sharding_is_input_invariant(cfg):
    kw = {"n_per_env": 500} if cfg == 3 else {}
    full = scenes.CONFIGS[cfg](seed=5, n_envs=4, **kw)
    part = scenes.CONFIGS[cfg](seed=5, n_envs=2, env_offset=2, **kw)
    assert np.array_equal(full.x[2:], part.x)
    assert np.array_equal(full.v[2:], part.v)
    assert np.array_equal(full.actions[2:], part.actions)


def test_seeded_determinism():
    a = scenes.config1(seed=3)
    b = scenes.config1(seed=3)
    c = scenes.config1(seed=4)
    assert np.array_equal(a.v, b.v) and not np.array_equal(a.v, c.v)
    assert abs(a.v.std() - 0.5) < 0.02


def test_kmeans_groups_cover():
    sc = scenes.config2(n_envs=1)
    g = sc.group[0]
    assert set(np.unique(g)) == set(range(8))


@pytest.mark.parametrize("cfg", [3, 4])
def test_task_vjp_matches_fd(cfg):
    kw = {"n_per_env": 200} if cfg == 3 else {"lattice_counts": (4, 4, 2)}
    sc = scenes.CONFIGS[cfg](seed=1, n_envs=2, n_ctrl=5, **kw)
    rng = np.random.default_rng(0)
    cvo, _ = sc.task.forward(sc.actions)
    g = rng.standard_normal(cvo.shape)
    ga = sc.task.vjp(sc.actions, g, None)
    h = 1e-6
    for idx in [(0, 0, 0), (1, 2, 1), (0, 4, 2)]:
        ap = sc.actions.copy()
        am = sc.actions.copy()
        ap[idx] += h
        am[idx] -= h
        fd = ((sc.task.forward(ap)[0] - sc.task.forward(am)[0]) * g).sum() / (2 * h)
        assert abs(ga[idx] - fd) < 1e-6 * max(1, abs(fd))


@pytest.mark.parametrize("spec", [{"kind": "com_target", "target": (0.5, 0.4, 0.5)}, {"kind": "neg_mean_z"},
                                  {"kind": "var_z"},
                                  {"kind": "fluid_move", "target": (0.55, 0.5, 0.2), "spill_half": 0.15,
                                   "spill_temp": 0.01}])
def test_loss_gradient_fd_and_torch(spec):
    import torch
    from paper_2412_12089_b200.losses import loss_and_dobs_torch
    rng = np.random.default_rng(2)
    obs = rng.random((3, 4, 7))
    L, d = loss_and_dobs(spec, obs)
    h = 1e-7
    for idx in [(0, 0, 0), (1, 3, 2), (2, 1, 5), (0, 2, 6)]:
        op = obs.copy()
        om = obs.copy()
        op[idx] += h
        om[idx] -= h
        fd = (loss_and_dobs(spec, op)[0][idx[0]] - loss_and_dobs(spec, om)[0][idx[0]]) / (2 * h)
        assert abs(d[idx] - fd) < 1e-5 * max(1, abs(fd))
    Lt, dt = loss_and_dobs_torch(spec, torch.tensor(obs))
    assert np.allclose(Lt.numpy(), L) and np.allclose(dt.numpy(), d, atol=1e-6)


def test_lattice_reset_host_matches_direct_restatement():
    """scenes.lattice_reset_host (the host twin of the device reset
    dm_reset_lattice) against a direct restatement of the draws: cfg1's
    jittered lattice + Box-Muller velocities and cfg4's origin-offset lattice,
    bit for bit (env.hpp:66-96, mpm.hpp:371-395, rng.hpp:11-55)."""
    from paper_2412_12089_b200.rng import RngStream
    dx = 1.0 / 32
    sc = scenes.config1(seed=7, n_envs=2, env_offset=3)
    base = scenes.lattice((0.3, 0.3, 0.3), (16, 16, 16), (0.2 / 16,) * 3)
    N = base.shape[0]
    for e in range(2):
        r = RngStream(7, 3 + e)
        jit = r.uniform(-0.25 * dx, 0.25 * dx, 3 * N).reshape(N, 3)
        assert np.array_equal(sc.x[e], base + jit)
        assert np.array_equal(sc.v[e], 0.5 * r.normals(3 * N).reshape(N, 3))
    sc4 = scenes.config4(seed=2, n_envs=3, n_ctrl=2, n_sub=4, lattice_counts=(4, 4, 2))
    half = 0.15
    for e in range(3):
        r = RngStream(2, e)
        d = r.uniform(-0.01, 0.01, 2)
        org = np.array([0.5 - half, 0.5 - half, 0.15]) + np.array([d[0], d[1], 0.0])
        assert np.array_equal(sc4.x[e], scenes.lattice(org, (4, 4, 2), np.array([0.3, 0.3, 0.15]) / (4, 4, 2)))
        assert np.allclose(sc4.task.center0[e][:2], org[:2] + half, rtol=0, atol=1e-15)


def test_lattice_reset_draw_order_shares_the_action_stream():
    """cfg4: the origin draws come first in the env's stream, the per-step
    actions continue after them (one stream per env, env.hpp:71)."""
    from paper_2412_12089_b200.rng import RngStream
    sc = scenes.config4(seed=5, n_envs=2, n_ctrl=3, n_sub=4, lattice_counts=(4, 4, 2))
    for e in range(2):
        u = RngStream(5, e).uniform(-1.0, 1.0, 2 + 9)
        assert np.array_equal(sc.actions[e], u[2:].reshape(3, 3))


@pytest.mark.skipif(not __import__("pyoracle").have_ref(), reason="oracle/_ref not built (needs /root/reference)")
def test_samplers_match_reference_bitwise():
    """scenes.sample_box / sample_cylinder restate mpm.hpp:371-423 with the
    reference's own expression order: positions and volumes bit-identical."""
    import pyoracle as O
    cases = [("box", (0.27, 0.42, 0.1625), (0.16, 0.16, 0.08), 0.05, 8),
             ("box", (0.3, 0.3, 0.3), (0.2, 0.2, 0.2), 1 / 32, 27),
             ("box", (0.35, 0.35, 0.15), (0.3, 0.3, 0.15), 1 / 48, 8)]
    for kind, a, b, dx, ppc in cases:
        x, vol = scenes.sample_box(a, b, dx, ppc)
        xr, vr = O.ref_sample(kind, a, b, dx, ppc)
        assert np.array_equal(x, xr) and vol == vr
    x, vol = scenes.sample_cylinder((0.5, 0.5, 0.1), 0.08, 0.12, 1 / 40, 8)
    xr, vr = O.ref_sample("cylinder", (0.5, 0.5, 0.1), (0.08, 0.12), 1 / 40, 8)
    assert x.shape[0] > 100 and np.array_equal(x, xr) and vol == vr
