"""GPU: device-side env reset (dm_reset_lattice)
against the host generator scenes.lattice_reset_host, bit for bit in fp32:
full reset for cfg1 (jitter + Box-Muller velocities), cfg2 (per-particle
actuation groups) and cfg4 (per-env origin draws), and a masked reset that
regenerates only the done envs (EnvBatch::reset_env, env.hpp:93-96)."""
import numpy as np
import pytest

from paper_2412_12089_b200 import api, scenes

pytestmark = pytest.mark.gpu


def _check_env(st, e, x, v):
    assert np.array_equal(st["x"][e], x.astype(np.float32))
    # Box-Muller uses the device's double log / cos: identical after fp32 rounding
    assert np.array_equal(st["v"][e], v.astype(np.float32))
    eye = np.tile(np.eye(3, dtype=np.float32).ravel(), (x.shape[0], 1))
    assert np.array_equal(st["F"][e], eye) and not st["C"][e].any()


@pytest.mark.parametrize("cfg,kw", [(1, {"n_envs": 2, "env_offset": 5}), (2, {"n_envs": 2, "n_ctrl": 1}),
                                     (4, {"n_envs": 3, "n_ctrl": 1, "lattice_counts": (8, 8, 4)})])
def test_device_reset_matches_host(cfg, kw):
    sc = scenes.CONFIGS[cfg](seed=11, **kw)
    spec, seed = sc.extra["reset"], sc.extra["seed"]
    b = api.from_scene(sc)
    d = b.reset_lattice(spec, seed, sc.env_offset, particle_group=sc.extra.get("particle_group"))
    x, v, dh = scenes.lattice_reset_host(spec, seed, sc.env_offset, sc.n_envs)
    assert np.array_equal(d, dh)
    st = b.get_state()
    for e in range(sc.n_envs):
        _check_env(st, e, x[e], v[e])
        assert np.array_equal(x[e], sc.x[e]) and np.array_equal(v[e], sc.v[e])
    assert b.tape_steps == 0
    # the regenerated state steps like the uploaded one
    cvo, act = sc.cvo_act()
    o1 = b.step(cvo[:, 0] if sc.colliders else None, act[:, 0] if getattr(sc.task, "n_act", 0) else None)
    b.set_state(sc.x, sc.v, sc.F, sc.C, sc.material, sc.group)
    o2 = b.step(cvo[:, 0] if sc.colliders else None, act[:, 0] if getattr(sc.task, "n_act", 0) else None)
    assert np.array_equal(o1, o2)
    b.close()


def test_masked_reset_keeps_other_envs():
    sc = scenes.config4(seed=3, n_envs=3, n_ctrl=2, n_sub=4, lattice_counts=(8, 8, 4))
    spec, seed = sc.extra["reset"], sc.extra["seed"]
    b = api.from_scene(sc)
    b.set_state(sc.x, sc.v, sc.F, sc.C, sc.material, sc.group)
    cvo, _ = sc.cvo_act()
    b.step(cvo[:, 0])
    before = b.get_state()
    mask = np.array([0, 1, 0], np.uint8)
    b.reset_lattice(spec, seed, sc.env_offset, env_mask=mask)
    after = b.get_state()
    x, v, _ = scenes.lattice_reset_host(spec, seed, sc.env_offset, sc.n_envs)
    _check_env(after, 1, x[1], v[1])
    for e in (0, 2):
        for k in "xvFC":
            assert np.array_equal(after[k][e], before[k][e])
    assert b.tape_steps == 0
    b.step(cvo[:, 1])  # the new initial state is steppable
    b.close()


def test_reset_spec_validation():
    sc = scenes.config4(seed=3, n_envs=2, n_ctrl=1, n_sub=2, lattice_counts=(4, 4, 2))
    b = api.from_scene(sc)
    bad = dict(sc.extra["reset"], counts=(4, 4, 3))
    with pytest.raises(ValueError, match="particles_per_env"):
        b.reset_lattice(bad, 0)
    b.close()
