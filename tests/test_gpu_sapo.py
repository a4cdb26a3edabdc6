"""GPU: config-5 pieces -- pooled group observables (forward vs the fp64
oracle state, adjoint vs central FD through the oracle), the incremental
backward (== one-shot backward, bitwise), and one SAPO iteration with the
policy in the loop."""
import numpy as np
import pytest

import pyoracle as O
from paper_2412_12089_b200 import api, scenes

pytestmark = pytest.mark.gpu


def group_obs_np(x, v, group, G=8):
    out = []
    for g in range(G):
        m = group == g
        xs, vs = x[m], v[m]
        mz = xs[:, 2].mean()
        out += list(xs.mean(0)) + list(vs.mean(0)) + [((xs[:, 2] - mz) ** 2).mean(), np.linalg.norm(vs, axis=1).mean()]
    return np.array(out)


def small_cfg2(n_envs=2, n_ctrl=2, n_sub=4):
    sc = scenes.config2(seed=3, n_envs=n_envs, n_ctrl=n_ctrl, n_sub=n_sub)
    sc.extra["obs_groups"] = 8
    return sc


def test_group_obs_forward_matches_oracle():
    sc = small_cfg2()
    b = api.from_scene(sc)
    out = api.run_scene(b, sc, want_grad=False)
    cvo, act = sc.cvo_act()
    for e in range(sc.n_envs):
        st, _, _ = O.rollout(sc.sim, sc.materials, [], sc.env_state(e), sc.n_ctrl, sc.n_sub, act=act[e])
        want = group_obs_np(st["x"], st["v"], sc.group[e])
        got = out["obs"][-1, e, 7:]
        assert np.allclose(got, want, rtol=2e-4, atol=2e-6), np.abs(got - want).max()


def test_incremental_backward_equals_one_shot():
    sc = small_cfg2(n_envs=3, n_ctrl=3)
    b = api.from_scene(sc)
    rng = np.random.default_rng(0)
    cvo, act = sc.cvo_act()
    b.set_state(sc.x, sc.v, sc.F, sc.C, sc.material, sc.group)
    for t in range(sc.n_ctrl):
        b.step(None, act[:, t])
    dobs = rng.standard_normal((sc.n_ctrl, sc.n_envs, b.obs_dim)).astype(np.float32) * 1e-2
    full = b.backward(dobs=dobs)
    b.backward_begin()
    dact = []
    for t in range(sc.n_ctrl - 1, -1, -1):
        _, a = b.backward_step(dobs[t])
        dact.append(a)
    inc = b.backward_end()
    assert np.array_equal(np.stack(dact[::-1]), full["act"])
    for k in ("x", "v", "F", "C", "E"):
        assert np.array_equal(inc[k], full[k]), k


def test_group_obs_gradient_vs_fd():
    """d (w . group_obs) / d (initial x, v) vs central FD of the fp64 oracle."""
    sc = small_cfg2(n_envs=1, n_ctrl=1, n_sub=3)
    b = api.from_scene(sc)
    cvo, act = sc.cvo_act()
    rng = np.random.default_rng(1)
    w = rng.standard_normal(64)
    b.set_state(sc.x, sc.v, sc.F, sc.C, sc.material, sc.group)
    b.step(None, act[:, 0])
    dobs = np.zeros((1, 1, b.obs_dim), np.float32)
    dobs[0, 0, 7:] = w
    g = b.backward(dobs=dobs)

    st0 = {k: np.asarray(getattr(sc, k)[0], np.float64) for k in ("x", "v", "F", "C")}
    st0["group"] = sc.group[0]
    st0["material"] = sc.material[0]

    def L(st):
        out, _, _ = O.rollout(sc.sim, sc.materials, [], st, 1, sc.n_sub, act=act[0, :1])
        return w @ group_obs_np(out["x"], out["v"], sc.group[0])

    idx = rng.choice(sc.n_per_env, 6, replace=False)
    for p in idx:
        for field, a, h in (("x", 2, 1e-6), ("v", 0, 1e-5), ("v", 2, 1e-5)):
            sp = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in st0.items()}
            sm = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in st0.items()}
            sp[field][p, a] += h
            sm[field][p, a] -= h
            fd = (L(sp) - L(sm)) / (2 * h)
            got = g[field][0, p, a]
            assert abs(got - fd) <= 2e-3 * max(abs(fd), 1e-3), (field, p, a, got, fd)


def test_sapo_iteration_runs():
    from paper_2412_12089_b200.sapo import SapoTrainer
    tr = SapoTrainer(seed=0, n_envs=4, horizon=4, n_sub=4, critic_passes=2, hidden=(32, 32, 32))
    p0 = [p.detach().clone() for p in tr.actor.parameters()]
    s1 = tr.iteration()
    s2 = tr.iteration()
    for s in (s1, s2):
        assert all(np.isfinite(v) for v in s.values()), s
    assert s1["grad_norm"] > 0
    moved = sum(float((p - q).abs().sum()) for p, q in zip(tr.actor.parameters(), p0))
    assert moved > 0


def test_sapo_checkpoint_resume_bitwise(tmp_path):
    """Trainer persistence in the DSIMCKPT container (checkpoint_io.hpp:140-205):
    run 2 iterations, save, run 2 more; a fresh trainer restored from the file
    runs the same 2 iterations bit for bit (test_cli.cpp:130-151)."""
    import torch
    from paper_2412_12089_b200 import ckpt
    from paper_2412_12089_b200.sapo import SapoTrainer
    kw = dict(seed=1, n_envs=3, horizon=3, n_sub=4, critic_passes=2, hidden=(32, 32, 32))
    a = SapoTrainer(**kw)
    a.iteration()
    a.iteration()
    path = str(tmp_path / "trainer.ckpt")
    ckpt.save_checkpoint(ckpt.snapshot_trainer(a), path)
    ra = [a.iteration(), a.iteration()]
    torch.manual_seed(123)  # different network init: parameters must come from the file
    b = SapoTrainer(**kw)
    ckpt.restore_trainer(b, ckpt.load_checkpoint(path))
    rb = [b.iteration(), b.iteration()]
    assert ra == rb
    for p, q in zip(list(a.actor.parameters()) + list(a.critics.parameters()),
                    list(b.actor.parameters()) + list(b.critics.parameters())):
        assert torch.equal(p, q)
    assert float(a.log_alpha) == float(b.log_alpha) and a.iter == b.iter == 4
