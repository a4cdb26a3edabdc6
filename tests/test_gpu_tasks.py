"""The reference's MPM tasks through the task-level C ABI (GPU).

MiniFluidMove (tasks.hpp:502-645) and MiniRollFlat (tasks.hpp:232-369) as
EnvBatch<Task> (env.hpp:55-117) on the GPU simulator, against the reference's
own task code compiled unchanged (fixtures tests/golden/task_*.npz from
tests/golden/make_task_golden.py): observations and rewards per step within
1e-5, the auto-reset at episode_len (T = 6 > episode_len = 4: the gradient
is cut there), and dL/dactions for L = sum w_r rewards + sum w_o obs against
central differences of the reference's double forward and its tape gradient
at cosine >= 0.999, rel L2 <= 1e-3.
"""
import os

import numpy as np
import pytest

from helpers import cosine, rel_l2
from paper_2412_12089_b200 import api

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _fixture(name):
    fx = np.load(os.path.join(GOLDEN, "task_%s.npz" % name))
    cfg = dict(zip([str(k) for k in fx["cfg_keys"]], [float(v) for v in fx["cfg_vals"]]))
    for k in ("grid_n", "ppc", "substeps", "episode_len", "cloud_k"):
        cfg[k] = int(cfg[k])
    cfg["kind"] = int(fx["kind"])
    return fx, cfg


@pytest.mark.parametrize("name", ["fluid_move", "roll_flat"])
def test_task_rewards_obs_and_action_gradients(name):
    fx, cfg = _fixture(name)
    E, T = int(fx["n_envs"]), int(fx["T"])
    env = api.TaskBatch(cfg, E, seed=int(fx["seed"]), horizon=T)
    assert env.obs_dim == fx["obs"].shape[2] and env.act_dim == fx["actions"].shape[2]
    obs0 = env.observe()
    assert rel_l2(obs0, fx["obs"][0]) <= 1e-6
    for t in range(T):
        r, d = env.step(fx["actions"][t])
        ref = fx["rewards"][t]
        assert np.all(np.abs(r - ref) <= 1e-5 * np.maximum(np.abs(ref), 1e-2)), (t, r, ref)
        assert list(d) == [(t + 1) % cfg["episode_len"] == 0] * E  # EnvBatch::step done + auto-reset
        o = env.observe()
        for e in range(E):
            assert rel_l2(o[e], fx["obs"][t + 1][e]) <= 1e-5, (t, e, rel_l2(o[e], fx["obs"][t + 1][e]))
    da = env.backward(fx["w_r"], fx["w_o"])
    for ref in (fx["dact_fd"], fx["dact_tape"]):
        assert cosine(da, ref) >= 0.999 and rel_l2(da, ref) <= 1e-3, (cosine(da, ref), rel_l2(da, ref))
    # after the backward the tape restarts from the current state: keep stepping
    r, _ = env.step(fx["actions"][0])
    assert np.isfinite(r).all()
    env.close()


def test_task_errors_and_plain_stepping():
    cfg = api.task_config("fluid_move", episode_len=3)
    env = api.TaskBatch(cfg, 2, seed=1, horizon=2)
    a = np.zeros((2, 2))
    env.step(a)
    env.step(a)
    with pytest.raises(RuntimeError, match="tape capacity"):
        env.step(a)
    env.backward(np.ones((2, 2)))
    for _ in range(5):  # plain stepping (EnvBatch::step): a full tape restarts itself
        r, d = env.step(a, record=False)
        assert np.isfinite(r).all()
    with pytest.raises(ValueError, match="unrecorded"):
        env.backward(np.ones((env.tape_steps, 2)))
    with pytest.raises(ValueError):
        api.TaskBatch(dict(cfg, substeps=0), 1)
