"""CPU: the task fixtures (tests/golden/task_*.npz) reproduce from the
reference's own tasks (oracle/_ref, tasks.hpp compiled unchanged) -- the
double forward bit for bit -- and their two gradient references (reference
tape, central differences) agree.  The GPU comparison is
tests/test_gpu_tasks.py."""
import os

import numpy as np
import pytest

import pyoracle as O
from helpers import cosine, rel_l2

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name", ["fluid_move", "roll_flat"])
def test_task_fixture(name):
    fx = np.load(os.path.join(GOLDEN, "task_%s.npz" % name))
    assert cosine(fx["dact_tape"], fx["dact_fd"]) >= 0.99999 and rel_l2(fx["dact_tape"], fx["dact_fd"]) <= 1e-5
    if not O.have_ref():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    cfg = dict(zip([str(k) for k in fx["cfg_keys"]], [float(v) for v in fx["cfg_vals"]]))
    r, o, _ = O.ref_task_rollout(int(fx["kind"]), cfg, int(fx["n_envs"]), int(fx["seed"]), 0, fx["actions"])
    assert np.array_equal(r, fx["rewards"]) and np.array_equal(o, fx["obs"])
