"""The committed BASELINE-config gradient fixtures (tests/golden/cfg*_grad.npz,
made by tests/golden/make_config_golden.py from the reference build) still
describe the scenes scenes.py builds: same fp32 initial state (sha256), sane
contents.  CPU only; the GPU comparison is tests/test_gpu_config_parity.py."""
import os

import numpy as np
import pytest

from config_cases import GRAD_CASES, case_scene, state_sha

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("case", GRAD_CASES)
def test_fixture_matches_scene(case):
    fx = np.load(os.path.join(GOLDEN, "%s_grad.npz" % case))
    sc, st, cols, act, loss = case_scene(case)
    assert state_sha(st) == str(fx["sha"])
    N = sc.n_per_env
    assert fx["gx"].shape == (N, 3) and fx["gF"].shape == (N, 9) and int(fx["n_sub"]) == sc.n_sub
    for k in ("gx", "gv", "gF", "gC"):
        assert np.isfinite(fx[k]).all()
    assert np.linalg.norm(fx["gx"]) > 0 and np.linalg.norm(fx["gv"]) > 0
