"""Reference error paths and tape checks through the C ABI (GPU).

  * mpm_step's CFL warning (mpm.hpp:355-361; test_mpm.cpp:300-308): once per
    violating control step, on the velocities at its entry -- and not again
    for a later step that no longer violates it
  * det(F) <= 0 (mpm.hpp:168-169, 203-205) and substeps < 1 (mpm.hpp:354)
  * replay verification (tape.hpp:234-241) with a fault-injected
    non-deterministic forward, in the style of test_tape.cpp:311-323
  * dm_observe between a full rollout and the backward leaves the gradients
    unchanged; a keep-pool allocation failure falls back to the replay
  * the *_device path reports device-detected errors at the next sync
"""
import numpy as np
import pytest

from helpers import random_block, to_f32_state
from paper_2412_12089_b200 import api

pytestmark = pytest.mark.gpu

SIM16 = {"dims": (16, 16, 16), "dx": 1 / 16, "dt": 1e-4, "gravity": (0, 0, -9.8), "boundary": "slip"}
FLUID = {"kind": "fluid", "E": 2e4, "nu": 0.3, "rho": 1000, "volume": 1e-4, "bulk": 2e4}
EP = {"kind": "elastoplastic", "E": 5e3, "nu": 0.2, "rho": 1, "volume": 1e-4, "yield_stress": 20}
FCR = {"kind": "fixed_corotated", "E": 1e4, "nu": 0.3, "rho": 1, "volume": 1e-4}
SPHERE = [{"kind": "sphere", "center": (0.5, 0.5, 0.66), "radius": 0.08, "velocity": (0.1, 0, -0.3)}]


def batch_for(st, mats, cols=(), n_sub=2, max_steps=2, sim=SIM16, E=1):
    b = api.MpmBatch(sim, list(mats), list(cols), E, st["x"].shape[0], n_sub, max_steps)
    stack = lambda k: np.stack([st[k]] * E)
    b.set_state(stack("x"), stack("v"), stack("F"), stack("C"), stack("material"), stack("group"))
    return b


def cvo_of(cols, E=1):
    if not cols:
        return None
    c = cols[0]
    row = np.array([*c["center"], *c.get("velocity", (0, 0, 0)), *c.get("omega", (0, 0, 0))], np.float32)
    return np.broadcast_to(row, (E, 1, 9)).copy()


def test_cfl_warning_once_per_violating_step(capfd):
    rng = np.random.default_rng(5)
    st = to_f32_state(random_block(rng, 256, 0.44, 0.56, vs=0.0, fs=0.0, cs=0.0))
    st["v"][17] = (0.0, 0.0, 800.0)  # 800 * 1e-4 >= 1/16: violates at the first step's entry
    b = batch_for(st, [FCR], n_sub=1, max_steps=2)
    b.step()
    first = capfd.readouterr().err
    assert first.count("CFL") == 1, first
    # the grid transfer spreads the light particle's momentum: below the limit
    # at the second step's entry, so no second warning (the word is per step)
    assert np.abs(b.get_state()["v"]).max() * 1e-4 < 1 / 16
    b.step()
    assert "CFL" not in capfd.readouterr().err


@pytest.mark.parametrize("mat,name", [(FLUID, "stress_fluid"), (EP, "stress_elastoplastic"),
                                      (FCR, "stress_fixed_corotated")])
def test_det_f_nonpositive(mat, name):
    rng = np.random.default_rng(2)
    st = to_f32_state(random_block(rng, 64, 0.4, 0.6, fs=0.0))
    st["F"][3] = np.diag([-1.0, 1.0, 1.0]).ravel()
    b = batch_for(st, [mat], n_sub=1, max_steps=1)
    with pytest.raises(RuntimeError, match=name + r": det\(F\) <= 0.*particle 3"):
        b.step()


def test_substeps_below_one():
    with pytest.raises(ValueError, match="mpm_step: substeps < 1"):
        api.MpmBatch(SIM16, [FCR], [], 1, 8, 0, 1)


def _rollout(st, mats, cols, T, S, max_steps, inject=None, observe_between=False, E=2):
    b = batch_for(st, mats, cols, n_sub=S, max_steps=max_steps, E=E)
    cvo = cvo_of(cols, E)
    obs = [b.step(cvo) for _ in range(T)]
    if observe_between:
        moved = None if cvo is None else (cvo + np.float32(0.05)).astype(np.float32)
        b.observe(moved)
    if inject is not None:
        b.debug_inject(*inject)
    dobs = np.zeros((T, E, 7), np.float32)
    dobs[:, :, 5] = 1.0  # var_z
    dobs[-1, :, 2] = 0.3
    g = b.backward(dobs=dobs)
    b.close()
    return np.stack(obs), g


@pytest.mark.parametrize("max_steps", [3, 4])  # the last step replayed, or kept from the forward
def test_replay_fault_injection_detected(max_steps):
    rng = np.random.default_rng(8)
    st = to_f32_state(random_block(rng, 200, 0.42, 0.58))
    _rollout(st, [EP], SPHERE, 3, 4, max_steps)  # clean: the replays verify
    with pytest.raises(RuntimeError, match=r"checkpoint replay: non-deterministic forward \(exit value 15 changed\)"):
        _rollout(st, [EP], SPHERE, 3, 4, max_steps, inject=(0, 1, 5))


def test_observe_after_full_rollout_keeps_gradients():
    rng = np.random.default_rng(9)
    st = to_f32_state(random_block(rng, 200, 0.42, 0.58))
    _, g0 = _rollout(st, [EP], SPHERE, 3, 4, 3)
    _, g1 = _rollout(st, [EP], SPHERE, 3, 4, 3, observe_between=True)
    for k in ("x", "v", "F", "C", "cvo", "E"):
        assert np.array_equal(g0[k], g1[k]), k


def test_keep_pool_allocation_failure_falls_back_to_replay(monkeypatch):
    rng = np.random.default_rng(10)
    st = to_f32_state(random_block(rng, 200, 0.42, 0.58))
    o0, g0 = _rollout(st, [FLUID], SPHERE, 2, 4, 2)
    monkeypatch.setenv("DIFFMPM_DEBUG_FAIL_KEEP_POOL", "1")
    o1, g1 = _rollout(st, [FLUID], SPHERE, 2, 4, 2)
    assert np.array_equal(o0, o1)
    for k in ("x", "v", "F", "C", "cvo", "E"):
        assert np.array_equal(g0[k], g1[k]), k


def test_device_path_reports_at_sync():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    st = random_block(rng, 8, 0.4, 0.6)
    st["x"][0] = (0.01, 0.5, 0.5)
    b = api.MpmBatch(SIM16, [FLUID], [], 1, 8, 1, 2)
    dev = torch.device("cuda")
    T = lambda a: torch.as_tensor(np.asarray(a, np.float32)[None], device=dev)
    with torch.cuda.stream(b.torch_stream()):
        b.set_state(T(st["x"]), T(st["v"]), T(st["F"]), T(st["C"]))
        obs = torch.zeros((1, 7), device=dev)
        b.step(None, None, obs)  # no host synchronisation: returns OK
        with pytest.raises(RuntimeError, match="particle 0 outside grid interior"):
            b.sync()
