"""The small-batch scheduling modes (GPU, through the C ABI).

dm_create picks CTA-cooperative tiles (`coop`: a group of 2 or 4 warps of a
CTA shares a tile's chunks; `grid_coop`: the 4 warps share its owned nodes)
from the batch size; DIFFMPM_COOP / DIFFMPM_GRID_COOP / DIFFMPM_COOP_CG force
them.  Every mode must be
deterministic run to run (the replay verification relies on it) and agree
with the others up to the fp32 summation order of the per-warp partials.
"""
import os

import numpy as np
import pytest

from paper_2412_12089_b200 import api, scenes

pytestmark = pytest.mark.gpu

# (COOP, grid COOP, COOP group size in warps)
MODES = [("0", "0", "4"), ("1", "0", "2"), ("1", "0", "4"), ("1", "1", "4")]


def _run(sc, coop, grid_coop, cg):
    old = {k: os.environ.get(k) for k in ("DIFFMPM_COOP", "DIFFMPM_GRID_COOP", "DIFFMPM_COOP_CG")}
    os.environ["DIFFMPM_COOP"], os.environ["DIFFMPM_GRID_COOP"], os.environ["DIFFMPM_COOP_CG"] = coop, grid_coop, cg
    try:
        b = api.from_scene(sc)  # the mode is read when the context is created
        r1 = api.run_scene(b, sc)
        r2 = api.run_scene(b, sc)
        b.close()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    for k in r1:
        if isinstance(r1[k], np.ndarray):
            assert np.array_equal(r1[k], r2[k]), (coop, grid_coop, cg, k)
    return r1


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


@pytest.mark.parametrize("cfg", [2, 4])
def test_modes_deterministic_and_consistent(cfg):
    kw = {"seed": 3, "n_envs": 3, "n_ctrl": 2}
    sc = scenes.CONFIGS[cfg](**kw)
    runs = {m: _run(sc, *m) for m in MODES}
    ref = runs[("0", "0", "4")]
    full = lambda r: np.concatenate([np.asarray(r[k], np.float64).ravel() for k in ("x", "v", "F", "C")])
    for m, r in runs.items():
        assert _rel(r["obs"], ref["obs"]) <= 1e-4, (m, "obs")
        # the full per-env state gradient (a field the loss does not depend on,
        # e.g. dL/dF0 of a centre-of-mass loss, is rounding noise on its own)
        assert _rel(full(r), full(ref)) <= 1e-4, (m, "dL/dstate", _rel(full(r), full(ref)))
        scale = np.linalg.norm(full(ref))
        for k in ("cvo", "act"):
            if k not in ref:
                continue
            if np.linalg.norm(ref[k]) <= 1e-6 * scale:  # the loss does not depend on it: noise
                assert np.linalg.norm(r[k]) <= 1e-4 * scale, (m, k)
            else:
                assert _rel(r[k], ref[k]) <= 1e-4, (m, k, _rel(r[k], ref[k]))


def test_stress_cache_on_off_consistent():
    """The elastoplastic stress cache (G2P writes P F'^T, the next P2G reads it
    instead of a new SVD) changes only fp32 rounding: a cfg3 rollout with it
    and with DIFFMPM_NO_TAU_CACHE=1 agree (states 1e-5, the full per-env
    gradient 1e-4), and each is deterministic."""
    sc = scenes.CONFIGS[3](seed=4, n_envs=2, n_ctrl=2)

    def run(no_cache):
        old = os.environ.get("DIFFMPM_NO_TAU_CACHE")
        if no_cache:
            os.environ["DIFFMPM_NO_TAU_CACHE"] = "1"
        else:
            os.environ.pop("DIFFMPM_NO_TAU_CACHE", None)
        try:
            b = api.from_scene(sc)
            r1, r2 = api.run_scene(b, sc), api.run_scene(b, sc)
            st = b.get_state()
            b.close()
        finally:
            if old is None:
                os.environ.pop("DIFFMPM_NO_TAU_CACHE", None)
            else:
                os.environ["DIFFMPM_NO_TAU_CACHE"] = old
        for k in r1:
            if isinstance(r1[k], np.ndarray):
                assert np.array_equal(r1[k], r2[k]), (no_cache, k)
        return r1, st

    (ra, sa), (rb, sb) = run(False), run(True)
    for k in "xvFC":
        assert _rel(sa[k], sb[k]) <= 1e-5, (k, _rel(sa[k], sb[k]))
    full = lambda r: np.concatenate([np.asarray(r[k], np.float64).ravel() for k in ("x", "v", "F", "C")])
    assert _rel(full(ra), full(rb)) <= 1e-4, _rel(full(ra), full(rb))
    assert _rel(ra["cvo"], rb["cvo"]) <= 1e-4


@pytest.mark.parametrize("cfg", [1, 2])
def test_launch_chaining_bitwise(cfg):
    """Programmatic dependent launch (DIFFMPM_PDL) and the one-CTA work-list
    ordering change only when kernels start, never what they compute: a
    rollout (forward, replay, adjoint) with launch chaining on equals the one
    with it off bit for bit (cfg2: from the second control step on, the
    work list is ordered by k_order_small -- the active-tile count is known
    after the first)."""
    sc = scenes.CONFIGS[2](seed=5, n_envs=2, n_ctrl=2) if cfg == 2 else scenes.CONFIGS[1](seed=5, n_sub=12)

    def run(pdl):
        old = os.environ.get("DIFFMPM_PDL")
        os.environ["DIFFMPM_PDL"] = pdl
        try:
            b = api.from_scene(sc)
            r = api.run_scene(b, sc)
            b.close()
        finally:
            if old is None:
                os.environ.pop("DIFFMPM_PDL", None)
            else:
                os.environ["DIFFMPM_PDL"] = old
        return r

    on, off = run("1"), run("0")
    for k in off:
        if isinstance(off[k], np.ndarray):
            assert np.array_equal(on[k], off[k]), k
