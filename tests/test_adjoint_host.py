"""CPU: the hand-written adjoint (device code in paper_2412_12089_b200/csrc,
compiled by g++ in fp64 via tests/native/adjoint_check.cpp) against the
reference-tape gradient oracle, on every law x collider family.  Tolerance:
fp64 round-off (rel L2 <= 1e-9), far tighter than the GPU fp32 gate."""
import numpy as np
import pytest

import hostcheck as H
import pyoracle as O
from helpers import random_block, rel_l2
from paper_2412_12089_b200.losses import loss_and_dobs

pytestmark = pytest.mark.skipif(not O.have_ref(), reason="needs oracle/_ref (reference tape)")

G16 = {"dims": (16, 16, 16), "dx": 1 / 16, "dt": 2e-4, "gravity": (0, 0, -9.8), "boundary": "slip"}
FLUID_LOSS = {"kind": "fluid_move", "target": (0.55, 0.5, 0.2), "spill_half": 0.1, "spill_temp": 0.01,
              "tier_threshold": 0.02, "tier_low": 1.0, "tier_high": 2.0}
CASES = {
    "fcr": ({"kind": "fixed_corotated", "E": 1e4, "nu": 0.3, "rho": 1, "volume": 1e-4}, [], {"kind": "var_z"}, "sticky"),
    "nh_act": ({"kind": "neo_hookean", "E": 3e4, "nu": 0.3, "rho": 1, "volume": 1e-4, "act_strength": 1e4}, [],
               {"kind": "var_z"}, "slip"),
    "ep_yield_cyl": ({"kind": "elastoplastic", "E": 5e3, "nu": 0.2, "rho": 1, "volume": 1e-4, "yield_stress": 20},
                     [{"kind": "cylinder", "normal": (0, 1, 0), "radius": 0.05, "length": 0.3,
                       "center": (0.5031, 0.4987, 0.6029), "velocity": (0.1, 0, -0.3), "omega": (0, 5, 0)}],
                     {"kind": "var_z"}, "slip"),
    "ep_sphere_box_plane": (
        {"kind": "elastoplastic", "E": 5e3, "nu": 0.2, "rho": 1, "volume": 1e-4, "yield_stress": 20, "wide_yield": 1},
        [{"kind": "sphere", "center": (0.5, 0.5, 0.66), "radius": 0.08, "velocity": (0.1, 0, -0.3)},
         {"kind": "box", "center": (0.3513, 0.5021, 0.4987), "half": (0.0511, 0.1013, 0.0493), "velocity": (0.3, 0, 0)},
         {"kind": "plane", "center": (0, 0, 0.42), "normal": (0, 0, 1), "velocity": (0, 0, 0.1)}],
        {"kind": "var_z"}, "slip"),
    "fluid_visc_hollow": (
        {"kind": "fluid", "E": 2e4, "nu": 0.3, "rho": 1000, "volume": 1e-4, "bulk": 2e4, "viscosity": 0.5},
        [{"kind": "hollow_box", "half": (0.1013, 0.0987, 0.1021), "thickness": 0.0911,
          "center": (0.5017, 0.4983, 0.4529), "velocity": (0.2, -0.1, 0.05)}], FLUID_LOSS, "slip"),
}


@pytest.mark.parametrize("name", list(CASES))
def test_hand_adjoint_matches_reference_tape(name):
    law, cols, loss, boundary = CASES[name]
    rng = np.random.default_rng(len(name))
    st = random_block(rng, 64, 0.42, 0.58, groups=2)
    sim = dict(G16, boundary=boundary, mu_b=0.3)
    act = rng.uniform(-1, 1, (2, 2)) if law["kind"] == "neo_hookean" else None
    ref = O.rollout_grad(sim, [law], cols, st, 2, 4, loss, act=act, seg=1)
    hc = H.rollout(O, sim, [law], cols, st, 2, 4, act=act, loss=loss, dobs_fn=lambda o: loss_and_dobs(loss, o)[1])
    assert np.abs(ref["obs"] - hc["obs"]).max() < 1e-12
    for k in ("x", "v", "F", "C", "cvo", "act", "E"):
        r = np.asarray(ref[k])
        if r.size == 0 or np.abs(r).max() == 0:
            continue
        assert rel_l2(hc[k], r) <= 1e-9, (k, rel_l2(hc[k], r))


def test_elastoplastic_case_yields():
    """The ep case must exercise the return map (otherwise its adjoint is untested)."""
    law = CASES["ep_yield_cyl"][0]
    rng = np.random.default_rng(len("ep_yield_cyl"))
    st = random_block(rng, 64, 0.42, 0.58, groups=2)
    cy = law["yield_stress"] / (2 * law["E"] / (2 * 1.2))
    dev = []
    for f in st["F"]:
        s = np.linalg.svd(f.reshape(3, 3), compute_uv=False)
        e = np.log(s)
        dev.append(np.linalg.norm(e - e.mean()))
    assert np.mean(np.array(dev) > cy) > 0.2
