"""Generates tests/golden/oracle_golden.npz from the reference build
(oracle/_ref/libref.so = /root/reference headers compiled unchanged).
Run here (the reference is not on the GPU box): python tests/golden/make_golden.py

Contents:
  in_x/v/F/C, ref_x/v/F/C : 8 substeps of the reference mpm_step<double>
                            (elastoplastic, moving sphere, slip boundary)
  bin_x, bin_keys, bin_perm: fp32 positions, (4^3 tile, cell) keys and stable
                            permutation computed independently in numpy
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as O  # noqa: E402

rng = np.random.default_rng(20241217)
n = 64
st = {"x": 0.4 + 0.2 * rng.random((n, 3)), "v": 0.3 * rng.standard_normal((n, 3)),
      "F": np.tile(np.eye(3).ravel(), (n, 1)) + 0.02 * rng.standard_normal((n, 9)), "C": 0.5 * rng.standard_normal((n, 9))}
sim = {"dims": (16, 16, 16), "dx": 1 / 16, "dt": 1e-3, "gravity": (0, 0, -9.81), "boundary": "slip"}
mats = [{"kind": "elastoplastic", "E": 1e4, "nu": 0.3, "rho": 1000, "volume": 1e-5, "yield_stress": 50}]
cols = [{"kind": "sphere", "center": (0.5, 0.5, 0.75), "radius": 0.1, "velocity": (0.1, 0, -0.2)}]
ref, _ = O.ref_rollout(sim, mats, cols, st, 8)

bx = (0.1 + 0.8 * rng.random((2000, 3))).astype(np.float32)
g = np.floor((bx * np.float32(48.0)).astype(np.float32) - np.float32(0.5)).astype(np.int64)
keys = ((((g[:, 0] >> 2) * 12 + (g[:, 1] >> 2)) * 12 + (g[:, 2] >> 2)) * 64 +
        ((g[:, 0] & 3) * 4 + (g[:, 1] & 3)) * 4 + (g[:, 2] & 3)).astype(np.int32)
perm = np.argsort(keys, kind="stable").astype(np.int32)
np.savez_compressed(os.path.join(HERE, "oracle_golden.npz"),
                    **{"in_" + k: st[k] for k in "xvFC"}, **{"ref_" + k: ref[k] for k in "xvFC"},
                    bin_x=bx, bin_keys=keys, bin_perm=perm)
print("wrote oracle_golden.npz")
