"""One small rollout (fwd+bwd) of a config for ncu captures."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_12089_b200 import api, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--envs", type=int, default=64)
ap.add_argument("--ctrl", type=int, default=1)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
kw = {"n_envs": a.envs}
if a.config != 1:
    kw["n_ctrl"] = a.ctrl
sc = scenes.CONFIGS[a.config](seed=0, **kw)
b = api.from_scene(sc)
for _ in range(a.reps):
    out = api.run_scene(b, sc)
print("loss", float(out["loss"].mean()), "launches", b.launches)
