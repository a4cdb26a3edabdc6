import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2412_12089_b200 import api, scenes
for envs, ctrl in [(2, 2), (2, 32), (32, 4)]:
    sc = scenes.config2(seed=0, n_envs=envs, n_ctrl=ctrl)
    b = api.from_scene(sc)
    try:
        out = api.run_scene(b, sc, want_grad=False)
        print(envs, ctrl, "fwd ok", out["obs"][-1, 0, :3])
        out = api.run_scene(b, sc, want_grad=True)
        print(envs, ctrl, "fwd+bwd ok", float(out["loss"].mean()))
    except Exception as e:
        print(envs, ctrl, "ERR", e)
        break
