"""Dumps GPU gradients of the BASELINE-config fixture cases (for FD checks on CPU)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)
import numpy as np
from config_cases import case_scene
from paper_2412_12089_b200 import api
from paper_2412_12089_b200.losses import loss_and_dobs
out = {}
for case in sys.argv[1:]:
    sc, st, cols, act, loss = case_scene(case)
    ls = sc.loss
    b = api.MpmBatch(sc.sim, sc.materials, sc.colliders, 1, sc.n_per_env, sc.n_sub, 1,
                     num_groups=getattr(sc.task, "n_act", 0), checkpoint_every=sc.checkpoint_every,
                     spill_half=ls.get("spill_half", 0.0), spill_temp=ls.get("spill_temp", 0.0))
    b.set_state(st["x"][None], st["v"][None], st["F"][None], st["C"][None], sc.material, sc.group)
    cv = np.stack([np.asarray(c["cvo"])[0] for c in cols]).astype(np.float32)[None] if cols else None
    obs = b.step(cv, act[:1].astype(np.float32) if b.G else None)
    L, dobs = loss_and_dobs(loss, np.transpose(obs[None], (1, 0, 2)))
    g = b.backward(dobs=np.ascontiguousarray(np.transpose(dobs, (1, 0, 2)), dtype=np.float32))
    for k in "xvFC":
        out[case + "_" + k] = g[k][0]
    out[case + "_L"] = L
    b.close()
np.savez(os.path.join(ROOT, "gpurun_out", "gpu_grads.npz"), **out)
