"""Diagnostic: every BASELINE-config parity metric (no asserts), JSON to stdout."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)
import numpy as np
import pyoracle as O
from config_cases import ENV_SUBSET, GRAD_CASES, case_scene
from helpers import cosine, field_rel, rel_l2, to_f32_state
from paper_2412_12089_b200 import api
from paper_2412_12089_b200.losses import loss_and_dobs

rep = {}
def batch(sc, E, n_sub, max_steps, ck=None):
    ls = sc.loss
    return api.MpmBatch(sc.sim, sc.materials, sc.colliders, E, sc.n_per_env, n_sub, max_steps,
                        num_groups=getattr(sc.task, "n_act", 0), checkpoint_every=sc.checkpoint_every if ck is None else ck,
                        spill_half=ls.get("spill_half", 0.0), spill_temp=ls.get("spill_temp", 0.0))
cvo_row = lambda cols, t: np.stack([np.asarray(c["cvo"])[t] for c in cols]).astype(np.float32)
which = sys.argv[1:] or ["sub", "end", "grad"]
only = os.environ.get("ONLY")  # e.g. "4:677,3:255"
sel = {int(a): [int(b)] for a, b in (x.split(":") for x in only.split(","))} if only else None
for cfg in (2, 3, 4):
    if "sub" not in which: break
    if sel is not None and cfg not in sel: continue
    for e in (sel[cfg] if sel else ENV_SUBSET[cfg][:2]):
        sc, st, cols, act, _ = case_scene("cfg%d_e%d" % (cfg, e))
        b = batch(sc, 1, 1, 1, ck=0)
        cur = st
        worst = {k: 0.0 for k in "xvFC"}
        for q in range(sc.n_sub):
            s32 = to_f32_state(cur)
            c1 = [dict(c, cvo=np.asarray(c["cvo"])[:1]) for c in cols]
            a1 = None if act is None else act[:1]
            ref_f32in, _, _ = O.rollout(sc.sim, sc.materials, c1, s32, 1, 1, act=a1)
            b.set_state(s32["x"][None], s32["v"][None], s32["F"][None], s32["C"][None], sc.material, sc.group)
            b.step(cvo_row(cols, 0)[None] if b.K else None, a1.astype(np.float32) if a1 is not None else None)
            g = b.get_state()
            for k in "xvFC":
                r = field_rel(g[k][0], ref_f32in[k], sc.n_per_env)
                worst[k] = max(worst[k], r)
                if r > 1e-5:
                    d = np.linalg.norm(g[k][0].reshape(sc.n_per_env, -1) - ref_f32in[k].reshape(sc.n_per_env, -1), axis=1)
                    o = np.argsort(-d)[:5]
                    print(json.dumps({"over": [cfg, e, q, k, r, float(np.linalg.norm(ref_f32in[k])),
                                               [int(i) for i in o], [float(d[i]) for i in o],
                                               [list(map(float, s32["x"][i])) for i in o[:3]],
                                               [list(map(float, ref_f32in[k].reshape(sc.n_per_env, -1)[i])) for i in o[:2]],
                                               [list(map(float, g[k][0].reshape(sc.n_per_env, -1)[i])) for i in o[:2]],
                                               "frac_top5 %.3f" % float(np.sqrt((d[o]**2).sum()) / np.linalg.norm(d))]}), flush=True)
            cur, _, _ = O.rollout(sc.sim, sc.materials, c1, cur, 1, 1, act=a1)
        rep["sub_cfg%d_e%d" % (cfg, e)] = worst
        print(json.dumps({"sub_cfg%d_e%d" % (cfg, e): worst}), flush=True)
        b.close()
for cfg in (2, 3, 4):
    if "end" not in which: break
    for e in ENV_SUBSET[cfg][:2]:
        sc, st, cols, act, loss = case_scene("cfg%d_e%d" % (cfg, e), n_ctrl=2)
        b = batch(sc, 1, sc.n_sub, 2)
        b.set_state(st["x"][None], st["v"][None], st["F"][None], st["C"][None], sc.material, sc.group)
        for t in range(2):
            b.step(cvo_row(cols, t)[None] if b.K else None, act[t:t+1].astype(np.float32) if b.G else None)
        g = b.get_state()
        ref, _, _ = O.rollout(sc.sim, sc.materials, cols, st, 2, sc.n_sub, act=act, loss=loss)
        r = {k: field_rel(g[k][0], ref[k], sc.n_per_env) for k in "xvFC"}
        r.update({"norm_" + k: float(np.linalg.norm(ref[k])) for k in "vC"})
        print(json.dumps({"end_cfg%d_e%d" % (cfg, e): r}), flush=True)
        b.close()
for case in GRAD_CASES:
    if "grad" not in which: break
    fx = np.load(os.path.join(ROOT, "tests", "golden", "%s_grad.npz" % case))
    sc, st, cols, act, loss = case_scene(case)
    b = batch(sc, 1, sc.n_sub, 1)
    b.set_state(st["x"][None], st["v"][None], st["F"][None], st["C"][None], sc.material, sc.group)
    obs = b.step(cvo_row(cols, 0)[None] if b.K else None, act[:1].astype(np.float32) if b.G else None)
    L, dobs = loss_and_dobs(loss, np.transpose(obs[None], (1, 0, 2)))
    g = b.backward(dobs=np.ascontiguousarray(np.transpose(dobs, (1, 0, 2)), dtype=np.float32))
    r = {"loss_rel": abs(L[0] - float(fx["loss"])) / max(1e-30, abs(float(fx["loss"])))}
    for k in "xvFC":
        a, rr = g[k][0].ravel(), fx["g" + k].ravel()
        r[k] = [cosine(a, rr), rel_l2(a, rr), float(np.linalg.norm(rr)), float(np.linalg.norm(a))]
    full_a = np.concatenate([g[k][0].ravel() for k in "xvFC"]); full_r = np.concatenate([fx["g" + k].ravel() for k in "xvFC"])
    r["full"] = [cosine(full_a, full_r), rel_l2(full_a, full_r)]
    full_a = np.concatenate([g[k][0].ravel() for k in "xvC"]); full_r = np.concatenate([fx["g" + k].ravel() for k in "xvC"])
    r["full_noF"] = [cosine(full_a, full_r), rel_l2(full_a, full_r)]
    if b.K: r["cvo"] = [cosine(g["cvo"][:, 0], fx["gcvo"]), rel_l2(g["cvo"][:, 0], fx["gcvo"])]
    if b.G: r["act"] = [cosine(g["act"][:, 0], fx["gact"]), rel_l2(g["act"][:, 0], fx["gact"])]
    r["E"] = [float(g["E"][0, 0]), float(fx["gE"][0])]
    print(json.dumps({case: r}), flush=True)
    b.close()
