"""BASELINE-config parity cases shared by the fixture generator
(tests/golden/make_config_golden.py, run where /root/reference exists) and
the GPU tests (tests/test_gpu_config_parity.py).

A case is "cfg<k>_e<env>[_<tag>]": env <env> of config <k> built by scenes.py
from its seed and global env index (an env's inputs do not depend on which
envs share the batch), its state rounded to fp32, one control step at the
config's real substep count and checkpoint interval (cfg1: the whole
50-substep rollout).  The env subset per config is SURVEY 8(d)'s first,
last and two seeded random envs.
"""
from __future__ import annotations

import hashlib

import numpy as np

from helpers import to_f32_state

ENV_SUBSET = {2: [0, 31, 7, 22], 3: [0, 255, 41, 170], 4: [0, 1023, 118, 677]}
GRAD_CASES = ["cfg1_e0", "cfg1_e0_varz", "cfg2_e0", "cfg2_e31", "cfg3_e0", "cfg3_e255", "cfg4_e0", "cfg4_e1023"]


def state_sha(st) -> str:
    h = hashlib.sha256()
    for k in ("x", "v", "F", "C"):
        h.update(np.ascontiguousarray(np.asarray(st[k], np.float32)).tobytes())
    return h.hexdigest()


def config_env(cfg: int, env: int, n_ctrl: int = 1):
    """Scene holding env `env` of config `cfg` (1 env, n_ctrl control steps)."""
    from paper_2412_12089_b200 import scenes
    if cfg == 1:
        return scenes.config1(seed=3)
    if cfg == 2:
        return scenes.config2(seed=0, n_envs=1, env_offset=env, n_ctrl=n_ctrl)
    if cfg == 3:
        return scenes.config3(seed=0, n_envs=1, env_offset=env, n_ctrl=n_ctrl)
    return scenes.config4(seed=0, n_envs=1, env_offset=env, n_ctrl=n_ctrl)


def case_scene(case: str, n_ctrl: int = 1):
    """(scene, fp32-rounded env state, per-env collider specs with per-step
    poses, actions [T, A] or None, loss spec) of a case."""
    parts = case.split("_")
    cfg, env = int(parts[0][3:]), int(parts[1][1:])
    tag = parts[2] if len(parts) > 2 else ""
    sc = config_env(cfg, env, n_ctrl)
    loss = {"kind": "var_z"} if tag == "varz" else sc.loss
    st = to_f32_state(sc.env_state(0))
    cvo, act = sc.cvo_act()
    # the GPU consumes fp32 kinematics and actuation: the oracle gets the
    # identical (fp32-rounded) values
    cvo = np.asarray(cvo, np.float32).astype(np.float64)
    act = np.asarray(act, np.float32).astype(np.float64)
    cols = sc.env_cols(0, cvo) if sc.colliders else []
    a = act[0] if getattr(sc.task, "n_act", 0) else None
    return sc, st, cols, a, loss
