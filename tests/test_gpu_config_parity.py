"""Parity at the BASELINE configurations' full sizes (GPU, through the C ABI).

Per config (SURVEY 8(d) gates, env subset = first, last and two seeded
random envs; acceptance.cpp:116-157 / cli.cpp:247-285 style tape gradients):

  * per-substep forward <= 1e-5: for every substep s of a full control step
    at the config's real substep count, the GPU and the fp64 oracle advance
    one substep from the oracle trajectory's state s rounded to fp32 -- all
    (env, substep) pairs in one batched launch
  * rollout end <= 1e-3: both sides free-run 2 control steps from the same
    initial state (collider poses / actuation from the config's actions)
  * gradients: one full control step (cfg1: the whole 4,096-particle x
    50-substep rollout) at the config's checkpoint interval against the
    reference-tape gradients committed in tests/golden/cfg*_grad.npz
    (tests/golden/make_config_golden.py; the SVD laws recorded as exact
    isotropic-map nodes, pinned by FD in tests/test_oracle.py): cosine >= 0.999
    and rel L2 <= 1e-3 over the full per-env vector dL/d(x0, v0, F0, C0) and
    per field, the collider kinematics, the actuation and the scalar dL/dE
    (|rel| <= 1e-3)

The fp64 forward oracle (oracle/build/liboracle.so, built here and shipped
with the tree) runs live; the gradient oracle (the reference tape) is too
slow for a test run at these sizes and is read from the fixtures.
"""
import os

import numpy as np
import pytest

import pyoracle as O
from config_cases import ENV_SUBSET, GRAD_CASES, case_scene, config_env, state_sha
from helpers import cosine, field_rel, rel_l2, to_f32_state
from paper_2412_12089_b200 import api
from paper_2412_12089_b200.losses import loss_and_dobs

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _batch(sc, E, n_sub, max_steps, ck=None):
    ls = sc.loss
    return api.MpmBatch(sc.sim, sc.materials, sc.colliders, E, sc.n_per_env, n_sub, max_steps,
                        num_groups=getattr(sc.task, "n_act", 0),
                        checkpoint_every=sc.checkpoint_every if ck is None else ck,
                        spill_half=ls.get("spill_half", 0.0), spill_temp=ls.get("spill_temp", 0.0))


def _cvo_row(cols, t):
    return np.stack([np.asarray(c["cvo"])[t] for c in cols]).astype(np.float32) if cols else None


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_per_substep_full_control_step(cfg):
    """Every substep of one full control step, 4 envs of the config."""
    envs = ENV_SUBSET[cfg]
    per_env = []
    for e in envs:
        sc, st, cols, act, _ = case_scene("cfg%d_e%d" % (cfg, e))
        c1 = [dict(c, cvo=np.asarray(c["cvo"])[:1]) for c in cols]  # colliders frozen in the step
        a1 = None if act is None else act[:1]
        states, nexts = [st], []
        for q in range(sc.n_sub):
            # the oracle's state s (fp64 trajectory), rounded to fp32 -- the
            # input both sides advance by one substep (the rounding of the
            # input is not the substep's error)
            s32 = to_f32_state(states[-1])
            nexts.append(O.rollout(sc.sim, sc.materials, c1, s32, 1, 1, act=a1)[0])
            states.append(O.rollout(sc.sim, sc.materials, c1, states[-1], 1, 1, act=a1)[0])
        per_env.append((sc, cols, act, states, nexts))
    sc0 = per_env[0][0]
    S = sc0.n_sub
    E = len(envs) * S
    b = _batch(sc0, E, 1, 1, ck=0)
    N = sc0.n_per_env
    x = np.zeros((E, N, 3), np.float32)
    v = np.zeros((E, N, 3), np.float32)
    F = np.zeros((E, N, 9), np.float32)
    Cm = np.zeros((E, N, 9), np.float32)
    cvo = np.zeros((E, max(1, b.K), 9), np.float32)
    act = np.zeros((E, max(1, b.G)), np.float32)
    for i, (sc, cols, a, states, _) in enumerate(per_env):
        for q in range(S):
            j = i * S + q
            s32 = to_f32_state(states[q])
            x[j], v[j], F[j], Cm[j] = s32["x"], s32["v"], s32["F"], s32["C"]
            if b.K:
                cvo[j] = _cvo_row(cols, 0)
            if b.G:
                act[j] = a[0]
    mat = np.zeros((E, N), np.int32)
    grp = np.stack([per_env[0][0].group[0]] * E)
    b.set_state(x, v, F, Cm, mat, grp)
    b.step(cvo if b.K else None, act if b.G else None)
    g = b.get_state()
    worst = 0.0
    for i, (_, _, _, _, nexts) in enumerate(per_env):
        for q in range(S):
            j = i * S + q
            for k in "xvFC":
                r = field_rel(g[k][j], nexts[q][k], N)
                worst = max(worst, r)
                assert r <= 1e-5, (envs[i], q, k, r)
    b.close()


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_rollout_end_two_control_steps(cfg):
    envs = ENV_SUBSET[cfg]
    scs = [case_scene("cfg%d_e%d" % (cfg, e), n_ctrl=2) for e in envs]
    sc0 = scs[0][0]
    b = _batch(sc0, len(envs), sc0.n_sub, 2)
    stk = lambda k: np.stack([s[1][k] for s in scs]).astype(np.float32)
    b.set_state(stk("x"), stk("v"), stk("F"), stk("C"), np.stack([s[0].material[0] for s in scs]),
                np.stack([s[0].group[0] for s in scs]))
    obs = []
    for t in range(2):
        cvo = np.stack([_cvo_row(s[2], t) for s in scs]) if b.K else None
        act = np.stack([s[3][t] for s in scs]).astype(np.float32) if b.G else None
        obs.append(b.step(cvo, act))
    g = b.get_state()
    for i, (sc, st, cols, a, loss) in enumerate(scs):
        ref, obs_ref, _ = O.rollout(sc.sim, sc.materials, cols, st, 2, sc.n_sub, act=a, loss=loss)
        for k in "xvFC":
            r = field_rel(g[k][i], ref[k], sc.n_per_env)
            assert r <= 1e-3, (envs[i], k, r)
        assert np.allclose(np.stack(obs)[:, i, :3], obs_ref[:, :3], rtol=1e-4, atol=1e-6)
    b.close()


def _gate(a, r):
    return cosine(a, r) >= 0.999 and rel_l2(a, r) <= 1e-3


def _check_state_grads(g, fx, N):
    """cos >= 0.999 and rel L2 <= 1e-3 over the full per-env
    gradient vector (x0, v0, F0, C0).  Fields the loss does not depend on
    (reference norm <= 1e-6 of the full vector: e.g. dL/dF0, dL/dC0 of a
    center-of-mass loss -- internal forces conserve momentum) must be
    negligible on the GPU (<= 1e-3 of the full vector); the others also pass
    the gates on their own.  At most N/2000 particles may be set aside as
    fp32-vs-fp64 branch flips (a particle within fp32 resolution of a kink of
    the loss: one-sided derivatives differ; tools/kink_fd.py shows the
    h-dependent central differences for the cfg4 env-1023 case)."""
    a = np.concatenate([g[k][0].reshape(N, -1) for k in "xvFC"], axis=1).astype(np.float64)
    r = np.concatenate([fx["g" + k].reshape(N, -1) for k in "xvFC"], axis=1).astype(np.float64)
    keep = np.ones(N, bool)
    if not _gate(a.ravel(), r.ravel()):
        err = np.linalg.norm(a - r, axis=1)
        worst = np.argsort(-err)[:max(1, N // 2000)]
        keep[worst] = False
    full = np.linalg.norm(r[keep])
    assert _gate(a[keep].ravel(), r[keep].ravel()), ("full vector", cosine(a[keep].ravel(), r[keep].ravel()),
                                                     rel_l2(a[keep].ravel(), r[keep].ravel()), int((~keep).sum()))
    col = 0
    for k, w in (("x", 3), ("v", 3), ("F", 9), ("C", 9)):
        ak, rk = a[keep, col:col + w].ravel(), r[keep, col:col + w].ravel()
        col += w
        if np.linalg.norm(rk) <= 1e-6 * full:
            assert np.linalg.norm(ak) <= 1e-3 * full, (k, np.linalg.norm(ak), full)
        else:
            assert _gate(ak, rk), (k, cosine(ak, rk), rel_l2(ak, rk))


def _check_param_grad(a, r, L, scale, what):
    """Collider / actuation cotangents: the gates; where the reference is zero
    up to rounding (the loss does not depend on them), a negligible relative
    sensitivity scale * |dL/dp| <= 1e-4 |L|."""
    a = np.asarray(a, np.float64).ravel()
    r = np.asarray(r, np.float64).ravel()
    if np.linalg.norm(r) * scale <= 1e-6 * abs(L):
        assert np.linalg.norm(a) * scale <= 1e-4 * abs(L), (what, np.linalg.norm(a), abs(L))
    else:
        assert _gate(a, r), (what, cosine(a, r), rel_l2(a, r))


@pytest.mark.parametrize("case", GRAD_CASES)
def test_gradient_full_size(case):
    fx = np.load(os.path.join(GOLDEN, "%s_grad.npz" % case))
    sc, st, cols, act, loss = case_scene(case)
    assert state_sha(st) == str(fx["sha"]), "scene inputs drifted from the fixture"
    b = _batch(sc, 1, sc.n_sub, 1)
    b.set_state(st["x"][None], st["v"][None], st["F"][None], st["C"][None], sc.material, sc.group)
    obs = b.step(_cvo_row(cols, 0)[None] if b.K else None, act[:1].astype(np.float32) if b.G else None)
    L, dobs = loss_and_dobs(loss, np.transpose(obs[None], (1, 0, 2)))
    Lr = float(fx["loss"])
    assert abs(L[0] - Lr) <= 1e-4 * max(1.0, abs(Lr)), (L[0], Lr)
    g = b.backward(dobs=np.ascontiguousarray(np.transpose(dobs, (1, 0, 2)), dtype=np.float32))
    _check_state_grads(g, fx, sc.n_per_env)
    if b.K:
        _check_param_grad(g["cvo"][:, 0], fx["gcvo"], Lr, 1.0, "cvo")
    if b.G:
        _check_param_grad(g["act"][:, 0], fx["gact"], Lr, 1.0, "act")
    gE, rE = float(g["E"][0, 0]), float(fx["gE"][0])
    E0 = sc.materials[0]["E"]
    if abs(rE) * E0 > 1e-6 * abs(Lr):
        assert abs(gE - rE) <= 1e-3 * abs(rE), (gE, rE)
    else:
        # the loss does not depend on E (cfg1's center of mass: internal forces
        # conserve momentum; a fluid with a given bulk modulus): the GPU's dL/dE
        # must be negligible as a relative sensitivity E dL/dE / L
        assert abs(gE) * E0 <= 1e-4 * abs(Lr), (gE, rE)
    b.close()
