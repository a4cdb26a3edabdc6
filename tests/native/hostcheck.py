"""TEST INFRASTRUCTURE ONLY: ctypes binding for tests/native/libadjcheck.so
(fp64 host instantiation of the device physics + hand-written adjoint)."""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libadjcheck.so")


def build():
    src = os.path.join(HERE, "adjoint_check.cpp")
    deps = [src] + [os.path.join(HERE, "..", "..", "paper_2412_12089_b200", "csrc", f)
                    for f in ("dm_math.cuh", "dm_physics.cuh", "dm_transfer.cuh")]
    if not os.path.exists(SO) or os.path.getmtime(SO) < max(os.path.getmtime(d) for d in deps):
        subprocess.check_call(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                               "-o", SO, src])
    return C.CDLL(SO)


def rollout(O, sim, mats, cols, state, n_ctrl, n_sub, act=None, loss=None, dobs_fn=None):
    """Returns obs (and gradients when dobs_fn maps obs -> dobs)."""
    L = build()
    n, x, v, F, Cm, mat, grp = O._state_arrays(state)
    cvo = O.cvo_from_cols(cols, n_ctrl)
    nact = 0 if act is None else np.asarray(act).shape[-1]
    a = np.ascontiguousarray(np.zeros((n_ctrl, 1)) if act is None else np.asarray(act, dtype=np.float64).reshape(n_ctrl, nact))
    obs = np.zeros((n_ctrl, 7))
    half = loss.get("spill_half", 0.0) if loss else 0.0
    temp = loss.get("spill_temp", 0.0) if loss else 0.0
    err = C.create_string_buffer(512)
    g = [np.zeros((n, 3)), np.zeros((n, 3)), np.zeros((n, 9)), np.zeros((n, 9))]
    gcvo = np.zeros_like(cvo)
    gact = np.zeros_like(a)
    gE = np.zeros(max(1, len(mats)))
    args = [C.byref(O.make_sim(sim)), O.make_mats(mats), len(mats), O.make_cols(cols), len(cols), O._dp(cvo), O._dp(a),
            nact, n, O._dp(x), O._dp(v), O._dp(F), O._dp(Cm), O._ip(mat), O._ip(grp), n_ctrl, n_sub,
            C.c_double(half), C.c_double(temp), O._dp(obs)]
    rc = L.hc_rollout(*args, None, *(O._dp(q) for q in g), O._dp(gcvo), O._dp(gact), O._dp(gE), err, 512)
    if rc != 0:
        raise RuntimeError(err.value.decode())
    if dobs_fn is None:
        return obs
    dobs = np.ascontiguousarray(dobs_fn(obs))
    rc = L.hc_rollout(*args, O._dp(dobs), *(O._dp(q) for q in g), O._dp(gcvo), O._dp(gact), O._dp(gE), err, 512)
    if rc != 0:
        raise RuntimeError(err.value.decode())
    return {"obs": obs, "x": g[0], "v": g[1], "F": g[2], "C": g[3], "cvo": gcvo[:, :len(cols)], "act": gact[:, :nact],
            "E": gE[:len(mats)]}


def build_cpp_smoke():
    """Builds tests/native/cpp_adapter_smoke against the in-tree libdiffmpm.so."""
    root = os.path.dirname(os.path.dirname(HERE))
    exe = os.path.join(HERE, "cpp_adapter_smoke")
    src = os.path.join(HERE, "cpp_adapter_smoke.cpp")
    libdir = os.path.join(root, "paper_2412_12089_b200")
    deps = [src, os.path.join(root, "include", "diffmpm", "mpm_batch.hpp"), os.path.join(root, "include", "diffmpm.h")]
    if not os.path.exists(exe) or os.path.getmtime(exe) < max(os.path.getmtime(d) for d in deps):
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-I", os.path.join(root, "include"), "-o", exe, src,
                               "-L", libdir, "-ldiffmpm", f"-Wl,-rpath,{libdir}", "-Wl,-rpath,$ORIGIN/../../paper_2412_12089_b200"])
    return exe
