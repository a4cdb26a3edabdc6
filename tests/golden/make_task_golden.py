"""Generates tests/golden/task_{fluid_move,roll_flat}.npz from the reference's
own tasks (tasks.hpp MiniFluidMove / MiniRollFlat compiled unchanged into
oracle/_ref/libref.so) stepped as EnvBatch does (env.hpp:55-117):

  rewards [T][E], obs [T+1][E][od]   the double forward with the given actions
  dact_tape [T][E][A]                dL/dactions on the reference tape
                                     (step_checkpointed restated; MiniFluidMove:
                                     no SVD on its path)
  dact_fd  [T][E][A]                 central differences of the double forward
                                     (MiniRollFlat's elastoplastic law takes
                                     Tape::svd3x3, whose clamped adjoint is off
                                     at repeated singular values -- F = I)
  for L = sum w_r * rewards + sum_{t>=1} w_o * obs, episode_len 4 < T = 6 so
  the rollout crosses an auto-reset.  Run here (the reference is not on the
  GPU box):  python tests/golden/make_task_golden.py
"""
import os
import sys
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as O  # noqa: E402

T = 6
CASES = {"fluid_move": (0, 3, 7, {"substeps": 40}), "roll_flat": (1, 2, 11, {"substeps": 20})}


def base_cfg(over):
    c = dict(grid_n=20, ppc=8, dt=0.02, substeps=40, episode_len=4, cloud_k=16, container_half=0.1, fill=0.08,
             speed=0.25, start_x=0.35, start_y=0.5, target_x=0.65, target_y=0.5, spill_temp=0.01, block_size=0.2,
             block_height=0.1, roller_radius=0.07, roller_speed=0.25, h_flat=0.1, youngs=1e5, yield_stress=2e3)
    c.update(over)
    return c


def inputs(name):
    kind, E, seed, over = CASES[name]
    cfg = base_cfg(over)
    od, A = O.ref_task_dims(kind, cfg)
    rng = np.random.default_rng(seed)
    a = rng.uniform(-0.9, 0.9, (T, E, A))
    w_r = rng.standard_normal((T, E))
    w_o = rng.standard_normal((T + 1, E, od)) * 0.1
    w_o[0] = 0.0  # the reset observation carries no gradient
    return kind, E, seed, cfg, a, w_r, w_o


def loss(args):
    name, a = args
    kind, E, seed, cfg, _, w_r, w_o = inputs(name)
    r, o, _ = O.ref_task_rollout(kind, cfg, E, seed, 0, a)
    return float((w_r * r).sum() + (w_o * o).sum())


def make(name):
    kind, E, seed, cfg, a, w_r, w_o = inputs(name)
    r, o, d_tape = O.ref_task_rollout(kind, cfg, E, seed, 0, a, w_r=w_r, w_o=w_o)
    jobs, idx = [], []
    h = 1e-6
    for t in range(T):
        for e in range(E):
            for k in range(a.shape[2]):
                for sg in (1, -1):
                    ap = a.copy()
                    ap[t, e, k] += sg * h
                    jobs.append((name, ap))
                idx.append((t, e, k))
    with Pool(min(8, os.cpu_count() or 1)) as p:
        L = p.map(loss, jobs)
    d_fd = np.zeros_like(a)
    for j, (t, e, k) in enumerate(idx):
        d_fd[t, e, k] = (L[2 * j] - L[2 * j + 1]) / (2 * h)
    np.savez_compressed(os.path.join(HERE, "task_%s.npz" % name), kind=kind, n_envs=E, seed=seed, T=T,
                        cfg_keys=np.array(list(cfg)), cfg_vals=np.array([float(v) for v in cfg.values()]),
                        actions=a, w_r=w_r, w_o=w_o, rewards=r, obs=o, dact_tape=d_tape, dact_fd=d_fd)
    c = float(d_fd.ravel() @ d_tape.ravel() / (np.linalg.norm(d_fd) * np.linalg.norm(d_tape)))
    print(name, "tape vs FD: cos %.6f rel %.2e" % (c, np.linalg.norm(d_fd - d_tape) / np.linalg.norm(d_fd)), flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:] or list(CASES):
        make(n)
