"""Does a small batch leave the GPU idle enough that two independent halves
on two streams finish sooner than the whole batch on one?  (Probe for the
strong-scaling shard: cfg4 at 128 envs.)

usage: python tools/concurrency_probe.py [--envs 128] [--parts 2] [--reps 3]
Prints ms per rollout (fwd+bwd, device path) for 1 context of E envs and for
`parts` contexts of E/parts envs driven concurrently from host threads."""
import argparse
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_12089_b200 import api, scenes  # noqa: E402
from paper_2412_12089_b200.losses import loss_and_dobs_torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--envs", type=int, default=128)
ap.add_argument("--parts", type=int, default=2)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
dev = torch.device("cuda", 0)


def make(n_envs, env_offset):
    sc = scenes.CONFIGS[a.config](seed=0, n_envs=n_envs, env_offset=env_offset)
    b = api.from_scene(sc)
    E, N, T = sc.n_envs, sc.n_per_env, sc.n_ctrl
    K, G = b.K, b.G
    cvo, act = sc.cvo_act()
    f32 = lambda x: torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32), device=dev)
    x0, v0, F0, C0 = f32(sc.x), f32(sc.v), f32(sc.F), f32(sc.C)
    mat = torch.as_tensor(sc.material, dtype=torch.int32, device=dev)
    grp = torch.as_tensor(sc.group, dtype=torch.int32, device=dev)
    cvo_d = f32(np.transpose(cvo[:, :, :max(K, 1)], (1, 0, 2, 3))) if K else None
    act_d = f32(np.transpose(act[:, :, :max(G, 1)], (1, 0, 2))) if G else None
    obs_d = torch.zeros((T, E, 7), dtype=torch.float32, device=dev)
    out = {"x": torch.empty((E, N, 3), device=dev), "v": torch.empty((E, N, 3), device=dev),
           "F": torch.empty((E, N, 9), device=dev), "C": torch.empty((E, N, 9), device=dev),
           "cvo": torch.empty((T, E, max(K, 1), 9), device=dev) if K else None,
           "act": torch.empty((T, E, max(G, 1)), device=dev) if G else None,
           "E": torch.empty((E, b.n_materials), dtype=torch.float64, device=dev)}
    stream = torch.cuda.ExternalStream(b.stream_ptr, device=dev)

    def roll():
        with torch.cuda.stream(stream):
            b.set_state(x0, v0, F0, C0, mat, grp)
            for t in range(T):
                b.step(None if cvo_d is None else cvo_d[t], None if act_d is None else act_d[t], obs_d[t])
            _, dobs = loss_and_dobs_torch(sc.loss, obs_d.transpose(0, 1))
            b.backward(dobs=dobs.transpose(0, 1).contiguous(), out=out)
        stream.synchronize()
    return roll, b


def timed(rolls):
    for r in rolls:  # warm-up
        r()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.reps):
        if len(rolls) == 1:
            rolls[0]()
        else:
            th = [threading.Thread(target=r) for r in rolls]
            for x in th:
                x.start()
            for x in th:
                x.join()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / a.reps * 1e3


one, b1 = make(a.envs, 0)
ms1 = timed([one])
b1.close()
del one, b1
torch.cuda.empty_cache()
per = a.envs // a.parts
parts = [make(per, p * per) for p in range(a.parts)]
msp = timed([r for r, _ in parts])
print("one context of %d envs: %.1f ms/rollout; %d concurrent contexts of %d envs: %.1f ms/rollout (%.2fx)" %
      (a.envs, ms1, a.parts, per, msp, ms1 / msp))
