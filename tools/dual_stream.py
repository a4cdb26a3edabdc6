"""Experiment: env partitions on separate contexts (separate CUDA streams)
driven from host threads, vs one context with all envs (cfg4, device path as
in bench.py)."""
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_12089_b200 import api, scenes  # noqa: E402
from paper_2412_12089_b200.losses import loss_and_dobs_torch  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ctrl = int(sys.argv[2]) if len(sys.argv) > 2 else 2
parts = int(sys.argv[3]) if len(sys.argv) > 3 else 2
dev = torch.device("cuda", 0)


class Runner:
    def __init__(self, sc):
        self.sc = sc
        self.b = api.from_scene(sc)
        f32 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32), device=dev)
        cvo, act = sc.cvo_act()
        K = self.b.K
        self.x0, self.v0, self.F0, self.C0 = f32(sc.x), f32(sc.v), f32(sc.F), f32(sc.C)
        self.mat = torch.as_tensor(sc.material, dtype=torch.int32, device=dev)
        self.grp = torch.as_tensor(sc.group, dtype=torch.int32, device=dev)
        self.cvo = f32(np.transpose(cvo[:, :, :max(K, 1)], (1, 0, 2, 3)))
        T, En, N = sc.n_ctrl, sc.n_envs, sc.n_per_env
        self.obs = torch.zeros((T, En, 7), dtype=torch.float32, device=dev)
        self.out = {"x": torch.empty((En, N, 3), device=dev), "v": torch.empty((En, N, 3), device=dev),
                    "F": torch.empty((En, N, 9), device=dev), "C": torch.empty((En, N, 9), device=dev),
                    "cvo": torch.empty((T, En, max(K, 1), 9), device=dev), "act": None,
                    "E": torch.empty((En, self.b.n_materials), dtype=torch.float64, device=dev)}
        self.stream = torch.cuda.ExternalStream(self.b.stream_ptr, device=dev)

    def run(self, n=1):
        for _ in range(n):
            self.b.set_state(self.x0, self.v0, self.F0, self.C0, self.mat, self.grp)
            for t in range(self.sc.n_ctrl):
                self.b.step(self.cvo[t], None, self.obs[t])
            with torch.cuda.stream(self.stream):
                _, dobs = loss_and_dobs_torch(self.sc.loss, self.obs.transpose(0, 1))
                d = dobs.transpose(0, 1).contiguous()
            self.b.backward(dobs=d, out=self.out)
        torch.cuda.synchronize()


full = scenes.config4(seed=0, n_envs=E, n_ctrl=ctrl)
units = E * full.n_per_env * ctrl * full.n_sub
r = Runner(full)
r.run(1)
t0 = time.perf_counter()
r.run(2)
print("single ctx   : %.3e particle-substeps/s" % (2 * units / (time.perf_counter() - t0)), flush=True)
r.b.close()
del r
torch.cuda.empty_cache()
rs = [Runner(scenes.config4(seed=0, n_envs=E // parts, env_offset=p * (E // parts), n_ctrl=ctrl)) for p in range(parts)]
for q in rs:
    q.run(1)
t0 = time.perf_counter()
for q in rs:
    q.run(2)
print("%d ctx serial : %.3e" % (parts, 2 * units / (time.perf_counter() - t0)), flush=True)
t0 = time.perf_counter()
th = [threading.Thread(target=q.run, args=(2,)) for q in rs]
for t in th:
    t.start()
for t in th:
    t.join()
print("%d ctx threads: %.3e" % (parts, 2 * units / (time.perf_counter() - t0)), flush=True)
