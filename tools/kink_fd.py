"""Diagnostic (CPU, needs the oracle): central differences of the fp64
forward rollout loss w.r.t. single particle coordinates at several step
sizes.  An h-dependent FD (one-sided derivatives that differ) marks a
particle within fp32 resolution of a kink of the loss, where the fp32 GPU
and the fp64 oracle legitimately take different branches -- the particles
tests/test_gpu_config_parity.py may set aside (<= N/2000).

  python tools/kink_fd.py cfg4_e1023 13899 13400 13401
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)
from multiprocessing import Pool  # noqa: E402

import numpy as np  # noqa: E402
import pyoracle as O  # noqa: E402
from config_cases import case_scene  # noqa: E402

CASE = sys.argv[1] if len(sys.argv) > 1 else "cfg4_e1023"
PARTICLES = [int(a) for a in sys.argv[2:]] or [13899, 13400, 13401]
HS = (1e-5, 1e-6, 1e-7)


def loss(args):
    p, a, h = args
    sc, st, cols, act, ls = case_scene(CASE)
    s = {k: (np.array(v, dtype=np.float64, copy=True) if k in "xvFC" else v) for k, v in st.items()}
    s["x"][p, a] += h
    return O.rollout(sc.sim, sc.materials, cols, s, 1, sc.n_sub, act=act, loss=ls)[2]


if __name__ == "__main__":
    jobs = [(p, a, sg * h) for p in PARTICLES for a in (0, 1, 2) for h in HS for sg in (1, -1)]
    with Pool(min(8, os.cpu_count() or 1)) as pool:
        r = pool.map(loss, jobs)
    i = 0
    for p in PARTICLES:
        for a in (0, 1, 2):
            fds = []
            for h in HS:
                fds.append((r[i] - r[i + 1]) / (2 * h))
                i += 2
            spread = (max(fds) - min(fds)) / max(abs(np.mean(fds)), 1e-30)
            print("particle %d axis %d  FD(h=%s) = %s  spread %.2e%s" % (
                p, a, "/".join("%.0e" % h for h in HS), " ".join("%.6e" % f for f in fds), spread,
                "  <- kink" if spread > 1e-2 else ""))
