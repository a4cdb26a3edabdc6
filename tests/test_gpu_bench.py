"""GPU: the bench.py contract on a small workload -- one JSON line with the
driver's keys, single rank and two ranks (torchrun, gloo for the timing
reduction, both ranks on cuda:0 with independent env partitions)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"}


def _line(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_bench_single_rank():
    r = subprocess.run([sys.executable, "bench.py", "--envs", "8", "--ctrl", "1", "--steps", "1", "--warmup", "1",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert KEYS <= set(d), KEYS - set(d)
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["scaling"] == "strong" and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert 0 < d["roofline"]["frac"] < 1


@pytest.mark.parametrize("weak", [False, True])
def test_bench_two_ranks(weak):
    """Default: BASELINE's envs split across the ranks (strong); --weak: every
    rank simulates them."""
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(29533 + int(weak)), "bench.py", "--gpus",
                        "2", "--envs", "8", "--ctrl", "1", "--steps", "1", "--warmup", "1", "--no-e2e",
                        "--no-cpu-baseline"] + (["--weak"] if weak else []),
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["scaling"] == ("weak" if weak else "strong")
    assert d["config"]["envs"] == (16 if weak else 8)
    assert d["value"] > 0
