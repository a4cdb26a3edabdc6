#!/usr/bin/env python
"""Benchmark: batched differentiable MLS-MPM, forward + backward.

Metric (BASELINE.json): particle-substeps/s of forward + full adjoint over a
checkpointed substep tape.  Default workload = config 4 (FluidMove-like:
1,024 envs x 16,384 particles, 48^3 grid, 16 control steps x 32 substeps),
the configuration BASELINE.json shards over 1/2/4/8 GPUs.  Envs are
independent partitions (no simulator collective): by default the config's
1,024 envs are split across the ranks (strong scaling, BASELINE's "sharded
over 1/2/4/8 GPUs"; rank r owns global envs [r E/N, (r+1) E/N)); `--weak`
gives every rank the config's full env count instead.

One step = one whole rollout: set the initial state, 16 recorded control
steps (512 substeps), loss over the per-step observables, backward through
all 512 substeps (per-control-step recompute segments, algo.hpp:79-104)
down to the initial state, collider kinematics and Young's modulus.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`value`  : device-resident inputs (torch CUDA tensors through the *_device ABI).
`e2e`    : the same rollout through the host-pointer C ABI from pinned host
           memory, H2D of the initial state / per-step kinematics / dobs and
           D2H of observations and all cotangents inside the timed region.
`--impl reference`: the reference's own CPU implementation
           (oracle/_ref/libref.so = /root/reference headers compiled
           unchanged: mpm_step<Value> + Tape with per-substep checkpoint
           segments) on a bounded sample of the same workload, all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-substeps/s fwd+bwd"
UNIT = "particle-substeps/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", type=int, default=4)
    p.add_argument("--envs", type=int, default=0, help="override total envs (default: the config's)")
    p.add_argument("--ctrl", type=int, default=0, help="override control steps")
    p.add_argument("--checkpoint-every", type=int, default=-1)
    p.add_argument("--weak", action="store_true", help="every rank simulates the config's envs (default: split them)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--profile-out", default="")
    return p.parse_args()


# ---------------- distributed plumbing ----------------

def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def init_dist(world, local):
    if world <= 1:
        return None
    import torch
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    # BENCH_DIST_BACKEND=gloo lets the multi-rank path run with several ranks
    # on one device (tests only; the timing reduction is a scalar all-reduce)
    backend = os.environ.get("BENCH_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
    if backend == "nccl":
        torch.cuda.set_device(local)
    dist.init_process_group(backend)
    return dist


def max_over_ranks(dist, value: float) -> float:
    if dist is None:
        return value
    import torch
    on_gpu = torch.cuda.is_available() and dist.get_backend() == "nccl"
    t = torch.tensor([value], dtype=torch.float64, device="cuda" if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ---------------- clocks ----------------

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([c.strip() for c in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------- reference CPU arm ----------------

def reference_sample(scene, n_threads: int, n_sub: int = 1):
    """The reference's own CPU path (mpm_step<Value> + Tape, per-substep
    checkpoint segments, restated step_checkpointed) on n_threads envs of the
    scene in parallel (one tape per worker, tape.hpp:78-79).  Fluid law with
    lambda = the config's bulk modulus and the container as plane walls +
    floor (the reference has no hollow-box SDF or viscosity; the
    particle-substep cost is the same transfer/tape work).
    Returns (particle-substeps, wall seconds, sample description)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    mat = dict(scene.materials[0])
    if mat["kind"] == "fluid":
        nu = mat.get("nu", 0.3)
        lam = mat.get("bulk", 0.0) or mat["E"] * nu / ((1 + nu) * (1 - 2 * nu))
        mat = dict(mat, E=lam * (1 + nu) * (1 - 2 * nu) / nu, bulk=0.0, viscosity=0.0)
    elif mat["kind"] not in ("elastoplastic", "fluid"):
        mat = dict(mat, kind="elastoplastic", yield_stress=1e9)
    cvo, _ = scene.cvo_act()
    results = [None] * n_threads
    sim = dict(scene.sim, boundary="slip")

    def work(i):
        e = i % scene.n_envs
        c = cvo[e, 0, 0, 0:3] if scene.colliders else np.array([0.5, 0.5, 0.3])
        h = scene.colliders[0].get("half", (0.15, 0.15, 0.15)) if scene.colliders else (0.15, 0.15, 0.15)
        cols = [{"kind": "plane", "center": (c[0] - h[0], 0, 0), "normal": (1, 0, 0)},
                {"kind": "plane", "center": (c[0] + h[0], 0, 0), "normal": (-1, 0, 0)},
                {"kind": "plane", "center": (0, c[1] - h[1], 0), "normal": (0, 1, 0)},
                {"kind": "plane", "center": (0, c[1] + h[1], 0), "normal": (0, -1, 0)}]
        st = scene.env_state(e)
        t0 = time.perf_counter()
        O.ref_grad(sim, [mat], cols, st, n_sub, (0.55, 0.5, 0.2), seg=1)
        results[i] = time.perf_counter() - t0

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(i,)) for i in range(n_threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    wall = time.perf_counter() - t0
    units = n_threads * scene.n_per_env * n_sub
    desc = (f"{n_threads} env(s) x {scene.n_per_env} particles x {n_sub} substep(s) fwd+bwd, reference "
            f"mpm_step<Value> + Tape (per-substep checkpoint segments), fp64, {n_threads} thread(s)")
    return units, wall, desc


def cpu_info():
    """(usable host threads, CPU model) of this host."""
    try:
        n = len(os.sched_getaffinity(0))
    except Exception:
        n = os.cpu_count() or 1
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return max(1, n), model


def cpu_threads(bytes_per_thread=0):
    """Every host thread, bounded by the memory the per-thread tapes need
    (one reference tape per worker, tape.hpp:78-79)."""
    n, _ = cpu_info()
    if bytes_per_thread > 0:
        try:
            import psutil
            n = max(1, min(n, int(0.8 * psutil.virtual_memory().available // bytes_per_thread)))
        except Exception:
            pass
    return n


def ref_tape_bytes(scene):
    """Peak reference-tape bytes of one worker: ~2,200 nodes x 33 B per
    particle-substep, one substep segment at a time."""
    return int(scene.n_per_env * 2200 * 33 * 1.3)


def run_reference(args, scene, rank, dist):
    if rank != 0:
        return
    nt = cpu_threads(ref_tape_bytes(scene))
    vals = []
    for i in range(args.warmup + args.steps):
        units, wall, desc = reference_sample(scene, nt, 1)
        if i >= args.warmup:
            vals.append(units / wall)
    v = float(np.mean(vals))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * scene.n_per_env * nt / v,
            "higher_is_better": True, "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": scene.name, "sample": desc},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": nt, "kind": "reference", "sample": desc,
                             "host_threads": cpu_info()[0], "cpu_model": cpu_info()[1]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------- our arm ----------------

ALG_BYTES = {  # algorithmic HBM bytes per particle per launch
    "bin": 12, "p2g": 96, "g2p": 48 + 96, "g2p_adj": 48 + 96 + 48, "p2g_adj": 96 + 48 + 96,
}
# grid / grid_adj / env_reduce / obs are per-node or per-env work (reported in kernel_ms_per_step)


def run_ours(args, scene, rank, world, local, dist):
    import torch
    if torch.cuda.device_count() < world:  # several ranks sharing a device (multi-rank test only)
        local = local % max(1, torch.cuda.device_count())
    from paper_2412_12089_b200 import api
    from paper_2412_12089_b200.losses import loss_and_dobs, loss_and_dobs_torch

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    E, N, T, S = scene.n_envs, scene.n_per_env, scene.n_ctrl, scene.n_sub
    ck = scene.checkpoint_every if args.checkpoint_every < 0 else args.checkpoint_every
    batch = api.from_scene(scene, checkpoint_every=ck, device=local)
    K, G = batch.K, batch.G
    cvo, act = scene.cvo_act()
    f32 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32), device=dev)
    x0, v0, F0, C0 = f32(scene.x), f32(scene.v), f32(scene.F), f32(scene.C)
    mat = torch.as_tensor(scene.material, dtype=torch.int32, device=dev)
    grp = torch.as_tensor(scene.group, dtype=torch.int32, device=dev)
    cvo_d = f32(np.transpose(cvo[:, :, :max(K, 1)], (1, 0, 2, 3))) if K else None  # [T,E,K,9]
    act_d = f32(np.transpose(act[:, :, :max(G, 1)], (1, 0, 2))) if G else None      # [T,E,G]
    obs_d = torch.zeros((T, E, 7), dtype=torch.float32, device=dev)
    out = {"x": torch.empty((E, N, 3), device=dev), "v": torch.empty((E, N, 3), device=dev),
           "F": torch.empty((E, N, 9), device=dev), "C": torch.empty((E, N, 9), device=dev),
           "cvo": torch.empty((T, E, max(K, 1), 9), device=dev) if K else None,
           "act": torch.empty((T, E, max(G, 1)), device=dev) if G else None,
           "E": torch.empty((E, batch.n_materials), dtype=torch.float64, device=dev)}
    torch.cuda.synchronize()

    stream = torch.cuda.ExternalStream(batch.stream_ptr, device=dev)

    def rollout_device():
        # the loss reads obs_d and writes dobs: on the context stream, ordered
        # with the simulator's kernels (no host synchronisation in the step)
        with torch.cuda.stream(stream):
            batch.set_state(x0, v0, F0, C0, mat, grp)
            for t in range(T):
                batch.step(None if cvo_d is None else cvo_d[t], None if act_d is None else act_d[t], obs_d[t])
            _, dobs = loss_and_dobs_torch(scene.loss, obs_d.transpose(0, 1))
            batch.backward(dobs=dobs.transpose(0, 1).contiguous(), out=out)

    # host (pinned) buffers for the end-to-end arm
    def pinned(a, dtype=np.float32):
        t = torch.empty(a.shape, dtype=torch.float32 if dtype == np.float32 else torch.int32).pin_memory()
        t.numpy()[...] = a
        return t.numpy()

    hx, hv, hF, hC = (pinned(scene.x), pinned(scene.v), pinned(scene.F), pinned(scene.C))
    hmat, hgrp = pinned(scene.material, np.int32), pinned(scene.group, np.int32)
    hcvo = [np.ascontiguousarray(pinned(cvo[:, t, :K])) for t in range(T)] if K else None
    hact = [np.ascontiguousarray(pinned(act[:, t, :G])) for t in range(T)] if G else None

    # pinned output buffers for the host backward (D2H at full DMA rate)
    hout = {"x": pinned(np.zeros((E, N, 3))), "v": pinned(np.zeros((E, N, 3))), "F": pinned(np.zeros((E, N, 9))),
            "C": pinned(np.zeros((E, N, 9))), "cvo": pinned(np.zeros((T, E, K, 9))) if K else None,
            "act": pinned(np.zeros((T, E, G))) if G else None,
            "E": np.zeros((E, batch.n_materials), np.float64)}

    def rollout_host():
        batch.set_state(hx, hv, hF, hC, hmat, hgrp)
        obs = np.zeros((T, E, 7), np.float32)
        for t in range(T):
            obs[t] = batch.step(hcvo[t] if K else None, hact[t] if G else None)
        _, dobs = loss_and_dobs(scene.loss, np.transpose(obs, (1, 0, 2)))
        return batch.backward(dobs=np.ascontiguousarray(np.transpose(dobs, (1, 0, 2)), dtype=np.float32), out=hout)

    h2d = (hx.nbytes + hv.nbytes + hF.nbytes + hC.nbytes + hmat.nbytes + hgrp.nbytes +
           (sum(a.nbytes for a in hcvo) if K else 0) + (sum(a.nbytes for a in hact) if G else 0) + T * E * 7 * 4)
    d2h = T * E * 7 * 4 + E * N * 24 * 4 + (T * E * K * 9 * 4 if K else 0) + (T * E * G * 4 if G else 0) + E * 8 * batch.n_materials

    units_rank = E * N * T * S
    # warm-up
    for _ in range(args.warmup):
        rollout_device()
    torch.cuda.synchronize()
    launches0 = batch.launches
    barrier(dist)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            rollout_device()
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(dist)
    ms_rank = ev0.elapsed_time(ev1) / args.steps
    launches = (batch.launches - launches0) // args.steps
    # per-kernel-class times from a separate profiled rollout (CUDA events
    # around every launch on the context stream; not in the timed region)
    batch.profile(True)
    rollout_device()
    torch.cuda.synchronize()
    prof = batch.profile(False)
    prof_steps = 1

    # forward only (the rollout without the backward), same device timing
    def forward_device():
        with torch.cuda.stream(stream):
            batch.set_state(x0, v0, F0, C0, mat, grp)
            for t in range(T):
                batch.step(None if cvo_d is None else cvo_d[t], None if act_d is None else act_d[t], obs_d[t])
            batch.sync()  # forward errors / CFL of the rollout (the backward would read them)

    forward_device()
    barrier(dist)
    torch.cuda.synchronize()
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev2.record(stream)
    for _ in range(args.steps):
        forward_device()
    ev3.record(stream)
    torch.cuda.synchronize()
    fwd_ms = max_over_ranks(dist, ev2.elapsed_time(ev3) / args.steps)
    ms = max_over_ranks(dist, ms_rank)
    value = units_rank * world / (ms / 1e3)

    e2e = None
    if not args.no_e2e:
        rollout_host()
        torch.cuda.synchronize()
        barrier(dist)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            rollout_host()
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(dist, (time.perf_counter() - t0) * 1e3 / args.steps)
        barrier(dist)
        e2e = {"value": units_rank * world / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms}

    if rank != 0:
        return
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
        hbm, peak_src = float(peaks["hbm_gbs"]), "measured"
    except Exception:
        hbm, peak_src = 6650.0, "fallback"
    # dominant kernel (largest total time in the timed region)
    kern = {k: v for k, v in prof.items() if k in ALG_BYTES and v[1] > 0}
    dom = max(kern, key=lambda k: kern[k][0])
    dom_ms, dom_n = kern[dom]
    per_launch_units = E * N  # every launch of these kernels sweeps all particles once
    achieved = ALG_BYTES[dom] * per_launch_units / (dom_ms / dom_n / 1e3) / 1e9
    total_prof = sum(v[0] for v in prof.values())
    # DRAM traffic of the dominant kernel from the committed ncu --set full
    # capture (profiles/ncu_summary_cfg<N>.json, bytes per particle), per launch here
    # of this config (profiles/ncu_summary_cfg<N>.json; none committed: null)
    traffic, traffic_src = None, None
    try:
        name = "ncu_summary_cfg%d.json" % args.config
        with open(os.path.join(ROOT, "profiles", name)) as f:
            ks = json.load(f)
        kinfo = ks["kernels"][dom]
        traffic = kinfo["dram_bytes_per_particle"] * per_launch_units
        traffic_src = "profiles/%s (%s, %s)" % (name, kinfo["kernel"], ks.get("source", ""))
    except Exception:
        pass
    path_gbs = 480.0 * units_rank / (ms_rank / 1e3) / 1e9

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        nt = cpu_threads(ref_tape_bytes(scene))
        units, wall, desc = reference_sample(scene, nt, 1)
        cpu = {"value": units / wall, "unit": UNIT, "cores": nt, "kind": "reference", "sample": desc,
               "host_threads": cpu_info()[0], "cpu_model": cpu_info()[1]}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": scene.name, "envs": E * world, "particles_per_env": N, "control_steps": T,
                   "substeps_per_step": S, "grid": list(scene.sim["dims"]), "checkpoint_every": ck or S,
                   "particle_substeps_per_step": units_rank * world,
                   "l2": "inputs larger than L2 (state %.2f GB per rank)" % (E * N * 96 / 1e9)},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src,
                     "alg_bytes_per_particle": ALG_BYTES[dom], "kernel_share": dom_ms / total_prof,
                     "path_alg_gbs": path_gbs, "path_frac": path_gbs / hbm},
        "forward_only": {"value": units_rank * world / (fwd_ms / 1e3), "unit": UNIT, "ms_per_step": fwd_ms,
                         "note": "the same rollout without the backward (north_star: forward and forward+backward)"},
        "kernel_ms_per_step": {k: v[0] / prof_steps for k, v in prof.items() if v[1]},
        "kernel_ms_source": "one profiled rollout after the timed region (CUDA events per launch)",
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "e2e": e2e,
    }
    print(json.dumps(line), flush=True)
    if args.profile_out:
        with open(args.profile_out, "w") as f:
            json.dump(line, f, indent=1)


def run_sapo(args, rank, world, local, dist):
    """Config 5: full SAPO iterations (rollout with the policy in the loop,
    analytic gradient through the simulator, twin-critic TD(lambda), NCCL
    all-reduce of actor/critic gradients).  512 envs per GPU (weak scaling)."""
    import torch
    from paper_2412_12089_b200.sapo import SapoTrainer
    torch.cuda.set_device(local)
    per = (args.envs // world) if args.envs else 512
    H = args.ctrl or 32
    tr = SapoTrainer(seed=0, n_envs=per, env_offset=rank * per, n_global=per * world, horizon=H, n_sub=16,
                     dist=dist, device=local)
    for _ in range(args.warmup):
        tr.iteration()
    launches0 = tr.sim.launches
    barrier(dist)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            stats = tr.iteration()
        torch.cuda.synchronize()
        ms_rank = (time.perf_counter() - t0) * 1e3 / args.steps
    ms = max_over_ranks(dist, ms_rank)
    if rank != 0:
        return
    units = per * world * tr.N * H * 16
    line = {"metric": METRIC, "value": units / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "cfg5_sapo_iteration", "envs": per * world, "envs_per_gpu": per,
                       "particles_per_env": tr.N, "horizon": H, "substeps_per_step": 16,
                       "critic_passes": tr.critic_passes, "nets": "actor 64-256x3-16, twin critics 64-256x3-1, ELU+LN"},
            "env_steps_per_s": per * world * H / (ms / 1e3), "gpu_launches": int((tr.sim.launches - launches0) // args.steps),
            "clocks": clk.summary(), "last_iteration": stats,
            "timing": "host wall clock around whole iterations (sim + torch nets + NCCL), max over ranks"}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference" and rank != 0:
        return
    dist = init_dist(world, local) if args.impl == "ours" else None
    if args.config == 5 and args.impl == "ours":
        run_sapo(args, rank, world, local, dist)
        if dist is not None:
            dist.destroy_process_group()
        return
    from paper_2412_12089_b200 import scenes
    total = args.envs or {1: 1, 2: 32, 3: 256, 4: 1024, 5: 512}[args.config]
    if args.config == 5:
        args.config = 2  # the reference arm times config 5's simulator (config 2 physics)
    # strong scaling (default): the config's envs are split across the ranks
    # (rank r: global envs [r per, (r+1) per), no simulator collective);
    # --weak: every rank simulates the config's envs
    if args.impl == "ours":
        per = total if args.weak else total // world
    else:  # the reference arm: one env per host thread (bounded by the tapes' memory)
        n_cfg = {1: 4096, 2: 20480, 3: 30000, 4: 16384}[args.config]
        per = min(total, cpu_threads(int(n_cfg * 2200 * 33 * 1.3)))
    kw = {"n_envs": per, "env_offset": rank * per if args.impl == "ours" else 0}
    if args.ctrl:
        kw["n_ctrl"] = args.ctrl
    scene = scenes.CONFIGS[args.config](seed=0, **kw)
    if args.impl == "reference":
        run_reference(args, scene, rank, dist)
    else:
        run_ours(args, scene, rank, world, local, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
