"""CPU, world_size 2 over gloo: the env-sharded multi-GPU path's host logic.

Envs shard with no simulator collective; each rank builds
its env range from global env indices, so every env's inputs -- and hence its
oracle trajectory -- are identical to the unsharded run.  bench.py's timing
reduction is a MAX all-reduce over ranks."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": str(rank),
                       "WORLD_SIZE": str(world)})
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    import bench
    import pyoracle as O
    from paper_2412_12089_b200 import scenes
    total = 4
    per = total // world
    sc = scenes.config4(seed=9, n_envs=per, env_offset=rank * per, n_ctrl=1, n_sub=2, lattice_counts=(4, 4, 2))
    cvo, _ = sc.cvo_act()
    obs = []
    for e in range(per):
        _, o, _ = O.rollout(sc.sim, sc.materials, sc.env_cols(e, cvo), sc.env_state(e), 1, 2, loss=sc.loss)
        obs.append(o[0])
    t = torch.tensor(np.array(obs))
    gathered = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    mx = bench.max_over_ranks(dist, float(rank + 1))
    if rank == 0:
        out.put((torch.cat(gathered).numpy(), mx))
    dist.barrier()
    dist.destroy_process_group()


def test_env_sharding_world2_matches_single():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    sharded, mx = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import pyoracle as O
    from paper_2412_12089_b200 import scenes
    sc = scenes.config4(seed=9, n_envs=4, n_ctrl=1, n_sub=2, lattice_counts=(4, 4, 2))
    cvo, _ = sc.cvo_act()
    single = np.array([O.rollout(sc.sim, sc.materials, sc.env_cols(e, cvo), sc.env_state(e), 1, 2, loss=sc.loss)[1][0]
                       for e in range(4)])
    assert np.array_equal(sharded, single)
    assert mx == 2.0


def _grad_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_2412_12089_b200.sapo import SapoTrainer, MLP
    net = MLP([4, 8, 1])
    torch.manual_seed(rank)
    for p in net.parameters():
        dist.broadcast(p.data, 0)
    x = torch.full((3, 4), float(rank + 1))
    net(x).sum().backward()
    fake = SapoTrainer.__new__(SapoTrainer)
    fake.dist = dist
    fake.dev = torch.device("cpu")
    SapoTrainer._allreduce_grads(fake, list(net.parameters()))
    tot = SapoTrainer._allreduce_scalar(fake, float(rank + 1))
    if rank == 0:
        out.put(([p.grad.clone() for p in net.parameters()], tot, [p.detach().clone() for p in net.parameters()]))
    dist.barrier()
    dist.destroy_process_group()


def test_sapo_gradient_allreduce_world2():
    """Actor/critic gradients are summed over ranks (each rank's loss carries
    1/N_global), as the NCCL path does on GPUs."""
    import torch
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grad_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    grads, tot, params = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_2412_12089_b200.sapo import MLP
    net = MLP([4, 8, 1])
    with torch.no_grad():
        for p, q_ in zip(net.parameters(), params):
            p.copy_(q_)
    for r in range(2):
        net(torch.full((3, 4), float(r + 1))).sum().backward()
    for p, g in zip(net.parameters(), grads):
        assert torch.allclose(p.grad, g, atol=1e-6)
    assert tot == 3.0
