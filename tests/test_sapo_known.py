"""SAPO learner known answers on the torch path (cpu, and cuda under -m gpu).

  * soft TD(lambda) targets vs the n-step brute force of acceptance.cpp:211-249
    (criterion 3: 1000 random trials, horizon 5, 3 envs, episode cuts),
    max |err| < 1e-12, and alpha = 0 equals plain TD(lambda) with zero
    entropy bit for bit
  * the reference AdamW (nets.hpp:282-328; test_nets.cpp:281-324): hand first
    step, zero gradient, clip before the moments, NaN skip, decoupled decay
  * objective reductions (test_algo.cpp:197-247): SAPO with alpha = 0 and one
    critic equals SHAC (value and leaf gradients), APG equals SHAC with a
    zero critic (reward-leaf gradients)
"""
import math

import numpy as np
import pytest
import torch

from paper_2412_12089_b200.rng import RngStream
from paper_2412_12089_b200.sapo import (AdamWRef, actor_objective_apg, actor_objective_sapo, actor_objective_shac,
                                        soft_td_lambda)

DEVICES = [pytest.param("cpu"), pytest.param("cuda", marks=pytest.mark.gpu)]


def td_lambda_bruteforce(reward, ent, done, vmin, alpha, gamma, lam):
    """acceptance.cpp:211-249 restated: lambda-weighted n-step returns up to
    the episode end (test infrastructure, plain loops in fp64)."""
    H, N = reward.shape
    out = np.zeros((H, N))
    for i in range(N):
        for t in range(H):
            e = t
            while e < H - 1 and not done[e, i]:
                e += 1
            cut = bool(done[e, i])

            def nstep(n, boot):
                g, disc = 0.0, 1.0
                for k in range(n):
                    g += disc * (reward[t + k, i] + alpha[i] * ent[t + k, i])
                    disc *= gamma[i]
                if boot:
                    g += disc * vmin[t + n, i]
                return g

            seg = e - t + 1
            v, w = 0.0, 1.0
            for n in range(1, seg):
                v += (1.0 - lam[i]) * w * nstep(n, True)
                w *= lam[i]
            v += w * nstep(seg, not cut)
            out[t, i] = v
    return out


@pytest.mark.parametrize("dev", DEVICES)
def test_soft_td_lambda_vs_bruteforce(dev):
    rng = RngStream(3, 0)
    H, n_env, trials = 5, 3, 1000
    N = n_env * trials
    reward = np.zeros((H, N))
    ent = np.zeros((H, N))
    done = np.zeros((H, N), np.uint8)
    vmin = np.zeros((H + 1, N))
    gamma = np.zeros(N)
    lam = np.zeros(N)
    alpha = np.zeros(N)
    for tr in range(trials):
        sl = slice(tr * n_env, (tr + 1) * n_env)
        for t in range(H):
            for i in range(n_env):
                reward[t, tr * n_env + i] = rng.normal()
                ent[t, tr * n_env + i] = rng.uniform(0.0, 1.0)
                done[t, tr * n_env + i] = 1 if rng.uniform(0.0, 1.0) < 0.25 else 0
        for t in range(H + 1):
            for i in range(n_env):
                vmin[t, tr * n_env + i] = rng.normal()
        gamma[sl] = rng.uniform(0.8, 1.0)
        lam[sl] = rng.uniform(0.0, 1.0)
        alpha[sl] = rng.uniform(0.0, 0.5)
    want = td_lambda_bruteforce(reward, ent, done, vmin, alpha, gamma, lam)
    T = lambda a: torch.as_tensor(a, dtype=torch.float64, device=dev)
    got = soft_td_lambda(T(reward), T(ent), T(vmin), T(alpha), T(gamma), T(lam), done=T(done))
    assert float((got.cpu().numpy() - want).__abs__().max()) < 1e-12
    # alpha = 0 reduces to plain TD(lambda) (zero entropy, alpha 1) bit for bit
    soft0 = soft_td_lambda(T(reward), T(ent), T(vmin), 0.0, T(gamma), T(lam), done=T(done))
    plain = soft_td_lambda(T(reward), torch.zeros_like(T(ent)), T(vmin), 1.0, T(gamma), T(lam), done=T(done))
    assert torch.equal(soft0, plain)


@pytest.mark.parametrize("dev", DEVICES)
def test_adamw_reference_semantics(dev, capsys):
    P = lambda *v: torch.nn.Parameter(torch.tensor(v, dtype=torch.float64, device=dev))
    # hand-computed first step: gradient 1 clipped to 0.5, then one Adam step of size lr
    p = P(1.0)
    opt = AdamWRef([p], lr=0.1, betas=(0.9, 0.999))
    p.grad = torch.tensor([1.0], dtype=torch.float64, device=dev)
    assert opt.step()
    assert abs(float(p.detach()) - 0.9) < 1e-6
    # zero gradients, zero decay: unchanged
    q = P(0.3, -0.7)
    opt = AdamWRef([q])
    q.grad = torch.zeros_like(q)
    opt.step()
    assert q.tolist() == [0.3, -0.7]
    # large gradients are clipped (global norm 10 -> 0.5) before the moments
    r = P(0.0, 0.0)
    opt = AdamWRef([r])
    r.grad = torch.tensor([6.0, 8.0], dtype=torch.float64, device=dev)
    opt.step()
    m = opt.state[r]["m"].tolist()
    assert math.isclose(m[0], (1.0 - 0.7) * 0.3, rel_tol=1e-12) and math.isclose(m[1], (1.0 - 0.7) * 0.4, rel_tol=1e-12)
    # the clip norm is global over all of the optimizer's parameters
    a, b = P(0.0), P(0.0)
    opt = AdamWRef([a, b])
    a.grad = torch.tensor([6.0], dtype=torch.float64, device=dev)
    b.grad = torch.tensor([8.0], dtype=torch.float64, device=dev)
    opt.step()
    assert math.isclose(float(opt.state[b]["m"]), 0.3 * 0.4, rel_tol=1e-12)
    # NaN gradient: the step is skipped (no update, no moments, no step count)
    s = P(0.5)
    opt = AdamWRef([s])
    s.grad = torch.tensor([float("nan")], dtype=torch.float64, device=dev)
    assert opt.step() is False
    assert float(s.detach()) == 0.5 and opt.step_count == 0 and not opt.state[s]
    assert "AdamW: non-finite gradient, step skipped" in capsys.readouterr().err
    # decoupled weight decay
    w = P(2.0)
    opt = AdamWRef([w], lr=0.1, weight_decay=0.01)
    w.grad = torch.zeros_like(w)
    opt.step()
    assert math.isclose(float(w.detach()), 2.0 - 0.1 * 0.01 * 2.0, rel_tol=1e-12)


def _synthetic(dev, H, N, C, seed, zero_terminal=False):
    """Leaves: rewards [H, N], entropies [H, N], terminal critic values [C, N]."""
    r = RngStream(seed, 0)
    rew = torch.tensor([[r.normal() for _ in range(N)] for _ in range(H)], dtype=torch.float64, device=dev)
    ent = torch.tensor([[r.uniform(0.0, 1.0) for _ in range(N)] for _ in range(H)], dtype=torch.float64, device=dev)
    term = torch.tensor([[0.0 if zero_terminal else r.normal() for _ in range(N)] for _ in range(C)],
                        dtype=torch.float64, device=dev)
    return [x.requires_grad_(True) for x in (rew, ent, term)]


@pytest.mark.parametrize("dev", DEVICES)
def test_objective_reductions(dev):
    gamma = 0.97
    rew, ent, term = _synthetic(dev, 6, 4, 1, 17)
    l_sapo = actor_objective_sapo(rew, ent, term, 0.0, gamma)
    l_shac = actor_objective_shac(rew, ent, term, gamma)
    assert abs(float(l_sapo) - float(l_shac)) < 1e-12
    ga = torch.autograd.grad(l_sapo, [rew, ent, term], allow_unused=True)
    ra, ea, ta = _synthetic(dev, 6, 4, 1, 17)
    gb = torch.autograd.grad(actor_objective_shac(ra, ea, ta, gamma), [ra, ea, ta], allow_unused=True)
    for x, y in zip(ga, gb):
        if x is None or y is None:
            assert (x is None or not x.abs().max()) and (y is None or not y.abs().max())
            continue
        assert (x - y).abs().max() <= 1e-13
    # APG equals SHAC with an identically-zero critic (value, reward-leaf gradients)
    rew, ent, term = _synthetic(dev, 6, 4, 1, 23, zero_terminal=True)
    la = actor_objective_apg(rew, ent, gamma)
    lb = actor_objective_shac(rew, ent, term, gamma)
    assert abs(float(la) - float(lb)) < 1e-12
    (g_a,) = torch.autograd.grad(la, [rew])
    (g_b,) = torch.autograd.grad(lb, [rew])
    assert (g_a - g_b).abs().max() <= 1e-13
    # SAPO needs a critic
    with pytest.raises(ValueError):
        actor_objective_sapo(rew, ent, term[:0], 0.1, gamma)
