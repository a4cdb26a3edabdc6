"""SAPO training iteration on the GPU simulator (config 5).

Restates the reference learner around the hot path (algo.hpp:121-191
collect_rollout, 196-230 actor_objective_sapo, 243-265 soft TD(lambda),
292-327 critic_update, 348-357 temperature_update, 677-760 train_iteration;
nets.hpp:100-205 LayerNorm MLP and squashed-Gaussian policy, 294-328 AdamW)
with torch for the networks and the diffmpm batch (api.MpmBatch) for the
simulator.  The analytic policy gradient flows through the simulator with the
incremental backward (dm_backward_step): for t = H-1 .. 0 the cotangent of
obs_{t+1} (direct terms + the actor's input path) is injected, the
simulator returns d loss / d action_t, and the actor VJP closes the loop.

Data parallel: each rank owns a contiguous range of envs; the only
collectives are NCCL all-reduces of the actor and critic gradients and of a
few scalars (temperature gap, metrics) -- SURVEY.md 8(e).  Each rank scales
its loss by 1 / N_global so the all-reduced sum is the global mean
(algo.hpp:221), and gradient-norm clipping happens after the all-reduce.
"""
from __future__ import annotations

import math
import time

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as Fn

from . import api, scenes
from .rng import RngStream

K_LOG_SQRT_2PI = 0.9189385332046727


class MLP(nn.Module):
    """LayerNorm MLP with ELU on hidden layers (nets.hpp:100-139)."""

    def __init__(self, dims, out_scale=1.0):
        super().__init__()
        self.lin = nn.ModuleList([nn.Linear(a, b) for a, b in zip(dims[:-1], dims[1:])])
        self.norm = nn.ModuleList([nn.LayerNorm(d, eps=1e-5) for d in dims[1:-1]])
        with torch.no_grad():
            self.lin[-1].weight.mul_(out_scale)
            self.lin[-1].bias.zero_()

    def forward(self, x):
        for i, l in enumerate(self.lin):
            x = l(x)
            if i < len(self.lin) - 1:
                x = Fn.elu(self.norm[i](x))
        return x


class Actor(nn.Module):
    """Squashed Gaussian policy (nets.hpp:143-205): trunk -> (mean, log sigma)."""

    def __init__(self, obs_dim, act_dim, hidden=(256, 256, 256)):
        super().__init__()
        self.act_dim = act_dim
        self.trunk = MLP([obs_dim, *hidden, 2 * act_dim], out_scale=0.01)

    def sample(self, obs, noise):
        out = self.trunk(obs)
        mu, ls = out[:, :self.act_dim], out[:, self.act_dim:].clamp(-5.0, 2.0)
        u = mu + ls.exp() * noise
        a = torch.tanh(u)
        logp = (-0.5 * noise * noise - K_LOG_SQRT_2PI - ls).sum(-1)
        logp = logp - (2.0 * (math.log(2.0) - u - Fn.softplus(-2.0 * u))).sum(-1)
        return a, logp


def normalize_entropy(h, target):  # algo.hpp:38-43
    a = abs(target)
    return (h + a) * (1.0 / (2.0 * a))


def soft_td_lambda(reward, ent, vmin, alpha, gamma, lam, done=None):
    """soft_td_lambda_from_values (algo.hpp:240-265): backward recursion
    vt_t = (r_t + alpha hhat_t) + gamma ((1 - lambda) vmin_{t+1} + lambda vt_{t+1}),
    bootstrap dropped where done[t] (episode boundary).  reward, ent, done:
    [H, N]; vmin: [H+1, N]; alpha / gamma / lam: scalars or [N] tensors."""
    H = reward.shape[0]
    if vmin.shape[0] != H + 1:
        raise ValueError("soft_td_lambda: need H+1 value rows")
    targets = torch.empty_like(reward)
    nxt = vmin[H]
    for t in range(H - 1, -1, -1):
        boot = gamma * ((1.0 - lam) * vmin[t + 1] + lam * nxt)
        if done is not None:
            boot = torch.where(done[t].bool(), torch.zeros_like(boot), boot)
        targets[t] = reward[t] + alpha * ent[t] + boot
        nxt = targets[t]
    return targets


def actor_objective(reward, ent, terminal_values, alpha, gamma, boot="mean"):
    """actor_objective (algo.hpp:196-230):
    loss = -(1/N) sum_i [ sum_t gamma^t (r_t + alpha hhat_t) + gamma^H V(s_H) ]
    reward, ent: [H, N] (autograd tensors); terminal_values: [C, N];
    boot: "mean" (SAPO, mean over the C critics), "first" (SHAC), "none" (APG)."""
    H, N = reward.shape
    if boot != "none" and (terminal_values is None or terminal_values.shape[0] == 0):
        raise ValueError("actor_objective: no critics in buffer")
    acc = torch.zeros(N, dtype=reward.dtype, device=reward.device)
    disc = 1.0
    for t in range(H):
        step_r = reward[t] + alpha * ent[t] if alpha != 0.0 else reward[t]
        acc = acc + disc * step_r
        disc *= gamma
    if boot == "mean":
        acc = acc + (disc / terminal_values.shape[0]) * terminal_values.sum(0)
    elif boot == "first":
        acc = acc + disc * terminal_values[0]
    return (-1.0 / N) * acc.sum()


def actor_objective_sapo(reward, ent, terminal_values, alpha, gamma):
    return actor_objective(reward, ent, terminal_values, alpha, gamma, "mean")


def actor_objective_shac(reward, ent, terminal_values, gamma):
    return actor_objective(reward, ent, terminal_values, 0.0, gamma, "first")


def actor_objective_apg(reward, ent, gamma):
    return actor_objective(reward, ent, None, 0.0, gamma, "none")


class AdamWRef(torch.optim.Optimizer):
    """The reference optimizer (nets.hpp:282-328), not torch's AdamW:
      * a non-finite gradient (or squared norm) skips the whole step: no
        moment, step-count or parameter update; prints the reference's
        "AdamW: non-finite gradient, step skipped" to stderr; step() returns False
      * the global L2 norm of all the optimizer's gradients is clipped to
        clip_norm *inside* the step, before the moments
      * p -= lr (mhat / (sqrt(vhat) + eps) + weight_decay p), with
        mhat = m / (1 - beta1^k), vhat = v / (1 - beta2^k).
    Defaults are the reference's (lr 1e-3, betas (0.7, 0.95), eps 1e-8,
    weight_decay 0, clip_norm 0.5).  Runs on the parameters' device and dtype."""

    def __init__(self, params, lr=1e-3, betas=(0.7, 0.95), eps=1e-8, weight_decay=0.0, clip_norm=0.5):
        super().__init__(params, dict(lr=lr, betas=betas, eps=eps, weight_decay=weight_decay, clip_norm=clip_norm))
        self.step_count = 0

    @torch.no_grad()
    def step(self, closure=None):  # noqa: D401
        params = [p for g in self.param_groups for p in g["params"] if p.grad is not None]
        if not params:
            return False
        norm2 = torch.stack([(p.grad.double() * p.grad.double()).sum() for p in params]).sum()
        if not bool(torch.isfinite(norm2)):  # NaN / inf entries make the sum non-finite
            import sys
            print("AdamW: non-finite gradient, step skipped", file=sys.stderr)
            return False
        norm = math.sqrt(float(norm2))
        self.step_count += 1
        for g in self.param_groups:
            b1, b2 = g["betas"]
            clip = g["clip_norm"]
            scale = clip / norm if (clip > 0.0 and norm > clip) else 1.0
            bc1 = 1.0 - b1 ** self.step_count
            bc2 = 1.0 - b2 ** self.step_count
            for p in g["params"]:
                if p.grad is None:
                    continue
                st = self.state[p]
                if not st:
                    st["m"] = torch.zeros_like(p)
                    st["v"] = torch.zeros_like(p)
                gr = p.grad * scale if scale != 1.0 else p.grad
                st["m"].mul_(b1).add_(gr, alpha=1.0 - b1)
                st["v"].mul_(b2).add_(gr * gr, alpha=1.0 - b2)
                upd = (st["m"] / bc1) / ((st["v"] / bc2).sqrt() + g["eps"])
                if g["weight_decay"] != 0.0:
                    upd = upd + g["weight_decay"] * p
                p.sub_(g["lr"] * upd)
        return True


class SapoTrainer:
    def __init__(self, seed=0, n_envs=512, env_offset=0, n_global=None, horizon=32, n_sub=16, critic_passes=16,
                 hidden=(256, 256, 256), dist=None, device=0, gamma=0.99, lam=0.95, actor_lr=2e-3, critic_lr=5e-4,
                 alpha_lr=5e-3, init_alpha=1.0, total_iterations=100):
        self.dist = dist
        self.seed, self.env_offset = seed, env_offset
        self.dev = torch.device("cuda", device)
        self.scene = scenes.config2(seed=seed, n_envs=n_envs, env_offset=env_offset, n_ctrl=horizon, n_sub=n_sub)
        self.scene.extra["obs_groups"] = 8
        self.E, self.N, self.H, self.S = n_envs, self.scene.n_per_env, horizon, n_sub
        self.n_global = n_global or n_envs
        self.sim = api.from_scene(self.scene, device=device)
        self.od = self.sim.obs_dim
        self.act_dim = 8
        self.gamma, self.lam, self.critic_passes = gamma, lam, critic_passes
        g = torch.Generator().manual_seed(seed)
        torch.manual_seed(seed)
        self.actor = Actor(64, self.act_dim, hidden).to(self.dev)
        self.critics = nn.ModuleList([MLP([64, *hidden, 1]) for _ in range(2)]).to(self.dev)
        if dist is not None:  # identical initial weights on every rank
            for p in list(self.actor.parameters()) + list(self.critics.parameters()):
                dist.broadcast(p.data, 0)
        betas = (0.7, 0.95)
        # the reference AdamW: clip inside step (after the all-reduce), skip non-finite
        self.actor_opt = AdamWRef(self.actor.parameters(), lr=actor_lr, betas=betas, clip_norm=0.5)
        self.critic_opts = [AdamWRef(c.parameters(), lr=critic_lr, betas=betas, clip_norm=0.5) for c in self.critics]
        self.log_alpha = torch.tensor(math.log(init_alpha), device=self.dev, requires_grad=True)
        self.alpha_opt = AdamWRef([self.log_alpha], lr=alpha_lr, betas=betas, clip_norm=0.5)
        self.ent_target = -self.act_dim / 2.0
        self.iter = 0
        self.total_iterations = total_iterations
        self.base_lr = (actor_lr, critic_lr)
        f32 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32), device=self.dev)
        sc = self.scene
        self.x0, self.v0, self.F0, self.C0 = f32(sc.x), f32(sc.v), f32(sc.F), f32(sc.C)
        self.mat = torch.as_tensor(sc.material, dtype=torch.int32, device=self.dev)
        self.grp = torch.as_tensor(sc.group, dtype=torch.int32, device=self.dev)
        self.noise_gen = torch.Generator(device=self.dev).manual_seed(seed * 1000003 + env_offset)
        self.obs = torch.zeros((self.H + 1, self.E, self.od), device=self.dev)
        self.stream = torch.cuda.ExternalStream(self.sim.stream_ptr, device=self.dev)
        torch.cuda.synchronize()  # initial tensors (default stream) are ready before the context stream reads them

    def env_rng(self, i):
        """(key, counter) of env i's RngStream(seed, global index) (env.hpp:71):
        the config-2 reset draws nothing from it."""
        r = RngStream(self.seed, self.env_offset + i)
        return int(r.key), int(r.counter)

    # ---- collectives (NCCL) ----
    def _allreduce_grads(self, params):
        if self.dist is None:
            return
        grads = [p.grad for p in params if p.grad is not None]
        flat = torch.cat([g.reshape(-1) for g in grads])
        self.dist.all_reduce(flat)
        o = 0
        for g in grads:
            n = g.numel()
            g.copy_(flat[o:o + n].view_as(g))
            o += n

    def _allreduce_scalar(self, x):
        t = torch.as_tensor([x], dtype=torch.float64, device=self.dev)
        if self.dist is not None:
            self.dist.all_reduce(t)
        return float(t.item())

    def _policy_input(self, t):
        return self.obs[t, :, 7:7 + 64]

    def iteration(self):
        """One SAPO iteration.  Every torch op runs on the simulator context's
        stream, so the simulator kernels and the networks are ordered without
        host synchronisation (the *_device ABI contract)."""
        with torch.cuda.stream(self.stream):
            return self._iteration()

    def _iteration(self):
        frac = max(0.0, 1.0 - self.iter / self.total_iterations)
        for g in self.actor_opt.param_groups:
            g["lr"] = self.base_lr[0] * frac
        for o in self.critic_opts:
            for g in o.param_groups:
                g["lr"] = self.base_lr[1] * frac
        E, H = self.E, self.H
        alpha = float(self.log_alpha.detach().exp())
        # ---- rollout (collect_rollout, algo.hpp:121-191) ----
        self.sim.set_state(self.x0, self.v0, self.F0, self.C0, self.mat, self.grp)
        self.sim.observe(None, self.obs[0])  # reset observation (Task::observe)
        obs_in, acts, logps = [], [], []
        for t in range(H):
            o_in = self._policy_input(t).detach().clone().requires_grad_(True)
            noise = torch.randn((E, self.act_dim), generator=self.noise_gen, device=self.dev)
            a, logp = self.actor.sample(o_in, noise)
            obs_in.append(o_in)
            acts.append(a)
            logps.append(logp)
            act = a.detach().contiguous()
            self.sim.step(None, act, self.obs[t + 1])
        obs_next = self.obs[1:].detach().clone().requires_grad_(True)  # [H, E, od]
        reward = obs_next[:, :, 2]  # height reward: mean z after the step
        h_raw = -torch.stack(logps)  # [H, E]
        ent = normalize_entropy(h_raw, self.ent_target)
        disc = torch.tensor([self.gamma ** t for t in range(H)], device=self.dev)
        v_term = torch.stack([c(obs_next[H - 1, :, 7:7 + 64]).squeeze(-1) for c in self.critics])  # [C, E]
        ret = (disc[:, None] * (reward + alpha * ent)).sum(0) + (self.gamma ** H) * v_term.mean(0)
        # actor_objective_sapo (algo.hpp:226-229), this rank's share of -(1/N_global) sum_i
        loss = actor_objective_sapo(reward, ent, v_term, alpha, self.gamma) * (E / self.n_global)
        # direct partials: obs_{t+1} (reward, bootstrap) and the actor inputs obs_t
        params = list(self.actor.parameters())
        g_next, *g_in = torch.autograd.grad(loss, [obs_next] + obs_in[1:], retain_graph=True, allow_unused=True)
        g_next = g_next.detach()
        # ---- reverse sweep through the simulator (dm_backward_step) ----
        self.sim.backward_begin()
        dact = [None] * H
        dobs_t = torch.zeros((E, self.od), device=self.dev)
        dact_buf = torch.zeros((E, self.act_dim), device=self.dev)
        carry = torch.zeros((E, 64), device=self.dev)  # actor-input cotangent of obs_{t+1}
        for t in range(H - 1, -1, -1):
            dobs_t.copy_(g_next[t])
            if t + 1 < H:
                if g_in[t] is not None:  # obs_in[t+1] direct term
                    dobs_t[:, 7:7 + 64] += g_in[t]
                dobs_t[:, 7:7 + 64] += carry
            self.sim.backward_step(dobs_t, out_act=dact_buf)
            dact[t] = dact_buf.clone()
            # actor input path: obs_t -> a_t, cotangent dact_t
            if t > 0:
                (carry,) = torch.autograd.grad(acts[t], obs_in[t], grad_outputs=dact[t], retain_graph=True)
        self.sim.backward_end()
        surrogate = loss + sum((acts[t] * dact[t]).sum() for t in range(H))
        self.actor_opt.zero_grad(set_to_none=True)
        surrogate.backward()
        self._allreduce_grads(params)
        gnorm = torch.stack([(p.grad.double() ** 2).sum() for p in params if p.grad is not None]).sum().sqrt()
        self.actor_opt.step()  # global-norm clip to 0.5 and non-finite skip inside (nets.hpp:294-316)
        # ---- temperature (algo.hpp:348-357) ----
        gap = self._allreduce_scalar(float((h_raw.detach() - self.ent_target).sum())) / (H * self.n_global)
        self.alpha_opt.zero_grad(set_to_none=True)
        self.log_alpha.grad = torch.tensor(alpha * gap, device=self.dev)
        self.alpha_opt.step()
        alpha = float(self.log_alpha.detach().exp())
        # ---- critics: soft TD(lambda) targets + K full-batch passes (algo.hpp:243-327) ----
        with torch.no_grad():
            obs_all = self.obs[:, :, 7:7 + 64].detach()  # [H+1, E, 64]
            vmin = torch.stack([c(obs_all).squeeze(-1) for c in self.critics]).min(0).values
            targets = soft_td_lambda(reward.detach(), ent.detach(), vmin, alpha, self.gamma, self.lam)  # no dones in H
        closs = 0.0
        for _ in range(self.critic_passes):
            closs = 0.0
            for c, opt in zip(self.critics, self.critic_opts):
                opt.zero_grad(set_to_none=True)
                v = c(obs_all[:H]).squeeze(-1)
                lc = ((v - targets) ** 2).sum() / (H * self.n_global)
                lc.backward()
                self._allreduce_grads(list(c.parameters()))
                opt.step()  # clip + non-finite skip inside (critic_update, algo.hpp:318)
                closs += float(lc.detach())
        self.iter += 1
        ret_mean = self._allreduce_scalar(float(ret.detach().sum())) / self.n_global
        return {"actor_loss": self._allreduce_scalar(float(loss.detach())), "critic_loss": closs / 2, "return_mean": ret_mean,
                "alpha": alpha, "entropy_mean": gap + self.ent_target, "grad_norm": float(gnorm)}
