"""Task losses over per-control-step observables and their cotangents.

Observables per env per control step (7 floats, computed on the device after
every control step): center of mass (3), per-axis position variance (3) and
the smoothed spill fraction outside the container footprint (1).  These are
the reductions the reference tasks compute in ``step``/``observe``
(tasks.hpp:286-304, 330-338, 554-570, 604-615).  The loss is a scalar of
those observables, so its gradient w.r.t. them is formed here on the host and
fed to the device backward as ``dobs``.
"""
from __future__ import annotations

import numpy as np

OBS_DIM = 7


def tiered(d, threshold, low, high):
    """reward_distance_tiered (env.hpp:33-39): (1/(1+d))^2 x tier (gradient-blocked)."""
    mult = np.where(d > threshold, low, high)
    return mult / (1.0 + d) ** 2, mult


def loss_and_dobs(spec: dict, obs: np.ndarray):
    """obs: [..., T, 7] -> (loss [...], dobs [..., T, 7])."""
    obs = np.asarray(obs, dtype=np.float64)
    d = np.zeros_like(obs)
    kind = spec["kind"]
    if kind == "com_target":
        tgt = np.asarray(spec.get("target", (0.5, 0.4, 0.5)))
        diff = obs[..., -1, 0:3] - tgt
        L = (diff ** 2).sum(-1)
        d[..., -1, 0:3] = 2.0 * diff
    elif kind == "neg_mean_z":
        L = -obs[..., :, 2].sum(-1)
        d[..., :, 2] = -1.0
    elif kind == "var_z":
        L = obs[..., :, 5].sum(-1)
        d[..., :, 5] = 1.0
    elif kind == "fluid_move":
        tgt = np.asarray(spec["target"])
        diff = obs[..., 0:3] - tgt
        dist = np.sqrt((diff ** 2).sum(-1) + 1e-12)
        r, mult = tiered(dist, spec.get("tier_threshold", 0.02), spec.get("tier_low", 1.0), spec.get("tier_high", 2.0))
        L = (-(r - obs[..., 6])).sum(-1)
        dr_ddist = -2.0 * mult / (1.0 + dist) ** 3
        d[..., 0:3] = (-dr_ddist / dist)[..., None] * diff
        d[..., 6] = 1.0
    else:
        raise ValueError(f"unknown loss kind {kind!r}")
    return L, d


def loss_and_dobs_torch(spec: dict, obs):
    """Same as loss_and_dobs for a torch tensor obs [..., T, 7] (device-side)."""
    import torch
    o = obs.double()
    d = torch.zeros_like(o)
    kind = spec["kind"]
    if kind == "com_target":
        tgt = torch.tensor(spec.get("target", (0.5, 0.4, 0.5)), dtype=o.dtype, device=o.device)
        diff = o[..., -1, 0:3] - tgt
        L = (diff ** 2).sum(-1)
        d[..., -1, 0:3] = 2.0 * diff
    elif kind == "neg_mean_z":
        L = -o[..., :, 2].sum(-1)
        d[..., :, 2] = -1.0
    elif kind == "var_z":
        L = o[..., :, 5].sum(-1)
        d[..., :, 5] = 1.0
    elif kind == "fluid_move":
        tgt = torch.tensor(spec["target"], dtype=o.dtype, device=o.device)
        diff = o[..., 0:3] - tgt
        dist = torch.sqrt((diff ** 2).sum(-1) + 1e-12)
        thr, lo, hi = spec.get("tier_threshold", 0.02), spec.get("tier_low", 1.0), spec.get("tier_high", 2.0)
        mult = torch.where(dist > thr, torch.full_like(dist, lo), torch.full_like(dist, hi))
        r = mult / (1.0 + dist) ** 2
        L = (-(r - o[..., 6])).sum(-1)
        dr = -2.0 * mult / (1.0 + dist) ** 3
        d[..., 0:3] = (-dr / dist).unsqueeze(-1) * diff
        d[..., 6] = 1.0
    else:
        raise ValueError(f"unknown loss kind {kind!r}")
    return L, d.float()
