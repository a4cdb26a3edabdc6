"""Trainer / env persistence in the reference's DSIMCKPT container
(checkpoint_io.hpp:20-207), so a resumed run continues bit for bit.

Container (checkpoint_io.hpp:57-111): magic "DSIMCKPT", u32 version 1,
u32 entry count, then per entry (ascending name order, std::map) u32 name
length, name bytes, u64 value count, f64 values; little-endian.  Integer
state (iteration counters, RNG words) is stored as bit patterns
(pack_u64 / unpack_u64, checkpoint_io.hpp:50-55).

Entries written by snapshot_trainer mirror the reference's names
(checkpoint_io.hpp:140-170): meta, policy, opt.actor.{m,v,step},
critic.k, opt.critic.k.{m,v,step}, opt.alpha.{m,v,step}, and per env
env.i.{state,cursor,rng,ep_return} (state in the visit order x, v, F, C,
tasks.hpp:203-219).  Framework extras: sim.noise (the policy-noise
generator state) and sim.env_seed.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"DSIMCKPT"
VERSION = 1


class CheckpointError(RuntimeError):
    """ckpt::CheckpointError (checkpoint_io.hpp:24-26)."""


def pack_u64(x: int) -> float:
    return struct.unpack("<d", struct.pack("<Q", int(x) & 0xFFFFFFFFFFFFFFFF))[0]


def unpack_u64(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", float(x)))[0]


def save_checkpoint(arrays: dict, path: str) -> None:
    """save_checkpoint (checkpoint_io.hpp:57-78)."""
    try:
        f = open(path, "wb")
    except OSError:
        raise CheckpointError("cannot open checkpoint for write: " + path) from None
    with f:
        f.write(MAGIC)
        f.write(struct.pack("<II", VERSION, len(arrays)))
        for name in sorted(arrays):
            data = np.ascontiguousarray(arrays[name], dtype="<f8").ravel()
            nb = name.encode()
            f.write(struct.pack("<I", len(nb)))
            f.write(nb)
            f.write(struct.pack("<Q", data.size))
            f.write(data.tobytes())


def load_checkpoint(path: str) -> dict:
    """load_checkpoint (checkpoint_io.hpp:80-111): the same error texts."""
    try:
        f = open(path, "rb")
    except OSError:
        raise CheckpointError("cannot open checkpoint: " + path) from None
    with f:
        buf = f.read()
    if len(buf) < 8 or buf[:8] != MAGIC:
        raise CheckpointError("not a checkpoint file: " + path)
    o = 8
    if len(buf) < o + 8:
        raise CheckpointError("truncated checkpoint: " + path)
    version, n = struct.unpack_from("<II", buf, o)
    o += 8
    if version != VERSION:
        raise CheckpointError("unsupported checkpoint version " + str(version))
    out = {}
    for _ in range(n):
        if len(buf) < o + 4:
            raise CheckpointError("truncated checkpoint: " + path)
        (ln,) = struct.unpack_from("<I", buf, o)
        o += 4
        name = buf[o:o + ln].decode()
        o += ln
        if len(buf) < o + 8:
            raise CheckpointError("truncated checkpoint: " + path)
        (cnt,) = struct.unpack_from("<Q", buf, o)
        o += 8
        if len(buf) < o + 8 * cnt:
            raise CheckpointError("truncated checkpoint: " + path)
        out[name] = np.frombuffer(buf, dtype="<f8", count=cnt, offset=o).copy()
        o += 8 * cnt
    return out


def expect(c: dict, name: str, count: int) -> np.ndarray:
    """Checkpoint::expect (checkpoint_io.hpp:40-47)."""
    if name not in c:
        raise CheckpointError("checkpoint: missing entry '" + name + "'")
    a = c[name]
    if a.size != count:
        raise CheckpointError("checkpoint: entry '%s' has %d values, model needs %d" % (name, a.size, count))
    return a


# ---------------- trainer snapshot / restore ----------------

def _flat(params):
    import torch
    return torch.cat([p.detach().reshape(-1).double() for p in params]).cpu().numpy()


def _unflat(params, arr):
    import torch
    o = 0
    with torch.no_grad():
        for p in params:
            n = p.numel()
            p.copy_(torch.as_tensor(arr[o:o + n], dtype=p.dtype, device=p.device).view_as(p))
            o += n


def _put_opt(c, prefix, opt, params):
    """detail::put_opt (checkpoint_io.hpp:115-120): AdamW moments + step."""
    st = [opt.state.get(p, {}) for p in params]
    if all("m" in s for s in st):  # sapo.AdamWRef: moments m, v and the step count (nets.hpp:289-290)
        c[prefix + ".m"] = _flat([s["m"] for s in st])
        c[prefix + ".v"] = _flat([s["v"] for s in st])
        step = int(opt.step_count)
    else:
        c[prefix + ".m"] = np.zeros(0)
        c[prefix + ".v"] = np.zeros(0)
        step = 0
    c[prefix + ".step"] = np.array([pack_u64(step)])


def _get_opt(c, prefix, opt, params):
    """detail::get_opt (checkpoint_io.hpp:122-138)."""
    import torch
    n_params = sum(p.numel() for p in params)
    if prefix + ".m" not in c:
        raise CheckpointError("checkpoint: missing entry '" + prefix + ".m'")
    if prefix + ".v" not in c:
        raise CheckpointError("checkpoint: missing entry '" + prefix + ".v'")
    m, v = c[prefix + ".m"], c[prefix + ".v"]
    if m.size and m.size != n_params:
        raise CheckpointError("checkpoint: entry '%s.m' has %d values, model needs %d" % (prefix, m.size, n_params))
    if v.size != m.size:
        raise CheckpointError("checkpoint: optimizer moment shapes disagree in '" + prefix + "'")
    step = unpack_u64(expect(c, prefix + ".step", 1)[0])
    opt.state.clear()
    opt.step_count = step
    if m.size:
        o = 0
        for p in params:
            k = p.numel()
            opt.state[p] = {
                "m": torch.as_tensor(m[o:o + k], dtype=p.dtype, device=p.device).view_as(p).clone(),
                "v": torch.as_tensor(v[o:o + k], dtype=p.dtype, device=p.device).view_as(p).clone()}
            o += k


def snapshot_trainer(tr) -> dict:
    """snapshot_trainer (checkpoint_io.hpp:140-170) for sapo.SapoTrainer."""
    c = {}
    c["meta"] = np.array([float(tr.iter), float(tr.iter * tr.H * tr.E), float(tr.log_alpha.detach()),
                          float(getattr(tr, "last_return_mean", 0.0)), float(getattr(tr, "last_return_std", 0.0))])
    actor = list(tr.actor.parameters())
    c["policy"] = _flat(actor)
    _put_opt(c, "opt.actor", tr.actor_opt, actor)
    for k, (crit, opt) in enumerate(zip(tr.critics, tr.critic_opts)):
        ps = list(crit.parameters())
        c["critic.%d" % k] = _flat(ps)
        _put_opt(c, "opt.critic.%d" % k, opt, ps)
    _put_opt(c, "opt.alpha", tr.alpha_opt, [tr.log_alpha])
    # the state the next iteration starts from (SapoTrainer resets to it)
    st = {k: t.detach().cpu().numpy() for k, t in zip("xvFC", (tr.x0, tr.v0, tr.F0, tr.C0))}
    for i in range(tr.E):
        p = "env.%d" % i
        c[p + ".state"] = np.concatenate([st[k][i].astype(np.float64).ravel() for k in ("x", "v", "F", "C")])
        c[p + ".cursor"] = np.array([float(getattr(tr, "cursor", 0))])
        key, ctr = tr.env_rng(i)
        c[p + ".rng"] = np.array([pack_u64(key), pack_u64(ctr)])
        c[p + ".ep_return"] = np.array([0.0])
    g = tr.noise_gen.get_state().cpu().numpy().astype(np.uint8)
    pad = (-g.size) % 8
    words = np.concatenate([g, np.zeros(pad, np.uint8)]).view("<u8")
    c["sim.noise"] = np.array([pack_u64(int(w)) for w in words] + [pack_u64(g.size)])
    return c


def restore_trainer(tr, c: dict) -> None:
    """restore_trainer (checkpoint_io.hpp:172-205) for sapo.SapoTrainer."""
    import torch
    meta = expect(c, "meta", 5)
    actor = list(tr.actor.parameters())
    _unflat(actor, expect(c, "policy", sum(p.numel() for p in actor)))
    _get_opt(c, "opt.actor", tr.actor_opt, actor)
    for k, (crit, opt) in enumerate(zip(tr.critics, tr.critic_opts)):
        ps = list(crit.parameters())
        _unflat(ps, expect(c, "critic.%d" % k, sum(p.numel() for p in ps)))
        _get_opt(c, "opt.critic.%d" % k, opt, ps)
    _get_opt(c, "opt.alpha", tr.alpha_opt, [tr.log_alpha])
    N = tr.scene.n_per_env
    x, v, F, C = [], [], [], []
    for i in range(tr.E):
        s = expect(c, "env.%d.state" % i, 24 * N)
        x.append(s[:3 * N].reshape(N, 3))
        v.append(s[3 * N:6 * N].reshape(N, 3))
        F.append(s[6 * N:15 * N].reshape(N, 9))
        C.append(s[15 * N:].reshape(N, 9))
        expect(c, "env.%d.rng" % i, 2)
        expect(c, "env.%d.cursor" % i, 1)
        expect(c, "env.%d.ep_return" % i, 1)
    f32 = lambda a: torch.as_tensor(np.ascontiguousarray(np.stack(a), dtype=np.float32), device=tr.dev)
    tr.x0, tr.v0, tr.F0, tr.C0 = f32(x), f32(v), f32(F), f32(C)
    words = c["sim.noise"]
    n = unpack_u64(words[-1])
    raw = np.array([unpack_u64(w) for w in words[:-1]], dtype="<u8").view(np.uint8)[:n]
    tr.noise_gen.set_state(torch.as_tensor(raw.copy(), dtype=torch.uint8))
    with torch.no_grad():
        tr.log_alpha.copy_(torch.tensor(float(meta[2]), device=tr.dev))
    tr.iter = int(meta[0])
