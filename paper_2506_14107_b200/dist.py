"""Multi-GPU frame-group sharding.

The reference chains of the plan never cross a refresh I-frame except for the B-frames
17, 18, 19 of a 20-frame group, which reference the NEXT group's I-frame.  So each rank takes
a contiguous run of refresh groups and additionally computes the right-edge I-frame as a halo
(dense, reference-free, its embedding discarded): no activation ever crosses a GPU.  The only
collective is the final NCCL all_gather of embeddings and reuse masks (BASELINE.json: "NCCL
over NVLink used only to gather embeddings").  torch.distributed provides the process group;
the embed itself is libreusevit's.
"""
from __future__ import annotations

from typing import Tuple


def shard_frames(n_total: int, refresh: int, rank: int, world: int) -> Tuple[int, int, int]:
    """Contiguous refresh groups per rank.  Returns (first display frame f0, frames owned,
    frames computed including the halo I-frame).  f0 is a multiple of `refresh`, so the local
    plan_gop(n_loc, refresh) is the global plan restricted to [f0, f0 + n_loc) shifted by f0."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    groups = (n_total + refresh - 1) // refresh
    g0 = groups * rank // world
    g1 = groups * (rank + 1) // world
    f0 = min(n_total, g0 * refresh)
    f1 = min(n_total, g1 * refresh)
    halo = 1 if f1 < n_total else 0
    return f0, f1 - f0, f1 - f0 + halo


def _collective_device(group, like=None):
    """Device the collective runs on: NCCL needs CUDA tensors even on a rank with no work."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return like.device if like is not None else torch.device("cpu")


def gather_rows(parts, counts, group=None):
    """All-gather per-rank row blocks of different lengths (the a15 step).

    ``parts``: this rank's tensors [>= counts[rank], ...] (rows beyond counts[rank] ignored);
    ``counts``: rows owned by every rank (known to all ranks from the sharding, so no extra
    collective).  Each tensor is padded to max(counts) rows and gathered with ONE collective
    (NCCL ``all_gather_into_tensor`` over NVLink; the list form on gloo).  A rank that owns no
    rows still takes part (its padding lives on the collective's device).  Returns the valid
    rows of all ranks concatenated in rank order, one tensor per input."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n_max = max(max(counts), 1)
    out = []
    for t in parts:
        dev = _collective_device(group, t)
        pad = torch.zeros((n_max,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
        if counts[rank]:
            pad[:counts[rank]] = t[:counts[rank]].to(dev)
        full = torch.empty((world * n_max,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(full, pad, group=group)
        else:
            dist.all_gather(list(full.chunk(world)), pad, group=group)
        out.append(torch.cat([full[r * n_max:r * n_max + counts[r]] for r in range(world)]))
    return out


def max_over_ranks(value: float, group=None) -> float:
    """Max of a per-rank float (device-timed step times: the contract's max over ranks)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_collective_device(group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def embed_sharded(model, patches, codec, refresh: int = 20, group=None, **embed_kw):
    """Embed a whole video on all ranks of `group`: every rank embeds its shard (+ halo) with
    `model.embed` and the embeddings / masks are all-gathered.  `patches`/`codec` hold the
    full video (display order) on each rank.  Returns (Z [n_total, D], masks [n_total, L, N])
    on every rank, in display order."""
    import torch
    import torch.distributed as dist
    from .api import plan_gop

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n_total = patches.shape[0]
    f0, n_own, n_loc = shard_frames(n_total, refresh, rank, world)
    x = patches[f0:f0 + n_loc].contiguous()
    c = codec[f0:f0 + n_loc].clone()
    c[0] = 0.0                       # the shard starts with an I-frame (no previous frame)
    Z, M, _, _ = model.embed(x, c, plan_gop(n_loc, refresh), **embed_kw)
    Z = torch.as_tensor(Z)
    M = torch.as_tensor(M)
    if world == 1:
        return Z[:n_own], M[:n_own]
    counts = [shard_frames(n_total, refresh, r, world)[1] for r in range(world)]
    Zg, Mg = gather_rows([Z, M], counts, group)
    return Zg, Mg


# ------------------------------------------------------------------ multi-video
def reuse_estimate(p_motion: float, refresh: int = 20, T: int = 257, N: int = 256) -> float:
    """Expected reuse_all of the SPEC plan for per-step patch motion probability p (SURVEY §8(d)
    derivation: P frames (1-p)^4, B2 1-(1-(1-p)^2)^2, B1 1-p^2, weights 4:5:10 per 19 non-I
    frames of a 20-frame group, CLS never reused).  Used only to balance work across GPUs."""
    q = 1.0 - p_motion
    rp, rb2, rb1 = q ** 4, 1.0 - (1.0 - q * q) ** 2, 1.0 - p_motion ** 2
    non_i = (4 * rp + 5 * rb2 + 10 * rb1) / 19.0
    return non_i * (refresh - 1) / refresh * N / T


def lpt_assign(costs, world: int):
    """Longest-processing-time-first assignment of independent videos to `world` ranks
    (C5 balances by estimated cost sum(1 - r_hat) per video).  Returns, per rank,
    the video indices in ascending order (videos stay whole on one GPU; no halo needed)."""
    if world < 1:
        raise ValueError("world >= 1")
    loads = [0.0] * world
    out = [[] for _ in range(world)]
    for v in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        r = min(range(world), key=lambda k: (loads[k], k))
        out[r].append(v)
        loads[r] += costs[v]
    return [sorted(o) for o in out]


def combine_plans(plans):
    """Block-diagonal plan for several independent videos embedded in one call: frame indices
    of video k are offset by the frames before it, references stay inside each video, and the
    computation order is the videos' orders one after another (every reference still precedes
    its dependents).  The runtime then batches equal dependency levels across all videos."""
    import numpy as np
    offs, acc = [], 0
    for p in plans:
        offs.append(acc)
        acc += len(p["type"])
    shift = lambda a, o: np.where(np.asarray(a) >= 0, np.asarray(a) + o, -1).astype(np.int32)
    return {"type": np.concatenate([np.asarray(p["type"], np.int8) for p in plans]),
            "past": np.concatenate([shift(p["past"], o) for p, o in zip(plans, offs)]),
            "future": np.concatenate([shift(p["future"], o) for p, o in zip(plans, offs)]),
            "order": np.concatenate([np.asarray(p["order"], np.int32) + o for p, o in zip(plans, offs)]),
            "offsets": np.asarray(offs + [acc], np.int64)}


def embed_videos(model, videos, refresh: int = 20, **embed_kw):
    """Embed several independent videos [(patches [n_k, N, pp], codec [n_k, N]), ...] in ONE
    rv_embed with the combined plan (bigger level waves than one call per video).  Returns the
    per-video (Z, masks) in input order."""
    import torch
    from .api import plan_gop
    plans = [plan_gop(int(x.shape[0]), refresh) for x, _ in videos]
    cp = combine_plans(plans)
    xs = torch.cat([torch.as_tensor(x) for x, _ in videos]).contiguous()
    cs = torch.cat([torch.as_tensor(c) for _, c in videos]).contiguous()
    plan = {k: cp[k] for k in ("type", "past", "future", "order")}
    Z, M, _, _ = model.embed(xs, cs, plan, **embed_kw)
    Z, M = torch.as_tensor(Z), torch.as_tensor(M)
    o = cp["offsets"]
    return [(Z[o[k]:o[k + 1]], M[o[k]:o[k + 1]]) for k in range(len(videos))]


def embed_videos_sharded(model, videos, costs=None, refresh: int = 20, group=None, **embed_kw):
    """C5 on `world` GPUs: videos assigned to ranks by LPT on their estimated cost (default:
    frame count), each rank embeds its videos in one call, embeddings all-gathered (NCCL;
    gloo in the CPU tests).  Returns the list of per-video Z on every rank, in input order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lens = [int(x.shape[0]) for x, _ in videos]
    if costs is None:
        costs = [float(n) for n in lens]
    assign = lpt_assign(costs, world)
    mine = assign[rank]
    outs = embed_videos(model, [videos[v] for v in mine], refresh, **embed_kw) if mine else []
    if world == 1:
        return [z for z, _ in outs]
    D = int(outs[0][0].shape[1]) if outs else int(model.cfg.dim)
    # a rank without videos contributes an empty block of the model's output dtype (fp32 for
    # libreusevit); every rank must pass the same dtype to the collective
    dt = outs[0][0].dtype if outs else getattr(model, "out_dtype", torch.float32)
    z_mine = torch.cat([z for z, _ in outs]) if outs else torch.zeros((0, D), dtype=dt)
    counts = [sum(lens[v] for v in a) for a in assign]
    (zg,) = gather_rows([z_mine], counts, group)
    res = [None] * len(videos)
    off = 0
    for r in range(world):
        for v in assign[r]:
            res[v] = zg[off:off + lens[v]]
            off += lens[v]
    return res
