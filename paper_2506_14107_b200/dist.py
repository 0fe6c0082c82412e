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
    n_max = max(shard_frames(n_total, refresh, r, world)[1] for r in range(world))
    zp = torch.zeros((n_max,) + tuple(Z.shape[1:]), dtype=Z.dtype, device=Z.device)
    mp = torch.zeros((n_max,) + tuple(M.shape[1:]), dtype=M.dtype, device=M.device)
    zp[:n_own] = Z[:n_own]
    mp[:n_own] = M[:n_own]
    zg = torch.empty((world * n_max,) + tuple(Z.shape[1:]), dtype=Z.dtype, device=Z.device)
    mg = torch.empty((world * n_max,) + tuple(M.shape[1:]), dtype=M.dtype, device=M.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(zg, zp, group=group)
        dist.all_gather_into_tensor(mg, mp, group=group)
    else:                            # gloo (CPU tests): list form
        dist.all_gather(list(zg.chunk(world)), zp, group=group)
        dist.all_gather(list(mg.chunk(world)), mp, group=group)
    parts_z, parts_m = [], []
    for r in range(world):
        _, n_r, _ = shard_frames(n_total, refresh, r, world)
        parts_z.append(zg[r * n_max:r * n_max + n_r])
        parts_m.append(mg[r * n_max:r * n_max + n_r])
    return torch.cat(parts_z), torch.cat(parts_m)
