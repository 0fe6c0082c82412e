"""Multi-GPU host logic on CPU: frame-group sharding with a halo I-frame,
and a world_size-2 gloo run of embed_sharded whose per-rank "model" is the fp64 oracle —
the gathered result must equal the single-process embedding of the whole video exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2506_14107_b200.dist import shard_frames


@pytest.mark.parametrize("n_total", [1, 19, 20, 21, 41, 100, 901, 7200])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shards_cover_and_plans_agree(n_total, world):
    g = oracle.plan_gop(n_total, 20)
    covered = []
    for r in range(world):
        f0, n_own, n_loc = shard_frames(n_total, 20, r, world)
        assert f0 % 20 == 0 or n_own == 0
        covered += list(range(f0, f0 + n_own))
        if n_loc == 0:
            continue
        loc = oracle.plan_gop(n_loc, 20)
        for j in range(n_own):
            f = f0 + j
            assert loc["type"][j] == g["type"][f]
            for k in ("past", "future"):
                want = g[k][f] - f0 if g[k][f] >= 0 else -1
                assert loc[k][j] == want, (r, f, k)
        if n_loc > n_own:                       # halo = next group's I-frame
            assert loc["type"][n_own] == 0 and g["type"][f0 + n_own] == 0
    assert covered == list(range(n_total))


class OracleModel:
    """Stand-in for ReuseViT.embed on a CPU rank: the fp64 oracle."""
    def __init__(self, cfg, W, G):
        self.cfg, self.W, self.G = cfg, W, G

    def embed(self, x, c, plan, **kw):
        out = oracle.reuse_embed(self.cfg, self.W, self.G, np.asarray(x), np.asarray(c), plan)
        return torch.from_numpy(out["Z"]), torch.from_numpy(out["M"]), None, {}


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_14107_b200 import dist as rvdist
    import paper_2506_14107_b200.api as api
    api.plan_gop = lambda n, refresh=20, reorder=True: oracle.plan_gop(n, refresh, reorder)  # host plan, no .so
    cfg = synth.CONFIGS["tiny"]
    W = synth.make_vit(cfg, random_ln=True)
    G = synth.make_gates(cfg, restore_bias=True)
    x, c = synth.make_video(cfg, 41, 0.3, seed=2001)
    Z, M = rvdist.embed_sharded(OracleModel(cfg, W, G), torch.from_numpy(x), torch.from_numpy(c), refresh=20)
    if rank == 0:
        q.put((Z.numpy(), M.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_embed_sharded_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    Z, M = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    cfg = synth.CONFIGS["tiny"]
    W = synth.make_vit(cfg, random_ln=True)
    G = synth.make_gates(cfg, restore_bias=True)
    x, c = synth.make_video(cfg, 41, 0.3, seed=2001)
    ref = oracle.reuse_embed(cfg, W, G, x, c, oracle.plan_gop(41))
    assert np.array_equal(Z, ref["Z"]) and np.array_equal(M, ref["M"])
