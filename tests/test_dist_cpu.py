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
    out_dtype = torch.float64

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


# ------------------------------------------------------------------ multi-video (C5) sharding
import itertools  # noqa: E402

from paper_2506_14107_b200.dist import combine_plans, lpt_assign, reuse_estimate  # noqa: E402


def test_reuse_estimate_matches_survey_table():
    """SURVEY §8(d) reuse sweep (derived from the plan): reuse_all at p = 1 .. 0."""
    table = {1.0: 0.00, 0.6: 0.40, 0.4: 0.59, 0.3: 0.69, 0.2: 0.78, 0.1: 0.86, 0.05: 0.91, 0.0: 0.946}
    for p, r in table.items():
        assert abs(reuse_estimate(p) - r) < 0.006, (p, reuse_estimate(p), r)


@pytest.mark.parametrize("seed", range(6))
def test_lpt_within_graham_bound(seed):
    """Every video on exactly one rank; makespan within LPT's 4/3 - 1/(3m) of the optimum
    (brute force over all assignments of 8 videos to 3 ranks)."""
    rng = np.random.default_rng(seed)
    costs = list(rng.uniform(1, 10, 8))
    m = 3
    a = lpt_assign(costs, m)
    assert sorted(v for r in a for v in r) == list(range(8))
    mk = max(sum(costs[v] for v in r) for r in a)
    opt = min(max(sum(c for c, k in zip(costs, asg) if k == r) for r in range(m))
              for asg in itertools.product(range(m), repeat=8))
    assert mk <= (4 / 3 - 1 / (3 * m)) * opt + 1e-9


def test_combined_plan_is_block_diagonal_and_valid():
    plans = [oracle.plan_gop(n) for n in (21, 5, 40, 1)]
    cp = combine_plans(plans)
    n = int(cp["offsets"][-1])
    assert sorted(cp["order"].tolist()) == list(range(n))
    pos = {int(f): i for i, f in enumerate(cp["order"])}
    for k, p in enumerate(plans):
        o0, o1 = int(cp["offsets"][k]), int(cp["offsets"][k + 1])
        for f in range(o0, o1):
            assert cp["type"][f] == p["type"][f - o0]
            for key in ("past", "future"):
                r = int(cp[key][f])
                assert (r == -1) == (p[key][f - o0] == -1)
                if r >= 0:
                    assert o0 <= r < o1 and pos[r] < pos[f]
    # the oracle's level-batched schedule of the combined plan (S:410 math-neutral batching)
    lev = oracle.plan_levels({k: cp[k] for k in ("type", "past", "future", "order")})
    assert len(lev) == n


def _worker_videos(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_14107_b200 import dist as rvdist
    import paper_2506_14107_b200.api as api
    api.plan_gop = lambda n, refresh=20, reorder=True: oracle.plan_gop(n, refresh, reorder)
    cfg = synth.CONFIGS["tiny"]
    W = synth.make_vit(cfg, random_ln=True)
    G = synth.make_gates(cfg, restore_bias=True)
    vids = []
    for k, (n, p) in enumerate([(9, 0.1), (5, 0.4), (12, 0.2)]):
        x, c = synth.make_video(cfg, n, p, seed=2100 + k)
        vids.append((torch.from_numpy(x), torch.from_numpy(c)))
    costs = [x.shape[0] * (1 - rvdist.reuse_estimate(p)) for (x, _), p in zip(vids, [0.1, 0.4, 0.2])]
    Zs = rvdist.embed_videos_sharded(OracleModel(cfg, W, G), vids, costs=costs)
    if rank == 0:
        q.put([z.numpy() for z in Zs])
    dist.barrier()
    dist.destroy_process_group()


def test_embed_videos_sharded_gloo_world2():
    """C5: independent videos LPT-assigned to 2 ranks, one combined-plan embed per rank,
    gathered per video == each video embedded alone (fp64 oracle as the per-rank model)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_videos, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    Zs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    cfg = synth.CONFIGS["tiny"]
    W = synth.make_vit(cfg, random_ln=True)
    G = synth.make_gates(cfg, restore_bias=True)
    for k, (n, p) in enumerate([(9, 0.1), (5, 0.4), (12, 0.2)]):
        x, c = synth.make_video(cfg, n, p, seed=2100 + k)
        ref = oracle.reuse_embed(cfg, W, G, x, c, oracle.plan_gop(n))
        np.testing.assert_allclose(Zs[k], ref["Z"], rtol=0, atol=1e-12)


# ------------------------------------------------------------------ gather / max helpers (bench N > 1)
def _worker_gather(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_14107_b200 import dist as rvdist
    counts = [3, 0, 5][:world]                   # rank 1 owns nothing (fewer videos than ranks)
    own = counts[rank]
    Z = torch.full((own + 1, 4), float(rank)) + torch.arange(own + 1, dtype=torch.float32)[:, None]
    M = torch.full((own + 1, 2, 3), rank, dtype=torch.uint8)
    Zg, Mg = rvdist.gather_rows([Z, M], counts)
    mx = rvdist.max_over_ranks(10.0 + rank)
    # the videos path with more ranks than videos: a rank with no video still joins the gather
    cfg = synth.CONFIGS["tiny"]
    W = synth.make_vit(cfg, random_ln=True)
    G = synth.make_gates(cfg, restore_bias=True)
    import paper_2506_14107_b200.api as api
    api.plan_gop = lambda n, refresh=20, reorder=True: oracle.plan_gop(n, refresh, reorder)
    vids = []
    for k, n in enumerate((6, 4)):
        x, c = synth.make_video(cfg, n, 0.3, seed=2200 + k)
        vids.append((torch.from_numpy(x), torch.from_numpy(c)))
    Zs = rvdist.embed_videos_sharded(OracleModel(cfg, W, G), vids)
    if rank == 0:
        q.put((Zg.numpy(), Mg.numpy(), mx, [z.numpy() for z in Zs]))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_rows_and_max_gloo_world3():
    """The bench's N > 1 collective path on CPU: ragged per-rank blocks (one rank empty) gather
    into rank order; the step time is the max over ranks; a rank without videos takes part."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 3
    procs = [ctx.Process(target=_worker_gather, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    Zg, Mg, mx, Zs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    counts = [3, 0, 5]
    wantZ = np.concatenate([np.full((n, 4), float(r)) + np.arange(n)[:, None] for r, n in enumerate(counts)])
    wantM = np.concatenate([np.full((n, 2, 3), r, np.uint8) for r, n in enumerate(counts)])
    assert np.array_equal(Zg, wantZ) and np.array_equal(Mg, wantM)
    assert mx == 12.0
    cfg = synth.CONFIGS["tiny"]
    W = synth.make_vit(cfg, random_ln=True)
    G = synth.make_gates(cfg, restore_bias=True)
    for k, n in enumerate((6, 4)):
        x, c = synth.make_video(cfg, n, 0.3, seed=2200 + k)
        ref = oracle.reuse_embed(cfg, W, G, x, c, oracle.plan_gop(n))
        np.testing.assert_allclose(Zs[k], ref["Z"], rtol=0, atol=1e-12)
