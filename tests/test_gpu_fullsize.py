"""Parity at BASELINE.json's full size, in the launch configuration bench.py times
(ViT-L/14, 7,200-frame 1-hour video at 2 FPS, p = 0.2, one embed, CUDA graph),
on outputs the oracle can compute one by one: display frames 0-20 (prefix-closed: their
references are among them) vs the fp64 oracle.  And the multi-GPU sharding scheme (SURVEY
§8(e), D9) on one device: each of the 8 shards of the same video (contiguous refresh groups +
the right-edge I-frame halo) embedded alone reproduces the whole-video embeddings and masks of
its frames bit for bit (kernels are batch-invariant, so "N-GPU == 1-GPU bitwise")."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def video():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2506_14107_b200 import ReuseViT
    cfg = synth.CONFIGS["l14"]
    W = synth.make_vit(cfg)
    G = synth.make_gates(cfg)
    m = ReuseViT(cfg, 0)
    m.load_vit(synth.pack_vit(cfg, W))
    m.load_gates(synth.pack_gates(cfg, G))
    n = 7200
    x, c = synth.make_video_torch(cfg, n, 0.2, seed=2000)
    Z, M, _, st = m.embed(x, c)
    torch.cuda.synchronize()
    return cfg, W, G, m, x, c, Z, M, st


def test_fullsize_sampled_parity(video):
    cfg, W, G, m, x, c, Z, M, st = video
    frames = list(range(21))
    ref = oracle.reuse_embed(cfg, W, G, x[:21].cpu().numpy(), c[:21].cpu().numpy(), oracle.plan_gop(7200),
                             frames=frames)
    Zg = Z[:21].cpu().double().numpy()
    Zr = ref["Z"][:21]
    err = np.abs(Zg - Zr).max(axis=1) / np.abs(Zr).max(axis=1)
    cos = (Zg * Zr).sum(1) / np.linalg.norm(Zg, axis=1) / np.linalg.norm(Zr, axis=1)
    Mg = M[:21].cpu().numpy()
    band = np.abs(np.nan_to_num(ref["d"][:21], nan=1.0)) >= 1e-3
    agree = float((Mg == ref["M"][:21])[band].mean())
    print(f"7200 frames: reuse_all={st['reuse_all']:.3f} frames 0-20 max_rel_err={err.max():.2e} "
          f"min_cos={cos.min():.6f} mask_agree={agree:.5f}")
    assert err.max() <= 2e-2 and cos.min() >= 0.999 and agree >= 0.999
    assert 0.7 < st["reuse_all"] < 0.85


def test_shards_reproduce_whole_video_bitwise(video):
    from paper_2506_14107_b200 import plan_gop
    from paper_2506_14107_b200.dist import shard_frames
    cfg, W, G, m, x, c, Z, M, st = video
    Zc, Mc = Z.clone(), M.clone()
    world = 8
    for rank in range(world):
        f0, n_own, n_loc = shard_frames(7200, 20, rank, world)
        xs = x[f0:f0 + n_loc].contiguous()
        cs = c[f0:f0 + n_loc].clone()
        cs[0] = 0.0
        Zs, Ms, _, _ = m.embed(xs, cs, plan_gop(n_loc, 20))
        torch.cuda.synchronize()
        assert torch.equal(Zs[:n_own], Zc[f0:f0 + n_own]), rank
        assert torch.equal(Ms[:n_own], Mc[f0:f0 + n_own]), rank
