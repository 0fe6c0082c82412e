"""Gate trainer on the GPU (include/reusevit_train.h) against the fp64
training oracle (oracle/train_ref.py, pinned in tests/test_train_pins.py) on the same seeded
groups and Gumbel draws:
* soft forward (Eq. 11-12): Z, M_soft and the decision logits d;
* dense (M = 0) forward = the frozen ViT; forced hard masks = the hard-gated oracle;
* loss (Eq. 13-15) and the gradient of every gate array (ViT frozen);
* a toy training run (1-5-9-13-11-12 groups; annealed temperature) that meets
  R_target, and whose hard-gated inference (rv_embed with the trained RVG1 blob) keeps the
  embeddings closer to the dense ViT than random reuse decisions at the same reuse rate."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import train_ref as tr

pytestmark = pytest.mark.gpu
CFG = synth.CONFIGS["tiny"]


def _inputs(B, seed, tau_gate=0.7):
    W = synth.make_vit(CFG, random_ln=True)
    G = synth.make_gates(CFG, tau=tau_gate, restore_bias=True)
    plan = oracle.group_plan()
    x, c = synth.make_train_groups(CFG, B, plan["display"], seed=seed)
    g = synth.make_gumbel((B, 6, CFG.layers, CFG.N, 2), seed=seed + 1)
    return W, G, plan, x, c, g


def _trainer(W, G, plan, B, **kw):
    from paper_2506_14107_b200.train import GateTrainer
    return GateTrainer(CFG, synth.pack_vit(CFG, W), synth.pack_gates(CFG, G), plan, groups=B, **kw)


def _cuda(a):
    if a is None:
        return None
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


@pytest.mark.parametrize("tau", [1.0, 0.3])
def test_soft_forward_parity(cuda_ok, tau):
    B = 3
    W, G, plan, x, c, g = _inputs(B, seed=11)
    t = _trainer(W, G, plan, B)
    Z, M, d = t.forward(_cuda(x), _cuda(c), _cuda(g), tau)
    torch.cuda.synchronize()
    Gt = tr.gates_to_torch(G, requires_grad=False)
    for b in range(B):
        ref = tr.soft_forward(CFG, W, Gt, x[b], c[b], plan, g[b], tau)
        Zr = ref["Z"].numpy()
        err = np.abs(Z[b].cpu().numpy() - Zr).max() / np.abs(Zr).max()
        assert err < 1e-4, err
        Mr = ref["M"].numpy()
        assert np.abs(M[b].cpu().numpy() - Mr).max() < 1e-4
        dr = ref["d"].numpy()
        dg = d[b].cpu().numpy()
        has = ~np.isnan(dr)
        assert np.array_equal(np.isnan(dg), ~has)
        assert np.all(np.abs(dg[has] - dr[has]) <= 1e-4 * (1 + np.abs(dr[has])))
        assert 0.02 < Mr[plan["type"] != 0].mean() < 0.98     # a genuinely soft mix
    t.close()


def test_dense_and_hard_limits(cuda_ok):
    B = 2
    W, G, plan, x, c, g = _inputs(B, seed=21)
    t = _trainer(W, G, plan, B)
    Zd, Md, _ = t.forward(_cuda(x), _cuda(c), None, 1.0, dense=True)
    hard = [oracle.reuse_embed(CFG, W, G, x[b], c[b], plan) for b in range(B)]
    force = np.stack([h["M"] for h in hard]).astype(np.float32)
    Zh, Mh, _ = t.forward(_cuda(x), _cuda(c), _cuda(g), 1.0, force=_cuda(force))
    torch.cuda.synchronize()
    for b in range(B):
        Zr = oracle.dense_embed(CFG, W, x[b])
        assert np.abs(Zd[b].cpu().numpy() - Zr).max() / np.abs(Zr).max() < 1e-4
        Zr = hard[b]["Z"]
        assert np.abs(Zh[b].cpu().numpy() - Zr).max() / np.abs(Zr).max() < 1e-4
        assert np.array_equal(Mh[b].cpu().numpy(), force[b])
    assert float(Md.abs().sum()) == 0.0
    t.close()


@pytest.mark.parametrize("R_target", [0.9, 0.0])
def test_loss_and_gradient_parity(cuda_ok, R_target):
    """Hinge active (0.9) and inactive (0.0): every gate array's gradient within 1e-3 of the
    fp64 autograd gradient (relative, Frobenius); the loss terms within 1e-5."""
    B, tau, alpha = 3, 0.7, 2.0
    W, G, plan, x, c, g = _inputs(B, seed=31)
    t = _trainer(W, G, plan, B, alpha=alpha, r_target=R_target)
    log, grad = t.loss_grad(_cuda(x), _cuda(c), _cuda(g), tau)
    loss, gref, outs = tr.loss_and_grads(CFG, W, G, x, c, plan, g, tau, alpha, R_target)
    assert abs(log["l_total"] - loss) < 1e-5 * (1 + abs(loss))
    assert abs(log["l_sim"] - np.mean([float(o["l_sim"]) for o in outs])) < 1e-5
    assert abs(log["l_reuse"] - np.mean([float(o["l_reuse"]) for o in outs])) < 1e-5
    gg = grad.cpu().numpy().astype(np.float64)
    off = 0
    for name, shape in synth.gate_array_order(CFG):
        n = int(np.prod(shape))
        a, r = gg[off:off + n], gref[name].reshape(-1)
        off += n
        scale = np.linalg.norm(r)
        assert np.linalg.norm(a - r) <= 1e-3 * scale + 1e-9, (name, np.linalg.norm(a - r), scale)
    assert off == gg.size
    t.close()


def test_toy_training_meets_target_and_beats_random_reuse(cuda_ok):
    """A toy run (tools/train_gates.py settings): a random ViT whose CLS embedding depends on
    the frame content (init std 0.3), 256 training groups of 1-5-9-13-11-12 frames, minibatches
    of 16, 300 Adam steps, temperature annealed 5 -> 0.1, R_target = 0.5, alpha = 2.
    Checks: the loss falls below half its start; the hard-gated inference path (Eq. 4) with the
    trained RVG1 blob reuses >= 0.35 of the non-I tokens of held-out video (the initial
    recompute-leaning gates reuse none); its embeddings stay closer to the dense ViT (1 - cos)
    than random reuse decisions at the same per-layer rate, and than reusing everything."""
    from paper_2506_14107_b200 import ReuseViT
    W = synth.make_vit(CFG, random_ln=True, std=0.3)
    G0 = synth.init_train_gates(CFG)
    plan = oracle.group_plan()
    pool, B, steps = 256, 16, 300
    x, c = synth.make_train_groups(CFG, pool, plan["display"], seed=77)
    xd, cd = _cuda(x), _cuda(c)
    t = _trainer(W, G0, plan, B, alpha=2.0, r_target=0.5, lr=3e-3)
    rng = np.random.default_rng(78)
    logs = []
    for s in range(steps):
        idx = torch.from_numpy(rng.choice(pool, B, replace=False)).cuda()
        g = synth.make_gumbel((B, 6, CFG.layers, CFG.N, 2), seed=10_000 + s)
        logs.append(t.step(xd[idx].contiguous(), cd[idx].contiguous(), _cuda(g), tr.temperature(s, steps)))
    first = np.mean([l["l_total"] for l in logs[:10]])
    last = np.mean([l["l_total"] for l in logs[-10:]])
    print(f"train: l_total {first:.4f} -> {last:.4f}; last l_reuse {logs[-1]['l_reuse']:.3f} "
          f"l_sim {logs[-1]['l_sim']:.5f}")
    assert last < 0.5 * first
    assert logs[-1]["l_reuse"] >= 0.45           # the hinge holds the soft reuse near R_target
    blob = t.gates()
    t.close()
    # hard-gated inference with the trained gates on a held-out 41-frame video
    m = ReuseViT(CFG, 0)
    m.load_vit(synth.pack_vit(CFG, W))
    m.load_gates(blob)
    xv, cv = synth.make_video(CFG, 41, 0.2, seed=909)
    Z, M, _, st = m.embed(_cuda(xv), _cuda(cv))
    Zd, _, _, _ = m.embed(_cuda(xv), _cuda(cv), dense=True)
    torch.cuda.synchronize()
    Mh = M.cpu().numpy()
    types = oracle.plan_gop(41)["type"]
    nonI = types != 0
    reuse = Mh[nonI].mean()
    cos = lambda A, Bm: (A * Bm).sum(1) / np.linalg.norm(A, axis=1) / np.linalg.norm(Bm, axis=1)
    Zdn = Zd.cpu().numpy().astype(np.float64)
    err = lambda Zx: float(np.mean(1 - cos(Zx.cpu().numpy().astype(np.float64), Zdn)))
    err_trained = err(Z)
    # random decisions at the same per-layer rate, and all-reuse (forced masks, same path)
    fm = np.zeros_like(Mh)
    rr = np.random.default_rng(6)
    for l in range(CFG.layers):
        rate = Mh[nonI, l].mean()
        fm[nonI, l] = (rr.random((int(nonI.sum()), CFG.N)) < rate).astype(np.uint8)
    Zr, _, _, _ = m.embed(_cuda(xv), _cuda(cv), force_masks=torch.from_numpy(fm))
    fa = np.zeros_like(Mh)
    fa[nonI] = 1
    Za, _, _, _ = m.embed(_cuda(xv), _cuda(cv), force_masks=torch.from_numpy(fa))
    torch.cuda.synchronize()
    err_random, err_all = err(Zr), err(Za)
    print(f"hard inference: reuse {reuse:.3f}  1-cos trained {err_trained:.3e}  random {err_random:.3e}  "
          f"all-reuse {err_all:.3e}")
    assert reuse >= 0.35
    assert err_trained < 0.75 * err_random and err_trained < err_all
    m.close()
