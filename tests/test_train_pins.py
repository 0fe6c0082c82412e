"""Pins of the gate-training oracle (oracle/train_ref.py, §4)
against things other than itself:
* the soft forward at M_soft in {0, 1} (reading T2's limit) equals the hard-gated oracle
  (oracle.reuse_embed, itself pinned by brute force) and, at M = 0, the dense ViT;
* Eq. 11: Gumbel-Softmax as tau -> 0 samples the hard indicator (Monte Carlo);
* Eq. 12: blend examples of S:250-252 on the mask itself;
* Eq. 13-15: the SPEC worked examples and the hinge property;
* gradients: central finite differences of the fp64 loss;
* Adam: one step equals torch.optim.Adam (a library routine); annealing endpoints;
* the 1-5-9-13-11-12 group as a plan."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import train_ref as tr

CFG = synth.ViTConfig(layers=2, dim=64, heads=4, patch=16, img=48, ffn=128, hidden_r=64, hidden_g=8)


def _setup(B=1, seed=0):
    W = synth.make_vit(CFG, random_ln=True)
    G = synth.make_gates(CFG, tau=0.7, restore_bias=True)
    plan = oracle.group_plan()
    x, c = synth.make_train_groups(CFG, B, plan["display"], seed=seed)
    g = synth.make_gumbel((B, 6, CFG.layers, CFG.N, 2), seed=seed + 1)
    return W, G, plan, x, c, g


def test_group_plan_is_the_papers_pattern():
    """I-P-P (1, 5, 9), then 13 and the B_dist2 / B_dist1 frames 11, 12 of the last
    segment; computation order 1-5-9-13-11-12."""
    p = oracle.group_plan()
    assert p["display"].tolist() == [0, 4, 8, 10, 11, 12]
    F = oracle.FTYPES
    assert p["type"].tolist() == [F["I"], F["P"], F["P"], F["B2"], F["B1"], F["P"]]
    assert [int(p["display"][k]) + 1 for k in p["order"]] == [1, 5, 9, 13, 11, 12]
    assert p["past"].tolist() == [-1, 0, 1, 2, 3, 2] and p["future"].tolist() == [-1, -1, -1, 5, 5, -1]
    oracle.plan_levels(p)        # references precede their dependents


def test_soft_forward_hard_limit_equals_hard_oracle():
    """Reading T2: with the hard oracle's own masks forced into the soft forward (M in {0,1}),
    embeddings equal oracle.reuse_embed on the same frames and plan."""
    W, G, plan, x, c, g = _setup()
    hard = oracle.reuse_embed(CFG, W, G, x[0], c[0], plan)
    Gt = tr.gates_to_torch(G, requires_grad=False)
    soft = tr.soft_forward(CFG, W, Gt, x[0], c[0], plan, g[0], 1.0, force_masks=hard["M"])
    assert 0.05 < hard["M"][plan["type"] != 0].mean() < 0.95
    np.testing.assert_allclose(soft["Z"].numpy(), hard["Z"], rtol=0, atol=1e-10)
    # the decision logits of the soft pass are Eq. 3's (features identical in the limit)
    has = ~np.isnan(hard["d"])
    np.testing.assert_allclose(soft["d"].numpy()[has], hard["d"][has], rtol=0, atol=1e-10)


def test_soft_forward_dense_equals_vit():
    W, G, plan, x, c, g = _setup()
    Gt = tr.gates_to_torch(G, requires_grad=False)
    soft = tr.soft_forward(CFG, W, Gt, x[0], c[0], plan, g[0], 1.0, dense=True)
    np.testing.assert_allclose(soft["Z"].numpy(), oracle.dense_embed(CFG, W, x[0]), rtol=0, atol=1e-10)
    assert float(soft["M"].abs().sum()) == 0.0


def test_gumbel_softmax_low_temperature_samples_hard_indicator():
    """S:207 (reading: the "hard indicator" of a sample is the Gumbel-max decision
    1[d + g_reuse > g_recompute]): at temperature 0.01 the soft samples' mean distance to it
    over 10k samples is below 0.02; and those hard samples are Bernoulli(sigmoid(d))
    (Gumbel-max trick, 4.5 sigma), which is the tau -> 0 law of Eq. 11."""
    for d0 in (-2.0, -0.3, 0.4, 3.0):
        g = torch.from_numpy(synth.make_gumbel((10000, 2), seed=int(10 * d0) + 50).astype(np.float64))
        d = torch.full((10000,), d0, dtype=torch.float64)
        m = tr.gumbel_soft_mask(d, g[:, 0], g[:, 1], 0.01)
        hard = (d + g[:, 0] > g[:, 1]).double()
        assert float((m - hard).abs().mean()) < 0.02
        p = 1 / (1 + np.exp(-d0))
        assert abs(float(hard.mean()) - p) < 4.5 * np.sqrt(p * (1 - p) / 10000)
    with pytest.raises(ValueError):
        tr.gumbel_soft_mask(d, g[:, 0], g[:, 1], 0.0)


def test_soft_blend_examples():
    """S:250-252 on Eq. 11's output: large |d| / tau gives M -> {0, 1}; d = 0 with equal
    Gumbel draws gives exactly 0.5 (the arithmetic mean of the two paths), and dM/dd there is
    1 / (4 tau) (nonzero gradient through the gate)."""
    z = torch.zeros(3, dtype=torch.float64)
    assert torch.allclose(tr.gumbel_soft_mask(torch.tensor([-50.0, 0.0, 50.0], dtype=torch.float64), z, z, 1.0),
                          torch.tensor([0.0, 0.5, 1.0], dtype=torch.float64), atol=1e-12)
    d = torch.zeros(1, dtype=torch.float64, requires_grad=True)
    m = tr.gumbel_soft_mask(d, torch.zeros(1, dtype=torch.float64), torch.zeros(1, dtype=torch.float64), 0.5)
    (gd,) = torch.autograd.grad(m.sum(), d)
    assert abs(float(gd) - 1 / (4 * 0.5)) < 1e-12


def test_loss_examples_and_hinge():
    """S:446-466 worked examples of Eq. 13-15."""
    Z = torch.randn(4, 16, dtype=torch.float64)
    types = np.array([0, 1, 1, 2])
    M = torch.rand(4, 2, 5, dtype=torch.float64)
    assert abs(float(tr.group_losses(Z, Z, M, types, 2.0, 0.0)["l_sim"])) < 1e-12          # Z_hat = Z -> 0
    assert abs(float(tr.group_losses(Z, -Z, M, types, 2.0, 0.0)["l_sim"]) - 2.0) < 1e-12   # Z_hat = -Z -> 2
    for val in (0.0, 1.0):
        Mc = torch.full((4, 2, 5), val, dtype=torch.float64)
        assert float(tr.group_losses(Z, Z, Mc, types, 2.0, 0.0)["l_reuse"]) == val
    Mh = torch.zeros(4, 2, 5, dtype=torch.float64)
    Mh[:, :, :2] = 1.0
    Mh[:, :, 2] = 0.5                                                                      # 2.5 of 5
    assert abs(float(tr.group_losses(Z, Z, Mh, types, 2.0, 0.0)["l_reuse"]) - 0.5) < 1e-12
    # I-frame rows do not count
    MI = Mh.clone()
    MI[0] = 1.0
    assert abs(float(tr.group_losses(Z, Z, MI, types, 2.0, 0.0)["l_reuse"]) - 0.5) < 1e-12
    # l_sim = 0.1, l_reuse = 0.3, R_target = 0.5, alpha = 2 -> 0.5; l_reuse >= R_target -> l_sim
    Zh = Z.clone()
    lo = tr.group_losses(Z, Zh, torch.full((4, 2, 5), 0.3, dtype=torch.float64), types, 2.0, 0.5)
    assert abs(float(lo["l_total"]) - (float(lo["l_sim"]) + 2 * 0.2)) < 1e-12
    lo = tr.group_losses(Z, Zh, torch.full((4, 2, 5), 0.7, dtype=torch.float64), types, 2.0, 0.5)
    assert float(lo["l_total"]) == float(lo["l_sim"])
    with pytest.raises(ValueError):
        tr.group_losses(Z, Z, M, np.zeros(4), 2.0, 0.5)


def _fd_check(W, G, plan, x, c, g, tau, alpha, R_target, names, coords=3, h=1e-5, seed=0):
    loss, grads, outs = tr.loss_and_grads(CFG, W, G, x, c, plan, g, tau, alpha, R_target)
    feats = [o["features"] for o in outs]      # T3: the finite differences hold them fixed
    rng = np.random.default_rng(seed)
    Z_ref = []
    with torch.no_grad():
        Gt0 = tr.gates_to_torch(G, requires_grad=False)
        for b in range(x.shape[0]):
            Z_ref.append(tr.soft_forward(CFG, W, Gt0, x[b], c[b], plan, g[b], 1.0, dense=True)["Z"].numpy())

    def L(Gd):
        with torch.no_grad():
            v, _ = tr.batch_loss(CFG, W, tr.gates_to_torch(Gd, requires_grad=False), x, c, plan, g, tau, alpha,
                                 R_target, Z_ref=Z_ref, features=feats)
        return float(v)
    checked = 0
    for name in names:
        a = np.asarray(G[name], np.float64)
        for _ in range(coords):
            idx = tuple(int(rng.integers(s)) for s in a.shape)
            Gp = {k: np.asarray(v, np.float64).copy() for k, v in G.items()}
            Gm = {k: np.asarray(v, np.float64).copy() for k, v in G.items()}
            Gp[name][idx] += h
            Gm[name][idx] -= h
            fd = (L(Gp) - L(Gm)) / (2 * h)
            an = grads[name][idx]
            assert abs(fd - an) <= 1e-6 + 1e-4 * abs(an), (name, idx, fd, an)
            checked += 1
    return grads, checked


def test_gradients_match_finite_differences():
    """S:466 "gradient of total w.r.t. decision logits nonzero when hinge active [finite
    difference]" and S:268 gradient reachability: every gate array of both layers, autograd
    vs central differences of the fp64 loss, hinge active (R_target = 0.9)."""
    W, G, plan, x, c, g = _setup(B=2, seed=3)
    G = {k: np.asarray(v, np.float64) for k, v in G.items()}
    names = [n for n, _ in synth.gate_array_order(CFG)]
    grads, checked = _fd_check(W, G, plan, x, c, g, 0.7, 2.0, 0.9, names, coords=2)
    assert checked == 2 * len(names)
    last = f"L{CFG.layers - 1}."
    for n in names:
        if n.startswith(last) and n[len(last):] in ("Wr1", "br1", "Wr2", "br2"):
            # Z = LN_post(X_L[CLS]) never reads the last layer's patch outputs: exactly zero
            assert np.abs(grads[n]).max() == 0, n
        else:                            # reachability: no other gate array is cut off
            assert np.abs(grads[n]).max() > 0, n


def test_hinge_inactive_removes_reuse_gradient():
    """d l_total / d l_reuse = 0 when l_reuse > R_target: with R_target = 0 the
    gradient does not depend on alpha."""
    W, G, plan, x, c, g = _setup(seed=5)
    _, g0, _ = tr.loss_and_grads(CFG, W, G, x, c, plan, g, 0.7, 0.0, 0.0)
    _, g5, _ = tr.loss_and_grads(CFG, W, G, x, c, plan, g, 0.7, 5.0, 0.0)
    for k in g0:
        np.testing.assert_array_equal(g0[k], g5[k])
    _, g5b, _ = tr.loss_and_grads(CFG, W, G, x, c, plan, g, 0.7, 5.0, 1.0)     # active: differs
    assert any(np.abs(g5b[k] - g0[k]).max() > 0 for k in g0 if "Wd" in k or "bd" in k)


def test_adam_step_equals_torch_optim():
    rng = np.random.default_rng(0)
    p0 = rng.standard_normal(50)
    m = np.zeros(50)
    v = np.zeros(50)
    pt = torch.tensor(p0.copy(), requires_grad=True)
    opt = torch.optim.Adam([pt], lr=3e-3, betas=(0.9, 0.999), eps=1e-8)
    p = p0.copy()
    for t in range(1, 4):
        g = rng.standard_normal(50)
        p, m, v = tr.adam_step(p, g, m, v, t, 3e-3)
        pt.grad = torch.tensor(g)
        opt.step()
    np.testing.assert_allclose(p, pt.detach().numpy(), rtol=0, atol=1e-12)


def test_temperature_schedule():
    ts = [tr.temperature(s, 50) for s in range(50)]
    assert abs(ts[0] - 5.0) < 1e-12 and abs(ts[-1] - 0.1) < 1e-12
    assert all(a > b for a, b in zip(ts, ts[1:]))
