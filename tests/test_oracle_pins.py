"""Pins for the oracle (CPU only): each test ties oracle/ to something other than itself —
the paper's / SPEC's worked examples (tests/golden/), a library routine (torch fp64
F.layer_norm / F.scaled_dot_product_attention), pure-Python brute force on tiny frames,
or a closed-form invariant of the method."""
import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as Fnn

import oracle
import synth
from tests import bruteforce

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TINY = synth.CONFIGS["tiny"]
T_NAMES = {v: k for k, v in oracle.FTYPES.items()}


def _gold(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


# ------------------------------------------------------------------ plan (§3.1, §6.3)
def test_plan_golden_examples():
    g = _gold("plan.json")
    p5 = oracle.plan_gop(5)
    assert p5["order"].tolist() == g["n5"]["order"]
    assert [T_NAMES[int(t)] for t in p5["type"]] == g["n5"]["type_display"]
    assert p5["past"].tolist() == g["n5"]["past"]
    assert p5["future"].tolist() == g["n5"]["future"]
    p1 = oracle.plan_gop(1)
    assert p1["order"].tolist() == [0] and int(p1["type"][0]) == 0
    p8 = oracle.plan_gop(8)
    assert p8["order"].tolist() == g["n8"]["order"]
    for f in g["n8"]["past_only"]:
        assert p8["past"][f] >= 0 and p8["future"][f] == -1
    lev = oracle.plan_levels(p8)
    assert lev.tolist() == g["n8"]["levels"]
    assert np.bincount(lev).tolist() == g["n8"]["level_sizes"]
    p41 = oracle.plan_gop(41, refresh=20)
    assert np.flatnonzero(p41["type"] == 0).tolist() == g["n41_refresh20"]["I_frames"]


@pytest.mark.parametrize("n", list(range(1, 64)) + [256, 901, 7200])
def test_plan_dag_properties(n):
    """S:337 computed-before-used; S:339 B1 at distance 1, B2 at distance 2; every frame
    exactly once in the computation order."""
    p = oracle.plan_gop(n)
    assert sorted(p["order"].tolist()) == list(range(n))
    pos = np.empty(n, int)
    pos[p["order"]] = np.arange(n)
    for f in range(n):
        t = T_NAMES[int(p["type"][f])]
        for r in (p["past"][f], p["future"][f]):
            if r >= 0:
                assert pos[r] < pos[f]
        if t == "I":
            assert p["past"][f] == -1 and p["future"][f] == -1
        elif t == "B1":
            assert p["past"][f] == f - 1 and p["future"][f] in (-1, f + 1)
        elif t == "B2":
            assert p["past"][f] == f - 2 and p["future"][f] in (-1, f + 2)
        elif t == "P":
            assert p["past"][f] == f - 4 and p["future"][f] == -1


def test_refresh_overhead_below_5pct():
    """P:586-587 "keeps the overhead below 5%"; refresh 20 raises the I fraction by
    <= 5 percentage points over the no-refresh plan."""
    n = 7200
    with_refresh = np.mean(oracle.plan_gop(n, refresh=20)["type"] == 0)
    no_refresh = np.mean(oracle.plan_gop(n, refresh=4 * n)["type"] == 0)
    assert with_refresh - no_refresh <= 0.05 + 1e-12


def test_levels_c3_c4():
    """SURVEY §8 'Waves' (derived ASAP level sizes)."""
    assert np.bincount(oracle.plan_levels(oracle.plan_gop(256))).tolist() == [13, 13, 26, 52, 52, 52, 48]
    assert np.bincount(oracle.plan_levels(oracle.plan_gop(7200))).tolist() == [360, 360, 720, 1440, 1440, 1440, 1440]


def test_lowlatency_plan():
    """reordering disabled -> each frame references its predecessor."""
    p = oracle.plan_gop(41, reorder=False)
    assert p["order"].tolist() == list(range(41))
    assert np.flatnonzero(p["type"] == 0).tolist() == [0, 20, 40]
    assert all(p["past"][f] == f - 1 for f in range(41) if f % 20)


# ------------------------------------------------------------------ compaction (Eq. 5-6, §5.3)
def test_compaction_golden():
    g = _gold("compaction.json")
    idxC, idxR, qoff = oracle.compaction_indices(np.array(g["masks"], np.uint8))
    assert idxC.tolist() == g["idxC"] and idxR.tolist() == g["idxR"] and qoff.tolist() == g["qoff"]
    s = g["spec396"]
    T = s["T"]
    masks = np.ones((2, T), np.uint8)
    masks[0, :s["active_per_frame"][0]] = 0
    masks[1, :s["active_per_frame"][1]] = 0
    idxC, _, qoff = oracle.compaction_indices(masks)
    assert len(idxC) == s["rows"] and qoff[-1] == s["rows"]


def test_compaction_roundtrip_random():
    """S:216 reconstruct(filter(x)) = identity; partition covers all tokens."""
    rng = np.random.default_rng(0)
    for trial in range(50):
        n_w, T = rng.integers(1, 9), rng.integers(2, 40)
        masks = (rng.random((n_w, T)) < rng.random()).astype(np.uint8)
        idxC, idxR, qoff = oracle.compaction_indices(masks)
        assert len(idxC) + len(idxR) == n_w * T
        assert len(np.intersect1d(idxC, idxR)) == 0
        x = rng.standard_normal((n_w * T, 3))
        y = np.empty_like(x)
        y[idxC] = x[idxC]
        y[idxR] = x[idxR]
        assert np.array_equal(x, y)
        assert all((r % T) != 0 for r in idxR)            # CLS never reused
        for w in range(n_w):
            rows = idxC[qoff[w]:qoff[w + 1]]
            assert np.all(rows // T == w) and rows[0] % T == 0   # CLS leads its frame


# ------------------------------------------------------------------ Eq. 1 similarity
def test_similarity_examples():
    """identical -> s=1; past 0.2 / future 0.9 -> 0.9 from the future."""
    rng = np.random.default_rng(1)
    a = rng.standard_normal((5, 16))
    s, prov = oracle.similarity(a, a.copy(), None)
    np.testing.assert_allclose(s, 1.0, rtol=0, atol=1e-14)
    assert np.all(prov == 0)
    e1 = np.zeros((1, 3)); e1[0, 0] = 1
    past = np.array([[0.2, math.sqrt(1 - 0.04), 0.0]])
    fut = np.array([[0.9, 0.0, math.sqrt(1 - 0.81)]])
    s, prov = oracle.similarity(e1, past, fut)
    assert abs(s[0] - 0.9) < 1e-14 and prov[0] == 1
    s, prov = oracle.similarity(e1, e1.copy(), e1.copy())      # tie -> past
    assert prov[0] == 0
    z = np.zeros((1, 3))
    assert oracle.cosine(z, e1)[0] == 0.0                      # S:76 zero-norm -> 0


def test_cosine_bruteforce():
    rng = np.random.default_rng(2)
    a, b = rng.standard_normal((20, 33)), rng.standard_normal((20, 33))
    got = oracle.cosine(a, b)
    for i in range(20):
        assert abs(got[i] - bruteforce.cos(list(a[i]), list(b[i]))) < 1e-14


# ------------------------------------------------------------------ Eq. 2-4 gate
def _tiny_inputs(n=5, p=0.3, seed=2000, mode="bimodal", random_ln=True, restore_bias=True, **gk):
    W = synth.make_vit(TINY, random_ln=random_ln)
    G = synth.make_gates(TINY, restore_bias=restore_bias, **gk)
    x, c = synth.make_video(TINY, n, p, seed=seed, mode=mode)
    return W, G, x, c


def test_forced_logits_all_recompute_equals_dense():
    """S:205 final bias -10, zero weights -> all M=0; S:264/S:619 zero-reuse exactness:
    ReuseViT with M == 0 equals the dense ViT."""
    W, G, x, c = _tiny_inputs(n=8, zero_decision=True, final_bias=-10.0)
    plan = oracle.plan_gop(8)
    out = oracle.reuse_embed(TINY, W, G, x, c, plan)
    assert out["M"].sum() == 0
    Zd = oracle.dense_embed(TINY, W, x)
    np.testing.assert_allclose(out["Z"], Zd, rtol=0, atol=1e-12)


def test_forced_logits_all_reuse():
    """S:206 final bias +10 -> all patches reused; CLS still recomputed.  Closed
    form of the D1 reading: a P-frame with every patch reused has Z_f = Z_ref (its CLS sees
    exactly the reference's K/V at every layer)."""
    W, G, x, c = _tiny_inputs(n=5, zero_decision=True, final_bias=10.0)
    plan = oracle.plan_gop(5)
    out = oracle.reuse_embed(TINY, W, G, x, c, plan)
    nonI = plan["type"] != 0
    assert np.all(out["M"][nonI] == 1) and np.all(out["M"][~nonI] == 0)
    np.testing.assert_allclose(out["Z"][4], out["Z"][0], rtol=0, atol=1e-12)   # P-frame 4 -> I 0


def test_decision_mlp_standalone():
    """Eq. 3 as a two-layer MLP evaluated by hand-written loops."""
    G = synth.make_gates(TINY, structured=True)
    rng = np.random.default_rng(3)
    v = rng.standard_normal((6, 7))
    got = oracle.decision_mlp(G, 1, v)
    for i in range(6):
        h = bruteforce.matvec_rowvec(list(v[i]), G["L1.Wd1"].astype(float).tolist(), G["L1.bd1"].astype(float).tolist())
        ref = sum(bruteforce.qgelu(hh) * float(w) for hh, w in zip(h, G["L1.Wd2"])) + float(G["L1.bd2"][0])
        assert abs(got[i] - ref) < 1e-12


def test_structured_gate_threshold():
    """d ~ QG(16(s - 0.7)) - 1 => reuse iff s >~ 0.775 (other features add ~1e-3)."""
    G = synth.make_gates(TINY, structured=True)
    v = np.zeros((2, 7))
    v[0, 0], v[1, 0] = 0.70, 0.85
    d = oracle.decision_mlp(G, 0, v)
    assert d[0] < 0 < d[1]


# ------------------------------------------------------------------ Eq. 8-9 restoration
def test_restoration_zero_delta_and_standalone():
    """Delta = 0 with zero biases -> correction exactly 0; S:234 random Delta equals a
    standalone MLP evaluation."""
    G = synth.make_gates(TINY, restore_bias=False)
    assert np.all(oracle.restoration_mlp(G, 0, np.zeros((3, TINY.dim))) == 0)
    G = synth.make_gates(TINY, restore_bias=True)
    rng = np.random.default_rng(4)
    dR = rng.standard_normal((3, TINY.dim))
    got = oracle.restoration_mlp(G, 1, dR)
    for i in range(3):
        h = [bruteforce.qgelu(v) for v in bruteforce.matvec_rowvec(list(dR[i]), G["L1.Wr1"].astype(float).tolist(), G["L1.br1"].astype(float).tolist())]
        ref = bruteforce.matvec_rowvec(h, G["L1.Wr2"].astype(float).tolist(), G["L1.br2"].astype(float).tolist())
        np.testing.assert_allclose(got[i], ref, rtol=0, atol=1e-12)


# ------------------------------------------------------------------ dense path vs library
def _torch_vit(cfg, W, patches):
    """CLIP-style pre-norm ViT from torch library routines in float64."""
    t = {k: torch.from_numpy(np.asarray(v, np.float64)) for k, v in W.items()}
    x = torch.from_numpy(np.asarray(patches, np.float64))
    n = x.shape[0]
    D, H = cfg.dim, cfg.heads
    E = x @ t["W_pe"]
    X = torch.cat([t["cls"].expand(n, 1, D), E], dim=1) + t["pos"]
    X = Fnn.layer_norm(X, (D,), t["lnpre_g"], t["lnpre_b"], eps=1e-5)
    for l in range(cfg.layers):
        p = f"L{l}."
        h = Fnn.layer_norm(X, (D,), t[p + "ln1_g"], t[p + "ln1_b"], eps=1e-5)
        qkv = Fnn.linear(h, t[p + "Wqkv"].T, t[p + "bqkv"])
        q, k, v = qkv.split(D, dim=-1)
        sh = lambda z: z.reshape(n, -1, H, D // H).transpose(1, 2)
        o = Fnn.scaled_dot_product_attention(sh(q), sh(k), sh(v))
        o = o.transpose(1, 2).reshape(n, -1, D)
        X = X + Fnn.linear(o, t[p + "Wo"].T, t[p + "bo"])
        h = Fnn.layer_norm(X, (D,), t[p + "ln2_g"], t[p + "ln2_b"], eps=1e-5)
        a = Fnn.linear(h, t[p + "W1"].T, t[p + "b1"])
        a = a * torch.sigmoid(1.702 * a)
        X = X + Fnn.linear(a, t[p + "W2"].T, t[p + "b2"])
    return Fnn.layer_norm(X[:, 0], (D,), t["lnpost_g"], t["lnpost_b"], eps=1e-5).numpy()


@pytest.mark.parametrize("cfgname", ["tiny", "mid"])
def test_dense_equals_torch_library(cfgname):
    cfg = TINY if cfgname == "tiny" else synth.ViTConfig(layers=3, dim=96, heads=6, patch=8, img=40, ffn=384)
    W = synth.make_vit(cfg, random_ln=True, std=0.05)
    x, _ = synth.make_video(cfg, 3, 0.5)
    np.testing.assert_allclose(oracle.dense_embed(cfg, W, x), _torch_vit(cfg, W, x), rtol=0, atol=1e-10)


# ------------------------------------------------------------------ brute force, tiny
@pytest.mark.parametrize("mode,p,seed", [("bimodal", 0.3, 2000), ("continuous", 0.0, 2001)])
def test_oracle_equals_bruteforce_tiny(mode, p, seed):
    """Full ReuseViT path (decision, filtration, K/V reuse, attention, restoration,
    reconstruction) vs the pure-Python token-by-token implementation on tiny frames."""
    tau = 0.7 if mode == "bimodal" else 0.3
    W, G, x, c = _tiny_inputs(n=5, p=p, seed=seed, mode=mode, tau=tau)
    plan = oracle.plan_gop(5)
    out = oracle.reuse_embed(TINY, W, G, x, c, plan)
    Zb, Mb, db = bruteforce.run(TINY, W, G, x, c, plan)
    M = out["M"]
    assert 0 < M.sum() < M[plan["type"] != 0].size, "test needs a mix of reuse and recompute"
    for f in range(5):
        np.testing.assert_allclose(out["Z"][f], Zb[f], rtol=0, atol=1e-10)
        assert M[f].tolist() == Mb[f]
        if plan["type"][f] != 0:
            np.testing.assert_allclose(out["d"][f], np.array(db[f]), rtol=0, atol=1e-10)


def test_oracle_force_masks_bruteforce():
    """Forced masks (diagnostic mode): random mask pattern, both implementations agree."""
    W, G, x, c = _tiny_inputs(n=5, p=0.5, seed=2003)
    plan = oracle.plan_gop(5)
    rng = np.random.default_rng(5)
    fm = (rng.random((5, TINY.layers, TINY.N)) < 0.5).astype(np.uint8)
    fm[plan["type"] == 0] = 0
    out = oracle.reuse_embed(TINY, W, G, x, c, plan, force_masks=fm)
    Zb, Mb, _ = bruteforce.run(TINY, W, G, x, c, plan, force_masks=fm)
    assert np.array_equal(out["M"], fm)
    for f in range(5):
        np.testing.assert_allclose(out["Z"][f], Zb[f], rtol=0, atol=1e-10)


# ------------------------------------------------------------------ invariants
def test_duplicate_frame_invariant():
    """a P-frame identical to its reference is fully reused (s = 1 > tau) and,
    with zero restoration biases (Delta = 0 -> correction 0), Z_f = Z_ref exactly."""
    cfg = TINY
    W = synth.make_vit(cfg, random_ln=True)
    G = synth.make_gates(cfg, restore_bias=False)
    x, c = synth.make_video(cfg, 5, 0.5, duplicate_of={4: 0})
    c[4] = 0.0
    plan = oracle.plan_gop(5)
    out = oracle.reuse_embed(cfg, W, G, x, c, plan)
    assert np.all(out["M"][4] == 1)
    np.testing.assert_allclose(out["Z"][4], out["Z"][0], rtol=0, atol=1e-12)


def test_schedule_neutrality():
    """scheduling does not change math — level order == plan order, bitwise."""
    W, G, x, c = _tiny_inputs(n=8, p=0.3)
    plan = oracle.plan_gop(8)
    a = oracle.reuse_embed(TINY, W, G, x, c, plan)
    lev = oracle.plan_levels(plan)
    plan2 = dict(plan)
    plan2["order"] = np.array(sorted(plan["order"], key=lambda f: (lev[f], f)), np.int32)
    b = oracle.reuse_embed(TINY, W, G, x, c, plan2)
    assert np.array_equal(a["Z"], b["Z"]) and np.array_equal(a["M"], b["M"])


def test_frame_subset():
    W, G, x, c = _tiny_inputs(n=8, p=0.3)
    plan = oracle.plan_gop(8)
    full = oracle.reuse_embed(TINY, W, G, x, c, plan)
    sub = oracle.reuse_embed(TINY, W, G, x, c, plan, frames=[0, 4, 2, 1])
    for f in (0, 4, 2, 1):
        assert np.array_equal(full["Z"][f], sub["Z"][f])
    assert np.isnan(sub["Z"][3]).all()
    with pytest.raises(ValueError):
        oracle.reuse_embed(TINY, W, G, x, c, plan, frames=[0, 2])


# ------------------------------------------------------------------ accounting
def test_flops_closed_form():
    """dense L/14 = 162.0 GFLOP/frame, B/16 = 35.1; QKV+FFN dominate;
    restoration ~2.1% (L/14) / 2.8% (B/16) of QKV+W_o+FFN per reused token (SURVEY Q3,
    consistent with the paper's ~4% incl. decision)."""
    for name, gf in (("l14", 162.0), ("b16", 35.1)):
        cfg = synth.CONFIGS[name]
        f = oracle.flops_per_frame(cfg, np.full(cfg.layers, cfg.T), np.zeros(cfg.layers))
        assert abs(f / 1e9 - gf) < 0.05
    cfg = synth.CONFIGS["l14"]
    D = cfg.dim
    share_qkv_ffn = (6 + 16) * D * D / (24 * D * D + 4 * cfg.T * D)
    assert share_qkv_ffn > 0.85
    rest = 4 * D * cfg.hidden_r / (24 * D * D)
    assert 0.015 < rest < 0.04


def test_reuse_rates():
    """Eq. 14 mean of M; S:457-460 examples."""
    types = np.array([0, 1, 1])
    T = 5
    M = np.ones((3, 2, 4), np.uint8)
    M[0] = 0
    nonI, allr = oracle.reuse_rates(M, types, T)
    assert nonI == 1.0 and abs(allr - 16 / 30) < 1e-15
    M[:] = 0
    assert oracle.reuse_rates(M, types, T) == (0.0, 0.0)
    M[1:, :, :2] = 1
    assert oracle.reuse_rates(M, types, T)[0] == 0.5


# ------------------------------------------------------------------ embedding store (NEXT-4)
def test_store_topk_matches_exhaustive_scan():
    """S:530 'k=1 on 100 random records -> matches exhaustive scan': pure-Python loops."""
    rng = np.random.default_rng(5)
    E16 = oracle.to_fp16(rng.standard_normal((100, 24)))
    Q = rng.standard_normal((4, 24))
    idx, sc = oracle.topk_cosine(E16, Q, 3)
    for i in range(4):
        scores = []
        for r in range(100):
            e = [float(v) for v in E16[r]]
            q = [float(v) for v in Q[i]]
            dot = sum(a * b for a, b in zip(e, q))
            den = (sum(a * a for a in e) ** 0.5) * (sum(b * b for b in q) ** 0.5)
            scores.append((-(dot / den), r))
        best = sorted(scores)[:3]
        assert [r for _, r in best] == list(idx[i])
        assert np.allclose([-s for s, _ in best], sc[i], rtol=0, atol=1e-12)


def test_store_topk_examples():
    """S:529 query = stored vector -> that record first with score ~1; S:531 orthogonal query
    -> scores ~0 in index order; zero vector -> cosine 0; k > n returns all."""
    E = np.zeros((5, 8))
    E[np.arange(5), np.arange(5)] = 1.0
    E16 = oracle.to_fp16(E)
    idx, sc = oracle.topk_cosine(E16, E[3], 2)
    assert idx[0, 0] == 3 and abs(sc[0, 0] - 1.0) < 1e-12
    q = np.zeros(8)
    q[7] = 1.0                                        # orthogonal to every record
    idx, sc = oracle.topk_cosine(E16, q, 5)
    assert list(idx[0]) == [0, 1, 2, 3, 4] and np.all(sc == 0)
    idx, sc = oracle.topk_cosine(E16, np.zeros(8), 2)
    assert list(idx[0]) == [0, 1] and np.all(sc == 0)
    idx, sc = oracle.topk_cosine(E16, E[0], 7)
    assert list(idx[0, 5:]) == [-1, -1] and np.all(np.isinf(sc[0, 5:]))


def test_store_storage_arithmetic():
    """1024-dim fp16 at 2 FPS = 4 KB/s ~ 0.64% of a ~625 KB/s Full-HD H.264 stream."""
    bps = oracle.storage_bytes_per_second(1024, 2.0)
    assert bps == 4096 and abs(bps / (625 * 1024) * 100 - 0.64) < 0.005


# ------------------------------------------------------------------ SPEC chain variant (NEXT-1)
from tests import bruteforce_chain  # noqa: E402


@pytest.mark.parametrize("mode,p,seed", [("bimodal", 0.3, 2000), ("continuous", 0.0, 2001)])
def test_chain_oracle_equals_bruteforce_tiny(mode, p, seed):
    """Chain variant (FFN_l -> QKV_{l+1} gated, dense attention + W_o, S:218-220 / S:271-272) vs
    the pure-Python token-by-token implementation: embeddings and masks."""
    tau = 0.7 if mode == "bimodal" else 0.3
    W, G, x, c = _tiny_inputs(n=5, p=p, seed=seed, mode=mode, tau=tau)
    plan = oracle.plan_gop(5)
    out = oracle.reuse_embed_chain(TINY, W, G, x, c, plan)
    Zb, Mb = bruteforce_chain.run(TINY, W, G, x, c, plan)
    M = out["M"]
    assert 0 < M.sum() < M[plan["type"] != 0].size, "test needs a mix of reuse and recompute"
    for f in range(5):
        np.testing.assert_allclose(out["Z"][f], Zb[f], rtol=0, atol=1e-10)
        assert M[f].tolist() == Mb[f]


def test_chain_oracle_force_masks_bruteforce():
    W, G, x, c = _tiny_inputs(n=5, p=0.5, seed=2003)
    plan = oracle.plan_gop(5)
    rng = np.random.default_rng(6)
    fm = (rng.random((5, TINY.layers, TINY.N)) < 0.5).astype(np.uint8)
    fm[plan["type"] == 0] = 0
    out = oracle.reuse_embed_chain(TINY, W, G, x, c, plan, force_masks=fm)
    Zb, Mb = bruteforce_chain.run(TINY, W, G, x, c, plan, force_masks=fm)
    assert np.array_equal(out["M"], fm)
    for f in range(5):
        np.testing.assert_allclose(out["Z"][f], Zb[f], rtol=0, atol=1e-10)


def test_chain_oracle_zero_masks_equal_torch_library():
    """S:264 exactness at zero reuse, for the chain variant: forced M = 0 -> plain ViT."""
    cfg = TINY
    W, G, x, c = _tiny_inputs(n=5, p=0.5, seed=2004)
    plan = oracle.plan_gop(5)
    fm = np.zeros((5, cfg.layers, cfg.N), np.uint8)
    out = oracle.reuse_embed_chain(cfg, W, G, x, c, plan, force_masks=fm)
    np.testing.assert_allclose(out["Z"], _torch_vit(cfg, W, x), rtol=0, atol=1e-10)


def test_chain_duplicate_frame_invariant():
    """S:260/S:265 in the chain variant: a P-frame identical to its reference reuses every
    patch token (x' identical -> s = 1) and, with zero restoration biases, Z_f = Z_ref."""
    cfg = TINY
    W = synth.make_vit(cfg, random_ln=True)
    G = synth.make_gates(cfg, restore_bias=False)
    x, c = synth.make_video(cfg, 5, 0.5, duplicate_of={4: 0})
    c[4] = 0.0
    plan = oracle.plan_gop(5)
    out = oracle.reuse_embed_chain(cfg, W, G, x, c, plan)
    assert out["M"][4].all()
    np.testing.assert_allclose(out["Z"][4], out["Z"][0], rtol=0, atol=1e-12)
