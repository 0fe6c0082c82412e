"""Per-kernel GPU tests through the C-ABI stage entry points (include/reusevit_stages.h).

* GEMM (tcgen05/TMEM/TMA): vs a plain PyTorch fp32 matmul of the same bf16 operands.
* attention (compacted queries over all keys): vs plain PyTorch fp32 softmax attention of the
  same bf16 q/K/V, and the CLS head-mean probabilities.
* score (Eq. 1-4): teacher-forced with the ORACLE's X_{l-1} and t; d within 1e-5*(1+|d|),
  masks equal outside the 1e-3 band, provider/cntC consistent.
* compaction (Eq. 5-6): bit-exact vs oracle.compaction_indices.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(cuda_ok):
    return torch.device("cuda:0")


def _model(cfg, gates=True, **gk):
    from paper_2506_14107_b200 import ReuseViT
    m = ReuseViT(cfg, 0)
    W = synth.make_vit(cfg, random_ln=True)
    m.load_vit(synth.pack_vit(cfg, W))
    G = synth.make_gates(cfg, restore_bias=True, **gk)
    if gates:
        m.load_gates(synth.pack_gates(cfg, G))
    return m, W, G


# ------------------------------------------------------------------------- GEMM
@pytest.mark.parametrize("M,N,K", [(1, 64, 64), (100, 192, 64), (128, 256, 1024), (300, 768, 768),
                                   (1000, 3072, 1024), (4097, 1024, 4096), (257, 128, 1024),
                                   (513, 1024, 128), (20000, 4096, 1024),
                                   # CTA-pair path (BN = 256): a lone row, rank 1 holding 1 row, ragged tails
                                   (1, 256, 64), (129, 1024, 256), (383, 512, 4096), (70001, 1024, 1024)])
def test_gemm_vs_torch(dev, M, N, K):
    m, _, _ = _model(synth.CONFIGS["tiny"], gates=False)
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16)
    B = (0.05 * torch.randn(N, K, generator=g)).to(torch.bfloat16)
    bias = torch.randn(N, generator=g)
    ref = A.float() @ B.float().T + bias
    out = m.stage_gemm(A.to(dev), B.to(dev), bias.to(dev))
    torch.cuda.synchronize()
    err = (out.cpu() - ref).abs().max().item()
    assert err <= 1e-3 * (1 + ref.abs().max().item()), err
    # QuickGELU epilogue, bf16 output
    out2 = m.stage_gemm(A.to(dev), B.to(dev), bias.to(dev), act=1, out_bf16=True)
    torch.cuda.synchronize()
    ref2 = ref * torch.sigmoid(1.702 * ref)
    err2 = (out2.cpu().float() - ref2).abs().max().item()
    assert err2 <= 1e-2 * (1 + ref2.abs().max().item()), err2


def test_gemm_row_position_invariance(dev):
    """Batch invariance: a row's result does not depend on M or its position."""
    m, _, _ = _model(synth.CONFIGS["tiny"], gates=False)
    g = torch.Generator(device="cpu").manual_seed(0)
    A = torch.randn(1000, 1024, generator=g).to(torch.bfloat16).to(dev)
    B = (0.05 * torch.randn(1024, 1024, generator=g)).to(torch.bfloat16).to(dev)
    full = m.stage_gemm(A, B)
    part = m.stage_gemm(A[333:334].contiguous(), B)
    shifted = m.stage_gemm(A[300:700].contiguous(), B)
    torch.cuda.synchronize()
    assert torch.equal(full[333], part[0])
    assert torch.equal(full[300:700], shifted)


@pytest.mark.parametrize("M,N,K,act", [(700, 1024, 128, 0), (5000, 768, 128, 0), (1000, 1024, 1024, 0),
                                       (300, 4096, 1024, 1)])
def test_gemm_row_mapped_epilogue_vs_torch(dev, M, N, K, act):
    """Row-mapped epilogue (W_o / FC2 / restoration R2, Eq. 9-10): gathered fp32 residual rows,
    scattered output rows (entries < 0 skipped); K = 128 takes the short-K streaming variant."""
    cfg = synth.CONFIGS["b16"]
    m, _, _ = _model(cfg, gates=False)
    g = torch.Generator(device=dev).manual_seed(M + N)
    A = (0.5 * torch.randn(M, K, device=dev, generator=g)).to(torch.bfloat16)
    B = (0.05 * torch.randn(N, K, device=dev, generator=g)).to(torch.bfloat16)
    bias = torch.randn(N, device=dev, generator=g)
    rows = 3 * M
    resid = torch.randn(rows, N, device=dev, generator=g)
    rrows = torch.randperm(rows, device=dev, generator=g)[:M].to(torch.int32)
    orows = torch.randperm(rows, device=dev, generator=g)[:M].to(torch.int32)
    orows[::7] = -1
    out = torch.full((rows, N), 7.0, device=dev)
    m.stage_gemm_rows(A, B, out, bias=bias, act=act, resid=resid, resid_rows=rrows, out_rows=orows)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().T + bias
    if act:
        ref = ref * torch.sigmoid(1.702 * ref)
    ref = ref + resid[rrows.long()]
    keep = orows >= 0
    got = out[orows[keep].long()]
    assert (got - ref[keep]).abs().max().item() < 2e-2 * (1 + ref.abs().max().item() * 1e-2)
    untouched = torch.ones(rows, dtype=torch.bool, device=dev)
    untouched[orows[keep].long()] = False
    assert torch.all(out[untouched] == 7.0)


# ------------------------------------------------------------------------- attention
# use_tc: False mma.sync; True tcgen05 (persistent kernel for T <= 257, general kernel for
# T = 577); 2 the general tcgen05 kernel (128-query tiles, online softmax over key blocks)
@pytest.mark.parametrize("cfgname,use_tc", [("tiny", False), ("b16", False), ("l14", False), ("l14_336", False),
                                            ("b16", True), ("l14", True), ("l14_336", True), ("b16", 2),
                                            ("l14", 2)])
def test_attention_vs_torch(dev, cfgname, use_tc):
    cfg = synth.CONFIGS[cfgname]
    m, _, _ = _model(cfg, gates=False)
    T, D, H, dh = cfg.T, cfg.dim, cfg.heads, cfg.dh
    rng = np.random.default_rng(1)
    slots = 5
    n_w = 4
    slot_of = np.array([3, 0, 4, 1], np.int32)
    nq = np.array([T, 1, 37, 130 if T > 130 else T - 3])      # full frame, CLS only, ragged
    qoff = np.concatenate([[0], np.cumsum(nq)]).astype(np.int32)
    q = torch.from_numpy(rng.standard_normal((qoff[-1], D)).astype(np.float32)).to(torch.bfloat16)
    KV = torch.from_numpy(rng.standard_normal((slots * T, 2 * D)).astype(np.float32)).to(torch.bfloat16)
    wdesc = np.zeros((n_w, 4), np.int32)
    wdesc[:, 0] = slot_of
    out = torch.zeros((qoff[-1], D), dtype=torch.bfloat16, device=dev)
    pcls = torch.zeros((slots, H, cfg.N), dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream()
    m.stage_attention(torch.from_numpy(wdesc).to(dev), torch.from_numpy(qoff).to(dev), q.to(dev), KV.to(dev),
                      out, pcls, st, use_tc=use_tc)
    torch.cuda.synchronize()
    for w in range(n_w):
        s = slot_of[w]
        Kf = KV[s * T:(s + 1) * T].float().reshape(T, H, 2, dh)[:, :, 0].transpose(0, 1)
        Vf = KV[s * T:(s + 1) * T].float().reshape(T, H, 2, dh)[:, :, 1].transpose(0, 1)
        qf = q[qoff[w]:qoff[w + 1]].float().reshape(-1, H, dh).transpose(0, 1)
        P = torch.softmax(qf @ Kf.transpose(1, 2) / dh ** 0.5, dim=-1)
        ref = (P @ Vf).transpose(0, 1).reshape(-1, D)
        got = out[qoff[w]:qoff[w + 1]].cpu().float()
        assert (got - ref).abs().max().item() < 2e-2 * (1 + ref.abs().max().item())
        tref = P[:, 0, 1:]                       # per-head CLS softmax row over patch keys
        assert (pcls[s].cpu() - tref).abs().max().item() < 1e-4


@pytest.mark.parametrize("cfgname,use_tc", [("b16", False), ("l14", False), ("l14_336", False), ("b16", True),
                                            ("l14", True), ("l14_336", True), ("l14", 2)])
def test_attention_wave_kvsrc(dev, cfgname, use_tc):
    """A level-wave-sized launch: 300 frames in shuffled slots, ragged query counts (1 .. T,
    mostly the 30-70 of the paper's reuse rates), K/V rows read through a random reuse-cache
    table (a7: reused tokens point at another slot's row of the same token), vs torch fp32."""
    cfg = synth.CONFIGS[cfgname]
    m, _, _ = _model(cfg, gates=False)
    T, D, H, dh = cfg.T, cfg.dim, cfg.heads, cfg.dh
    rng = np.random.default_rng(7)
    n_w = 300
    slot_of = rng.permutation(n_w).astype(np.int32)
    nq = rng.integers(30, 71, n_w)
    nq[::20] = T
    nq[5::37] = 1
    nq[7::41] = 64
    nq[9::43] = 65
    qoff = np.concatenate([[0], np.cumsum(nq)]).astype(np.int32)
    kvsrc = np.arange(n_w * T, dtype=np.int32).reshape(n_w, T)
    other = rng.integers(0, n_w, (n_w, T))
    reuse = rng.random((n_w, T)) < 0.7
    reuse[:, 0] = False
    kvsrc[reuse] = (other * T + np.arange(T)[None, :])[reuse]
    g = torch.Generator(device=dev).manual_seed(3)
    q = torch.randn(int(qoff[-1]), D, device=dev, generator=g).to(torch.bfloat16)
    KV = torch.randn(n_w * T, 2 * D, device=dev, generator=g).to(torch.bfloat16)
    wdesc = np.zeros((n_w, 4), np.int32)
    wdesc[:, 0] = slot_of
    out = torch.zeros((int(qoff[-1]), D), dtype=torch.bfloat16, device=dev)
    pcls = torch.zeros((n_w, H, cfg.N), dtype=torch.float32, device=dev)
    kv_d = torch.from_numpy(kvsrc).to(dev)
    m.stage_attention(torch.from_numpy(wdesc).to(dev), torch.from_numpy(qoff).to(dev), q, KV, out, pcls,
                      torch.cuda.current_stream(), use_tc=use_tc, kvsrc=kv_d)
    torch.cuda.synchronize()
    worst, worst_p = 0.0, 0.0
    for w in range(n_w):
        s = int(slot_of[w])
        rows = kv_d[s].long()
        Kf = KV[rows].float().reshape(T, H, 2, dh)[:, :, 0].transpose(0, 1)
        Vf = KV[rows].float().reshape(T, H, 2, dh)[:, :, 1].transpose(0, 1)
        qf = q[qoff[w]:qoff[w + 1]].float().reshape(-1, H, dh).transpose(0, 1)
        P = torch.softmax(qf @ Kf.transpose(1, 2) / dh ** 0.5, dim=-1)
        ref = (P @ Vf).transpose(0, 1).reshape(-1, D)
        got = out[qoff[w]:qoff[w + 1]].float()
        worst = max(worst, (got - ref).abs().max().item() / (1 + ref.abs().max().item()))
        worst_p = max(worst_p, (pcls[s] - P[:, 0, 1:]).abs().max().item())
    assert worst < 2e-2, worst
    assert worst_p < 1e-4, worst_p


@pytest.mark.parametrize("boost_block", [0, 2, 4])
def test_attention_tcg_online_rescale(dev, boost_block):
    """The general tcgen05 kernel's lazy online softmax: keys of one 128-key block are scaled
    up 6x so that block dominates the row maxima.  Block 0 boosted: no later rescale; blocks
    2 / 4 (the ragged last block of T = 577): the running max jumps by far more than 2^8 and
    O in TMEM is rescaled mid-row.  Output and CLS probabilities vs torch fp32."""
    cfg = synth.CONFIGS["l14_336"]
    m, _, _ = _model(cfg, gates=False)
    T, D, H, dh = cfg.T, cfg.dim, cfg.heads, cfg.dh
    g = torch.Generator(device=dev).manual_seed(40 + boost_block)
    n_w = 3
    nq = np.array([T, 130, 1])
    qoff = np.concatenate([[0], np.cumsum(nq)]).astype(np.int32)
    q = torch.randn(int(qoff[-1]), D, device=dev, generator=g).to(torch.bfloat16)
    KVf = torch.randn(n_w * T, 2 * D, device=dev, generator=g)
    for w in range(n_w):
        lo = w * T + boost_block * 128
        KVf[lo:min(lo + 128, (w + 1) * T), :D] *= 6.0
    KV = KVf.to(torch.bfloat16)
    wdesc = np.zeros((n_w, 4), np.int32)
    wdesc[:, 0] = np.arange(n_w)
    out = torch.zeros((int(qoff[-1]), D), dtype=torch.bfloat16, device=dev)
    pcls = torch.zeros((n_w, H, cfg.N), dtype=torch.float32, device=dev)
    m.stage_attention(torch.from_numpy(wdesc).to(dev), torch.from_numpy(qoff).to(dev), q, KV, out, pcls,
                      torch.cuda.current_stream(), use_tc=2)
    torch.cuda.synchronize()
    for w in range(n_w):
        Kf = KV[w * T:(w + 1) * T].float().reshape(T, H, 2, dh)[:, :, 0].transpose(0, 1)
        Vf = KV[w * T:(w + 1) * T].float().reshape(T, H, 2, dh)[:, :, 1].transpose(0, 1)
        qf = q[qoff[w]:qoff[w + 1]].float().reshape(-1, H, dh).transpose(0, 1)
        P = torch.softmax(qf @ Kf.transpose(1, 2) / dh ** 0.5, dim=-1)
        ref = (P @ Vf).transpose(0, 1).reshape(-1, D)
        got = out[qoff[w]:qoff[w + 1]].float()
        assert (got - ref).abs().max().item() < 2e-2 * (1 + ref.abs().max().item())
        assert (pcls[w] - P[:, 0, 1:]).abs().max().item() < 1e-4


# ------------------------------------------------------------------------- score (teacher forced)
# generic (tiny), VPL = 6 (B/16, D = 768) and VPL = 8 (L/14 and L/14@336, D = 1024: the path the
# bench runs) loops; bimodal (bench workloads) and continuous (s spread over (0, 1), tokens near
# the threshold: SURVEY §8(d) continuous stress mode, tau = 0.3)
@pytest.mark.parametrize("cfgname,mode,n", [("tiny", "continuous", 8), ("b16", "bimodal", 9), ("b16", "continuous", 9),
                                            ("l14", "bimodal", 6), ("l14", "continuous", 6),
                                            ("l14_336", "bimodal", 6), ("l14_336", "continuous", 6)])
def test_score_teacher_forced(dev, cfgname, mode, n):
    cfg = synth.CONFIGS[cfgname]
    tau = 0.7 if mode == "bimodal" else 0.3
    m, W, G = _model(cfg, tau=tau)
    x, c = synth.make_video(cfg, n, 0.3 if mode == "bimodal" else 0.0, seed=2010, mode=mode)
    plan = oracle.plan_gop(n)
    ref = oracle.reuse_embed(cfg, W, G, x, c, plan, trace=True)
    T, N, D, L = cfg.T, cfg.N, cfg.dim, cfg.layers
    lev = oracle.plan_levels(plan)
    frames = [f for f in plan["order"] if plan["type"][f] != 0]
    wdesc = np.array([[f, plan["past"][f], plan["future"][f], plan["type"][f]] for f in frames], np.int32)
    st = torch.cuda.current_stream()
    checked = 0
    for l in range(L):
        X = np.stack([ref["X"][f][l] for f in range(n)]).astype(np.float32)      # [n, T, D]
        t = np.nan_to_num(ref["t"][:, l, :], nan=0.0).astype(np.float32)
        Xd = torch.from_numpy(X).to(dev)
        masks = torch.zeros((n, L, N), dtype=torch.uint8, device=dev)
        scores = torch.zeros((n, L, N), dtype=torch.float32, device=dev)
        wmask = torch.zeros((len(frames), T), dtype=torch.uint8, device=dev)
        wprov = torch.zeros_like(wmask)
        cntR = torch.zeros(len(frames), dtype=torch.int32, device=dev)
        m.stage_score(l, Xd, torch.from_numpy(wdesc).to(dev), torch.from_numpy(t).to(dev),
                      torch.from_numpy(c).to(dev), None, masks, scores, wmask, wprov, cntR, st)
        torch.cuda.synchronize()
        d_ref = ref["d"][:, l, :]
        d_gpu = scores[:, l, :].cpu().double().numpy()
        for f in frames:
            assert np.all(np.abs(d_gpu[f] - d_ref[f]) <= 1e-5 * (1 + np.abs(d_ref[f]))), (l, f)
            band = np.abs(d_ref[f]) >= 1e-3
            assert np.array_equal(masks[f, l].cpu().numpy()[band], ref["M"][f, l][band])
            checked += band.sum()
        # provider (Eq. 1 argmax, ties -> past) on frames with two references, wherever the two
        # fp64 cosines differ by more than fp32 rounding can reorder
        pv = wprov.cpu().numpy()
        for k, f in enumerate(frames):
            pa, fu = plan["past"][f], plan["future"][f]
            if pa >= 0 and fu >= 0:
                cur = X[f, 1:].astype(np.float64)
                cos = lambda r: (cur * X[r, 1:]).sum(1) / np.sqrt((cur * cur).sum(1) * (X[r, 1:].astype(np.float64) ** 2).sum(1))
                sp, sf = cos(pa), cos(fu)
                clear = np.abs(sp - sf) > 1e-5
                assert np.array_equal(pv[k, 1:][clear], (sf > sp)[clear].astype(np.uint8)), (l, f)
                assert np.array_equal(ref["prov"][f, l][clear], (sf > sp)[clear].astype(np.int8))
        wm = wmask.cpu().numpy()
        assert np.all(wm[:, 0] == 0)
        assert np.array_equal(cntR.cpu().numpy(), wm.sum(1))
    assert checked > 0


# ------------------------------------------------------------------------- compaction
def _compaction_case(dev, cfg, n_w, p, seed):
    """Random level-wave of n_w frames (random slots, providers, masks at reuse rate p) through
    rv_stage_compact; bit-exact vs oracle.compaction_indices (north star: compaction indices and
    gathered token order bit-exact given the same mask)."""
    from paper_2506_14107_b200 import ReuseViT
    m = ReuseViT(cfg, 0)            # compaction needs only T from the context (no weights)
    T = cfg.T
    rng = np.random.default_rng(seed)
    masks = (rng.random((n_w, T)) < p).astype(np.uint8)
    masks[:, 0] = rng.integers(0, 2, n_w)            # the kernel must ignore CLS's flag
    prov = (rng.random((n_w, T)) < 0.5).astype(np.uint8)
    n_slots = n_w + 7
    slots = rng.permutation(n_slots)[:n_w].astype(np.int32)
    past = rng.integers(0, n_slots, n_w).astype(np.int32)
    fut = rng.integers(0, n_slots, n_w).astype(np.int32)
    wdesc = np.stack([slots, past, fut, np.ones(n_w, np.int32)], 1).astype(np.int32)
    cm = masks.copy()
    cm[:, 0] = 0
    cntR = cm.sum(1).astype(np.int32)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    idxC = torch.full((n_w * T,), -1, dtype=torch.int32, device=dev)
    idxR = torch.full((n_w * T,), -1, dtype=torch.int32, device=dev)
    provrow = torch.full((n_w * T,), -1, dtype=torch.int32, device=dev)
    qoff = torch.zeros(n_w + 1, dtype=torch.int32, device=dev)
    counts = torch.zeros(2, dtype=torch.int32, device=dev)
    m.stage_compact(d(wdesc), d(masks), d(prov), d(cntR), idxC, idxR, provrow, qoff, counts,
                    torch.cuda.current_stream())
    torch.cuda.synchronize()
    eC, eR, eq = oracle.compaction_indices(masks)
    MC, MR = counts.cpu().tolist()
    assert MC == len(eC) and MR == len(eR) and MC + MR == n_w * T
    # GPU rows are global slot*T + token; map back to the oracle's wave-local w*T + token
    w_of_slot = np.full(n_slots, -1, np.int64)
    w_of_slot[slots] = np.arange(n_w)
    to_local = lambda r: w_of_slot[r // T] * T + r % T
    gC = idxC[:MC].cpu().numpy().astype(np.int64)
    gR = idxR[:MR].cpu().numpy().astype(np.int64)
    assert np.array_equal(to_local(gC), eC)
    assert np.array_equal(to_local(gR), eR)
    assert np.array_equal(qoff.cpu().numpy(), eq)
    w, tok = eR // T, eR % T
    want = np.where(prov[w, tok] == 1, fut[w], past[w]).astype(np.int64) * T + tok
    assert np.array_equal(provrow[:MR].cpu().numpy().astype(np.int64), want)
    # untouched tails
    assert torch.all(idxC[MC:] == -1) and torch.all(idxR[MR:] == -1)
    m.close()


@pytest.mark.parametrize("n_w,p", [(1, 0.5), (7, 0.0), (7, 1.0), (40, 0.3), (300, 0.9)])
def test_compaction_bitexact(dev, n_w, p):
    _compaction_case(dev, synth.CONFIGS["tiny"], n_w, p, seed=n_w)


# T = 257 (L/14) and 577 (L/14@336): several 256-token chunks per frame and a ragged tail;
# n_w up to the 1,440 / 1,536-frame waves of the 7,200-frame bench (the O(n_w) offset sum)
@pytest.mark.parametrize("cfgname", ["l14", "l14_336"])
@pytest.mark.parametrize("n_w", [1, 45, 1440, 1536])
@pytest.mark.parametrize("p", [0.0, 0.3, 0.9, 1.0])
def test_compaction_bitexact_fullsize(dev, cfgname, n_w, p):
    _compaction_case(dev, synth.CONFIGS[cfgname], n_w, p, seed=1000 * n_w + int(p * 10))
