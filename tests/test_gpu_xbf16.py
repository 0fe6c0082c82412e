"""RV_X_BF16 (SURVEY §8(b) "experimental bf16 residual"): the residual stream X is stored in bf16
(LN statistics, the decision, GEMM accumulators and residual adds still in fp32, one rounding
on store).  Same bar as the fp32-residual path against the fp64 oracle (BASELINE.json north
star): per-frame normwise max relative error <= 2e-2, cosine >= 0.999, masks agree
on >= 99.9% of tokens outside |d| < 1e-3; plus bitwise wavefront == serial waves and the
chain-variant contract error."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.test_gpu_parity import build, mask_agreement, metrics

pytestmark = pytest.mark.gpu

CASES = [("tiny", 41, 41, 0.2, "bimodal"), ("b16", 32, 32, 0.3, "bimodal"), ("l14", 64, 21, 0.2, "bimodal"),
         ("l14_336", 24, 9, 0.2, "bimodal"), ("b16", 16, 16, 0.0, "continuous"), ("l14", 9, 9, 0.0, "continuous")]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-n{c[1]}-{c[4]}" for c in CASES])
def test_x_bf16_parity(cuda_ok, case):
    cfgname, n, n_check, p, mode = case
    cfg = synth.CONFIGS[cfgname]
    m, W, G = build(cfg, **({"tau": 0.3} if mode == "continuous" else {}))
    x, c = synth.make_video(cfg, n, p, seed=(2500 if mode == "continuous" else 2000) + n, mode=mode)
    plan = oracle.plan_gop(n)
    xd, cd = torch.from_numpy(x).cuda(), torch.from_numpy(c).cuda()
    Z, M, S, st = m.embed(xd, cd, want_scores=True, x_bf16=True)
    Z32, M32, _, _ = m.embed(xd, cd, want_scores=True)
    torch.cuda.synchronize()
    frames = list(range(n_check))
    ref = oracle.reuse_embed(cfg, W, G, x, c, plan, frames=frames)
    err, cos = metrics(Z.cpu().numpy()[frames], ref["Z"][frames])
    err32, _ = metrics(Z32.cpu().numpy()[frames], ref["Z"][frames])
    agree, cnt = mask_agreement(M.cpu().numpy(), ref, frames)
    d_gpu = S.cpu().numpy()[frames].astype(np.float64)
    has = ~np.isnan(ref["d"][frames])
    assert np.array_equal(np.isnan(d_gpu), ~has)
    print(f"x_bf16 {cfgname} n={n} {mode}: reuse_all={st['reuse_all']:.3f} max_err={err.max():.3e} "
          f"(fp32 residual {err32.max():.3e}) min_cos={cos.min():.6f} mask_agree={agree:.5f} ({cnt} tokens)")
    assert err.max() <= 2e-2 and cos.min() >= 0.999 and agree >= 0.999


@pytest.mark.parametrize("cfgname,n,p", [("b16", 32, 0.3), ("l14", 64, 0.2)])
def test_x_bf16_wavefront_equals_serial(cuda_ok, cfgname, n, p):
    cfg = synth.CONFIGS[cfgname]
    m, W, G = build(cfg)
    x, c = synth.make_video(cfg, n, p, seed=3100 + n)
    xd, cd = torch.from_numpy(x).cuda(), torch.from_numpy(c).cuda()
    Z0, M0, _, st0 = m.embed(xd, cd, serial_waves=True, x_bf16=True)
    Z1, M1, _, st1 = m.embed(xd, cd, x_bf16=True)
    Z2, M2, _, _ = m.embed(xd, cd, x_bf16=True, graph=False)
    torch.cuda.synchronize()
    assert st0["wave_ring"] == 0 and st1["wave_ring"] >= 3
    assert torch.equal(Z0, Z1) and torch.equal(M0, M1) and torch.equal(Z0, Z2) and torch.equal(M0, M2)


def test_x_bf16_rejected_with_chain(cuda_ok):
    from paper_2506_14107_b200._lib import ReuseViTError
    cfg = synth.CONFIGS["tiny"]
    m, W, G = build(cfg)
    x, c = synth.make_video(cfg, 8, 0.3, seed=2000)
    with pytest.raises(ReuseViTError, match="ECONTRACT"):
        m.embed(torch.from_numpy(x).cuda(), torch.from_numpy(c).cuda(), chain=True, x_bf16=True)
