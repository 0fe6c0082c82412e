"""Fused restoration kernel (k_restore.cu: Eq. 8-10 over the compacted reused rows, hr kept on
chip) against the two-GEMM restoration (RV_RESTORE_GEMMS: R1 over every wave row with hr through
HBM, then R2).  Same K order and epilogue arithmetic, so every embedding, mask and decision
logit is bitwise equal, in the serial and the wavefront schedule and with the bf16 residual
stream; end-to-end parity of the fused path against the oracle is test_gpu_parity.py."""
import pytest
import torch

import synth
from tests.test_gpu_parity import build

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfgname,n,p,kw", [("b16", 32, 0.3, {}), ("l14", 64, 0.2, {}), ("l14", 64, 0.2, {"serial_waves": True}),
                                            ("l14_336", 24, 0.2, {}), ("l14", 41, 0.1, {"x_bf16": True}),
                                            ("b16", 21, 0.5, {"no_compaction": True}), ("l14", 41, 0.2, {"chain": True})])
def test_fused_restore_equals_gemms(cuda_ok, cfgname, n, p, kw):
    cfg = synth.CONFIGS[cfgname]
    m, W, G = build(cfg)
    x, c = synth.make_video(cfg, n, p, seed=4100 + n)
    xd, cd = torch.from_numpy(x).cuda(), torch.from_numpy(c).cuda()
    Z0, M0, S0, st0 = m.embed(xd, cd, want_scores=True, restore_gemms=True, **kw)
    Z1, M1, S1, st1 = m.embed(xd, cd, want_scores=True, **kw)
    torch.cuda.synchronize()
    assert st1["reuse_all"] > 0.3
    assert torch.equal(M0, M1)
    assert torch.equal(torch.nan_to_num(S0, nan=-7.0), torch.nan_to_num(S1, nan=-7.0))
    assert torch.equal(Z0, Z1), (Z0 - Z1).abs().max().item()
