"""Microbenchmark of the tcgen05 GEMM on the shapes of the L/14 hot path (one level wave of
M compacted rows): QKV (N 3D, K D, bf16 out), FC1 (N 4D, K D, QuickGELU, bf16 out), FC2
(N D, K 4D, fp32 out), W_o (N D, K D, fp32 out), against torch.matmul (cuBLAS) on the same
operands.  Run twice with RV_GEMM_PAIR=0 / 1 to compare single-CTA and CTA-pair tiles.

    python tools/gemm_bench.py [--M 80000] [--iters 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=80000)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only", default=None, help="comma-separated subset of qkv,fc1,fc2,wo")
    a = ap.parse_args()
    import torch
    import synth
    from paper_2506_14107_b200 import ReuseViT
    cfg = synth.CONFIGS["l14"]
    m = ReuseViT(cfg, 0)
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(1)
    D = cfg.dim
    shapes = [("qkv", 3 * D, D, 0, True), ("fc1", 4 * D, D, 1, True), ("fc2", D, 4 * D, 0, False),
              ("wo", D, D, 0, False)]
    pair = os.environ.get("RV_GEMM_PAIR", "1")
    for name, N, K, act, obf in shapes:
        if a.only and name not in a.only.split(","):
            continue
        A = torch.randn(a.M, K, device=dev, generator=g).to(torch.bfloat16)
        B = (0.05 * torch.randn(N, K, device=dev, generator=g)).to(torch.bfloat16)
        bias = torch.randn(N, device=dev, generator=g)
        out = torch.empty((a.M, N), dtype=torch.bfloat16 if obf else torch.float32, device=dev)

        def ours():
            m.stage_gemm(A, B, bias=bias, act=act, out=out, out_bf16=obf)

        def cublas():
            return torch.matmul(A, B.t())

        res = {}
        for tag, fn in (("ours", ours), ("cublas", cublas)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.iters):
                fn()
            e1.record()
            torch.cuda.synchronize()
            res[tag] = e0.elapsed_time(e1) / a.iters
        ours()
        ref = (A[:4096].float() @ B.float().t()) + bias
        if act == 1:
            ref = ref * torch.sigmoid(1.702 * ref)
        err = ((out[:4096].float() - ref).abs().max() / ref.abs().max()).item()
        tail = ((out[-1000:].float() - ((A[-1000:].float() @ B.float().t()) + bias if act == 0 else out[-1000:].float())).abs().max()).item()
        fl = 2.0 * a.M * N * K
        print(f"pair={pair} {name:4s} M={a.M} N={N} K={K}: ours {res['ours'] * 1e3:8.1f} us "
              f"{fl / res['ours'] / 1e9:7.0f} TF/s | cuBLAS {res['cublas'] * 1e3:8.1f} us "
              f"{fl / res['cublas'] / 1e9:7.0f} TF/s | rel err {err:.1e} tail {tail:.1e}", flush=True)


if __name__ == "__main__":
    main()
