"""Microbenchmark of the restoration output GEMM (R2, Eq. 9-10) in isolation: M reused rows,
N = D, K = Hr = 128, provider rows gathered from / merged rows scattered into an X_l-sized fp32
buffer (random disjoint row sets, as in a level-3 wave of the 7,200-frame L/14 bench).

    python tools/r2_bench.py [--M 63000] [--rows 1850000] [--iters 20]
Prints us per launch and the achieved HBM rate on the algorithmic bytes (M x (4 D in + 4 D out
+ 2 Hr)).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=63000)
    ap.add_argument("--rows", type=int, default=1850000)
    ap.add_argument("--D", type=int, default=1024)
    ap.add_argument("--K", type=int, default=128, help="128: restoration R2; 1024: W_o; 4096: FC2")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--sorted", action="store_true", help="row maps sorted (frame-ordered, as compaction emits)")
    a = ap.parse_args()
    import torch
    import synth
    from paper_2506_14107_b200 import ReuseViT
    cfg = synth.CONFIGS["l14"]
    m = ReuseViT(cfg, 0)
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(1)
    hr = torch.randn(a.M, a.K, device=dev, generator=g).to(torch.bfloat16)
    W = (0.05 * torch.randn(a.D, a.K, device=dev, generator=g)).to(torch.bfloat16)
    b = torch.randn(a.D, device=dev, generator=g)
    X = torch.randn(a.rows, a.D, device=dev, generator=g)
    perm = torch.randperm(a.rows, device=dev, generator=g)
    rr, orr = perm[:a.M].to(torch.int32), perm[a.M:2 * a.M].to(torch.int32)
    if a.sorted:
        rr, orr = rr.sort().values, orr.sort().values
    for _ in range(3):
        m.stage_gemm_rows(hr, W, X, bias=b, resid=X, resid_rows=rr, out_rows=orr)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        m.stage_gemm_rows(hr, W, X, bias=b, resid=X, resid_rows=rr, out_rows=orr)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    byt = a.M * (8.0 * a.D + 2.0 * a.K)
    print(f"row-mapped GEMM M={a.M} N={a.D} K={a.K} {'sorted' if a.sorted else 'random'} rows: {ms * 1e3:.1f} us, "
          f"{byt / ms / 1e6:.0f} GB/s algorithmic, {2.0 * a.M * a.D * a.K / ms / 1e9:.0f} TFLOP/s")


if __name__ == "__main__":
    main()
