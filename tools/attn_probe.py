"""Time the two attention kernels on one synthetic L/14 wave (stage API, no graph).

    python tools/attn_probe.py [--frames 288] [--nq 57] [--iters 20]
Every frame of the wave has `nq` compact queries (frame 0 of every 20 has all T, like the
I frames); K/V rows are the frame's own (kvsrc = identity).  Prints ms per launch.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=288)
    ap.add_argument("--nq", type=int, default=57)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only", default="both", choices=["both", "tc", "sync", "tcg", "all"])
    ap.add_argument("--config", default="l14")
    a = ap.parse_args()
    import numpy as np
    import torch
    import synth
    from paper_2506_14107_b200 import ReuseViT, _lib
    if os.environ.get("RV_LIB"):   # experiment build (paper_2506_14107_b200.build.build_variant)
        _lib.load_library(os.environ["RV_LIB"])
    cfg = synth.CONFIGS[a.config]
    T, D, H = cfg.T, cfg.dim, cfg.heads
    m = ReuseViT(cfg, 0)
    m.load_vit(synth.pack_vit(cfg, synth.make_vit(cfg)))
    n_w = a.frames
    nq = np.array([T if w % 20 == 0 else a.nq for w in range(n_w)])
    qoff = np.concatenate([[0], np.cumsum(nq)]).astype(np.int32)
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(int(qoff[-1]), D, device="cuda", generator=g).to(torch.bfloat16)
    KV = torch.randn(n_w * T, 2 * D, device="cuda", generator=g).to(torch.bfloat16)
    wdesc = torch.zeros(n_w, 4, dtype=torch.int32, device="cuda")
    wdesc[:, 0] = torch.arange(n_w, dtype=torch.int32)
    qo = torch.from_numpy(qoff).cuda()
    out = torch.zeros_like(q)
    pcls = torch.zeros(n_w, H, cfg.N, device="cuda")
    st = torch.cuda.current_stream()
    flops = 4.0 * float(qoff[-1]) * T * D
    modes = {"both": [0, 1], "tc": [1], "sync": [0], "tcg": [2], "all": [0, 1, 2]}[a.only]
    for use_tc in modes:
        for _ in range(3):
            m.stage_attention(wdesc, qo, q, KV, out, pcls, st, use_tc=use_tc)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            m.stage_attention(wdesc, qo, q, KV, out, pcls, st, use_tc=use_tc)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        print(f"{['mma.sync', 'tcgen05', 'tcgen05-general'][use_tc]}: {ms * 1e3:.1f} us/launch, {flops / ms / 1e9:.1f} TFLOP/s, "
              f"K/V {n_w * T * 2 * D * 2 / ms / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
