"""One (or a few) ReuseViT embeds for ncu: inputs are generated on the host (numpy) and copied
with a single H2D, so the only kernels in the process are libreusevit's.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file L.csv \
        python tools/prof_run.py --frames 1440
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="l14")
    ap.add_argument("--frames", type=int, default=1440)
    ap.add_argument("--p", type=float, default=0.2)
    ap.add_argument("--iters", type=int, default=1)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--counts-out", default=None, help="write the per-wave M_C / M_R counts (JSON)")
    a = ap.parse_args()
    import torch
    import synth
    from paper_2506_14107_b200 import ReuseViT
    cfg = synth.CONFIGS[a.config]
    x, c = synth.make_video(cfg, a.frames, a.p, seed=2000)
    m = ReuseViT(cfg, 0)
    m.load_vit(synth.pack_vit(cfg, synth.make_vit(cfg)))
    m.load_gates(synth.pack_gates(cfg, synth.make_gates(cfg)))
    xd, cd = torch.from_numpy(x).cuda(), torch.from_numpy(c).cuda()
    for _ in range(a.iters):
        Z, M, _, st = m.embed(xd, cd, graph=not a.no_graph)
    torch.cuda.synchronize()
    print({k: st[k] for k in ("reuse_all", "ms_compute", "n_launches")})
    if a.counts_out:
        import json
        wc = m.wave_counts()
        with open(a.counts_out, "w") as fh:
            json.dump({"frames": wc["frames"].tolist(), "M_C": wc["M_C"].tolist(), "M_R": wc["M_R"].tolist(),
                       "config": a.config, "n": a.frames, "p": a.p, "T": cfg.T, "D": cfg.dim, "F": cfg.ffn,
                       "Hr": cfg.hidden_r}, fh)


if __name__ == "__main__":
    main()
