#!/usr/bin/env python
"""Reuse-rate sweep and ablation ladder (BASELINE configs[2]: CLIP ViT-L/14
224 px ReuseViT, 256-frame clip, reuse-rate sweep 0-90%).

    python tools/sweep.py [--frames 256] [--out profiles/sweep_r1.json] [--parity-frames 9]

For every motion probability p in {1, .6, .4, .3, .2, .1, .05} (SURVEY §8(d) sweep table):
frames/s of the reuse path (CUDA events, median of 3 after warm-up), reuse rates (reuse_all
and Eq. 14's reuse_nonI), executed vs dense tensor FLOPs, speedup over the same kernels run
dense (RV_DENSE) and over a torch cuBLAS + SDPA dense ViT, and parity of the first
`--parity-frames` frames (prefix-closed) against the fp64 oracle.

Ablation ladder at p = 0.4 (~61% reuse, the paper's Fig. `fig:eval-ablation` point,
P:709-713), each step adding one mechanism:
  0. dense ViT            RV_DENSE: every token recomputed, no gates (the reference speed)
  1. masked dense         RV_NO_COMPACTION: hard gating decides, every token is still computed
                          and the reused tokens' outputs are replaced by the restoration (the
                          paper's "hard gating alone")
  2. per-frame compaction each frame compacted on its own (RV_WAVE_FRAME: one wave per frame)
  3. level-batched        cross-frame compaction of a level's frames, one 20-frame refresh group
                          (+ its right-edge I frame) resident at a time (no cached memory
                          compaction: the paper's batch-size limit)
  4. all groups resident  the default: every frame of the clip in one embed (level waves span
                          all groups; P:502-522 cached memory compaction makes this fit)
Writes one JSON document to --out and prints a summary table.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="l14")
    ap.add_argument("--frames", type=int, default=256)
    ap.add_argument("--ps", default="1,0.6,0.4,0.3,0.2,0.1,0.05")
    ap.add_argument("--ablation-p", type=float, default=0.4)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--parity-frames", type=int, default=9)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "sweep_r2.json"))
    a = ap.parse_args()

    import numpy as np
    import torch

    import bench
    import oracle
    import synth
    from paper_2506_14107_b200 import ReuseViT

    cfg = synth.CONFIGS[a.config]
    n = a.frames
    W = synth.make_vit(cfg)
    G = synth.make_gates(cfg)
    m = ReuseViT(cfg, 0)
    m.load_vit(synth.pack_vit(cfg, W))
    m.load_gates(synth.pack_gates(cfg, G))
    stream = torch.cuda.current_stream()
    L, N, D = cfg.layers, cfg.N, cfg.dim

    def outs(k):   # fixed output buffers: the cached CUDA graph is replayed, not re-captured
        return (torch.empty((k, D), device="cuda"), torch.empty((k, L, N), dtype=torch.uint8, device="cuda"),
                None)
    o_n = outs(n)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts), r

    def dense_flops_frame():
        N, T, D, F, pp = cfg.N, cfg.T, cfg.dim, cfg.ffn, cfg.pp
        return 2.0 * N * pp * D + cfg.layers * T * (8.0 * D * D + 4.0 * D * F + 4.0 * T * D)

    doc = {"config": {"model": a.config, "frames": n, "T": cfg.T, "refresh": 20,
                      "generator": "SURVEY §8(d) bimodal motion, seed 2000 + frames"},
           "sweep": [], "ablation": None}
    x0, c0 = synth.make_video_torch(cfg, n, 1.0, seed=2000 + n)
    ms_dense, _ = timed(lambda: m.embed(x0, c0, dense=True, out=o_n))
    dense_fps = n / (ms_dense / 1e3)
    torch_fps = bench.torch_dense_fps(cfg, W, x0)
    doc["own_dense_fps"] = dense_fps
    doc["torch_dense_fps"] = torch_fps
    print(f"dense: own {dense_fps:.0f} fps, torch {torch_fps:.0f} fps")
    for p in [float(v) for v in a.ps.split(",")]:
        x, c = synth.make_video_torch(cfg, n, p, seed=2000 + n)
        ms, (Z, M, _, st) = timed(lambda: m.embed(x, c, out=o_n))
        ms_ser, _ = timed(lambda: m.embed(x, c, out=o_n, serial_waves=True))
        fps = n / (ms / 1e3)
        rec = {"p": p, "fps": fps, "ms": ms, "reuse_all": st["reuse_all"], "reuse_nonI": st["reuse_nonI"],
               "wave_ring": st["wave_ring"], "fps_serial_waves": n / (ms_ser / 1e3),
               "flops_exec_per_frame": st["flops_exec"] / n, "flops_dense_per_frame": dense_flops_frame(),
               "speedup_vs_own_dense": fps / dense_fps, "speedup_vs_torch_dense": fps / torch_fps}
        if a.parity_frames > 0:
            frames = list(range(a.parity_frames))
            xh, ch = x.cpu().numpy(), c.cpu().numpy()
            ref = oracle.reuse_embed(cfg, W, G, xh, ch, oracle.plan_gop(n), frames=frames)
            Zg = Z.cpu().double().numpy()[frames]
            Zr = ref["Z"][frames]
            err = np.abs(Zg - Zr).max(axis=1) / np.abs(Zr).max(axis=1)
            cos = (Zg * Zr).sum(1) / np.linalg.norm(Zg, axis=1) / np.linalg.norm(Zr, axis=1)
            Mg = M.cpu().numpy()[frames]
            band = np.abs(np.nan_to_num(ref["d"][frames], nan=1.0)) >= 1e-3
            rec["parity"] = {"frames": len(frames), "max_rel_err": float(err.max()), "min_cos": float(cos.min()),
                             "mask_agree": float((Mg == ref["M"][frames])[band].mean())}
        doc["sweep"].append(rec)
        print(f"p={p:<5} reuse_all={rec['reuse_all']:.3f} nonI={rec['reuse_nonI']:.3f} fps={fps:8.0f} "
              f"x{rec['speedup_vs_own_dense']:.2f} vs own dense  GFLOP/frame {rec['flops_exec_per_frame'] / 1e9:6.1f}"
              + f"  (serial waves {rec['fps_serial_waves']:.0f}, ring {rec['wave_ring']})"
              + (f"  err {rec['parity']['max_rel_err']:.1e} cos {rec['parity']['min_cos']:.6f}" if "parity" in rec else ""))

    # ---- ablation ladder on n_ab = 20 k + 1 frames (k refresh groups, each with its right-edge
    # I frame: step 3 then runs k equal 21-frame embeds, one cached graph)
    p = a.ablation_p
    k_groups = (n - 1) // 20 if (n - 1) % 20 == 0 else n // 20 + 1
    n_ab = 20 * k_groups + 1
    x, c = synth.make_video_torch(cfg, n_ab, p, seed=2000 + n)
    o_ab = outs(n_ab)
    ms_dense_ab, _ = timed(lambda: m.embed(x, c, dense=True, out=o_ab))
    ms_full, (_, _, _, st) = timed(lambda: m.embed(x, c, out=o_ab))
    ms_full_ser, _ = timed(lambda: m.embed(x, c, out=o_ab, serial_waves=True))
    ms_masked, _ = timed(lambda: m.embed(x, c, no_compaction=True, out=o_ab))
    ms_frame, _ = timed(lambda: m.embed(x, c, per_frame_waves=True, out=o_ab))
    xb, cb, o_g = torch.empty_like(x[:21]), torch.empty_like(c[:21]), outs(21)

    def per_group():
        for g in range(k_groups):
            xb.copy_(x[20 * g:20 * g + 21])
            cb.copy_(c[20 * g:20 * g + 21])
            m.embed(xb, cb, out=o_g)
        return None
    ms_group, _ = timed(per_group)
    halo = k_groups * 21 - n_ab
    ms_dense = ms_dense_ab
    n = n_ab
    ladder = [("dense ViT (RV_DENSE)", ms_dense), ("masked dense: hard gating, no compaction (RV_NO_COMPACTION)", ms_masked),
              ("per-frame compaction (RV_WAVE_FRAME)", ms_frame),
              ("level-batched, one refresh group resident", ms_group),
              ("all groups resident, serial level waves (RV_SERIAL_WAVES)", ms_full_ser),
              ("all groups resident, wavefront over layers (default)", ms_full)]
    doc["ablation"] = {"p": p, "frames": n_ab, "reuse_all": st["reuse_all"], "halo_frames_step3": halo,
                       "steps": [{"step": k, "name": nm, "ms": v, "fps": n / (v / 1e3), "speedup": ms_dense / v}
                                 for k, (nm, v) in enumerate(ladder)],
                       "paper": {"hard gating": 1.25, "+ sparse compaction": 1.45, "+ memory compaction": 1.62,
                                 "cite": "P:709-713, at 61% reuse, RTX 3090"}}
    print(f"ablation at p={p} (reuse_all {st['reuse_all']:.3f}):")
    for s in doc["ablation"]["steps"]:
        print(f"  {s['step']}. {s['name']:<45} {s['fps']:8.0f} fps  x{s['speedup']:.2f}")
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(doc, fh, indent=1)


if __name__ == "__main__":
    main()
