"""Time small-clip embeds (C2: B/16 x 32 frames; C3: L/14 x 256) with the fused restoration vs the
two restoration GEMMs (RV_RESTORE_GEMMS), wavefront vs serial waves.  CUDA events, median of 20.

    python tools/small_probe.py [--config b16 --frames 32 --p 0.1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="b16")
    ap.add_argument("--frames", type=int, default=32)
    ap.add_argument("--p", type=float, default=0.1)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    import torch
    import synth
    from paper_2506_14107_b200 import ReuseViT, _lib
    if os.environ.get("RV_LIB"):   # experiment build (paper_2506_14107_b200.build.build_variant)
        _lib.load_library(os.environ["RV_LIB"])
    cfg = synth.CONFIGS[a.config]
    m = ReuseViT(cfg, 0)
    m.load_vit(synth.pack_vit(cfg, synth.make_vit(cfg)))
    m.load_gates(synth.pack_gates(cfg, synth.make_gates(cfg)))
    x, c = synth.make_video(cfg, a.frames, a.p, seed=2000)
    xd, cd = torch.from_numpy(x).cuda(), torch.from_numpy(c).cuda()
    import time
    stream = torch.cuda.current_stream()
    emb = torch.empty((a.frames, cfg.dim), dtype=torch.float32, device="cuda")
    masks = torch.empty((a.frames, cfg.layers, cfg.N), dtype=torch.uint8, device="cuda")
    for kw in ({}, {"restore_gemms": True}, {}, {"restore_gemms": True}):
        # the bench loop: one profiled step, warm-up, then embed_async + wait per step, events
        # around the whole loop; host time per step alongside
        m.embed_async(xd, cd, out=(emb, masks, None), stream=stream, profile=True, **kw)
        m.wait()
        for _ in range(3):
            m.embed_async(xd, cd, out=(emb, masks, None), stream=stream, **kw)
            m.wait()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.perf_counter()
        th = 0.0
        for _ in range(a.iters):
            h0 = time.perf_counter()
            m.embed_async(xd, cd, out=(emb, masks, None), stream=stream, **kw)
            th += time.perf_counter() - h0
            m.wait()
        e1.record(stream)
        torch.cuda.synchronize()
        print(f"bench loop {kw}: {e0.elapsed_time(e1) / a.iters:.3f} ms/step (wall {(time.perf_counter() - t0) / a.iters * 1e3:.3f}, "
              f"embed_async host {th / a.iters * 1e3:.3f} ms)")
    for kw in ({}, {"restore_gemms": True}, {"serial_waves": True}, {"serial_waves": True, "restore_gemms": True}):
        outs = None
        ts = []
        for it in range(a.iters + 3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            h = m.embed_async(xd, cd, out=outs, **kw)
            e1.record()
            st = m.wait(h)
            outs = (h["emb"], h["masks"], None)
            torch.cuda.synchronize()
            if it >= 3:
                ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(f"{a.config} x{a.frames} p={a.p} {kw}: {ts[len(ts) // 2]:.3f} ms  ring={st['wave_ring']} "
              f"-> {a.frames / ts[len(ts) // 2] * 1e3:.0f} frames/s")


if __name__ == "__main__":
    main()
