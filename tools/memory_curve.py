"""Cached memory compaction, measured (§5.2; Fig. `fig:tmp-memory-profile`
P:683-700 analogue): for videos of n frames (ViT-L/14, p = 0.2), the
device bytes the library allocates for one embed with the layer-wise cache (X ping-pong + one
K/V layer, the default) and with RV_KEEP_ALL_CACHE (every layer's X and K/V), plus the embed
time and the device memory in use (cudaMemGetInfo) after each.  Keep-all stops fitting in the
B200's HBM long before the 7,200-frame workload; the layer-wise cache holds it with room to
spare.  Prints one JSON line.

    python tools/memory_curve.py [--frames 64,256,1024,2048,3072,4096,7200] [--out f.json]"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2506_14107_b200 import ReuseViT  # noqa: E402
from paper_2506_14107_b200._lib import ReuseViTError  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="l14")
    ap.add_argument("--frames", default="64,256,1024,2048,3072,4096,7200")
    ap.add_argument("--p", type=float, default=0.2)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    W, G = synth.make_vit(cfg), synth.make_gates(cfg)
    rows = []
    total = torch.cuda.mem_get_info()[1]
    for n in [int(v) for v in a.frames.split(",")]:
        x, c = synth.make_video_torch(cfg, n, a.p, seed=2000, device="cuda")
        for mode in ("layerwise", "keep_all"):
            m = ReuseViT(cfg, 0)
            m.load_vit(synth.pack_vit(cfg, W))
            m.load_gates(synth.pack_gates(cfg, G))
            rec = {"frames": n, "mode": mode}
            try:
                m.embed(x, c, keep_all_cache=(mode == "keep_all"), want_masks=False)   # allocate + capture
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                _, _, _, st = m.embed(x, c, keep_all_cache=(mode == "keep_all"), want_masks=False)
                e1.record()
                torch.cuda.synchronize()
                free, _ = torch.cuda.mem_get_info()
                rec.update({"ok": True, "cache_bytes": st["peak_cache_bytes"], "device_bytes": st["device_bytes"],
                            "cache_bytes_per_frame": st["peak_cache_bytes"] / n, "ms": e0.elapsed_time(e1),
                            "frames_per_s": n / (e0.elapsed_time(e1) / 1e3), "gpu_mem_in_use": total - free,
                            "reuse_all": st["reuse_all"]})
            except ReuseViTError as ex:
                rec.update({"ok": False, "error": str(ex)[:160]})
            rows.append(rec)
            print(json.dumps(rec), file=sys.stderr, flush=True)
            m.close()
            del m
            torch.cuda.empty_cache()
        del x, c
        torch.cuda.empty_cache()
    out = {"config": a.config, "p": a.p, "hbm_bytes": total, "rows": rows}
    s = json.dumps(out)
    print(s)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(s + "\n")


if __name__ == "__main__":
    main()
