"""Bitwise check of the fused restoration against the two GEMMs (RV_RESTORE_GEMMS) on an L/14
clip, for an experiment build (RV_LIB=...): python tools/restore_check.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import synth
    from paper_2506_14107_b200 import ReuseViT, _lib
    if os.environ.get("RV_LIB"):
        _lib.load_library(os.environ["RV_LIB"])
    for name, n, p, kw in (("l14", 64, 0.2, {}), ("l14", 64, 0.2, {"serial_waves": True}), ("b16", 32, 0.3, {}),
                           ("l14", 41, 0.1, {"x_bf16": True})):
        cfg = synth.CONFIGS[name]
        m = ReuseViT(cfg, 0)
        m.load_vit(synth.pack_vit(cfg, synth.make_vit(cfg, random_ln=True)))
        m.load_gates(synth.pack_gates(cfg, synth.make_gates(cfg, restore_bias=True)))
        x, c = synth.make_video(cfg, n, p, seed=4100 + n)
        xd, cd = torch.from_numpy(x).cuda(), torch.from_numpy(c).cuda()
        Z0, M0, _, _ = m.embed(xd, cd, restore_gemms=True, **kw)
        Z1, M1, _, st = m.embed(xd, cd, **kw)
        torch.cuda.synchronize()
        ok = torch.equal(Z0, Z1) and torch.equal(M0, M1)
        print(f"{name} n={n} {kw}: reuse {st['reuse_all']:.3f} bitwise {'OK' if ok else 'MISMATCH'} "
              f"max|dZ| {(Z0 - Z1).abs().max().item():.3e}")
        m.close()


if __name__ == "__main__":
    main()
