"""Toy gate-training run on the GPU (§4): GateTrainer (libreusevit
C-ABI, include/reusevit_train.h) on 1-5-9-13-11-12 frame groups of synthetic video, then
hard-gated inference (rv_embed, Eq. 4) with the trained RVG1 blob on held-out video, compared
with random reuse decisions at the same per-layer rate and with reusing everything.

    python tools/train_gates.py [--std 0.1] [--steps 300] [--r-target 0.5] [--out f.json]
Prints one JSON line (training log excerpt + evaluation)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2506_14107_b200 import ReuseViT, plan_gop  # noqa: E402
from paper_2506_14107_b200.train import GateTrainer  # noqa: E402

# the training group (P:482, 1-based 1-5-9-13-11-12) as a plan over its 6 frames, built from the
# library's own plan: display frames [0, 4, 8, 10, 11, 12] of plan_gop(13), references inside
GROUP_DISPLAY = [0, 4, 8, 10, 11, 12]


def group_plan():
    full = plan_gop(13)
    loc = {f: k for k, f in enumerate(GROUP_DISPLAY)}
    typ = np.array([full["type"][f] for f in GROUP_DISPLAY], np.int8)
    past = np.array([loc.get(int(full["past"][f]), -1) if full["past"][f] >= 0 else -1 for f in GROUP_DISPLAY],
                    np.int32)
    fut = np.array([loc.get(int(full["future"][f]), -1) if full["future"][f] >= 0 else -1 for f in GROUP_DISPLAY],
                   np.int32)
    order = np.array([loc[int(f)] for f in full["order"] if int(f) in loc], np.int32)
    return {"type": typ, "past": past, "future": fut, "order": order}


def temperature(step, steps, t0=5.0, t1=0.1):   # S:487 exponential annealing
    return t0 * (t1 / t0) ** (step / max(steps - 1, 1))


def cos_rows(A, B):
    return (A * B).sum(1) / np.linalg.norm(A, axis=1) / np.linalg.norm(B, axis=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tiny")
    ap.add_argument("--std", type=float, default=0.02, help="ViT init std (random weights)")
    ap.add_argument("--p-lo", type=float, default=0.05)
    ap.add_argument("--p-hi", type=float, default=0.4)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--pool", type=int, default=256)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--lr", type=float, default=3e-3)
    ap.add_argument("--alpha", type=float, default=2.0)
    ap.add_argument("--r-target", type=float, default=0.5)
    ap.add_argument("--eval-p", type=float, default=0.2)
    ap.add_argument("--seed", type=int, default=77)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    W = synth.make_vit(cfg, random_ln=True, std=a.std)
    G0 = synth.init_train_gates(cfg)
    plan = group_plan()
    x, c = synth.make_train_groups(cfg, a.pool, GROUP_DISPLAY, seed=a.seed, p_range=(a.p_lo, a.p_hi))
    xd, cd = torch.from_numpy(x).cuda(), torch.from_numpy(c).cuda()
    tr = GateTrainer(cfg, synth.pack_vit(cfg, W), synth.pack_gates(cfg, G0), plan, groups=a.batch, alpha=a.alpha,
                     r_target=a.r_target, lr=a.lr)
    rng = np.random.default_rng(a.seed + 1)
    log = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for s in range(a.steps):
        idx = torch.from_numpy(rng.choice(a.pool, a.batch, replace=False)).cuda()
        g = torch.from_numpy(synth.make_gumbel((a.batch, 6, cfg.layers, cfg.N, 2), seed=10_000 + s)).cuda()
        lg = tr.step(xd[idx].contiguous(), cd[idx].contiguous(), g, temperature(s, a.steps))
        if s % max(1, a.steps // 20) == 0 or s == a.steps - 1:
            log.append({"step": s, "tau": round(temperature(s, a.steps), 4), **{k: round(v, 6) for k, v in lg.items()
                                                                                  if k != "step"}})
    ev1.record()
    torch.cuda.synchronize()
    ms_step = ev0.elapsed_time(ev1) / a.steps
    blob = tr.gates()
    tr.close()
    # hard-gated inference (Eq. 4) with the trained gates on held-out video
    m = ReuseViT(cfg, 0)
    m.load_vit(synth.pack_vit(cfg, W))
    n = 41
    xv, cv = synth.make_video(cfg, n, a.eval_p, seed=909)
    xv, cv = torch.from_numpy(xv).cuda(), torch.from_numpy(cv).cuda()
    types = plan_gop(n)["type"]
    nonI = types != 0
    res = {}
    for name, gates in (("init", G0), ("trained", None)):
        m.load_gates(blob if gates is None else synth.pack_gates(cfg, gates))
        Z, M, _, st = m.embed(xv, cv)
        Zd, _, _, _ = m.embed(xv, cv, dense=True)
        torch.cuda.synchronize()
        Mh = M.cpu().numpy()
        Zn, Zdn = Z.cpu().double().numpy(), Zd.cpu().double().numpy()
        res[name] = {"reuse_nonI": float(Mh[nonI].mean()),
                     "reuse_by_layer": [round(float(v), 3) for v in Mh[nonI].mean(axis=(0, 2))],
                     "one_minus_cos": float(np.mean(1 - cos_rows(Zn, Zdn)))}
        if gates is None:
            rr = np.random.default_rng(6)
            fm = np.zeros_like(Mh)
            for l in range(cfg.layers):
                rate = Mh[nonI, l].mean()
                fm[nonI, l] = (rr.random((int(nonI.sum()), cfg.N)) < rate).astype(np.uint8)
            Zr, _, _, _ = m.embed(xv, cv, force_masks=torch.from_numpy(fm))
            fa = np.zeros_like(Mh)
            fa[nonI] = 1
            Za, _, _, _ = m.embed(xv, cv, force_masks=torch.from_numpy(fa))
            torch.cuda.synchronize()
            res["random_same_rate"] = {"one_minus_cos": float(np.mean(1 - cos_rows(Zr.cpu().double().numpy(), Zdn)))}
            res["all_reuse"] = {"one_minus_cos": float(np.mean(1 - cos_rows(Za.cpu().double().numpy(), Zdn)))}
    out = {"config": a.config, "vit_std": a.std, "p_range": [a.p_lo, a.p_hi], "steps": a.steps, "batch": a.batch,
           "pool": a.pool, "alpha": a.alpha, "r_target": a.r_target, "lr": a.lr, "ms_per_step": ms_step,
           "log": log, "eval": {"frames": n, "p": a.eval_p, **res}}
    s = json.dumps(out)
    print(s, flush=True)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(s + "\n")


if __name__ == "__main__":
    main()
