"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Training-time ReuseViT (§4): the soft-gated forward
pass (Eq. 11-12), the loss (Eq. 13-15) over grouped frames (the 1-5-9-13-11-12
pattern) and its gradient with respect to the decision and restoration layers only (the ViT
stays frozen).  Plain PyTorch fp64 on the CPU, frame-sequential in computation order
like oracle/reusevit_ref.py; the gradient is torch autograd (a library primitive) over that
plain forward, pinned in tests/test_train_pins.py by central finite differences.

Readings ("Gate training"):
* T1  Eq. 11 with two logits, reuse = d_i and recompute = 0: M_soft,i is the reuse
      probability of a 2-class Gumbel-Softmax, softmax([(d_i + g_i1), g_i0] / tau)[0].  The
      Gumbel draws g are INPUTS (random numbers the method draws are passed in).
* T2  Eq. 12's blend applies to every quantity the hard gate selects between under reading
      D1: the layer output (M_soft * restored + (1 - M_soft) * recomputed) and the key /
      value the token contributes to attention (M_soft * provider's + (1 - M_soft) * own).
      With M_soft in {0, 1} the soft forward is the hard forward of reusevit_ref exactly.
      Every token's recompute branch (LN1 -> QKV -> attention over all keys -> W_o -> FFN)
      and, for patches of non-I frames, its restoration branch are both evaluated.
* T3  The decision features (s_i, provider, t_i, r, c_i; Eq. 1-2) are inputs of the
      decision layer and carry no gradient (stop-gradient); the provider is Eq. 1's argmax.
* T4  L_sim averages 1 - cos(Z, Z_hat) over the group's frames (I included: 0 for it when
      the I-frame is exact); L_reuse averages M_soft over the non-I frames' patch tokens and
      all layers; the hinge of Eq. 15 per group; a batch averages group losses.
"""
from __future__ import annotations

import math
from typing import Dict, Optional

import numpy as np
import torch

from .reusevit_ref import FTYPES, plan_gop

_T64 = torch.float64

# P:482 "grouping six frames in the pattern 1-5-9-13-11-12" (1-based display indices)
GROUP_PATTERN = (1, 5, 9, 13, 11, 12)


def group_plan(pattern=GROUP_PATTERN, refresh: int = 20) -> Dict[str, np.ndarray]:
    """The training group as a plan over local frames 0..G-1: the display
    frames of ``pattern`` (1-based) keep their types and references from the inference plan
    (plan_gop), restricted to the group; local index = position in ascending
    display order.  For 1-5-9-13-11-12 this is I, P(I), P, P, B2(9, 13), B1(11, 13) with
    computation order 1, 5, 9, 13, 11, 12 — every reference inside the group (the pattern
    is prefix-closed in plan_gop's DAG).  Returns dict(type, past, future, order, display)."""
    disp = sorted(p - 1 for p in pattern)
    full = plan_gop(max(disp) + 1, refresh)
    loc = {f: k for k, f in enumerate(disp)}
    G = len(disp)
    typ = np.zeros(G, np.int8)
    past = np.full(G, -1, np.int32)
    fut = np.full(G, -1, np.int32)
    for f in disp:
        k = loc[f]
        typ[k] = full["type"][f]
        for key, arr in (("past", past), ("future", fut)):
            r = int(full[key][f])
            if r >= 0:
                if r not in loc:
                    raise ValueError(f"pattern is not closed: frame {f + 1} needs {r + 1}")
                arr[k] = loc[r]
    order = np.array([loc[f] for f in full["order"] if f in loc], np.int32)
    return {"type": typ, "past": past, "future": fut, "order": order, "display": np.array(disp, np.int32)}


def _t(a):
    return a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a), dtype=_T64)


def _ln(x, g, b, eps=1e-5):
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    return (x - mu) / torch.sqrt(var + eps) * g + b


def _qg(x):
    return x * torch.sigmoid(1.702 * x)


def gumbel_soft_mask(d, g_reuse, g_recompute, tau: float):
    """Eq. 11: M_soft = GumbelSoftmax(MLP_decision(v)) with the two logits (reuse d,
    recompute 0) of reading T1: softmax over [(d + g_reuse) / tau, g_recompute / tau], the
    reuse class's probability."""
    if tau <= 0:
        raise ValueError("temperature must be > 0 (S:203)")
    logits = torch.stack([(d + g_reuse) / tau, (torch.zeros_like(d) + g_recompute) / tau], dim=-1)
    return torch.softmax(logits, dim=-1)[..., 0]


def soft_forward(cfg, W, G, patches, codec, plan, gumbel, tau: float, *, dense: bool = False,
                 force_masks=None, features=None) -> Dict[str, torch.Tensor]:
    """Soft-gated ReuseViT forward of one frame group (Eq. 1-12 under readings D1, T1-T3).

    ``G`` maps RVG1 names (synth.gate_array_order) to fp64 tensors (they may require grad);
    ``W`` the frozen ViT (numpy or tensors); ``patches`` [n, N, pp]; ``codec`` [n, N];
    ``plan`` over the n frames; ``gumbel`` [n, L, N, 2] Gumbel(0, 1) draws (index 0 for the
    reuse logit, 1 for the recompute logit); ``dense``: M = 0 everywhere (the frozen ViT's
    own embedding Z of Eq. 13); ``force_masks`` [n, L, N]: constant M (soft-to-hard limit);
    ``features``: the decision features {(f, l): (v, provider frames)} of an earlier pass to
    use instead of recomputing them (T3 makes them constants: a finite-difference check of
    the gradient must hold them fixed).  Returns Z [n, D], M [n, L, N] (0 for I-frames),
    d [n, L, N] (NaN without decision) and the features used."""
    L, D, H, N, T = cfg.layers, cfg.dim, cfg.heads, cfg.N, cfg.T
    dh = D // H
    Wt = {k: _t(v) for k, v in W.items()}
    n = patches.shape[0]
    pt, ct, gt = _t(patches), _t(codec), _t(gumbel)
    onehot = torch.eye(4, dtype=_T64)
    Xc: Dict[int, list] = {}      # frame -> [X_0 .. X_L]
    KVc: Dict[int, list] = {}     # frame -> [(K_l, V_l)] of the soft-blended keys / values
    Z = [None] * n
    Mrows = [[torch.zeros(N, dtype=_T64) for _ in range(L)] for _ in range(n)]
    d_all = torch.full((n, L, N), float("nan"), dtype=_T64)
    feats = {}
    for f in [int(v) for v in plan["order"]]:
        ftype = int(plan["type"][f])
        refs = {0: int(plan["past"][f]), 1: int(plan["future"][f])}
        E = pt[f] @ Wt["W_pe"]
        X = [_ln(torch.cat([Wt["cls"][None, :], E], 0) + Wt["pos"], Wt["lnpre_g"], Wt["lnpre_b"])]
        KV = []
        t = torch.full((N,), 1.0 / N, dtype=_T64)
        for l in range(L):
            Xp = X[l]
            pre = f"L{l}."
            decide = not dense and ftype != FTYPES["I"] and (refs[0] >= 0 or refs[1] >= 0)
            if decide:
                # Eq. 1 (T3: features carry no gradient): s_i, provider = argmax, ties -> past
                with torch.no_grad():
                    cur = Xp[1:].detach()
                    best, prov = None, None
                    for k in (0, 1):
                        if refs[k] < 0:
                            continue
                        R = Xc[refs[k]][l][1:].detach()
                        den = torch.sqrt((cur * cur).sum(1) * (R * R).sum(1))
                        c = torch.where(den > 0, (cur * R).sum(1) / torch.where(den > 0, den, torch.ones_like(den)),
                                        torch.zeros_like(den))
                        if best is None:
                            best, prov = c, torch.full((N,), k, dtype=torch.long)
                        else:
                            take = c > best
                            best = torch.where(take, c, best)
                            prov = torch.where(take, torch.full_like(prov, k), prov)
                    v = torch.cat([best[:, None], t.detach()[:, None], onehot[ftype][None, :].expand(N, 4),
                                   ct[f][:, None]], 1)
                prov_f = [refs[int(k)] for k in prov]
                if features is not None:
                    v, prov_f = features[(f, l)]
                feats[(f, l)] = (v, prov_f)
                # Eq. 3 decision MLP, Eq. 11 soft mask
                hd = _qg(v @ G[pre + "Wd1"] + G[pre + "bd1"])
                d = hd @ G[pre + "Wd2"] + G[pre + "bd2"][0]
                d_all[f, l] = d.detach()
                M = gumbel_soft_mask(d, gt[f, l, :, 0], gt[f, l, :, 1], tau)
                if force_masks is not None:
                    M = _t(force_masks[f, l]).to(_T64)
            else:
                M = torch.zeros(N, dtype=_T64)
            Mrows[f][l] = M
            # recompute branch for every token (Eq. 7), keys / values blended (T2)
            h1 = _ln(Xp, Wt[pre + "ln1_g"], Wt[pre + "ln1_b"])
            qkv = h1 @ Wt[pre + "Wqkv"] + Wt[pre + "bqkv"]
            q, kc, vc = qkv[:, :D], qkv[:, D:2 * D], qkv[:, 2 * D:]
            if decide:
                Kp = torch.stack([KVc[prov_f[i]][l][0][1 + i] for i in range(N)])
                Vp = torch.stack([KVc[prov_f[i]][l][1][1 + i] for i in range(N)])
                K = torch.cat([kc[:1], M[:, None] * Kp + (1 - M[:, None]) * kc[1:]], 0)
                V = torch.cat([vc[:1], M[:, None] * Vp + (1 - M[:, None]) * vc[1:]], 0)
            else:
                K, V = kc, vc
            KV.append((K, V))
            pcls = []
            heads = []
            for h in range(H):
                sl = slice(h * dh, (h + 1) * dh)
                P = torch.softmax(q[:, sl] @ K[:, sl].T / math.sqrt(dh), dim=-1)
                heads.append(P @ V[:, sl])
                pcls.append(P[0, 1:])
            o = torch.cat(heads, 1)
            t = torch.stack(pcls).mean(0).detach()          # D5, no gradient (T3)
            x1 = Xp + o @ Wt[pre + "Wo"] + Wt[pre + "bo"]
            h2 = _ln(x1, Wt[pre + "ln2_g"], Wt[pre + "ln2_b"])
            Ct = x1 + _qg(h2 @ Wt[pre + "W1"] + Wt[pre + "b1"]) @ Wt[pre + "W2"] + Wt[pre + "b2"]
            if decide:
                # Eq. 8-9 restoration branch for every patch token, Eq. 12 blend
                Rin = torch.stack([Xc[prov_f[i]][l][1 + i] for i in range(N)])
                Rout = torch.stack([Xc[prov_f[i]][l + 1][1 + i] for i in range(N)])
                hr = _qg((Xp[1:] - Rin) @ G[pre + "Wr1"] + G[pre + "br1"])
                Rhat = Rout + hr @ G[pre + "Wr2"] + G[pre + "br2"]
                Xn = torch.cat([Ct[:1], M[:, None] * Rhat + (1 - M[:, None]) * Ct[1:]], 0)
            else:
                Xn = Ct
            X.append(Xn)
        Z[f] = _ln(X[L][0], Wt["lnpost_g"], Wt["lnpost_b"])
        Xc[f] = X
        KVc[f] = KV
    Mt = torch.stack([torch.stack(r) for r in Mrows])
    return {"Z": torch.stack(Z), "M": Mt, "d": d_all, "features": feats}


def group_losses(Z_ref, Z_hat, M, types, alpha: float, R_target: float) -> Dict[str, torch.Tensor]:
    """Eq. 13-15 over one frame group (grouped averaging P:466-468, reading T4):
    L_sim = mean_f (1 - cos(Z_f, Z_hat_f)); L_reuse = mean of M over non-I frames, layers and
    patch tokens (Eq. 14); L = L_sim + alpha * max(0, R_target - L_reuse) (Eq. 15)."""
    Z_ref, Z_hat = _t(Z_ref), _t(Z_hat)
    num = (Z_ref * Z_hat).sum(1)
    den = torch.sqrt((Z_ref * Z_ref).sum(1) * (Z_hat * Z_hat).sum(1))
    cos = torch.where(den > 0, num / torch.where(den > 0, den, torch.ones_like(den)), torch.zeros_like(den))
    l_sim = (1 - cos).mean()
    nonI = torch.as_tensor(np.asarray(types) != FTYPES["I"])
    if not bool(nonI.any()):
        raise ValueError("reuse loss needs a non-I frame (S:456 empty mask set)")
    l_reuse = M[nonI].mean()
    total = l_sim + alpha * torch.clamp(R_target - l_reuse, min=0.0)
    return {"l_sim": l_sim, "l_reuse": l_reuse, "l_total": total, "cos": cos}


def gates_to_torch(G: Dict[str, np.ndarray], requires_grad: bool = True) -> Dict[str, torch.Tensor]:
    return {k: torch.tensor(np.asarray(v, np.float64), dtype=_T64, requires_grad=requires_grad) for k, v in G.items()}


def batch_loss(cfg, W, Gt, patches, codec, plan, gumbel, tau, alpha, R_target, Z_ref=None, features=None):
    """Mean over a batch of groups (reading T4) of Eq. 15.  ``patches`` [B, n, N, pp],
    ``codec`` [B, n, N], ``gumbel`` [B, n, L, N, 2]; ``Z_ref`` [B, n, D] (default: the frozen
    ViT's embeddings, soft_forward(dense=True)).  Returns (mean total, per-group dicts)."""
    B = patches.shape[0]
    outs, tot = [], 0.0
    for b in range(B):
        if Z_ref is None:
            with torch.no_grad():
                zr = soft_forward(cfg, W, Gt, patches[b], codec[b], plan, gumbel[b], 1.0, dense=True)["Z"]
        else:
            zr = _t(Z_ref[b])
        fw = soft_forward(cfg, W, Gt, patches[b], codec[b], plan, gumbel[b], tau,
                          features=None if features is None else features[b])
        lo = group_losses(zr, fw["Z"], fw["M"], plan["type"], alpha, R_target)
        lo.update(fw)
        lo["Z_ref"] = zr
        outs.append(lo)
        tot = tot + lo["l_total"]
    return tot / B, outs


def loss_and_grads(cfg, W, G, patches, codec, plan, gumbel, tau, alpha, R_target):
    """Eq. 15 batch loss and its gradient w.r.t. every gate array (RVG1 names), by autograd
    over soft_forward.  Returns (loss float, {name: grad ndarray}, per-group outputs)."""
    Gt = gates_to_torch(G)
    loss, outs = batch_loss(cfg, W, Gt, patches, codec, plan, gumbel, tau, alpha, R_target)
    grads = torch.autograd.grad(loss, list(Gt.values()), allow_unused=True)
    gd = {k: (g.detach().numpy() if g is not None else np.zeros_like(np.asarray(G[k], np.float64)))
          for k, g in zip(Gt.keys(), grads)}
    return float(loss.detach()), gd, outs


def adam_step(p, g, m, v, t: int, lr: float, b1: float = 0.9, b2: float = 0.999, eps: float = 1e-8):
    """One Adam update ("plain Adam-style adaptive step (beta = 0.9/0.999)"), bias
    corrected, written out: m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
    p -= lr * (m / (1-b1^t)) / (sqrt(v / (1-b2^t)) + eps).  Returns (p, m, v) as new arrays."""
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    mh = m / (1 - b1 ** t)
    vh = v / (1 - b2 ** t)
    return p - lr * mh / (np.sqrt(vh) + eps), m, v


def temperature(step: int, steps: int, t0: float = 5.0, t1: float = 0.1) -> float:
    """Exponential annealing t0 -> t1 over the step budget ("gradually
    lowering the Gumbel-Softmax temperature")."""
    if steps <= 1:
        return t1
    return t0 * (t1 / t0) ** (step / (steps - 1))
