"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SPEC chain variant of ReuseViT: the paper-literal reading of Eq. 7
"QKV(FFN(C))" and of §3.2 / §8 "only FFN and QKV", fixed by SPEC's
reuse_forward design.  Readings ("chain variant"):
  * one decision per token and layer l = 1..L gates the token-independent chain
    FFN_l -> QKV_{l+1} (FFN_L alone for l = L); QKV_1 is computed for every token
    (the layer-0 chain is not gated: "decision layers count L");
  * attention and the output projection W_o run densely over all T tokens in every layer
    ("attention itself is always computed densely with all tokens"); a reused
    token's q, k, v of layer l+1 are its provider's (the chain output reused raw);
  * the decision and the restoration see the chain's input x'_l = X_{l-1} + Attn.Wo + bo
    ("Delta R_i = R_cur_i - R_ref_i (block inputs)"): s_i = max cos(x'^f_i, x'^ref_i)
    (Eq. 1), X_l^f[i] = X_l^prov[i] + MLP_rest(x'^f_i - x'^prov_i) (Eq. 8-9, "cached block
    output + MLP_restoration");
  * t for decision l = head-mean CLS attention row of layer l-1, uniform for l = 1;
  * CLS never reused; ties to the past reference; d = 0 -> recompute (as the D1 oracle).
Pins (tests/test_oracle_pins.py): M = 0 -> the torch fp64 library ViT; duplicate frame ->
Z_f = Z_ref; forced masks -> pure-Python brute force (tests/bruteforce_chain.py).
Correspondence to the authors' trained model: parity unpinned (no code or weights exist).
"""
from __future__ import annotations

from typing import Dict, List, Optional

import numpy as np

from .reusevit_ref import (FTYPES, _attention_rows, decision_mlp, layer_norm, patch_embed, quick_gelu,
                           restoration_mlp, similarity)

_F64 = np.float64


def _qkv(W, l: int, X: np.ndarray) -> np.ndarray:
    """LN1_l then the QKV projection of layer l (0-based l), rows of X."""
    pre = f"L{l}."
    h = layer_norm(X, W[pre + "ln1_g"], W[pre + "ln1_b"])
    return h @ np.asarray(W[pre + "Wqkv"], _F64) + np.asarray(W[pre + "bqkv"], _F64)


def reuse_embed_chain(cfg, W: Dict[str, np.ndarray], G: Optional[Dict[str, np.ndarray]],
                      patches: np.ndarray, codec: np.ndarray, plan: Dict[str, np.ndarray],
                      dense: bool = False, force_masks: Optional[np.ndarray] = None,
                      frames: Optional[List[int]] = None) -> Dict[str, np.ndarray]:
    """Chain-variant forward, frame-sequentially in plan['order'].  Same outputs
    as oracle.reuse_embed: Z [n, D], M [n, L, N] uint8, d [n, L, N] (NaN where no decision)."""
    L, D, H, N, T = cfg.layers, cfg.dim, cfg.heads, cfg.N, cfg.T
    n = patches.shape[0]
    order = [int(f) for f in plan["order"]]
    if frames is not None:
        want = set(int(f) for f in frames)
        for f in want:
            for r in (plan["past"][f], plan["future"][f]):
                if r >= 0 and r not in want:
                    raise ValueError(f"frame {f} needs reference {r} outside the subset")
        order = [f for f in order if f in want]
    Z = np.full((n, D), np.nan)
    M_all = np.zeros((n, L, N), np.uint8)
    d_all = np.full((n, L, N), np.nan)
    Xc: Dict[int, List[np.ndarray]] = {}     # frame -> [X_0 .. X_L]
    XPc: Dict[int, List[np.ndarray]] = {}    # frame -> [x'_1 .. x'_L]  (chain inputs)
    QKVc: Dict[int, List[np.ndarray]] = {}   # frame -> [qkv_1 .. qkv_L]  ([T, 3D] each)
    onehot = np.eye(4)
    for f in order:
        ftype = int(plan["type"][f])
        refs = {0: int(plan["past"][f]), 1: int(plan["future"][f])}
        has_refs = not dense and ftype != FTYPES["I"] and (refs[0] >= 0 or refs[1] >= 0)
        X = [patch_embed(W, patches[f])]
        XP: List[np.ndarray] = []
        QKV = [_qkv(W, 0, X[0])]                      # layer-0 chain: QKV_1 of every token
        t = np.full(N, 1.0 / N)                       # decision 1 uses uniform t
        for l in range(L):                            # 0-based layer index: layer l+1
            pre = f"L{l}."
            qkv = QKV[l]
            o, Pm = _attention_rows(qkv[:, :D], qkv[:, D:2 * D], qkv[:, 2 * D:], H)   # dense
            t_att = Pm[:, 0, 1:].mean(axis=0)
            xp = X[l] + o @ np.asarray(W[pre + "Wo"], _F64) + np.asarray(W[pre + "bo"], _F64)
            XP.append(xp)
            # ---- decision on the chain input x' (Eq. 1-4)
            M = np.zeros(N, np.uint8)
            prov = np.full(N, -1, np.int8)
            if has_refs:
                Tp = XPc[refs[0]][l][1:] if refs[0] >= 0 else None
                Tf = XPc[refs[1]][l][1:] if refs[1] >= 0 else None
                s, prov = similarity(xp[1:], Tp, Tf)
                v = np.concatenate([s[:, None], t[:, None], np.repeat(onehot[ftype][None, :], N, axis=0),
                                    np.asarray(codec[f], _F64)[:, None]], axis=1)
                d = decision_mlp(G, l, v)
                M = (d > 0).astype(np.uint8)
                if force_masks is not None:
                    M = np.asarray(force_masks[f, l], np.uint8).copy()
                d_all[f, l] = d
            M_all[f, l] = M
            C = np.concatenate([[0], 1 + np.flatnonzero(M == 0)])
            R = 1 + np.flatnonzero(M == 1)
            prov_tok = np.full(T, -1, np.int64)
            prov_tok[R] = [refs[int(prov[i - 1])] for i in R]
            # ---- chain FFN_l (C), restoration of the block output (R), Eq. 10 merge
            Xn = np.empty((T, D), _F64)
            h2 = layer_norm(xp[C], W[pre + "ln2_g"], W[pre + "ln2_b"])
            ff = quick_gelu(h2 @ np.asarray(W[pre + "W1"], _F64) + np.asarray(W[pre + "b1"], _F64))
            Xn[C] = xp[C] + ff @ np.asarray(W[pre + "W2"], _F64) + np.asarray(W[pre + "b2"], _F64)
            if len(R):
                dR = xp[R] - np.stack([XPc[prov_tok[i]][l][i] for i in R])
                Xn[R] = np.stack([Xc[prov_tok[i]][l + 1][i] for i in R]) + restoration_mlp(G, l, dR)
            X.append(Xn)
            # ---- chain QKV_{l+1}: computed for C, the provider's for R
            if l + 1 < L:
                qn = np.empty((T, 3 * D), _F64)
                qn[C] = _qkv(W, l + 1, Xn[C])
                for i in R:
                    qn[i] = QKVc[prov_tok[i]][l + 1][i]
                QKV.append(qn)
            t = t_att
        Z[f] = layer_norm(X[L][0], W["lnpost_g"], W["lnpost_b"])
        Xc[f], XPc[f], QKVc[f] = X, XP, QKV
    return {"Z": Z, "M": M_all, "d": d_all}
