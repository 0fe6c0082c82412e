"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Plain float64 NumPy ReuseViT, frame-sequential in the plan's computation order.
Citations: ``P:n`` = /root/reference/PAPER.md line n, ``S:n`` = SPEC.md line n,
``SURVEY`` = /root/repo/SURVEY.md section.  Readings of ambiguous passages: DESIGN.md §3.
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional

import numpy as np

# Frame types, one-hot order of the reference-type feature r.
FTYPES = {"I": 0, "P": 1, "B2": 2, "B1": 3}
_F64 = np.float64


# ----------------------------------------------------------------------------- helpers
def layer_norm(x: np.ndarray, g: np.ndarray, b: np.ndarray, eps: float = 1e-5) -> np.ndarray:
    """LN(x) = (x - mean) / sqrt(var + eps) * g + b over the last axis, biased variance
    (pre-norm CLIP ViT).  Pinned: torch F.layer_norm (fp64)."""
    x = np.asarray(x, dtype=_F64)
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * np.asarray(g, _F64) + np.asarray(b, _F64)


def quick_gelu(x: np.ndarray) -> np.ndarray:
    """QuickGELU(x) = x * sigmoid(1.702 x) (OpenAI-CLIP activation; "All models use
    CLIP")."""
    x = np.asarray(x, dtype=_F64)
    return x / (1.0 + np.exp(-1.702 * x))


def cosine(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Row-wise cos(a,b) = a.b / sqrt(|a|^2 |b|^2); 0 when the denominator is 0
    (Eq. 1; zero-norm convention S:45, S:76 / SURVEY Q9).  Pinned: brute force."""
    a = np.asarray(a, _F64)
    b = np.asarray(b, _F64)
    num = (a * b).sum(axis=-1)
    den = np.sqrt((a * a).sum(axis=-1) * (b * b).sum(axis=-1))
    out = np.zeros_like(num)
    nz = den > 0
    out[nz] = num[nz] / den[nz]
    return out


# ----------------------------------------------------------------------------- plan
def plan_gop(n: int, refresh: int = 20, reorder: bool = True) -> Dict[str, np.ndarray]:
    """Frame typing and computation order ("I -> (P -> B_dist2 -> B_dist1 ->
    B_dist1)"; P:583-587 I-frame every 20th frame; S:308-316 plan_gop; S:341-342 tail).

    5-frame unit over display indices [4u .. 4u+4]: anchor 4u+4 is P referencing 4u (or I
    when (4u+4) % refresh == 0), 4u+2 is B2 referencing (4u, 4u+4), 4u+1 and 4u+3 are B1
    referencing their immediate neighbours.  Computation order per unit: anchor, B2, B1, B1
    ("computation order 0,4,2,1,3").  A future reference beyond the last frame is
    dropped (past-only degradation).  ``reorder=False`` is the low-latency mode
    (P:579-581): every non-I frame is a P referencing its predecessor.
    Returns display-indexed arrays type (int8, FTYPES), past, future (int32, -1 = none)
    and the computation order (int32).  Pinned: S:314-316 examples (tests/golden/plan.json)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if refresh < 4 or refresh % 4 != 0:
        raise ValueError("refresh must be a multiple of 4 (S:310)")
    typ = np.zeros(n, np.int8)
    past = np.full(n, -1, np.int32)
    fut = np.full(n, -1, np.int32)
    order: List[int] = []
    if not reorder:
        for i in range(n):
            if i % refresh == 0:
                typ[i] = FTYPES["I"]
            else:
                typ[i] = FTYPES["P"]
                past[i] = i - 1
            order.append(i)
        return {"type": typ, "past": past, "future": fut, "order": np.array(order, np.int32)}
    order.append(0)
    typ[0] = FTYPES["I"]
    u = 0
    while 4 * u + 1 < n:
        a0, a1 = 4 * u, 4 * u + 4
        if a1 < n:
            if a1 % refresh == 0:
                typ[a1] = FTYPES["I"]
            else:
                typ[a1] = FTYPES["P"]
                past[a1] = a0
            order.append(a1)
        have_a1 = a1 < n
        b2 = a0 + 2
        if b2 < n:
            typ[b2] = FTYPES["B2"]
            past[b2] = a0
            fut[b2] = a1 if have_a1 else -1
            order.append(b2)
        for b1 in (a0 + 1, a0 + 3):
            if b1 < n:
                typ[b1] = FTYPES["B1"]
                past[b1] = b1 - 1
                fut[b1] = b1 + 1 if b1 + 1 < n else -1
                order.append(b1)
        u += 1
    return {"type": typ, "past": past, "future": fut, "order": np.array(order, np.int32)}


def plan_levels(plan: Dict[str, np.ndarray]) -> np.ndarray:
    """ASAP dependency level of every frame: 0 for reference-free frames, else
    1 + max(level of its references) (SURVEY D8 reading of P:571-574 batching; the
    level schedule is a GPU batching choice and is math-neutral)."""
    n = len(plan["type"])
    lev = np.full(n, -1, np.int64)
    for f in plan["order"]:
        refs = [r for r in (plan["past"][f], plan["future"][f]) if r >= 0]
        for r in refs:
            if lev[r] < 0:
                raise ValueError("reference used before it is computed (S:316)")
        lev[f] = 0 if not refs else 1 + max(lev[r] for r in refs)
    return lev


# ----------------------------------------------------------------------------- model pieces
def patch_embed(W: Dict[str, np.ndarray], patches_f: np.ndarray) -> np.ndarray:
    """X_0 = LN_pre(concat(cls, patches @ W_pe) + pos): patches are linearly embedded, a
    CLS token is added, positions are added (CLIP ln_pre).
    Returns [T, D] float64.  Pinned: torch fp64 library ViT."""
    E = np.asarray(patches_f, _F64) @ np.asarray(W["W_pe"], _F64)
    X = np.concatenate([np.asarray(W["cls"], _F64)[None, :], E], axis=0) + np.asarray(W["pos"], _F64)
    return layer_norm(X, W["lnpre_g"], W["lnpre_b"])


def similarity(T_cur: np.ndarray, T_past: Optional[np.ndarray], T_future: Optional[np.ndarray]):
    """Eq. 1: s_i = max(cos(T_cur_i, T_past_i), cos(T_cur_i, T_future_i)) over the
    *available* references; also returns the provider (0 = past, 1 = future) that attains
    the max, ties -> past.  Inputs are [N, D] patch rows."""
    refs = [(0, T_past), (1, T_future)]
    best = None
    prov = None
    for k, R in refs:
        if R is None:
            continue
        c = cosine(T_cur, R)
        if best is None:
            best, prov = c, np.full(c.shape, k, np.int8)
        else:
            take = c > best            # strict: ties keep the past reference
            best = np.where(take, c, best)
            prov = np.where(take, np.int8(k), prov)
    return best, prov


def decision_mlp(G: Dict[str, np.ndarray], l: int, v: np.ndarray) -> np.ndarray:
    """Eq. 3: d_i = MLP_decision(v_i), a two-layer MLP 7 -> Hg -> 1 with
    QuickGELU (hidden size and activation are a reading, parity unpinned
    against the paper's trained model; pinned here by forced-logit and brute-force tests)."""
    h = quick_gelu(np.asarray(v, _F64) @ np.asarray(G[f"L{l}.Wd1"], _F64) + np.asarray(G[f"L{l}.bd1"], _F64))
    return h @ np.asarray(G[f"L{l}.Wd2"], _F64) + np.asarray(G[f"L{l}.bd2"], _F64)[0]


def restoration_mlp(G: Dict[str, np.ndarray], l: int, dR: np.ndarray) -> np.ndarray:
    """Eq. 9 MLP_restoration(Delta R_i): two-layer MLP D -> 128 -> D (P:377
    "hidden size of 128"), QuickGELU."""
    h = quick_gelu(np.asarray(dR, _F64) @ np.asarray(G[f"L{l}.Wr1"], _F64) + np.asarray(G[f"L{l}.br1"], _F64))
    return h @ np.asarray(G[f"L{l}.Wr2"], _F64) + np.asarray(G[f"L{l}.br2"], _F64)


def _attention_rows(q: np.ndarray, K: np.ndarray, V: np.ndarray, H: int):
    """Multi-head self-attention for the query rows q [m, D] over all T keys/values of the
    frame (every recomputed query attends to all tokens).  Scale 1/sqrt(d_h)
    (SURVEY Q14).  Returns (o [m, D], p [H, m, T] softmax probabilities)."""
    m, D = q.shape
    dh = D // H
    o = np.empty((m, D), _F64)
    P = np.empty((H, m, K.shape[0]), _F64)
    for h in range(H):
        sl = slice(h * dh, (h + 1) * dh)
        S = q[:, sl] @ K[:, sl].T / math.sqrt(dh)
        S = S - S.max(axis=1, keepdims=True)
        E = np.exp(S)
        P[h] = E / E.sum(axis=1, keepdims=True)
        o[:, sl] = P[h] @ V[:, sl]
    return o, P


# ----------------------------------------------------------------------------- forward
def reuse_embed(cfg, W: Dict[str, np.ndarray], G: Optional[Dict[str, np.ndarray]],
                patches: np.ndarray, codec: np.ndarray, plan: Dict[str, np.ndarray],
                dense: bool = False, force_masks: Optional[np.ndarray] = None,
                frames: Optional[List[int]] = None, trace: bool = False) -> Dict[str, np.ndarray]:
    """ReuseViT forward, frame-sequentially in ``plan['order']`` (P:576-578 reordering
    inside the forward pass; results returned in display order).

    Per frame f and layer l = 1..L (SURVEY §8(c) algorithm, D1 layer-gated reading):
      * I-frames / ``dense``: M = 0 (no references).
      * else Eq. 1 s_i and provider; v_i = [s_i, t_i, onehot(r), c_i] (Eq. 2);
        d_i = MLP_decision(v_i) (Eq. 3); M_i = 1 iff d_i > 0 (Eq. 4);
        ``force_masks[f, l-1]`` overrides M (diagnostic).
      * C = {CLS} u {i: M_i = 0}, R = {i: M_i = 1} (Eq. 5-6; CLS never reused,
        S:182).
      * C rows: LN1 -> QKV (Eq. 7 QKV part); R rows take K_l, V_l of the provider
        (reused QKV computation); attention of C queries over all T keys; t for the
        next layer = head-mean CLS probability over patch keys;
        x' = X + o Wo + bo; X_l = x' + FFN(LN2 x') (Eq. 7 FFN part).
      * R rows: Delta = X^f_{l-1} - X^prov_{l-1} (Eq. 8); X_l = X^prov_l +
        MLP_restoration(Delta) (Eq. 9).
      * Rows merged in token order (Eq. 10).
    Z_f = LN_post(X_L[CLS]).

    ``frames`` restricts computation to a prefix-closed subset (every reference of a listed
    frame must be listed); outputs of other frames are NaN.  Returns dict with Z [n, D],
    M [n, L, N] uint8, d [n, L, N] float64 (NaN where no decision ran), prov [n, L, N]
    int8 (-1 where none), s [n, L, N], t [n, L, N] (the t fed to the decision),
    and if ``trace`` X [n][L+1] arrays."""
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
    # remaining dependents, to free caches once no later frame needs them
    dependents = {f: 0 for f in order}
    for f in order:
        for r in (plan["past"][f], plan["future"][f]):
            if r >= 0:
                dependents[int(r)] += 1

    Z = np.full((n, D), np.nan)
    M_all = np.zeros((n, L, N), np.uint8)
    d_all = np.full((n, L, N), np.nan)
    s_all = np.full((n, L, N), np.nan)
    t_all = np.full((n, L, N), np.nan)
    prov_all = np.full((n, L, N), -1, np.int8)
    Xc: Dict[int, List[np.ndarray]] = {}   # frame -> [X_0..X_L]       (ActivationCache)
    KVc: Dict[int, List[tuple]] = {}       # frame -> [(K_1,V_1)..]
    tr = {} if trace else None
    dh_onehot = np.eye(4)

    for f in order:
        ftype = int(plan["type"][f])
        refs = {0: int(plan["past"][f]), 1: int(plan["future"][f])}
        X = [patch_embed(W, patches[f])]
        KV: List[tuple] = []
        t = np.full(N, 1.0 / N)                      # layer 1 uses uniform t
        for l in range(L):
            Xp = X[l]
            pre = f"L{l}."
            # ---- decision (Eq. 1-4)
            M = np.zeros(N, np.uint8)
            prov = np.full(N, -1, np.int8)
            if not dense and ftype != FTYPES["I"] and (refs[0] >= 0 or refs[1] >= 0):
                Tp = Xc[refs[0]][l][1:] if refs[0] >= 0 else None
                Tf = Xc[refs[1]][l][1:] if refs[1] >= 0 else None
                s, prov = similarity(Xp[1:], Tp, Tf)
                v = np.concatenate([s[:, None], t[:, None],
                                    np.repeat(dh_onehot[ftype][None, :], N, axis=0),
                                    np.asarray(codec[f], _F64)[:, None]], axis=1)
                d = decision_mlp(G, l, v)
                M = (d > 0).astype(np.uint8)                   # Eq. 4, strict
                if force_masks is not None:
                    M = np.asarray(force_masks[f, l], np.uint8).copy()
                d_all[f, l] = d
                s_all[f, l] = s
                t_all[f, l] = t
                prov_all[f, l] = prov
            M_all[f, l] = M
            # ---- filtration (Eq. 5-6): token 0 = CLS always in C
            C = np.concatenate([[0], 1 + np.flatnonzero(M == 0)])
            R = 1 + np.flatnonzero(M == 1)
            prov_tok = np.full(T, -1, np.int64)
            prov_tok[R] = [refs[int(prov[i - 1])] for i in R]
            # ---- recompute path, QKV part (Eq. 7)
            h1 = layer_norm(Xp[C], W[pre + "ln1_g"], W[pre + "ln1_b"])
            qkv = h1 @ np.asarray(W[pre + "Wqkv"], _F64) + np.asarray(W[pre + "bqkv"], _F64)
            q = qkv[:, :D]
            K = np.empty((T, D), _F64)
            V = np.empty((T, D), _F64)
            K[C] = qkv[:, D:2 * D]
            V[C] = qkv[:, 2 * D:]
            for i in R:                                   # reused QKV computation
                Kp, Vp = KVc[prov_tok[i]][l]
                K[i] = Kp[i]
                V[i] = Vp[i]
            KV.append((K, V))
            o, Pm = _attention_rows(q, K, V, H)
            t = Pm[:, 0, 1:].mean(axis=0)                  # C[0] is CLS
            # ---- recompute path, FFN part (Eq. 7)
            x1 = Xp[C] + o @ np.asarray(W[pre + "Wo"], _F64) + np.asarray(W[pre + "bo"], _F64)
            h2 = layer_norm(x1, W[pre + "ln2_g"], W[pre + "ln2_b"])
            ff = quick_gelu(h2 @ np.asarray(W[pre + "W1"], _F64) + np.asarray(W[pre + "b1"], _F64))
            Ctil = x1 + ff @ np.asarray(W[pre + "W2"], _F64) + np.asarray(W[pre + "b2"], _F64)
            # ---- restoration (Eq. 8-9) and reconstruction (Eq. 10)
            Xn = np.empty((T, D), _F64)
            Xn[C] = Ctil
            if len(R):
                Rcur = Xp[R]
                Rref = np.stack([Xc[prov_tok[i]][l][i] for i in R])
                Rtil_ref = np.stack([Xc[prov_tok[i]][l + 1][i] for i in R])
                Xn[R] = Rtil_ref + restoration_mlp(G, l, Rcur - Rref)
            X.append(Xn)
        Z[f] = layer_norm(X[L][0], W["lnpost_g"], W["lnpost_b"])
        Xc[f] = X
        KVc[f] = KV
        if trace:
            tr[f] = X
        for r in set(v for v in refs.values() if v >= 0):
            dependents[r] -= 1
            if dependents[r] == 0 and not trace:
                del Xc[r], KVc[r]
        if dependents[f] == 0 and not trace:
            del Xc[f], KVc[f]
    out = {"Z": Z, "M": M_all, "d": d_all, "prov": prov_all, "s": s_all, "t": t_all}
    if trace:
        out["X"] = tr
    return out


def dense_embed(cfg, W, patches: np.ndarray) -> np.ndarray:
    """Plain ViT forward of every frame (M = 0 everywhere): the no-reuse special case
    ("forcing M = 0 yields Z_hat = dense Z").  Returns Z [n, D]."""
    n = patches.shape[0]
    plan = {"type": np.zeros(n, np.int8), "past": np.full(n, -1, np.int32),
            "future": np.full(n, -1, np.int32), "order": np.arange(n, dtype=np.int32)}
    return reuse_embed(cfg, W, None, patches, np.zeros((n, cfg.N)), plan, dense=True)["Z"]


# ----------------------------------------------------------------------------- compaction
def compaction_indices(masks: np.ndarray):
    """Stream compaction of one level-wave (Eq. 5-6; §5.3 P:535-538 "gathering
    active tokens ... into contiguous memory"): ``masks`` [n_w, T] uint8 for the wave's
    frames in ascending computation-order position, column 0 = CLS (ignored: always C).
    Rows are enumerated w*T + token.  Returns (idxC, idxR, qoff) with
    idxC = flatnonzero(token == 0 or M == 0), idxR = flatnonzero(M == 1 and token > 0),
    qoff = [0, cumsum(|C_w|)] (SURVEY §8(c) compaction-index oracle).
    Pinned: tests/golden/compaction.json (SURVEY worked vector)."""
    masks = np.asarray(masks, np.uint8)
    n_w, T = masks.shape
    isC = (masks == 0)
    isC[:, 0] = True
    flatC = isC.reshape(-1)
    idxC = np.flatnonzero(flatC).astype(np.int32)
    idxR = np.flatnonzero(~flatC).astype(np.int32)
    qoff = np.concatenate([[0], np.cumsum(isC.sum(axis=1))]).astype(np.int32)
    return idxC, idxR, qoff


# ----------------------------------------------------------------------------- accounting
def flops_per_frame(cfg, n_C: np.ndarray, n_R: np.ndarray) -> float:
    """Executed tensor FLOPs of one frame given per-layer recompute/reuse counts
    (SURVEY §8(d)): 2*N*pp*D (patch embed) + sum_l [n_C,l*(24 D^2 + 4 T D) + n_R,l*4*D*Hr].
    24D^2 = QKV 6D^2 + W_o 2D^2 + FFN 16D^2 (F = 4D); 4TD = attention QK^T + PV."""
    D, T, N, pp, Hr, F = cfg.dim, cfg.T, cfg.N, cfg.pp, cfg.hidden_r, cfg.ffn
    per_c = 2 * D * 3 * D + 2 * D * D + 2 * D * F * 2 + 4 * T * D
    per_r = 2 * D * Hr * 2
    return float(2 * N * pp * D + np.sum(np.asarray(n_C) * per_c) + np.sum(np.asarray(n_R) * per_r))


def reuse_rates(M: np.ndarray, types: np.ndarray, T: int):
    """Eq. 14 reuse rate = mean of M over layers and patch tokens, over non-I frames
    (``reuse_nonI``); ``reuse_all`` = reused token-layers / all T token-layers of all frames
    (the FLOP-relevant form)."""
    M = np.asarray(M, np.float64)
    nonI = np.asarray(types) != FTYPES["I"]
    reuse_nonI = float(M[nonI].mean()) if nonI.any() else 0.0
    reuse_all = float(M.sum() / (M.shape[0] * M.shape[1] * T))
    return reuse_nonI, reuse_all
