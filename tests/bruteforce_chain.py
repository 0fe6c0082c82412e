"""Pure-Python, token-by-token brute force of the SPEC chain variant for
TINY configs — a pin for oracle/chain_ref.py, written with explicit loops over tokens, heads
and elements (plain Python floats), following S:218-220 / S:230 / S:271-272:
  layer l: dense attention of every token (q, k, v of layer l) -> x' = X + o Wo + bo;
           decision on x' (Eq. 1-4, t = previous layer's CLS attention, uniform first);
           C: X_l = x' + FFN(LN2 x'), qkv_{l+1} = QKV_{l+1}(LN1 X_l);
           R: X_l = X_l^prov + MLP_rest(x'^f - x'^prov), qkv_{l+1} = qkv_{l+1}^prov.
"""
import math

from tests.bruteforce import _mat, _vec, cos, ln, matvec_rowvec, qgelu


def run(cfg, W, G, patches, codec, plan, force_masks=None):
    L, D, H, N, T = cfg.layers, cfg.dim, cfg.heads, cfg.N, cfg.T
    dh = D // H
    Wl = {k: (_mat(v) if getattr(v, "ndim", 1) == 2 else _vec(v)) for k, v in W.items()}
    Gl = {k: (_mat(v) if getattr(v, "ndim", 1) == 2 else _vec(v)) for k, v in G.items()} if G else {}
    X, XP, QKV = {}, {}, {}
    Zs, Ms = {}, {}

    def qkv_of(l, x):
        p = f"L{l}."
        return matvec_rowvec(ln(x, Wl[p + "ln1_g"], Wl[p + "ln1_b"]), Wl[p + "Wqkv"], Wl[p + "bqkv"])

    for f in [int(v) for v in plan["order"]]:
        ftype = int(plan["type"][f])
        past, fut = int(plan["past"][f]), int(plan["future"][f])
        toks = [list(Wl["cls"])] + [matvec_rowvec(_vec(patches[f][i]), Wl["W_pe"], [0.0] * D) for i in range(N)]
        toks = [ln([toks[i][k] + Wl["pos"][i][k] for k in range(D)], Wl["lnpre_g"], Wl["lnpre_b"]) for i in range(T)]
        Xf, XPf = [toks], []
        QKVf = [[qkv_of(0, toks[i]) for i in range(T)]]
        t = [1.0 / N] * N
        Mf = []
        for l in range(L):
            p = f"L{l}."
            qkv = QKVf[l]
            xp = []
            t_next = [0.0] * N
            for i in range(T):                       # dense attention + W_o for every token
                o = [0.0] * D
                for h in range(H):
                    logits = []
                    for j in range(T):
                        acc = 0.0
                        for k in range(dh):
                            acc += qkv[i][h * dh + k] * qkv[j][D + h * dh + k]
                        logits.append(acc / math.sqrt(dh))
                    mx = max(logits)
                    e = [math.exp(v - mx) for v in logits]
                    ssum = sum(e)
                    pr = [v / ssum for v in e]
                    if i == 0:
                        for j in range(1, T):
                            t_next[j - 1] += pr[j] / H
                    for k in range(dh):
                        acc = 0.0
                        for j in range(T):
                            acc += pr[j] * qkv[j][2 * D + h * dh + k]
                        o[h * dh + k] = acc
                y = matvec_rowvec(o, Wl[p + "Wo"], Wl[p + "bo"])
                xp.append([Xf[l][i][k] + y[k] for k in range(D)])
            XPf.append(xp)
            M = [0] * N
            prov = [None] * N
            if ftype != 0:
                onehot = [1.0 if k == ftype else 0.0 for k in range(4)]
                for i in range(N):
                    best, who = None, None
                    for r in (past, fut):
                        if r < 0:
                            continue
                        c = cos(xp[1 + i], XP[r][l][1 + i])
                        if best is None or c > best:
                            best, who = c, r
                    v = [best, t[i]] + onehot + [float(codec[f][i])]
                    hid = [qgelu(hv) for hv in matvec_rowvec(v, Gl[p + "Wd1"], Gl[p + "bd1"])]
                    di = sum(hid[j] * Gl[p + "Wd2"][j] for j in range(len(hid))) + Gl[p + "bd2"][0]
                    M[i] = 1 if di > 0 else 0
                    if force_masks is not None:
                        M[i] = int(force_masks[f][l][i])
                    prov[i] = who
            Mf.append(M)
            new = [None] * T
            nq = [None] * T
            for i in range(T):
                if i == 0 or M[i - 1] == 0:
                    h2 = ln(xp[i], Wl[p + "ln2_g"], Wl[p + "ln2_b"])
                    ff = matvec_rowvec([qgelu(v) for v in matvec_rowvec(h2, Wl[p + "W1"], Wl[p + "b1"])],
                                       Wl[p + "W2"], Wl[p + "b2"])
                    new[i] = [xp[i][k] + ff[k] for k in range(D)]
                    if l + 1 < L:
                        nq[i] = qkv_of(l + 1, new[i])
                else:
                    src = prov[i - 1]
                    delta = [xp[i][k] - XP[src][l][i][k] for k in range(D)]
                    hr = [qgelu(v) for v in matvec_rowvec(delta, Gl[p + "Wr1"], Gl[p + "br1"])]
                    corr = matvec_rowvec(hr, Gl[p + "Wr2"], Gl[p + "br2"])
                    new[i] = [X[src][l + 1][i][k] + corr[k] for k in range(D)]
                    if l + 1 < L:
                        nq[i] = QKV[src][l + 1][i]
            Xf.append(new)
            if l + 1 < L:
                QKVf.append(nq)
            t = t_next
        X[f], XP[f], QKV[f] = Xf, XPf, QKVf
        Zs[f] = ln(Xf[L][0], Wl["lnpost_g"], Wl["lnpost_b"])
        Ms[f] = Mf
    return Zs, Ms
