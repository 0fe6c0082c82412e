"""Pure-Python, token-by-token, element-by-element ReuseViT for TINY configs.

A pin for the oracle (tests only): written independently of oracle/ with explicit
loops over tokens, heads and vector elements, plain Python floats (IEEE double), no
NumPy arithmetic.  It follows PAPER.md §3 Eq. 1-10 in order:

  Eq. 1  s_i = max(cos(T_cur_i, T_past_i), cos(T_cur_i, T_future_i))
  Eq. 2  v_i = concat(s_i, t_i, r_i, c_i)
  Eq. 3  d_i = MLP_decision(v_i)
  Eq. 4  M_i = 1 iff d_i > 0
  Eq. 5-6 C / R partition
  Eq. 7  recompute tokens: QKV and FFN
  Eq. 8-9 Delta R_i = R_cur_i - R_ref_i ; R_hat = R_tilde_ref + MLP_rest(Delta)
  Eq. 10 reconstruction in token order
with the readings of DESIGN.md §3 (layer-gated decision, provider = argmax with ties to
the past reference, t = previous-layer CLS attention head-mean, CLS never reused).
"""
import math


def _vec(a):
    return [float(x) for x in a]


def _mat(a):
    return [[float(x) for x in row] for row in a]


def matvec_rowvec(x, W, b):
    """y[j] = sum_k x[k] * W[k][j] + b[j]."""
    n_out = len(W[0])
    out = []
    for j in range(n_out):
        acc = 0.0
        for k in range(len(x)):
            acc += x[k] * W[k][j]
        out.append(acc + b[j])
    return out


def ln(x, g, b, eps=1e-5):
    n = len(x)
    mu = sum(x) / n
    var = sum((v - mu) * (v - mu) for v in x) / n
    inv = 1.0 / math.sqrt(var + eps)
    return [(x[k] - mu) * inv * g[k] + b[k] for k in range(n)]


def qgelu(v):
    return v / (1.0 + math.exp(-1.702 * v))


def cos(a, b):
    dot = sum(a[k] * b[k] for k in range(len(a)))
    na = sum(v * v for v in a)
    nb = sum(v * v for v in b)
    den = math.sqrt(na * nb)
    return 0.0 if den == 0.0 else dot / den


def run(cfg, W, G, patches, codec, plan, force_masks=None):
    """Returns (Z dict frame->list, M dict frame->[L][N], d dict frame->[L][N])."""
    L, D, H, N, T = cfg.layers, cfg.dim, cfg.heads, cfg.N, cfg.T
    dh = D // H
    Wl = {k: (_mat(v) if getattr(v, "ndim", 1) == 2 else _vec(v)) for k, v in W.items()}
    Gl = {k: (_mat(v) if getattr(v, "ndim", 1) == 2 else _vec(v)) for k, v in G.items()} if G else {}
    X = {}   # frame -> [layer][token] -> vector
    KV = {}  # frame -> [layer] -> (K tokens, V tokens)
    Zs, Ms, ds = {}, {}, {}
    for f in [int(v) for v in plan["order"]]:
        ftype = int(plan["type"][f])
        past, fut = int(plan["past"][f]), int(plan["future"][f])
        # patch embedding + CLS + positions + ln_pre
        toks = [list(Wl["cls"])]
        for i in range(N):
            toks.append(matvec_rowvec(_vec(patches[f][i]), Wl["W_pe"], [0.0] * D))
        toks = [[toks[i][k] + Wl["pos"][i][k] for k in range(D)] for i in range(T)]
        toks = [ln(tk, Wl["lnpre_g"], Wl["lnpre_b"]) for tk in toks]
        Xf = [toks]
        KVf = []
        t = [1.0 / N] * N
        Mf, df = [], []
        for l in range(L):
            p = f"L{l}."
            cur = Xf[l]
            M = [0] * N
            d = [float("nan")] * N
            prov = [None] * N
            if ftype != 0:
                onehot = [1.0 if k == ftype else 0.0 for k in range(4)]
                for i in range(N):
                    best, who = None, None
                    for who_k, r in (("past", past), ("future", fut)):
                        if r < 0:
                            continue
                        c = cos(cur[1 + i], X[r][l][1 + i])
                        if best is None or c > best:
                            best, who = c, r
                    v = [best, t[i]] + onehot + [float(codec[f][i])]
                    hidden = matvec_rowvec(v, Gl[p + "Wd1"], Gl[p + "bd1"])
                    hidden = [qgelu(h) for h in hidden]
                    di = sum(hidden[j] * Gl[p + "Wd2"][j] for j in range(len(hidden))) + Gl[p + "bd2"][0]
                    d[i] = di
                    M[i] = 1 if di > 0 else 0
                    if force_masks is not None:
                        M[i] = int(force_masks[f][l][i])
                    prov[i] = who
            Mf.append(M)
            df.append(d)
            C = [0] + [1 + i for i in range(N) if M[i] == 0]
            R = [1 + i for i in range(N) if M[i] == 1]
            K = [None] * T
            V = [None] * T
            Q = {}
            for i in C:
                h = ln(cur[i], Wl[p + "ln1_g"], Wl[p + "ln1_b"])
                qkv = matvec_rowvec(h, Wl[p + "Wqkv"], Wl[p + "bqkv"])
                Q[i] = qkv[:D]
                K[i] = qkv[D:2 * D]
                V[i] = qkv[2 * D:]
            for i in R:
                src = prov[i - 1]
                K[i] = KV[src][l][0][i]
                V[i] = KV[src][l][1][i]
            KVf.append((K, V))
            new = [None] * T
            t_next = [0.0] * N
            for i in C:
                o = [0.0] * D
                for h in range(H):
                    logits = []
                    for j in range(T):
                        acc = 0.0
                        for k in range(dh):
                            acc += Q[i][h * dh + k] * K[j][h * dh + k]
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
                            acc += pr[j] * V[j][h * dh + k]
                        o[h * dh + k] = acc
                x1 = matvec_rowvec(o, Wl[p + "Wo"], Wl[p + "bo"])
                x1 = [cur[i][k] + x1[k] for k in range(D)]
                h2 = ln(x1, Wl[p + "ln2_g"], Wl[p + "ln2_b"])
                ff = [qgelu(v) for v in matvec_rowvec(h2, Wl[p + "W1"], Wl[p + "b1"])]
                ff = matvec_rowvec(ff, Wl[p + "W2"], Wl[p + "b2"])
                new[i] = [x1[k] + ff[k] for k in range(D)]
            for i in R:
                src = prov[i - 1]
                delta = [cur[i][k] - X[src][l][i][k] for k in range(D)]
                hr = [qgelu(v) for v in matvec_rowvec(delta, Gl[p + "Wr1"], Gl[p + "br1"])]
                corr = matvec_rowvec(hr, Gl[p + "Wr2"], Gl[p + "br2"])
                new[i] = [X[src][l + 1][i][k] + corr[k] for k in range(D)]
            Xf.append(new)
            t = t_next
        X[f] = Xf
        KV[f] = KVf
        Zs[f] = ln(Xf[L][0], Wl["lnpost_g"], Wl["lnpost_b"])
        Ms[f] = Mf
        ds[f] = df
    return Zs, Ms, ds
