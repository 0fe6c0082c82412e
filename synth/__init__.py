"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no cosine, no gating, no
compaction, no ViT math).  It only draws random numbers and lays them out in the
interface orders the two sides agree on:

* ``ViTConfig``      — model dimensions (SURVEY §8 notation, BASELINE.json configs).
* ``make_vit``       — random-init ViT weights, dict in RVW1 declaration order
                       ("flat f32 arrays in declared order").
* ``make_gates``     — decision + restoration weights, dict per layer in RVG1 order
                       (SPEC.md:280), including the structured "learned-like" gate of
                       SURVEY §8(d) (``Wd1[s,0]=16, bd1[0]=-16*tau, Wd2[0]=1, bd2=-1``).
* ``make_video``     — patch-space frames ``[n, N, pp]`` with controlled inter-frame
                       motion probability ``p`` plus the codec-metadata stub ``c``
                       ("motion vectors and residuals").
* ``pack_vit`` / ``pack_gates`` — flatten the dicts to the little-endian fp32 blobs
                       that ``rv_load_vit`` / ``rv_load_gates`` take (include/reusevit.h).

Seeds: weights 1234, gates 1235, video v -> 2000+v, numpy PCG64.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List

import numpy as np

__all__ = [
    "ViTConfig", "CONFIGS", "make_vit", "make_gates", "make_video", "make_video_torch",
    "pack_vit", "pack_gates", "vit_array_order", "gate_array_order", "make_gumbel", "make_train_groups",
    "init_train_gates",
]


@dataclasses.dataclass(frozen=True)
class ViTConfig:
    """Model dimensions.  ``N=(img/patch)^2`` patch tokens, ``T=N+1`` with CLS,
    ``pp=3*patch^2`` pixels per patch (channel-major (3,P,P) flatten)."""
    layers: int
    dim: int
    heads: int
    patch: int
    img: int
    ffn: int
    hidden_r: int = 128   # restoration hidden size, PAPER.md:377 ("hidden size of 128")
    hidden_g: int = 32    # decision-MLP hidden size (SURVEY D4 / Q4 reading)

    @property
    def N(self) -> int:
        return (self.img // self.patch) ** 2

    @property
    def T(self) -> int:
        return self.N + 1

    @property
    def pp(self) -> int:
        return 3 * self.patch * self.patch

    @property
    def dh(self) -> int:
        return self.dim // self.heads


# BASELINE.json "configs" (SURVEY §8 notation table).
CONFIGS: Dict[str, ViTConfig] = {
    "tiny": ViTConfig(layers=2, dim=64, heads=4, patch=16, img=64, ffn=256),
    "b16": ViTConfig(layers=12, dim=768, heads=12, patch=16, img=224, ffn=3072),
    "l14": ViTConfig(layers=24, dim=1024, heads=16, patch=14, img=224, ffn=4096),
    "l14_336": ViTConfig(layers=24, dim=1024, heads=16, patch=14, img=336, ffn=4096),
}


def vit_array_order(cfg: ViTConfig) -> List[tuple]:
    """(name, shape) in RVW1 declaration order (SURVEY §8(c) "Parameters")."""
    D, T, F, pp = cfg.dim, cfg.T, cfg.ffn, cfg.pp
    order = [("W_pe", (pp, D)), ("cls", (D,)), ("pos", (T, D)),
             ("lnpre_g", (D,)), ("lnpre_b", (D,))]
    for l in range(cfg.layers):
        order += [
            (f"L{l}.ln1_g", (D,)), (f"L{l}.ln1_b", (D,)),
            (f"L{l}.Wqkv", (D, 3 * D)), (f"L{l}.bqkv", (3 * D,)),
            (f"L{l}.Wo", (D, D)), (f"L{l}.bo", (D,)),
            (f"L{l}.ln2_g", (D,)), (f"L{l}.ln2_b", (D,)),
            (f"L{l}.W1", (D, F)), (f"L{l}.b1", (F,)),
            (f"L{l}.W2", (F, D)), (f"L{l}.b2", (D,)),
        ]
    order += [("lnpost_g", (D,)), ("lnpost_b", (D,))]
    return order


def gate_array_order(cfg: ViTConfig) -> List[tuple]:
    """(name, shape) in RVG1 declaration order (SURVEY §8(c) "Gates (RVG1)")."""
    D, Hr, Hg = cfg.dim, cfg.hidden_r, cfg.hidden_g
    order = []
    for l in range(cfg.layers):
        order += [
            (f"L{l}.Wd1", (7, Hg)), (f"L{l}.bd1", (Hg,)),
            (f"L{l}.Wd2", (Hg,)), (f"L{l}.bd2", (1,)),
            (f"L{l}.Wr1", (D, Hr)), (f"L{l}.br1", (Hr,)),
            (f"L{l}.Wr2", (Hr, D)), (f"L{l}.br2", (D,)),
        ]
    return order


def make_vit(cfg: ViTConfig, seed: int = 1234, random_ln: bool = False,
             std: float = 0.02) -> Dict[str, np.ndarray]:
    """Random-init ViT weights: matrices, embeddings and linear biases ~ N(0, std)
    ("scaled Gaussian, std 0.02"); LN gamma=1, beta=0 unless ``random_ln``
    (tests use random LN parameters so a swapped gamma/beta cannot pass)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out: Dict[str, np.ndarray] = {}
    for name, shape in vit_array_order(cfg):
        base = name.split(".")[-1]
        if base.endswith("_g"):
            out[name] = (1.0 + 0.1 * rng.standard_normal(shape)) if random_ln else np.ones(shape)
        elif base.endswith("_b") and base.startswith("ln"):
            out[name] = (0.1 * rng.standard_normal(shape)) if random_ln else np.zeros(shape)
        else:
            out[name] = std * rng.standard_normal(shape)
        out[name] = out[name].astype(np.float32)
    return out


def make_gates(cfg: ViTConfig, seed: int = 1235, tau: float = 0.7, slope: float = 16.0,
               structured: bool = True, restore_bias: bool = False,
               final_bias: float | None = None, zero_decision: bool = False,
               restore_std: float = 0.02) -> Dict[str, np.ndarray]:
    """Decision + restoration weights per layer (RVG1 order).

    ``structured`` builds SURVEY §8(d)'s learned-like gate: ``Wd1 ~ N(0,.02)`` then
    ``Wd1[s,0]=slope``, ``bd1[0]=-slope*tau``; ``Wd2 ~ N(0,.02)`` then ``Wd2[0]=1``,
    ``bd2=-1``.  ``zero_decision`` zeroes every decision weight so that ``d == bd2``
    (with ``final_bias`` = +-10 this is SPEC.md:205-206's forced-logit example).
    Restoration weights ~ N(0, restore_std); biases zero unless ``restore_bias``.
    Feature order of Wd1's 7 rows: [s, t, 1[I], 1[P], 1[B2], 1[B1], c]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out: Dict[str, np.ndarray] = {}
    for l in range(cfg.layers):
        Hg, Hr, D = cfg.hidden_g, cfg.hidden_r, cfg.dim
        Wd1 = 0.02 * rng.standard_normal((7, Hg))
        bd1 = 0.02 * rng.standard_normal(Hg)
        Wd2 = 0.02 * rng.standard_normal(Hg)
        bd2 = 0.02 * rng.standard_normal(1)
        if structured:
            Wd1[0, 0] = slope
            bd1[0] = -slope * tau
            Wd2[0] = 1.0
            bd2[0] = -1.0
        if zero_decision:
            Wd1[:] = 0
            bd1[:] = 0
            Wd2[:] = 0
            bd2[:] = 0
        if final_bias is not None:
            bd2[0] = final_bias
        Wr1 = restore_std * rng.standard_normal((D, Hr))
        br1 = 0.02 * rng.standard_normal(Hr) if restore_bias else np.zeros(Hr)
        Wr2 = restore_std * rng.standard_normal((Hr, D))
        br2 = 0.02 * rng.standard_normal(D) if restore_bias else np.zeros(D)
        for k, v in (("Wd1", Wd1), ("bd1", bd1), ("Wd2", Wd2), ("bd2", bd2),
                     ("Wr1", Wr1), ("br1", br1), ("Wr2", Wr2), ("br2", br2)):
            out[f"L{l}.{k}"] = np.asarray(v, dtype=np.float32)
    return out


def _pack(d: Dict[str, np.ndarray], order) -> np.ndarray:
    parts = []
    for name, shape in order:
        a = np.asarray(d[name], dtype=np.float32)
        if a.shape != tuple(shape):
            raise ValueError(f"{name}: shape {a.shape} != {shape}")
        parts.append(a.reshape(-1))
    return np.ascontiguousarray(np.concatenate(parts).astype("<f4"))


def pack_vit(cfg: ViTConfig, w: Dict[str, np.ndarray]) -> np.ndarray:
    """Flat little-endian fp32 blob in RVW1 declaration order (no header)."""
    return _pack(w, vit_array_order(cfg))


def pack_gates(cfg: ViTConfig, g: Dict[str, np.ndarray]) -> np.ndarray:
    """Flat little-endian fp32 blob in RVG1 declaration order (no header)."""
    return _pack(g, gate_array_order(cfg))


def make_video(cfg: ViTConfig, n: int, p: float, seed: int = 2000, mode: str = "bimodal",
               noise: float = 0.02, duplicate_of: dict | None = None):
    """Patch-space frames ``[n, N, pp]`` fp32 in display order and codec stub ``[n, N]``.

    ``bimodal`` (SURVEY §8(d) generator): frame 0 ~ N(0,1) iid; at each display step each
    patch independently *moves* with probability ``p`` (fresh N(0,1) content), otherwise it
    stays plus N(0, noise^2).  ``continuous`` (mask-parity stress mode):
    ``x <- sqrt(1-a^2) x + a*fresh`` with ``a ~ U(0,1)`` per patch per step.
    Codec stub ``c[f,i] = RMS(x_f[i] - x_{f-1}[i])`` (0 for frame 0).
    ``duplicate_of`` = {dst: src} copies frame src into dst afterwards (T-DUP tests)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    N, pp = cfg.N, cfg.pp
    x = np.empty((n, N, pp), dtype=np.float32)
    x[0] = rng.standard_normal((N, pp), dtype=np.float32)
    for f in range(1, n):
        prev = x[f - 1]
        if mode == "bimodal":
            move = rng.random(N) < p
            fresh = rng.standard_normal((N, pp), dtype=np.float32)
            stay = prev + noise * rng.standard_normal((N, pp), dtype=np.float32)
            x[f] = np.where(move[:, None], fresh, stay)
        elif mode == "continuous":
            a = rng.random(N).astype(np.float32)[:, None]
            fresh = rng.standard_normal((N, pp), dtype=np.float32)
            x[f] = np.sqrt(1 - a * a) * prev + a * fresh
        else:
            raise ValueError(mode)
    if duplicate_of:
        for dst, src in duplicate_of.items():
            x[dst] = x[src]
    codec = np.zeros((n, N), dtype=np.float32)
    if n > 1:
        codec[1:] = np.sqrt(np.mean((x[1:] - x[:-1]) ** 2, axis=2))
    return x, codec


def make_video_torch(cfg: ViTConfig, n: int, p: float, seed: int = 2000, device="cuda",
                     noise: float = 0.02):
    """Same distribution as ``make_video(mode='bimodal')`` drawn with a torch generator
    on ``device`` (different random stream; used by bench.py for the 7,200-frame
    workload where numpy generation would dominate).  Returns (patches fp32 [n,N,pp],
    codec fp32 [n,N]) on ``device``."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    N, pp = cfg.N, cfg.pp
    x = torch.empty((n, N, pp), dtype=torch.float32, device=device)
    x[0] = torch.randn((N, pp), generator=g, device=device)
    for f in range(1, n):
        move = torch.rand((N, 1), generator=g, device=device) < p
        fresh = torch.randn((N, pp), generator=g, device=device)
        stay = x[f - 1] + noise * torch.randn((N, pp), generator=g, device=device)
        x[f] = torch.where(move, fresh, stay)
    codec = torch.zeros((n, N), dtype=torch.float32, device=device)
    if n > 1:
        codec[1:] = ((x[1:] - x[:-1]) ** 2).mean(dim=2).sqrt()
    return x, codec


def make_gumbel(shape, seed: int) -> np.ndarray:
    """Standard Gumbel(0, 1) draws -log(-log(U)), U ~ U(0, 1) (PCG64), float32: the random
    numbers Eq. 11's Gumbel-Softmax draws, passed to both sides as inputs."""
    rng = np.random.Generator(np.random.PCG64(seed))
    u = rng.random(shape)
    u = np.clip(u, 1e-12, 1.0 - 1e-12)
    return (-np.log(-np.log(u))).astype(np.float32)


def make_train_groups(cfg: ViTConfig, B: int, display, seed: int, p_range=(0.05, 0.4)):
    """B training groups (P:478-482 grouped frames): each group is drawn from its own
    ``max(display)+1``-frame bimodal clip with motion p ~ U(p_range); returns the frames at the
    given 0-based display indices (ascending) as (patches [B, G, N, pp], codec [B, G, N]).
    The codec stub stays relative to the previous DISPLAY frame of the clip."""
    rng = np.random.Generator(np.random.PCG64(seed))
    disp = sorted(int(d) for d in display)
    n = disp[-1] + 1
    xs, cs = [], []
    for b in range(B):
        p = float(rng.uniform(*p_range))
        x, c = make_video(cfg, n, p, seed=int(rng.integers(1 << 31)))
        xs.append(x[disp])
        cs.append(c[disp])
    return np.stack(xs), np.stack(cs)


def init_train_gates(cfg: ViTConfig, seed: int = 1236) -> Dict[str, np.ndarray]:
    """Initial gates of a training run ("restoration MLP's final layer is
    zero-initialized; decision MLP final bias initialized to -1 (recompute-leaning)"):
    decision and first restoration layer ~ N(0, 0.02), Wr2 = 0, biases 0, bd2 = -1."""
    return make_gates(cfg, seed=seed, structured=False, final_bias=-1.0, restore_bias=False,
                      restore_std=0.02) | {f"L{l}.Wr2": np.zeros((cfg.hidden_r, cfg.dim), np.float32)
                                          for l in range(cfg.layers)}
