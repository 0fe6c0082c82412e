"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Embedding-store query of the paper's workflow (§6.1; SURVEY §8(f) NEXT-4;
SPEC embed-store S:501-549): per-frame embeddings stored as fp16 ("1024-dimensional FP16
embeddings at ~2KB each") and retrieved by brute-force cosine similarity, top-k descending,
ties broken by (video_id, frame_index), i.e. by record order in a key-sorted store.
Pinned in tests/test_oracle_pins.py by a pure-Python exhaustive scan, the S:529-531 examples
(stored vector first with score 1; orthogonal query -> 0 with index tie order) and the P:553-554
storage arithmetic.
"""
from __future__ import annotations

import numpy as np


def to_fp16(Z: np.ndarray) -> np.ndarray:
    """Store format: IEEE half, round to nearest even (numpy's float16 cast)."""
    return np.asarray(Z, dtype=np.float64).astype(np.float16)


def cosine_scores(E16: np.ndarray, Q: np.ndarray) -> np.ndarray:
    """cos(q, e) = q.e / (|q| |e|) in float64 on the stored fp16 values; 0 for a zero norm
    (S:76).  Returns [nq, n]."""
    E = np.asarray(E16, dtype=np.float64)
    Qd = np.atleast_2d(np.asarray(Q, dtype=np.float64))
    dots = Qd @ E.T
    den = np.linalg.norm(Qd, axis=1)[:, None] * np.linalg.norm(E, axis=1)[None, :]
    out = np.zeros_like(dots)
    np.divide(dots, den, out=out, where=den > 0)
    return out


def topk_cosine(E16: np.ndarray, Q: np.ndarray, k: int):
    """Top-k records per query: (idx [nq, k] int64, score [nq, k] float64), descending cosine,
    equal scores by lower record index; entries past the store size are -1 / -inf (S:528
    "k > count -> return all")."""
    S = cosine_scores(E16, Q)
    nq, n = S.shape
    idx = -np.ones((nq, k), np.int64)
    sc = np.full((nq, k), -np.inf)
    for i in range(nq):
        order = np.lexsort((np.arange(n), -S[i]))     # primary: score desc; secondary: index asc
        m = min(k, n)
        idx[i, :m] = order[:m]
        sc[i, :m] = S[i, order[:m]]
    return idx, sc


def storage_bytes_per_second(dim: int = 1024, fps: float = 2.0, bytes_per_value: int = 2) -> float:
    """fp16 embeddings of `dim` values at `fps` frames per second."""
    return dim * bytes_per_value * fps
