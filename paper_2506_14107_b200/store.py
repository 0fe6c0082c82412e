"""Embedding store on the device (paper §6.1): per-frame fp16
embeddings keyed by (video id, frame index), brute-force cosine top-k queries, compute on a
miss.  Conversion and query run in libreusevit (rv_f32_to_f16, rv_topk_cosine); this class only
keeps the device buffer and the host-side index (argument marshalling).

    store = EmbeddingStore(dim=1024, capacity=7200)
    store.put("video0", frames, Z)                       # Z: fp32 [n, D] CUDA tensor
    idx, score = store.query(q, k=5)                     # q: fp32 [nq, D] CUDA tensor
    store.key(idx[0, 0])                                 # -> ("video0", frame index)
Records are kept in (video id, frame index) order, so the library's tie order (lower record
index first) is SPEC's (video_id, frame_index) order and results do not depend on insertion
order.
"""
from __future__ import annotations

import bisect
import ctypes

from . import _lib
from ._lib import check


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


class EmbeddingStore:
    def __init__(self, dim: int, capacity: int = 1024, device: int = 0):
        import torch
        self.dim, self.device = dim, torch.device("cuda", device)
        self.lib = _lib.load_library()
        self.keys: list = []                     # sorted (video_id, frame_index)
        self.emb = torch.empty((max(capacity, 1), dim), dtype=torch.float16, device=self.device)

    def __len__(self):
        return len(self.keys)

    @staticmethod
    def bytes_per_frame(dim: int) -> int:
        """fp16 payload per stored frame (2 D bytes: ~2 KB at D = 1024)."""
        return 2 * dim

    def get(self, video_id: str, frame: int):
        """fp16 embedding of (video_id, frame) or None (a miss: the caller embeds the frame)."""
        i = bisect.bisect_left(self.keys, (video_id, frame))
        if i < len(self.keys) and self.keys[i] == (video_id, frame):
            return self.emb[i]
        return None

    def put(self, video_id: str, frames, Z):
        """Insert fp32 embeddings Z [n, D] (CUDA) of the given frame indices (overwrites)."""
        import torch
        assert Z.dim() == 2 and Z.shape[1] == self.dim and Z.is_cuda and Z.dtype == torch.float32
        Z = Z.contiguous()
        z16 = torch.empty(Z.shape, dtype=torch.float16, device=self.device)
        stream = torch.cuda.current_stream(self.device)
        check(self.lib, self.lib.rv_f32_to_f16(_ptr(Z), _ptr(z16), Z.numel(), ctypes.c_void_p(stream.cuda_stream)))
        for row, f in enumerate(list(frames)):
            key = (video_id, int(f))
            i = bisect.bisect_left(self.keys, key)
            if i < len(self.keys) and self.keys[i] == key:
                self.emb[i] = z16[row]
                continue
            if len(self.keys) == self.emb.shape[0]:
                grown = torch.empty((2 * self.emb.shape[0], self.dim), dtype=torch.float16, device=self.device)
                grown[:len(self.keys)] = self.emb[:len(self.keys)]
                self.emb = grown
            n = len(self.keys)
            if i < n:
                self.emb[i + 1:n + 1] = self.emb[i:n].clone()
            self.emb[i] = z16[row]
            self.keys.insert(i, key)

    def query(self, q, k: int):
        """Top-k records by cosine similarity for each query row: (idx [nq, k] int32 record
        indices (-1 past the store size), score [nq, k] fp32), descending, ties -> lower index."""
        import torch
        if q.dim() == 1:
            q = q[None]
        assert q.is_cuda and q.dtype == torch.float32 and q.shape[1] == self.dim and len(self.keys) > 0
        q = q.contiguous()
        n, nq = len(self.keys), q.shape[0]
        tmp = torch.empty((nq, n), dtype=torch.float32, device=self.device)
        idx = torch.empty((nq, k), dtype=torch.int32, device=self.device)
        score = torch.empty((nq, k), dtype=torch.float32, device=self.device)
        stream = torch.cuda.current_stream(self.device)
        check(self.lib, self.lib.rv_topk_cosine(_ptr(self.emb), n, self.dim, _ptr(q), nq, k, _ptr(tmp), _ptr(idx),
                                                _ptr(score), ctypes.c_void_p(stream.cuda_stream)))
        return idx, score

    def key(self, record: int):
        return self.keys[int(record)]
