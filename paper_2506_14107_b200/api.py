"""Python binding of libreusevit (argument marshalling only).

    m = ReuseViT(cfg, device=0)            # cfg: any object with layers, dim, heads, patch,
    m.load_vit(vit_blob); m.load_gates(g)  #      img, ffn, hidden_r, hidden_g attributes
    Z, masks, scores, stats = m.embed(patches, codec)          # plan_gop(n, 20) by default

``patches`` [n, N, pp] / ``codec`` [n, N] may be CUDA torch tensors (device path, results
are CUDA tensors in stream order) or host arrays (numpy / CPU torch; the library copies
them host->device and results back).  Torch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from . import _lib
from ._lib import (RV_ATTN_SYNC, RV_CHAIN, RV_DENSE, RV_DEVICE_PTRS, RV_FORCE_MASKS, RV_KEEP_ALL_CACHE,
                   RV_NO_COMPACTION, RV_NO_GRAPH, RV_PROFILE, RV_SERIAL_WAVES, RV_WAVE_FRAME, RV_X_BF16, RV_RESTORE_GEMMS, RvConfig, RvKernelProf, RvPlan, RvStats,
                   check, load_library)

__all__ = ["ReuseViT", "plan_gop", "plan_check", "vit_blob_floats", "gate_blob_floats"]


def _cfg(cfg) -> RvConfig:
    return RvConfig(*(int(getattr(cfg, k)) for k in ("layers", "dim", "heads", "patch", "img", "ffn",
                                                     "hidden_r", "hidden_g")))


def _plan_struct(plan: dict):
    n = len(plan["type"])
    arrs = {
        "type": np.ascontiguousarray(plan["type"], dtype=np.int8),
        "past": np.ascontiguousarray(plan["past"], dtype=np.int32),
        "future": np.ascontiguousarray(plan["future"], dtype=np.int32),
        "order": np.ascontiguousarray(plan["order"], dtype=np.int32),
    }
    st = RvPlan(n, arrs["type"].ctypes.data_as(ctypes.POINTER(ctypes.c_int8)),
                arrs["past"].ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                arrs["future"].ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                arrs["order"].ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    return st, arrs   # keep arrs alive while st is used


def plan_gop(n: int, refresh: int = 20, reorder: bool = True) -> dict:
    """rv_plan_gop: display-indexed type/past/future and the computation order."""
    lib = load_library()
    out = {"type": np.zeros(n, np.int8), "past": np.zeros(n, np.int32), "future": np.zeros(n, np.int32),
           "order": np.zeros(n, np.int32)}
    st, keep = _plan_struct(out)
    check(lib, lib.rv_plan_gop(n, refresh, 1 if reorder else 0, ctypes.byref(st)))
    return keep


def plan_check(plan: dict) -> None:
    lib = load_library()
    st, _keep = _plan_struct(plan)
    check(lib, lib.rv_plan_check(ctypes.byref(st)))


def vit_blob_floats(cfg) -> int:
    c = _cfg(cfg)
    return int(load_library().rv_vit_blob_floats(ctypes.byref(c)))


def gate_blob_floats(cfg) -> int:
    c = _cfg(cfg)
    return int(load_library().rv_gate_blob_floats(ctypes.byref(c)))


def _ptr(x):
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return ctypes.c_void_p(x.data_ptr())
    return ctypes.c_void_p(x.ctypes.data)


class ReuseViT:
    """One libreusevit context on one CUDA device."""

    def __init__(self, cfg, device: int = 0):
        self.lib = load_library()
        self.cfg = cfg
        self.c = _cfg(cfg)
        self.N = (cfg.img // cfg.patch) ** 2
        self.T = self.N + 1
        self.pp = 3 * cfg.patch * cfg.patch
        self.device = device
        h = ctypes.c_void_p()
        check(self.lib, self.lib.rv_create(ctypes.byref(self.c), device, ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.rv_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ weights
    def load_vit(self, blob: np.ndarray):
        b = np.ascontiguousarray(blob, dtype=np.float32)
        check(self.lib, self.lib.rv_load_vit(self.h, b.ctypes.data_as(_lib.P_f32), b.size), self.h)

    def load_gates(self, blob: np.ndarray):
        b = np.ascontiguousarray(blob, dtype=np.float32)
        check(self.lib, self.lib.rv_load_gates(self.h, b.ctypes.data_as(_lib.P_f32), b.size), self.h)

    # ------------------------------------------------------------------ embed
    def embed_async(self, patches, codec, plan: Optional[dict] = None, *, refresh: int = 20,
                    reorder: bool = True, dense: bool = False, force_masks=None, want_masks: bool = True,
                    want_scores: bool = False, stream=None, graph: bool = True, out=None,
                    profile: bool = False, attn_tc: bool = True,
                    per_frame_waves: bool = False, chain: bool = False, no_compaction: bool = False,
                    keep_all_cache: bool = False, serial_waves: bool = False, x_bf16: bool = False,
                    restore_gemms: bool = False):
        """Enqueue one embed; returns a handle for ``wait``.  ``x_bf16``: experimental bf16
        residual stream (RV_X_BF16).  ``restore_gemms``: diagnostic, restoration as two GEMMs
        (RV_RESTORE_GEMMS) instead of the fused kernel.  ``out`` optionally supplies the
        output buffers (emb, masks, scores) to reuse across calls (same pointers -> the
        cached CUDA graph is replayed)."""
        import torch
        n = patches.shape[0]
        if plan is None:
            plan = plan_gop(n, refresh, reorder)
        st, keep = _plan_struct(plan)
        L, N, D = self.cfg.layers, self.N, self.cfg.dim
        device_path = isinstance(patches, torch.Tensor) and patches.is_cuda
        flags = ((RV_DENSE if dense else 0) | (0 if graph else RV_NO_GRAPH) | (RV_PROFILE if profile else 0)
                 | (0 if attn_tc else RV_ATTN_SYNC)
                 | (RV_WAVE_FRAME if per_frame_waves else 0) | (RV_CHAIN if chain else 0)
                 | (RV_NO_COMPACTION if no_compaction else 0) | (RV_KEEP_ALL_CACHE if keep_all_cache else 0)
                 | (RV_SERIAL_WAVES if serial_waves else 0) | (RV_X_BF16 if x_bf16 else 0)
                 | (RV_RESTORE_GEMMS if restore_gemms else 0))
        if force_masks is not None:
            flags |= RV_FORCE_MASKS
        if device_path:
            flags |= RV_DEVICE_PTRS
            dev = patches.device
            if not patches.is_contiguous() or patches.dtype != torch.float32:
                raise ValueError("patches must be contiguous float32")
            if not (isinstance(codec, torch.Tensor) and codec.is_cuda and codec.dtype == torch.float32
                    and codec.is_contiguous()):
                raise ValueError("codec must be a contiguous float32 CUDA tensor on the device path")
            if out is None:
                emb = torch.empty((n, D), dtype=torch.float32, device=dev)
                masks = torch.empty((n, L, N), dtype=torch.uint8, device=dev) if (want_masks or force_masks is not None) else None
                scores = torch.empty((n, L, N), dtype=torch.float32, device=dev) if want_scores else None
            else:
                emb, masks, scores = out
            if force_masks is not None:
                masks = force_masks.to(device=dev, dtype=torch.uint8).contiguous()
            if stream is None:
                stream = torch.cuda.current_stream(dev)
            sptr = ctypes.c_void_p(stream.cuda_stream)
        else:
            patches = np.ascontiguousarray(patches.numpy() if hasattr(patches, "numpy") else patches, dtype=np.float32)
            codec = np.ascontiguousarray(codec.numpy() if hasattr(codec, "numpy") else codec, dtype=np.float32)
            if out is None:
                emb = np.empty((n, D), np.float32)
                masks = np.empty((n, L, N), np.uint8) if (want_masks or force_masks is not None) else None
                scores = np.empty((n, L, N), np.float32) if want_scores else None
            else:
                emb, masks, scores = out
            if force_masks is not None:
                masks = np.ascontiguousarray(force_masks, dtype=np.uint8)
            sptr = ctypes.c_void_p(stream.cuda_stream) if stream is not None else None
        check(self.lib, self.lib.rv_embed(self.h, _ptr(patches), _ptr(codec), ctypes.byref(st), flags, sptr,
                                          _ptr(emb), _ptr(masks), _ptr(scores)), self.h)
        return {"emb": emb, "masks": masks, "scores": scores, "keep": (keep, patches, codec)}

    def wait(self, handle=None) -> dict:
        s = RvStats()
        check(self.lib, self.lib.rv_wait(self.h, ctypes.byref(s)), self.h)
        L = self.cfg.layers
        return {"reuse_nonI": s.reuse_nonI, "reuse_all": s.reuse_all, "flops_exec": s.flops_exec,
                "flops_dense": s.flops_dense, "bytes_alg": s.bytes_alg,
                "peak_cache_bytes": int(s.peak_cache_bytes), "keepall_cache_bytes": int(s.keepall_cache_bytes),
                "ms_total": s.ms_total, "ms_compute": s.ms_compute, "n_levels": s.n_levels,
                "n_launches": s.n_launches, "reuse_by_layer": list(s.reuse_by_layer[:L]),
                "device_bytes": int(s.device_bytes), "wave_ring": int(s.wave_ring)}

    def wave_counts(self) -> dict:
        """Level-wave structure of the last embed (after ``wait``): frames per wave and the
        per-layer recomputed / reused row counts."""
        k = self.lib.rv_wave_counts(self.h, None, None, 0)
        if k < 0:
            check(self.lib, k, self.h)
        frames = np.zeros(k, np.int32)
        counts = np.zeros((self.cfg.layers, k, 2), np.int32)
        check_k = self.lib.rv_wave_counts(self.h, frames.ctypes.data_as(ctypes.c_void_p),
                                          counts.ctypes.data_as(ctypes.c_void_p), k)
        if check_k < 0:
            check(self.lib, check_k, self.h)
        return {"frames": frames, "M_C": counts[:, :, 0], "M_R": counts[:, :, 1]}

    def profile(self) -> list:
        """Per-kernel-class records of the last ``profile=True`` embed (after ``wait``)."""
        buf = (RvKernelProf * 32)()
        k = self.lib.rv_profile(self.h, buf, 32)
        if k < 0:
            check(self.lib, k, self.h)
        return [{"name": buf[i].name.decode(), "launches": buf[i].launches, "ms": buf[i].ms,
                 "flops": buf[i].flops, "bytes": buf[i].bytes} for i in range(k)]

    def embed(self, patches, codec, plan: Optional[dict] = None, **kw):
        """Synchronous embed: returns (Z [n,D], masks [n,L,N] or None, scores or None, stats)."""
        hnd = self.embed_async(patches, codec, plan, **kw)
        stats = self.wait(hnd)
        return hnd["emb"], hnd["masks"], hnd["scores"], stats

    # ------------------------------------------------------------------ stages (tests)
    def stage_score(self, layer, X, wdesc, t, codec, force, masks, scores, wmask, wprov, cntR, stream):
        check(self.lib, self.lib.rv_stage_score(self.h, layer, _ptr(X), wdesc.shape[0], _ptr(wdesc), _ptr(t),
                                                _ptr(codec), _ptr(force), _ptr(masks), _ptr(scores), _ptr(wmask),
                                                _ptr(wprov), _ptr(cntR), ctypes.c_void_p(stream.cuda_stream)), self.h)

    def stage_compact(self, wdesc, wmask, wprov, cntR, idxC, idxR, provrow, qoff, counts, stream):
        check(self.lib, self.lib.rv_stage_compact(self.h, wdesc.shape[0], _ptr(wdesc), _ptr(wmask), _ptr(wprov),
                                                  _ptr(cntR), _ptr(idxC), _ptr(idxR), _ptr(provrow), _ptr(qoff),
                                                  _ptr(counts), ctypes.c_void_p(stream.cuda_stream)), self.h)

    def stage_gemm(self, A, B, bias=None, act=0, out=None, out_bf16=False, stream=None):
        import torch
        M, K = A.shape
        N = B.shape[0]
        if out is None:
            out = torch.empty((M, N), dtype=torch.bfloat16 if out_bf16 else torch.float32, device=A.device)
        stream = stream or torch.cuda.current_stream(A.device)
        check(self.lib, self.lib.rv_stage_gemm(self.h, M, N, K, _ptr(A), _ptr(B), _ptr(bias), act, _ptr(out),
                                               1 if out_bf16 else 0, ctypes.c_void_p(stream.cuda_stream)), self.h)
        return out

    def stage_gemm_rows(self, A, B, out, bias=None, act=0, resid=None, resid_rows=None, out_rows=None,
                        stream=None):
        """out[out_rows[m]] = act(A[m] B^T + bias) + resid[resid_rows[m]] (row-mapped epilogue)."""
        import torch
        M, K = A.shape
        N = B.shape[0]
        stream = stream or torch.cuda.current_stream(A.device)
        check(self.lib, self.lib.rv_stage_gemm_rows(
            self.h, M, N, K, _ptr(A), _ptr(B), _ptr(bias), act, _ptr(resid), _ptr(resid_rows),
            resid.shape[1] if resid is not None else 0, _ptr(out), _ptr(out_rows), out.shape[1],
            1 if out.dtype == torch.bfloat16 else 0, ctypes.c_void_p(stream.cuda_stream)), self.h)
        return out

    def stage_attention(self, wdesc, qoff, q, KV, out, pcls, stream, use_tc=False, kvsrc=None):
        """use_tc: False/0 mma.sync, True/1 tcgen05 (persistent kernel where T <= 257), 2 general tcgen05."""
        check(self.lib, self.lib.rv_stage_attention(self.h, wdesc.shape[0], _ptr(wdesc), _ptr(qoff), _ptr(q),
                                                    q.shape[0], _ptr(KV), _ptr(kvsrc), _ptr(out), _ptr(pcls),
                                                    int(use_tc),
                                                    ctypes.c_void_p(stream.cuda_stream)), self.h)
