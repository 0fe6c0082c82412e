"""Python binding of libreusevit's gate trainer (include/reusevit_train.h; SURVEY §8(f) NEXT-2,
PAPER.md §4): argument marshalling only — the soft-gated forward (Eq. 11-12), the loss
(Eq. 13-15), the reverse pass and Adam all run in the library's CUDA kernels.

    tr = GateTrainer(cfg, vit_blob, gate_blob, group_plan, groups=B, alpha=2.0, r_target=0.5)
    log = tr.step(patches, codec, gumbel, tau)     # CUDA tensors [B,G,N,pp], [B,G,N], [B,G,L,N,2]
    m.load_gates(tr.gates())                        # trained RVG1 blob -> the inference path
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import RV_TRAIN_DENSE, RV_TRAIN_FORCE, RvTrainConfig, RvTrainLog, load_library
from .api import _cfg

__all__ = ["GateTrainer"]


def _dptr(t, name):
    import torch
    if t is None:
        return None
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous float32 CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


class GateTrainer:
    """Trains the decision + restoration layers of a frozen ViT on groups of frames."""

    def __init__(self, cfg, vit_blob, gate_blob, plan: dict, groups: int, device: int = 0, alpha: float = 2.0,
                 r_target: float = 0.5, lr: float = 1e-3, betas=(0.9, 0.999), eps: float = 1e-8):
        self.lib = load_library()
        self.cfg = cfg
        self.G = len(plan["type"])
        self.B = groups
        self.N = (cfg.img // cfg.patch) ** 2
        self.device = device
        self._plan = {k: np.ascontiguousarray(plan[k], dtype=np.int8 if k == "type" else np.int32)
                      for k in ("type", "past", "future", "order")}
        p = self._plan
        tc = RvTrainConfig(groups, self.G, p["type"].ctypes.data_as(ctypes.POINTER(ctypes.c_int8)),
                           p["past"].ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                           p["future"].ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                           p["order"].ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                           alpha, r_target, lr, betas[0], betas[1], eps)
        vb = np.ascontiguousarray(vit_blob, dtype=np.float32)
        gb = np.ascontiguousarray(gate_blob, dtype=np.float32)
        self.n_gate = gb.size
        c = _cfg(cfg)
        h = ctypes.c_void_p()
        self._check(self.lib.rv_trainer_create(ctypes.byref(c), device, vb.ctypes.data_as(_lib.P_f32), vb.size,
                                               gb.ctypes.data_as(_lib.P_f32), gb.size, ctypes.byref(tc),
                                               ctypes.byref(h)), None)
        self.h = h

    def _check(self, st, h):
        if st != 0:
            msg = self.lib.rv_trainer_last_error(h)
            raise _lib.ReuseViTError(st, msg.decode() if msg else "")

    def close(self):
        if getattr(self, "h", None):
            self.lib.rv_trainer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _stream(self, stream):
        import torch
        s = stream or torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(s.cuda_stream)

    def forward(self, patches, codec, gumbel, tau: float, dense: bool = False, force=None, stream=None):
        """Soft forward of B groups: returns (Z [B,G,D], M [B,G,L,N], d [B,G,L,N]) CUDA tensors."""
        import torch
        B = patches.shape[0]
        L, D, N = self.cfg.layers, self.cfg.dim, self.N
        dev = patches.device
        Z = torch.empty((B, self.G, D), dtype=torch.float32, device=dev)
        M = torch.empty((B, self.G, L, N), dtype=torch.float32, device=dev)
        d = torch.empty((B, self.G, L, N), dtype=torch.float32, device=dev)
        flags = (RV_TRAIN_DENSE if dense else 0) | (RV_TRAIN_FORCE if force is not None else 0)
        self._check(self.lib.rv_trainer_forward(self.h, _dptr(patches, "patches"), _dptr(codec, "codec"),
                                                _dptr(gumbel, "gumbel"), B, float(tau), flags,
                                                _dptr(force, "force"), _dptr(Z, "Z"), _dptr(M, "M"), _dptr(d, "d"),
                                                self._stream(stream)), self.h)
        return Z, M, d

    @staticmethod
    def _log(lg):
        return {"l_sim": lg.l_sim, "l_reuse": lg.l_reuse, "l_total": lg.l_total, "cos_mean": lg.cos_mean,
                "step": lg.step}

    def loss_grad(self, patches, codec, gumbel, tau: float, stream=None):
        """Eq. 15 batch loss and its gradient w.r.t. the RVG1 gate blob: (log, grad CUDA tensor)."""
        import torch
        g = torch.empty(self.n_gate, dtype=torch.float32, device=patches.device)
        lg = RvTrainLog()
        self._check(self.lib.rv_trainer_loss_grad(self.h, _dptr(patches, "patches"), _dptr(codec, "codec"),
                                                  _dptr(gumbel, "gumbel"), patches.shape[0], float(tau),
                                                  _dptr(g, "grad"), ctypes.byref(lg), self._stream(stream)), self.h)
        return self._log(lg), g

    def step(self, patches, codec, gumbel, tau: float, stream=None) -> dict:
        lg = RvTrainLog()
        self._check(self.lib.rv_trainer_step(self.h, _dptr(patches, "patches"), _dptr(codec, "codec"),
                                             _dptr(gumbel, "gumbel"), patches.shape[0], float(tau), ctypes.byref(lg),
                                             self._stream(stream)), self.h)
        return self._log(lg)

    def gates(self) -> np.ndarray:
        """Current gates as an RVG1 blob (host float32), for ReuseViT.load_gates."""
        out = np.empty(self.n_gate, np.float32)
        self._check(self.lib.rv_trainer_gates(self.h, out.ctypes.data_as(_lib.P_f32)), self.h)
        return out
