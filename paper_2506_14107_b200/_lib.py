"""ctypes declarations of libreusevit.so (include/reusevit.h, include/reusevit_stages.h).

Argument marshalling only: every step of the hot path runs in the library's CUDA kernels.
There is no fallback — if the shared library is missing this raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libreusevit.so")

c_i32, c_u32, c_sz, c_vp = ctypes.c_int32, ctypes.c_uint32, ctypes.c_size_t, ctypes.c_void_p
P_f32 = ctypes.POINTER(ctypes.c_float)

RV_OK = 0
STATUS = {0: "RV_OK", -1: "RV_ECONFIG", -2: "RV_ESHAPE", -3: "RV_EPLAN", -4: "RV_ECACHE",
          -5: "RV_ECONTRACT", -6: "RV_ECUDA", -7: "RV_ENOMEM", -8: "RV_EBUSY"}
RV_DEVICE_PTRS, RV_DENSE, RV_FORCE_MASKS, RV_NO_GRAPH, RV_PROFILE, RV_ATTN_SYNC, RV_WAVE_FRAME, RV_CHAIN = (
    1, 2, 4, 8, 16, 32, 64, 128)
RV_NO_COMPACTION, RV_KEEP_ALL_CACHE, RV_SERIAL_WAVES, RV_X_BF16, RV_RESTORE_GEMMS = 256, 512, 1024, 2048, 4096
RV_I, RV_P, RV_B2, RV_B1 = 0, 1, 2, 3


class RvConfig(ctypes.Structure):
    _fields_ = [(k, c_i32) for k in ("layers", "dim", "heads", "patch", "img", "ffn", "hidden_r", "hidden_g")]


class RvPlan(ctypes.Structure):
    _fields_ = [("n", c_i32), ("type", ctypes.POINTER(ctypes.c_int8)), ("past", ctypes.POINTER(c_i32)),
                ("future", ctypes.POINTER(c_i32)), ("order", ctypes.POINTER(c_i32))]


class RvStats(ctypes.Structure):
    _fields_ = [("reuse_nonI", ctypes.c_double), ("reuse_all", ctypes.c_double),
                ("flops_exec", ctypes.c_double), ("flops_dense", ctypes.c_double),
                ("bytes_alg", ctypes.c_double), ("peak_cache_bytes", ctypes.c_uint64),
                ("keepall_cache_bytes", ctypes.c_uint64), ("ms_total", ctypes.c_float),
                ("ms_compute", ctypes.c_float), ("n_levels", c_i32), ("n_launches", c_i32),
                ("reuse_by_layer", ctypes.c_float * 64), ("device_bytes", ctypes.c_uint64), ("wave_ring", c_i32)]


class RvKernelProf(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 24), ("launches", c_i32), ("ms", ctypes.c_double),
                ("flops", ctypes.c_double), ("bytes", ctypes.c_double)]


class RvTrainConfig(ctypes.Structure):
    _fields_ = [("groups", c_i32), ("group_size", c_i32), ("type", ctypes.POINTER(ctypes.c_int8)),
                ("past", ctypes.POINTER(c_i32)), ("future", ctypes.POINTER(c_i32)), ("order", ctypes.POINTER(c_i32)),
                ("alpha", ctypes.c_float), ("r_target", ctypes.c_float), ("lr", ctypes.c_float),
                ("beta1", ctypes.c_float), ("beta2", ctypes.c_float), ("eps", ctypes.c_float)]


class RvTrainLog(ctypes.Structure):
    _fields_ = [("l_sim", ctypes.c_double), ("l_reuse", ctypes.c_double), ("l_total", ctypes.c_double),
                ("cos_mean", ctypes.c_double), ("step", c_i32)]


RV_TRAIN_DENSE, RV_TRAIN_FORCE = 1, 2


class ReuseViTError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


# (name, restype, argtypes) for every exported symbol the headers declare.
SIGNATURES = {
    "rv_create": (c_i32, [ctypes.POINTER(RvConfig), ctypes.c_int, ctypes.POINTER(c_vp)]),
    "rv_vit_blob_floats": (c_sz, [ctypes.POINTER(RvConfig)]),
    "rv_gate_blob_floats": (c_sz, [ctypes.POINTER(RvConfig)]),
    "rv_load_vit": (c_i32, [c_vp, P_f32, c_sz]),
    "rv_load_gates": (c_i32, [c_vp, P_f32, c_sz]),
    "rv_plan_gop": (c_i32, [c_i32, c_i32, c_i32, ctypes.POINTER(RvPlan)]),
    "rv_plan_check": (c_i32, [ctypes.POINTER(RvPlan)]),
    "rv_embed": (c_i32, [c_vp, c_vp, c_vp, ctypes.POINTER(RvPlan), c_u32, c_vp, c_vp, c_vp, c_vp]),
    "rv_wait": (c_i32, [c_vp, ctypes.POINTER(RvStats)]),
    "rv_profile": (c_i32, [c_vp, ctypes.POINTER(RvKernelProf), c_i32]),
    "rv_last_error": (ctypes.c_char_p, [c_vp]),
    "rv_status_string": (ctypes.c_char_p, [c_i32]),
    "rv_destroy": (None, [c_vp]),
    "rv_stage_score": (c_i32, [c_vp, c_i32, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "rv_stage_compact": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "rv_stage_gemm": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_i32, c_vp, c_i32, c_vp]),
    "rv_stage_gemm_rows": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, ctypes.c_int64,
                                   c_vp, c_vp, ctypes.c_int64, c_i32, c_vp]),
    "rv_stage_attention": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp]),
    "rv_wave_counts": (c_i32, [c_vp, c_vp, c_vp, c_i32]),
    "rv_f32_to_f16": (c_i32, [c_vp, c_vp, ctypes.c_int64, c_vp]),
    "rv_topk_cosine": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp]),
    # gate trainer (include/reusevit_train.h)
    "rv_trainer_create": (c_i32, [ctypes.POINTER(RvConfig), ctypes.c_int, P_f32, c_sz, P_f32, c_sz,
                                  ctypes.POINTER(RvTrainConfig), ctypes.POINTER(c_vp)]),
    "rv_trainer_forward": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i32, ctypes.c_float, c_u32, c_vp, c_vp, c_vp, c_vp,
                                   c_vp]),
    "rv_trainer_loss_grad": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i32, ctypes.c_float, c_vp, ctypes.POINTER(RvTrainLog),
                                     c_vp]),
    "rv_trainer_step": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i32, ctypes.c_float, ctypes.POINTER(RvTrainLog), c_vp]),
    "rv_trainer_gates": (c_i32, [c_vp, P_f32]),
    "rv_trainer_last_error": (ctypes.c_char_p, [c_vp]),
    "rv_trainer_destroy": (None, [c_vp]),
}

_LIB = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the in-tree libreusevit.so (built by __graft_entry__.build()).  Raises if absent:
    the product path has no CPU or library fallback."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def check(lib, status: int, ctx=None):
    if status != RV_OK:
        msg = lib.rv_last_error(ctx)
        raise ReuseViTError(status, msg.decode() if msg else "")
