"""CPU-side checks of libreusevit.so (no GPU needed): the library loads, exports every symbol
the public headers declare, its host-only plan logic matches the oracle's plan (which is pinned
to SPEC.md's examples), and its error paths behave (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2506_14107_b200 import build as b
    b.build()
    from paper_2506_14107_b200 import _lib
    return _lib.load_library()


def _declared_symbols():
    names = set()
    for h in sorted(f for f in os.listdir(os.path.join(ROOT, "include")) if f.endswith(".h")):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(rv_[a-z_]+)\s*\(", src))
    return names


def test_exports_every_declared_symbol(lib):
    declared = _declared_symbols()
    assert {"rv_create", "rv_embed", "rv_wait", "rv_stage_gemm", "rv_trainer_step"} <= declared
    for name in declared:
        assert hasattr(lib, name), name


def test_sm100a_code_in_library(lib):
    """The library carries sm_100a tcgen05 code (SASS UTCHMMA / UTMALDG / LDTM)."""
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    from paper_2506_14107_b200._lib import LIB_PATH
    sass = subprocess.run([cuobjdump, "-sass", LIB_PATH], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnem in sass, mnem
    assert "sm_100a" in subprocess.run([cuobjdump, "-lelf", LIB_PATH], capture_output=True, text=True).stdout


@pytest.mark.parametrize("reorder", [True, False])
def test_plan_matches_oracle(lib, reorder):
    from paper_2506_14107_b200 import plan_gop
    for n in list(range(1, 80)) + [256, 901, 7200]:
        for refresh in (20, 8):
            a = plan_gop(n, refresh, reorder)
            b = oracle.plan_gop(n, refresh, reorder)
            for k in ("type", "past", "future", "order"):
                assert np.array_equal(a[k], b[k]), (n, refresh, k)


def test_plan_check_errors(lib):
    from paper_2506_14107_b200 import ReuseViTError, plan_check
    good = oracle.plan_gop(9)
    plan_check(good)
    bad = {k: v.copy() for k, v in good.items()}
    bad["order"] = bad["order"][::-1].copy()          # reference after dependent
    with pytest.raises(ReuseViTError) as e:
        plan_check(bad)
    assert e.value.status == -3
    bad = {k: v.copy() for k, v in good.items()}
    bad["type"][3] = 7
    with pytest.raises(ReuseViTError):
        plan_check(bad)
    bad = {k: v.copy() for k, v in good.items()}
    bad["past"][0] = 2                                  # I-frame with a reference
    with pytest.raises(ReuseViTError):
        plan_check(bad)
    bad = {k: v.copy() for k, v in good.items()}
    bad["order"][1] = bad["order"][0]                  # not a permutation
    with pytest.raises(ReuseViTError):
        plan_check(bad)


def test_blob_sizes(lib):
    from paper_2506_14107_b200 import gate_blob_floats, vit_blob_floats
    for name in ("tiny", "b16", "l14"):
        cfg = synth.CONFIGS[name]
        assert vit_blob_floats(cfg) == sum(int(np.prod(s)) for _, s in synth.vit_array_order(cfg))
        assert gate_blob_floats(cfg) == sum(int(np.prod(s)) for _, s in synth.gate_array_order(cfg))


def test_create_errors_without_gpu(lib):
    """Invalid config -> RV_ECONFIG; on a host without an sm_100 device -> RV_ECUDA (the
    library has no CPU fallback)."""
    import torch
    from paper_2506_14107_b200 import ReuseViT, ReuseViTError
    bad = synth.ViTConfig(layers=2, dim=96, heads=5, patch=16, img=64, ffn=256)
    with pytest.raises(ReuseViTError) as e:
        ReuseViT(bad)
    assert e.value.status == -1
    if not torch.cuda.is_available():
        with pytest.raises(ReuseViTError) as e:
            ReuseViT(synth.CONFIGS["tiny"])
        assert e.value.status == -6
