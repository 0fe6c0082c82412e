"""Shared test configuration.  ``-m gpu`` tests need a CUDA device and the in-tree
``paper_2506_14107_b200/lib/libreusevit.so``; everything else runs on CPU."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


if os.environ.get("RV_LIB"):   # experiment builds (build.build_variant) under the same tests
    from paper_2506_14107_b200 import _lib as _rv_lib
    _rv_lib.load_library(os.environ["RV_LIB"])


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU")


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
