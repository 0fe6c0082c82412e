"""paper_2506_14107_b200 — B200-native (sm_100a) ReuseViT hot path of Deja Vu (arxiv 2506.14107).

The product is ``lib/libreusevit.so`` (C-ABI: include/reusevit.h); this package is its thin
ctypes binding.  Build with ``__graft_entry__.build()``.  See DESIGN.md.
"""
from .api import ReuseViT, gate_blob_floats, plan_check, plan_gop, vit_blob_floats  # noqa: F401
from ._lib import ReuseViTError, load_library  # noqa: F401
from .store import EmbeddingStore  # noqa: F401
