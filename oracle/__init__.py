"""ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (NumPy, float64) of the ReuseViT
forward pass of Deja Vu (arxiv 2506.14107, §3, Eq. 1-10) written from the
paper.  It exists to prove the CUDA path right.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import it.  It shares no code with ``paper_2506_14107_b200/`` (the product)
and imports nothing from it; the only shared module is ``synth`` (seeded inputs).

Every function cites the passage it follows.  Readings of ambiguous passages are the
ones listed in DESIGN.md §3.

Pins (tests/test_oracle_pins.py, ``-m "not gpu"``) tie it to things other than itself:
torch-fp64 library ViT for the dense path, pure-Python brute force on tiny frames,
the SPEC/SURVEY worked examples under tests/golden/, and closed-form invariants
(all-reuse => Z_f = Z_ref, duplicate frame, forced logits, Delta=0 restoration).
Functions without such a pin say "parity unpinned" in their docstring.
"""
from .reusevit_ref import (  # noqa: F401
    FTYPES, layer_norm, quick_gelu, cosine, plan_gop, plan_levels, patch_embed,
    similarity, decision_mlp, restoration_mlp, reuse_embed, dense_embed,
    compaction_indices, flops_per_frame, reuse_rates,
)
from .store_ref import to_fp16, cosine_scores, topk_cosine, storage_bytes_per_second  # noqa: F401
from .chain_ref import reuse_embed_chain  # noqa: F401
from .train_ref import (  # noqa: F401
    GROUP_PATTERN, group_plan, gumbel_soft_mask, soft_forward, group_losses, gates_to_torch, batch_loss,
    loss_and_grads, adam_step, temperature,
)
