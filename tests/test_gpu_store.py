"""Embedding store on the GPU (paper §6.1) vs the fp64 oracle
(oracle/store_ref.py): fp16 conversion bit-exact (RNE), cosine scores within fp32 rounding,
top-k order equal wherever the oracle's consecutive scores are separated by more than that
rounding, insertion-order invariance, and the compute-on-miss workflow on real embeddings."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda_ok():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return True


def _check_topk(idx_g, sc_g, E16, Q, k):
    idx_r, sc_r = oracle.topk_cosine(E16, Q, k)
    sc_all = oracle.cosine_scores(E16, Q)
    for i in range(Q.shape[0]):
        for t in range(k):
            if idx_r[i, t] < 0:
                assert idx_g[i, t] == -1
                continue
            # the GPU's pick has (within fp32 rounding) the oracle's score at this rank
            assert abs(sc_g[i, t] - sc_r[i, t]) < 2e-6
            assert abs(sc_all[i, idx_g[i, t]] - sc_r[i, t]) < 2e-6
            gap_prev = sc_r[i, t - 1] - sc_r[i, t] if t > 0 else np.inf
            gap_next = sc_r[i, t] - sc_r[i, t + 1] if t + 1 < k and idx_r[i, t + 1] >= 0 else np.inf
            if min(gap_prev, gap_next) > 4e-6:
                assert idx_g[i, t] == idx_r[i, t]


def test_store_topk_vs_oracle(cuda_ok):
    from paper_2506_14107_b200 import EmbeddingStore
    rng = np.random.default_rng(11)
    n, D, k = 3000, 1024, 10
    Z = rng.standard_normal((n, D)).astype(np.float32)
    Z[17] = 0.0                                            # zero norm: cosine 0
    perm = rng.permutation(n)
    store = EmbeddingStore(D, capacity=64)                  # grows
    for chunk in np.array_split(perm, 7):                   # shuffled insertion order
        store.put("v0", chunk.tolist(), torch.from_numpy(Z[chunk]).cuda())
    assert len(store) == n and store.key(5) == ("v0", 5)
    E16 = store.emb[:n].cpu().numpy()
    assert np.array_equal(E16.view(np.uint16), oracle.to_fp16(Z).view(np.uint16))   # RNE, bit-exact
    Q = rng.standard_normal((6, D)).astype(np.float32)
    Q[0] = Z[1234]                                         # S:529 stored vector -> first, score ~1
    Q[1] = 0.0
    idx, sc = store.query(torch.from_numpy(Q).cuda(), k)
    idx, sc = idx.cpu().numpy(), sc.cpu().numpy()
    assert idx[0, 0] == 1234 and abs(sc[0, 0] - 1.0) < 1e-3
    assert list(idx[1]) == list(range(k)) and np.all(sc[1] == 0)
    _check_topk(idx, sc, E16, Q, k)
    # insertion-order invariance: same store content, different order -> same answer
    store2 = EmbeddingStore(D, capacity=n)
    store2.put("v0", list(range(n)), torch.from_numpy(Z).cuda())
    idx2, sc2 = store2.query(torch.from_numpy(Q).cuda(), k)
    assert np.array_equal(idx, idx2.cpu().numpy()) and np.array_equal(sc, sc2.cpu().numpy())
    # k > n returns every record then -1
    small = EmbeddingStore(D, capacity=4)
    small.put("v1", [0, 1, 2], torch.from_numpy(Z[:3]).cuda())
    i3, s3 = small.query(torch.from_numpy(Q[2:3]).cuda(), 5)
    assert sorted(i3[0, :3].cpu().tolist()) == [0, 1, 2] and i3[0, 3:].cpu().tolist() == [-1, -1]


def test_store_compute_on_miss_workflow(cuda_ok):
    """cached embeddings are returned when present, otherwise the frames are embedded
    (rv_embed) and stored; a query with a frame's own embedding retrieves that frame."""
    from paper_2506_14107_b200 import EmbeddingStore, ReuseViT
    cfg = synth.CONFIGS["b16"]
    m = ReuseViT(cfg, 0)
    m.load_vit(synth.pack_vit(cfg, synth.make_vit(cfg)))
    m.load_gates(synth.pack_gates(cfg, synth.make_gates(cfg)))
    x, c = synth.make_video(cfg, 24, 0.5, seed=41)
    store = EmbeddingStore(cfg.dim, capacity=8)
    assert store.get("clip", 3) is None                     # miss -> compute
    Z, _, _, _ = m.embed(torch.from_numpy(x).cuda(), torch.from_numpy(c).cuda())
    store.put("clip", range(24), Z)
    hit = store.get("clip", 3)
    assert hit is not None and torch.equal(hit, Z[3].half())
    idx, sc = store.query(Z[7:8], 3)
    assert store.key(idx[0, 0].item()) == ("clip", 7) and sc[0, 0].item() > 0.999
