"""The a15 collective on real hardware: an NCCL process group (world size 1 -- gpurun and the
round-end tiers have one GPU; NCCL refuses two ranks on one device) runs the same
``gather_rows`` / ``max_over_ranks`` code the multi-GPU bench uses, over ``ReuseViT`` outputs on
cuda:0.  The gathered embeddings and masks must equal the embed's own bitwise.  World sizes
2-3 of the same functions run on gloo in tests/test_dist_cpu.py."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, sys.argv[1])
import synth
from paper_2506_14107_b200 import ReuseViT
from paper_2506_14107_b200.dist import embed_sharded, gather_rows, max_over_ranks, shard_frames
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
assert dist.get_backend() == "nccl"
cfg = synth.CONFIGS["b16"]
m = ReuseViT(cfg, 0)
m.load_vit(synth.pack_vit(cfg, synth.make_vit(cfg)))
m.load_gates(synth.pack_gates(cfg, synth.make_gates(cfg)))
x, c = synth.make_video(cfg, 45, 0.2, seed=77)
x, c = torch.from_numpy(x).cuda(), torch.from_numpy(c).cuda()
Z, M, _, _ = m.embed(x, c)
Zs, Ms = embed_sharded(m, x, c)
f0, n_own, n_loc = shard_frames(45, 20, 0, 1)
Zg, Mg = gather_rows([Z, M.view(45, -1)], [n_own])      # NCCL all_gather_into_tensor
torch.cuda.synchronize()
assert Zg.is_cuda and torch.equal(Zg, Z) and torch.equal(Mg.view_as(M), M)
assert torch.equal(Zs, Z) and torch.equal(Ms, M)
assert max_over_ranks(3.5) == 3.5
t = torch.tensor([2.0], device="cuda")
dist.all_reduce(t, op=dist.ReduceOp.MAX)
assert t.item() == 2.0
dist.destroy_process_group()
print("NCCL_OK", torch.cuda.nccl.version())
"""


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_gather_world1(cuda_ok):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), NCCL_DEBUG="WARN")
    r = subprocess.run([sys.executable, "-c", _SCRIPT, ROOT], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "NCCL_OK" in r.stdout
