"""bench.py's N > 1 path on the one-GPU box: two ranks (torchrun, gloo, both on cuda:0 through
the RV_BENCH_GLOO_ONE_GPU test hook) run the frame-group sharding with its halo I-frame, the
embedding / mask gather, the max-over-ranks timing and the rank-0 JSON line, for the C4-style
video workload and the C5 multi-video workload, so that the first 8-GPU run cannot die on an
untested branch.  The NCCL collective itself is covered by tests/test_gpu_dist.py."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("extra", [["--config", "b16", "--frames", "84"],
                                   ["--workload", "c5", "--videos", "4", "--video-frames", "20"]],
                         ids=["video", "c5"])
def test_bench_two_ranks_one_gpu(cuda_ok, extra, tmp_path):
    out = tmp_path / "line.json"
    env = dict(os.environ, RV_BENCH_GLOO_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-cpu", "--no-baselines", "--out", str(out)] + extra
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-5000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["ms_per_step"] > 0
    assert json.loads(out.read_text()) == d
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
