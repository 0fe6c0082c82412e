# r2b: new general tcgen05 attention — correctness, then speed vs the other kernels
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" 2>&1 | tail -15
for args in "--config l14_336 --frames 288 --nq 127" "--config l14 --frames 288 --nq 57" "--config l14 --frames 288 --nq 257" "--config l14_336 --frames 288 --nq 577"; do echo "== $args"; timeout 120 python tools/attn_probe.py $args --only all; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "chain or l14_336" 2>&1 | tail -5
