set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 400 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" 2>&1 | tail -3
for args in "--config l14_336 --frames 288 --nq 127" "--config l14_336 --frames 288 --nq 577" "--config l14 --frames 288 --nq 257" "--config l14 --frames 1440 --nq 47"; do
  timeout 120 python tools/attn_probe.py $args --only tcg
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "chain or l14_336" 2>&1 | tail -3
