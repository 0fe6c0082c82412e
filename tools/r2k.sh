set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 400 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" 2>&1 | tail -3
for args in "--config l14 --frames 288 --nq 57" "--config l14 --frames 1440 --nq 47" "--config l14 --frames 288 --nq 257" "--config b16 --frames 288 --nq 40"; do
  timeout 120 python tools/attn_probe.py $args --only tc
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "embed_parity or wavefront" 2>&1 | tail -3
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-baselines --out gpurun_out/bench_r2k_c4.json > gpurun_out/bench_r2k_c4.log 2>&1
grep -h '"value"' gpurun_out/bench_r2k_c4.json | cut -c1-200
