set -x
timeout 400 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "chain or l14_336" 2>&1 | tail -2
for args in "--config l14_336 --frames 288 --nq 127" "--config l14_336 --frames 288 --nq 577" "--config l14 --frames 288 --nq 257"; do
  timeout 120 python tools/attn_probe.py $args --only tcg
done
timeout 600 python bench.py --chain --steps 5 --warmup 3 --no-cpu --no-baselines --no-e2e --out gpurun_out/bench_r2r_chain.json > gpurun_out/bench_r2r_chain.log 2>&1
grep -h '"value"' gpurun_out/bench_r2r_chain.json | cut -c1-150
