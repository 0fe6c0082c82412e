set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "chain" 2>&1 | tail -3
timeout 400 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" 2>&1 | tail -3
timeout 600 python bench.py --chain --steps 5 --warmup 3 --no-cpu --no-baselines --no-e2e --out gpurun_out/bench_r2q_chain.json > gpurun_out/bench_r2q_chain.log 2>&1
timeout 600 python bench.py --chain --attn-sync --steps 5 --warmup 3 --no-cpu --no-baselines --no-e2e --out gpurun_out/bench_r2q_chain_sync.json > gpurun_out/bench_r2q_chain_sync.log 2>&1
grep -h '"value"' gpurun_out/bench_r2q_chain*.json | cut -c1-150
