set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 ./build/gather_rate > gpurun_out/gather_rate_r2g.txt 2>&1; cat gpurun_out/gather_rate_r2g.txt
timeout 600 python bench.py --chain --steps 5 --warmup 3 --no-cpu --no-baselines --no-e2e --out gpurun_out/bench_r2g_chain.json > gpurun_out/bench_r2g_chain.log 2>&1
timeout 600 python bench.py --config b16 --frames 32 --p 0.1 --cpu-frames 32 --steps 20 --warmup 5 --out gpurun_out/bench_r2g_c2_p0.1.json > gpurun_out/bench_r2g_c2_p0.1.log 2>&1
timeout 600 python bench.py --config b16 --frames 32 --p 0.3 --cpu-frames 32 --steps 20 --warmup 5 --out gpurun_out/bench_r2g_c2_p0.3.json > gpurun_out/bench_r2g_c2_p0.3.log 2>&1
grep -h '"value"' gpurun_out/bench_r2g_*.json | cut -c1-200
