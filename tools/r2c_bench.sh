set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 --out gpurun_out/bench_r2c_c5.json > gpurun_out/bench_r2c_c5.log 2>&1
timeout 600 python bench.py --chain --steps 5 --warmup 3 --no-cpu --out gpurun_out/bench_r2c_chain.json > gpurun_out/bench_r2c_chain.log 2>&1
tail -3 gpurun_out/bench_r2c_c5.log gpurun_out/bench_r2c_chain.log
