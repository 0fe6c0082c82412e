set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash tools/profile_round.sh r2 > gpurun_out/profile_round_r2.log 2>&1
timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 --out gpurun_out/bench_r2s_c5.json > gpurun_out/bench_r2s_c5.log 2>&1
timeout 900 python bench.py --p 0.05 --steps 10 --warmup 3 --out gpurun_out/bench_r2s_c4_p0.05.json > gpurun_out/bench_r2s_c4_p0.05.log 2>&1
grep -h '"value"' gpurun_out/bench_r2*.json | cut -c1-160
ls -la gpurun_out | tail -30
