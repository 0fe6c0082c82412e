#!/bin/bash
# Final round-2 measurement on one B200: the profile round (bench line, reference arm, ncu launch
# list, full captures of score / attention / FC1 / restore / general attention), then the C5,
# C4 p = 0.05, chain, 900-frame shard, x_bf16 and C2 lines.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash tools/profile_round.sh r2f > gpurun_out/profile_round_r2f.log 2>&1
B="python bench.py --no-cpu --no-baselines"
timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 --out gpurun_out/bench_r2f_c5.json > gpurun_out/bench_r2f_c5.log 2>&1
timeout 900 python bench.py --p 0.05 --steps 10 --warmup 3 --out gpurun_out/bench_r2f_c4_p0.05.json > gpurun_out/bench_r2f_c4_p0.05.log 2>&1
timeout 900 $B --chain --steps 3 --out gpurun_out/bench_r2f_chain.json > gpurun_out/bench_r2f_chain.log 2>&1
timeout 900 $B --frames 900 --steps 10 --out gpurun_out/bench_r2f_900.json > gpurun_out/bench_r2f_900.log 2>&1
timeout 900 python bench.py --x-bf16 --out gpurun_out/bench_r2f_xbf16.json > gpurun_out/bench_r2f_xbf16.log 2>&1
timeout 900 python bench.py --config b16 --frames 32 --p 0.1 --steps 20 --out gpurun_out/bench_r2f_c2_p0.1.json > gpurun_out/bench_r2f_c2.log 2>&1
timeout 900 python tools/sweep.py --out gpurun_out/sweep_r2f.json > gpurun_out/sweep_r2f.log 2>&1
grep -h '"value"' gpurun_out/bench_r2f*.json | cut -c1-160
ls -la gpurun_out | tail -40
