#!/bin/bash
# Round-2 closing bench lines (after the host-path fix): C4 headline with e2e / baselines /
# oracle, reference arm, C4 p = 0.05, C5, chain, 900-frame shard, x_bf16, C2, C3 sweep.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
O=gpurun_out
timeout 900 python bench.py --out $O/bench_r2g_c4.json > $O/bench_r2g_c4.log 2>&1
timeout 900 python bench.py --impl reference --out $O/bench_r2g_reference.json > $O/bench_r2g_reference.log 2>&1
timeout 900 python bench.py --p 0.05 --steps 10 --out $O/bench_r2g_c4_p0.05.json > $O/bench_r2g_c4_p0.05.log 2>&1
timeout 900 python bench.py --workload c5 --steps 3 --out $O/bench_r2g_c5.json > $O/bench_r2g_c5.log 2>&1
timeout 900 python bench.py --chain --steps 3 --no-cpu --out $O/bench_r2g_chain.json > $O/bench_r2g_chain.log 2>&1
timeout 900 python bench.py --frames 900 --steps 10 --no-cpu --out $O/bench_r2g_900.json > $O/bench_r2g_900.log 2>&1
timeout 900 python bench.py --x-bf16 --out $O/bench_r2g_xbf16.json > $O/bench_r2g_xbf16.log 2>&1
timeout 900 python bench.py --config b16 --frames 32 --p 0.1 --steps 20 --out $O/bench_r2g_c2_p0.1.json > $O/bench_r2g_c2.log 2>&1
timeout 900 python bench.py --config b16 --frames 32 --p 0.3 --steps 20 --out $O/bench_r2g_c2_p0.3.json > $O/bench_r2g_c2b.log 2>&1
timeout 1200 python tools/sweep.py --out $O/sweep_r2g.json > $O/sweep_r2g.log 2>&1
grep -h '"value"' $O/bench_r2g*.json | cut -c1-120
