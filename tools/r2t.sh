#!/bin/bash
# r2t: head-interleaved K/V cache layout (k_h v_h per token): attention + parity tests, bench
# lines for C4 (product lib and the A8_L2_PREFETCH=256 variant), C5 and the chain variant.
set -x
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -m gpu -x -q > $O/gputest_r2t_kv.log 2>&1
tail -3 $O/gputest_r2t_kv.log
B="python bench.py --no-cpu --no-e2e --no-baselines"
timeout 600 $B --out $O/bench_r2t_c4.json > $O/bench_r2t_c4.log 2>&1
RV_LIB=build/var_l2.so timeout 600 $B --out $O/bench_r2t_c4_l2.json > $O/bench_r2t_c4_l2.log 2>&1
timeout 900 $B --workload c5 --steps 3 --out $O/bench_r2t_c5.json > $O/bench_r2t_c5.log 2>&1
timeout 900 $B --chain --steps 3 --out $O/bench_r2t_chain.json > $O/bench_r2t_chain.log 2>&1
for f in $O/bench_r2t_*.json; do echo $f; python -c "
import json,sys; d=json.load(open('$f')); k={x['name']:x['ms'] for x in d['kernels']}
print(round(d['value']), d['clocks']['sm_mhz'], 'attn', k.get('attention'), 'step', round(d['ms_per_step'],1))"; done
