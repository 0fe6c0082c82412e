#!/bin/bash
# Round profiling on one B200 (run under gpurun from the repo root): the bench line, the
# reference arm, the ncu launch list of the bench command itself, and one `ncu --set full`
# capture per dominant kernel class (tools/prof_run.py, 1,440-frame L/14 video, layer 0,
# dependency level 3 = a 288-frame wave).  Summarise afterwards on the CPU box with
#   python tools/summarize_profiles.py --round R --launches gpurun_out/launches_R.csv \
#     --rep attention=gpurun_out/prof_R_attn.ncu-rep --rep score=... --rep gemm_fc1=... --rep gemm_r2=...
set -u
R=${1:-r1c}
O=gpurun_out
mkdir -p $O
timeout 600 python bench.py --out $O/bench_${R}.json > $O/bench_${R}.log 2>&1
timeout 600 python bench.py --impl reference --out $O/bench_${R}_reference.json > $O/bench_${R}_reference.log 2>&1
KR='regex:score_kernel|compact_kernel|gather_ln|attn|gemm_tc_kernel|restore_kernel|patch_to_bf16|embed_finish|ln_post'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" --csv --log-file $O/launches_${R}.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-baselines > $O/ncu_launches_${R}.log 2>&1
NCU="ncu --set full --import-source on --clock-control none -c 1"
timeout 600 $NCU -k regex:attn_tc --launch-skip 3 -o $O/prof_${R}_attn python tools/prof_run.py --frames 1440 > /dev/null 2>&1
timeout 600 $NCU -k regex:score_kernel --launch-skip 3 -o $O/prof_${R}_score python tools/prof_run.py --frames 1440 > /dev/null 2>&1
# gemm_tc_kernel launches: PE, then QKV / W_o / FC1 / FC2 per wave -> FC1 of wave 3 is launch 15;
# restore_kernel: one per wave with references (waves 1-6 of layer 0) -> wave 3 is launch 2
timeout 600 $NCU -k regex:gemm_tc_kernel --launch-skip 15 -o $O/prof_${R}_fc1 python tools/prof_run.py --frames 1440 > /dev/null 2>&1
timeout 600 $NCU -k regex:restore_kernel --launch-skip 2 -o $O/prof_${R}_restore python tools/prof_run.py --frames 1440 > /dev/null 2>&1
# the general tcgen05 attention (L/14@336, T = 577; BASELINE configs[4] shape), level-3 wave
timeout 600 $NCU -k regex:attn_tcg --launch-skip 3 -o $O/prof_${R}_attng python tools/prof_run.py --config l14_336 --frames 480 > /dev/null 2>&1
ls -la $O | tail -20
