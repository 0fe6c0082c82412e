set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
RV_LIB=build_var/ag_trace/libreusevit_agtrace.so timeout 120 python tools/attn_probe.py --config l14_336 --frames 288 --nq 127 --only tcg --iters 1 > gpurun_out/ag_trace_577_r2h.txt 2>&1
tail -2 gpurun_out/ag_trace_577_r2h.txt
timeout 120 python tools/attn_probe.py --config l14_336 --frames 288 --nq 127 --only tcg
for p in 0.1 0.3; do timeout 600 python bench.py --config b16 --frames 32 --p $p --no-cpu --no-e2e --steps 50 --warmup 5 --out gpurun_out/bench_r2h_c2_p$p.json > gpurun_out/bench_r2h_c2_p$p.log 2>&1; done
grep -h '"value"' gpurun_out/bench_r2h_*.json | cut -c1-200
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "score" 2>&1 | tail -3
