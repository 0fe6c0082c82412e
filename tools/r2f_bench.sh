set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --steps 10 --warmup 3 --out gpurun_out/bench_r2f_c4.json > gpurun_out/bench_r2f_c4.log 2>&1
RV_LIB=build_var/libreusevit_wf2048.so timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-baselines --out gpurun_out/bench_r2f_c4_wf2048.json > gpurun_out/bench_r2f_c4_wf2048.log 2>&1
timeout 600 python bench.py --frames 900 --steps 10 --warmup 3 --no-cpu --no-baselines --out gpurun_out/bench_r2f_900.json > gpurun_out/bench_r2f_900.log 2>&1
grep -h '"value"' gpurun_out/bench_r2f_*.json | cut -c1-300
