set -x
python bench.py --steps 10 --warmup 3 --out gpurun_out/bench_c4_p0.2.json > gpurun_out/bench_c4_p0.2.log 2>&1
python bench.py --p 0.05 --steps 10 --warmup 3 --out gpurun_out/bench_c4_p0.05.json > gpurun_out/bench_c4_p0.05.log 2>&1
python bench.py --config b16 --frames 32 --p 0.3 --cpu-frames 32 --steps 20 --warmup 5 --out gpurun_out/bench_c2_p0.3.json > gpurun_out/bench_c2_p0.3.log 2>&1
python bench.py --config b16 --frames 32 --p 0.1 --cpu-frames 32 --steps 20 --warmup 5 --out gpurun_out/bench_c2_p0.1.json > gpurun_out/bench_c2_p0.1.log 2>&1
python bench.py --workload c5 --steps 3 --warmup 3 --out gpurun_out/bench_c5.json > gpurun_out/bench_c5.log 2>&1
python bench.py --chain --steps 5 --warmup 3 --no-cpu --out gpurun_out/bench_chain.json > gpurun_out/bench_chain.log 2>&1
python tools/sweep.py --out gpurun_out/sweep_r2.json > gpurun_out/sweep_r2.log 2>&1
python tools/memory_curve.py --out gpurun_out/memory_curve_r2.json > gpurun_out/memory_curve_r2.log 2>&1
ls -la gpurun_out | tail -30
