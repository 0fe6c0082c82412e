set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "wavefront or misaligned or per_frame or determinism or embed_parity" 2>&1 | tail -5
timeout 900 python tools/sweep.py --out gpurun_out/sweep_r2e.json 2>&1 | tail -20
for f in 900 1800; do timeout 600 python tools/sweep.py --frames $f --ps 0.2 --parity-frames 0 --reps 3 --out gpurun_out/shard_r2e_$f.json 2>&1 | tail -9; done
