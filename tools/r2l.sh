set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2000 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2l.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gputest_r2l.log
