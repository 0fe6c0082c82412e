set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2b.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gputest_r2b.log
for args in "--config l14_336 --frames 288 --nq 127" "--config l14 --frames 288 --nq 57" "--config l14 --frames 288 --nq 257"; do echo "== $args"; timeout 300 python tools/attn_probe.py $args --only all; done
