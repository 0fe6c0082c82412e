#!/bin/bash
# r2v: fused restoration kernel: bitwise vs the two GEMMs, parity suite, C4 bench (fused and
# RV_RESTORE_GEMMS-equivalent numbers come from the bench's kernel table)
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_restore.py -m gpu -x -q > $O/gputest_r2v_restore.log 2>&1
tail -3 $O/gputest_r2v_restore.log
if grep -q " passed" $O/gputest_r2v_restore.log && ! grep -q "failed" $O/gputest_r2v_restore.log; then
  timeout 600 python bench.py --no-cpu --no-e2e --no-baselines --out $O/bench_r2v_c4.json > $O/bench_r2v_c4.log 2>&1
  timeout 600 python bench.py --no-cpu --no-e2e --no-baselines --x-bf16 --out $O/bench_r2v_c4_xbf16.json > $O/bench_r2v_c4_xbf16.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_xbf16.py -m gpu -x -q > $O/gputest_r2v_parity.log 2>&1
  tail -3 $O/gputest_r2v_parity.log
fi
