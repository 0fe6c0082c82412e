set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sanitizer.py tests/test_gpu_store.py tests/test_gpu_train.py tests/test_gpu_bench_multirank.py -q > gpurun_out/gputest_r2n.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gputest_r2n.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
bash tools/r2m.sh
