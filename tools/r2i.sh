set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for lib in "" build_var/poly2/libreusevit.so build_var/poly3/libreusevit.so build_var/poly4/libreusevit.so; do
  echo "== lib $lib"
  for args in "--config l14_336 --frames 288 --nq 127" "--config l14_336 --frames 288 --nq 577" "--config l14 --frames 288 --nq 257"; do
    RV_LIB=$lib timeout 120 python tools/attn_probe.py $args --only tcg
  done
done
RV_LIB=build_var/poly3/libreusevit.so timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" 2>&1 | tail -3
