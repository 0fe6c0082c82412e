set -x
RV_LIB=build_var/ag_trace/libreusevit_agtrace.so timeout 120 python tools/attn_probe.py --config l14_336 --frames 288 --nq 127 --only tcg --iters 1 > gpurun_out/ag_trace_577_r2m.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_tcg -c 1 --launch-skip 2 -o gpurun_out/prof_r2m_tcg python tools/attn_probe.py --config l14_336 --frames 288 --nq 127 --only tcg --iters 2 > gpurun_out/prof_r2m_tcg.log 2>&1
ls -la gpurun_out/prof_r2m_tcg*
