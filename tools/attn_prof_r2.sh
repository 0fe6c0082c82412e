python tools/attn_probe.py --config l14_336 --frames 288 --nq 127 --only all
python tools/attn_probe.py --config l14 --frames 288 --nq 57 --only all
python tools/attn_probe.py --config l14 --frames 288 --nq 257 --only all
ncu --set full --import-source on --clock-control none -k regex:attn_tcg -c 1 -o gpurun_out/prof_r2_tcg python tools/attn_probe.py --config l14_336 --frames 288 --nq 127 --only tcg --iters 1 > /dev/null 2>&1
ls -la gpurun_out/prof_r2_tcg*
