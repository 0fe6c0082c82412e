#!/bin/bash
# r2u: ncu --set full of attn_tc_kernel and the R2 GEMM on a 1,440-frame level wave of the
# 7,200-frame C4 video (layer 0, dependency level 3), the shapes the bench spends its time on
O=gpurun_out
NCU="ncu --set full --import-source on --clock-control none -c 1"
timeout 900 $NCU -k regex:attn_tc --launch-skip 3 -o $O/prof_r2u_attn7200 python tools/prof_run.py --frames 7200 > $O/prof_r2u_attn.log 2>&1
timeout 900 $NCU -k regex:gemm_tc_kernel --launch-skip 22 -o $O/prof_r2u_r2_7200 python tools/prof_run.py --frames 7200 > $O/prof_r2u_r2.log 2>&1
timeout 900 $NCU -k regex:gemm_tc_kernel --launch-skip 21 -o $O/prof_r2u_r1_7200 python tools/prof_run.py --frames 7200 > $O/prof_r2u_r1.log 2>&1
ls -la $O/*.ncu-rep
