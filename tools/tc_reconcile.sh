#!/bin/bash
# Tensor-pipe evidence for the tcgen05 kernels: ncu over every GEMM launch of
# layer 0 of a 1,440-frame L/14 embed (patch embed, then per level-wave QKV, W_o, FC1, FC2
# [, R1, R2]) and that layer's 7 attention launches, with the UTCHMMA bf16->fp32 math-op counter
# next to the duration, DRAM bytes and the tensor-pipe activity counters.  Reconciled on the CPU
# box by tools/tc_reconcile.py against the algorithmic / tile-padded 2*M*N*K of each launch.
set -u
O=gpurun_out
mkdir -p $O
M="gpu__time_duration.sum,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum,sm__inst_executed_pipe_tc.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second"
timeout 300 python tools/prof_run.py --frames 1440 --counts-out $O/tc_counts.json > $O/tc_counts.log 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:gemm_tc -c 41 --csv \
  --log-file $O/tc_gemm.csv python tools/prof_run.py --frames 1440 > /dev/null 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:attn_tc -c 7 --csv \
  --log-file $O/tc_attn.csv python tools/prof_run.py --frames 1440 > /dev/null 2>&1
ls -la $O/tc_*
