"""Reconcile the ncu tensor-pipe counters with the algorithmic FLOPs of each tcgen05 launch
(VERDICT r1 item 5).  Input: gpurun_out/tc_gemm.csv, tc_attn.csv (ncu --csv, tools/tc_reconcile.sh)
and tc_counts.json (per-layer, per-wave M_C / M_R of the same embed).

For every launch: algorithmic FLOPs (2 M N K with the real compacted M; attention 4 nq T D),
UTCHMMA math ops counted by ncu (sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32: executed
multiply-add lanes incl. tile padding), their ratio, and three rates over the ncu duration:
alg FLOP/s, counted FLOP/s, and the tensor-pipe activity counters.

    python tools/tc_reconcile.py [gpurun_out] > profiles/tc_reconcile_r2.md
"""
import csv
import json
import os
import sys
from collections import defaultdict


def load(path):
    rows = defaultdict(dict)
    names = {}
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    for r in csv.DictReader(lines):
        i = int(r["ID"])
        names[i] = r["Kernel Name"]
        v = r["Metric Value"].replace(",", "")
        try:
            rows[i][r["Metric Name"]] = float(v)
        except ValueError:
            rows[i][r["Metric Name"]] = v
    return [(names[i], rows[i]) for i in sorted(rows)]


def main():
    d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    cnt = json.load(open(os.path.join(d, "tc_counts.json")))
    T, D, F, Hr, n = cnt["T"], cnt["D"], cnt["F"], cnt["Hr"], cnt["n"]
    N = T - 1
    frames = cnt["frames"]
    MC, MR = cnt["M_C"][0], cnt["M_R"][0]
    peak = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json")))
    # expected layer-0 GEMM launch sequence
    seq = [("PE", n * N, D, 640)]
    for w, nw in enumerate(frames):
        seq += [("QKV", MC[w], 3 * D, D), ("W_o", MC[w], D, D), ("FC1", MC[w], F, D), ("FC2", MC[w], D, F)]
        if MR[w] > 0 or w > 0:
            seq += [("R1", MR[w], Hr, D, nw * T), ("R2", MR[w], D, Hr)]
    g = load(os.path.join(d, "tc_gemm.csv"))
    print("# tcgen05 tensor-pipe counters vs algorithmic FLOPs (layer 0, 1,440-frame L/14 embed, p = 0.2)\n")
    print("ncu `--clock-control none`, one launch per row. `alg` = 2·M·N·K with the real compacted M "
          "(R1: M = reused rows; it runs over all n_w·T wave rows); `utc` = UTCHMMA math ops counted "
          "by ncu (×1 = FLOPs if the counter counts FLOPs, see the ratio column); rates over the ncu "
          "duration; `pipe%` = sm__pipe_tensor_cycles_active, `hmma%` = the hmma subpipe, `smem-tc%` = "
          "sm__mem_tensor_cycles_active (tensor-core operand reads).\n")
    print("`pred%` = utc TF/s / (8,192 dense bf16 FLOP per clock per SM x 148 SMs x the launch's SM clock "
          "`sm__cycles_elapsed.avg.per_second`): the tensor-pipe activity the counted FLOPs imply.\n")
    print("| # | GEMM | M | N | K | us | MHz | alg TF/s | utc/alg | utc TF/s | pipe% | pred% | smem-tc% | DRAM GB/s |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    agg = defaultdict(lambda: [0.0, 0.0, 0.0])
    for i, ((name, m), s) in enumerate(zip(g, seq)):
        kind, M, Nn, K = s[:4]
        us = m["gpu__time_duration.sum"] / 1e3
        alg = 2.0 * M * Nn * K
        utc = m.get("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum", 0.0)
        dram = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        agg[kind][0] += us
        agg[kind][1] += alg
        agg[kind][2] += utc
        clk = m.get("sm__cycles_elapsed.avg.per_second", 0.0)
        pred = utc / (us * 1e-6) / (8192.0 * 148 * clk) * 100 if clk else 0.0
        print(f"| {i} | {kind} | {M} | {Nn} | {K} | {us:.1f} | {clk / 1e6:.0f} | {alg / us / 1e6:.0f} | "
              f"{utc / alg if alg else 0:.3f} | {utc / us / 1e6:.0f} | "
              f"{m.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0):.1f} | {pred:.1f} | "
              f"{m.get('sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0):.1f} | {dram / us / 1e3:.0f} |")
    print("\n| GEMM class (layer 0) | us | alg TF/s | utc/alg | utc TF/s | frac of sustained bf16 peak (utc) |")
    print("|---|---|---|---|---|---|")
    pk = peak.get("bf16_tflops_sustained") or peak.get("bf16_tflops")
    for k, (us, alg, utc) in agg.items():
        print(f"| {k} | {us:.0f} | {alg / us / 1e6:.0f} | {utc / alg if alg else 0:.3f} | {utc / us / 1e6:.0f} | "
              f"{utc / us / 1e6 / pk:.2f} |" if pk else f"| {k} | {us:.0f} | {alg / us / 1e6:.0f} | | | |")
    a = load(os.path.join(d, "tc_attn.csv"))
    print("\n| attention wave | frames | queries | us | alg TF/s (4 nq T D) | utc/alg | utc TF/s | pipe% | pred% | DRAM GB/s |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for w, (name, m) in enumerate(a):
        us = m["gpu__time_duration.sum"] / 1e3
        alg = 4.0 * MC[w] * T * D
        utc = m.get("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum", 0.0)
        dram = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        clk = m.get("sm__cycles_elapsed.avg.per_second", 0.0)
        pred = utc / (us * 1e-6) / (8192.0 * 148 * clk) * 100 if clk else 0.0
        print(f"| {w} | {frames[w]} | {MC[w]} | {us:.1f} | {alg / us / 1e6:.0f} | {utc / alg:.3f} | {utc / us / 1e6:.0f} | "
              f"{m.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0):.1f} | {pred:.1f} | "
              f"{dram / us / 1e3:.0f} |")


if __name__ == "__main__":
    main()
