"""Summarise ncu captures into profiles/ (run here, on the CPU box, after gpurun brings the
reports back).

    python tools/summarize_profiles.py --round r1 --launches gpurun_out/launches_r1.csv \
        --rep fc1=gpurun_out/prof_r1g_fc1.ncu-rep --rep attn=gpurun_out/prof_r1g_attn.ncu-rep ...

Writes profiles/launches_<round>.csv (the raw per-launch list), profiles/launch_shares_<round>.csv
(per kernel class: launches, summed cold-cache time, share), profiles/ncu_<name>_<round>.txt
(key counters of each --set full capture) and merges dram bytes per launch into
profiles/ncu_traffic.json (read by bench.py for the roofline `traffic` field).
"""
import argparse
import csv
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
GEMM_ORDER_FULL = ["gemm_qkv", "gemm_wo", "gemm_fc1", "gemm_fc2", "gemm_r1", "gemm_r2"]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def classify(names):
    """Map the launch sequence to kernel classes (gemm launches are told apart by their
    position inside a wave: score starts a wave; then qkv, wo, fc1, fc2[, r1, r2])."""
    out = []
    gi = None
    ln = 0
    for n in names:
        if "score_kernel" in n:
            gi, ln = 0, 0
            out.append("score")
        elif "compact_kernel" in n:
            out.append("compact")
        elif "gather_ln" in n:
            out.append("gather_ln1" if ln == 0 else "ln2")
            ln += 1
        elif "rgather" in n or "gather_rows" in n:
            out.append("rgather")
        elif "attn" in n:
            out.append("attention")
        elif "restore_kernel" in n:
            out.append("restore")
        elif "gemm_tc_kernel" in n:
            if gi is None:
                out.append("gemm_pe")
            else:
                out.append(GEMM_ORDER_FULL[min(gi, 5)])
                gi += 1
        elif "patch_to_bf16" in n:
            out.append("patch_to_bf16")
        elif "embed_finish" in n:
            out.append("embed_finish")
        elif "ln_post" in n:
            out.append("ln_post")
            gi = None
        else:
            out.append("other")
    return out


def launches(path, rnd):
    rows = list(csv.reader(open(path)))
    hdr = None
    recs = []
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                unit = d.get("Metric Unit", "ns")
                scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
                recs.append((d["Kernel Name"], v * scale))
    shutil.copy(path, os.path.join(PROF, f"launches_{rnd}.csv"))
    cls = classify([n for n, _ in recs])
    agg = {}
    for (n, ms), c in zip(recs, cls):
        a = agg.setdefault(c, [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(PROF, f"launch_shares_{rnd}.csv"), "w") as fh:
        fh.write("class,launches,ms_cold_serialised,share\n")
        for c, (k, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
            fh.write(f"{c},{k},{ms:.3f},{ms / tot:.4f}\n")
    return agg, tot


def ncu_keys(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return {}
    h, u, v = rows[0], rows[1], rows[2]
    res = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else "?"}
    for k in KEYS:
        hits = [i for i, name in enumerate(h) if name == k or name.endswith("." + k)]
        if hits:
            i = hits[0]
            res[k] = f"{v[i]} {u[i]}".strip()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r1")
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[])
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        agg, tot = launches(a.launches, a.round)
        print(f"{sum(v[0] for v in agg.values())} launches, {tot:.1f} ms cold-serialised")
        for c, (k, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
            print(f"  {c:14s} {k:6d} {ms:9.2f} ms  {ms / tot:6.1%}")
    tpath = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for spec in a.rep:
        name, rep = spec.split("=", 1)
        d = ncu_keys(rep)
        with open(os.path.join(PROF, f"ncu_{name}_{a.round}.txt"), "w") as fh:
            fh.write(f"# ncu --set full --clock-control none, one launch ({os.path.basename(rep)})\n")
            for k, v in d.items():
                fh.write(f"{k}: {v}\n")
        print(name, d)
        try:
            rd = float(d["dram__bytes_read.sum"].split()[0].replace(",", ""))
            wr = float(d["dram__bytes_write.sum"].split()[0].replace(",", ""))
            unit = d["dram__bytes_read.sum"].split()[1]
            mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            traffic[name] = {"dram_bytes_per_launch": (rd + wr) * mul, "source": os.path.basename(rep),
                             "note": "one ncu --set full launch (tools/prof_run.py, 1,440 frames)"}
        except Exception:
            pass
    with open(tpath, "w") as fh:
        json.dump(traffic, fh, indent=1)


if __name__ == "__main__":
    main()
