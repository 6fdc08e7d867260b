"""Summarize ncu captures into the text files committed under profiles/ (run in the build container).

    python profiles/summarize.py <round-tag> gpurun_out/<tag>_launches.csv gpurun_out/<tag>_*.ncu-rep
"""
import collections
import csv
import io
import os
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "L2 Hit Rate", "L1/TEX Hit Rate"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(list)
    for d in data:
        if d.get("Metric Name") == "gpu__time_duration.sum":
            agg[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"]) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    out = ["kernel | launches | mean us | total us | share", "---|---|---|---|---"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k} | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} | {sum(v) / tot:.3f}")
    return "\n".join(out)


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    out, name = [], None
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        name = name or d.get("Kernel Name")
        if d.get("Metric Name") in KEYS:
            out.append(f"{d['Metric Name']} = {d['Metric Value']} {d['Metric Unit']}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) >= 3:
        h, units, vals = rr[0], rr[1], rr[2]
        for key in ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]:
            if key in h:
                i = h.index(key)
                out.append(f"{key} = {vals[i]} {units[i]}")
    return f"## {os.path.basename(path)}: {name}\n" + "\n".join(out)


def main(argv):
    tag = argv[0]
    parts = []
    for p in argv[1:]:
        parts.append(f"# launch list {os.path.basename(p)}\n" + launches(p) if p.endswith(".csv") else report(p))
    dst = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"{tag}_ncu_summary.md")
    with open(dst, "w") as f:
        f.write("\n\n".join(parts) + "\n")
    print(dst)


if __name__ == "__main__":
    main(sys.argv[1:])
