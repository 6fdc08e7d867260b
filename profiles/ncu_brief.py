"""Brief ncu summary: duration, occupancy, IPC, stall mix, per-unit SASS opcode histogram.

    python profiles/ncu_brief.py gpurun_out/<rep>.ncu-rep [units]
"""
import collections
import csv
import io
import subprocess
import sys


def ncu(path, *args):
    return subprocess.run(["ncu", "-i", path, *args], capture_output=True, text=True).stdout


def main(path, units=4096):
    for r in csv.reader(io.StringIO(ncu(path, "--page", "details", "--csv"))):
        if len(r) > 14 and any(k in r[12] for k in ["Duration", "Registers Per", "Dynamic Shared", "Issue Slots Busy",
                                                     "Achieved Active Warps", "Executed Ipc A", "DRAM Throughput"]):
            print(f"{r[12]} = {r[14]} {r[13]}")
    rows = list(csv.reader(io.StringIO(ncu(path, "--page", "raw", "--csv"))))
    d = dict(zip(rows[0], rows[2] if len(rows) > 2 else rows[1]))
    st = []
    for k, v in d.items():
        if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
            try:
                st.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", ""))))
            except ValueError:
                pass
    tot = sum(x for _, x in st) or 1
    print("stalls:", ", ".join(f"{k} {x / tot:.2f}" for k, x in sorted(st, key=lambda t: -t[1])[:7]))
    hdr, agg, n_all = None, collections.Counter(), 0
    for r in csv.reader(io.StringIO(ncu(path, "--page", "source", "--csv", "--print-source", "sass"))):
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            row = dict(zip(hdr, r))
            toks = row.get("Source", "").split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            try:
                n = float(row.get("Instructions Executed", "0") or 0)
            except ValueError:
                continue
            agg[op.split(".")[0]] += n
            n_all += n
    print(f"warp instructions per unit: {n_all / units:.0f}")
    print("  " + ", ".join(f"{k} {v / units:.0f}" for k, v in agg.most_common(16)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 4096)
