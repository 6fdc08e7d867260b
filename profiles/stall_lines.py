"""Top source lines per stall reason from an ncu report (--import-source on, -lineinfo).

    python profiles/stall_lines.py gpurun_out/<rep>.ncu-rep [reasons=long_sb,short_sb,wait] [top=8]
"""
import csv
import io
import subprocess
import sys


def main(path, reasons="long_sb,short_sb,wait", top=8):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    hdr, fname, rows = None, None, []
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r[0] == "Line No":
            hdr = r
        elif hdr and len(r) == len(hdr) and r[0].isdigit():
            rows.append((fname, int(r[0]), r[1].strip()[:90], dict(zip(hdr, r))))
    allst = sum(float(d.get("Warp Stall Sampling (All Samples)", 0) or 0) for *_, d in rows) or 1
    for rs in reasons.split(","):
        col = "stall_" + rs
        vals = [(float(d.get(col, 0) or 0), f, ln, src) for f, ln, src, d in rows]
        tot = sum(v for v, *_ in vals) or 1
        print(f"{rs}: {tot / allst:.2f} of all samples")
        for v, f, ln, src in sorted(vals, key=lambda t: -t[0])[:top]:
            print(f"  {v / tot:6.3f} {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3] or []), *([int(sys.argv[3])] if len(sys.argv) > 3 else []))
