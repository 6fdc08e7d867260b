"""Top source lines by executed warp instructions (per unit) from an ncu report.

    python profiles/inst_lines.py gpurun_out/<rep>.ncu-rep <units> [top]
"""
import csv
import io
import subprocess
import sys


def main(path, units, top=30):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, hdr, agg, tot = None, None, {}, 0
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0] and len(r) > 7 and r[7].isdigit():
            s = int(r[7])
            agg[(fname, int(r[0]), r[1].strip()[:90])] = s
            tot += s
    print(f"total warp instructions {tot}, per unit {tot / units:.0f}")
    for (f, ln, src), s in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{s / tot:6.3f} {s / units:8.0f} {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 30)
