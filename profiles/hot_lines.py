"""Top source lines by warp-stall samples from an ncu report (--import-source on, -lineinfo).

    python profiles/hot_lines.py gpurun_out/<rep>.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main(path, top=30):
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
        if hdr and r[0] and len(r) > 4 and r[4].isdigit():
            s = int(r[4] or 0)
            agg[(fname, int(r[0]), r[1].strip()[:90])] = s
            tot += s
    for (f, ln, src), s in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{s / max(tot, 1):6.3f} {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
