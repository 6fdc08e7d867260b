"""Warp-stall samples aggregated by SASS opcode and stall reason: python profiles/stall_by_op.py <rep>"""
import collections, csv, io, subprocess, sys
txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = collections.defaultdict(lambda: collections.Counter()); tot = 0
for r in rows[2:]:
    if len(r) != len(hdr): continue
    toks = r[idx["Source"]].split()
    if not toks: continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0] + ("." + op.split(".")[1] if op.startswith(("LDS", "LDCU", "LDG", "STS")) and "." in op else "")
    for k in st:
        v = int(r[idx[k]] or 0); agg[op][k[6:]] += v; tot += v
for op, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:14]:
    n = sum(c.values())
    print(f"{n / tot:6.3f} {op:10s} " + " ".join(f"{k}={v / tot:.3f}" for k, v in c.most_common(5) if v / tot >= 0.003))
