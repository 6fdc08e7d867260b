"""Kernel timing study tool (GPU): average device time of one PC apply and one Jv at a
BASELINE configuration, CUDA events on the library's stream, inputs resident in HBM.
Variant libraries are selected with TPDG_GPU_LIB=...; with --save / --check the PC output is
stored / compared (rel-L2) so that A/B builds can be checked against each other.

  python tools/ktime.py --case cfg2 --p 15 [--reps 50] [--save f.npy | --check f.npy]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1704_04549_b200 as T  # noqa: E402


def build(case, p):
    if case == "cfg4":
        return T.setup_advection("const3d", 16, 16, 16, p=10, vel=(1.0, 0.7, 0.4)), 0.01
    if case == "cfg1":
        return T.setup_advection("const2d", 8, 8, p=8, vel=(1.0, 0.5, 0.0)), 0.01
    return T.setup_advection("swirl2d", 64, 64, p=p), 0.005


def timed(fn, stream, reps):
    s = torch.cuda.ExternalStream(stream)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1000.0 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="cfg2")
    ap.add_argument("--p", type=int, default=15)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--save")
    ap.add_argument("--check")
    a = ap.parse_args()
    sysm, dt = build(a.case, a.p)
    ctx = T.Context(0)
    op = T.LinearizedOperator(ctx, sysm, dt)
    pc = T.form_ksvd(op)
    b = T.uniform_vector(12345, sysm.N, 1.0)
    d_in = torch.from_numpy(b).cuda()
    d_out = torch.empty_like(d_in)
    d_jv = torch.empty_like(d_in)
    res = {"case": a.case, "p": a.p if a.case == "cfg2" else None, "N": sysm.N}
    res["pc_us"] = timed(lambda: pc.apply_device(d_in, d_out), ctx.stream(), a.reps)
    res["jv_us"] = timed(lambda: op.apply_device(d_in, d_jv), ctx.stream(), a.reps)
    y = d_out.cpu().numpy()
    if a.save:
        np.save(a.save, y)
    if a.check and os.path.exists(a.check):
        z = np.load(a.check)
        res["pc_rel_vs_saved"] = float(np.linalg.norm(y - z) / np.linalg.norm(z))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
