#!/usr/bin/env python
"""Benchmark: KSVD-preconditioned matrix-free GMRES on B200 (BASELINE.json configs[1]).

Workload (N=1 headline): 2D scalar linear advection, velocity (sin 2 pi y, cos 2 pi x), periodic
unit square, 64x64 quads, Gauss-Lobatto p=15 (q=16, mu=17), backward Euler dt=0.005, operator
A = M - dt J, right KSVD (r=2) preconditioner formed on the device, GMRES(30) to rel. tol 1e-10,
RHS uniform[-1,1] from std::mt19937_64(12345). Synthetic inputs with exactly the config's
shapes (there is no dataset). One step = one full GMRES solve from x0 = 0 on resident inputs.

value  = GDOF-iterations/s = N * iterations / t_solve (device CUDA events, max over ranks)
e2e    = same metric through the C ABI with HOST buffers (pinned H2D of b + D2H of x per step)
--impl reference : the reference CPU implementation (oracle/_ref/tpdg_ref_bench, compiled
                   in place from the unmodified reference) on this box's host cores.
Multi-GPU (torchrun): element rows partitioned across ranks, NCCL halo + allreduce (strong
scaling of the fixed 64x64 problem).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "preconditioned GMRES GDOF-iterations/s; Kronecker-apply GDOF/s vs roofline"
REF_BENCH = os.path.join(ROOT, "oracle", "_ref", "tpdg_ref_bench")
GOLDEN_ITS = {4: 17, 8: 18, 15: 25, 20: 39, 30: 21}  # reference GMRES counts, tests/golden/cfg2_p*.npz


def workload(p, case="cfg2"):
    if case == "cfg4":
        return ("cfg4: 3D advection, velocity (1, 0.7, 0.4), periodic unit cube, 16x16x16 hexes, Gauss-Lobatto "
                "p=10, backward Euler dt=0.01, A = M - dt J, right 3D KSVD (rank-1 x rank-2) preconditioner, "
                "GMRES(30) rel tol 1e-10, RHS uniform[-1,1] mt19937_64(12345), fp64")
    if case == "cfg1":
        return ("cfg1: 2D advection, velocity (1, 0.5), periodic unit square, 8x8 quads, Gauss-Lobatto p=8, "
                "backward Euler dt=0.01, right KSVD r=2, GMRES(30) rel tol 1e-10, RHS uniform[-1,1], fp64")
    return (f"cfg2: 2D advection, velocity (sin 2pi y, cos 2pi x), periodic unit square, 64x64 quads, "
            f"Gauss-Lobatto p={p}, backward Euler dt=0.005, A = M - dt J, right KSVD r=2 preconditioner, "
            f"GMRES(30) rel tol 1e-10, RHS uniform[-1,1] mt19937_64(12345), fp64")


def build_case(T, case, p):
    """(system, dt, golden case name, golden iteration count) of a BASELINE configuration."""
    if case == "cfg4":
        return T.setup_advection("const3d", 16, 16, 16, p=10, vel=(1.0, 0.7, 0.4)), 0.01, "cfg4", 159
    if case == "cfg1":
        return T.setup_advection("const2d", 8, 8, p=8, vel=(1.0, 0.5, 0.0)), 0.01, "cfg1", 11
    return T.setup_advection("swirl2d", 64, 64, p=p), 0.005, f"cfg2_p{p}", GOLDEN_ITS.get(p)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        if self.index < 0:
            return self
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def run_reference_bench(case, threads, max_its, reps, timeout=1800):
    out = subprocess.run([REF_BENCH, "bench", case, str(threads), str(max_its), str(reps)], capture_output=True,
                         text=True, timeout=timeout, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# --------------------------------------------------------------------------- reference arm
def main_reference(args, rank):
    if rank != 0:
        return 0
    if not os.path.exists(REF_BENCH):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/tpdg_ref_bench not built"}))
        return 0
    th = cpu_threads()
    ref_case = {"cfg4": "cfg4", "cfg1": "cfg1"}.get(args.case, f"cfg2_p{args.p}")
    r = run_reference_bench(ref_case, th, 2000, args.warmup + args.steps)
    times = r["gmres_s"][args.warmup:]
    t = statistics.median(times)
    N, its = r["N"], r["gmres_its"]
    value = N * its / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GDOF-it/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload(args.p, args.case), "N": N, "iterations": its, "p": args.p},
        "cpu_baseline": {"value": value, "unit": "GDOF-it/s", "cores": th, "kind": "reference",
                         "sample": f"{args.steps} full GMRES solves ({its} iterations each) after {args.warmup} "
                                   f"warm-up solves; unmodified reference, g++ -O3 -march=x86-64-v3, "
                                   f"thread_count()={th}; form {r['form_s']:.3f} s, "
                                   f"PC apply {r['pc_apply_s']:.3f} s, Jv {r['jv_s']:.3f} s"},
        "e2e": {"value": value, "unit": "GDOF-it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "form_s": r["form_s"], "fallbacks": r["fallbacks"],
    }
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------------- our arm
def main_ours(args, rank, world, local_rank):
    import torch
    import paper_1704_04549_b200 as T

    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
        obj = [T.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    else:
        torch.cuda.set_device(local_rank)
        nccl_id = None
    dev = torch.device("cuda", local_rank)
    ctx = T.Context(local_rank, rank, world, nccl_id)
    p = args.p
    sysm, dt, ref_case, ref_its = build_case(T, args.case, p)
    op = T.LinearizedOperator(ctx, sysm, dt)
    N = sysm.N
    e0, e1 = op.e_begin, op.e_end
    npe = sysm.npe
    b_host = T.uniform_vector(12345, N, 1.0)[e0 * npe:e1 * npe].copy()

    def barrier():
        if dist:
            dist.barrier()

    # ---- form (timed separately; once per solve in the reference's newton_linear_solve):
    # one warm-up formation, then the median of 3
    pc = T.form_ksvd(op)
    form_times = []
    for _ in range(3):
        pc.close()  # release the previous preconditioner outside the timed region (cudaFree synchronizes)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        pc = T.form_ksvd(op)
        torch.cuda.synchronize()
        form_times.append(time.perf_counter() - t0)
    form_s = statistics.median(form_times)
    nfb = len(pc.fallbacks)

    b = torch.from_numpy(b_host).to(dev)
    x = torch.zeros_like(b)
    cfg = T.GmresConfig(tol=1e-10, restart=30, max_iterations=2000, side="right")
    stream = torch.cuda.ExternalStream(ctx.stream())

    for _ in range(args.warmup):
        its, conv, _ = T.gmres_device(op, pc, b, x, cfg)
    torch.cuda.synchronize()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launches()
    its_list = []
    with ClockSampler(local_rank if not args.no_clocks else -1) as clk:
        torch.cuda.synchronize()
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            its, conv, _ = T.gmres_device(op, pc, b, x, cfg)
            its_list.append(its)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    t_ms = ev0.elapsed_time(ev1)
    launches = ctx.launches() - launches0
    # per-kernel breakdown: a separate pass with CUDA events around every PC / Jv / MGS launch
    # (the events cost ~7 %, so they stay out of the timed region above)
    prof = {"pc_apply": (0.0, 0), "jv": (0.0, 0), "mgs": (0.0, 0)}
    t_prof_ms = t_ms
    if not args.no_profile:
        ctx.profile(True)
        T.gmres_device(op, pc, b, x, cfg)  # grows the event pool
        ctx.profile_read()
        ctx.profile(True)
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            T.gmres_device(op, pc, b, x, cfg)
        ev1.record(stream)
        torch.cuda.synchronize()
        t_prof_ms = ev0.elapsed_time(ev1)
        prof = ctx.profile_read()
        ctx.profile(False)
    t_max = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    t_ms = float(t_max.item())
    its_total = int(sum(its_list))
    value = N * its_total / (t_ms * 1e-3) / 1e9

    # ---- end to end through the C ABI with host buffers (pinned)
    bh = torch.from_numpy(b_host).pin_memory()
    xh = torch.empty_like(bh).pin_memory()
    bh_np, xh_np = bh.numpy(), xh.numpy()
    T.gmres(op, pc, bh_np, cfg, out=xh_np)  # warm
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_its = 0
    for _ in range(args.steps):
        res = T.gmres(op, pc, bh_np, cfg, out=xh_np)
        e2e_its += res.iterations
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    e2e_t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = N * e2e_its / float(e2e_t.item()) / 1e9

    # ---- roofline of the dominant kernel class (algorithmic bytes per SURVEY.md sec.8d)
    hbm, hbm_kind = peaks()
    q, mu, nc, d = sysm.q, sysm.mu, sysm.n_c, sysm.dim
    n_loc = e1 - e0
    n1 = nc * q
    if d == 2:
        bytes_pc = n_loc * 8.0 * (2 * n1 * q + 3 * n1 * n1 + 3 * q * q)
        flops_pc = n_loc * 7.0 * n1 * q * (n1 + q)
    else:  # B = 8 (2 n1 q^2 + n1^2 + 6 q^2), F = 2 n1^2 q^2 + 14 n1 q^3
        bytes_pc = n_loc * 8.0 * (2 * n1 * q * q + n1 * n1 + 6 * q * q)
        flops_pc = n_loc * (2.0 * n1 * n1 * q * q + 14.0 * n1 * q ** 3)
    bytes_jv = n_loc * 8.0 * (2 * nc * q ** d + mu ** d * (1 + d * nc * nc) + 4 * d * mu ** (d - 1) * nc * nc)
    n_local = n_loc * nc * npe
    # MGS region of iteration k (0-based in its cycle): 8 (5 (k+1) + 3) bytes per DOF
    per_solve_its = its_list[0] if its_list else 0
    ks = [i % 30 for i in range(per_solve_its)]
    bytes_mgs_per_it = [n_local * 8.0 * (5 * (k + 1) + 3) for k in ks]
    kern = {}
    for name, algo in (("pc_apply", bytes_pc), ("jv", bytes_jv)):
        ms, cnt = prof[name]
        if cnt:
            avg = ms / cnt
            kern[name] = {"launches": cnt, "avg_us": avg * 1e3, "share": ms / t_prof_ms,
                          "algorithmic_bytes": algo, "achieved_gbs": algo / (avg * 1e-3) / 1e9}
    ms, cnt = prof["mgs"]
    if cnt:
        algo = float(np.mean(bytes_mgs_per_it)) if bytes_mgs_per_it else 0.0
        kern["mgs"] = {"launches": cnt, "avg_us": ms / cnt * 1e3, "share": ms / t_prof_ms,
                       "algorithmic_bytes": algo, "achieved_gbs": algo / (ms / cnt * 1e-3) / 1e9}
    dom = max(kern, key=lambda k: kern[k]["share"]) if kern else None
    roof = None
    traffic = {}
    try:  # per-launch DRAM bytes of the same kernels from an ncu --set full capture (profiles/)
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f)
    except Exception:
        pass
    if "mgs_bytes_per_pass" in traffic and ks:
        traffic["mgs"] = traffic["mgs_bytes_per_pass"] * float(np.mean([k + 2 for k in ks]))
    if dom:
        ach = kern[dom]["achieved_gbs"]
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "peak_kind": hbm_kind,
                "traffic": traffic.get(dom) if (p == 15 and args.case == "cfg2") else None,
                "algorithmic_bytes_per_launch": kern[dom]["algorithmic_bytes"]}
    kron = None
    if "pc_apply" in kern:
        avg_s = kern["pc_apply"]["avg_us"] * 1e-6
        # T_roof = max(B / BW_HBM, F / P_FP64); P_FP64 measured on the box (tools/fp64_peak.cu)
        p64 = 37.06
        try:
            with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
                p64 = float(json.load(f)["fp64_dmma_tflops"])
        except Exception:
            pass
        # 2D default kernel (kron_ew.cu) is bit-faithful: separate mul / add roundings, one flop per
        # FP64 instruction, so its FP64 ceiling is half the DFMA rate; TPDG_GPU_KRON=mma and the 3D
        # kernel use DMMA products (peak: measured DMMA rate)
        faithful = d == 2 and os.environ.get("TPDG_GPU_KRON", "ew")[:1] not in ("m",)
        p64_dfma = 35.91
        try:
            with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
                p64_dfma = float(json.load(f)["fp64_dfma_tflops"])
        except Exception:
            pass
        p_eff = p64_dfma / 2 if faithful else p64
        t_roof = max(bytes_pc / (hbm * 1e9), flops_pc / (p_eff * 1e12))
        kron = {"value": n_local / avg_s / 1e9 * world, "unit": "GDOF/s",
                "roofline_frac": t_roof / avg_s,
                "bound": "hbm" if bytes_pc / hbm * 1e-9 >= flops_pc / p_eff * 1e-12 else "fp64",
                "arithmetic": "bit-faithful (no FMA)" if faithful else "DMMA / FMA",
                "flops_per_launch": flops_pc, "achieved_tflops": flops_pc / avg_s / 1e12, "fp64_peak_tflops": p_eff,
                "hbm_frac": bytes_pc / (hbm * 1e9) / avg_s}

    # ---- CPU baseline (rank 0, N = 1): the unmodified reference on this host
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and os.path.exists(REF_BENCH):
        th = cpu_threads()
        try:
            r = run_reference_bench(ref_case, th, 2000, 1, timeout=900)
            v = r["N"] * r["gmres_its"] / r["gmres_s"][-1] / 1e9
            cpu = {"value": v, "unit": "GDOF-it/s", "cores": th, "kind": "reference",
                   "sample": f"one full GMRES solve ({r['gmres_its']} iterations) of the same workload, unmodified "
                             f"reference (oracle/_ref/tpdg_ref_bench, g++ -O3 -march=x86-64-v3), "
                             f"thread_count()={th}; form {r['form_s']:.3f} s, PC apply {r['pc_apply_s']:.3f} s, "
                             f"Jv {r['jv_s']:.3f} s"}
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": "GDOF-it/s", "cores": th, "kind": "reference", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GDOF-it/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(p, args.case), "N": N,
                       "iterations_per_solve": its_list[0] if its_list else None,
                       "reference_iterations": ref_its, "fallbacks": nfb, "p": p if args.case == "cfg2" else None,
                       "parallelism": f"element rows x{world}",
                       "l2": "inputs larger than L2 (Krylov basis 31 x N x 8 B + factors + operator data > 126 MB)"},
            "roofline": roof, "kron_apply": kron, "kernels": kern, "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "GDOF-it/s", "h2d_bytes_per_step": 8 * n_local * world,
                    "d2h_bytes_per_step": 8 * n_local * world},
            "gpu_launches": launches, "clocks": clk.summary(), "form_ms": form_s * 1e3,
        }
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--p", type=int, default=15, choices=[4, 8, 15, 20, 30], help="cfg2 polynomial degree")
    ap.add_argument("--case", default="cfg2", choices=["cfg2", "cfg1", "cfg4"],
                    help="BASELINE config (headline: cfg2 = configs[1]; others for measurement)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true", help="diagnostic: do not sample nvidia-smi")
    ap.add_argument("--no-profile", action="store_true", help="diagnostic: no per-kernel events")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return main_reference(args, rank)
    return main_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
