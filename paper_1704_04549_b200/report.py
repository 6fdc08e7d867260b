"""Scan reports in the reference's format.

The reference's harness writes one CSV row per (case, p, dt, preconditioner) cell
(harness/experiment.hpp:32-46: `report_csv_header`, `report_row_csv`, precision 12) and maps
exceptions to failure codes (experiment.hpp:98-105). This module emits the same columns for
B200 runs of the BASELINE configurations, so that GPU scans drop into the reference's tooling:

    python -m paper_1704_04549_b200.report --p 4 8 15 20 30 --out scan.csv

A cell here is one backward-Euler step of the linear advection problem = one linear solve
(newton_steps = 1); form_seconds / pc_apply_seconds / total_seconds are wall / device times of
the KSVD formation, of all preconditioner applications inside GMRES (CUDA events on the
library's stream) and of the whole cell. l2_error is empty (no exact solution is used here).
"""
import argparse
import dataclasses
import math
import sys
import time

import numpy as np

# harness/experiment.hpp:32-35
REPORT_CSV_HEADER = ("case,p,dt,precond,avg_gmres_iters,total_gmres_iters,newton_steps,form_seconds,"
                     "pc_apply_seconds,total_seconds,l2_error,status,failure_code")


@dataclasses.dataclass
class ReportRow:
    """ReportRow (harness/experiment.hpp:13-30)."""
    case_id: str
    p: int
    dt: float
    precond: str = "ksvd_full"
    avg_gmres: float = 0.0
    total_gmres: int = 0
    newton_steps: int = 0
    form_seconds: float = 0.0
    pc_apply_seconds: float = 0.0
    total_seconds: float = 0.0
    l2_error: float = float("nan")
    status: str = "ok"
    failure_code: str = ""
    gmres_per_solve: list = dataclasses.field(default_factory=list)


def _num(x):
    """C++ ostream << double with precision(12) (default float field): %.12g."""
    if isinstance(x, (int, np.integer)):
        return str(int(x))
    return f"{x:.12g}"


def report_row_csv(r: ReportRow) -> str:
    """report_row_csv (harness/experiment.hpp:37-46)."""
    cols = [r.case_id, _num(r.p), _num(r.dt), r.precond, _num(r.avg_gmres), _num(r.total_gmres),
            _num(r.newton_steps), _num(r.form_seconds), _num(r.pc_apply_seconds), _num(r.total_seconds),
            _num(r.l2_error) if math.isfinite(r.l2_error) else "", r.status, r.failure_code]
    return ",".join(cols)


def failure_code_for(exc: BaseException) -> str:
    """failure_code_for (harness/experiment.hpp:98-105) over this package's exception classes."""
    from . import ConfigError, ConvergenceError, GmresFailure, SingularError, StateError
    if isinstance(exc, GmresFailure):
        return "gmres_max_iterations"
    if isinstance(exc, StateError):
        return "non_physical_state"
    if isinstance(exc, SingularError):
        return "singular_block"
    if isinstance(exc, ConvergenceError):
        return "nonlinear_divergence"
    if isinstance(exc, ConfigError):
        return "config_error"
    return "internal_error"


def write_report_csv(rows, path):
    """write_report_csv (harness/experiment.hpp:193-198)."""
    with open(path, "w") as f:
        f.write(REPORT_CSV_HEADER + "\n")
        for r in rows:
            f.write(report_row_csv(r) + "\n")


def run_cell(ctx, case, p, tol=1e-10, restart=30, max_iterations=2000, seed=12345, precond="ksvd_full"):
    """One BASELINE cell on the device: formation, then one GMRES solve of a seeded RHS.
    precond: "ksvd_full" (the KSVD preconditioner) or "jacobi_full" (exact block Jacobi)."""
    from . import (GmresConfig, LinearizedOperator, form_block_jacobi, form_ksvd, gmres, setup_advection,
                   uniform_vector)
    if case == "cfg4":
        sysm, dt, name = setup_advection("const3d", 16, 16, 16, p=p, vel=(1.0, 0.7, 0.4)), 0.01, "advection_3d"
    elif case == "cfg1":
        sysm, dt, name = setup_advection("const2d", 8, 8, p=p, vel=(1.0, 0.5, 0.0)), 0.01, "advection_const"
    else:
        sysm, dt, name = setup_advection("swirl2d", 64, 64, p=p), 0.005, "advection_swirl"
    row = ReportRow(case_id=name, p=p, dt=dt, precond=precond)
    t0 = time.perf_counter()
    try:
        op = LinearizedOperator(ctx, sysm, dt)
        ctx.sync()
        tf = time.perf_counter()
        pc = form_block_jacobi(op) if precond == "jacobi_full" else form_ksvd(op)
        ctx.sync()
        row.form_seconds = time.perf_counter() - tf
        b = uniform_vector(seed, sysm.N, 1.0)
        ctx.profile(True)
        res = gmres(op, pc, b, GmresConfig(tol=tol, restart=restart, max_iterations=max_iterations))
        prof = ctx.profile_read()
        ctx.profile(False)
        row.pc_apply_seconds = prof["pc_apply"][0] * 1e-3
        row.gmres_per_solve = [res.iterations]
        row.total_gmres = res.iterations
        row.avg_gmres = float(res.iterations)
        row.newton_steps = 1
    except Exception as exc:  # the reference records the failure and continues the scan
        row.status = "failed"
        row.failure_code = failure_code_for(exc)
    row.total_seconds = time.perf_counter() - t0
    return row


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--case", default="cfg2", choices=["cfg1", "cfg2", "cfg4"])
    ap.add_argument("--p", type=int, nargs="+", default=[4, 8, 15, 20, 30])
    ap.add_argument("--precond", nargs="+", default=["ksvd_full"], choices=["ksvd_full", "jacobi_full"])
    ap.add_argument("--out", default="-")
    a = ap.parse_args(argv)
    from . import Context
    ctx = Context(0)
    rows = [run_cell(ctx, a.case, p, precond=pk) for p in a.p for pk in a.precond]
    if a.out == "-":
        print(REPORT_CSV_HEADER)
        for r in rows:
            print(report_row_csv(r))
    else:
        write_report_csv(rows, a.out)
    return 0 if all(r.status == "ok" for r in rows) else 1


if __name__ == "__main__":
    sys.exit(main())
