"""Sensitivity of the PC apply to arithmetic order (study tool, GPU): for every golden case, the
apply with the reference's own factors vs the reference's output (rel-L2), and the GMRES count.
Run against variant builds via TPDG_GPU_LIB=... to decide which stages must stay faithful."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import _oracle as O  # noqa: E402
import paper_1704_04549_b200 as T  # noqa: E402

CASES = ["cfg1", "cfg2s_p4", "cfg2s_p8", "cfg2s_p15", "pert2d", "adv3d_p3", "adv3d_p4", "euler2d", "euler2d_small",
         "euler3d"]


def main():
    ctx = T.Context(0)
    out = {}
    for case in CASES:
        z = O.load_raw(case)
        s = T.System.from_golden(z)
        mode = "small" if int(z["meta"][6]) else "full"
        op = T.LinearizedOperator(ctx, s, float(z["meta"][5]), block_mode=mode)
        pc = T.import_factors(op, z["factors"], z["has_factors"])
        err = O.rel_l2(pc.apply(z["rhs"]), z["pc_out"])
        res = T.gmres(op, pc, z["rhs"], T.GmresConfig(tol=1e-10, restart=30, max_iterations=2000))
        out[case] = {"pc_rel": float(f"{err:.3e}"), "its": res.iterations, "ref_its": int(z["gmres_meta"][0])}
    for p in [int(x) for x in os.environ.get("FULL_P", "15").split()]:
        s = T.setup_advection("swirl2d", 64, 64, p=p)
        z = O.load_raw(f"cfg2_p{p}")
        op = T.LinearizedOperator(ctx, s, 0.005)
        pc = T.form_ksvd(op)
        b = T.uniform_vector(12345, s.N, 1.0)
        res = T.gmres(op, pc, b, T.GmresConfig(tol=1e-10, restart=30, max_iterations=2000))
        out[f"cfg2_p{p}"] = {"its": res.iterations, "ref_its": int(z["gmres_meta"][0])}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
