"""Bit-identity check of the blocked dense LU (GPU study tool): block-Jacobi applies of golden cases, written as
JSON; run once with TPDG_GPU_DENSE_LU=unblocked and compare (tests/ and DESIGN.md cite the result)."""
import os, sys, json
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import _oracle as O
import paper_1704_04549_b200 as T
ctx = T.Context(0)
out = {}
for case in ["cfg1", "cfg2s_p8", "cfg2s_p15", "euler2d", "adv3d_p4"]:
    z = O.load_raw(case)
    s = T.System.from_golden(z)
    mode = "small" if int(z["meta"][6]) else "full"
    op = T.LinearizedOperator(ctx, s, float(z["meta"][5]), block_mode=mode)
    pc = T.form_block_jacobi(op)
    out[case] = pc.apply(z["rhs"]).tolist()
json.dump(out, open(sys.argv[1], "w"))
