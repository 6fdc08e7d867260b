"""Exact block-Jacobi preconditioner on the device (form_block_jacobi, precond/block_jacobi.hpp:38-72),
the paper's comparison baseline: apply vs a dense solve of the oracle's assembled diagonal blocks
(assemble_diag_block(_small), ops/linearized.hpp:245-285), the budget's ConfigError, and GMRES."""
import numpy as np
import pytest

import _oracle as O
import paper_1704_04549_b200 as T

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return T.Context(0)


@pytest.mark.parametrize("case", ["cfg1", "cfg2s_p8", "adv3d_p3", "euler2d", "euler2d_small"])
def test_block_jacobi_apply_and_gmres(ctx, case):
    z = O.load_raw(case)
    osys = O.System(z)
    s = T.System.from_golden(z)
    mode = "small" if int(z["meta"][6]) else "full"
    op = T.LinearizedOperator(ctx, s, float(z["meta"][5]), block_mode=mode)
    pc = T.form_block_jacobi(op)
    assert pc.fallbacks == []
    x = z["rhs"]
    y = pc.apply(x)
    ref = np.empty_like(x)
    nc = osys.n_c if osys.small else 1
    blk = osys.npe if osys.small else osys.n_c * osys.npe
    for e in range(osys.n_elements):
        for c in range(nc):
            o = (e * nc + c) * blk
            ref[o:o + blk] = np.linalg.solve(osys.block(e, c), x[o:o + blk])
    err = O.rel_l2(y, ref)
    print(f"{case}: block-Jacobi apply rel-L2 vs dense solve {err:.2e}")
    assert err <= 1e-12
    res = T.gmres(op, pc, x, T.GmresConfig(tol=1e-10, restart=30, max_iterations=2000))
    assert res.converged
    assert res.iterations <= int(z["gmres_meta"][0]) + 2  # exact block inverse: no worse than the KSVD


def test_block_jacobi_budget(ctx):
    z = O.load_raw("cfg1")
    op = T.LinearizedOperator(ctx, T.System.from_golden(z), float(z["meta"][5]))
    with pytest.raises(T.ConfigError):
        T.form_block_jacobi(op, max_total_entries=1000)


def test_blocked_dense_lu_is_bit_identical():
    """The panel-blocked dense LU (default) gives the same factors as the unblocked kernel: block-Jacobi applies of
    golden cases compared bit for bit between two processes (TPDG_GPU_DENSE_LU is read once per process)."""
    import json
    import os
    import subprocess
    import sys
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for mode in ("", "unblocked"):
        fd, path = tempfile.mkstemp(suffix=".json")
        os.close(fd)
        env = dict(os.environ, TPDG_GPU_DENSE_LU=mode)
        r = subprocess.run([sys.executable, os.path.join(root, "tools", "dense_lu_compare.py"), path], env=env,
                           cwd=root, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.load(open(path)))
        os.unlink(path)
    for case in outs[0]:
        assert np.array_equal(np.array(outs[0][case]), np.array(outs[1][case])), case
