"""Parity of the CUDA path (through the C ABI) against the reference's golden outputs and the oracle.

Tolerances (north star, BASELINE.json):
  * Jv (matrix-free operator): rel-L2 <= 1e-12.
  * Shuffled products, PC apply with the reference's own factors: bit-exact expected (faithful
    kernels, no FMA, reference order); asserted <= 1e-14 / 1e-12 rel-L2.
  * Kronecker blocks P = A1 (x) B1 + A2 (x) B2 formed on the GPU: <= 1e-10 rel-Frobenius.
  * GMRES(30) to 1e-10: identical iteration counts.
"""
import numpy as np
import pytest

import _oracle as O
import paper_1704_04549_b200 as T

pytestmark = pytest.mark.gpu

SMALL = ["cfg1", "cfg2s_p4", "cfg2s_p8", "cfg2s_p15", "pert2d", "adv3d_p3", "adv3d_p4",
         "euler2d", "euler2d_small", "euler3d"]


@pytest.fixture(scope="module")
def ctx():
    return T.Context(0)


_cache = {}


def op_for(ctx, case):
    if case not in _cache:
        z = O.load_raw(case)
        s = T.System.from_golden(z)
        mode = "small" if int(z["meta"][6]) else "full"
        _cache[case] = (z, T.LinearizedOperator(ctx, s, float(z["meta"][5]), block_mode=mode))
    return _cache[case]


def kron_blocks(z_meta, fac, n_c_blk):
    """Dense P of one block from raw factors (2D: a1 b1 a2 b2; 3D: a1 b1 c1 b2 c2)."""
    dim, q = int(z_meta[0]), int(z_meta[2]) + 1
    n1 = n_c_blk * q
    if dim == 2:
        o = 0
        a1 = fac[o:o + n1 * n1].reshape(n1, n1); o += n1 * n1
        b1 = fac[o:o + q * q].reshape(q, q); o += q * q
        a2 = fac[o:o + n1 * n1].reshape(n1, n1); o += n1 * n1
        b2 = fac[o:o + q * q].reshape(q, q)
        return np.kron(a1, b1) + np.kron(a2, b2)
    o = 0
    a1 = fac[o:o + n1 * n1].reshape(n1, n1); o += n1 * n1
    mats = []
    for _ in range(4):
        mats.append(fac[o:o + q * q].reshape(q, q)); o += q * q
    b1, c1, b2, c2 = mats
    return np.kron(a1, np.kron(b1, c1)) + np.kron(a1, np.kron(b2, c2))


@pytest.mark.parametrize("case", SMALL)
def test_jv_matches_reference(ctx, case):
    z, op = op_for(ctx, case)
    out = op.jacobian_apply(z["jv_in"])
    assert O.rel_l2(out, z["jv_out"]) <= 1e-12


@pytest.mark.parametrize("case", SMALL)
def test_shuffled_products_match_reference(ctx, case):
    z, op = op_for(ctx, case)
    comps = int(z["meta"][1]) if op.small else 1
    E = int(z["meta"][4])
    for e in (0, E - 1):
        for c in range(comps):
            t = f"e{e}c{c}"
            av = op.shuffled_apply(e, z[f"shuf_{t}_v"], comp=c)
            atu = op.shuffled_apply(e, z[f"shuf_{t}_u"], transpose=True, comp=c)
            assert O.rel_l2(av, z[f"shuf_{t}_av"]) <= 1e-14, (t, O.rel_l2(av, z[f"shuf_{t}_av"]))
            assert O.rel_l2(atu, z[f"shuf_{t}_atu"]) <= 1e-14


@pytest.mark.parametrize("case", SMALL)
def test_pc_apply_with_reference_factors(ctx, case):
    """Faithful apply: the reference's factors in, the reference's P^{-1} b out."""
    z, op = op_for(ctx, case)
    pc = T.import_factors(op, z["factors"], z["has_factors"])
    assert [f for f in pc.fallbacks] == [tuple(x) for x in z["fallbacks"].reshape(-1, 2)]
    out = pc.apply(z["rhs"])
    assert O.rel_l2(out, z["pc_out"]) <= 1e-12, O.rel_l2(out, z["pc_out"])


@pytest.mark.parametrize("case", SMALL)
def test_form_blocks_and_fallbacks(ctx, case):
    z, op = op_for(ctx, case)
    pc = T.form_ksvd(op)
    assert [f for f in pc.fallbacks] == [tuple(x) for x in z["fallbacks"].reshape(-1, 2)]
    has = z["has_factors"]
    flen = None
    off = 0
    worst = 0.0
    ncb = 1 if op.small else int(z["meta"][1])
    for blk in range(pc.nblk):
        fac, h = pc.factors(blk)
        assert h == bool(has[blk])
        if not h:
            continue
        flen = fac.size
        ref = z["factors"][off:off + flen]
        off += flen
        P = kron_blocks(z["meta"], fac, ncb)
        Pr = kron_blocks(z["meta"], ref, ncb)
        worst = max(worst, np.linalg.norm(P - Pr) / np.linalg.norm(Pr))
    assert worst <= 1e-10, worst


@pytest.mark.parametrize("case", SMALL)
def test_gmres_counts_match_reference(ctx, case):
    z, op = op_for(ctx, case)
    pc = T.form_ksvd(op)
    res = T.gmres(op, pc, z["rhs"], T.GmresConfig(tol=1e-10, restart=30, max_iterations=2000))
    assert res.iterations == int(z["gmres_meta"][0])
    assert res.converged
    # both solutions satisfy ||b - A x|| <= 1e-10 ||b||
    assert O.rel_l2(res.x, z["gmres_x"]) <= 1e-6


@pytest.mark.parametrize("case", SMALL)
def test_pc_apply_formed_on_gpu(ctx, case):
    """End-to-end apply with GPU-formed factors vs the reference: formation (with glibc's libm in
    standardize_2x2, csrc/glibm.cuh) and apply both follow the reference's arithmetic."""
    z, op = op_for(ctx, case)
    pc = T.form_ksvd(op)
    err = O.rel_l2(pc.apply(z["rhs"]), z["pc_out"])
    print(f"{case}: GPU-formed PC apply rel-L2 vs reference = {err:.3e}")
    assert err <= 1e-12


@pytest.mark.parametrize("case", ["cfg1", "cfg2s_p15", "adv3d_p4", "euler2d"])
def test_pc_apply_faithful_path(ctx, case):
    """TPDG_GPU_FAITHFUL=1 (read when a PC is built) selects the order-faithful, FMA-free kernels."""
    import os
    z, op = op_for(ctx, case)
    os.environ["TPDG_GPU_FAITHFUL"] = "1"
    try:
        pc = T.import_factors(op, z["factors"], z["has_factors"])
    finally:
        del os.environ["TPDG_GPU_FAITHFUL"]
    out = pc.apply(z["rhs"])
    assert O.rel_l2(out, z["pc_out"]) <= 1e-12, O.rel_l2(out, z["pc_out"])
    res = T.gmres(op, pc, z["rhs"], T.GmresConfig(tol=1e-10, restart=30, max_iterations=2000))
    assert res.iterations == int(z["gmres_meta"][0])
