"""Multi-rank data plane on ONE GPU (in-process transport, tpdg_gpu_ctx_create_loopback): each rank is a
host thread with its own context, stream and operator over its element rows / slabs; the halo moves
only the face node layers (n_c q^(d-1) doubles per cut face, the rest of every halo block is NaN) on a
separate stream while the interior elements run, and the GMRES dots are all-reduced (fixed rank order).

Gates: the distributed Jv equals the single-rank Jv bit for bit, the
element-local preconditioner apply likewise, and distributed GMRES takes the reference's iteration
count. The same code path runs over NCCL when the contexts are created with an ncclUniqueId."""
import threading

import numpy as np
import pytest

import _oracle as O
import paper_1704_04549_b200 as T

pytestmark = pytest.mark.gpu


def run_ranks(nranks, fn):
    hub = T.Loopback(nranks)
    out, errs = [None] * nranks, []

    def work(r):
        try:
            ctx = T.Context(0, r, loopback=hub)
            out[r] = fn(ctx, r)
            ctx.close()
        except Exception as e:  # surfaced in the main thread
            errs.append((r, repr(e)))

    th = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    hub.close()
    assert not errs, errs
    return out


CASES = [  # (name, system builder, dt, reference GMRES count or golden case, ranks)
    ("cfg2_p8", lambda: T.setup_advection("swirl2d", 64, 64, p=8), 0.005, 18, 2),
    ("cfg2_p15", lambda: T.setup_advection("swirl2d", 64, 64, p=15), 0.005, 25, 4),
    ("cfg4", lambda: T.setup_advection("const3d", 16, 16, 16, p=10, vel=(1.0, 0.7, 0.4)), 0.01, 159, 2),
]


@pytest.mark.parametrize("name,build,dt,ref_its,nranks", CASES, ids=[c[0] for c in CASES])
def test_loopback_jv_pc_gmres(name, build, dt, ref_its, nranks):
    s = build()
    b = T.uniform_vector(12345, s.N, 1.0)
    ctx1 = T.Context(0)
    op1 = T.LinearizedOperator(ctx1, s, dt)
    jv_ref = op1.jacobian_apply(b)
    pc1 = T.form_ksvd(op1)
    pc_ref = pc1.apply(b)
    blk = s.n_c * s.npe

    def rank_fn(ctx, r):
        op = T.LinearizedOperator(ctx, s, dt)
        lo, hi = op.e_begin * blk, op.e_end * blk
        jv = op.jacobian_apply(b[lo:hi])
        pc = T.form_ksvd(op)
        pa = pc.apply(b[lo:hi])
        res = T.gmres(op, pc, b[lo:hi], T.GmresConfig(tol=1e-10, restart=30, max_iterations=2000))
        return lo, hi, jv, pa, res.iterations, res.converged

    res = run_ranks(nranks, rank_fn)
    its = set()
    for lo, hi, jv, pa, n_its, conv in res:
        assert np.array_equal(jv, jv_ref[lo:hi]), f"{name}: distributed Jv differs from the single-rank Jv"
        assert np.array_equal(pa, pc_ref[lo:hi]), f"{name}: element-local PC apply differs"
        assert conv
        its.add(n_its)
    print(f"{name}: {nranks} ranks, GMRES iterations {sorted(its)} (reference {ref_its})")
    assert its == {ref_its}


@pytest.mark.parametrize("case,nranks", [("euler2d", 2), ("euler2d_small", 2), ("adv3d_p4", 2), ("euler3d", 2),
                                          ("cfg1", 3), ("cfg2s_p8", 2)])
def test_loopback_golden_cases(case, nranks):
    """Small golden cases (n_c = 4 / 5, small block mode, 3D, 3 ranks): distributed Jv within 1e-12 of the
    reference's, and distributed GMRES with the reference's own factors (import_factors, element-local)
    taking the reference's iteration count."""
    z = O.load_raw(case)
    s = T.System.from_golden(z)
    dt = float(z["meta"][5])
    mode = "small" if int(z["meta"][6]) else "full"
    blk = s.n_c * s.npe
    nb_per_elem = s.n_c if mode == "small" else 1
    flen = z["factors"].size // max(1, int(np.sum(z["has_factors"])))

    def rank_fn(ctx, r):
        op = T.LinearizedOperator(ctx, s, dt, block_mode=mode)
        lo, hi = op.e_begin * blk, op.e_end * blk
        jv = op.jacobian_apply(z["jv_in"][lo:hi])
        has = z["has_factors"][op.e_begin * nb_per_elem:op.e_end * nb_per_elem]
        first = int(np.sum(z["has_factors"][:op.e_begin * nb_per_elem]))
        fac = z["factors"][first * flen:(first + int(np.sum(has))) * flen]
        pc = T.import_factors(op, fac, has)
        res = T.gmres(op, pc, z["rhs"][lo:hi], T.GmresConfig(tol=1e-10, restart=30, max_iterations=2000))
        return lo, hi, jv, res.iterations, res.converged

    for lo, hi, jv, its, conv in run_ranks(nranks, rank_fn):
        assert O.rel_l2(jv, z["jv_out"][lo:hi]) <= 1e-12
        assert conv and its == int(z["gmres_meta"][0]), (its, int(z["gmres_meta"][0]))
