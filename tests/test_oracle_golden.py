"""Pin the C oracle (oracle/tpdg_oracle.c) against the reference's own outputs.

The golden fixtures are produced by the unmodified reference compiled in place
(oracle/ref_driver.cpp, tests/golden/make_golden.py). The oracle restates the
reference's summation order and is compiled without FMA contraction, so it is
expected to agree BIT FOR BIT; that is what the tests assert.
"""
import numpy as np
import pytest

import _oracle as O

SMALL = ["cfg1", "cfg2s_p4", "cfg2s_p8", "cfg2s_p15", "pert2d", "adv3d_p3", "adv3d_p4",
         "euler2d", "euler2d_small", "euler3d", "cfg3s", "cfg5s"]


@pytest.fixture(scope="module", params=SMALL)
def sys_(request):
    return O.load(request.param)


def test_rng_restatement(sys_):
    # libstdc++ mt19937_64 + normal_distribution (tensor/lanczos.hpp:61-72)
    assert np.array_equal(O.seeded_unit_vector(len(sys_["start_vec"])), sys_["start_vec"])
    # mt19937_64 + uniform_real_distribution (tests/support/test_rng.hpp:20-25)
    assert np.array_equal(O.uniform_vector(12345, sys_.N, float(sys_["meta"][10])), sys_["rhs"])


def test_jacobian_apply_bit_exact(sys_):
    assert np.array_equal(sys_.jv(sys_["jv_in"]), sys_["jv_out"])


def test_shuffled_products_bit_exact(sys_):
    comps = sys_.n_c if sys_.small else 1
    for e in (0, sys_.n_elements - 1):
        for c in range(comps):
            t = f"e{e}c{c}"
            assert np.array_equal(sys_.shuffled(e, sys_[f"shuf_{t}_v"], comp=c), sys_[f"shuf_{t}_av"])
            assert np.array_equal(sys_.shuffled(e, sys_[f"shuf_{t}_u"], True, comp=c), sys_[f"shuf_{t}_atu"])


def test_assembled_block(sys_):
    if sys_.small:
        pytest.skip("full-mode blocks only in the fixture")
    for e in (0, sys_.n_elements - 1):
        assert np.array_equal(sys_.block(e).ravel(), sys_[f"block_e{e}"])


def test_form_apply_gmres_bit_exact(sys_):
    pc = sys_.form()
    assert np.array_equal(pc.has(), sys_["has_factors"])
    assert np.array_equal(pc.fallbacks().ravel(), sys_["fallbacks"])
    has = pc.has()
    fac = np.concatenate([pc.factors(i) for i in range(pc.nblk) if has[i]])
    assert np.array_equal(fac, sys_["factors"])
    assert np.array_equal(pc.apply(sys_["rhs"]), sys_["pc_out"])
    x, its, hist, conv = pc.gmres(sys_["rhs"])
    assert its == int(sys_["gmres_meta"][0]) and conv
    assert np.array_equal(hist, sys_["gmres_hist"])
    assert np.array_equal(x, sys_["gmres_x"])


def test_kronecker_block_error_is_optimal(sys_):
    """||P - A||_F equals the optimal two-term error for 2D full mode
    (reference tests/unit/test_precond.cpp:155-171)."""
    if sys_.dim != 2 or sys_.small:
        pytest.skip("2D full mode")
    pc = sys_.form()
    q, n1 = sys_.q, sys_.n_c * sys_.q
    for e in (0, sys_.n_elements - 1):
        f = pc.factors(e)
        a1, b1 = f[: n1 * n1].reshape(n1, n1), f[n1 * n1: n1 * n1 + q * q].reshape(q, q)
        a2 = f[n1 * n1 + q * q: 2 * n1 * n1 + q * q].reshape(n1, n1)
        b2 = f[2 * n1 * n1 + q * q:].reshape(q, q)
        P = np.kron(a1, b1) + np.kron(a2, b2)
        A = sys_[f"block_e{e}"].reshape(n1 * q, n1 * q)
        # Van Loan shuffle (tensor/shuffle.hpp:16-25) and its singular values
        At = A.reshape(n1, q, n1, q).transpose(2, 0, 3, 1).reshape(n1 * n1, q * q)
        sv = np.linalg.svd(At, compute_uv=False)
        opt = np.sqrt(np.sum(sv[2:] ** 2))
        assert np.linalg.norm(P - A) <= (1 + 1e-6) * opt + 1e-12 * np.linalg.norm(A)
