"""Jv parity at the exact BASELINE sizes the bench runs (GPU): the full 64x64 cfg2 meshes at
p = 4, 8, 15, 20, 30 (jv2d_mma<5,6> ... <31,32>) and the full 16^3 cfg4 mesh (jv3d_sized<11,12>),
each compared elementwise with the oracle's jacobian_apply (oracle/tpdg_oracle.c, bit-exact to the
reference's ops/linearized.hpp:201-240) on the bench's own seeded RHS. Gate: rel-L2 <= 1e-12
(north star) and max-abs relative to max |y| <= 1e-12."""
import numpy as np
import pytest

import _oracle as O
import paper_1704_04549_b200 as T

pytestmark = pytest.mark.gpu


def oracle_system(s, dt, grid):
    a = s.arrays
    meta = np.array([s.dim, s.n_c, s.p, s.mu, s.n_elements, dt, 0, *grid, 1.0, 1.0])
    arrays = {"meta": meta, "ref_g": a["g"], "ref_d": a["d"], "ref_gw": a["gw"], "ref_dw": a["dw"], "ref_w": a["w"],
              "jdet": a["jdet"], "face_w": a["face_w"], "conn": a["conn"], "dft": a["dft"], "dfm": a["dfm"],
              "dfp": a["dfp"], "start_vec": np.zeros(1)}
    return O.System(arrays)


@pytest.fixture(scope="module")
def ctx():
    return T.Context(0)


def check(ctx, s, dt, grid, label):
    op = T.LinearizedOperator(ctx, s, dt)
    osys = oracle_system(s, dt, grid)
    for seed in (12345, 7):
        b = T.uniform_vector(seed, s.N, 1.0)
        y = op.jacobian_apply(b)
        yr = osys.jv(b)
        rel = O.rel_l2(y, yr)
        mx = float(np.max(np.abs(y - yr)) / np.max(np.abs(yr)))
        print(f"{label} seed {seed}: N = {s.N}, Jv rel-L2 {rel:.3e}, max-abs/max {mx:.3e}")
        assert rel <= 1e-12 and mx <= 1e-12


@pytest.mark.parametrize("p", [4, 8, 15, 20, 30])
def test_cfg2_full_mesh_jv(ctx, p):
    s = T.setup_advection("swirl2d", 64, 64, p=p)
    check(ctx, s, 0.005, (64, 64, 1), f"cfg2 p={p}")


def test_cfg4_full_mesh_jv(ctx):
    s = T.setup_advection("const3d", 16, 16, 16, p=10, vel=(1.0, 0.7, 0.4))
    check(ctx, s, 0.01, (16, 16, 16), "cfg4")


def test_cfg1_jv(ctx):
    s = T.setup_advection("const2d", 8, 8, p=8, vel=(1.0, 0.5, 0.0))
    check(ctx, s, 0.01, (8, 8, 1), "cfg1")
