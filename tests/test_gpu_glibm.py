"""Device libm of the KSVD formation (csrc/glibm.cuh through tpdg_gpu_libm_eval) against the host libm
bit for bit on >= 10^7 arguments per function: the ranges standardize_2x2 produces (tensor/schur.hpp:
91-108: theta in [-pi/2, pi], atan2 of arbitrary entry differences/sums, atan of sqrt ratios) plus wide
log-uniform and adversarial arguments (quadrant and table boundaries, tiny, huge, specials)."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import paper_1704_04549_b200 as T

HERE = os.path.dirname(os.path.abspath(__file__))
pytestmark = pytest.mark.gpu
N = 10_000_000


@pytest.fixture(scope="module")
def host_libm(tmp_path_factory):
    so = tmp_path_factory.mktemp("libm") / "libm_batch.so"
    subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", os.path.join(HERE, "libm_batch.c"), "-o", str(so), "-lm"])
    L = C.CDLL(str(so))
    dp = C.POINTER(C.c_double)
    L.libm_batch.argtypes = [C.c_int, C.c_long, dp, dp, dp]

    def run(fn, x, y=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        yy = np.ascontiguousarray(y if y is not None else x, dtype=np.float64)
        L.libm_batch(fn, x.size, x.ctypes.data_as(dp), yy.ctypes.data_as(dp), out.ctypes.data_as(dp))
        return out
    return run


@pytest.fixture(scope="module")
def ctx():
    return T.Context(0)


def _logu(rng, n, emin, emax):
    return np.ldexp(1.0 + rng.random(n), rng.integers(emin, emax + 1, n)) * rng.choice([-1.0, 1.0], n)


def _special():
    v = [0.0, -0.0, 1.0, -1.0, 0.0625, 16.0, float.fromhex("0x1.49ff2p52"), 5e-324, 2.2250738585072014e-308, 1e300, np.inf,
         -np.inf, np.pi, np.pi / 2, np.pi / 4, 0.85546875, 2.426265, 0.126, 1e-8, 3 * np.pi / 4]
    v = np.array(v + [-a for a in v])
    nodes = np.arange(0, 112) / 128.0  # sincos table nodes and their neighbours
    nodes = np.concatenate([nodes, np.nextafter(nodes, 1), np.nextafter(nodes, -1)])
    return np.concatenate([v, nodes, -nodes])


def _bits_equal(a, b):
    return np.count_nonzero(a.view(np.uint64) != b.view(np.uint64))


@pytest.mark.parametrize("fn", ["sin", "cos"])
def test_sincos_bitwise(ctx, host_libm, fn):
    rng = np.random.default_rng(11)
    x = np.concatenate([rng.uniform(-np.pi / 2, np.pi, N // 2), _logu(rng, N // 4, -40, 6),
                        rng.uniform(-1e5, 1e5, N // 4), _special()])
    code = {"sin": 0, "cos": 1}[fn]
    got = T.libm_eval(ctx, fn, x)
    assert _bits_equal(got, host_libm(code, x)) == 0


def test_atan_bitwise(ctx, host_libm):
    rng = np.random.default_rng(12)
    x = np.concatenate([np.sqrt(rng.random(N // 2) * 100.0), _logu(rng, N // 2, -40, 60), _special()])
    assert _bits_equal(T.libm_eval(ctx, "atan", x), host_libm(2, x)) == 0


def test_atan2_bitwise(ctx, host_libm):
    rng = np.random.default_rng(13)
    y = np.concatenate([rng.uniform(-2, 2, N // 4), _logu(rng, N // 4, -40, 40), _logu(rng, N // 4, -1070, 1023),
                        _logu(rng, N // 4, -5, 5)])
    x = np.concatenate([rng.uniform(-2, 2, N // 4), _logu(rng, N // 4, -40, 40), _logu(rng, N // 4, -1070, 1023),
                        y[3 * N // 4:] * rng.uniform(0.9, 1.1, N - 3 * N // 4)])
    s = _special()
    y = np.concatenate([y, np.repeat(s, s.size)])
    x = np.concatenate([x, np.tile(s, s.size)])
    got = T.libm_eval(ctx, "atan2", y, x)
    assert _bits_equal(got, host_libm(3, y, x)) == 0
