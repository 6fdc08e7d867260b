"""CPU-side checks of the drop-in boundary (no GPU needed).

* libtpdg_gpu.so loads and exports every entry point include/tpdg_gpu.h declares;
* the host-side input production (setup_advection) reproduces the reference's arrays bit for bit;
* the host RNG restates libstdc++ exactly (RHS vectors, Lanczos start vectors);
* argument validation maps onto the reference's exception classes.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import _oracle as O
import paper_1704_04549_b200 as T

HEADER = os.path.join(O.ROOT, "include", "tpdg_gpu.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(tpdg_(?:gpu_|setup_|uniform|seeded|halo_plan_)\w*)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(T.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(T.EXPORTS)


def test_version_string():
    assert b"sm_100a" in T.lib().tpdg_gpu_version()


MAP = {"g": "ref_g", "d": "ref_d", "gw": "ref_gw", "dw": "ref_dw", "w": "ref_w", "jdet": "jdet", "face_w": "face_w",
       "conn": "conn", "dft": "dft", "dfm": "dfm", "dfp": "dfp"}


@pytest.mark.parametrize("case,kind,n,p,vel", [
    ("cfg1", "const2d", (8, 8, 1), 8, (1.0, 0.5, 0.0)),
    ("cfg2s_p4", "swirl2d", (8, 8, 1), 4, (0, 0, 0)),
    ("cfg2s_p8", "swirl2d", (4, 4, 1), 8, (0, 0, 0)),
    ("cfg2s_p15", "swirl2d", (2, 2, 1), 15, (0, 0, 0)),
    ("adv3d_p3", "const3d", (2, 2, 2), 3, (1.0, 0.7, 0.4)),
    ("adv3d_p4", "const3d", (3, 3, 3), 4, (1.0, 0.7, 0.4)),
])
def test_setup_matches_reference_bitwise(case, kind, n, p, vel):
    z = O.load_raw(case)
    s = T.setup_advection(kind, n[0], n[1], n[2], p=p, vel=vel)
    for k, g in MAP.items():
        assert np.array_equal(s.arrays[k], z[g]), k


def test_rng_matches_reference():
    z = O.load_raw("cfg1")
    assert np.array_equal(T.uniform_vector(12345, z["rhs"].size), z["rhs"])
    assert np.array_equal(T.seeded_unit_vector(z["start_vec"].size), z["start_vec"])
    z3 = O.load_raw("adv3d_p4")
    assert np.array_equal(T.seeded_unit_vector(z3["start_vec"].size), z3["start_vec"])
    assert np.array_equal(T.seeded_unit_vector(z3["start_vec2"].size), z3["start_vec2"])


def test_setup_validation_raises_config_error():
    with pytest.raises(T.ConfigError):
        T.setup_advection("swirl2d", 0, 4, p=3)
    with pytest.raises(T.ConfigError):
        T.setup_advection("swirl2d", 4, 4, p=0)


def test_partition_covers_all_elements():
    for E in (64, 4096, 4097):
        for N in (1, 2, 3, 8):
            ranges = [T.partition(E, N, r) for r in range(N)]
            assert ranges[0][0] == 0 and ranges[-1][1] == E
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(N - 1))
