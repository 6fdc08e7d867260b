"""build_cache of scalar upwind advection on the device vs the host restatement
(host_setup.cpp, checked bit-exact against the reference's build_cache arrays in the golden tests)."""
import numpy as np
import pytest

import paper_1704_04549_b200 as T

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,args,exact", [("const2d", dict(nx=8, ny=8, p=8, vel=(1.0, 0.5, 0.0)), True),
                                             ("swirl2d", dict(nx=16, ny=16, p=15), False),
                                             ("const3d", dict(nx=4, ny=4, nz=4, p=10, vel=(1.0, 0.7, 0.4)), True)])
def test_device_cache_matches_host(kind, args, exact):
    ctx = T.Context(0)
    s = T.setup_advection(kind, **args)
    dft, dfm, dfp = T.build_advection_cache(ctx, s)
    for name, got in (("dft", dft), ("dfm", dfm), ("dfp", dfp)):
        ref = s.arrays[name]
        if exact:
            assert np.array_equal(got, ref), name
        else:  # CUDA sin / cos vs glibc: <= 1-2 ulp of the velocity
            assert np.max(np.abs(got - ref)) <= 4e-16 * max(1.0, np.max(np.abs(ref))), name
