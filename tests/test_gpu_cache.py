"""build_cache of scalar upwind advection on the device vs the host restatement
(host_setup.cpp, checked bit-exact against the reference's build_cache arrays in the golden tests)."""
import numpy as np
import pytest

import paper_1704_04549_b200 as T

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,args", [("const2d", dict(nx=8, ny=8, p=8, vel=(1.0, 0.5, 0.0))),
                                       ("swirl2d", dict(nx=16, ny=16, p=15)), ("swirl2d", dict(nx=64, ny=64, p=15)),
                                       ("const3d", dict(nx=4, ny=4, nz=4, p=10, vel=(1.0, 0.7, 0.4)))])
def test_device_cache_matches_host(kind, args):
    ctx = T.Context(0)
    s = T.setup_advection(kind, **args)
    dft, dfm, dfp = T.build_advection_cache(ctx, s)
    for name, got in (("dft", dft), ("dfm", dfm), ("dfp", dfp)):
        ref = s.arrays[name]
        # the swirl field's sin / cos run in glibc's arithmetic on the device (csrc/glibm.cuh)
        assert np.array_equal(got, ref), name
