"""The formation's libm restatement (csrc/glibm.cuh: glibc 2.39 sin/cos/atan/atan2, FMA builds), compiled
for the host, against the host libm bit for bit (reference call site tensor/schur.hpp:91-108)."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _glibc_is_pinned():
    out = subprocess.run(["ldd", "--version"], capture_output=True, text=True).stdout
    return "2.39" in out.splitlines()[0] if out else False


@pytest.mark.skipif(not _glibc_is_pinned(), reason="host libm is not glibc 2.39 (the reference's golden build)")
def test_glibm_host_build_matches_libm(tmp_path):
    exe = tmp_path / "glibm_check"
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", os.path.join(HERE, "glibm_check.c"), "-o", str(exe),
                           "-lm"])
    r = subprocess.run([str(exe), "4000000", "7"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    assert "mismatches: sin 0 cos 0 atan 0 atan2 0" in r.stdout
