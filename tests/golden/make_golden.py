"""Regenerate the golden fixtures from the reference itself (run in the build container).

    python tests/golden/make_golden.py [case ...]

Builds oracle/_ref/tpdg_ref_golden (the UNMODIFIED reference headers from
/root/reference compiled in place with the reference's CMake Release flags, see
oracle/Makefile), runs `golden <case>` for every case and packs the dumped
.npy arrays into tests/golden/<case>.npz. The fixtures are committed; the GPU
box never sees /root/reference.
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))

CASES = ["cfg1", "cfg2s_p4", "cfg2s_p8", "cfg2s_p15", "pert2d", "adv3d_p3", "adv3d_p4",
         "euler2d", "euler2d_small", "euler3d",
         # full-size BASELINE configs: fallback decisions + GMRES counts/histories only
         "cfg2_p4", "cfg2_p8", "cfg2_p15", "cfg2_p20", "cfg2_p30", "cfg4",
         # Euler stand-ins of configs[2] / configs[4] (LLF): reduced sizes, then fixed-budget histories at size
         "cfg3s", "cfg5s", "cfg3", "cfg5"]


def main(argv):
    cases = argv or CASES
    subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "ref"])
    exe = os.path.join(ROOT, "oracle", "_ref", "tpdg_ref_golden")
    for case in cases:
        with tempfile.TemporaryDirectory() as tmp:
            subprocess.check_call([exe, "golden", case, tmp])
            arrays = {f[:-4]: np.load(os.path.join(tmp, f)) for f in sorted(os.listdir(tmp)) if f.endswith(".npy")}
        out = os.path.join(HERE, case + ".npz")
        np.savez_compressed(out, **arrays)
        print(f"{case}: {len(arrays)} arrays, {os.path.getsize(out) / 1024:.0f} KiB")


if __name__ == "__main__":
    main(sys.argv[1:])
