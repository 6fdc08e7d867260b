"""The multi-rank GMRES orthogonalization code path (one fused w-update + partial-dot kernel and one
allreduce per MGS pass, capi.cu) exercised on one GPU: TPDG_GPU_MULTI_MGS=1 selects it with a
single rank (the allreduce is then the identity), and the iteration counts must still be the
reference's. The NCCL exchange itself needs >= 2 GPUs; its host-side plan and the distributed
arithmetic are covered by tests/test_multirank_cpu.py (gloo, world_size 2)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import _oracle as O
import paper_1704_04549_b200 as T
ctx = T.Context(0)
out = {{}}
for case in ["cfg1", "cfg2s_p8", "cfg2s_p15", "adv3d_p3", "euler2d"]:
    z = O.load_raw(case)
    s = T.System.from_golden(z)
    mode = "small" if int(z["meta"][6]) else "full"
    op = T.LinearizedOperator(ctx, s, float(z["meta"][5]), block_mode=mode)
    pc = T.import_factors(op, z["factors"], z["has_factors"])
    res = T.gmres(op, pc, z["rhs"], T.GmresConfig(tol=1e-10, restart=30, max_iterations=2000))
    out[case] = [res.iterations, int(z["gmres_meta"][0]), O.rel_l2(res.x, z["gmres_x"])]
s = T.setup_advection("swirl2d", 64, 64, p=15)
op = T.LinearizedOperator(ctx, s, 0.005)
res = T.gmres(op, T.form_ksvd(op), T.uniform_vector(12345, s.N, 1.0), T.GmresConfig(tol=1e-10, restart=30))
out["cfg2_p15"] = [res.iterations, 25, 0.0]
print(json.dumps(out))
"""


def test_multi_rank_mgs_path_single_gpu():
    env = dict(os.environ, TPDG_GPU_MULTI_MGS="1")
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    print(out)
    for case, (its, ref, xerr) in out.items():
        assert its == ref, (case, its, ref)
        assert xerr <= 1e-6, (case, xerr)
