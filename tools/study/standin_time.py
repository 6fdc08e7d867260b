"""Per-kernel timing of the Euler stand-ins at their configured sizes (cfg3: 32^2 p15 n_c4; cfg5: 8^3 p7 n_c5)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np
import torch
import paper_1704_04549_b200 as T

CASES = (("cfg3", (32, 32, 1), 15, 0.05), ("cfg5", (8, 8, 8), 7, 0.01))
only = sys.argv[1:]  # optional case names
for kind, n, p, dt in CASES:
    if only and kind not in only:
        continue
    ctx = T.Context(0)
    s = T.setup_euler(kind, n[0], n[1], n[2], p=p)
    t0 = time.perf_counter(); T.build_euler_cache(ctx, s); t_cache = time.perf_counter() - t0
    op = T.LinearizedOperator(ctx, s, dt)
    t0 = time.perf_counter(); pc = T.form_ksvd(op); torch.cuda.synchronize(); t_form = time.perf_counter() - t0
    b = T.uniform_vector(12345, s.N, 1e-3)
    db = torch.from_numpy(b).cuda(); dx = torch.zeros_like(db)
    cfg = T.GmresConfig(tol=1e-10, restart=30, max_iterations=40)
    T.gmres_device(op, pc, db, dx, cfg)
    ctx.profile(True); T.gmres_device(op, pc, db, dx, cfg); ctx.profile_read(); ctx.profile(True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    its, conv, _ = T.gmres_device(op, pc, db, dx, cfg)
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    prof = ctx.profile_read()
    print(kind, "N", s.N, "its", its, "GDOF-it/s %.3f" % (s.N * its / t / 1e9), "cache %.3f s form %.3f s" % (t_cache, t_form),
          {k: round(v[0] / max(v[1], 1) * 1e3, 1) for k, v in prof.items()}, flush=True)
