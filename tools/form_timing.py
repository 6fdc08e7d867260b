"""KSVD formation wall time at cfg2 p=15 (GPU study tool): with / without releasing the previous PC first."""
import time, sys
sys.path.insert(0, ".")
import torch
import paper_1704_04549_b200 as T
torch.cuda.set_device(0)
ctx = T.Context(0)
s = T.setup_advection("swirl2d", 64, 64, p=15)
op = T.LinearizedOperator(ctx, s, 0.005)
pc = T.form_ksvd(op)
for mode in ["noclose", "close", "close_sync"]:
    ts = []
    for i in range(3):
        if mode != "noclose": pc.close()
        if mode == "close_sync": torch.cuda.synchronize(); time.sleep(0.05)
        torch.cuda.synchronize()
        t0 = time.perf_counter(); pc = T.form_ksvd(op); torch.cuda.synchronize(); ts.append(round((time.perf_counter() - t0) * 1e3, 1))
    print(mode, ts)
