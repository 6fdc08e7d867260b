"""Run the oracle's KSVD formation on a full BASELINE configuration with the trig-logging shim
(LD_PRELOAD=/tmp/trig_log.so TRIG_LOG=...). Usage: trig_log_run.py cfg2 15 | cfg4."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
import paper_1704_04549_b200 as T
import _oracle as O
case = sys.argv[1]
if case == "cfg4":
    s, dt, p, dims = T.setup_advection("const3d", 16, 16, 16, p=10, vel=(1.0, 0.7, 0.4)), 0.01, 10, 3
else:
    p = int(sys.argv[2]); s, dt, dims = T.setup_advection("swirl2d", 64, 64, p=p), 0.005, 2
n = s.q ** dims
arrays = {"meta": np.array([dims, 1, p, s.mu, s.n_elements, dt, 0, 0, 0, 1, 1.0, 1.0]),
          "ref_g": s.arrays["g"], "ref_d": s.arrays["d"], "ref_gw": s.arrays["gw"], "ref_dw": s.arrays["dw"],
          "ref_w": s.arrays["w"], "jdet": s.arrays["jdet"], "face_w": s.arrays["face_w"], "conn": s.arrays["conn"],
          "dft": s.arrays["dft"], "dfm": s.arrays["dfm"], "dfp": s.arrays["dfp"]}
if dims == 2:
    arrays["start_vec"] = T.seeded_unit_vector(s.q * s.q)
else:
    arrays["start_vec"] = T.seeded_unit_vector(s.q ** 4)
    arrays["start_vec2"] = T.seeded_unit_vector(s.q * s.q)
osys = O.System(arrays)
pc = osys.form()
print("formed", case, p, "fallbacks", len(pc.fallbacks()))
