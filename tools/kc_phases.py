"""KC phase timestamps (debug flag): one solve, phase deltas of the last KC launch."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2511_19036_b200 as P
from fmg_inputs import CONFIGS, default_schedule
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
P._lib.fmg_debug_kc.argtypes = [C.c_int, C.c_void_p]
P._lib.fmg_debug_kc(1, None)  # before the graph is captured
s = P.Solver(cfg["dim"], cfg["p"], cfg["levels"], default_schedule(cfg["dim"], cfg["p"]))
s.solve(); s.solve(); s.solve()
buf = np.zeros(256, dtype=np.uint64)
n = P._lib.fmg_debug_kc(0, buf.ctypes.data)
t = buf[:min(n, 256)].astype(np.int64)
print("KC phases of the last launch:", n, "stamps; deltas (us):", np.round(np.diff(t) / 1e3, 2).tolist(),
      "total", (t[-1] - t[0]) / 1e3)
