"""K4 phase timestamps (debug build): one solve, print phase deltas of the last K4."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2511_19036_b200 as P
from fmg_inputs import CONFIGS, default_schedule
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
s = P.Solver(cfg["dim"], cfg["p"], cfg["levels"], default_schedule(cfg["dim"], cfg["p"]))
s.solve()
P._lib.fmg_debug_k4(1, None)
s.solve(); s.solve()
buf = np.zeros(64, dtype=np.uint64)
P._lib.fmg_debug_k4.argtypes = [C.c_int, C.c_void_p]
P._lib.fmg_debug_k4(0, buf.ctypes.data)
t = buf.astype(np.int64)
n = int(np.argmax(t == 0)) if (t == 0).any() else 64
print("K4 phases (us):", np.round(np.diff(t[:n]) / 1e3, 2).tolist(), "total", (t[n-1] - t[0]) / 1e3)
