"""Debug helper: locate a failing launch at a 3D config (direct, non-graph run)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_19036_b200 as P
from fmg_inputs import default_schedule
d, p = int(sys.argv[1]), int(sys.argv[2])
for lev in [int(a) for a in sys.argv[3].split(",")]:
    s = P.Solver(d, p, lev, default_schedule(d, p))
    for mode in ("upto", "graph"):
        try:
            if mode == "upto":
                s.solve_upto(lev - 1, 3)
            else:
                s.solve()
            print(d, p, lev, mode, "ok", flush=True)
        except Exception as e:
            print(d, p, lev, mode, "FAIL", e, flush=True)
    s.close()
