"""Per-FMG-level relative errors of the GPU solution at full size (tools only)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_19036_b200 as P
from fmg_inputs import CONFIGS, default_schedule

for cfg in sys.argv[1:]:
    c = CONFIGS[cfg]
    d, p, lv = c["dim"], c["p"], c["levels"]
    s = P.Solver(d, p, lv, default_schedule(d, p))
    prev = None
    for L in range(max(1, lv - 5), lv):
        s.solve_upto(L, s.schedule.n_ir)
        e = s.errors()
        line = f"{cfg} L={L} l2={e[0]:.4e} h1semi={e[1]:.4e}"
        if prev is not None:
            line += f"  log2 ratios l2={math.log2(e[0] / prev[0]):+.3f} h1={math.log2(e[1] / prev[1]):+.3f}"
        print(line, flush=True)
        prev = e
    s.close()
