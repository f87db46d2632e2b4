"""One C2 solve with nu = 2 (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_19036_b200 as P
from fmg_inputs import CONFIGS, default_schedule
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
s = default_schedule(cfg["dim"], cfg["p"])
s["nu"] = int(sys.argv[2]) if len(sys.argv) > 2 else 2
sv = P.Solver(cfg["dim"], cfg["p"], cfg["levels"], P.Schedule.from_dict(s))
sv.solve()
print("ok")
