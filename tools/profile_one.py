"""One compact-FMG solve of a config (for ncu captures).  Usage:
python tools/profile_one.py C2 [nsolves] [fp32]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_19036_b200 as P
from fmg_inputs import CONFIGS, default_schedule
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
sch = default_schedule(cfg["dim"], cfg["p"])
if len(sys.argv) > 3 and sys.argv[3] == "fp32":  # FP32 cFas (reading R28)
    sch["cfas_fp32"] = 1
s = P.Solver(cfg["dim"], cfg["p"], cfg["levels"], sch)
for _ in range(n):
    s.solve()
print("ok", s.info())
