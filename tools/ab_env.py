"""A/B of env-var settings read at fmg_create (tools only):
   python tools/ab_env.py CFG "FMG_LC=3" "FMG_LC=4" ...
AB_FP32=1: FP32 cFas schedules.  Creates one context per setting in one process, then times them alternately
(CUDA events, no L2 flush), 3 rounds."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2511_19036_b200 as P
from fmg_inputs import CONFIGS, default_schedule

cfg = CONFIGS[sys.argv[1]]
solvers = []
for spec in sys.argv[2:]:
    saved = dict(os.environ)
    for kv in spec.split():
        k, v = kv.split("=", 1)
        os.environ[k] = v
    sch = default_schedule(cfg["dim"], cfg["p"])
    if os.environ.get("AB_FP32") == "1":  # FP32 cFas (reading R28)
        sch["cfas_fp32"] = 1
    s = P.Solver(cfg["dim"], cfg["p"], cfg["levels"], sch)
    s.solve()  # graph captured under this setting
    os.environ.clear()
    os.environ.update(saved)
    solvers.append((spec, s))
n = int(os.environ.get("AB_N", "20"))
res = {spec: [] for spec, _ in solvers}
for _ in range(3):
    for spec, s in solvers:
        for _ in range(3):
            s.solve_async()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            s.solve_async()
        b.record()
        b.synchronize()
        res[spec].append(a.elapsed_time(b) / n)
for spec, v in res.items():
    print(f"{sys.argv[1]} {spec:24s} " + " ".join(f"{x:.4f}" for x in v) + f"  min {min(v):.4f} ms")
