"""Warm per-launch device times of one solve (events around every launch in
the captured graph).  Prints the launches of the last IR iteration and a
per-FMG-level summary."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_19036_b200 as P
from fmg_inputs import CONFIGS, default_schedule
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
s = P.Solver(cfg["dim"], cfg["p"], cfg["levels"], default_schedule(cfg["dim"], cfg["p"]),
             stream=torch.cuda.current_stream())
s.enable_kernel_timing(4)
for _ in range(3):
    s.solve()
t = s.kernel_times() * 1e3
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); s.solve_async(); e1.record(); torch.cuda.synchronize()
print("solve ms (timed, with events)", e0.elapsed_time(e1), "launches", len(t), "sum of launch us", t.sum())
print("last 40 launches (us):", np.round(t[-40:], 2).tolist())
