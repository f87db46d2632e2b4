"""Experiment: solve time vs number of levels (separates per-launch overhead
from fine-level work).  Prints one line per configuration."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_19036_b200 as P
from fmg_inputs import default_schedule

def run(d, p, levels, reps=10):
    s = P.Solver(d, p, levels, default_schedule(d, p), stream=torch.cuda.current_stream())
    for _ in range(3):
        s.solve_async()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        s.solve_async()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    info = s.info()
    print(f"d={d} p={p} levels={levels:2d} ms={ms:8.3f} launches={int(info['launches_per_solve'])} us/launch={ms*1e3/info['launches_per_solve']:.2f}", flush=True)
    s.close()

for args in [(2, 2, l) for l in range(1, 11)] + [(2, 1, 7)] + [(3, 1, l) for l in range(4, 9)] + [(3, 3, l) for l in range(3, 8)]:
    try:
        run(*args)
    except Exception as e:
        print(args, "failed", e)
