"""N4 timing sweep (tools only): ms per batched 1D solve for a few
(p, m, levels, smoother, batch) configurations, CUDA events on the context's
stream, native assembly and loads."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2511_19036_b200 as P

CFGS_ENV = os.environ.get("N4_CFGS")
CFGS = [(1, 1, 16, "lex", 1184), (1, 1, 16, "lex", 2368), (1, 1, 16, "mcgs", 592), (1, 1, 12, "lex", 2368),
        (1, 1, 12, "mcgs", 1184), (3, 1, 10, "lex", 2368), (5, 2, 7, "lex", 2368), (5, 2, 7, "mcgs", 1184)]
if CFGS_ENV:  # "p,m,levels,smoother,batch;..."
    CFGS = [(int(a), int(b), int(c), d, int(e)) for a, b, c, d, e in (x.split(",") for x in CFGS_ENV.split(";"))]
ROWS = {(1, 1): (4, 5, 3), (3, 1): (4, 7, 4), (5, 2): (5, 8, 5)}
st = torch.cuda.Stream()
for p, m, levels, sm, batch in CFGS:
    N, b1, b2 = ROWS[(p, m)]
    s = P.Solver1D(p, m, levels, N, b1, b2, smoother=sm, batch=batch, stream=st)
    s.set_load([P.fmg1d_load(p, m, l) for l in range(levels)])
    s.solve()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(3):
            s.solve_async()
        e1.record(st)
    s.sync()
    ms = e0.elapsed_time(e1) / 3
    n = s.n[-1]
    print(f"p={p} m={m} levels={levels} {sm:4s} batch={batch} n_L={n}: {ms:.3f} ms/solve  "
          f"{batch * n / ms / 1e6:.3f} G DoF/s", flush=True)
    s.close()
