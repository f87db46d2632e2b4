"""Quick fine3 parity probe: python tools/f3_check.py [d p levels]..."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import oracle as O
import paper_2511_19036_b200 as P
from fmg_inputs import default_schedule

cases = [(3, 1, 3), (3, 2, 3), (3, 3, 3), (3, 1, 5), (3, 2, 4), (3, 3, 4)]
if len(sys.argv) > 1:
    a = list(map(int, sys.argv[1:]))
    cases = [tuple(a[i:i + 3]) for i in range(0, len(a), 3)]
for d, p, lev in cases:
    oc = O.CFMG(d, p, lev, O.schedule(d, p))
    oc.solve()
    gs = P.Solver(d, p, lev, P.Schedule.from_dict(default_schedule(d, p)))
    t0 = time.time()
    gs.solve()
    torch.cuda.synchronize()
    ok = True
    no, ng = oc.norms(), gs.norms()
    m = no != 0
    rel = np.abs(ng[m] - no[m]) / no[m] if m.any() else np.zeros(1)
    msg = [f"norm rel max {rel.max():.2e}"]
    for l in range(lev):
        for which in (0, 1):
            mo, eo, wo = oc.section(which, l)
            mg, eg, wg = gs.section(which, l)
            if wo != wg or not np.array_equal(eo, eg) or not np.array_equal(mo, mg):
                ok = False
                nb = len(eo)
                bad = np.nonzero(eo != eg)[0]
                msg.append(f"{'ur'[which]}{l}: w {wo}/{wg} exps bad {len(bad)}/{nb} first {bad[:5]}")
    print(d, p, lev, "OK" if ok and rel.max() <= 1e-6 else "FAIL", "; ".join(msg), f"{time.time()-t0:.2f}s", flush=True)
