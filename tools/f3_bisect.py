"""First (FMG level, IR iteration) where the GPU sections leave the oracle:
python tools/f3_bisect.py d p levels"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2511_19036_b200 as P
from fmg_inputs import default_schedule
d, p, lev = map(int, sys.argv[1:4])
s = O.schedule(d, p)
for L in range(1, lev):
    for it in range(1, s.n_ir + 1):
        oc = O.CFMG(d, p, lev, s)
        oc.solve_upto(L, it)
        gs = P.Solver(d, p, lev, P.Schedule.from_dict(default_schedule(d, p)))
        try:
            gs.solve_upto(L, it)
        except Exception as e:
            print("L", L, "it", it, "ERROR", e, flush=True)
            sys.exit(1)
        bad = []
        for l in range(L + 1):
            for which in (0, 1):
                mo, eo, wo = oc.section(which, l)
                mg, eg, wg = gs.section(which, l)
                if wo != wg or not np.array_equal(eo, eg) or not np.array_equal(mo, mg):
                    bad.append(f"{'ur'[which]}{l}")
        print("L", L, "it", it, "OK" if not bad else "BAD " + " ".join(bad), flush=True)
        if bad:
            sys.exit(1)
