import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2511_19036_b200 as P
from fmg_inputs import default_schedule
d, p, lev = map(int, sys.argv[1:4])
try:
    s = P.Solver(d, p, lev, P.Schedule.from_dict(default_schedule(d, p)))
    s.solve()
    print("ok", os.environ.get("FMG_TMA"), os.environ.get("FMG_TPB"), os.environ.get("FMG_CFS"))
except Exception as e:
    print("FAIL", os.environ.get("FMG_TMA"), os.environ.get("FMG_TPB"), os.environ.get("FMG_CFS"), e)
