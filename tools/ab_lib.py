"""A/B timing of libfmg.so builds (tools only): python tools/ab_lib.py CFG lib1.so [lib2.so ...]
Times fmg_solve_async of config CFG with CUDA events (no L2 flush), each lib
in turn, 3 rounds; the libraries are loaded side by side with ctypes."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_19036_b200 as P
from fmg_inputs import CONFIGS, default_schedule

cfg = CONFIGS[sys.argv[1]]
libs = []
for path in sys.argv[2:]:
    L = C.CDLL(os.path.abspath(path), mode=C.RTLD_LOCAL)
    L.fmg_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    L.fmg_solve_async.argtypes = [C.c_void_p]
    libs.append((path, L))
sched = P.Schedule.from_dict(default_schedule(cfg["dim"], cfg["p"]))
st = torch.cuda.Stream()
ctxs = []
for path, L in libs:
    h = C.c_void_p()
    rc = L.fmg_create(cfg["dim"], cfg["p"], cfg["levels"], C.byref(sched), C.c_void_p(st.cuda_stream), C.byref(h))
    assert rc == 0, (path, rc)
    ctxs.append(h)
res = {p: [] for p, _ in libs}
for rnd in range(3):
    for (path, L), h in zip(libs, ctxs):
        with torch.cuda.stream(st):
            for _ in range(3):
                L.fmg_solve_async(h)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(int(os.environ.get("AB_N", "20"))):
                L.fmg_solve_async(h)
            b.record(st)
        st.synchronize()
        res[path].append(a.elapsed_time(b) / int(os.environ.get("AB_N", "20")))
for p, v in res.items():
    print(f"{p}: " + " ".join(f"{x:.4f}" for x in v) + f"  min {min(v):.4f} ms")
