"""bench.py -- compact-FMG solve throughput on B200 (BASELINE.json metric).

One step = one full compact FMG solve (Alg 3.3, all FMG levels, N IR
iterations each: every §8(a) row S1-S11) of the configured workload, issued
through the C-ABI (fmg_solve_async) with the context resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

Default workload: C4 (3D Q3, 256^3 elements, 8-level FMG), the largest
configuration that runs on one GPU (BASELINE.json configs[3]; C5 needs 8).
Multi-GPU: 3D configs run ONE problem in z slabs over the ranks (NCCL halo
exchange, strong scaling); 2D configs do not shard (replicas
only), so each rank solves its own instance (weak).
--impl reference: the CPU oracle (oracle/, plain sequential C) on the same
config, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from fmg_inputs import CONFIGS, default_schedule, unknowns  # noqa: E402

METRIC = "FMG solve DoF/s and effective HBM GB/s vs 8 TB/s roofline at 1/2/4/8 B200"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_PEAK_TFLOPS = 37.2  # 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz; measured 34.0
FP32_PEAK_TFLOPS = 74.4  # 148 SMs x 128 FFMA/clk x 2 x 1.965 GHz (the FP32 cFas lines, reading R28)


def peaks():
    try:
        with open(PEAKS_FILE) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6536.7), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """Samples SM clock and throttle reasons through NVML every 5 ms during the
    timed region (nvidia-smi's 200 ms period is longer than a C2 step)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.stop_ev = threading.Event()
        self.th = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def loop():
                while not self.stop_ev.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((sm, rs))
                    except Exception:
                        pass
                    time.sleep(0.005)

            self.th = threading.Thread(target=loop, daemon=True)
            self.th.start()
        except Exception:
            self.th = None

    def stop(self):
        self.stop_ev.set()
        if self.th:
            self.th.join(timeout=1)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        reasons = set()
        for _, rs in self.samples:
            for nm, bit in self.REASONS.items():
                if rs & bit:
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def reduce_max(value: float, device=None) -> float:
    """Max of a per-rank scalar over all ranks (timings are max-over-ranks);
    identity without an initialised process group."""
    import torch
    import torch.distributed as tdist
    if not (tdist.is_available() and tdist.is_initialized()) or tdist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return float(t.item())


def aggregate(unknowns_per_rank: int, world: int, ms_max: float) -> float:
    """Whole-job DoF/s: every rank solves its own replica (2D configs do not
    shard), timed by the slowest rank."""
    return unknowns_per_rank * world / (ms_max * 1e-3)


def kernel_model(cfg, sched, cls):
    """Algorithmic work of one launch of the roofline kernel,
    counted per stored point of the finest level at the finest FMG level:

    * flops: FP64 operations of the canonical expression trees (
      an FMA counts 2), halo recompute and the codec's integer work excluded;
    * section bytes: only the compact sections the launch must
      read or write at their widths at FMG level L = Lmax, plus one int8
      exponent per 32-entry block.  FP64 temporaries are not algorithmic
      bytes: §8(d) defines them as on-chip values.
    Returns (flops, section_bytes)."""
    d, p, levels = cfg["dim"], cfg["p"], cfg["levels"]
    n = p << levels
    NX = (n + 31) // 32 * 32
    pts = NX * n * (n if d == 3 else 1)
    t = 2 * p + 1
    a_flops = (8 * t + 1) if d == 2 else (14 * t + 2)   # canonical A tree, FMA = 2 flops
    wr_b = sched["b_r"] / 8 + 1 / 32
    wu_b = sched["b_u"] / 8 + 1 / 32
    if cls == 0:   # residual: t_L = f - A u_L (f = ((C g) g) g), r_L = enc(t_L) written
        flops = a_flops + (d - 1) + 2
        byts = wr_b
    else:          # cls 5: last Chebyshev step (finalise) at the finest level:
        # y_1 = inv_theta invD b (2), A y_1, q, d, y (5), correction (2 adds); ú_L read + written
        flops = 2 + a_flops + 5 + 2
        byts = 2 * wu_b
    return flops * pts, byts * pts


KERNEL_LABEL = {(2, 0): "k_m_residual (fine level)", (3, 0): "k_f3_staged / k_f3_residual (fine level)",
                (2, 5): "k_m_cheb final step (fine level)",
                (3, 5): "last Chebyshev step (k_f3_staged2<3, 4> at p = 3, k_f3_cheb at p = 1) + k_f3_tpb<1> "
                        "finalisation (fine level)"}


def roofline_entry(cfg, sched, args, avg_launch_ms, launches, hbm, hbm_src):
    """The contract's roofline object for the fine-level roofline kernel.  The
    binding roof is the larger of the two model times: FP64 flops at the
    derived FP64 peak (the 3D configs: "alu") or the §8(d) section bytes at
    the measured HBM copy bandwidth."""
    flops, byts = kernel_model(cfg, sched, args.roofline_class)
    t_hbm = byts / (hbm * 1e9)
    t_alu = flops / (FP64_PEAK_TFLOPS * 1e12)
    sec = avg_launch_ms * 1e-3
    if t_alu >= t_hbm and sched.get("cfas_fp32") and args.roofline_class == 5:
        # FP32 cFas: the Chebyshev step's arithmetic is float (the correction's 2 adds excepted)
        roof = {"bound": "alu", "achieved": flops / sec / 1e12, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                "peak_source": "derived FP32: 148 SMs x 128 FFMA/clk x 2 x 1.965 GHz (DESIGN.md §7)"}
    elif t_alu >= t_hbm:
        roof = {"bound": "alu", "achieved": flops / sec / 1e12, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "peak_source": "derived FP64: 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz (DESIGN.md §7; "
                               "tools/fp64_peak.cu measured 34.0)"}
    else:
        roof = {"bound": "hbm", "achieved": byts / sec / 1e9, "peak": hbm, "unit": "GB/s",
                "peak_source": hbm_src}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["hbm_section_frac"] = byts / sec / 1e9 / hbm
    roof["traffic"] = args.traffic
    if args.traffic is None and args.smoother == "chebyshev" and args.nu == 1 and not sched.get("cfas_fp32"):
        # the committed ncu capture of this kernel (profiles/traffic.json)
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
                t = json.load(fh)[args.config][str(args.roofline_class)]
            roof["traffic"] = t["bytes"]
            roof["traffic_source"] = t["source"]
            if "fp64_pipe_pct" in t:
                roof["fp64_pipe_frac_ncu"] = t["fp64_pipe_pct"] / 100.0
        except (OSError, KeyError, ValueError):
            pass
    label = KERNEL_LABEL[(cfg["dim"], args.roofline_class)]
    if cfg["dim"] == 3 and (args.smoother == "mcgs" or args.nu > 1):  # (level-by-level kernels, fmg_march3.cu)
        label = {0: "k_m3_residual (fine level)", 5: "k_m3_cheb final step (fine level)"}.get(args.roofline_class, label)
    if args.smoother == "mcgs" and args.roofline_class == 5:
        label = label.replace("cheb final step", "gs final colour step")
    roof["kernel"] = label
    roof["avg_launch_ms"] = avg_launch_ms
    roof["launches_timed"] = launches
    roof["alg_flops_per_launch"] = flops
    roof["section_bytes_per_launch"] = byts
    return roof


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2511_19036_b200 as P

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = CONFIGS[args.config]
    sched = default_schedule(cfg["dim"], cfg["p"])
    sched["smoother"] = {"chebyshev": 0, "mcgs": 1}[args.smoother]
    sched["nu"] = args.nu
    sched["cfas_fp32"] = int(args.cfas_fp32)
    P.use_torch_allocator(True)
    stream = torch.cuda.current_stream()
    dist_slabs = world > 1 and cfg["dim"] == 3  # 3D: one problem in z slabs over the ranks (NCCL)
    if dist_slabs:
        import torch.distributed as tdist
        uid = [P.nccl_unique_id() if rank == 0 else None]
        tdist.broadcast_object_list(uid, src=0)
        solver = P.Solver(cfg["dim"], cfg["p"], cfg["levels"], sched, stream=stream, dist=(rank, world, uid[0]))
    else:
        solver = P.Solver(cfg["dim"], cfg["p"], cfg["levels"], sched, stream=stream)
    info_unk = unknowns(cfg["dim"], cfg["p"], cfg["levels"])

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    for _ in range(args.warmup):
        solver.solve_async()
    torch.cuda.synchronize()
    solver.solve()  # error check (FMG_ERANGE) once before timing
    info = solver.info()
    exp_ref = torch.empty(solver.export_size(), dtype=torch.uint8).pin_memory()
    solver.export_solution(exp_ref)
    stream.synchronize()

    dist = world > 1
    if dist:
        import torch.distributed as tdist
    clocks = Clocks(local_rank)
    clocks.start()
    times = []
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        solver.solve_async()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    if dist:
        tdist.barrier()
    ck = clocks.stop()
    ms = reduce_max(sum(times) / len(times), dev)
    # every repeat is bit-identical: the compact solution after
    # the timed solves equals the one before them, byte for byte
    exp_chk = torch.empty_like(exp_ref)
    solver.export_solution(exp_chk)
    stream.synchronize()
    repeat_identical = bool(torch.equal(exp_ref, exp_chk))

    # ---- roofline kernel: CUDA events around each launch of its class, in a
    # separate graph and OUTSIDE the timed region above (the events would
    # otherwise sit inside the timed solves)
    solver.enable_kernel_timing(args.roofline_class)
    ktimes, klaunch = 0.0, 0
    for _ in range(max(2, min(args.steps, 5))):
        flush.zero_()
        solver.solve_async()
        kt, kn = solver.kernel_time()
        ktimes += kt
        klaunch += kn
    solver.enable_kernel_timing(-1)

    # ---- end to end through the C-ABI with host buffers --------------------
    rhs_host = torch.from_numpy(solver.get_rhs()).pin_memory()
    exp_host = torch.empty(solver.export_size(), dtype=torch.uint8).pin_memory()
    e2e_times = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        solver.set_rhs(rhs_host)            # H2D: the separable RHS tables
        solver.solve_async()
        solver.export_solution(exp_host)    # D2H: every compact solution section
        stream.synchronize()
        e2e_times.append((time.perf_counter() - t0) * 1e3)
    e2e_ms = reduce_max(sum(e2e_times) / len(e2e_times), dev)

    if rank != 0:
        return
    hbm, hbm_src = peaks()
    avg_launch_ms = ktimes / max(klaunch, 1)
    roof = roofline_entry(cfg, sched, args, avg_launch_ms, klaunch, hbm, hbm_src)

    eff_gbs = info["alg_bytes_per_solve"] / (ms * 1e-3) / 1e9
    nrep = 1 if dist_slabs else world  # slabs: one problem on all ranks (strong); else replicas (weak)
    out = {
        "metric": METRIC,
        "value": aggregate(info_unk, nrep, ms),
        "unit": "DoF/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong" if dist_slabs else "weak",
        "vs_baseline": None,
        "dtype": "f64 (cFas f32)" if args.cfas_fp32 else "f64",
        "data": "synthetic (manufactured solution u = prod sin(pi x_k); no dataset)",
        "config": {"workload": args.config + ": " + cfg["desc"], "dim": cfg["dim"], "p": cfg["p"],
                   "levels": cfg["levels"], "unknowns": info_unk,
                   "schedule": sched, "l2": "flushed (256 MB write) before every timed step",
                   "parallelism": (f"z slabs x{world} (NCCL halo exchange)" if dist_slabs else
                                   f"replicas x{world}" if world > 1 else "single GPU")},
        "effective_hbm_gbs": eff_gbs,
        "hbm_roofline_frac_nominal_8tbs": eff_gbs / 8000.0,
        "hbm_roofline_frac_measured": eff_gbs / hbm,
        "alg_bytes_per_solve": info["alg_bytes_per_solve"],
        "roofline": roof,
        "e2e": {"value": aggregate(info_unk, nrep, e2e_ms), "unit": "DoF/s",
                "h2d_bytes_per_step": rhs_host.numel() * 8, "d2h_bytes_per_step": exp_host.numel(),
                "ms_per_step": e2e_ms},
        "gpu_launches": int(info["launches_per_solve"]) * args.steps,
        "repeat_bit_identical": repeat_identical,
        "device_bytes": solver.device_bytes(),
        "clocks": ck,
    }
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.config, args.smoother, args.nu, int(args.cfas_fp32))
    print(json.dumps(out))


# ------------------------------------------------------------------ N4 --
# the paper's 1D B-spline workloads (include/fmg1d.h), a
# batch of independent problems per launch (one CTA per problem).  Default:
# 1D Poisson, p = 1, Table 3's row (N = 4, b1 = 5, b2 = 3),
# L = 15 (n_L = 65535, inside FP64's range b3 + (p+m+1) L <= 53), the paper's
# lexicographic Gauss-Seidel, batch 4736 = 32 problems per SM (one warp
# each).
N4_ROWS = {(1, 1): (4, 5, 3), (2, 1): (3, 5, 4), (3, 1): (4, 7, 4), (4, 1): (5, 8, 4), (5, 1): (9, 9, 5),
           (3, 2): (6, 4, 4), (4, 2): (4, 6, 4), (5, 2): (5, 8, 5), (6, 2): (5, 11, 5), (7, 2): (11, 12, 6)}


def n4_alg_bytes(p, m, levels, N, b1, b2):
    """Algorithmic bytes of one 1D solve: per IR iteration at
    FMG level L, f_L (8 B/DoF) plus, per level l <= L, the compact sections the
    method reads and writes -- u_l read twice (standard form, correction) and
    written once, r_l written and read, y_l written and read twice (cFas,
    correction): (3 w_u + 5 w_r) / 8 B/DoF -- and the final solution (8 B/DoF)."""
    n = [(1 << (l + 1)) + p - 2 * m for l in range(levels)]
    tot = 0.0
    for L in range(1, levels):
        per_it = 8 * n[L] + sum(n[l] * (3 * (b1 + (p + 1) * (L - l)) + 5 * (b2 + m * (L - l))) / 8
                                for l in range(L + 1))
        tot += N * per_it
    return tot + 8 * n[-1]


def run_n4(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_2511_19036_b200 as P

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    p, m, levels, batch = args.n4_p, args.n4_m, args.n4_levels, args.n4_batch
    if batch is None:  # fill the resident problems once: 32 per SM
        # with one warp per problem, 4 per SM with a 256-thread CTA per problem
        warp_per_problem = args.n4_smoother == "lex" or (1 << levels) + p - 2 * m <= 2048
        batch = 148 * (32 if warp_per_problem else 4)
    N, b1, b2 = N4_ROWS[(p, m)]
    stream = torch.cuda.current_stream()
    s = P.Solver1D(p, m, levels, N, b1, b2, smoother=args.n4_smoother, batch=batch, stream=stream)
    loads = [P.fmg1d_load(p, m, l) for l in range(levels)]
    # distinct problems: problem b solves with load (1 + b / batch) f
    scale = 1.0 + np.arange(batch)[:, None] / batch
    fb = [np.ascontiguousarray(scale * v[None, :]) for v in loads]
    s.set_load(fb)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        s.solve_async()
    s.sync()
    dist = world > 1
    if dist:
        import torch.distributed as tdist
        tdist.barrier()
    clocks = Clocks(local_rank)
    clocks.start()
    times = []
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s.solve_async()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    s.sync()
    if dist:
        tdist.barrier()
    ck = clocks.stop()
    ms = reduce_max(sum(times) / len(times), dev)
    # end to end: pinned host loads in, host solutions out, every step
    fpin = [torch.from_numpy(v).pin_memory() for v in fb]
    fnp = [t.numpy() for t in fpin]
    upin = torch.empty((batch, s.n[-1]), dtype=torch.float64).pin_memory()
    e2e = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.solve_host(fnp, upin.numpy())
        e2e.append((time.perf_counter() - t0) * 1e3)
    e2e_ms = reduce_max(sum(e2e) / len(e2e), dev)
    if rank != 0:
        return
    hbm, hbm_src = peaks()
    byts = n4_alg_bytes(p, m, levels, N, b1, b2) * batch
    unk = s.n[-1] * batch
    roof = {"bound": "hbm", "achieved": byts / (ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
            "peak_source": hbm_src, "traffic": args.traffic,
            "kernel": f"k_fmg1d<{p}> (the whole batched solve is one launch)",
            "avg_launch_ms": ms, "alg_bytes_per_launch": byts,
            "note": "compact-section bytes only (DESIGN.md §12); the lexicographic sweep is a "
                    "sequential latency chain per problem, so the fraction is low by construction"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    out = {
        "metric": METRIC,
        "value": unk * world / (ms * 1e-3),
        "unit": "DoF/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (the paper's manufactured 1D problems, loads scaled per problem; no dataset)",
        "config": {"workload": f"N4: 1D {'Poisson' if m == 1 else 'biharmonic'} B-spline p={p}, "
                               f"{levels} levels, batch {batch}, {args.n4_smoother} GS",
                   "p": p, "m": m, "levels": levels, "batch": batch, "unknowns_per_problem": s.n[-1],
                   "schedule": {"N": N, "b1": b1, "b2": b2, "smoother": args.n4_smoother},
                   "l2": "flushed (256 MB write) before every timed step",
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
        "roofline": roof,
        "e2e": {"value": unk * world / (e2e_ms * 1e-3), "unit": "DoF/s",
                "h2d_bytes_per_step": int(sum(v.nbytes for v in fb)), "d2h_bytes_per_step": int(upin.numel() * 8),
                "ms_per_step": e2e_ms},
        "gpu_launches": args.steps,
        "clocks": ck,
    }
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = n4_oracle_sample(p, m, levels, args.n4_smoother)[0]
    print(json.dumps(out))


def n4_oracle_sample(p, m, levels, smoother):
    """The oracle (oracle/bspline1d.py) on one problem of the workload, with
    fewer levels when the full depth would exceed ~20 s; solve time only."""
    import oracle.bspline1d as B
    N, b1, b2 = N4_ROWS[(p, m)]
    lev = min(levels, 12)
    o = B.CFMG1D(p, m, lev, N, b1, b2, B.poisson_f if m == 1 else B.biharm_f, smoother=smoother)
    t0 = time.perf_counter()
    o.solve()
    dt = time.perf_counter() - t0
    n = len(o.f[-1])
    return ({"value": n / dt, "unit": "DoF/s", "cores": 1, "kind": "oracle",
             "sample": f"one 1D solve, p={p} m={m}, {lev} levels ({n} unknowns), {dt:.2f} s (solve only)"}, dt)


def cpu_baseline(config, smoother="chebyshev", nu=1, cfas_fp32=0):
    import oracle as O
    cfg = CONFIGS[config]
    d, p, lev = cfg["dim"], cfg["p"], cfg["levels"]
    # bounded sample: the full solve when it fits ~30 s, else the same solver
    # on fewer levels (same d, p, schedule)
    sample_lev = lev
    while sample_lev > 2 and (p << sample_lev) ** d > 5_000_000:
        sample_lev -= 1
    s = O.schedule(d, p, smoother=smoother, nu=nu, cfas_fp32=cfas_fp32)
    c = O.CFMG(d, p, sample_lev, s)
    t0 = time.perf_counter()
    c.solve()
    dt = time.perf_counter() - t0
    unk = unknowns(d, p, sample_lev)
    cores = int(O.lib().orc_threads())
    return {"value": unk / dt, "unit": "DoF/s", "cores": cores, "kind": "oracle",
            "sample": f"one full compact FMG solve, {d}D Q{p}, {sample_lev} levels ({unk} unknowns), "
                      f"{dt:.2f} s on {cores} OpenMP thread(s)"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle as O
    cfg = CONFIGS[args.config]
    d, p, lev = cfg["dim"], cfg["p"], cfg["levels"]
    sample_lev = lev
    while sample_lev > 2 and (p << sample_lev) ** d > 5_000_000:
        sample_lev -= 1
    s = O.schedule(d, p, smoother=args.smoother, nu=args.nu, cfas_fp32=int(args.cfas_fp32))
    c = O.CFMG(d, p, sample_lev, s)
    for _ in range(args.warmup):
        c.solve()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        c.solve()
        ts.append(time.perf_counter() - t0)
    ms = 1e3 * sum(ts) / len(ts)
    unk = unknowns(d, p, sample_lev)
    cores = int(O.lib().orc_threads())
    v = unk / (ms * 1e-3)
    out = {
        "impl": "reference",
        "metric": METRIC, "value": v, "unit": "DoF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (manufactured solution)",
        "config": {"workload": args.config + ": " + cfg["desc"], "dim": d, "p": p, "levels": lev,
                   "sample_levels": sample_lev},
        "cpu_baseline": {"value": v, "unit": "DoF/s", "cores": cores, "kind": "oracle",
                         "sample": f"each step one full oracle solve with {sample_lev} levels "
                                   f"on {cores} OpenMP thread(s)"},
        "e2e": {"value": v, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--roofline-class", type=int, default=5, choices=[0, 5])
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per launch of the roofline kernel (profiles/)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nu", type=int, default=1,
                    help="compact V(0,1) cycles per IR iteration (SURVEY 8f N2; one GPU, 2D/3D, Chebyshev degree >= 2 or mcgs)")
    ap.add_argument("--cfas-fp32", action="store_true",
                    help="cFas in FP32 (DESIGN.md reading R28; 3D, Chebyshev): z, b, y, w in float")
    ap.add_argument("--smoother", default="chebyshev", choices=["chebyshev", "mcgs"],
                    help="cFas smoother: Chebyshev-Jacobi (default) or multicolour Gauss-Seidel (SURVEY 8f N1)")
    ap.add_argument("--workload", default="fmg", choices=["fmg", "n4"],
                    help="fmg: the 2D/3D compact FMG (--config); n4: the 1D B-spline batch (SURVEY 8f N4)")
    ap.add_argument("--n4-p", type=int, default=1)
    ap.add_argument("--n4-m", type=int, default=1)
    ap.add_argument("--n4-levels", type=int, default=16)
    ap.add_argument("--n4-batch", type=int, default=None,
                    help="problems per launch (default: one resident wave, DESIGN.md §12)")
    ap.add_argument("--n4-smoother", default="lex", choices=["lex", "mcgs"])
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if args.workload == "n4":
            if rank == 0:
                base, dt0 = n4_oracle_sample(args.n4_p, args.n4_m, args.n4_levels, args.n4_smoother)
                ts = [n4_oracle_sample(args.n4_p, args.n4_m, args.n4_levels, args.n4_smoother)[1]
                      for _ in range(args.steps)]
                v = base["value"] * dt0 / (sum(ts) / len(ts))  # same problem each step
                print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": "DoF/s",
                                  "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                                  "ms_per_step": 1e3 * sum(ts) / len(ts), "higher_is_better": True,
                                  "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                                  "data": "synthetic (manufactured 1D problem)",
                                  "config": {"workload": "N4 1D B-spline (oracle sample)", "p": args.n4_p,
                                             "m": args.n4_m, "levels": args.n4_levels},
                                  "cpu_baseline": dict(base, value=v),
                                  "e2e": {"value": v, "unit": "DoF/s", "h2d_bytes_per_step": 0,
                                          "d2h_bytes_per_step": 0}}))
            return
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.workload == "n4":
            run_n4(args, rank, world, local_rank)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as tdist
            tdist.destroy_process_group()


if __name__ == "__main__":
    main()
