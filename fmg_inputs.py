"""Inputs shared by the oracle tests and the product path: the benchmark
configurations, the solver schedules, and seeded synthetic vectors for codec
tests.  Holds NO arithmetic of the method (no operators, no codec, no tables):
only problem parameters and random numbers (DESIGN.md §4 input recipe).
"""
from __future__ import annotations

import numpy as np

# BASELINE.json configs (C1..C5).  levels = k-level FMG: solver levels 0..k-1,
# element size h_l = 2^-(l+1) (reading R3).
CONFIGS = {
    "C1": dict(dim=2, p=1, levels=7, desc="2D Poisson Q1 128x128 elements, 7-level FMG"),
    "C2": dict(dim=2, p=2, levels=10, desc="2D Poisson Q2 1024x1024 elements, 10-level FMG"),
    "C3": dict(dim=3, p=1, levels=9, desc="3D Poisson Q1 512^3 elements, 9-level FMG"),
    "C4": dict(dim=3, p=3, levels=8, desc="3D Poisson Q3 256^3 elements, 8-level FMG"),
    "C5": dict(dim=3, p=1, levels=12, desc="3D Poisson Q1 4096^3 elements, 12-level FMG"),
    # not a BASELINE config: C5's discretisation one level coarser, 8.6 G unknowns
    # = C5's per-GPU share at 8 GPUs, the largest Q1 cube one B200 holds
    # (SURVEY §8d-6 fallback: "a 2048^3 Q1 11-level problem")
    "C5h": dict(dim=3, p=1, levels=11, desc="3D Poisson Q1 2048^3 elements, 11-level FMG (C5 per-GPU share)"),
}

# Chebyshev upper bounds: 1.05 x lambda_max(D^-1 A) from the p-periodic block
# symbol (reading R4): Q1 1.5 (2D, 3D); 2D Q2 1.5523; 2D Q3 2.1586;
# 3D Q2 1.3393; 3D Q3 2.3350.
_LAMBDA_HI = {(2, 1): 1.575, (3, 1): 1.575, (2, 2): 1.63, (3, 2): 1.41,
              (2, 3): 2.27, (3, 3): 2.45}

# (b_u, b_r, N, Chebyshev degree, alpha) per degree p.
_SCHED = {1: (4, 4, 3, 2, 4.0), 2: (5, 4, 3, 2, 4.0), 3: (6, 4, 3, 3, 8.0)}


def default_schedule(d: int, p: int) -> dict:
    b_u, b_r, n_ir, k, alpha = _SCHED[p]
    return dict(b_u=b_u, k_u=p + 1, b_r=b_r, k_r=1, n_ir=n_ir, cheb_degree=k,
                lambda_hi=_LAMBDA_HI[(d, p)], alpha=alpha)


def unknowns(d: int, p: int, levels: int) -> int:
    """Interior unknowns of the finest level: (p 2^levels - 1)^d."""
    return (p * (1 << levels) - 1) ** d


def codec_vectors(n: int, seed: int, kind: str = "smooth") -> np.ndarray:
    """Seeded synthetic codec inputs (SURVEY §8d-2 recipe): smooth sum of sines
    plus 2^-s Gaussian noise, or plain Gaussian, or an adversarial mix of
    exact ties, powers of two, zero blocks and exponent-bump blocks."""
    rng = np.random.Generator(np.random.PCG64(seed))
    i = np.arange(n, dtype=np.float64)
    if kind == "smooth":
        a = rng.standard_normal(8)
        k = rng.uniform(1e-4, 0.3, 8)
        ph = rng.uniform(0, 2 * np.pi, 8)
        x = sum(a[j] * np.sin(k[j] * i + ph[j]) for j in range(8))
        s = rng.choice([10, 30])
        return x + 2.0 ** (-s) * rng.standard_normal(n)
    if kind == "gauss":
        return rng.standard_normal(n) * 2.0 ** rng.integers(-40, 40)
    if kind == "adversarial":
        x = rng.standard_normal(n)
        blocks = x.reshape(-1, 32)
        for b in range(blocks.shape[0]):
            t = b % 5
            e = int(rng.integers(-20, 20))
            if t == 0:
                blocks[b] = 0.0
            elif t == 1:   # powers of two with random signs
                blocks[b] = rng.choice([-1, 1], 32) * 2.0 ** rng.integers(e - 6, e, 32)
            elif t == 2:   # exact ties at a width-6 grid: (k + 1/2) 2^(e-q)
                kk = rng.integers(-30, 30, 32)
                blocks[b] = (kk + 0.5) * 2.0 ** (e - 5)
            elif t == 3:   # max rounds up to 2^q at width 4 -> exponent bump
                blocks[b] = rng.uniform(-1, 1, 32) * 2.0 ** e
                blocks[b, 0] = (2.0 - 2.0 ** -5) * 2.0 ** e
            else:          # sign-symmetric pairs
                v = rng.standard_normal(16) * 2.0 ** e
                blocks[b] = np.concatenate([v, -v])
        return blocks.reshape(-1)
    if kind == "staircase":
        # streaming-exponent inputs (N3): magnitudes trending up from the
        # subnormal range to 2^1000 over the vector, so the running maximum
        # rises ~2000 times at positions spread over every CTA chunk; 5 % zeros,
        # some exponent-bump values (2 - 2^-5) 2^e
        e_lo, e_hi = -1070.0, 1000.0
        t = (i / max(n, 1)) ** 1.5
        e = np.floor(e_lo + (e_hi - e_lo) * t + rng.integers(-40, 3, n)).astype(np.int64)
        e = np.clip(e, -1074, 1000)
        x = rng.uniform(0.5, 1.0, n) * rng.choice([-1.0, 1.0], n)
        bump = rng.random(n) < 0.02
        x[bump] = np.sign(x[bump]) * (1.0 - 2.0 ** -6)
        x = np.ldexp(x, e)
        x[rng.random(n) < 0.05] = 0.0
        return x
    raise ValueError(kind)
