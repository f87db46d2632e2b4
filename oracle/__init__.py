"""ctypes binding of the CPU oracle (liboracle.so).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_2511_19036_b200`` never imports it.

The oracle is a plain sequential FP64 C implementation of compact FMG
(Alg 3.3 o Alg 3.2 o Alg 3.1) written from the paper; see
``oracle/oracle.h`` and DESIGN.md §3 for the canonical evaluation order.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build() -> str:
    """Compile liboracle.so in-tree (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        srcs = [os.path.join(_HERE, f) for f in os.listdir(_HERE) if f.endswith((".c", ".h"))]
        if not os.path.exists(path) or any(os.path.getmtime(s) > os.path.getmtime(path) for s in srcs):
            build()
        L = C.CDLL(path)
        dp = C.POINTER(C.c_double)
        L.orc_bfp_encode.argtypes = [dp, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_bfp_decode.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, dp]
        L.orc_stream_encode.argtypes = [dp, C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_stream_decode.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int, dp]
        L.orc_apply_A.argtypes = [C.c_int, C.c_int, C.c_int, dp, dp]
        L.orc_prolong.argtypes = [C.c_int, C.c_int, C.c_int, dp, dp]
        L.orc_restrict.argtypes = [C.c_int, C.c_int, C.c_int, dp, dp]
        L.orc_rhs_table.argtypes = [C.c_int, C.c_int, dp]
        L.orc_rhs.argtypes = [C.c_int, C.c_int, C.c_int, dp]
        L.orc_rhs_const.argtypes = [C.c_int]
        L.orc_rhs_const.restype = C.c_double
        L.orc_inv_diag.argtypes = [C.c_int, C.c_int, C.c_int, dp]
        L.orc_coef_A.argtypes = [C.c_int, dp, dp]
        L.orc_coef_P.argtypes = [C.c_int, dp]
        L.orc_coef_R.argtypes = [C.c_int, dp]
        L.orc_coarse_n.argtypes = [C.c_int, C.c_int]
        L.orc_coarse_matrix.argtypes = [C.c_int, C.c_int, dp]
        L.orc_coarse_inverse.argtypes = [C.c_int, C.c_int, dp]
        L.orc_cheb_coefs.argtypes = [C.c_void_p, dp, dp, dp]
        L.orc_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_create_streamed.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_stream_bytes.argtypes = [C.c_void_p]
        L.orc_stream_bytes.restype = C.c_int64
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_solve.argtypes = [C.c_void_p]
        L.orc_solve_upto.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.orc_residual.argtypes = [C.c_void_p, C.c_int, dp]
        L.orc_cfas_correct.argtypes = [C.c_void_p, C.c_int]
        L.orc_norms.argtypes = [C.c_void_p]
        L.orc_norms.restype = dp
        L.orc_get_section.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_int)]
        L.orc_set_section.argtypes = [C.c_void_p, C.c_int, C.c_int, dp, C.c_int]
        L.orc_get_array.argtypes = [C.c_void_p, C.c_int, C.c_int, dp]
        L.orc_decode_solution.argtypes = [C.c_void_p, C.c_int, dp]
        L.orc_errors.argtypes = [C.c_int, C.c_int, C.c_int, dp, dp]
        L.orc_std_solve.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, dp]
        L.orc_std_vcycle_rho.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, dp]
        _LIB = L
    return _LIB


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Schedule(C.Structure):
    """Mirror of orc_schedule (oracle.h)."""

    _fields_ = [("b_u", C.c_int), ("k_u", C.c_int), ("b_r", C.c_int), ("k_r", C.c_int),
                ("n_ir", C.c_int), ("cheb_degree", C.c_int),
                ("lambda_hi", C.c_double), ("alpha", C.c_double), ("smoother", C.c_int),
                ("nu", C.c_int), ("cfas_fp32", C.c_int)]


SMOOTHERS = {"chebyshev": 0, "mcgs": 1, "lexgs": 2}


def schedule(d: int, p: int, b_u=None, b_r=None, n_ir=None, k_u=None, k_r=1,
             cheb_degree=None, lambda_hi=None, alpha=None, smoother="chebyshev", nu=1,
             cfas_fp32=0) -> Schedule:
    """Default schedule of DESIGN.md §5 (same numbers the product path uses)."""
    from fmg_inputs import default_schedule
    s = default_schedule(d, p)
    over = dict(b_u=b_u, b_r=b_r, n_ir=n_ir, k_u=k_u, k_r=k_r, cheb_degree=cheb_degree,
                lambda_hi=lambda_hi, alpha=alpha)
    for k, v in over.items():
        if v is not None:
            s[k] = v
    return Schedule(s["b_u"], s["k_u"], s["b_r"], s["k_r"], s["n_ir"], s["cheb_degree"],
                    s["lambda_hi"], s["alpha"], SMOOTHERS[smoother] if isinstance(smoother, str) else smoother,
                    nu, int(cfas_fp32))


@dataclass
class Geom:
    d: int
    p: int
    l: int

    @property
    def n(self):
        return self.p << (self.l + 1)

    @property
    def NX(self):
        return (self.n + 31) // 32 * 32

    @property
    def shape(self):
        n = self.n
        return (n, n, self.NX) if self.d == 3 else (1, n, self.NX)

    @property
    def size(self):
        s = self.shape
        return s[0] * s[1] * s[2]


def bfp_encode(x: np.ndarray, width: int):
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = x.size
    mant = np.zeros((n // 32) * width, dtype=np.uint32)
    exps = np.zeros(n // 32, dtype=np.int8)
    rc = lib().orc_bfp_encode(_dp(x), n, width, mant.ctypes.data, exps.ctypes.data)
    return rc, mant, exps


def bfp_decode(mant: np.ndarray, exps: np.ndarray, n: int, width: int):
    x = np.zeros(n, dtype=np.float64)
    rc = lib().orc_bfp_decode(mant.ctypes.data, exps.ctypes.data, n, width, _dp(x))
    return rc, x


def stream_encode(x: np.ndarray, width: int):
    """Streaming-exponent BFP -> (rc, mant, xexp[:K], xstart[:K])."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = x.size
    mant = np.zeros((n // 32) * width, dtype=np.uint32)
    xexp = np.zeros(width, dtype=np.int32)
    xstart = np.zeros(width, dtype=np.int64)
    nb = np.zeros(1, dtype=np.int32)
    rc = lib().orc_stream_encode(_dp(x), n, width, mant.ctypes.data, xexp.ctypes.data, xstart.ctypes.data,
                                 nb.ctypes.data)
    k = int(nb[0])
    return rc, mant, xexp[:k].copy(), xstart[:k].copy()


def stream_decode(mant: np.ndarray, xexp: np.ndarray, xstart: np.ndarray, n: int, width: int):
    x = np.zeros(n, dtype=np.float64)
    xexp = np.ascontiguousarray(xexp, dtype=np.int32)
    xstart = np.ascontiguousarray(xstart, dtype=np.int64)
    rc = lib().orc_stream_decode(np.ascontiguousarray(mant, dtype=np.uint32).ctypes.data, xexp.ctypes.data,
                                 xstart.ctypes.data, len(xexp), n, width, _dp(x))
    return rc, x


def apply_A(d, p, l, u):
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros_like(u)
    lib().orc_apply_A(d, p, l, _dp(u), _dp(out))
    return out


def apply_A_f32(d, p, l, u):
    u = np.ascontiguousarray(u, dtype=np.float32)
    out = np.zeros_like(u)
    fp = C.POINTER(C.c_float)
    lib().orc_apply_A_f32(d, p, l, u.ctypes.data_as(fp), out.ctypes.data_as(fp))
    return out


def prolong_f32(d, p, lf, coarse):
    coarse = np.ascontiguousarray(coarse, dtype=np.float32)
    out = np.zeros(Geom(d, p, lf).shape, dtype=np.float32)
    fp = C.POINTER(C.c_float)
    lib().orc_prolong_f32(d, p, lf, coarse.ctypes.data_as(fp), out.ctypes.data_as(fp))
    return out


def prolong(d, p, lf, coarse):
    coarse = np.ascontiguousarray(coarse, dtype=np.float64)
    out = np.zeros(Geom(d, p, lf).shape)
    lib().orc_prolong(d, p, lf, _dp(coarse), _dp(out))
    return out


def restrict(d, p, lf, fine):
    fine = np.ascontiguousarray(fine, dtype=np.float64)
    out = np.zeros(Geom(d, p, lf - 1).shape)
    lib().orc_restrict(d, p, lf, _dp(fine), _dp(out))
    return out


def rhs_table(p, l):
    g = np.zeros(p << (l + 1))
    lib().orc_rhs_table(p, l, _dp(g))
    return g


def rhs(d, p, l):
    f = np.zeros(Geom(d, p, l).shape)
    lib().orc_rhs(d, p, l, _dp(f))
    return f


def inv_diag(d, p, l):
    v = np.zeros(Geom(d, p, l).shape)
    lib().orc_inv_diag(d, p, l, _dp(v))
    return v


def coef_A(p):
    K = np.zeros((p, 2 * p + 1)); M = np.zeros((p, 2 * p + 1))
    lib().orc_coef_A(p, _dp(K), _dp(M))
    return K, M


def coef_P(p):
    W = np.zeros((2 * p, p + 1))
    lib().orc_coef_P(p, _dp(W))
    return W


def coef_R(p):
    R = np.zeros((p, 4 * p - 1))
    lib().orc_coef_R(p, _dp(R))
    return R


def coarse_matrix(d, p):
    n0 = lib().orc_coarse_n(d, p)
    A = np.zeros((n0, n0))
    lib().orc_coarse_matrix(d, p, _dp(A))
    return A


def coarse_inverse(d, p):
    n0 = lib().orc_coarse_n(d, p)
    A = np.zeros((n0, n0))
    rc = lib().orc_coarse_inverse(d, p, _dp(A))
    assert rc == 0
    return A


def cheb_coefs(s: Schedule):
    it = np.zeros(1); al = np.zeros(8); be = np.zeros(8)
    lib().orc_cheb_coefs(C.byref(s), _dp(it), _dp(al), _dp(be))
    return it[0], al, be


def errors(d, p, l, uhat):
    uhat = np.ascontiguousarray(uhat, dtype=np.float64)
    e = np.zeros(3)
    lib().orc_errors(d, p, l, _dp(uhat), _dp(e))
    return e


def std_solve(d, p, levels, s: Schedule, cycles: int):
    out = np.zeros(Geom(d, p, levels - 1).shape)
    rc = lib().orc_std_solve(d, p, levels, C.byref(s), cycles, _dp(out))
    assert rc == 0
    return out


def vcycle_rho(d, p, levels, s: Schedule, iters=30):
    r = np.zeros(1)
    lib().orc_std_vcycle_rho(d, p, levels, C.byref(s), iters, _dp(r))
    return float(r[0])


class CFMG:
    """Oracle compact FMG context (orc_ctx)."""

    def __init__(self, d: int, p: int, levels: int, s: Schedule, streamed: bool = False):
        """streamed: the plane-streamed mode (Alg 5.3/5.4 at plane granularity,
        orc_stream.c), bit-identical to the simple mode in linear space."""
        self.d, self.p, self.levels, self.s = d, p, levels, s
        self.Lmax = levels - 1
        h = C.c_void_p()
        create = lib().orc_create_streamed if streamed else lib().orc_create
        rc = create(d, p, levels, C.byref(s), C.byref(h))
        if rc:
            raise ValueError(f"orc_create failed rc={rc}")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    def solve(self):
        rc = lib().orc_solve(self.h)
        if rc:
            raise RuntimeError(f"orc_solve rc={rc}")

    def solve_upto(self, L, iters_last):
        rc = lib().orc_solve_upto(self.h, L, iters_last)
        if rc:
            raise RuntimeError(f"orc_solve_upto rc={rc}")

    def residual(self, L):
        nr = np.zeros(L + 1)
        rc = lib().orc_residual(self.h, L, _dp(nr))
        assert rc == 0
        return nr

    def smooth(self, l: int, b: np.ndarray) -> np.ndarray:
        """The schedule's cFas smoother on level l from y = 0 (orc_smooth)."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        y = np.zeros_like(b)
        rc = lib().orc_smooth(self.h, l, _dp(b), _dp(y))
        assert rc == 0
        return y

    def cfas_correct(self, L):
        rc = lib().orc_cfas_correct(self.h, L)
        assert rc == 0

    def stream_bytes(self) -> int:
        """Peak bytes of the streamed mode's plane windows (0 in simple mode)."""
        return int(lib().orc_stream_bytes(self.h))

    def norms(self):
        n = (self.Lmax + 1) * self.s.n_ir * (self.Lmax + 1)
        ptr = lib().orc_norms(self.h)
        return np.ctypeslib.as_array(ptr, shape=(n,)).copy().reshape(
            self.Lmax + 1, self.s.n_ir, self.Lmax + 1)

    def section(self, which: int, l: int):
        g = Geom(self.d, self.p, l)
        w = C.c_int()
        lib().orc_get_section(self.h, which, l, None, None, C.byref(w))
        mant = np.zeros((g.size // 32) * w.value, dtype=np.uint32)
        exps = np.zeros(g.size // 32, dtype=np.int8)
        lib().orc_get_section(self.h, which, l, mant.ctypes.data, exps.ctypes.data, C.byref(w))
        return mant, exps, w.value

    def set_section(self, which: int, l: int, x: np.ndarray, width: int):
        x = np.ascontiguousarray(x, dtype=np.float64)
        rc = lib().orc_set_section(self.h, which, l, _dp(x), width)
        assert rc == 0

    def array(self, which: int, l: int):
        out = np.zeros(Geom(self.d, self.p, l).shape)
        lib().orc_get_array(self.h, which, l, _dp(out))
        return out

    def solution(self, L=None):
        L = self.Lmax if L is None else L
        out = np.zeros(Geom(self.d, self.p, L).shape)
        lib().orc_decode_solution(self.h, L, _dp(out))
        return out

    def errors(self, L=None):
        L = self.Lmax if L is None else L
        return errors(self.d, self.p, L, self.solution(L))
