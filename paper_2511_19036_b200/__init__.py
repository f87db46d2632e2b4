"""Thin Python binding of libfmg.so (include/fmg.h) -- the B200 compact-FMG hot
path of arXiv 2511.19036.

Argument marshalling only: every step of the method runs in the CUDA kernels
of ``csrc/``.  PyTorch provides device memory (through the allocator hook),
streams and tensors.  There is no CPU fallback: importing this package raises
if the extension has not been built.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("FMG_LIB") or os.path.join(_HERE, "libfmg.so")

if not os.path.exists(_SO):
    raise ImportError(f"libfmg.so not built ({_SO}); run `python -c 'import __graft_entry__ as g; g.build()'`")

_lib = C.CDLL(_SO)

FMG_OK, FMG_EINVAL, FMG_ERANGE, FMG_ENOMEM, FMG_ECUDA, FMG_ESTATE, FMG_ENCCL = range(7)


class FmgError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {_lib.fmg_strerror(code).decode()} (code {code})")
        self.code = code


class Schedule(C.Structure):
    """fmg_schedule (include/fmg.h)."""

    _fields_ = [("b_u", C.c_int), ("k_u", C.c_int), ("b_r", C.c_int), ("k_r", C.c_int),
                ("n_ir", C.c_int), ("cheb_degree", C.c_int),
                ("lambda_hi", C.c_double), ("alpha", C.c_double), ("smoother", C.c_int),
                ("nu", C.c_int), ("cfas_fp32", C.c_int)]

    @classmethod
    def from_dict(cls, d: dict) -> "Schedule":
        sm = d.get("smoother", 0)
        sm = {"chebyshev": 0, "mcgs": 1}[sm] if isinstance(sm, str) else sm
        return cls(d["b_u"], d["k_u"], d["b_r"], d["k_r"], d["n_ir"], d["cheb_degree"],
                   d["lambda_hi"], d["alpha"], sm, d.get("nu", 1), int(d.get("cfas_fp32", 0)))


_vp = C.c_void_p
_dp = C.POINTER(C.c_double)
_lib.fmg_strerror.restype = C.c_char_p
_lib.fmg_strerror.argtypes = [C.c_int]
_lib.fmg_create.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(Schedule), _vp, C.POINTER(_vp)]
_lib.fmg_create_slabs.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(Schedule), C.c_int, _vp, C.POINTER(_vp)]
_lib.fmg_create_dist.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(Schedule), C.c_int, C.c_int, _vp, _vp,
                                 C.POINTER(_vp)]
_lib.fmg_nccl_unique_id.argtypes = [_vp]
# host-staged transport callback: fn(user, n, peer[], send[], buf[], bytes[]) -> 0
_XFER_FN = C.CFUNCTYPE(C.c_int, _vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(_vp),
                       C.POINTER(C.c_int64))
_lib.fmg_create_hostx.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(Schedule), C.c_int, C.c_int, _XFER_FN, _vp,
                                  _vp, C.POINTER(_vp)]
_lib.fmg_slab_plan.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _vp, C.c_int]
_lib.fmg_solve.argtypes = [_vp]
_lib.fmg_solve_async.argtypes = [_vp]
_lib.fmg_solve_upto.argtypes = [_vp, C.c_int, C.c_int]
_lib.fmg_norms.argtypes = [_vp, _dp]
_lib.fmg_residual.argtypes = [_vp, _dp]
_lib.fmg_get_solution.argtypes = [_vp, _vp]
_lib.fmg_errors.argtypes = [_vp, _dp]
_lib.fmg_get_section.argtypes = [_vp, C.c_int, C.c_int, _vp, _vp, C.POINTER(C.c_int)]
_lib.fmg_info.argtypes = [_vp, _dp]
_lib.fmg_memory_model.argtypes = [C.c_int, C.c_int, C.c_int, _vp, _dp, C.c_int]
_lib.fmg_device_bytes.argtypes = [_vp]
_lib.fmg_device_bytes.restype = C.c_int64
_lib.fmg_enable_kernel_timing.argtypes = [_vp, C.c_int]
_lib.fmg_kernel_time.argtypes = [_vp, _dp, C.POINTER(C.c_int)]
_lib.fmg_kernel_times.argtypes = [_vp, _vp, C.c_int]
_lib.fmg_destroy.argtypes = [_vp]
_lib.fmg_destroy.restype = None
_lib.fmg_rhs_size.argtypes = [_vp]
_lib.fmg_rhs_size.restype = C.c_int64
_lib.fmg_set_rhs.argtypes = [_vp, _vp]
_lib.fmg_export_solution.argtypes = [_vp, _vp, C.c_int64]
_lib.fmg_export_solution.restype = C.c_int64
_lib.fmg_get_rhs.argtypes = [_vp, _vp]
_lib.bfp_encode.argtypes = [_vp, C.c_int64, C.c_int, _vp, _vp, _vp]
_lib.bfp_decode.argtypes = [_vp, _vp, C.c_int64, C.c_int, _vp, _vp]
_lib.bfp_status.argtypes = [_vp]
_lib.bfp_stream_work_bytes.argtypes = [C.c_int64]
_lib.bfp_stream_work_bytes.restype = C.c_int64
_lib.bfp_stream_encode.argtypes = [_vp, C.c_int64, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp]
_lib.bfp_stream_decode.argtypes = [_vp, _vp, _vp, _vp, C.c_int64, C.c_int, _vp, _vp]

_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p)
_lib.fmg_set_allocator.argtypes = [_ALLOC_FN, _FREE_FN, C.c_void_p]

EXPORTS = ["fmg_set_allocator", "fmg_create", "fmg_create_slabs", "fmg_create_dist", "fmg_create_hostx",
           "fmg_nccl_unique_id",
           "fmg_slab_plan", "fmg_solve_async", "fmg_solve", "fmg_solve_upto",
           "fmg_norms", "fmg_residual", "fmg_get_solution", "fmg_errors", "fmg_get_section",
           "fmg_info", "fmg_memory_model", "fmg_device_bytes", "fmg_enable_kernel_timing", "fmg_kernel_time", "fmg_kernel_times", "fmg_destroy",
           "fmg_rhs_size", "fmg_set_rhs", "fmg_get_rhs", "fmg_export_solution",
           "fmg_strerror", "bfp_encode", "bfp_decode", "bfp_status",
           "bfp_stream_work_bytes", "bfp_stream_encode", "bfp_stream_decode"]


def _check(rc: int, what: str):
    if rc != FMG_OK:
        raise FmgError(rc, what)


_torch_alloc_refs = None


def use_torch_allocator(enable: bool = True):
    """Back every context's device memory by torch's caching allocator."""
    global _torch_alloc_refs
    import torch

    if not enable:
        _lib.fmg_set_allocator(_ALLOC_FN(), _FREE_FN(), None)
        _torch_alloc_refs = None
        return

    def _alloc(nbytes, user):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), torch.cuda.current_device())
        except Exception:
            return None

    def _free(ptr, nbytes, user):
        torch.cuda.caching_allocator_delete(ptr)

    _torch_alloc_refs = (_ALLOC_FN(_alloc), _FREE_FN(_free))
    _check(_lib.fmg_set_allocator(_torch_alloc_refs[0], _torch_alloc_refs[1], None), "fmg_set_allocator")


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for fmg_create_dist (call on rank 0, broadcast)."""
    buf = C.create_string_buffer(128)
    _check(_lib.fmg_nccl_unique_id(buf), "fmg_nccl_unique_id")
    return buf.raw


def slab_plan(nz: int, nslabs: int, rank: int, depth: int, gather: bool = False):
    """Host-only ghost-plane exchange plan of one z slab (fmg_slab_plan):
    list of (peer, z0, z1, send)."""
    n = _lib.fmg_slab_plan(nz, nslabs, rank, depth, int(gather), None, 0)
    if n < 0:
        raise FmgError(-n, "fmg_slab_plan")
    out = (C.c_int * (4 * max(n, 1)))()
    _lib.fmg_slab_plan(nz, nslabs, rank, depth, int(gather), out, n)
    return [tuple(out[4 * i:4 * i + 4]) for i in range(n)]


def host_transport_gloo(group=None):
    """A host-staged transport for Solver(hostx=...): every piece of an
    exchange as torch.distributed isend / irecv (e.g. over gloo), then wait."""
    import torch
    import torch.distributed as tdist

    def transport(pieces):
        reqs = []
        for peer, send, arr in pieces:
            t = torch.from_numpy(arr)
            reqs.append(tdist.isend(t, peer, group=group) if send else tdist.irecv(t, peer, group=group))
        for r in reqs:
            r.wait()

    return transport


def _stream_ptr(stream):
    if stream is None:
        return None
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


class Solver:
    """A compact-FMG context (fmg_create ... fmg_destroy)."""

    def __init__(self, dim: int, p: int, levels: int, schedule: Schedule | dict | None = None,
                 stream=None, slabs: int = 1, dist: tuple | None = None, hostx: tuple | None = None):
        """slabs > 1: virtual z slabs on this device (fmg_create_slabs).
        dist = (rank, nranks, uid): this process is z-slab `rank` of `nranks`
        GPUs (fmg_create_dist); uid from nccl_unique_id() on rank 0.
        hostx = (rank, nranks, transport): z-slab `rank` with a host-staged
        transport (fmg_create_hostx); transport(pieces) receives a list of
        (peer, send, numpy uint8 view) and must complete every piece, e.g.
        torch.distributed isend / irecv over gloo (see host_transport_gloo)."""
        if schedule is None:
            from fmg_inputs import default_schedule
            schedule = default_schedule(dim, p)
        if isinstance(schedule, dict):
            schedule = Schedule.from_dict(schedule)
        self.dim, self.p, self.levels, self.schedule = dim, p, levels, schedule
        self.stream = stream
        h = C.c_void_p()
        self._xfer = None
        if hostx is not None:
            rank, nranks, transport = hostx
            import numpy as np

            def _cb(user, n, peer, send, buf, nbytes):
                try:
                    pieces = [(peer[i], send[i], np.ctypeslib.as_array(C.cast(buf[i], C.POINTER(C.c_uint8)),
                                                                        shape=(nbytes[i],)))
                              for i in range(n)]
                    transport(pieces)
                    return 0
                except Exception:  # (reported to the library as a transport failure)
                    import traceback
                    traceback.print_exc()
                    return 1

            self._xfer = _XFER_FN(_cb)
            _check(_lib.fmg_create_hostx(dim, p, levels, C.byref(schedule), nranks, rank, self._xfer, None,
                                         _stream_ptr(stream), C.byref(h)), "fmg_create_hostx")
        elif dist is not None:
            rank, nranks, uid = dist
            ub = C.create_string_buffer(bytes(uid), 128)
            _check(_lib.fmg_create_dist(dim, p, levels, C.byref(schedule), nranks, rank, ub, _stream_ptr(stream),
                                        C.byref(h)), "fmg_create_dist")
        elif slabs > 1:  # virtual z slabs on one device (fmg_create_slabs)
            _check(_lib.fmg_create_slabs(dim, p, levels, C.byref(schedule), slabs, _stream_ptr(stream),
                                         C.byref(h)), "fmg_create_slabs")
        else:
            _check(_lib.fmg_create(dim, p, levels, C.byref(schedule), _stream_ptr(stream), C.byref(h)),
                   "fmg_create")
        self._h = h

    def close(self):
        # (at interpreter shutdown the module globals may already be cleared)
        if getattr(self, "_h", None) and _lib is not None:
            _lib.fmg_destroy(self._h)
            self._h = None

    __del__ = close

    # -- Alg 3.3 ----------------------------------------------------------
    def solve(self):
        _check(_lib.fmg_solve(self._h), "fmg_solve")

    def solve_async(self):
        _check(_lib.fmg_solve_async(self._h), "fmg_solve_async")

    def solve_upto(self, L: int, iters_last: int):
        _check(_lib.fmg_solve_upto(self._h, L, iters_last), "fmg_solve_upto")

    def norms(self):
        import numpy as np
        n = self.levels * self.schedule.n_ir * self.levels
        out = np.zeros(n)
        _check(_lib.fmg_norms(self._h, out.ctypes.data_as(_dp)), "fmg_norms")
        return out.reshape(self.levels, self.schedule.n_ir, self.levels)

    def residual(self):
        import numpy as np
        out = np.zeros(self.levels)
        _check(_lib.fmg_residual(self._h, out.ctypes.data_as(_dp)), "fmg_residual")
        return out

    def geom(self, l: int):
        n = self.p << (l + 1)
        NX = (n + 31) // 32 * 32
        return (n, n, NX) if self.dim == 3 else (1, n, NX)

    def solution(self, L: int | None = None):
        import torch
        L = self.levels - 1 if L is None else L
        out = torch.empty(self.geom(L), dtype=torch.float64, device="cuda")
        _check(_lib.fmg_get_solution(self._h, C.c_void_p(out.data_ptr())), "fmg_get_solution")
        return out

    def errors(self):
        import numpy as np
        e = np.zeros(3)
        _check(_lib.fmg_errors(self._h, e.ctypes.data_as(_dp)), "fmg_errors")
        return e

    def section(self, which: int, l: int):
        import numpy as np
        w = C.c_int()
        _check(_lib.fmg_get_section(self._h, which, l, None, None, C.byref(w)), "fmg_get_section")
        shp = self.geom(l)
        nblk = shp[0] * shp[1] * shp[2] // 32
        mant = np.zeros(nblk * w.value, dtype=np.uint32)
        exps = np.zeros(nblk, dtype=np.int8)
        _check(_lib.fmg_get_section(self._h, which, l, mant.ctypes.data, exps.ctypes.data, C.byref(w)),
               "fmg_get_section")
        return mant, exps, w.value

    def info(self) -> dict:
        import numpy as np
        v = np.zeros(10)
        _check(_lib.fmg_info(self._h, v.ctypes.data_as(_dp)), "fmg_info")
        keys = ["dim", "p", "levels", "NX", "NY", "NZ", "unknowns", "stored_bits", "alg_bytes_per_solve",
                "launches_per_solve"]
        return dict(zip(keys, v.tolist()))

    def device_bytes(self) -> int:
        """Device memory this context holds (all slabs)."""
        return int(_lib.fmg_device_bytes(self._h))

    def rhs_size(self) -> int:
        return int(_lib.fmg_rhs_size(self._h))

    def get_rhs(self):
        import numpy as np
        out = np.zeros(self.rhs_size())
        _check(_lib.fmg_get_rhs(self._h, out.ctypes.data), "fmg_get_rhs")
        return out

    def set_rhs(self, host_tables):
        """host_tables: numpy float64 array or pinned torch CPU tensor (async copy)."""
        ptr = host_tables.data_ptr() if hasattr(host_tables, "data_ptr") else host_tables.ctypes.data
        _check(_lib.fmg_set_rhs(self._h, C.c_void_p(ptr)), "fmg_set_rhs")

    def export_size(self) -> int:
        return int(_lib.fmg_export_solution(self._h, None, 0))

    def export_solution(self, host_buf):
        """Asynchronous D2H copy of every compact solution section (storage
        layout, see fmg.h) into a pinned torch CPU uint8 tensor."""
        rc = _lib.fmg_export_solution(self._h, C.c_void_p(host_buf.data_ptr()), host_buf.numel())
        if rc < 0:
            raise FmgError(-rc, "fmg_export_solution")

    def enable_kernel_timing(self, cls: int):
        _check(_lib.fmg_enable_kernel_timing(self._h, cls), "fmg_enable_kernel_timing")

    def kernel_times(self):
        import numpy as np
        buf = np.zeros(20000, dtype=np.float32)
        n = _lib.fmg_kernel_times(self._h, buf.ctypes.data, buf.size)
        return buf[:max(n, 0)].copy()

    def kernel_time(self):
        t = C.c_double()
        n = C.c_int()
        _check(_lib.fmg_kernel_time(self._h, C.byref(t), C.byref(n)), "fmg_kernel_time")
        return t.value, n.value


def bfp_encode(x, width: int, stream=None):
    """Encode a CUDA float64 tensor (numel % 32 == 0) -> (mant uint32-as-int32, exps int8)."""
    import torch
    assert x.is_cuda and x.dtype == torch.float64 and x.is_contiguous()
    n = x.numel()
    mant = torch.empty((n // 32) * width, dtype=torch.int32, device=x.device)
    exps = torch.empty(n // 32, dtype=torch.int8, device=x.device)
    st = _stream_ptr(stream if stream is not None else torch.cuda.current_stream())
    _check(_lib.bfp_encode(C.c_void_p(x.data_ptr()), n, width, C.c_void_p(mant.data_ptr()),
                           C.c_void_p(exps.data_ptr()), st), "bfp_encode")
    return mant, exps


def bfp_decode(mant, exps, n: int, width: int, stream=None):
    import torch
    x = torch.empty(n, dtype=torch.float64, device=mant.device)
    st = _stream_ptr(stream if stream is not None else torch.cuda.current_stream())
    _check(_lib.bfp_decode(C.c_void_p(mant.data_ptr()), C.c_void_p(exps.data_ptr()), n, width,
                           C.c_void_p(x.data_ptr()), st), "bfp_decode")
    return x


MEMORY_KEYS = ["unknowns", "u_mantissa_bits", "r_mantissa_bits", "eq61_u", "eq61_u_bound", "eq61_r",
               "eq61_r_bound", "exponent_bits_fixed", "exponent_bits_streaming", "eq62_ut_bits",
               "eq63_z_bits", "fp64_temporary_bytes", "section_bytes"]


def memory_model(dim: int, p: int, levels: int, schedule=None) -> dict:
    """Storage accounting of a solve (Eq 6.1-6.3; host only,
    no device work): see fmg_memory_model in include/fmg.h."""
    import numpy as np
    if schedule is None:
        from fmg_inputs import default_schedule
        schedule = default_schedule(dim, p)
    if isinstance(schedule, dict):
        schedule = Schedule.from_dict(schedule)
    v = np.zeros(len(MEMORY_KEYS))
    _check(_lib.fmg_memory_model(dim, p, levels, C.byref(schedule), v.ctypes.data_as(_dp), len(MEMORY_KEYS)),
           "fmg_memory_model")
    return dict(zip(MEMORY_KEYS, v.tolist()))


def bfp_stream_encode(x, width: int, stream=None):
    """Streaming-exponent BFP of a CUDA float64 tensor
    (numel % 32 == 0) -> (mant int32[n w / 32], xexp int32[width],
    xstart int64[width], nblocks int32[1]); the first nblocks table entries are
    valid.  All outputs stay on the device."""
    import torch
    assert x.is_cuda and x.dtype == torch.float64 and x.is_contiguous()
    n = x.numel()
    dev = x.device
    mant = torch.empty((n // 32) * width, dtype=torch.int32, device=dev)
    xexp = torch.zeros(width, dtype=torch.int32, device=dev)
    xstart = torch.zeros(width, dtype=torch.int64, device=dev)
    nb = torch.zeros(1, dtype=torch.int32, device=dev)
    wb = _lib.bfp_stream_work_bytes(n)
    if wb < 0:
        raise FmgError(-wb, "bfp_stream_work_bytes")
    work = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
    st = _stream_ptr(stream if stream is not None else torch.cuda.current_stream())
    _check(_lib.bfp_stream_encode(C.c_void_p(x.data_ptr()), n, width, C.c_void_p(mant.data_ptr()),
                                  C.c_void_p(xexp.data_ptr()), C.c_void_p(xstart.data_ptr()),
                                  C.c_void_p(nb.data_ptr()), C.c_void_p(work.data_ptr()), st),
           "bfp_stream_encode")
    return mant, xexp, xstart, nb


def bfp_stream_decode(mant, xexp, xstart, nblocks, n: int, width: int, stream=None):
    import torch
    x = torch.empty(n, dtype=torch.float64, device=mant.device)
    st = _stream_ptr(stream if stream is not None else torch.cuda.current_stream())
    _check(_lib.bfp_stream_decode(C.c_void_p(mant.data_ptr()), C.c_void_p(xexp.data_ptr()),
                                  C.c_void_p(xstart.data_ptr()), C.c_void_p(nblocks.data_ptr()), n, width,
                                  C.c_void_p(x.data_ptr()), st), "bfp_stream_decode")
    return x


def bfp_status(stream=None) -> int:
    import torch
    st = _stream_ptr(stream if stream is not None else torch.cuda.current_stream())
    return _lib.bfp_status(st)


# ------------------------------------------------- 1D B-spline FMG (N4) --
# include/fmg1d.h: the paper's 1D Poisson / biharmonic workloads, a batch of
# problems per launch (one CTA per problem).  Marshalling only.
FMG1D_LEX, FMG1D_MCGS = 0, 1


class Schedule1D(C.Structure):
    _fields_ = [("N", C.c_int), ("b1", C.c_int), ("b2", C.c_int), ("smoother", C.c_int)]


_PP = C.POINTER(_vp)
_lib.fmg1d_size.argtypes = [C.c_int, C.c_int, C.c_int]
_lib.fmg1d_ell_width.argtypes = [C.c_int, C.c_int, C.c_int]
_lib.fmg1d_assemble_operator.argtypes = [C.c_int, C.c_int, C.c_int, _vp]
_lib.fmg1d_assemble_prolongation.argtypes = [C.c_int, C.c_int, C.c_int, _vp]
_lib.fmg1d_assemble_load.argtypes = [C.c_int, C.c_int, C.c_int, _vp]
_lib.fmg1d_create.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(Schedule1D), C.c_int, _PP, _PP, _vp, _vp,
                              C.POINTER(_vp)]
_lib.fmg1d_destroy.argtypes = [_vp]
_lib.fmg1d_set_load.argtypes = [_vp, _PP]
_lib.fmg1d_solve_async.argtypes = [_vp]
_lib.fmg1d_sync.argtypes = [_vp]
_lib.fmg1d_solve_host.argtypes = [_vp, _PP, _vp]
_lib.fmg1d_solution.argtypes = [_vp, C.c_int, _vp]
_lib.fmg1d_solution_device.argtypes = [_vp, C.POINTER(_vp)]
_lib.fmg1d_section.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, C.POINTER(C.c_int)]

EXPORTS += ["fmg1d_size", "fmg1d_ell_width", "fmg1d_assemble_operator", "fmg1d_assemble_prolongation",
            "fmg1d_assemble_load", "fmg1d_create", "fmg1d_destroy", "fmg1d_set_load", "fmg1d_solve_async",
            "fmg1d_sync", "fmg1d_solve_host", "fmg1d_solution", "fmg1d_solution_device", "fmg1d_section"]


def fmg1d_size(p: int, m: int, l: int) -> int:
    n = _lib.fmg1d_size(p, m, l)
    if n < 0:
        raise FmgError(FMG_EINVAL, "fmg1d_size")
    return n


def fmg1d_operator(p: int, m: int, l: int):
    """Native band of A_l, shape (n_l, 2p+1) (host assembly)."""
    import numpy as np
    a = np.zeros((fmg1d_size(p, m, l), 2 * p + 1))
    _check(_lib.fmg1d_assemble_operator(p, m, l, a.ctypes.data), "fmg1d_assemble_operator")
    return a


def fmg1d_prolongation(p: int, m: int, l: int):
    """Native ELL values of P_l, shape (n_l, kp_l) (host assembly)."""
    import numpy as np
    a = np.zeros((fmg1d_size(p, m, l), _lib.fmg1d_ell_width(p, m, l)))
    _check(_lib.fmg1d_assemble_prolongation(p, m, l, a.ctypes.data), "fmg1d_assemble_prolongation")
    return a


def fmg1d_load(p: int, m: int, l: int):
    """Native load vector of the paper's manufactured problem at level l."""
    import numpy as np
    a = np.zeros(fmg1d_size(p, m, l))
    _check(_lib.fmg1d_assemble_load(p, m, l, a.ctypes.data), "fmg1d_assemble_load")
    return a


def _ptr_array(arrs):
    return (_vp * len(arrs))(*[None if a is None else a.ctypes.data for a in arrs])


class Solver1D:
    """A batch of 1D B-spline compact-FMG problems (fmg1d_create ... fmg1d_destroy).
    Ab / Pv / A0inv: operator arrays in the layouts of include/fmg1d.h, or None
    for the library's native assembly."""

    def __init__(self, p: int, m: int, levels: int, N: int, b1: int, b2: int, smoother: str = "lex",
                 batch: int = 1, Ab=None, Pv=None, A0inv=None, stream=None):
        import numpy as np
        self.p, self.m, self.levels, self.batch = p, m, levels, batch
        self.n = [fmg1d_size(p, m, l) for l in range(levels)]
        self.sched = Schedule1D(N, b1, b2, FMG1D_LEX if smoother == "lex" else FMG1D_MCGS)
        keep = []
        ab = pv = None
        if Ab is not None:
            keep += [np.ascontiguousarray(a, dtype=np.float64) for a in Ab]
            ab = _ptr_array(keep[-len(Ab):])
        if Pv is not None:
            pvs = [None if a is None else np.ascontiguousarray(a, dtype=np.float64) for a in Pv]
            keep += [a for a in pvs if a is not None]
            pv = _ptr_array(pvs)
        a0 = None
        if A0inv is not None:
            a0 = np.ascontiguousarray(A0inv, dtype=np.float64)
            keep.append(a0)
        h = _vp()
        _check(_lib.fmg1d_create(p, m, levels, C.byref(self.sched), batch, ab, pv,
                                 None if a0 is None else a0.ctypes.data, _stream_ptr(stream), C.byref(h)),
               "fmg1d_create")
        self._h = h

    def set_load(self, f):
        """f[l]: (batch, n_l) or (n_l,) (broadcast over the batch) host arrays."""
        import numpy as np
        self._f = [np.ascontiguousarray(np.broadcast_to(np.asarray(v, dtype=np.float64), (self.batch, self.n[l])))
                   for l, v in enumerate(f)]
        _check(_lib.fmg1d_set_load(self._h, _ptr_array(self._f)), "fmg1d_set_load")

    def solve_async(self):
        _check(_lib.fmg1d_solve_async(self._h), "fmg1d_solve_async")

    def sync(self):
        _check(_lib.fmg1d_sync(self._h), "fmg1d_sync")

    def solve(self):
        self.solve_async()
        self.sync()

    def solve_host(self, f, out=None):
        """End to end: host loads in, host solutions (batch, n_L) out."""
        import numpy as np
        self._f = [np.ascontiguousarray(np.broadcast_to(np.asarray(v, dtype=np.float64), (self.batch, self.n[l])))
                   for l, v in enumerate(f)]
        if out is None:
            out = np.zeros((self.batch, self.n[-1]))
        _check(_lib.fmg1d_solve_host(self._h, _ptr_array(self._f), out.ctypes.data), "fmg1d_solve_host")
        return out

    def solution(self, b: int = 0):
        import numpy as np
        u = np.zeros(self.n[-1])
        _check(_lib.fmg1d_solution(self._h, b, u.ctypes.data), "fmg1d_solution")
        return u

    def section(self, which: int, l: int, b: int = 0):
        """(mant, exps, w) of section which (0 u, 1 r, 2 y) at level l."""
        import numpy as np
        nblk = (self.n[l] + 31) // 32
        mant = np.zeros(nblk * 64, dtype=np.uint32)
        exps = np.zeros(nblk, dtype=np.int8)
        w = C.c_int()
        _check(_lib.fmg1d_section(self._h, which, l, b, mant.ctypes.data, exps.ctypes.data, C.byref(w)),
               "fmg1d_section")
        return mant[: nblk * w.value], exps, w.value

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.fmg1d_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
