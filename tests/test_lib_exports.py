"""CPU checks of the C-ABI boundary: libfmg.so loads (no GPU needed for dlopen)
and exports every function include/*.h declares; the oracle library builds.
No compute calls are made here."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    inc = os.path.join(ROOT, "include")
    src = "".join(open(os.path.join(inc, h)).read() for h in sorted(os.listdir(inc)) if h.endswith(".h"))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(\w+)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n.startswith(("fmg_", "bfp_", "fmg1d_"))))


def test_header_declares_boundary():
    names = declared_functions()
    for n in ["fmg_create", "fmg_solve", "fmg_residual", "bfp_encode", "bfp_decode", "fmg_destroy",
              "fmg1d_create", "fmg1d_solve_async", "fmg1d_section", "fmg1d_assemble_operator"]:
        assert n in names


def test_libfmg_exports_every_declared_symbol():
    so = os.path.join(ROOT, "paper_2511_19036_b200", "libfmg.so")
    assert os.path.exists(so), "libfmg.so not built"
    lib = ctypes.CDLL(so)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_export_list_matches_header():
    import paper_2511_19036_b200 as P
    assert sorted(P.EXPORTS) == declared_functions()


def test_strerror_and_argument_validation_without_gpu():
    import paper_2511_19036_b200 as P
    lib = P._lib
    assert lib.fmg_strerror(0) == b"ok"
    # argument validation happens before any device call
    s = P.Schedule(4, 2, 4, 1, 3, 2, 1.575, 4.0)
    h = ctypes.c_void_p()
    assert lib.fmg_create(4, 1, 5, ctypes.byref(s), None, ctypes.byref(h)) == P.FMG_EINVAL
    assert lib.fmg_create(2, 4, 5, ctypes.byref(s), None, ctypes.byref(h)) == P.FMG_EINVAL
    bad = P.Schedule(50, 2, 4, 1, 3, 2, 1.575, 4.0)  # w_u(0,L) > 54
    assert lib.fmg_create(2, 1, 5, ctypes.byref(bad), None, ctypes.byref(h)) == P.FMG_EINVAL
    assert lib.bfp_encode(None, 31, 4, None, None, None) == P.FMG_EINVAL
    assert lib.bfp_encode(None, 32, 55, None, None, None) == P.FMG_EINVAL
    assert lib.bfp_decode(None, None, 32, 1, None, None) == P.FMG_EINVAL
    assert lib.bfp_encode(None, 0, 4, None, None, None) == P.FMG_OK
