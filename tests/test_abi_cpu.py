"""CPU-side checks of the C ABI boundary (no GPU compute): the library builds
and loads, exports every entry point declared in include/afn.h, and rejects
bad arguments without touching memory."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "afn.h")
LIB = os.path.join(ROOT, "paper_2304_05460_b200", "libafn.so")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import importlib.util
        spec = importlib.util.spec_from_file_location(
            "afn_build", os.path.join(ROOT, "paper_2304_05460_b200", "build.py"))
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        mod.build()
    import paper_2304_05460_b200 as afn
    return afn


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:afn_status|void|int64_t|int32_t|const char\*)\s+(\w+)\s*\(", src, re.M)
    return sorted(set(names))


def test_header_declares_the_north_star_calls():
    names = header_functions()
    for required in ("kernel_matvec", "afn_build", "afn_apply", "afn_pcg_solve"):
        assert required in names


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [n for n in header_functions() if n not in exported]
    assert not missing, missing
    # the binding wraps exactly the declared set
    assert set(lib.EXPORTED) == set(header_functions())


def test_abi_version_and_struct_layout(lib):
    import ctypes as C
    assert lib.abi_version() == 6
    # afn_params: 2 doubles, int64, 4 int32, int64, uint64, 4 int32 = 72 bytes
    assert C.sizeof(lib.Params) == 72
    assert C.sizeof(lib.Info) == 8 * 4 + 4 * 4 + 8 * 9 + 4 * 2 + 8 * 4 + 4 * 2 + 4 * 2 + 8 * 4
    # (kmv_plan, kmv_reserved; kmv_units64/32, kmv_pairs64/32)
    assert C.sizeof(lib.Report) == 4 * 4 + 8 * 6 + 8


def test_host_pointers_are_rejected_without_compute(lib):
    import ctypes as C
    import numpy as np
    X = np.zeros((4, 3))
    v = np.zeros(4)
    y = np.zeros(4)
    st = lib._lib.kernel_matvec(X.ctypes.data_as(C.c_void_p), 4, 3, 0, 1.0, 1e-4,
                                v.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), None)
    assert st == 1  # AFN_ERR_ARG
    assert b"device pointer" in lib._lib.afn_last_error()
    # bad sizes are rejected first
    st = lib._lib.kernel_matvec(None, 0, 3, 0, 1.0, 1e-4, None, None, None)
    assert st == 1
    h = C.c_void_p()
    p = lib.make_params(1.0, 1e-4, 10, lib.W_MAX + 1)  # w > AFN_W_MAX
    st = lib._lib.afn_build(X.ctypes.data_as(C.c_void_p), 4, 3, C.byref(p), None, C.byref(h))
    assert st == 1 and not h.value
    # allocator: alloc and free must come together; NULL/NULL restores the pool
    fake = C.cast(lib._ALLOC_FN(lambda n, s, c: None), C.c_void_p)
    assert lib._lib.afn_set_allocator(fake, None, None) == 1
    assert lib._lib.afn_set_allocator(None, None, None) == 0
    # CG on host pointers: rejected before any compute
    b = np.zeros(4)
    st = lib._lib.afn_cg_solve(None, X.ctypes.data_as(C.c_void_p), 4, 3, 0, 1.0, 1e-4,
                               b.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), 1e-4, 10, 0,
                               None, None)
    assert st == 1


def test_cutoff_mode_and_w_product_arguments(lib):
    """afn_set_cutoff_mode takes 0..3 only; afn_w_product
    returns AFN_ERR_ARG, without computing, for bad arguments (here host
    pointers, an unknown method, the cutoff method with d > 3)."""
    import ctypes as C
    for m in (0, 1, 2, 3):
        assert lib._lib.afn_set_cutoff_mode(m) == 0
    for m in (-1, 4, 99):
        assert lib._lib.afn_set_cutoff_mode(m) == 1  # AFN_ERR_ARG
    assert lib._lib.afn_set_cutoff_mode(0) == 0
    assert lib.WPROD_CUT == 2
    # (host pointers: argument checks come first, no compute without a GPU)
    import numpy as np
    X1, Xr, Li, W = np.zeros((4, 3)), np.zeros((8, 3)), np.eye(4), np.zeros((8, 4))
    P = lambda a: a.ctypes.data_as(C.c_void_p)
    assert lib._lib.afn_w_product(P(X1), 4, P(Xr), 8, 3, 0, 1.0, P(Li), 7, P(W), None) == 1
    X1b, Xrb = np.zeros((4, 5)), np.zeros((8, 5))
    assert lib._lib.afn_w_product(P(X1b), 4, P(Xrb), 8, 5, 0, 1.0, P(Li), 2, P(W), None) == 1


def test_binding_has_no_cpu_fallback():
    """The product package never imports the oracle and never computes on the host."""
    pkg = os.path.join(ROOT, "paper_2304_05460_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in src.replace("oracle/", ""), fn
            assert "import numpy" not in src or fn == "__init__.py"
