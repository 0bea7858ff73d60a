"""CPU-side checks of the C-ABI boundary: the library builds for sm_100a,
loads without a GPU, and exports every entry point include/itsk_b200.h declares."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "itsk_b200.h")


def _ensure_built():
    from paper_2311_04362_b200 import build

    return build.build()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(itsk_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_entry_points():
    names = declared_functions()
    for must in ("itsk_sparse_sign_pattern", "itsk_sketch", "itsk_qr_aug", "itsk_trsv", "itsk_trsv_pair",
                 "itsk_normest", "itsk_condest", "itsk_fused_pass", "itsk_loop_begin", "itsk_loop_step_pre",
                 "itsk_loop_step_post", "itsk_loop_graph_create", "itsk_loop_graph_launch"):
        assert must in names


def test_library_loads_and_exports_every_symbol():
    path = _ensure_built()
    lib = ctypes.CDLL(path)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    for n in declared_functions():
        assert re.search(rf"\bT {n}$", out, flags=re.M), n


def test_python_binding_covers_header():
    from paper_2311_04362_b200 import _lib

    assert set(declared_functions()) == set(_lib.exported_symbols())
    lib = _lib.load()
    assert lib.itsk_version() >= 100


def test_sm100a_cubin_only():
    path = _ensure_built()
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out


def test_no_device_is_reported_not_faked():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2311_04362_b200 import _lib

    lib = _lib.load()
    assert lib.itsk_device_check(0) != 0
    from paper_2311_04362_b200 import SolverConfig, gen_randsvd, iterative_sketching

    p = gen_randsvd(200, 5, 10.0, 1e-3, 0)
    with pytest.raises(RuntimeError):
        iterative_sketching(p.a, p.b, SolverConfig(d=50))


def test_workspace_queries_without_device():
    from paper_2311_04362_b200 import _lib

    lib = _lib.load()
    b = ctypes.c_int64()
    assert lib.itsk_pattern_workspace(4000, 200000, 8, ctypes.byref(b)) == 0 and b.value > 0
    assert lib.itsk_qr_workspace(4000, 200, ctypes.byref(b)) == 0 and b.value > 0
    assert lib.itsk_pattern_workspace(3, 10, 4, ctypes.byref(b)) == _lib.ITSK_EINVAL
    assert b"zeta" in lib.itsk_last_error() or lib.itsk_last_error()


def test_ctypes_structs_match_the_compiled_abi():
    """The ctypes mirrors of the parameter structs have the sizes the library
    was compiled with (a field added on one side only would shift every
    later field)."""
    import ctypes

    from paper_2311_04362_b200 import _lib

    lib = _lib.load()
    assert lib.itsk_struct_size(0) == ctypes.sizeof(_lib.LoopParams)
    assert lib.itsk_struct_size(1) == ctypes.sizeof(_lib.LoopResult)
    assert lib.itsk_struct_size(2) == ctypes.sizeof(_lib.PeerParams)
    assert lib.itsk_struct_size(7) == -1
