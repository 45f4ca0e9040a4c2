"""CPU checks of the drop-in boundary: the sm_100a library loads and exports every
entry point include/*.h declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    inc = os.path.join(ROOT, "include")
    for name in os.listdir(inc):
        if name.endswith(".h"):
            text = open(os.path.join(inc, name)).read()
            text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
            syms |= set(re.findall(r"\b(rtn_[a-z0-9_]+)\s*\(", text))
    return syms


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("rtn_ctx_create", "rtn_apply_normal", "rtn_cg_solve", "rtn_newton_step",
                 "rtn_reconstruct_frame", "rtn_fft2", "rtn_make_weights_inv"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    import paper_1701_08361_b200 as pb
    lib = pb.load_library()
    missing = [s for s in sorted(declared_symbols()) if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.rtn_abi_version() == 1


def test_compute_fails_loudly_without_gpu():
    import paper_1701_08361_b200 as pb
    lib = pb.load_library()
    if lib.rtn_device_count() > 0:
        return  # on a GPU box the gpu-marked tests cover this path
    plan = pb.raw_plan(16, 1)
    try:
        pb.Context(plan)
    except RuntimeError as e:
        assert "CUDA" in str(e) or "device" in str(e)
    else:
        raise AssertionError("context creation succeeded without a GPU")


def test_size_coverage_table():
    import paper_1701_08361_b200 as pb
    lib = pb.load_library()
    for G in (16, 24, 32, 48, 64, 72, 96, 128, 160, 192, 256, 320, 384, 512):
        assert lib.rtn_grid_supported(G) == 1, G
    for G in (34, 130, 1000):
        assert lib.rtn_grid_supported(G) == 0, G


def test_cpp_drop_in_links_against_the_c_abi():
    """the C++ drop-in (the reference's nlinv.hpp / fft.hpp API over include/rtnlinv_b200.h)
    is built and defines the reference's hot-path symbols; no device call is made"""
    import subprocess
    so = os.path.join(ROOT, "paper_1701_08361_b200", "compat", "_build", "librtnlinv_compat.so")
    if not os.path.exists(so):
        import pytest
        pytest.skip("compat library not built (needs the reference headers)")
    syms = subprocess.run(["nm", "-DC", "--defined-only", so], capture_output=True, text=True).stdout
    for name in ("rtnlinv::apply_normal(", "rtnlinv::cg_solve(", "rtnlinv::newton_step(",
                 "rtnlinv::reconstruct_frame(", "rtnlinv::reconstruct_series(", "rtnlinv::make_step_cache(",
                 "rtnlinv::fft::forward(", "rtnlinv::fft::count("):
        assert name in syms, name
    deps = subprocess.run(["ldd", so], capture_output=True, text=True).stdout
    assert "librtnlinv_b200.so" in deps
