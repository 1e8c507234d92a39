"""The C ABI library loads and exports every entry point ``include/glsim_cuda.h``
declares (no device calls: runs on the CPU-only build box too)."""

import ctypes
import os
import re

import pytest

from paper_2203_06117_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "glsim_cuda.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_native.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build_native()
    return ctypes.CDLL(_native.LIB_PATH)


def test_header_declares_the_engine():
    syms = declared_symbols()
    for s in ("gs_design_create", "gs_stim_create", "gs_engine_create", "gs_run_stats",
              "gs_run_arena", "gs_dwell_sweep", "gs_init_values", "gs_last_error"):
        assert s in syms


def test_every_declared_symbol_is_exported(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_the_header():
    assert sorted(_native.SIGNATURES) == declared_symbols()


def test_version_and_error_string_without_device(lib):
    lib.gs_version.restype = ctypes.c_int
    assert lib.gs_version() >= 1
    lib.gs_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.gs_last_error(), bytes)


def test_library_is_built_for_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
