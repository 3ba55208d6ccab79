"""CPU-side checks of the C-ABI library: it loads and exports every symbol
include/dfx.h declares (no compute calls without a GPU)."""

import ctypes
import os
import re

from paper_2110_10802_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dfx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dfx_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header():
    lib = _lib.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_header():
    assert sorted(declared_symbols()) == sorted(_lib.EXPORTED)


def test_gemm_args_layout_matches_header():
    # 4 int32 + 5 int64 + (ptr + 4 int64) * 2 + ptr + 3 int64 + 2 float + ptr + (ptr + 3 int64) * 2
    assert ctypes.sizeof(_lib.GemmArgs) == 4 * 4 + 5 * 8 + 2 * 40 + 32 + 8 + 8 + 2 * 32 + 16


def test_cpu_only_calls_do_not_need_gpu():
    lib = _lib.load()
    assert lib.dfx_version() == 1
    assert lib.dfx_bdrln_bwd_workspace(4096, 768) > 0
    assert lib.dfx_colsum_workspace(4096, 768) > 0
