"""The C-ABI library builds for sm_100a, loads, and exports every entry
point declared in include/dlrsn.h (no GPU needed)."""

import ctypes
import os
import re

from conftest import REPO
from paper_2601_18705_b200 import _lib
from paper_2601_18705_b200.build import build


def header_functions():
    text = open(os.path.join(REPO, "include", "dlrsn.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(dlrsn_\w+)\s*\(", text, re.M)))


def test_library_builds_and_exports_header():
    path = build()
    lib = ctypes.CDLL(path)
    names = header_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(names) == _lib.exported_symbols()


def test_host_layout_queries_without_gpu():
    lib = _lib.load()
    assert lib.dlrsn_version() >= 1
    # SK slab sizes: strips of 32 rows, nx+31 skewed steps, 4 dofs per lane
    assert lib.dlrsn_sk_vec_len(70, 70) == 3 * (70 + 31) * 128
    assert lib.dlrsn_sk_scalar_len(5, 33) == 2 * 36 * 32
    assert lib.dlrsn_sweep_workspace_bytes(10, 40, 3, 2) >= 2 * 3 * 10 * 2 * 2 * 8


def test_group_struct_matches_c_layout():
    # struct dlrsn_group: 2 ints + 8 ints + 3*8 doubles, 8-byte aligned
    assert _lib.GROUP_DTYPE.itemsize == 4 * 10 + 8 * 24
    assert ctypes.sizeof(_lib.CellOps) == 2 * 4 + 8 * (4 + 16 * 3 + 4 * 3)
