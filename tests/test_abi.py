"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/apsp_warm.h declares; its pure host functions (layout, workspace
size, status strings) behave as documented.  No kernel is launched here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "apsp_warm.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:apsp_status|size_t|int64_t|int32_t|const char\*)\s+(\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def L():
    from paper_2412_15122_b200 import _lib
    return _lib


def test_header_declares_north_star_calls():
    names = declared_functions()
    for f in ["apsp_cold_fw", "apsp_add_node", "apsp_remove_node", "apsp_update_edge", "sp_pair_query"]:
        assert f in names


def test_library_exports_every_declared_symbol(L):
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(L.lib, name), name
    assert sorted(L.SYMBOLS) == names


def test_layout_partition(L):
    ld, r0, rows = L.apsp_layout(1000, 1, 0)
    assert (ld, r0, rows) == (1024, 0, 1000)
    for world in (2, 3, 4, 8):
        covered = []
        for rank in range(world):
            ld, r0, rows = L.apsp_layout(32768 + 64, world, rank)
            assert ld % 32 == 0 and r0 % 128 == 0
            covered.extend(range(r0, r0 + rows))
        assert covered == list(range(32768 + 64))
    with pytest.raises(L.ApspError):
        L.apsp_layout(0, 1, 0)
    with pytest.raises(L.ApspError):
        L.apsp_layout(10, 2, 2)


def test_workspace_bytes(L):
    a = L.apsp_workspace_bytes(L.APSP_I32, 1000)
    b = L.apsp_workspace_bytes(L.APSP_I32, 2000)
    assert a >= 4 * 1000 * 1024 and b > a
    assert L.apsp_workspace_bytes(7, 1000) == 0
    # every rank holds the whole WT replica (cap x ld) whatever its share of D
    assert L.apsp_workspace_bytes(L.APSP_F32, 1000, 4) >= 4 * 1000 * 1024


def test_status_strings(L):
    for s in range(10):
        assert L.lib.apsp_status_string(s)
    # null-handle calls are rejected without touching a device
    assert L.lib.apsp_cold_fw(None) == 1
    assert L.lib.apsp_size(None) == -1
    info = L.UpdateInfo()
    assert ctypes.sizeof(info) == 4 * 4 + 8 * 3 + 8 + 8
