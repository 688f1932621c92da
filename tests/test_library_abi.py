"""The C-ABI library loads and exports every symbol include/domdec_b200.h declares (CPU)."""

import ctypes
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    text = open(os.path.join(ROOT, "include", "domdec_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(dd3?_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = declared()
    assert "dd_cell_solve" in names and "dd_grid_lse" in names
    assert len(names) >= 20


def test_library_exports_every_declared_symbol():
    from paper_2410_08859_b200 import _lib

    h = _lib.load()
    for name in declared():
        assert hasattr(h, name), name
    assert set(declared()) <= set(_lib.EXPORTS) | {"dd_set_error"}
    assert h.dd_abi_version() == 1


def test_workspace_layout_matches_python_mirror():
    from paper_2410_08859_b200 import _lib
    from paper_2410_08859_b200.engine import _ws_total

    h = _lib.load()
    for nw0, nw1, ny0, ny1 in [(8, 8, 20, 20), (16, 16, 40, 37), (1, 4, 1, 32), (2, 2, 9, 1)]:
        assert h.dd_cell_ws_size(nw0, nw1, ny0, ny1) == int(
            _ws_total(nw0, nw1, np.array([ny0]), np.array([ny1]))[0])


def test_product_path_refuses_without_device():
    import pytest
    from paper_2410_08859_b200 import _lib

    h = _lib.load()
    if h.dd_device_count() > 0:
        pytest.skip("a device is visible")
    with pytest.raises(_lib.LibraryError):
        _lib.lib()


def test_cluster_workspace_layout_matches_python_mirror():
    from paper_2410_08859_b200 import _lib
    from paper_2410_08859_b200.engine import _cluster_ws

    h = _lib.load()
    for nw0, nw1, ny0, ny1, c in [(16, 16, 140, 150, 8), (8, 8, 30, 40, 2), (16, 16, 33, 17, 16)]:
        assert h.dd_cell_cluster_ws(nw0, nw1, ny0, ny1, c) == int(
            _cluster_ws(nw0, nw1, np.array([ny0]), np.array([ny1]), c)[0])


def test_three_axis_workspace_layout_matches_python_mirror():
    from paper_2410_08859_b200 import _lib
    from paper_2410_08859_b200.volume import _i32, _ws_total

    h = _lib.load()
    for w, n in [((8, 8, 8), (20, 21, 19)), ((1, 4, 4), (1, 9, 12)), ((1, 1, 2), (1, 1, 7))]:
        got = h.dd3_cell_ws_size(_i32(w), _i32(n))
        want = int(_ws_total(w, np.array([n[0]]), np.array([n[1]]), np.array([n[2]]))[0])
        assert got == want
