"""CPU-side checks of the C ABI: the library builds, loads, and exports every
symbol include/probestream.h declares (no compute calls without a GPU)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "probestream.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(ps_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))


@pytest.fixture(scope="module")
def libpath():
    from paper_2103_05875_b200 import build_native

    return build_native.build()


def test_header_declares_entry_points():
    names = declared_functions()
    for must in ("ps_detect_changed", "ps_select", "ps_assign_slots", "ps_build_update",
                 "ps_pack_color", "ps_pack_visibility", "ps_pack_delta", "ps_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(str(libpath))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_shim_binds_every_declared_symbol(libpath):
    from paper_2103_05875_b200 import _native

    bound = set(_native.exported_symbols())
    assert set(declared_functions()) <= bound
    lib = _native.lib()
    assert lib.ps_abi_version() == _native.ABI_VERSION
    assert lib.ps_widened_width(3) == 4 and lib.ps_widened_width(18) == 24
    assert lib.ps_widened_width(0) == 0 and lib.ps_widened_width(-1) == -1


def test_workspace_queries_are_pure(libpath):
    from paper_2103_05875_b200 import _native

    lib = _native.lib()
    for n in (1, 31, 32, 33, 131072):
        assert lib.ps_detect_workspace_bytes(n) > 0
        assert lib.ps_select_workspace_bytes(n) >= lib.ps_compact_workspace_bytes(n)
        assert lib.ps_assign_workspace_bytes(n, max(1, n // 2)) > 0


def test_errors_map_to_reference_classes(libpath):
    from paper_2103_05875_b200 import _native
    from paper_2103_05875_b200.errors import LayoutMismatchError, SlotOverflowError

    # a layout error raised before any launch (block_rows inconsistent)
    lib = _native.lib()
    st = lib.ps_detect_changed(0, None, None, 10, 4, 7, None, 0.0, 0, None, None, None, None, 0, None)
    assert st == _native.PS_ERR_LAYOUT
    with pytest.raises(LayoutMismatchError):
        _native.check(st)
    assert issubclass(LayoutMismatchError, ValueError)
    assert issubclass(SlotOverflowError, RuntimeError)
    st = lib.ps_pack_color(None, -1, 3, 3, None, None)
    with pytest.raises(ValueError):
        _native.check(st)
