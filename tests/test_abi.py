"""CPU-side checks of the C-ABI library: it builds, loads, exports every
symbol include/swdb.h declares, and validates arguments before touching the
GPU.  No compute call is made here (no GPU in this container)."""
import os
import re

import numpy as np
import pytest

import paper_1702_07195_b200 as sw
from paper_1702_07195_b200 import build as swbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    swbuild.build()
    return sw.load_library()


def _header_functions():
    text = open(os.path.join(ROOT, "include", "swdb.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sw_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    names = _header_functions()
    for n in ("sw_db_load", "sw_search", "sw_topk", "sw_search_dev", "sw_db_free", "sw_last_error"):
        assert n in names


def test_library_exports_every_header_symbol(lib):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", sw.library_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (sw_[a-z0-9_]+)", out))
    missing = [n for n in _header_functions() if n not in exported]
    assert not missing, missing
    assert set(sw.EXPORTS) == set(_header_functions())


def test_version_and_error_string(lib):
    assert "sm_100a" in sw.sw_version()
    assert isinstance(sw.sw_last_error(), str)


@pytest.mark.parametrize("res,offs,msg", [
    (np.array([1, 2, 3], np.uint8), np.array([0, 3, 2]), "non-decreasing"),
    (np.array([1, 2, 24], np.uint8), np.array([0, 3]), "code >= 24"),
    (np.array([1, 2, 3], np.uint8), np.array([1, 3]), "offsets[0]"),
    (np.array([], np.uint8), np.array([0]), "count"),
])
def test_db_load_validation(lib, res, offs, msg):
    with pytest.raises(sw.SWError) as e:
        sw.sw_db_load(res, offs)
    assert e.value.code == -1
    assert msg in str(e.value)


def test_streamed_load_validation(lib):
    with pytest.raises(sw.SWError) as e:
        sw.sw_db_load_streamed(np.array([1, 2, 3], np.uint8), np.array([0, 3]), 0)
    assert e.value.code == -1


def test_search_before_load_is_enodb(lib):
    sw.sw_db_free()
    with pytest.raises(sw.SWError) as e:
        sw.sw_search(np.array([0, 1], np.uint8), np.zeros((24, 24), np.int8), 10, 2)
    assert e.value.code == -4
    with pytest.raises(sw.SWError) as e:
        sw.sw_topk(5)
    assert e.value.code == -5


def test_tile_table(lib):
    assert sw.sw_tile_supported(32, 16)
    assert not sw.sw_tile_supported(7, 16)
    with pytest.raises(sw.SWError):
        sw.sw_set_tile(7, 16)
    sw.sw_set_tile(0)


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    import paper_1702_07195_b200.swdb as mod
    monkeypatch.setattr(mod, "_lib", None)
    monkeypatch.setattr(mod, "LIB", str(tmp_path / "nope.so"))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mod.load_library()
