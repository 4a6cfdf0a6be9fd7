"""The C-ABI library loads and exports every symbol include/*.h declares.

No compute is called here (no GPU in the build container); the GPU tests
exercise every entry point.
"""
import ctypes
import glob
import os
import re

import pytest

from paper_1912_02165_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    names = set()
    for hdr in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(hdr).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(wf_[a-z0-9_]+)\s*\(", text))
    return names


def test_header_declares_the_bound_api():
    declared = _declared_symbols()
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared_symbols():
        assert hasattr(lib, name), name


def test_binding_loads_and_reports_version():
    lib = _lib.load()
    assert lib.wf_version() >= 100
    assert isinstance(_lib.last_error(), str)


def test_scratch_queries_need_no_gpu():
    spec = _lib.wf_layer(64, 64, 64, 56, 56, 3, 1, 1)
    lib = _lib.load()
    # 36 positions x 98 blocks x (bf16 hi/lo U slab + f32 M)
    u = 36 * 98 * 2 * 128 * 64 * 2
    m = 36 * 64 * 98 * 128 * 4
    assert lib.wf_three_stage_scratch_bytes(ctypes.byref(spec), 6, 0) == u + m
    assert lib.wf_three_stage_scratch_bytes(ctypes.byref(spec), 9, 0) == 0
    assert lib.wf_mma_pack_bytes(6, 64, 64, 0) == 36 * 2 * 64 * 64 * 2


def test_status_codes_map_to_reference_errors():
    import paper_1912_02165_b200 as wf
    with pytest.raises(wf.InvalidParameterError):
        _lib.check(_lib.WF_ERR_PARAM, "x")
    with pytest.raises(wf.ShapeMismatchError):
        _lib.check(_lib.WF_ERR_SHAPE, "x")
    with pytest.raises(wf.UnsupportedConfigError):
        _lib.check(_lib.WF_ERR_UNSUPPORTED, "x")
    with pytest.raises(wf.NativeLibraryError):
        _lib.check(_lib.WF_ERR_CUDA, "x")
    _lib.check(_lib.WF_OK, "x")


def test_missing_library_fails_loudly(tmp_path):
    import paper_1912_02165_b200 as wf
    saved = _lib._lib
    try:
        _lib._lib = None
        with pytest.raises(wf.NativeLibraryError):
            _lib.load(str(tmp_path / "nope.so"))
    finally:
        _lib._lib = saved
