"""ctypes binding of the sm_100a C ABI (include/winofuse_b200.h).

The library is built in-tree (``make`` or ``__graft_entry__.build()``) as
``paper_1912_02165_b200/libwinofuse_b200.so``.  There is deliberately no
fallback: if the library is missing every GPU entry point raises
:class:`NativeLibraryError`.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (InvalidParameterError, NativeLibraryError, ShapeMismatchError,
                     UnsupportedConfigError, WinofuseError)

LIB_NAME = "libwinofuse_b200.so"
LIB_PATH = os.environ.get("WF_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

WF_OK, WF_ERR_PARAM, WF_ERR_SHAPE, WF_ERR_UNSUPPORTED, WF_ERR_CUDA, WF_ERR_SCRATCH = range(6)
WF_WINOGRAD, WF_FFT16 = 0, 1
WF_PREC_3XBF16, WF_PREC_BF16, WF_PREC_3XFP16 = 0, 1, 2
WF_PHASE_FORWARD, WF_PHASE_MULTIPLY, WF_PHASE_INVERSE = 1, 2, 4
WF_FUSED_AUTO, WF_FUSED_WS, WF_FUSED_ITEMQ, WF_FUSED_WAVES, WF_FUSED_WS_ROW = 0, 1, 2, 3, 4
WF_FUSED_COUNTERS_CLEAN, WF_FUSED_INSTRUMENT = 1, 2

PRECISIONS = {"3xbf16": WF_PREC_3XBF16, "bf16": WF_PREC_BF16, "3xfp16": WF_PREC_3XFP16}
# operand format of the device MMA pack per precision mode
PACK_FORMAT = {"3xbf16": "bf16", "bf16": "bf16", "3xfp16": "fp16"}
TRANSFORMS = {"winograd": WF_WINOGRAD, "fft": WF_FFT16}
# fused-engine variants (EngineConfig.fused_variant <-> WF_FUSED_*)
VARIANTS = {"auto": WF_FUSED_AUTO, "ws": WF_FUSED_WS, "itemq": WF_FUSED_ITEMQ, "waves": WF_FUSED_WAVES,
            "ws_row": WF_FUSED_WS_ROW}
VARIANT_NAMES = {v: k for k, v in VARIANTS.items()}


class wf_layer(ctypes.Structure):
    """Mirror of the C struct (and of LayerSpec, reference tensor.py:36-78)."""

    _fields_ = [(name, ctypes.c_int) for name in
                ("batch", "in_channels", "out_channels", "height", "width", "kernel",
                 "pad_lo", "pad_hi")]


class wf_fused_opts(ctypes.Structure):
    """Mirror of the C struct wf_fused_opts (zero = defaults)."""

    _fields_ = [("variant", ctypes.c_int), ("flags", ctypes.c_int), ("ring_bytes", ctypes.c_size_t),
                ("lag", ctypes.c_int), ("gbatch", ctypes.c_int)]


_vp, _i, _sz, _fp = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p
_LP = ctypes.POINTER(wf_layer)
_OP = ctypes.POINTER(wf_fused_opts)
_IP = ctypes.POINTER(ctypes.c_int)
_ULLP = ctypes.POINTER(ctypes.c_ulonglong)

# name -> (restype, argtypes); the exported symbol set checked by the tests.
SIGNATURES = {
    "wf_version": (_i, []),
    "wf_last_error": (ctypes.c_char_p, []),
    "wf_device_sm_count": (_i, []),
    "wf_kernel_launches": (ctypes.c_ulonglong, []),
    "wf_filter_transform": (_i, [_fp, _fp, _i, _i, _i, _vp]),
    "wf_mma_pack_bytes": (_sz, [_i, _i, _i, _i]),
    "wf_mma_pack": (_i, [_fp, _vp, _i, _i, _i, _i, _vp]),
    "wf_mma_pack_ex": (_i, [_fp, _vp, _i, _i, _i, _i, _i, _vp]),
    "wf_three_stage_scratch_bytes": (_sz, [_LP, _i, _i]),
    "wf_conv_three_stage": (_i, [_fp, _vp, _fp, _vp, _sz, _LP, _i, _i, _i, _vp]),
    "wf_conv_three_stage_phases": (_i, [_fp, _vp, _fp, _vp, _sz, _LP, _i, _i, _i, _i, _vp]),
    "wf_fused_scratch_bytes": (_sz, [_LP, _i, _i, _i]),
    "wf_fused_scratch_bytes_ex": (_sz, [_LP, _i, _i, _OP]),
    "wf_fused_variant": (_i, [_LP, _i, _i, _OP]),
    "wf_conv_fused": (_i, [_fp, _vp, _fp, _vp, _sz, _LP, _i, _i, _i, _i, _vp]),
    "wf_conv_fused_ex": (_i, [_fp, _vp, _fp, _vp, _sz, _LP, _i, _i, _i, _OP, _IP, _vp]),
    "wf_conv_fused_planned": (_i, [_fp, _vp, _fp, _vp, _sz, _LP, _i, _i, _i, _i, _vp]),
    "wf_fused_instrument_read": (_i, [_LP, _i, _i, _OP, _ULLP, _i, _ULLP, _IP]),
    "wf_conv_direct": (_i, [_fp, _fp, _fp, _LP, _vp]),
    "wf_forward_tiles": (_i, [_fp, _fp, _LP, _i, _i, _i, _i, _i, _vp]),
    "wf_multiply_positions": (_i, [_fp, _fp, _fp, _i, _i, _i, _i, _i, _vp]),
    "wf_inverse_tiles": (_i, [_fp, _fp, _LP, _i, _i, _i, _i, _i, _vp]),
}

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and return the native library; raise if it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeLibraryError(
                f"{LIB_NAME} not found at {path}; build it with `make` or "
                f"__graft_entry__.build() (there is no CPU fallback)")
        try:
            lib = ctypes.CDLL(path)
        except OSError as exc:
            raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().wf_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    """Map a WF_ERR_* status to the reference's exception types."""
    if rc == WF_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == WF_ERR_PARAM:
        raise InvalidParameterError(msg)
    if rc == WF_ERR_SHAPE:
        raise ShapeMismatchError(msg)
    if rc == WF_ERR_UNSUPPORTED:
        raise UnsupportedConfigError(msg)
    if rc in (WF_ERR_CUDA, WF_ERR_SCRATCH):
        raise NativeLibraryError(msg)
    raise WinofuseError(msg)


def layer_struct(spec) -> wf_layer:
    return wf_layer(spec.batch, spec.in_channels, spec.out_channels, spec.height, spec.width,
                    spec.kernel, spec.pad_lo, spec.pad_hi)


def fused_opts(variant: str = "auto", flags: int = 0, ring_bytes: int | None = None, lag: int = 0,
               gbatch: int = 0) -> wf_fused_opts:
    if variant not in VARIANTS:
        raise InvalidParameterError(f"unknown fused variant {variant!r} (one of {sorted(VARIANTS)})")
    return wf_fused_opts(VARIANTS[variant], flags, int(ring_bytes or 0), int(lag), int(gbatch))
