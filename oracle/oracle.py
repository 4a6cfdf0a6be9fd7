"""Python face of the CPU oracle (TEST INFRASTRUCTURE ONLY).

* :func:`direct_conv_f64` -- numpy FP64 direct cross-correlation built from
  shifted slices, restating the reference test oracle
  (pkg/tests/helpers.py:18-33).
* ctypes wrappers of oracle/winofuse_oracle.c: the reference's fused and
  three-stage float32 engines and their kernels (kernels.py, engines.py).
* :func:`max_rel_error` -- the reference's tolerance metric
  max|got - ref| / max|ref| (bench.py:59-64).
* :func:`default_basis` -- the default bt32 / at32 / g of tile T, read from the
  reference-generated golden fixture tests/golden/basis.json (no reference
  import at run time).
"""

from __future__ import annotations

import ctypes
import json
import os
import subprocess
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "liboracle.so")
GOLDEN = os.path.join(ROOT, "tests", "golden")


class OracleLayer(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in
                ("batch", "c_in", "c_out", "height", "width", "kernel", "pad_lo", "pad_hi")]


_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = ctypes.CDLL(LIB)
        f = ctypes.POINTER(ctypes.c_float)
        L = ctypes.POINTER(OracleLayer)
        i = ctypes.c_int
        lib.oracle_direct_conv.argtypes = [f, f, f, L]
        lib.oracle_forward_tiles.argtypes = [f, f, i, i, i, f, i, L, i]
        lib.oracle_inverse_tiles.argtypes = [f, f, i, i, i, i, f, L, i]
        lib.oracle_matmul_rows.argtypes = [f, f, f, i, i, i]
        lib.oracle_multiply_positions.argtypes = [f, f, f, i, i, i, i, i]
        lib.oracle_conv_fused.argtypes = [f, f, f, f, f, L, i, i, i]
        lib.oracle_conv_fused.restype = i
        lib.oracle_conv_three_stage.argtypes = [f, f, f, f, f, L, i, i]
        lib.oracle_conv_three_stage.restype = i
        lib.oracle_max_threads.restype = i
        _lib = lib
    return _lib


def _fp(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def layer(spec) -> OracleLayer:
    return OracleLayer(spec.batch, spec.in_channels, spec.out_channels, spec.height, spec.width,
                       spec.kernel, spec.pad_lo, spec.pad_hi)


def _out_dims(spec):
    return (spec.batch, spec.out_channels, spec.height + spec.pad_lo + spec.pad_hi - spec.kernel + 1,
            spec.width + spec.pad_lo + spec.pad_hi - spec.kernel + 1)


_BASIS = None


def default_basis(tile: int):
    """(bt32, at32, g64) of the default basis, from the golden fixture."""
    global _BASIS
    if _BASIS is None:
        with open(os.path.join(GOLDEN, "basis.json")) as fh:
            _BASIS = json.load(fh)
    entry = _BASIS[f"T{tile}_K3"]
    conv = lambda rows: np.array([[float(Fraction(v)) for v in r] for r in rows])  # noqa: E731
    return (np.ascontiguousarray(conv(entry["bt"]), np.float32),
            np.ascontiguousarray(conv(entry["at"]), np.float32), conv(entry["g"]))


def transform_kernels(w: np.ndarray, tile: int) -> np.ndarray:
    """(T*T, C, C') f32 pack: G w G^T in f64, one rounding (transforms.py:63-80)."""
    _, _, g = default_basis(tile)
    spatial = np.matmul(np.matmul(g, w.astype(np.float64)), g.T)
    return np.ascontiguousarray(spatial.transpose(2, 3, 1, 0).reshape(tile * tile, w.shape[1], w.shape[0]),
                                np.float32)


def conv_fused(x: np.ndarray, pack: np.ndarray, spec, tile: int, r: int = 24, threads: int = 1):
    bt, at, _ = default_basis(tile)
    out = np.zeros(_out_dims(spec), np.float32)
    load().oracle_conv_fused(_fp(np.ascontiguousarray(x, np.float32)), _fp(np.ascontiguousarray(pack, np.float32)),
                             _fp(out), _fp(bt), _fp(at), ctypes.byref(layer(spec)), tile, r, threads)
    return out


def conv_three_stage(x: np.ndarray, pack: np.ndarray, spec, tile: int, threads: int = 1):
    bt, at, _ = default_basis(tile)
    out = np.zeros(_out_dims(spec), np.float32)
    rc = load().oracle_conv_three_stage(_fp(np.ascontiguousarray(x, np.float32)),
                                        _fp(np.ascontiguousarray(pack, np.float32)), _fp(out), _fp(bt), _fp(at),
                                        ctypes.byref(layer(spec)), tile, threads)
    if rc != 0:
        raise MemoryError("oracle three-stage intermediates")
    return out


def direct_conv_f32(x: np.ndarray, w: np.ndarray, spec) -> np.ndarray:
    """The reference's direct engine (kernels.py:22-49): f64 accumulate, f32 out."""
    out = np.zeros(_out_dims(spec), np.float32)
    load().oracle_direct_conv(_fp(np.ascontiguousarray(x, np.float32)), _fp(np.ascontiguousarray(w, np.float32)),
                              _fp(out), ctypes.byref(layer(spec)))
    return out


def forward_tiles(x, spec, tile, t0, t1, rows, row0=0):
    bt, _, _ = default_basis(tile)
    dst = np.zeros((tile * tile, rows, spec.in_channels), np.float32)
    load().oracle_forward_tiles(_fp(np.ascontiguousarray(x, np.float32)), _fp(bt), t0, t1, row0, _fp(dst), rows,
                                ctypes.byref(layer(spec)), tile)
    return dst


def inverse_tiles(res, spec, tile, t0, t1, row0=0, out=None):
    _, at, _ = default_basis(tile)
    if out is None:
        out = np.zeros(_out_dims(spec), np.float32)
    load().oracle_inverse_tiles(_fp(np.ascontiguousarray(res, np.float32)), _fp(at), t0, t1, row0, res.shape[1],
                                _fp(out), ctypes.byref(layer(spec)), tile)
    return out


def multiply_positions(left, pack, r_eff):
    res = np.zeros((left.shape[0], left.shape[1], pack.shape[2]), np.float32)
    load().oracle_multiply_positions(_fp(np.ascontiguousarray(left, np.float32)),
                                     _fp(np.ascontiguousarray(pack, np.float32)), _fp(res), left.shape[0],
                                     left.shape[1], r_eff, left.shape[2], pack.shape[2])
    return res


def direct_conv_f64(x: np.ndarray, w: np.ndarray, spec) -> np.ndarray:
    """FP64 correlation from shifted slices (reference tests/helpers.py:18-33)."""
    xp = np.pad(x.astype(np.float64), ((0, 0), (0, 0), (spec.pad_lo, spec.pad_hi), (spec.pad_lo, spec.pad_hi)))
    _, _, ho, wo = _out_dims(spec)
    w64 = w.astype(np.float64)
    out = np.zeros(_out_dims(spec), np.float64)
    for ky in range(spec.kernel):
        for kx in range(spec.kernel):
            out += np.einsum("bcyx,oc->boyx", xp[:, :, ky:ky + ho, kx:kx + wo], w64[:, :, ky, kx], optimize=True)
    return out


def max_rel_error(got, ref) -> float:
    """max|got - ref| / max|ref| (reference bench.py:59-64)."""
    a = np.asarray(got, np.float64)
    b = np.asarray(ref, np.float64)
    return float(np.max(np.abs(a - b))) / max(float(np.max(np.abs(b))), 1e-30)


def threads() -> int:
    return int(load().oracle_max_threads())


def fft_conv_f64(x: np.ndarray, pack: np.ndarray, spec) -> np.ndarray:
    """FP64 numpy restatement of the FFT-16 overlap-save convolution.

    No reference implementation exists (FFT parity is
    "unpinned" against the reference and anchored on the FP64 direct
    oracle).  Follows the definition of SURVEY.md 8(b): 16x16 windows at
    stride 14 (tile grid of reference tiling.py:66-75 with m = 14), rfft2,
    per-bin real-expanded GEMM with ``pack`` (144, 2C, 2C'), irfft2, keep the
    valid 14x14 block.  Used to check the pack expansion and tiling on CPU.
    """
    b, c, h, w = x.shape
    k = spec.kernel
    m = 17 - k
    _, _, ho, wo = _out_dims(spec)
    ty, tx = -(-ho // m), -(-wo // m)
    hp, wp = (ty - 1) * m + 16, (tx - 1) * m + 16
    xp = np.zeros((b, c, max(hp, spec.pad_lo + h), max(wp, spec.pad_lo + w)), np.float64)
    xp[:, :, spec.pad_lo:spec.pad_lo + h, spec.pad_lo:spec.pad_lo + w] = x
    wins = np.empty((b, ty, tx, c, 16, 16), np.float64)
    for i in range(ty):
        for j in range(tx):
            wins[:, i, j] = xp[:, :, i * m:i * m + 16, j * m:j * m + 16]
    spec_x = np.fft.rfft2(wins).reshape(b * ty * tx, c, 144)           # (tiles, C, 144)
    cp = pack.shape[2] // 2
    out = np.empty((b * ty * tx, cp, 144), np.complex128)
    p64 = pack.astype(np.float64)
    for p in range(144):
        a = np.concatenate([spec_x[:, :, p].real, spec_x[:, :, p].imag], axis=1)   # (tiles, 2C)
        r = a @ p64[p]                                                              # (tiles, 2C')
        out[:, :, p] = r[:, :cp] + 1j * r[:, cp:]
    blocks = np.fft.irfft2(out.reshape(b * ty * tx, cp, 16, 9), s=(16, 16))[:, :, :m, :m]
    y = blocks.reshape(b, ty, tx, cp, m, m).transpose(0, 3, 1, 4, 2, 5).reshape(b, cp, ty * m, tx * m)
    return y[:, :, :ho, :wo]
