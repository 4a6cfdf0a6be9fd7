"""Kernel packs and the typed stage functions (reference winofuse/transforms.py).

* :class:`KernelPack` -- the transformed kernels, ``data`` shaped (T*T, C, C')
  float32, read-only, position-major, exactly the reference layout
  (transforms.py:22-41).  On first use on a CUDA device the pack is also
  uploaded and converted once into the MMA-ready operand (bf16 hi/lo UMMA
  slabs, cached per device); engines never pay for it inside their timing.
* :func:`transform_kernels` -- G w G^T in float64, one f32 rounding
  (transforms.py:63-80); host numpy for host weights, the
  ``wf_filter_transform`` kernel for CUDA weights.
* :func:`forward_transform_tiles`, :func:`multiply_block`,
  :func:`inverse_transform_tiles` -- the three stages on reference layouts,
  executed by the sm_100a utility kernels of the C ABI.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import device as _dev
from .basis import FftBasis, WinogradBasis, default_points
from .errors import ShapeMismatchError, UnsupportedConfigError
from .tensor import LayerSpec, Tensor4D, aligned_empty
from .tiling import TilePlan


@dataclass(frozen=True)
class KernelPack:
    """Transformed kernels (T*T, C, C'), float32, read-only."""

    data: np.ndarray
    tile: int
    kernel_side: int
    c_in: int
    c_out: int
    transform: str = "winograd"
    _device: dict = field(default_factory=dict, compare=False, repr=False)

    @property
    def nbytes(self) -> int:
        return int(self.data.nbytes)

    @property
    def positions(self) -> int:
        return int(self.data.shape[0])

    def device_f32(self, dev):
        """Reference-layout pack on ``dev`` (uploaded once)."""
        key = ("f32", str(dev))
        t = self._device.get(key)
        if t is None:
            t = _dev.to_device(self.data, dev, name="pack")
            self._device[key] = t
        return t

    def device_mma(self, dev, precision: str = "3xbf16"):
        """MMA-ready operand on ``dev`` (bf16 or fp16 hi/lo UMMA slabs, per the
        precision mode's operand format; built once per device and format)."""
        fmt = _lib.PACK_FORMAT[precision]
        key = ("mma", str(dev), fmt)
        t = self._device.get(key)
        if t is None:
            lib = _lib.load()
            tf = _lib.TRANSFORMS[self.transform]
            nbytes = lib.wf_mma_pack_bytes(self.tile, self.c_in, self.c_out, tf)
            if nbytes == 0:
                _lib.check(_lib.WF_ERR_UNSUPPORTED, "mma pack")
            t = _dev.torch.empty(nbytes, dtype=_dev.torch.uint8, device=dev)
            src = self.device_f32(dev)
            _lib.check(lib.wf_mma_pack_ex(_dev.ptr(src), _dev.ptr(t), self.tile, self.c_in, self.c_out, tf,
                                          _lib.PRECISIONS[precision], _dev.stream_ptr(dev)), "wf_mma_pack")
            self._device[key] = t
        return t


@dataclass
class LeftHandBlock:
    """Transformed input tiles of one task: (T*T, rows, C), first r_eff rows valid."""

    data: np.ndarray
    r_eff: int

    @classmethod
    def empty(cls, tile: int, rows: int, c_in: int) -> "LeftHandBlock":
        return cls(data=aligned_empty((tile * tile, rows, c_in)), r_eff=rows)


def fft_pack_host(w64: np.ndarray) -> np.ndarray:
    """Real expansion of the conjugate kernel spectra, (144, 2C, 2C') float32.

    V[p][c][c'] = conj(rfft2(w[c'][c] zero-padded to 16x16))[p] (cross-
    correlation), computed in float64.  The complex product M = X V over c is
    a real GEMM [Re X | Im X] @ [[Re V, Im V], [-Im V, Re V]]: rows 0..C-1 of
    the pack multiply Re X, rows C..2C-1 Im X; columns 0..C'-1 give Re M,
    C'..2C'-1 Im M.
    """
    c_out, c_in = w64.shape[:2]
    padded = np.zeros((c_out, c_in, 16, 16), np.float64)
    padded[:, :, :w64.shape[2], :w64.shape[3]] = w64
    spec = np.conj(np.fft.rfft2(padded))                       # (C', C, 16, 9)
    v = spec.reshape(c_out, c_in, 144).transpose(2, 1, 0)      # (144, C, C')
    host = aligned_empty((144, 2 * c_in, 2 * c_out))
    host[:, :c_in, :c_out] = v.real
    host[:, :c_in, c_out:] = v.imag
    host[:, c_in:, :c_out] = -v.imag
    host[:, c_in:, c_out:] = v.real
    return host


def transform_kernels(kers, basis) -> KernelPack:
    """G w G^T for every (c', c), packed position-major (T*T, C, C').

    Host weights: float64 numpy, one f32 rounding (reference
    transforms.py:73-77).  CUDA weights: the same arithmetic on the device.
    With an :class:`FftBasis` the pack is the real-expanded conjugate kernel
    spectrum (144, 2C, 2C') of :func:`fft_pack_host` (one-time, host f64).
    """
    dims = _dev.dims_of(kers)
    if len(dims) != 4:
        raise ShapeMismatchError(f"kernel dims {dims} are not 4-D")
    if isinstance(basis, WinogradBasis) and tuple(basis.points) != tuple(default_points(basis.tile)):
        # the sm_100a kernels bake in the default nodes' B^T / A^T: a pack of
        # other nodes would be applied with the wrong data transforms
        raise UnsupportedConfigError("the sm_100a kernels implement the default interpolation nodes only "
                                     f"({', '.join(str(p) for p in default_points(basis.tile))})")
    c_out, c_in, kh, kw = dims
    if kh != basis.kernel or kw != basis.kernel:
        raise ShapeMismatchError(f"kernel dims {dims} do not match basis K={basis.kernel}")
    if isinstance(basis, FftBasis):
        if _dev.is_torch(kers):
            w64 = kers.detach().cpu().double().numpy()
        else:
            w64 = (kers.data if isinstance(kers, Tensor4D) else np.asarray(kers)).astype(np.float64)
        host = fft_pack_host(w64)
        host.setflags(write=False)
        return KernelPack(data=host, tile=basis.tile, kernel_side=basis.kernel, c_in=c_in, c_out=c_out,
                          transform="fft")
    t = basis.tile
    if _dev.is_torch(kers) and kers.is_cuda:
        dev = kers.device
        w = kers.contiguous().float()
        lib = _lib.load()
        out = _dev.torch.empty((t * t, c_in, c_out), dtype=_dev.torch.float32, device=dev)
        _lib.check(lib.wf_filter_transform(_dev.ptr(w), _dev.ptr(out), c_in, c_out, t,
                                           _dev.stream_ptr(dev)), "wf_filter_transform")
        host = aligned_empty((t * t, c_in, c_out))
        host[...] = out.cpu().numpy()
        host.setflags(write=False)
        pack = KernelPack(data=host, tile=t, kernel_side=basis.kernel, c_in=c_in, c_out=c_out)
        pack._device[("f32", str(dev))] = out
        return pack
    w64 = (kers.data if isinstance(kers, Tensor4D) else np.asarray(kers)).astype(np.float64)
    # (C', C, T, T): G w_{c'c} G^T in f64 for every kernel, then position-major
    spatial = np.matmul(np.matmul(basis.g, w64), basis.g.T)
    host = aligned_empty((t * t, c_in, c_out))
    host[...] = spatial.transpose(2, 3, 1, 0).reshape(t * t, c_in, c_out)  # (T, T, C, C')
    host.setflags(write=False)
    return KernelPack(data=host, tile=t, kernel_side=basis.kernel, c_in=c_in, c_out=c_out)


def multiply_flops(rows: int, c_in: int, c_out: int, tile: int, transform: str = "winograd") -> int:
    """Useful multiply-stage flops for ``rows`` tiles.

    Winograd: 2 * rows * C * C' * T^2.  FFT-16: 8 * rows * C * C' * 144
    (a complex multiply-add is 8 real flops).
    """
    if transform == "fft":
        return 8 * rows * c_in * c_out * 144
    return 2 * rows * c_in * c_out * tile * tile


# ------------------------------------------------------------ stage functions
def _block_array(block):
    return block.data if isinstance(block, LeftHandBlock) else block


def _check_range(pl: TilePlan, tiles: range) -> None:
    if tiles.step != 1 or tiles.start < 0 or tiles.stop > pl.n_tile or tiles.start >= tiles.stop:
        raise ShapeMismatchError(f"tile range {tiles} invalid for {pl.n_tile} tiles")


def _writeback(dst_np: np.ndarray, src_t) -> None:
    dst_np[...] = src_t.cpu().numpy()


def forward_transform_tiles(inp, spec: LayerSpec, pl: TilePlan, basis: WinogradBasis, tiles: range,
                            dst, row0: int = 0, device=None) -> None:
    """Gather + transform tiles [start, stop) into dst[:, row0 + i - start, :].

    GPU execution of reference transforms.py:94-109 (kernels.py:52-100).
    """
    if spec != pl.spec:
        raise ShapeMismatchError("layer spec does not match the tile plan")
    _check_range(pl, tiles)
    if _dev.dims_of(inp) != spec.input_dims():
        raise ShapeMismatchError(f"input dims {_dev.dims_of(inp)} mismatch layer")
    d = _block_array(dst)
    t = pl.tile
    if d.shape[0] != t * t or d.shape[2] != spec.in_channels or d.shape[1] < row0 + len(tiles):
        raise ShapeMismatchError(f"bad destination block {tuple(d.shape)}")
    dev = _dev.require_cuda(device if not _dev.is_torch(d) else d.device)
    x = _dev.to_device(inp, dev, name="input")
    out = d if _dev.is_torch(d) else _dev.to_device(d, dev, name="dst")
    lib = _lib.load()
    _lib.check(lib.wf_forward_tiles(_dev.ptr(x), _dev.ptr(out), _lib.layer_struct(spec), t, tiles.start,
                                    tiles.stop, row0, int(d.shape[1]), _dev.stream_ptr(dev)),
               "wf_forward_tiles")
    if not _dev.is_torch(d):
        _writeback(d, out)


def multiply_block(lhs, pack: KernelPack, dst, rows: int | None = None, device=None) -> int:
    """dst[p, :rows] = lhs[p, :rows] @ pack.data[p]; returns useful flops.

    GPU execution of reference transforms.py:112-131 (f32, ascending c).
    """
    left = _block_array(lhs)
    if rows is None:
        rows = lhs.r_eff if isinstance(lhs, LeftHandBlock) else int(left.shape[1])
    t2 = pack.tile * pack.tile
    if left.shape[0] != t2 or left.shape[2] != pack.c_in or left.shape[1] < rows:
        raise ShapeMismatchError(f"left block {tuple(left.shape)} mismatch")
    if dst.shape[0] != t2 or dst.shape[2] != pack.c_out or dst.shape[1] < rows:
        raise ShapeMismatchError(f"result block {tuple(dst.shape)} mismatch")
    dev = _dev.require_cuda(device)
    a = _dev.to_device(np.ascontiguousarray(left) if not _dev.is_torch(left) else left, dev, name="left")
    b = pack.device_f32(dev)
    if _dev.is_torch(dst):
        out = dst
    else:
        out = _dev.to_device(np.ascontiguousarray(dst), dev, name="dst")
    lib = _lib.load()
    _lib.check(lib.wf_multiply_positions(_dev.ptr(a), _dev.ptr(b), _dev.ptr(out), t2, int(left.shape[1]),
                                         int(rows), pack.c_in, pack.c_out, _dev.stream_ptr(dev)),
               "wf_multiply_positions")
    if not _dev.is_torch(dst):
        _writeback(dst, out)
    return multiply_flops(rows, pack.c_in, pack.c_out, pack.tile)


def inverse_transform_tiles(results, basis: WinogradBasis, pl: TilePlan, tiles: range, out,
                            row0: int = 0, device=None) -> None:
    """Output-transform rows of ``results`` and scatter them into ``out``.

    GPU execution of reference transforms.py:134-152 (kernels.py:103-141).
    """
    _check_range(pl, tiles)
    t = pl.tile
    if results.shape[0] != t * t or results.shape[2] != pl.spec.out_channels \
            or results.shape[1] < row0 + len(tiles):
        raise ShapeMismatchError(f"bad result block {tuple(results.shape)}")
    if _dev.dims_of(out) != pl.spec.output_dims():
        raise ShapeMismatchError(f"output dims {_dev.dims_of(out)} mismatch layer")
    dev = _dev.require_cuda(device)
    res = _dev.to_device(np.ascontiguousarray(results) if not _dev.is_torch(results) else results, dev,
                         name="results")
    if _dev.is_torch(out):
        y = out
    else:
        y = _dev.to_device(out.data if isinstance(out, Tensor4D) else out, dev, name="out")
    lib = _lib.load()
    _lib.check(lib.wf_inverse_tiles(_dev.ptr(res), _dev.ptr(y), _lib.layer_struct(pl.spec), t, tiles.start,
                                    tiles.stop, row0, int(results.shape[1]), _dev.stream_ptr(dev)),
               "wf_inverse_tiles")
    if not _dev.is_torch(out):
        _writeback(out.data if isinstance(out, Tensor4D) else out, y)
