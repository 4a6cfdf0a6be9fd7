"""Device plumbing: torch owns device memory and streams, the C ABI computes.

Host inputs (``Tensor4D`` / numpy) are copied to the selected CUDA device
(pinned staging, async copies on the current stream) and results copied
back; torch CUDA tensors are used in place.  Nothing here computes.
"""

from __future__ import annotations

import ctypes

import numpy as np

from .errors import NativeLibraryError, ShapeMismatchError
from .tensor import Tensor4D

try:  # torch is the device-memory / stream provider on the GPU box
    import torch
except ImportError:  # pragma: no cover - the image always has torch
    torch = None


def require_cuda(device=None):
    """Resolve ``device`` to a torch CUDA device or raise (no CPU fallback)."""
    if torch is None or not torch.cuda.is_available():
        raise NativeLibraryError("a CUDA device (B200, sm_100a) is required; none is available")
    if device is None or device == "cuda":
        return torch.device("cuda", torch.cuda.current_device())
    if isinstance(device, int):
        return torch.device("cuda", device)
    dev = torch.device(device)
    if dev.type != "cuda":
        raise NativeLibraryError(f"device {device!r} is not a CUDA device")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def stream_ptr(dev) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def is_torch(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


def to_device(x, dev, dims=None, name="tensor"):
    """Return a contiguous float32 CUDA tensor for x (Tensor4D / ndarray / torch)."""
    if isinstance(x, Tensor4D):
        arr = x.data
    elif isinstance(x, np.ndarray):
        arr = np.ascontiguousarray(x, dtype=np.float32)
    elif is_torch(x):
        t = x
        if dims is not None and tuple(t.shape) != tuple(dims):
            raise ShapeMismatchError(f"{name} dims {tuple(t.shape)} do not match {tuple(dims)}")
        if t.device != dev:
            t = t.to(dev)
        if t.dtype != torch.float32:
            t = t.float()
        return t.contiguous()
    else:
        raise ShapeMismatchError(f"cannot use {type(x).__name__} as {name}")
    if dims is not None and tuple(arr.shape) != tuple(dims):
        raise ShapeMismatchError(f"{name} dims {tuple(arr.shape)} do not match {tuple(dims)}")
    if not arr.flags.writeable:
        arr = arr.copy()
    host = torch.from_numpy(arr)
    if not host.is_pinned():
        host = host.pin_memory()
    return host.to(dev, non_blocking=True)


def dims_of(x):
    if isinstance(x, Tensor4D):
        return x.dims
    if isinstance(x, np.ndarray) or is_torch(x):
        return tuple(int(n) for n in x.shape)
    raise ShapeMismatchError(f"cannot use {type(x).__name__} as a tensor")


def to_host_tensor4d(t) -> Tensor4D:
    """Copy a CUDA tensor back into an aligned Tensor4D (synchronises)."""
    from .tensor import aligned_empty

    out = aligned_empty(tuple(t.shape))
    host = torch.empty(tuple(t.shape), dtype=torch.float32, pin_memory=True)
    host.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    out[...] = host.numpy()
    return Tensor4D(out)
