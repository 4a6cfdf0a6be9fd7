"""Batch sharding across GPUs (one process per GPU, no data-path collective).

Transformed-convolution tiles of different images are independent (the
reference's flat tile order is batch-major, tiling.py:8-11), so a layer
shards along the batch: rank r of W gets a contiguous slice of images, a
replica of the KernelPack, and writes its own output slice.  The only
communication is outside the data path (optional gather of outputs for
verification).  Bitwise property: concatenating the shards'
outputs reproduces the single-device output exactly, because every tile is
computed by the same kernels with the same operands.
"""

from __future__ import annotations

from dataclasses import replace

from .errors import InvalidParameterError
from .tensor import LayerSpec


def shard_range(batch: int, rank: int, world: int):
    """Contiguous [lo, hi) image range of ``rank`` (near-equal split)."""
    if world < 1 or not 0 <= rank < world:
        raise InvalidParameterError(f"bad rank {rank} of world {world}")
    step, extra = divmod(batch, world)
    lo = rank * step + min(rank, extra)
    hi = lo + step + (1 if rank < extra else 0)
    return lo, hi


def shard_spec(spec: LayerSpec, rank: int, world: int) -> LayerSpec | None:
    """The LayerSpec of rank's slice, or None when the rank gets no image."""
    lo, hi = shard_range(spec.batch, rank, world)
    if hi <= lo:
        return None
    return replace(spec, batch=hi - lo)


def run_sharded(x, spec: LayerSpec, rank: int, world: int, compute, gather=None):
    """Run ``compute(x_slice, spec_slice)`` on this rank's images.

    ``x`` is the full batch (host or device tensor, indexable on axis 0);
    ``compute`` returns the slice's output.  With a torch.distributed
    ``gather`` group (any backend) the full output is assembled on every
    rank by all_gather -- verification only, never on the timed path.
    """
    lo, hi = shard_range(spec.batch, rank, world)
    sub = shard_spec(spec, rank, world)
    out = compute(x[lo:hi], sub) if sub is not None else None
    if gather is None:
        return out
    import torch
    import torch.distributed as dist

    tail = tuple(spec.output_dims()[1:])
    local = torch.as_tensor(out) if out is not None else torch.empty((0,) + tail)
    sizes = [h - l for l, h in (shard_range(spec.batch, r, world) for r in range(world))]
    cap = max(sizes)
    padded = torch.zeros((cap,) + tail, dtype=local.dtype, device=local.device)   # equal sizes for gloo
    padded[:local.shape[0]] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=gather)
    return torch.cat([p[:n] for p, n in zip(parts, sizes)], dim=0)
