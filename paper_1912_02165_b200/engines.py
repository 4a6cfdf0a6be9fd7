"""Convolution engines on the B200 (reference winofuse/engines.py).

Same names, argument order and error behaviour as the reference:

* ``direct``      -- seven-loop correlation, FP64 accumulation (the oracle
  engine, engines.py:213-231), here an sm_100a FP64 kernel.
* ``three_stage`` -- forward transform of every tile, one tcgen05 GEMM per
  transform position, inverse transform, with full-size intermediates in HBM
  (engines.py:234-314).  Kept as the in-repo comparison point.
* ``fused``       -- the transformed tiles never make an HBM round trip
  (engines.py:317-444); requires a prebuilt :class:`KernelPack`.

Inputs may be host ``Tensor4D`` / ndarrays (copied to the device and the
result copied back into a ``Tensor4D``, like the reference returns) or torch
CUDA tensors (result stays on the device).  ``ConvStats.wall_s`` is the
device time of the engine's kernels measured with CUDA events on the
launching stream (transfers excluded, like the reference's timers).

GPU additions to :class:`EngineConfig`: ``device`` (None = current CUDA
device), ``transform`` ("winograd" | "fft"), ``precision`` ("3xbf16" |
"3xfp16" | "bf16"), ``fused_variant`` (which fused kernel runs: "auto" | "ws" |
"itemq" | "waves" | "ws_row", the last never picked by "auto") and ``ring_bytes`` (L2 ring budget of the persistent
fused kernels).  There is no CPU fallback: without the CUDA extension or a
GPU every engine raises :class:`NativeLibraryError`.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import device as _dev
from .basis import FftBasis, make_basis, make_fft_basis
from .errors import (IntermediateAllocationError, InvalidParameterError, ShapeMismatchError,
                     WinofuseError)
from .tensor import LayerSpec, Tensor4D, aligned_empty
from .tiling import plan as tile_plan
from .transforms import KernelPack, multiply_flops, transform_kernels

ENGINE_KINDS = ("direct", "three_stage", "fused")
PRECISIONS = ("3xbf16", "bf16", "3xfp16")
TRANSFORMS = ("winograd", "fft")
FFT_TILE = 16
_FP32 = 4


@dataclass
class EngineConfig:
    """Engine selection and tuning knobs (reference engines.py:45-79).

    ``r``: tiles per task (the paper's R).  ``workers``: 0 = every SM of the
    device (the GPU analogue of one worker per core).
    """

    kind: str = "fused"
    tile: int = 7
    r: int = 24
    workers: int = 0
    points: tuple | None = None
    instrumented: bool = False
    l2_budget_bytes: int | None = None
    device: object = None
    transform: str = "winograd"
    precision: str = "3xbf16"
    fused_variant: str = "auto"
    ring_bytes: int | None = None

    def __post_init__(self):
        if self.kind not in ENGINE_KINDS:
            raise InvalidParameterError(f"unknown engine kind {self.kind!r}")
        if self.transform not in TRANSFORMS:
            raise InvalidParameterError(f"unknown transform {self.transform!r}")
        if self.kind != "direct":
            if self.transform == "winograd" and not 4 <= self.tile <= 8:
                raise InvalidParameterError(f"tile side must be in [4, 8], got {self.tile}")
            if self.transform == "fft" and self.tile != FFT_TILE:
                raise InvalidParameterError(f"the FFT transform uses tile {FFT_TILE}, got {self.tile}")
        if self.r < 1:
            raise InvalidParameterError("tiles per task (r) must be >= 1")
        if self.workers < 0:
            raise InvalidParameterError("workers must be >= 0 (0 = auto)")
        if self.precision not in PRECISIONS:
            raise InvalidParameterError(f"unknown precision {self.precision!r}")
        if self.fused_variant not in _lib.VARIANTS:
            raise InvalidParameterError(f"unknown fused variant {self.fused_variant!r}")
        if self.ring_bytes is not None and self.ring_bytes < 0:
            raise InvalidParameterError("ring_bytes must be >= 0")

    def resolved_workers(self, cap: int | None = None) -> int:
        w = self.workers or _device_sm_count()
        if cap is not None:
            w = min(w, cap)
        return max(w, 1)


def _device_sm_count() -> int:
    try:
        if _dev.torch is not None and _dev.torch.cuda.is_available():
            return int(_dev.torch.cuda.get_device_properties(
                _dev.torch.cuda.current_device()).multi_processor_count)
    except Exception:  # pragma: no cover
        pass
    return os.cpu_count() or 1


@dataclass
class ConvStats:
    engine: str
    wall_s: float = 0.0
    flops: int = 0
    n_tile: int = 0
    n_task: int = 0
    r: int = 0
    r_eff_last: int = 0
    workers: int = 1
    intermediate_bytes: int = 0
    scratch_bytes: int = 0
    phase_s: dict = field(default_factory=dict)
    warnings: list = field(default_factory=list)
    overlap_violations: int | None = None
    task_flops: list | None = None
    task_trace: list | None = None
    device: str = ""
    precision: str = ""
    transform: str = ""
    variant: str = ""           # fused kernel that ran: "ws" | "itemq" | "waves" | "ws_row"
    blocks: int = 0             # 128-tile blocks (the GPU's tasks: one MMA M each)


# ------------------------------------------------------- scratch layout math
@dataclass(frozen=True)
class BufferLayout:
    """Byte layout of one overlapping operand/result scratch (engines.py:100-134).

    Operand slots of s_l = 4*R*C bytes packed against the end, result slots
    of s_r = 4*R*C' from the base; result p only overwrites operand bytes of
    positions already consumed.  On the GPU the same calculus sizes the
    on-chip scratch of one CTA task.
    """

    r: int
    c_in: int
    c_out: int
    tile: int
    s_l: int
    s_r: int
    s_max: int
    s_min: int
    capacity: int
    left_offsets: tuple
    result_offsets: tuple

    def left_offset(self, i: int) -> int:
        return self.left_offsets[i - 1]

    def result_offset(self, i: int) -> int:
        return self.result_offsets[i - 1]

    def __iter__(self):
        return iter((self.capacity, self.left_offsets, self.result_offsets))


def buffer_layout(r: int, c_in: int, c_out: int, tile: int) -> BufferLayout:
    if min(r, c_in, c_out, tile) < 1:
        raise InvalidParameterError("layout parameters must all be >= 1")
    npos = tile * tile
    s_l, s_r = _FP32 * r * c_in, _FP32 * r * c_out
    s_max, s_min = max(s_l, s_r), min(s_l, s_r)
    cap = npos * s_max + s_min
    res = tuple(p * s_r for p in range(npos))
    left = tuple(cap - (npos - p) * s_l for p in range(npos))
    if any(res[p] + s_r > left[p] for p in range(npos)):
        raise WinofuseError("scratch layout overlap (internal error)")
    return BufferLayout(r=r, c_in=c_in, c_out=c_out, tile=tile, s_l=s_l, s_r=s_r, s_max=s_max,
                        s_min=s_min, capacity=cap, left_offsets=left, result_offsets=res)


class SharedBuffer:
    """Host scratch with aliasing operand / result views (engines.py:158-174)."""

    def __init__(self, layout: BufferLayout):
        self.layout = layout
        self.flat = aligned_empty((layout.capacity // _FP32,), np.float32)
        p2 = layout.tile * layout.tile
        l0 = layout.left_offsets[0] // _FP32
        self.left = self.flat[l0:l0 + p2 * layout.r * layout.c_in].reshape(p2, layout.r, layout.c_in)
        self.result = self.flat[:p2 * layout.r * layout.c_out].reshape(p2, layout.r, layout.c_out)


# ----------------------------------------------------------------- helpers
def _check_input(inp, spec: LayerSpec) -> None:
    if _dev.dims_of(inp) != spec.input_dims():
        raise ShapeMismatchError(f"input dims {_dev.dims_of(inp)} do not match layer {spec.input_dims()}")


def _resolve_pack(kers, spec: LayerSpec, basis) -> KernelPack:
    if isinstance(kers, KernelPack):
        want = "fft" if isinstance(basis, FftBasis) else "winograd"
        if (kers.tile != basis.tile or kers.kernel_side != spec.kernel or kers.c_in != spec.in_channels
                or kers.c_out != spec.out_channels or kers.transform != want):
            raise ShapeMismatchError(
                f"kernel pack (T={kers.tile}, K={kers.kernel_side}, C={kers.c_in}, C'={kers.c_out}) "
                f"does not match layer/config")
        return kers
    if isinstance(kers, Tensor4D) or isinstance(kers, np.ndarray) or _dev.is_torch(kers):
        if _dev.dims_of(kers) != spec.kernel_dims():
            raise ShapeMismatchError(f"kernel dims {_dev.dims_of(kers)} do not match {spec.kernel_dims()}")
        return transform_kernels(kers, basis)
    raise ShapeMismatchError(f"cannot use {type(kers).__name__} as kernels")


def _basis_for(cfg: EngineConfig, spec: LayerSpec):
    if cfg.transform == "fft":
        return make_fft_basis(spec.kernel)
    if cfg.points is not None and tuple(str(p) for p in cfg.points) != \
            tuple(str(p) for p in make_basis(cfg.tile, spec.kernel).points):
        from .errors import UnsupportedConfigError
        raise UnsupportedConfigError("the sm_100a kernels bake in the default interpolation nodes")
    return make_basis(cfg.tile, spec.kernel, cfg.points)


def _intermediate_bytes(n_tile: int, spec: LayerSpec, cfg: EngineConfig) -> int:
    """Full-size transformed intermediates of the three-stage engine.

    Winograd: 4 * T^2 * n_tile * (C + C'); FFT-16: complex64 bins,
    8 * 144 * n_tile * (C + C') (SURVEY.md 8(d) Q_3stage).
    """
    if cfg.transform == "fft":
        return 8 * 144 * n_tile * (spec.in_channels + spec.out_channels)
    return _FP32 * cfg.tile * cfg.tile * n_tile * (spec.in_channels + spec.out_channels)


def _finish(y, host_result: bool):
    return _dev.to_host_tensor4d(y) if host_result else y


class _Timer:
    """CUDA-event timing on the launching stream."""

    def __init__(self, dev):
        self.dev = dev
        torch = _dev.torch
        self.start = torch.cuda.Event(enable_timing=True)
        self.stop = torch.cuda.Event(enable_timing=True)

    def __enter__(self):
        self.start.record(_dev.torch.cuda.current_stream(self.dev))
        return self

    def __exit__(self, *exc):
        self.stop.record(_dev.torch.cuda.current_stream(self.dev))

    def seconds(self) -> float:
        self.stop.synchronize()
        return self.start.elapsed_time(self.stop) * 1e-3


def _on(dev):
    """Make ``dev`` the current CUDA device around a native call: the
    library launches on the current device (cudaGetDevice)."""
    return _dev.torch.cuda.device(dev)


def _opts(cfg: EngineConfig, flags: int = 0):
    return _lib.fused_opts(cfg.fused_variant, flags, cfg.ring_bytes)


_SCRATCH = {}


def _scratch(dev, nbytes: int, tag: str):
    """Engine-owned scratch, reused across calls of the same size."""
    key = (str(dev), tag)
    buf = _SCRATCH.get(key)
    if buf is None or buf.numel() < nbytes:
        _SCRATCH.pop(key, None)
        buf = _dev.torch.empty(max(nbytes, 16), dtype=_dev.torch.uint8, device=dev)
        _SCRATCH[key] = buf
    return buf


# ----------------------------------------------------------------- engines
def conv_direct(inp, kers, spec: LayerSpec, config: EngineConfig | None = None):
    """Oracle engine: FP64 direct correlation on the GPU (engines.py:213-231)."""
    if isinstance(kers, KernelPack) or not (isinstance(kers, (Tensor4D, np.ndarray)) or _dev.is_torch(kers)):
        raise ShapeMismatchError("direct engine needs untransformed kernels")
    _check_input(inp, spec)
    if _dev.dims_of(kers) != spec.kernel_dims():
        raise ShapeMismatchError(f"kernel dims {_dev.dims_of(kers)} do not match {spec.kernel_dims()}")
    dev = _dev.require_cuda(config.device if config else None)
    x = _dev.to_device(inp, dev, name="input")
    w = _dev.to_device(kers, dev, name="kernels")
    y = _dev.torch.empty(spec.output_dims(), dtype=_dev.torch.float32, device=dev)
    lib = _lib.load()
    with _on(dev), _Timer(dev) as tm:
        _lib.check(lib.wf_conv_direct(_dev.ptr(x), _dev.ptr(w), _dev.ptr(y), _lib.layer_struct(spec),
                                      _dev.stream_ptr(dev)), "wf_conv_direct")
    stats = ConvStats(engine="direct", wall_s=tm.seconds(), flops=spec.direct_flops(), device=str(dev))
    return _finish(y, not _dev.is_torch(inp)), stats


def conv_three_stage(inp, kers, spec: LayerSpec, config: EngineConfig | None = None):
    """Staged engine with full-size transformed intermediates (engines.py:234-314)."""
    cfg = config or EngineConfig(kind="three_stage")
    basis = _basis_for(cfg, spec)
    _check_input(inp, spec)
    pack = _resolve_pack(kers, spec, basis)
    pl = tile_plan(spec, cfg.tile, out=basis.out)
    dev = _dev.require_cuda(cfg.device if not _dev.is_torch(inp) else inp.device)
    lib = _lib.load()
    layer = _lib.layer_struct(spec)
    tf = _lib.TRANSFORMS[cfg.transform]
    inter_bytes = _intermediate_bytes(pl.n_tile, spec, cfg)
    need = lib.wf_three_stage_scratch_bytes(layer, cfg.tile, tf)
    if need == 0:
        _lib.check(lib.wf_conv_three_stage(None, None, None, None, 0, layer, cfg.tile, tf, 0, None),
                   "wf_conv_three_stage")
    x = _dev.to_device(inp, dev, name="input")
    vpack = pack.device_mma(dev, cfg.precision)
    try:
        scratch = _dev.torch.empty(need, dtype=_dev.torch.uint8, device=dev)
    except _dev.torch.cuda.OutOfMemoryError as exc:
        raise IntermediateAllocationError(inter_bytes, "staged transform intermediates") from exc
    y = _dev.torch.empty(spec.output_dims(), dtype=_dev.torch.float32, device=dev)
    # one launch group per stage with an event between them: the reference's
    # per-stage phase_s (engines.py:263-302), here device time per stage
    torch = _dev.torch
    events = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    stream = torch.cuda.current_stream(dev)
    phases = (("forward", _lib.WF_PHASE_FORWARD), ("multiply", _lib.WF_PHASE_MULTIPLY),
              ("inverse", _lib.WF_PHASE_INVERSE))
    with _on(dev):
        events[0].record(stream)
        for i, (_, bit) in enumerate(phases):
            _lib.check(lib.wf_conv_three_stage_phases(_dev.ptr(x), _dev.ptr(vpack), _dev.ptr(y), _dev.ptr(scratch),
                                                      need, layer, cfg.tile, tf, _lib.PRECISIONS[cfg.precision],
                                                      bit, _dev.stream_ptr(dev)), "wf_conv_three_stage")
            events[i + 1].record(stream)
    events[-1].synchronize()
    phase_s = {name: events[i].elapsed_time(events[i + 1]) * 1e-3 for i, (name, _) in enumerate(phases)}
    wall = events[0].elapsed_time(events[-1]) * 1e-3
    stats = ConvStats(engine="three_stage", wall_s=wall,
                      flops=multiply_flops(pl.n_tile, spec.in_channels, spec.out_channels, cfg.tile,
                                           cfg.transform),
                      n_tile=pl.n_tile, workers=cfg.resolved_workers(), intermediate_bytes=inter_bytes,
                      scratch_bytes=int(need), phase_s=phase_s, device=str(dev),
                      precision=cfg.precision, transform=cfg.transform, blocks=-(-pl.n_tile // 128))
    return _finish(y, not _dev.is_torch(inp)), stats


def conv_fused(inp, pack: KernelPack, spec: LayerSpec, config: EngineConfig | None = None, *,
               task_order=None):
    """Fused engine: transformed tiles stay on chip (engines.py:317-444).

    Takes a prebuilt KernelPack only.  ``task_order`` must be a permutation
    of range(n_task); tasks write disjoint output tiles, so the output does
    not depend on it (the GPU schedules tasks itself; the order is
    validated and recorded for API compatibility).
    """
    cfg = config or EngineConfig(kind="fused")
    if not isinstance(pack, KernelPack):
        raise ShapeMismatchError("fused engine needs a prebuilt KernelPack (see transform_kernels)")
    basis = _basis_for(cfg, spec)
    _check_input(inp, spec)
    pack = _resolve_pack(pack, spec, basis)
    pl = tile_plan(spec, cfg.tile, out=basis.out)
    n_task = -(-pl.n_tile // cfg.r)
    if task_order is None:
        order = list(range(n_task))
    else:
        order = [int(i) for i in task_order]
        if sorted(order) != list(range(n_task)):
            raise InvalidParameterError(f"task_order must be a permutation of range({n_task})")
    dev = _dev.require_cuda(cfg.device if not _dev.is_torch(inp) else inp.device)
    lib = _lib.load()
    layer = _lib.layer_struct(spec)
    tf = _lib.TRANSFORMS[cfg.transform]
    layout = buffer_layout(cfg.r, spec.in_channels, spec.out_channels, cfg.tile)
    warnings = []
    if cfg.l2_budget_bytes and layout.capacity > cfg.l2_budget_bytes:
        warnings.append(f"scratch buffer {layout.capacity} B exceeds the configured L2 budget "
                        f"{cfg.l2_budget_bytes} B; lower R")
    flags = _lib.WF_FUSED_INSTRUMENT if cfg.instrumented else 0
    with _on(dev):
        opts = _opts(cfg)
        variant = lib.wf_fused_variant(layer, cfg.tile, tf, opts)
        if variant < 0:
            _lib.check(-variant, "wf_fused_variant")
        if flags and variant not in (_lib.WF_FUSED_WS, _lib.WF_FUSED_WS_ROW):
            warnings.append(f"instrumented mode is implemented by the warp-specialised kernel; the "
                            f"{_lib.VARIANT_NAMES[variant]!r} variant ran uninstrumented")
            flags = 0
        opts = _opts(cfg, flags)
        need = lib.wf_fused_scratch_bytes_ex(layer, cfg.tile, tf, opts)
        x = _dev.to_device(inp, dev, name="input")
        vpack = pack.device_mma(dev, cfg.precision)
        scratch = _scratch(dev, int(need), "fused")
        y = _dev.torch.empty(spec.output_dims(), dtype=_dev.torch.float32, device=dev)
        ran = ctypes.c_int(0)
        with _Timer(dev) as tm:
            _lib.check(lib.wf_conv_fused_ex(_dev.ptr(x), _dev.ptr(vpack), _dev.ptr(y), _dev.ptr(scratch), int(need),
                                            layer, cfg.tile, tf, _lib.PRECISIONS[cfg.precision], opts,
                                            ctypes.byref(ran), _dev.stream_ptr(dev)), "wf_conv_fused")
        wall = tm.seconds()
    workers = cfg.resolved_workers(n_task)
    flops = multiply_flops(pl.n_tile, spec.in_channels, spec.out_channels, cfg.tile, cfg.transform)
    n_blk = -(-pl.n_tile // 128)
    task_flops = trace = violations = None
    phase_s = {"fused": wall}
    if flags:
        with _on(dev):
            task_flops, trace, violations, phase_s = _read_instrumented(lib, layer, cfg, tf, opts, pl, spec, dev)
    stats = ConvStats(engine="fused", wall_s=wall, flops=flops, n_tile=pl.n_tile, n_task=n_task, r=cfg.r,
                      r_eff_last=pl.n_tile - (n_task - 1) * cfg.r, workers=workers,
                      scratch_bytes=int(need), phase_s=phase_s, warnings=warnings,
                      overlap_violations=violations, task_flops=task_flops, task_trace=trace,
                      device=str(dev), precision=cfg.precision, transform=cfg.transform,
                      variant=_lib.VARIANT_NAMES.get(ran.value, ""), blocks=n_blk)
    return _finish(y, not _dev.is_torch(inp)), stats


def _read_instrumented(lib, layer, cfg, tf, opts, pl, spec, dev):
    """Per-block ordering tickets of an instrumented warp-specialised launch ->
    (task_flops, task_trace, overlap_violations, phase_s).

    The GPU's tasks are 128-tile blocks.  A violation is an inverted ticket
    pair on a dependency edge of the dataflow: a block's GEMM started before
    its forward units ended or its inverse units started before its GEMM
    ended, or a ring slot was rewritten (forward of block b into U slot
    b % NU, GEMM of b into M slot b % NM) before the slot's previous
    consumer ended -- the GPU analogue of the reference's operand-overlap
    check (engines.py:382-396).  phase_s sums the per-CTA busy time of the
    forward units, the GEMM epilogue and the inverse units (the reference
    sums its workers' per-stage times, engines.py:432-434).
    """
    n_blk = -(-pl.n_tile // 128)
    ev = (ctypes.c_ulonglong * (8 * n_blk))()
    roles = (ctypes.c_ulonglong * 4)()
    ring = (ctypes.c_int * 2)()
    n = lib.wf_fused_instrument_read(layer, cfg.tile, tf, opts, ev, 8 * n_blk, roles, ring)
    if n < 0:
        _lib.check(-n, "wf_fused_instrument_read")
    e = np.frombuffer(ev, dtype=np.uint64).reshape(n_blk, 8)[:n]
    inv = np.uint64(0xFFFFFFFFFFFFFFFF)
    f_start, f_cta = e[:, 0] >> np.uint64(12), (e[:, 0] & np.uint64(0xFFF)).astype(int)
    f_end, g_start, g_end = inv - e[:, 1], e[:, 2], inv - e[:, 3]
    i_start, i_end = e[:, 4], inv - e[:, 5]
    nu, nm = int(ring[0]), int(ring[1])
    viol = int(np.sum(g_start < f_end)) + int(np.sum(i_start < g_end))
    if n > nu:
        viol += int(np.sum(f_start[nu:] < g_end[:-nu]))
    if n > nm:
        viol += int(np.sum(g_start[nm:] < i_end[:-nm]))
    order = np.argsort(f_start, kind="stable")
    trace = [(int(b), int(f_cta[b])) for b in order]
    task_flops = [multiply_flops(min(128, pl.n_tile - b * 128), spec.in_channels, spec.out_channels, cfg.tile,
                                 cfg.transform) for b in range(n)]
    clock_hz = float(roles[3]) * 1e3 or 1.965e9          # SM clock (kHz) reported by the library
    phase_s = {"forward": roles[0] / clock_hz, "multiply": roles[1] / clock_hz, "inverse": roles[2] / clock_hz}
    return task_flops, trace, viol, phase_s


def run_engine(kind: str, inp, kers, spec: LayerSpec, config: EngineConfig | None = None, **kw):
    """Dispatch by engine kind (reference engines.py:447-455)."""
    if kind == "direct":
        return conv_direct(inp, kers, spec, config)
    if kind == "three_stage":
        return conv_three_stage(inp, kers, spec, config)
    if kind == "fused":
        return conv_fused(inp, kers, spec, config, **kw)
    raise InvalidParameterError(f"unknown engine kind {kind!r}")


class LayerPlan:
    """Pre-planned layer: validated geometry, device pack, scratch and output.

    ``plan = LayerPlan(spec, pack, config)`` does every allocation and check
    once; ``plan(x)`` then only launches the engine's kernels on the current
    stream (no host synchronisation, no allocation), so it can be timed
    with CUDA events or captured into a CUDA graph.  Used by bench.py.

    The fused variant is resolved once at planning time (``self.variant``)
    and passed explicitly on every call.  A plan that owns its scratch
    zero-fills it once and calls with WF_FUSED_COUNTERS_CLEAN (the
    warp-specialised kernel leaves its dependency counters zero, so the
    per-call reset is skipped); a plan given a shared scratch
    (:class:`LayerStack`, :class:`HostPipeline`) never does.
    """

    def __init__(self, spec: LayerSpec, pack: KernelPack, config: EngineConfig | None = None, scratch=None):
        cfg = config or EngineConfig(kind="fused")
        if cfg.kind == "direct":
            raise InvalidParameterError("LayerPlan covers the transformed engines")
        if not isinstance(pack, KernelPack):
            raise ShapeMismatchError("LayerPlan needs a prebuilt KernelPack")
        basis = _basis_for(cfg, spec)
        self.pack = _resolve_pack(pack, spec, basis)
        self.spec, self.cfg = spec, cfg
        self.dev = _dev.require_cuda(cfg.device)
        self.lib = _lib.load()
        self.layer = _lib.layer_struct(spec)
        self.tf = _lib.TRANSFORMS[cfg.transform]
        self.prec = _lib.PRECISIONS[cfg.precision]
        self.variant = None
        with _on(self.dev):
            if cfg.kind == "fused":
                v = self.lib.wf_fused_variant(self.layer, cfg.tile, self.tf, _opts(cfg))
                if v < 0:
                    _lib.check(-v, "wf_fused_variant")
                self.variant = _lib.VARIANT_NAMES[v]
                self._pinned = _lib.fused_opts(self.variant, 0, cfg.ring_bytes)
                self.nbytes = int(self.lib.wf_fused_scratch_bytes_ex(self.layer, cfg.tile, self.tf, self._pinned))
            else:
                self.nbytes = int(self.lib.wf_three_stage_scratch_bytes(self.layer, cfg.tile, self.tf))
            if scratch is not None and scratch.numel() >= self.nbytes:
                self.scratch = scratch                    # shared with other plans on the same stream
                self.shared = True
            else:
                self.scratch = _dev.torch.zeros(max(self.nbytes, 16), dtype=_dev.torch.uint8, device=self.dev)
                self.shared = False
            self.vpack = self.pack.device_mma(self.dev, cfg.precision)
            self.out = _dev.torch.empty(spec.output_dims(), dtype=_dev.torch.float32, device=self.dev)
        self.ran = ctypes.c_int(0)

    @property
    def flags(self) -> int:
        return 0 if self.shared else _lib.WF_FUSED_COUNTERS_CLEAN

    def share_scratch(self, scratch) -> None:
        """Use ``scratch`` (at least ``nbytes``, shared with other plans on one stream)."""
        if scratch.numel() < self.nbytes:
            raise InvalidParameterError(f"shared scratch {scratch.numel()} B < {self.nbytes} B")
        self.scratch = scratch
        self.shared = True

    def _check(self, t, dims, name):
        if not _dev.is_torch(t) or not t.is_cuda or t.device != self.dev:
            raise ShapeMismatchError(f"{name} must be a CUDA tensor on {self.dev}")
        if t.dtype != _dev.torch.float32 or not t.is_contiguous():
            raise ShapeMismatchError(f"{name} must be a contiguous float32 tensor")
        if tuple(t.shape) != tuple(dims):
            raise ShapeMismatchError(f"{name} dims {tuple(t.shape)} do not match {tuple(dims)}")
        if t.data_ptr() % 16:
            raise ShapeMismatchError(f"{name} must be 16-byte aligned (bulk copies)")

    def __call__(self, x, out=None):
        """Launch on the current stream; x: contiguous f32 CUDA tensor (B, C, H, W)."""
        y = self.out if out is None else out
        self._check(x, self.spec.input_dims(), "input")
        if out is not None:
            self._check(out, self.spec.output_dims(), "output")
        stream = _dev.stream_ptr(self.dev)
        with _on(self.dev):
            if self.cfg.kind == "fused":
                self._pinned.flags = self.flags
                rc = self.lib.wf_conv_fused_ex(_dev.ptr(x), _dev.ptr(self.vpack), _dev.ptr(y),
                                               _dev.ptr(self.scratch), self.nbytes, self.layer, self.cfg.tile,
                                               self.tf, self.prec, self._pinned, ctypes.byref(self.ran), stream)
            else:
                rc = self.lib.wf_conv_three_stage(_dev.ptr(x), _dev.ptr(self.vpack), _dev.ptr(y),
                                                  _dev.ptr(self.scratch), self.nbytes, self.layer, self.cfg.tile,
                                                  self.tf, self.prec, stream)
        _lib.check(rc, "LayerPlan")
        return y


class LayerStack:
    """Back-to-back layers on one stream (layer chaining).

    ``LayerStack(specs, packs, configs)`` plans every layer once; calling it
    runs them in order on the current stream -- layer i's output buffer is
    layer i+1's input, with no host synchronisation, re-layout or copy in
    between (activations stay NCHW f32 in HBM).  The layers share one
    scratch buffer (the size of the largest), which is safe because they are
    stream-ordered; every plan then resets its own dependency counters per
    call.  As in the reference there is no bias, activation or pooling
    between layers, so consecutive specs must match:
    ``specs[i].output_dims() == specs[i + 1].input_dims()``.
    """

    def __init__(self, specs, packs, configs):
        specs, packs = list(specs), list(packs)
        configs = list(configs) if isinstance(configs, (list, tuple)) else [configs] * len(specs)
        if not specs or not (len(specs) == len(packs) == len(configs)):
            raise InvalidParameterError("LayerStack needs matching, non-empty specs / packs / configs")
        for i in range(len(specs) - 1):
            if specs[i].output_dims() != specs[i + 1].input_dims():
                raise ShapeMismatchError(f"layer {i} output {specs[i].output_dims()} does not feed layer {i + 1} "
                                         f"input {specs[i + 1].input_dims()}")
        self.plans = [LayerPlan(spec, pack, cfg) for spec, pack, cfg in zip(specs, packs, configs)]
        # one scratch, the largest, for every plan (stream-ordered use)
        shared = max((p.scratch for p in self.plans), key=lambda t: t.numel())
        for plan in self.plans:
            plan.share_scratch(shared)

    def __call__(self, x):
        """Launch every layer on the current stream; returns the last output."""
        for plan in self.plans:
            x = plan(x)
        return x

    @property
    def direct_flops(self) -> int:
        return sum(p.spec.direct_flops() for p in self.plans)


class HostPipeline:
    """One layer over host (pinned) buffers, batch-chunked so the PCIe copies
    overlap the compute.

    ``HostPipeline(spec, pack, config, chunks=8)(x_host, y_host)`` splits the
    batch into ``chunks`` contiguous slices (images are independent: the tile
    order is batch-major, reference tiling.py:8-11) and runs, per slice, the
    host->device copy on one stream, the layer on a second and the
    device->host copy on a third, chained by events -- so slice i+1 is
    uploading while slice i computes and slice i-1 downloads.  The result
    is bitwise the one of a single call on the whole batch (every engine
    path shares the same arithmetic).  Returns after the last download.
    """

    def __init__(self, spec: LayerSpec, pack: KernelPack, config: EngineConfig | None = None, chunks: int = 8,
                 graph: bool = True, split=None, depth: int = 1):
        cfg = config or EngineConfig(kind="fused")
        self.use_graph = graph
        self._graph = None
        self._graph_key = None
        self.spec, self.cfg = spec, cfg
        if split is not None:
            # explicit slice sizes (e.g. small first / last slices shorten the
            # pipeline's fill and drain)
            sizes = [int(v) for v in split]
            if not sizes or min(sizes) < 1 or sum(sizes) != spec.batch:
                raise InvalidParameterError("split must be positive slice sizes summing to the batch")
        else:
            if chunks < 1:
                raise InvalidParameterError("chunks must be >= 1")
            chunks = min(chunks, spec.batch)
            base, extra = divmod(spec.batch, chunks)
            sizes = [base + (1 if i < extra else 0) for i in range(chunks)]
        self.bounds = []
        b0 = 0
        for nb in sizes:
            self.bounds.append((b0, b0 + nb))
            b0 += nb
        torch = _dev.torch
        self.dev = _dev.require_cuda(cfg.device)
        self.plans = {}
        for nb in sorted({hi - lo for lo, hi in self.bounds}, reverse=True):
            sub = LayerSpec(nb, spec.in_channels, spec.out_channels, spec.height, spec.width, spec.kernel,
                            spec.pad_lo, spec.pad_hi)
            self.plans[nb] = LayerPlan(sub, pack, cfg)
        if len(self.plans) > 1:
            # slices of different sizes share the largest scratch (one compute stream)
            shared = max((p.scratch for p in self.plans.values()), key=lambda t: t.numel())
            for plan in self.plans.values():
                plan.share_scratch(shared)
        # `depth` sets of device staging buffers: submit() of call k + 1 uploads
        # while call k computes and downloads (depth 1: one call at a time)
        if depth < 1:
            raise InvalidParameterError("depth must be >= 1")
        self.depth = depth
        self.x_devs = [torch.empty(spec.input_dims(), dtype=torch.float32, device=self.dev) for _ in range(depth)]
        self.y_devs = [torch.empty(spec.output_dims(), dtype=torch.float32, device=self.dev) for _ in range(depth)]
        self.x_dev, self.y_dev = self.x_devs[0], self.y_devs[0]
        self.streams = [torch.cuda.Stream(self.dev) for _ in range(3)]
        n = len(self.bounds)
        self.ev_in = [[torch.cuda.Event() for _ in range(n)] for _ in range(depth)]
        self.ev_comp = [[torch.cuda.Event() for _ in range(n)] for _ in range(depth)]
        self.ev_done = [None] * depth       # last download of the call that used buffer set k
        self.ev_comp_done = [None] * depth  # last layer launch of that call
        self._calls = 0

    def __call__(self, x_host, y_host):
        """x_host (B, C, H, W) and y_host (B, C', H', W'): CPU f32 tensors, ideally pinned.

        With ``graph=True`` (default) the whole chunked pipeline -- copies,
        kernels and the cross-stream events -- is captured once per
        (x_host, y_host) pair into a CUDA graph and replayed, so the host
        issues one launch per call instead of ~10 per slice.
        """
        torch = _dev.torch
        key = (x_host.data_ptr(), y_host.data_ptr())
        if self.use_graph and x_host.is_pinned() and y_host.is_pinned():
            if self._graph is None or self._graph_key != key:
                self._issue(x_host, y_host)                    # warm: attributes, first-launch setup
                torch.cuda.synchronize(self.dev)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._issue(x_host, y_host)
                self._graph, self._graph_key = g, key
            self._graph.replay()
            torch.cuda.current_stream(self.dev).synchronize()
            return y_host
        self._issue(x_host, y_host)
        self.streams[2].synchronize()
        return y_host

    def _issue(self, x_host, y_host, k=0, fork=True):
        torch = _dev.torch
        s_in, s_comp, s_out = self.streams
        x_dev, y_dev = self.x_devs[k], self.y_devs[k]
        ev_in, ev_comp = self.ev_in[k], self.ev_comp[k]
        cur = torch.cuda.current_stream(self.dev)
        if fork:
            for s in self.streams:
                s.wait_stream(cur)
        for i, (lo, hi) in enumerate(self.bounds):
            with torch.cuda.stream(s_in):
                x_dev[lo:hi].copy_(x_host[lo:hi], non_blocking=True)
                ev_in[i].record(s_in)
            with torch.cuda.stream(s_comp):
                s_comp.wait_event(ev_in[i])
                self.plans[hi - lo](x_dev[lo:hi], out=y_dev[lo:hi])
                ev_comp[i].record(s_comp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_comp[i])
                y_host[lo:hi].copy_(y_dev[lo:hi], non_blocking=True)
        if fork:
            cur.wait_stream(s_out)

    def submit(self, x_host, y_host):
        """Queue one call without waiting for it (streaming use: a serving
        loop that feeds batches back to back).  Call k + 1 uploads into the
        next of the ``depth`` staging sets while call k computes and
        downloads, so in the steady state a call costs max(upload, download,
        compute) instead of their pipelined sum.  The three streams keep the
        calls in order; the only extra edges are the reuse of a staging set
        (upload after the layer launches that read it, layer launches after
        the downloads that read their output).  ``wait()`` returns when every
        submitted call has landed in its ``y_host``; the caller must not
        reuse a ``y_host`` (or change an ``x_host``) of a call still in flight.
        """
        torch = _dev.torch
        k = self._calls % self.depth
        s_in, s_comp, s_out = self.streams
        if self._calls == 0:
            cur = torch.cuda.current_stream(self.dev)
            for s in self.streams:
                s.wait_stream(cur)
        if self.ev_comp_done[k] is not None:
            s_in.wait_event(self.ev_comp_done[k])
            s_comp.wait_event(self.ev_done[k])
        self._issue(x_host, y_host, k, fork=False)
        self.ev_comp_done[k] = self.ev_comp[k][-1]
        ev = self.ev_done[k] or torch.cuda.Event()
        ev.record(s_out)
        self.ev_done[k] = ev
        self._calls += 1
        return ev

    def wait(self):
        """Block until every submitted call has been downloaded."""
        self.streams[2].synchronize()
