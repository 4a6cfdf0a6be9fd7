"""Machine models and fusion planning, CPU (reference) and B200.

Two halves:

* The reference's planner API, restated (roofline.py:40-254): a
  ``MachineModel`` read from the same JSON fields, the arithmetic-intensity
  helpers (``ai_l3`` = alpha R / 2, ``ai_mem`` = C C' / (2 (C + C'))), the R
  bounds (``r_lower_bound`` = ceil(2 CMR_L3 / alpha), ``r_upper_bound`` =
  floor(fraction L2 / 4 / (max(C, C') (T^2 + 1)))) and ``plan`` ->
  ``PlanReport`` -- so the reference's machine files and reports keep
  working unchanged.

* ``B200Model`` / ``plan_b200``: the same
  flop-per-byte accounting with the GPU's levels -- HBM, the 126 MB L2 (the
  paper's shared cache), and the per-SM SMEM + TMEM (the paper's private
  cache) -- with measured bandwidths.  It predicts, per layer, which
  engine variant runs (persistent L2-staged dataflow kernel vs L2 waves),
  the per-level times, and the fused / three-stage crossover.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from pathlib import Path

from .errors import InvalidParameterError, MachineModelError
from .tensor import LayerSpec

_FP32 = 4

# JSON field -> attribute (the reference's interchange contract, roofline.py:28-37)
_MODEL_FIELDS = {
    "name": "name",
    "peak_flops": "peak_flops",
    "mem_bandwidth_bytes_per_s": "mem_bandwidth",
    "l3_bandwidth_bytes_per_s": "l3_bandwidth",
    "l2_bytes_per_core": "l2_bytes",
    "l3_bytes": "l3_bytes",
    "cores": "cores",
}
_NUMERIC = ("peak_flops", "mem_bandwidth", "l3_bandwidth", "l2_bytes", "l3_bytes", "cores")


def _require_positive(**kw) -> None:
    for k, v in kw.items():
        if v <= 0:
            raise InvalidParameterError(f"{k} must be positive, got {v}")


def _require_fraction(fraction: float) -> None:
    if not 0.0 < fraction <= 1.0:
        raise InvalidParameterError(f"occupancy fraction must be in (0, 1], got {fraction}")


@dataclass(frozen=True)
class MachineModel:
    """A CPU machine: peak flop/s, memory and shared-cache bandwidth, cache sizes."""

    name: str
    peak_flops: float
    mem_bandwidth: float
    l3_bandwidth: float
    l2_bytes: int
    l3_bytes: int
    cores: int

    def __post_init__(self):
        for f in _NUMERIC:
            if getattr(self, f) <= 0:
                raise MachineModelError(f"machine field {f} must be positive")

    @property
    def cmr_mem(self) -> float:
        return self.peak_flops / self.mem_bandwidth

    @property
    def cmr_l3(self) -> float:
        return self.peak_flops / self.l3_bandwidth

    @classmethod
    def from_dict(cls, raw: dict) -> "MachineModel":
        missing = [f for f in _MODEL_FIELDS if f not in raw]
        if missing:
            raise MachineModelError(f"machine model is missing {missing[0]!r}")
        kw = {attr: raw[f] for f, attr in _MODEL_FIELDS.items()}
        if not isinstance(kw["name"], str) or not kw["name"]:
            raise MachineModelError("machine field 'name' must be a label")
        for attr in _NUMERIC:
            v = kw[attr]
            if isinstance(v, bool) or not isinstance(v, (int, float)):
                field_name = next(f for f, a in _MODEL_FIELDS.items() if a == attr)
                raise MachineModelError(f"machine field {field_name!r} must be a number")
        for attr in ("l2_bytes", "l3_bytes", "cores"):
            kw[attr] = int(kw[attr])
        return cls(**kw)

    @classmethod
    def from_file(cls, path) -> "MachineModel":
        p = Path(path)
        try:
            raw = json.loads(p.read_text())
        except OSError as exc:
            raise MachineModelError(f"cannot read machine model: {exc}") from exc
        except json.JSONDecodeError as exc:
            raise MachineModelError(f"machine model {p} is not valid JSON: {exc}") from exc
        if not isinstance(raw, dict):
            raise MachineModelError(f"machine model {p} must be an object")
        return cls.from_dict(raw)


def sample_model_path(name: str) -> Path:
    """Path of a machine model shipped with the package (machines/<name>.json)."""
    p = Path(__file__).parent / "machines" / f"{name}.json"
    if not p.exists():
        raise MachineModelError(f"no sample machine model {name!r}")
    return p


def l3_fit(c_in: int, c_out: int, tile: int, l3_bytes: int, fraction: float = 0.5):
    """(fits, bytes): whether the 4 C C' T^2 byte kernel pack fits its shared-cache share."""
    _require_positive(c_in=c_in, c_out=c_out, tile=tile, l3_bytes=l3_bytes)
    _require_fraction(fraction)
    need = _FP32 * c_in * c_out * tile * tile
    return need <= fraction * l3_bytes, need


def ai_l3(r: int, alpha: float = 1.0) -> float:
    """Shared-cache intensity of a task of R tiles: alpha R / 2 flop per byte of pack."""
    if r < 1:
        raise InvalidParameterError(f"R must be >= 1, got {r}")
    return alpha * r / 2.0


def ai_mem(c_in: int, c_out: int) -> float:
    """Memory intensity of the fused engine: C C' / (2 (C + C'))."""
    _require_positive(c_in=c_in, c_out=c_out)
    return c_in * c_out / (2.0 * (c_in + c_out))


def ai_mem_lower_bound(c_in: int, c_out: int) -> float:
    _require_positive(c_in=c_in, c_out=c_out)
    return min(c_in, c_out) / 4.0


def r_lower_bound(cmr_l3: float, alpha: float = 1.0) -> int:
    """Smallest R whose shared-cache intensity reaches the machine balance."""
    _require_positive(cmr_l3=cmr_l3, alpha=alpha)
    return math.ceil(2.0 * cmr_l3 / alpha)


def l2_element_budget(l2_bytes: int, fraction: float = 0.5) -> int:
    _require_positive(l2_bytes=l2_bytes)
    _require_fraction(fraction)
    return math.floor(fraction * l2_bytes / _FP32)


def r_upper_bound(c_in: int, c_out: int, tile: int, l2_bytes: int, fraction: float = 0.5) -> int:
    """Largest R whose scratch, <= 4 R max(C, C') (T^2 + 1) bytes, fits the private-cache share."""
    _require_positive(c_in=c_in, c_out=c_out, tile=tile, l2_bytes=l2_bytes)
    _require_fraction(fraction)
    return l2_element_budget(l2_bytes, fraction) // (max(c_in, c_out) * (tile * tile + 1))


@dataclass(frozen=True)
class PlanReport:
    layer: LayerSpec
    tile: int
    alpha: float
    machine: str
    l3_fits: bool
    l3_required_bytes: int
    r_lower: int
    r_upper: int
    chosen_r: int
    feasible: bool
    utilization: dict
    utilization_overall: float

    def format(self) -> str:
        u = self.utilization
        return "\n".join([
            f"machine: {self.machine}",
            (f"layer: B={self.layer.batch} C={self.layer.in_channels} C'={self.layer.out_channels} "
             f"D={self.layer.height} W={self.layer.width} K={self.layer.kernel}  T={self.tile}  "
             f"alpha={self.alpha:g}"),
            (f"kernel pack: {self.l3_required_bytes} bytes; fits shared-cache share: "
             f"{'yes' if self.l3_fits else 'NO'}"),
            (f"R lower bound (saturate shared cache): {self.r_lower}   "
             f"R upper bound (scratch fits L2 share): {self.r_upper}"),
            f"chosen R: {self.chosen_r}   feasible: {'yes' if self.feasible else 'NO'}",
            (f"predicted utilization: shared-cache {u['l3']:.3f}, memory {u['mem']:.3f} -> overall "
             f"{self.utilization_overall:.3f}"),
        ])


def plan(layer: LayerSpec, tile: int, machine: MachineModel, alpha: float = 1.0, l2_fraction: float = 0.5,
         l3_fraction: float = 0.5) -> PlanReport:
    """Fit checks and R bounds of the reference planner (roofline.py:221-254):
    chosen R = the upper bound; infeasible when it cannot reach the lower
    bound; utilization = min over levels of min(1, AI / CMR)."""
    fits, need = l3_fit(layer.in_channels, layer.out_channels, tile, machine.l3_bytes, l3_fraction)
    lo = r_lower_bound(machine.cmr_l3, alpha)
    hi = r_upper_bound(layer.in_channels, layer.out_channels, tile, machine.l2_bytes, l2_fraction)
    chosen = hi if hi >= 1 else 0
    u3 = min(1.0, ai_l3(chosen, alpha) / machine.cmr_l3) if chosen >= 1 else 0.0
    um = min(1.0, ai_mem(layer.in_channels, layer.out_channels) / machine.cmr_mem)
    return PlanReport(layer=layer, tile=tile, alpha=alpha, machine=machine.name, l3_fits=fits,
                      l3_required_bytes=need, r_lower=lo, r_upper=hi, chosen_r=chosen,
                      feasible=1 <= lo <= hi, utilization={"l3": u3, "mem": um},
                      utilization_overall=min(u3, um))


# ------------------------------------------------------------------ B200
@dataclass(frozen=True)
class B200Model:
    """The GPU's levels for the fusion plan (measured on this pool's B200s).

    hbm / l2 bandwidth in bytes/s (L2 -> SM streaming measured with bulk
    copies, tools/ubench), bf16 tensor peak in flop/s (MEASURED_PEAKS.json),
    on-chip capacities per SM."""

    name: str = "b200"
    sms: int = 148
    hbm_bandwidth: float = 6545.3e9
    l2_bandwidth: float = 12.4e12
    l2_bytes: int = 126 * 2**20
    smem_bytes_per_sm: int = 228 * 1024
    tmem_bytes_per_sm: int = 256 * 1024
    tensor_bf16_flops: float = 1657.2e12
    hbm_bytes: int = 180 * 10**9

    @classmethod
    def from_file(cls, path) -> "B200Model":
        raw = json.loads(Path(path).read_text())
        known = {f for f in cls.__dataclass_fields__}
        bad = [k for k in raw if k not in known]
        if bad:
            raise MachineModelError(f"unknown B200 model field {bad[0]!r}")
        return cls(**raw)


@dataclass(frozen=True)
class B200PlanReport:
    layer: LayerSpec
    tile: int
    transform: str
    passes: int
    n_tile: int
    block_tiles: int
    blocks: int
    fused_variant: str
    r_lower: int
    r_upper: int
    bytes: dict = field(default_factory=dict)      # per level, fused and three-stage
    seconds: dict = field(default_factory=dict)    # per level / engine prediction
    predicted_winner: str = ""
    fitted: dict = field(default_factory=dict)     # times from the measurement-fitted rates (B200Fit)

    def format(self) -> str:
        s, b = self.seconds, self.bytes
        return "\n".join([
            (f"B200 plan: B={self.layer.batch} C={self.layer.in_channels} C'={self.layer.out_channels} "
             f"D={self.layer.height} W={self.layer.width}  {self.transform} T={self.tile}  passes={self.passes}"),
            (f"tiles {self.n_tile} in {self.blocks} blocks of {self.block_tiles} (MMA M); fused variant: "
             f"{self.fused_variant}"),
            (f"R lower bound (saturate L2 with the pack stream): {self.r_lower}   "
             f"R upper bound (task scratch fits SMEM+TMEM): {self.r_upper}"),
            (f"HBM bytes fused {b['hbm_fused'] / 1e6:.1f} MB, three-stage {b['hbm_three'] / 1e6:.1f} MB; "
             f"L2 bytes fused {b['l2_fused'] / 1e6:.1f} MB"),
            (f"time (us): HBM fused {s['hbm_fused'] * 1e6:.1f}, L2 fused {s['l2_fused'] * 1e6:.1f}, tensor "
             f"{s['tensor'] * 1e6:.1f} -> fused {s['fused'] * 1e6:.1f}; three-stage {s['three'] * 1e6:.1f}"),
            (f"fitted to measured layers (machines/b200_fit.json): fused {self.fitted['fused'] * 1e6:.1f} us, "
             f"three-stage {self.fitted['three'] * 1e6:.1f} us" if self.fitted else "no fitted rates for this transform"),
            f"predicted winner: {self.predicted_winner}",
        ])


def plan_b200(layer: LayerSpec, tile: int, machine: B200Model | None = None, transform: str = "winograd",
              precision: str = "3xbf16", block_tiles: int = 128) -> B200PlanReport:
    """Per-level prediction for one layer on the B200.

    Fused (L2-staged dataflow): HBM moves input + output + pack; L2 moves,
    per tile, the transformed tiles U (hi + lo bf16) written and read and
    the products M written and read, plus the input windows (re-read T^2 /
    m^2 times) and the output.  Three-stage: U and M make an HBM round trip
    too.  Tensor: passes x F_gemm at the bf16 peak.  Each engine's time is
    its slowest level (no overlap loss modelled).  R on the GPU is the tile
    block of one MMA (M = 128): the L2 pack stream of a block reaches the
    L2 balance point when R >= 2 CMR_L2 (the reference's r_lower with the
    L2 as the shared cache), and a block's U + M must fit the per-SM
    on-chip memory for a single-SM fusion (r_upper) -- the reason the B200
    design stages through L2.
    """
    mach = machine or B200Model()
    passes = 1 if precision == "bf16" else 3
    c, cp = layer.in_channels, layer.out_channels
    if transform == "fft":
        m, pos, kdim, ndim = 14, 144, 2 * c, 2 * cp
        f_tile = 8 * 144 * c * cp
        pack = 8 * 144 * c * cp
    else:
        m, pos, kdim, ndim = tile - layer.kernel + 1, tile * tile, c, cp
        f_tile = 2 * c * cp * tile * tile
        pack = _FP32 * tile * tile * c * cp
    n_tile = layer.batch * -(-layer.out_height // m) * -(-layer.out_width // m)
    blocks = -(-n_tile // block_tiles)
    io = _FP32 * (layer.batch * c * layer.height * layer.width + layer.batch * cp * layer.out_height * layer.out_width)
    u_tile = pos * kdim * 4            # bf16 hi + lo
    m_tile = pos * ndim * 4            # f32
    window = _FP32 * layer.batch * c * layer.height * layer.width * (tile * tile) / (m * m) if transform != "fft" \
        else _FP32 * layer.batch * c * layer.height * layer.width * 256 / 196
    hbm_fused = io + pack
    hbm_three = hbm_fused + 2 * n_tile * (u_tile + m_tile)
    l2_fused = window + 2 * n_tile * (u_tile + m_tile) + _FP32 * layer.batch * cp * layer.out_height * layer.out_width \
        + blocks * pos * kdim * ndim * 4 / 2
    tensor = passes * f_tile * n_tile / mach.tensor_bf16_flops
    t_hbm_f, t_hbm_3 = hbm_fused / mach.hbm_bandwidth, hbm_three / mach.hbm_bandwidth
    t_l2 = l2_fused / mach.l2_bandwidth
    t_fused = max(t_hbm_f, t_l2, tensor)
    t_three = max(t_hbm_3, tensor, t_l2)
    cmr_l2 = mach.tensor_bf16_flops / passes / mach.l2_bandwidth
    r_lo = math.ceil(2.0 * cmr_l2)
    onchip = mach.smem_bytes_per_sm + mach.tmem_bytes_per_sm
    r_up = int(onchip // (u_tile + m_tile))
    cppad = -(-ndim // 16) * 16
    if transform == "fft":
        variant = "L2 waves (three kernels per wave)"
    elif cppad <= 64 or (cppad <= 128 and tile <= 8):
        variant = "persistent dataflow kernel (L2-staged rings)"
    else:
        variant = "L2 waves (three kernels per wave)"
    winner = "fused" if t_fused < 0.95 * t_three else ("three_stage" if t_three < 0.95 * t_fused else "tie")
    fitted = {}
    fit_path = Path(__file__).parent / "machines" / "b200_fit.json"
    if transform != "fft" and fit_path.exists():
        # rates fitted to measured layers (fit_b200): the prediction that decides the crossover
        fit = B200Fit.from_file(fit_path)
        ops = transform_ops(layer, tile)
        tens = passes * f_tile * n_tile
        tf = fit.t0_fused + max(l2_fused / fit.l2_rate, tens / (fit.tc_eff * mach.tensor_bf16_flops), ops / fit.cc_rate)
        t3 = 3 * fit.t0_launch + hbm_three / fit.hbm_rate + tens / (fit.tc_eff * mach.tensor_bf16_flops) + \
            ops / fit.cc_rate
        fitted = {"fused": tf, "three": t3}
        winner = "fused" if tf < t3 else "three_stage"
    return B200PlanReport(layer=layer, tile=tile, transform=transform, passes=passes, n_tile=n_tile,
                          block_tiles=block_tiles, blocks=blocks, fused_variant=variant, r_lower=r_lo, r_upper=r_up,
                          bytes={"hbm_fused": hbm_fused, "hbm_three": hbm_three, "l2_fused": l2_fused},
                          seconds={"hbm_fused": t_hbm_f, "hbm_three": t_hbm_3, "l2_fused": t_l2, "tensor": tensor,
                                   "fused": t_fused, "three": t_three},
                          predicted_winner=winner, fitted=fitted)


# ------------------------------------------------- B200 model fitted to measurements
# CUDA-core operations per transform line (the factored 1-D transforms of
# csrc/common.cuh: bt*_line / at*_line) and per bf16 hi/lo split of a value.
_BT_LINE = {4: 6, 5: 12, 6: 14, 7: 22, 8: 26}
_AT_LINE = {4: 4, 5: 8, 6: 10, 7: 16, 8: 20}
_SPLIT_OPS = 4


def transform_ops(layer: LayerSpec, tile: int) -> float:
    """CUDA-core operations of the forward (2T lines + T^2 splits per tile and
    input channel) and inverse (T + m lines per tile and output channel)
    transforms of one Winograd layer."""
    m = tile - layer.kernel + 1
    n_tile = layer.batch * -(-layer.out_height // m) * -(-layer.out_width // m)
    fwd = 2 * tile * _BT_LINE[tile] + _SPLIT_OPS * tile * tile
    inv = (tile + m) * _AT_LINE[tile]
    return float(n_tile) * (layer.in_channels * fwd + layer.out_channels * inv)


@dataclass(frozen=True)
class B200Fit:
    """Effective rates of the B200 engines, fitted to measured layer times
    (``fit_b200``).  Fused (L2-staged dataflow kernel):

        t_fused = t0_fused + max(L2 ring bytes / l2_rate, tensor / tc_eff, ops / cc_rate)

    Three-stage (three kernels, the intermediates make an HBM round trip):

        t_three = 3 t0_launch + HBM bytes / hbm_rate + tensor / tc_eff + ops / cc_rate
    """

    l2_rate: float          # bytes/s of ring traffic the fused kernel sustains
    hbm_rate: float         # bytes/s the stage kernels sustain
    cc_rate: float          # transform operations/s (all SMs)
    tc_eff: float           # fraction of the bf16 tensor peak the GEMMs reach
    t0_fused: float         # fixed cost of a fused launch (fill + drain), s
    t0_launch: float        # fixed cost per stage kernel, s
    rms_log_error: float = 0.0
    samples: int = 0

    def predict(self, layer: LayerSpec, tile: int, machine: "B200Model | None" = None, precision: str = "3xbf16"):
        """-> (t_fused, t_three) in seconds."""
        mach = machine or B200Model()
        rep = plan_b200(layer, tile, mach, precision=precision)
        tensor = rep.seconds["tensor"] * mach.tensor_bf16_flops
        ops = transform_ops(layer, tile)
        t_f = self.t0_fused + max(rep.bytes["l2_fused"] / self.l2_rate, tensor / (self.tc_eff * mach.tensor_bf16_flops),
                                  ops / self.cc_rate)
        t_3 = 3 * self.t0_launch + rep.bytes["hbm_three"] / self.hbm_rate + \
            tensor / (self.tc_eff * mach.tensor_bf16_flops) + ops / self.cc_rate
        return t_f, t_3

    def winner(self, layer: LayerSpec, tile: int, machine=None, precision: str = "3xbf16") -> str:
        t_f, t_3 = self.predict(layer, tile, machine, precision)
        return "fused" if t_f < t_3 else "three_stage"

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k in self.__dataclass_fields__}

    @classmethod
    def from_file(cls, path) -> "B200Fit":
        return cls(**json.loads(Path(path).read_text()))


def fit_b200(measurements, machine: "B200Model | None" = None) -> B200Fit:
    """Least-squares fit (in log time) of the B200Fit rates to measured
    Winograd layers: ``measurements`` = iterable of dicts with ``layer``
    (LayerSpec), ``tile``, ``fused_s`` (warp-specialised kernel) and
    ``three_s`` -- e.g. the per-layer rows of bench.py's per_config block
    (machines/b200_measured.json).  The reference fits nothing (its planner
    reads given machine numbers, roofline.py:227-254); on the B200 the
    achievable rates of the dataflow kernels are what decides the
    fused / three-stage crossover, so they are measured and fitted."""
    import numpy as np
    from scipy.optimize import least_squares

    mach = machine or B200Model()
    rows = list(measurements)
    if len(rows) < 6:
        raise InvalidParameterError("need at least 6 measured layers to fit the B200 model")
    feats = []
    for r in rows:
        rep = plan_b200(r["layer"], r["tile"], mach)
        feats.append((rep.bytes["l2_fused"], rep.bytes["hbm_three"], rep.seconds["tensor"] * mach.tensor_bf16_flops,
                      transform_ops(r["layer"], r["tile"]), r["fused_s"], r["three_s"]))
    f = np.array(feats, dtype=np.float64)

    def model(x):
        l2, hbm, cc, tc, t0f, t0l = np.exp(x)
        tens = f[:, 2] / (tc * mach.tensor_bf16_flops)
        ops = f[:, 3] / cc
        tf = t0f + np.maximum(np.maximum(f[:, 0] / l2, tens), ops)
        t3 = 3 * t0l + f[:, 1] / hbm + tens + ops
        return tf, t3

    def resid(x):
        tf, t3 = model(x)
        return np.concatenate([np.log(tf / f[:, 4]), np.log(t3 / f[:, 5])])

    x0 = np.log([5e12, 4e12, 3e13, 0.4, 10e-6, 5e-6])
    lo = np.log([1e11, 1e11, 1e11, 0.01, 1e-7, 1e-7])
    hi = np.log([1e15, 2e13, 1e16, 1.0, 1e-3, 1e-3])
    sol = least_squares(resid, x0, bounds=(lo, hi))
    p = np.exp(sol.x)
    err = float(np.sqrt(np.mean(resid(sol.x) ** 2)))
    return B200Fit(l2_rate=float(p[0]), hbm_rate=float(p[1]), cc_rate=float(p[2]), tc_eff=float(p[3]),
                   t0_fused=float(p[4]), t0_launch=float(p[5]), rms_log_error=err, samples=len(rows))


def measured_layers(path=None):
    """The measured per-layer table shipped with the package
    (machines/b200_measured.json: bench.py per_config rows) as fit_b200 input."""
    p = Path(path) if path else Path(__file__).parent / "machines" / "b200_measured.json"
    doc = json.loads(p.read_text())
    out = []
    for r in doc["layers"]:
        out.append({"layer": LayerSpec(r["batch"], r["c"], r["cp"], r["hw"], r["hw"], 3, 1, 1), "tile": r["tile"],
                    "fused_s": r["fused_ms"] * 1e-3, "three_s": r["three_stage_ms"] * 1e-3, "name": r["name"]})
    return out
