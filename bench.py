"""Benchmark: direct-convolution-equivalent TFLOP/s of the fused transformed
convolution layer on B200, with roofline fraction and the CPU baseline.

Default workload (BASELINE.json configs[1], "c2"): ResNet-50 stage-1 3x3
layer, Winograd F(4x4,3x3) (T=6), B=64, C=C'=64, 56x56, stride 1, pad 1,
fp32 N(0,1) inputs, He-normal weights, 3xBF16 tensor-core mode.  A step is
one fused layer over one batch already resident in HBM; the L2 (126 MB)
is flushed before every timed step because input + output (103 MB) would
otherwise stay L2-resident.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torch.distributed.run, one rank per GPU; the batch is
sharded (weak scaling: B=64 per rank, no collective on the data path) and
the time is the max over ranks.  ``--impl reference`` times the
reference's CPU algorithm (the bit-exact C port in oracle/, all host
threads) on a bounded sample and prints the same JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Direct-conv-equivalent TFLOP/s per layer & fraction of B200 roofline"
CONFIGS = {
    # name: (B per GPU, C, C', H=W, tile, weight std rule, input distribution)
    "c2": (64, 64, 64, 56, 6, "he", "normal"),
    "c1": (1, 64, 64, 56, 4, "inv_sqrt", "normal"),
    # c5 (the sweep / scaling config) at its C = 64, 56x56 point: B = 256 per GPU
    "c5": (256, 64, 64, 56, 8, "he", "uniform"),
    # tuning shapes (not bench lines): VGG-16 conv2_2 / conv3_x at B = 32
    "vgg1": (32, 3, 64, 224, 6, "he", "normal"),
    "vgg2": (32, 64, 64, 224, 6, "he", "normal"),
    "vgg3": (32, 64, 128, 112, 6, "he", "normal"),
    "vgg4": (32, 128, 128, 112, 6, "he", "normal"),
    "vgg6": (32, 256, 256, 56, 6, "he", "normal"),
    "vgg9": (32, 512, 512, 28, 6, "he", "normal"),
    "c5_32_112": (256, 32, 32, 112, 8, "he", "uniform"),
    "c5_16_112": (256, 16, 16, 112, 8, "he", "uniform"),
    "c5_128_56": (256, 128, 128, 56, 8, "he", "uniform"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--engine", default="fused", choices=["fused", "three_stage"])
    ap.add_argument("--precision", default="3xbf16", choices=["3xbf16", "bf16"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=4, help="batch slices of the host-buffer pipeline")
    ap.add_argument("--e2e-split", default=None, help="explicit slice sizes, e.g. 8,24,24,8 (overrides --e2e-chunks)")
    return ap.parse_args()


def layer_inputs(cfg_name, batch=None, seed=1234):
    import paper_1912_02165_b200 as wf
    b, c, cp, hw, t, rule, dist = CONFIGS[cfg_name]
    spec = wf.LayerSpec(batch or b, c, cp, hw, hw, 3, 1, 1)
    rng = np.random.default_rng(seed)
    if dist == "uniform":
        x = rng.uniform(-1.0, 1.0, spec.input_dims()).astype(np.float32)
    else:
        x = rng.standard_normal(spec.input_dims()).astype(np.float32)
    std = np.sqrt(2.0 / (9 * c)) if rule == "he" else 1.0 / np.sqrt(9 * c)
    w = (np.random.default_rng(seed + 1).standard_normal(spec.kernel_dims()) * std).astype(np.float32)
    return spec, t, x, w


def roofline_terms(spec, t, precision):
    """Algorithmic bytes / flops of one layer."""
    m = t - 2
    n_tile = spec.batch * -(-spec.out_height // m) * -(-spec.out_width // m)
    q_fused = 4 * (spec.batch * spec.in_channels * spec.height * spec.width
                   + spec.batch * spec.out_channels * spec.out_height * spec.out_width) \
        + 4 * t * t * spec.in_channels * spec.out_channels
    q_three = q_fused + 2 * 4 * t * t * n_tile * (spec.in_channels + spec.out_channels)
    f_gemm = 2 * n_tile * spec.in_channels * spec.out_channels * t * t
    return n_tile, q_fused, q_three, f_gemm


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """SM clocks / clock-event (throttle) reasons sampled during the timed region.

    Uses NVML directly (the same counters nvidia-smi reads) so that a timed
    region of a few milliseconds still gets many samples; falls back to one
    nvidia-smi query per sample when NVML is unavailable.
    """

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index, period_s=0.0005):
        self.index = index
        self.period = period_s
        self.samples = []            # (wall time, sm_mhz, reasons bitmask)
        self.window = None           # (t0, t1) of the timed region
        self.max_mhz = None
        self.source = "nvml"
        self._stop = threading.Event()
        self._thread = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None
            self.source = "nvidia-smi"

    def _sample(self):
        if self._nvml is not None:
            n = self._nvml
            sm = n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM)
            try:
                mask = n.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except AttributeError:
                mask = n.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
            return time.perf_counter(), float(sm), int(mask)
        out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                              "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip().split(",")
        self.max_mhz = float(out[1])
        return time.perf_counter(), float(out[0]), int(out[2].strip(), 16)

    def _run(self):
        while True:
            try:
                self.samples.append(self._sample())
            except Exception:
                pass
            if self._stop.is_set():
                break
            time.sleep(self.period)

    def __enter__(self):
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._thread.join(timeout=10)

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def summary(self):
        """Samples taken inside the timed region (wall-clock window from the
        first launch to the final synchronize); if the region was shorter
        than one sample period, the samples adjacent to it."""
        samples = self.samples
        if self.window is not None:
            t0, t1 = self.window
            inside = [s for s in samples if t0 <= s[0] <= t1]
            if not inside and samples:
                inside = sorted(samples, key=lambda s: min(abs(s[0] - t0), abs(s[0] - t1)))[:2]
            samples = inside
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["clock query unavailable"],
                    "samples": 0, "source": self.source}
        sm = [s[1] for s in samples]
        reasons = sorted({name for _, _, m in samples for bit, name in self.REASONS.items() if m & bit})
        return {"sm_mhz": statistics.median(sm), "sm_min_mhz": min(sm), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(samples), "source": self.source}


def cpu_baseline(cfg_name, t, spec_full, threads=None):
    """Time the reference algorithm (bit-exact C port, oracle/) on a bounded sample."""
    from oracle import oracle as O
    import paper_1912_02165_b200 as wf
    threads = threads or O.threads()
    sample_b = 2 if spec_full.batch >= 2 else 1
    spec, _, x, w = layer_inputs(cfg_name, batch=sample_b)
    pack = O.transform_kernels(w, t)
    O.conv_fused(x, pack, spec, t, 24, threads=threads)        # warm (page-in, thread pool)
    times = []
    deadline = time.perf_counter() + 15.0
    while len(times) < 3 or (time.perf_counter() < deadline and len(times) < 50):
        t0 = time.perf_counter()
        O.conv_fused(x, pack, spec, t, 24, threads=threads)
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    return {"value": spec.direct_flops() / med / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "port",
            "sample": f"{sample_b} image(s) of {cfg_name} ({spec.in_channels}->{spec.out_channels} @ "
                      f"{spec.height}x{spec.width}, T={t}), reference fused algorithm (R=24) in the bit-exact "
                      f"C port oracle/winofuse_oracle.c, median of {len(times)} runs"}


def dist_setup(n):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n and world > 1:
        raise SystemExit(f"--gpus {n} but WORLD_SIZE={world}")
    return rank, world, local


def run_reference(args):
    rank, world, _ = dist_setup(args.gpus)
    if rank != 0:
        return
    from oracle import oracle as O
    spec_full, t, _, _ = layer_inputs(args.config)
    b_total = spec_full.batch * max(world, 1)
    threads = O.threads()
    sample_b = 2 if spec_full.batch >= 2 else 1
    spec, _, x, w = layer_inputs(args.config, batch=sample_b)
    pack = O.transform_kernels(w, t)
    for _ in range(args.warmup):
        O.conv_fused(x, pack, spec, t, 24, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.conv_fused(x, pack, spec, t, 24, threads=threads)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = spec.direct_flops() * args.steps / total / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": f"synthetic {'U(-1,1)' if CONFIGS[args.config][6] == 'uniform' else 'N(0,1)'} inputs, "
                "He-normal weights (seeded)",
        "config": {"workload": f"{args.config}: F(4x4,3x3) conv, B={b_total}, C=C'={spec.in_channels}, "
                               f"{spec.height}x{spec.width}, pad 1 (CPU sample: {sample_b} image(s) per step)",
                   "tile": t, "engine": "fused (reference algorithm, R=24)"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "port",
                         "sample": f"{sample_b} image(s) per step of {args.config}; the reference's fused "
                                   f"algorithm in the bit-exact C port (oracle/winofuse_oracle.c)"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def traffic_from_profiles(cfg_name):
    """DRAM bytes per launch of the fused step from the committed ncu summary, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return d.get(cfg_name)
    return None


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_1912_02165_b200 as wf
    from paper_1912_02165_b200 import _lib

    rank, world, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    spec, t, x_np, w_np = layer_inputs(args.config, seed=1234 + 1000 * rank)
    pack = wf.transform_kernels(wf.Tensor4D(w_np), wf.make_basis(t))
    cfg = wf.EngineConfig(kind=args.engine, tile=t, precision=args.precision, device=dev)
    x_dev = torch.from_numpy(x_np).to(dev)
    pack.device_mma(dev)
    # L2 flush buffer (> 126 MB L2)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    plan = wf.LayerPlan(spec, pack, cfg)          # allocation + validation once, launches only below
    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        plan(x_dev)
    torch.cuda.synchronize(dev)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    launches0 = _lib.load().wf_kernel_launches()
    with ClockSampler(local) as clocks:
        time.sleep(0.05)                                            # sampler running before the region
        w0 = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()                                           # evict input/output from L2
            starts[i].record(stream)
            plan(x_dev)
            ends[i].record(stream)
        torch.cuda.synchronize(dev)
        clocks.mark(w0, time.perf_counter())
    launches = _lib.load().wf_kernel_launches() - launches0
    if world > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    if world > 1:
        tt = torch.tensor([total_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms = total_ms / args.steps

    # end to end through the public API with host buffers (pinned), H2D + D2H
    # inside: HostPipeline splits the batch into slices so the uploads,
    # the layer and the downloads of different slices overlap
    x_host = torch.from_numpy(x_np).pin_memory()
    y_host = torch.empty(spec.output_dims(), dtype=torch.float32, pin_memory=True)
    split = [int(v) for v in args.e2e_split.split(",")] if args.e2e_split else None
    pipe = wf.HostPipeline(spec, pack, cfg, chunks=args.e2e_chunks, split=split)
    for _ in range(2):
        pipe(x_host, y_host)
    torch.cuda.synchronize(dev)
    e2e_steps = max(3, min(args.steps, 10))
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        pipe(x_host, y_host)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())

    n_tile, q_fused, q_three, f_gemm = roofline_terms(spec, t, args.precision)

    if rank == 0:
        hbm_peak, bf16_peak, peak_kind = measured_peaks()
        b_total = spec.batch * world
        flops_total = spec.direct_flops() * world
        value = flops_total / (ms * 1e-3) / 1e12
        e2e_value = flops_total / (e2e_ms * 1e-3) / 1e12
        achieved = q_fused / (ms * 1e-3) / 1e9
        passes = 3 if args.precision == "3xbf16" else 1
        t_roof = max(q_fused / (hbm_peak * 1e9), passes * f_gemm / (bf16_peak * 1e12))
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            try:
                cpu = cpu_baseline(args.config, t, spec)
            except Exception as exc:  # the baseline is reported, never gating
                cpu = {"value": None, "unit": "TFLOP/s", "cores": 0, "kind": "port", "sample": f"failed: {exc}"}
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 io, bf16x3 split tensor-core (f32 accumulate)"
            if args.precision == "3xbf16" else "f32 io, bf16 tensor-core",
            "data": f"synthetic: seeded {'U(-1,1)' if CONFIGS[args.config][6] == 'uniform' else 'N(0,1)'} "
                    "inputs, He-normal weights (no dataset in the reference)",
            "config": {"workload": f"{args.config}: Winograd F({t - 2}x{t - 2},3x3) conv, B={b_total} "
                                   f"({spec.batch}/GPU), C=C'={spec.in_channels}, {spec.height}x{spec.width}, "
                                   f"stride 1, pad 1", "engine": args.engine, "tile": t,
                       "precision": args.precision, "l2": "flushed (256 MB write) before every timed step",
                       "images_per_s": b_total / (ms * 1e-3), "parallelism": f"batch shards x{world}"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic_from_profiles(args.config),
                         "peak_source": peak_kind,
                         "algorithmic_bytes_per_step": q_fused, "three_stage_bytes_per_step": q_three,
                         "t_roof_us": t_roof * 1e6, "t_roof_frac": t_roof / (ms * 1e-3),
                         "unit_of_launch": "one fused layer call (all its kernels)"},
            "e2e": {"value": e2e_value, "unit": "TFLOP/s", "h2d_bytes_per_step": int(x_np.nbytes),
                    "d2h_bytes_per_step": int(np.prod(spec.output_dims()) * 4), "ms_per_step": e2e_ms,
                    "api": f"HostPipeline({'split=' + args.e2e_split if args.e2e_split else 'chunks=' + str(args.e2e_chunks)}): "
                           "pinned host in/out, copies overlap compute"},
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
