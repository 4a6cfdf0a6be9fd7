"""Time one layer of a bench config (CUDA events, L2 flushed before every call).

    python tools/layer_time.py c2 [layer-index] [--engine fused|three_stage]
        [--variant auto|ws|itemq|waves] [--ring-mb N] [--reps N]

Prints the median / min time, the variant that ran and the roofline fraction.
Short enough to run under ncu (--reps 3).
"""
import argparse
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_02165_b200 as wf  # noqa: E402
from bench import CONFIGS, roofline_terms  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("layer", type=int, nargs="?", default=0)
ap.add_argument("--engine", default="fused")
ap.add_argument("--variant", default="auto")
ap.add_argument("--ring-mb", type=int, default=0)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--batch", type=int, default=0)
a = ap.parse_args()

ld = CONFIGS[a.config][a.layer]
spec, x, w = ld.inputs(batch=a.batch or None)
dev = torch.device("cuda", 0)
basis = wf.make_fft_basis(3) if ld.tile == 16 else wf.make_basis(ld.tile)
pack = wf.transform_kernels(wf.Tensor4D(w), basis)
cfg = wf.EngineConfig(kind=a.engine, tile=ld.tile, transform=ld.transform, device=dev, fused_variant=a.variant,
                      ring_bytes=(a.ring_mb << 20) or None)
plan = wf.LayerPlan(spec, pack, cfg)
xd = torch.from_numpy(x).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ts = []
for i in range(a.reps + 2):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan(xd)
    e1.record()
    e1.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1) * 1e3)
rt = roofline_terms(spec, ld.tile)
med = statistics.median(ts)
print(f"{ld.label()} B={spec.batch} {a.engine} variant={wf._lib.VARIANT_NAMES.get(plan.ran.value, '-')}: "
      f"median {med:.1f} us min {min(ts):.1f} us; roof {rt['t_roof'] * 1e6:.1f} us ({rt['bound']}) -> "
      f"frac {rt['t_roof'] * 1e6 / med:.3f}", flush=True)
