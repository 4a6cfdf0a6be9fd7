"""Per-layer measurements of every BASELINE config on one B200.

For each layer: fused and three-stage time (median of N CUDA-event-timed
calls through LayerPlan, L2 flushed before each), direct-equivalent TFLOP/s,
images/s and the roofline fraction t_roof / t with
t_roof = max(Q_fused / BW_HBM, passes * F_gemm / P_bf16) (MEASURED_PEAKS.json).

    python tools/bench_all.py [--reps N] [--configs c1,c2,c3,c4,c5] > profiles/rNN_all_configs.md
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1912_02165_b200 as wf  # noqa: E402

VGG = [(3, 64, 224), (64, 64, 224), (64, 128, 112), (128, 128, 112), (128, 256, 56), (256, 256, 56),
       (256, 256, 56), (256, 512, 28), (512, 512, 28), (512, 512, 28), (512, 512, 14), (512, 512, 14),
       (512, 512, 14)]


def layers(names):
    out = []
    if "c1" in names:
        out.append(("c1", "F(2,3) 64->64 @56", 1, 64, 64, 56, "winograd", 4, "inv_sqrt", "normal"))
    if "c2" in names:
        out.append(("c2", "F(4,3) 64->64 @56", 64, 64, 64, 56, "winograd", 6, "he", "normal"))
    if "c3" in names:
        for i, (c, cp, hw) in enumerate(VGG):
            out.append(("c3", f"VGG L{i + 1} {c}->{cp} @{hw}", 32, c, cp, hw, "winograd", 6, "he", "normal"))
    if "c4" in names:
        for c, hw in [(64, 56), (128, 28), (256, 14), (512, 7)]:
            out.append(("c4", f"FFT-16 {c}->{c} @{hw}", 128, c, c, hw, "fft", 16, "he", "normal"))
    if "c5" in names:
        for c in (16, 32, 64, 128):
            for hw in (28, 56, 112):
                out.append(("c5", f"F(6,3) {c}->{c} @{hw}", 256, c, c, hw, "winograd", 8, "he", "uniform"))
    return out


def roof(spec, transform, t, peaks):
    if transform == "fft":
        m, pos, pack = 14, 144, 8 * 144 * spec.in_channels * spec.out_channels
        f_gemm = 8 * 144 * spec.in_channels * spec.out_channels
    else:
        m, pos, pack = t - 2, t * t, 4 * t * t * spec.in_channels * spec.out_channels
        f_gemm = 2 * spec.in_channels * spec.out_channels * t * t
    n_tile = spec.batch * -(-spec.out_height // m) * -(-spec.out_width // m)
    f_gemm *= n_tile
    q = 4 * (spec.batch * spec.in_channels * spec.height * spec.width
             + spec.batch * spec.out_channels * spec.out_height * spec.out_width) + pack
    return max(q / (peaks["hbm_gbs"] * 1e9), 3 * f_gemm / (peaks["bf16_tflops"] * 1e12)), q


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    rows = []
    print("| config | layer | B | engine | ms | direct-eq TFLOP/s | images/s | t_roof us | roofline frac |")
    print("|---|---|---|---|---|---|---|---|---|")
    for cfg, name, b, c, cp, hw, transform, t, wrule, xdist in layers(args.configs.split(",")):
        spec = wf.LayerSpec(b, c, cp, hw, hw, 3, 1, 1)
        rng = np.random.default_rng(1234)
        std = np.sqrt(2.0 / (9 * c)) if wrule == "he" else 1.0 / np.sqrt(9 * c)
        w = (rng.standard_normal(spec.kernel_dims()) * std).astype(np.float32)
        if xdist == "uniform":
            x = torch.rand(spec.input_dims(), device=dev) * 2 - 1
        else:
            x = torch.randn(spec.input_dims(), device=dev)
        basis = wf.make_fft_basis() if transform == "fft" else wf.make_basis(t)
        pack = wf.transform_kernels(wf.Tensor4D(w), basis)
        t_roof, q = roof(spec, transform, t, peaks)
        for kind in ("fused", "three_stage"):
            try:
                plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind=kind, tile=t, transform=transform, device=dev))
            except Exception as exc:  # e.g. three-stage intermediates beyond HBM
                print(f"| {cfg} | {name} | {b} | {kind} | n/a ({type(exc).__name__}) | | | | |", flush=True)
                continue
            for _ in range(3):
                plan(x)
            ts = []
            for _ in range(args.reps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                plan(x)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e-3)
            sec = float(np.median(ts))
            tf = spec.direct_flops() / sec / 1e12
            row = dict(config=cfg, layer=name, batch=b, engine=kind, ms=sec * 1e3, tflops=tf, images_s=b / sec,
                       t_roof_us=t_roof * 1e6, frac=t_roof / sec, q_fused=q)
            rows.append(row)
            print(f"| {cfg} | {name} | {b} | {kind} | {sec * 1e3:.3f} | {tf:.1f} | {b / sec:.0f} | "
                  f"{t_roof * 1e6:.1f} | {t_roof / sec:.3f} |", flush=True)
            del plan
            torch.cuda.empty_cache()
    if args.json:
        with open(args.json, "w") as fh:
            for r in rows:
                fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
