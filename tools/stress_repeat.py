"""Repeat-call stress of the persistent fused kernels: N calls per layer on the
same plan, every result bitwise equal to the three-stage one (a lost
dependency or a ring slot reused too early shows up as a differing call).

    python tools/stress_repeat.py [calls]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_02165_b200 as wf  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 200
dev = torch.device("cuda", 0)
cases = [
    ((24, 64, 64, 56, 56, 3, 1, 1), 6, "ws", None),
    ((24, 64, 64, 56, 56, 3, 1, 1), 6, "ws", 12),          # small rings: slot reuse
    ((24, 64, 64, 56, 56, 3, 1, 1), 6, "ws_row", None),
    ((24, 64, 64, 56, 56, 3, 1, 1), 6, "ws_row", 12),
    ((8, 3, 64, 112, 112, 3, 1, 1), 6, "ws", None),
    ((8, 64, 128, 56, 56, 3, 1, 1), 6, "ws", None),       # two positions per G unit
    ((8, 64, 128, 56, 56, 3, 1, 1), 6, "ws", 16),
    ((8, 128, 256, 56, 56, 3, 1, 1), 6, "ws", None),
    ((8, 256, 256, 28, 28, 3, 1, 1), 6, "ws", None),
    ((64, 16, 16, 56, 56, 3, 1, 1), 8, "ws", None),        # batched G publishes
    ((32, 64, 64, 56, 56, 3, 1, 1), 8, "ws", None),
    ((16, 128, 128, 28, 28, 3, 1, 1), 8, "ws", 40),
    ((24, 48, 80, 56, 56, 3, 1, 1), 6, "itemq", None),
    ((8, 96, 96, 56, 56, 3, 1, 1), 8, "itemq", None),
    ((16, 512, 512, 28, 28, 3, 1, 1), 6, "waves", None),   # three wave lanes, CTA-pair GEMM
    ((16, 256, 512, 28, 28, 3, 1, 1), 6, "waves", None),
    ((32, 512, 512, 14, 14, 3, 1, 1), 6, "waves", None),
    ((32, 64, 64, 56, 56, 3, 1, 1), 16, "waves", None),    # FFT-16
    ((32, 256, 256, 14, 14, 3, 1, 1), 16, "waves", None),
]
failed = 0
for dims, t, variant, ring_mb in cases:
    spec = wf.LayerSpec(*dims)
    rng = np.random.default_rng(5)
    x = torch.from_numpy(rng.standard_normal(spec.input_dims()).astype(np.float32)).to(dev)
    w = (rng.standard_normal(spec.kernel_dims()) * np.sqrt(2.0 / (9 * dims[1]))).astype(np.float32)
    tf = "fft" if t == 16 else "winograd"
    pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_fft_basis() if t == 16 else wf.make_basis(t))
    ref = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="three_stage", tile=t, device=dev, transform=tf))(x).clone()
    plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=t, device=dev, fused_variant=variant, transform=tf,
                                                    ring_bytes=(ring_mb << 20) if ring_mb else None))
    bad = 0
    out = torch.empty_like(ref)
    for i in range(calls):
        plan(x, out=out)
        if not torch.equal(out, ref):
            bad += 1
    torch.cuda.synchronize()
    print(f"{dims} T={t} {variant} ring={ring_mb}: {calls} calls, {bad} differing (variant ran: {plan.variant})", flush=True)
    failed = failed + (bad > 0)
print("stress ok" if not failed else f"stress FAILED: {failed} cases")
sys.exit(1 if failed else 0)
