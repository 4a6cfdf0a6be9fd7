"""Time the FFT-16 engines on BASELINE config c4 shapes (B=128) via LayerPlan."""
import sys
import numpy as np
import torch
import paper_1912_02165_b200 as wf

dev = torch.device("cuda:0")
B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
for c, hw in [(64, 56), (128, 28), (256, 14), (512, 7)]:
    spec = wf.LayerSpec(B, c, c, hw, hw, 3, 1, 1)
    rng = np.random.default_rng(0)
    w = (rng.standard_normal(spec.kernel_dims()) * np.sqrt(2 / (9 * c))).astype(np.float32)
    x = torch.randn(spec.input_dims(), device=dev)
    pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_fft_basis())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    res = []
    for kind in ("fused", "three_stage"):
        plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind=kind, transform="fft", tile=16, device=dev))
        for _ in range(3):
            plan(x)
        ts = []
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); plan(x); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        res.append(f"{kind} {np.median(ts):8.1f}us")
    direct_tf = spec.direct_flops() / (np.median(ts) * 1e-6) / 1e12
    print(f"c4 C={c} HW={hw} B={B}: " + "  ".join(res), flush=True)
