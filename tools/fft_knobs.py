"""c4 (FFT-16, B=128) layers under a list of environment settings ("K=V,K=V;...")."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for c, hw in [(64, 56), (128, 28), (256, 14), (512, 7)]:
    spec = wf.LayerSpec(128, c, c, hw, hw, 3, 1, 1)
    rng = np.random.default_rng(0)
    w = (rng.standard_normal(spec.kernel_dims()) * np.sqrt(2 / (9 * c))).astype(np.float32)
    pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_fft_basis())
    x = torch.randn(spec.input_dims(), device=dev)
    for setting in sys.argv[1].split(";"):
        env = dict(kv.split("=") for kv in setting.split(",") if kv)
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=16, transform="fft", device=dev))
        ts = []
        for i in range(12):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); plan(x); b.record(); b.synchronize()
            if i >= 2: ts.append(a.elapsed_time(b) * 1e3)
        print(f"{c}@{hw} {setting or 'default':36s}: median {np.median(ts):7.1f} us", flush=True)
        del plan
        for k, v in saved.items():
            if v is None: os.environ.pop(k, None)
            else: os.environ[k] = v
