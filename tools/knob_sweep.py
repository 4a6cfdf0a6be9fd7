"""Time c2 through LayerPlan under a list of environment settings ("K=V,K=V;K=V...")."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf
from bench import layer_inputs
spec, t, x, w = layer_inputs(sys.argv[2] if len(sys.argv) > 2 else "c2")
dev = torch.device("cuda", 0)
pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(t))
xd = torch.from_numpy(x).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ref = None
for setting in sys.argv[1].split(";"):
    env = dict(kv.split("=") for kv in setting.split(",") if kv)
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=t, device=dev))
    ts = []
    for i in range(14):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); y = plan(xd); b.record(); b.synchronize()
        if i >= 2: ts.append(a.elapsed_time(b) * 1e3)
    yh = y.cpu().numpy()
    ref = yh if ref is None else ref
    print(f"{setting or 'default':40s}: median {np.median(ts):7.1f} us  min {min(ts):7.1f}  same={np.array_equal(yh, ref)}",
          flush=True)
    del plan
    for k, v in saved.items():
        if v is None: os.environ.pop(k, None)
        else: os.environ[k] = v
