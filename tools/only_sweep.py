"""Time the persistent kernel with only one item kind doing work (WF_ONLY) on c2.

    python tools/only_sweep.py [modes]   e.g. 0,4,1,5,6,2,3
"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf
from bench import layer_inputs
spec, t, x, w = layer_inputs("c2")
dev = torch.device("cuda", 0)
pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(t))
xd = torch.from_numpy(x).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
modes = sys.argv[1].split(",") if len(sys.argv) > 1 else ["4", "1", "2", "3"]
names = ["all", "F", "G", "I", "none", "F-nostore", "F-staging-only"]
for only in modes:
    os.environ["WF_ONLY"] = only
    plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=t, device=dev))
    ts = []
    for i in range(14):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); plan(xd); b.record(); b.synchronize()
        if i >= 2: ts.append(a.elapsed_time(b) * 1e3)
    print(f"only={only} ({names[int(only)]}): median {np.median(ts):7.1f} us", flush=True)
os.environ.pop("WF_ONLY")
