"""Run one layer a few times through LayerPlan (for ncu launch lists).

    python tools/one_layer.py B C Cp HW tile transform kind [reps]
"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf
b, c, cp, hw, t = (int(v) for v in sys.argv[1:6])
transform, kind = sys.argv[6], sys.argv[7]
reps = int(sys.argv[8]) if len(sys.argv) > 8 else 3
dev = torch.device("cuda", 0)
spec = wf.LayerSpec(b, c, cp, hw, hw, 3, 1, 1)
w = (np.random.default_rng(0).standard_normal(spec.kernel_dims()) * np.sqrt(2 / (9 * c))).astype(np.float32)
basis = wf.make_fft_basis() if transform == "fft" else wf.make_basis(t)
pack = wf.transform_kernels(wf.Tensor4D(w), basis)
plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind=kind, tile=t, transform=transform, device=dev))
x = torch.randn(spec.input_dims(), device=dev)
for _ in range(reps):
    plan(x)
torch.cuda.synchronize()
print("ok")
