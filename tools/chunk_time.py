import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf
dev = torch.device("cuda", 0)
for b in (8, 16, 32, 64):
    spec = wf.LayerSpec(b, 64, 64, 56, 56, 3, 1, 1)
    w = (np.random.default_rng(0).standard_normal(spec.kernel_dims()) * 0.06).astype(np.float32)
    pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(6))
    plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=6, device=dev))
    x = torch.randn(spec.input_dims(), device=dev)
    for _ in range(3): plan(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): plan(x)
    e1.record(); torch.cuda.synchronize()
    print(b, f"{e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
