"""Two persistent fused layers launched concurrently on two streams (the
co-residency hazard of spin-waiting persistent kernels): with cooperative
launches the driver schedules each grid whole, so neither can deadlock.
Run under `timeout`; prints the outputs' agreement with a serial run."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf

dev = torch.device("cuda", 0)
spec = wf.LayerSpec(16, 64, 64, 56, 56, 3, 1, 1)
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.standard_normal(spec.input_dims()).astype(np.float32)).to(dev)
w = (rng.standard_normal(spec.kernel_dims()) * np.sqrt(2.0 / 576)).astype(np.float32)
pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(6))
plans = {v: [wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=6, device=dev, fused_variant=v))
             for _ in range(2)] for v in ("ws", "itemq")}
ref = plans["ws"][0](x).clone()
streams = [torch.cuda.Stream(dev) for _ in range(2)]
for v, (pa, pb) in plans.items():
    for it in range(50):
        with torch.cuda.stream(streams[0]):
            ya = pa(x)
        with torch.cuda.stream(streams[1]):
            yb = pb(x)
    torch.cuda.synchronize()
    print(v, "concurrent x50 ok; bitwise", torch.equal(ya, ref), torch.equal(yb, ref), "ran", pa.ran.value, pb.ran.value,
          flush=True)
