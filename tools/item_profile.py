"""Per-item-kind wait/run cycles of the persistent fused kernel (WF_PROFILE=1)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
os.environ["WF_PROFILE"] = "1"
import paper_1912_02165_b200 as wf
from paper_1912_02165_b200 import _lib
from bench import layer_inputs
spec, t, x, w = layer_inputs(sys.argv[1] if len(sys.argv) > 1 else "c2")
dev = torch.device("cuda", 0)
pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(t))
plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=t, device=dev))
xd = torch.from_numpy(x).to(dev)
lib = _lib.load()
N = 512 * 16
buf = (ctypes.c_ulonglong * N)()
clk = 1.9e3
for it in range(3):
    lib.wf_debug_fused_profile(buf, N)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); plan(xd); e1.record(); torch.cuda.synchronize()
    lib.wf_debug_fused_profile(buf, N)
    a = np.array(buf[:], dtype=np.float64).reshape(512, 16)
    ctas = int((a[:, 2] + a[:, 5] + a[:, 8] > 0).sum())
    print(f"step {it}: {e0.elapsed_time(e1)*1e3:.1f} us, {ctas} CTAs")
    for k, name in enumerate("FGI"):
        n = a[:, 3 * k + 2].sum()
        print(f"   {name}: items {n:5.0f}  avg wait {a[:, 3*k].sum()/max(n,1)/clk:6.2f} us  avg run "
              f"{a[:, 3*k+1].sum()/max(n,1)/clk:6.2f} us   per CTA run {a[:, 3*k+1].sum()/ctas/clk:6.1f} "
              f"wait {a[:, 3*k].sum()/ctas/clk:6.1f} us")
    nf, ni = a[:, 2].sum(), a[:, 8].sum()
    print(f"   F phases per item: staging {a[:, 9].sum()/max(nf,1)/clk:.2f} us, transform+store {a[:, 10].sum()/max(nf,1)/clk:.2f} us")
    nall = a[:, 2].sum() + a[:, 5].sum() + a[:, 8].sum()
    print(f"   per item: completion publish (fence+atomic) {a[:, 14].sum()/max(nall,1)/clk:.2f} us, "
          f"dispatch (loop top to start) {a[:, 15].sum()/max(nall,1)/clk:.2f} us, thread-0 decode {a[:, 13].sum()/max(nall,1)/clk:.2f} us")
