"""Per-role accounting of the warp-specialised fused kernel (WF_WS_PROF=1) on c2.

    python tools/ws_prof.py [config] [env=val ...]
"""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
os.environ["WF_WS_PROF"] = "1"
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    os.environ[k] = v
import paper_1912_02165_b200 as wf
from paper_1912_02165_b200 import _lib
from bench import layer_inputs
spec, t, x, w = layer_inputs(sys.argv[1] if len(sys.argv) > 1 else "c2")
dev = torch.device("cuda", 0)
pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(t))
plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=t, device=dev))
xd = torch.from_numpy(x).to(dev)
lib = _lib.load()
N = 1024 * 32
buf = (ctypes.c_ulonglong * N)()
lib.wf_debug_ws_profile.argtypes = [ctypes.c_void_p, ctypes.c_int]
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
names = ["G-prod dep wait", "G-prod stage wait", "G-issue full wait", "G-issue tempty wait", "G-epi tfull wait",
         "G-epi busy", "FI-prod dep wait", "FI-prod slot wait", "FI-work full wait", "FI-work F busy",
         "FI-work I busy", "publish fence"]
extra = {21: "FI-work loop total", 22: "FI-prod busy F (issue)", 23: "FI-prod busy I (issue)", 24: "FI-prod I: expect_tx", 25: "FI-prod I: copy issue"}
clk = 1.9e3
for it in range(3):
    flush.zero_()
    torch.cuda.synchronize()
    lib.wf_debug_ws_profile(buf, N)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); plan(xd); e1.record(); torch.cuda.synchronize()
    lib.wf_debug_ws_profile(buf, N)
    a = np.array(buf[:], dtype=np.float64).reshape(1024, 32)
    ctas = int((a[:, 12] > 0).sum())
    a = a[:ctas]
    print(f"step {it}: {e0.elapsed_time(e1)*1e3:.1f} us, {ctas} CTAs, F units/CTA {a[:, 19].mean():.1f}, I {a[:, 20].mean():.1f}")
    for k, nm in enumerate(names):
        print(f"   {nm:22s} avg {a[:, k].mean()/clk:7.2f} us  max {a[:, k].max()/clk:7.2f}")
    for k, nm in extra.items():
        print(f"   {nm:22s} avg {a[:, k].mean()/clk:7.2f} us  max {a[:, k].max()/clk:7.2f}")
    st = a[:, 12].min()
    for k, nm in zip(range(13, 19), ["G-prod", "G-issue", "G-epi", "FI-prod", "FI-work", "publisher"]):
        e = (a[:, k] - st) / 1e3
        print(f"   end {nm:10s} min {e.min():7.1f} med {np.median(e):7.1f} max {e.max():7.1f} us")

# per-block event trace of the last step (ns): F start/end, G start/end, I start/end
tr = (ctypes.c_ulonglong * (4096 * 8))()
lib.wf_debug_ws_trace.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
lib.wf_debug_ws_trace(tr, 4096, 1)
flush.zero_(); torch.cuda.synchronize()
plan(xd); torch.cuda.synchronize()
lib.wf_debug_ws_trace(tr, 4096, 1)
nb = -(-(spec.batch * -(-spec.out_height // (t - 2)) * -(-spec.out_width // (t - 2))) // 128)
a = np.array(tr[:nb * 8], dtype=np.float64).reshape(nb, 8)
t0 = a[:, 0].min()
a = (a - t0) / 1e3
print("block  Fstart  Fend  Gstart  Gend  Istart  Iend   (us)   G-F  I-G")
for b in list(range(0, nb, max(1, nb // 16))) + [nb - 1]:
    r = a[b]
    print(f"{b:5d} {r[0]:7.1f} {r[1]:6.1f} {r[2]:6.1f} {r[3]:6.1f} {r[4]:7.1f} {r[5]:6.1f}   {r[3]-r[1]:5.1f} {r[4]-r[3]:5.1f}")
print(f"median Gend-Fend {np.median(a[:,3]-a[:,1]):.1f} us, Gstart-Fend {np.median(a[:,2]-a[:,1]):.1f}, Istart-Gend {np.median(a[:,4]-a[:,3]):.1f}, Fend-Fstart {np.median(a[:,1]-a[:,0]):.1f}, Iend-Istart {np.median(a[:,5]-a[:,4]):.1f}")
