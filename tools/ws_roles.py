"""Per-role time accounting of the warp-specialised fused kernel (instrumented
launch): average per CTA, in microseconds of SM clock.

    python tools/ws_roles.py [config] [layer]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_02165_b200 as wf  # noqa: E402
from paper_1912_02165_b200 import _lib  # noqa: E402
from bench import CONFIGS  # noqa: E402

SLOTS = ["GP dep wait", "GP stage wait", "GI A-full wait", "GI TMEM-empty wait", "GE TMEM-full wait", "GE busy",
         "FP dep wait", "FP slot wait", "FW data wait", "FW F units", "FW I units", "publish fences",
         "start", "end GP", "end GI", "end GE", "end FP", "end FW", "end Pub", "n F", "n I", "FW loop",
         "FP busy F", "FP busy I", "FP tx", "FP copy"]
cfg, layer = (sys.argv[1], int(sys.argv[2])) if len(sys.argv) > 2 else ("c2", 0)
ld = CONFIGS[cfg][layer]
spec, x, w = ld.inputs()
pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(ld.tile))
xd = torch.from_numpy(x).cuda()
c = wf.EngineConfig(tile=ld.tile, instrumented=True)
wf.conv_fused(xd, pack, spec, c)
y, st = wf.conv_fused(xd, pack, spec, c)
lib = _lib.load()
buf = (ctypes.c_ulonglong * (1024 * 32))()
lib.wf_debug_ws_profile(buf, 1024 * 32)
a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 32)[:148].astype(np.float64)
khz = torch.cuda.get_device_properties(0).clock_rate if hasattr(torch.cuda.get_device_properties(0), "clock_rate") \
    else 1965000
ghz = 1.965
print(f"{ld.label()}: wall {st.wall_s * 1e6:.1f} us, violations {st.overlap_violations}, phase_s "
      + ", ".join(f"{k} {v * 1e6:.0f} us" for k, v in st.phase_s.items()))
t0 = a[:, 12]
for i, name in enumerate(SLOTS):
    if name.startswith("end"):
        print(f"{name:22s} {np.mean(a[:, i] - t0) / 1e3:9.1f} us after start (max {np.max(a[:, i] - t0) / 1e3:.1f})")
    elif name.startswith("n ") or name == "start":
        if name != "start":
            print(f"{name:22s} {np.mean(a[:, i]):9.1f} per CTA")
    else:
        print(f"{name:22s} {np.mean(a[:, i]) / ghz / 1e3:9.1f} us per CTA (max {np.max(a[:, i]) / ghz / 1e3:.1f})")
