"""Run a few c2 layer steps (fused + three-stage) for ncu launch lists / captures."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf
from bench import layer_inputs

engine = sys.argv[1] if len(sys.argv) > 1 else "fused"
cfgname = sys.argv[2] if len(sys.argv) > 2 else "c2"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
spec, t, x, w = layer_inputs(cfgname)
dev = torch.device("cuda", 0)
pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(t))
xd = torch.from_numpy(x).to(dev)
cfg = wf.EngineConfig(kind=engine, tile=t)
for _ in range(steps):
    y, st = wf.run_engine(engine, xd, pack, spec, cfg)
torch.cuda.synchronize()
print(engine, cfgname, "last step us", st.wall_s * 1e6)
