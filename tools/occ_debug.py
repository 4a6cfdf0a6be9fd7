import numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf
spec = wf.LayerSpec(2, 64, 64, 20, 20, 3, 1, 1)
x = wf.new_tensor(spec.input_dims(), seed=1)
pack = wf.transform_kernels(wf.new_tensor(spec.kernel_dims(), seed=2), wf.make_basis(6))
y, st = wf.conv_fused(x, pack, spec, wf.EngineConfig(tile=6, fused_variant="itemq"))
print("ran", st.variant)
