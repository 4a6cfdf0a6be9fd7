"""Repeat-call check at the benchmark sizes: every layer of the BASELINE
configs, N fused calls on one plan, each bitwise equal to the three-stage
result (tools/stress_repeat.py does the same on small layers with ring reuse).

    python tools/stress_configs.py [calls] [configs]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_02165_b200 as wf  # noqa: E402
from bench import CONFIGS  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 100
configs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["c1", "c2", "c3", "c4", "c5"]
dev = torch.device("cuda", 0)
failed = 0
for cfg in configs:
    for ld in CONFIGS[cfg]:
        spec, x, w = ld.inputs()
        basis = wf.make_fft_basis(3) if ld.tile == 16 else wf.make_basis(ld.tile)
        pack = wf.transform_kernels(wf.Tensor4D(w), basis)
        xd = torch.from_numpy(x).to(dev)
        ref = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="three_stage", tile=ld.tile, transform=ld.transform,
                                                       device=dev))(xd).clone()
        plan = wf.LayerPlan(spec, pack, wf.EngineConfig(kind="fused", tile=ld.tile, transform=ld.transform, device=dev))
        out = torch.empty_like(ref)
        bad = 0
        for _ in range(calls):
            plan(xd, out=out)
            bad += int(not torch.equal(out, ref))
        failed += bad > 0
        print(f"{cfg} {ld.label()} B={spec.batch} ({plan.variant}): {calls} calls, {bad} differing", flush=True)
        del xd, ref, out, plan
        torch.cuda.empty_cache()
print("stress ok" if not failed else f"stress FAILED: {failed} layers")
sys.exit(1 if failed else 0)
