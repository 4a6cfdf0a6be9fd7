"""End-to-end (pinned host buffers) time of the c2 layer through HostPipeline:
one call at a time (graph replay / plain streams) and streaming submit() with
double-buffered staging, per slice count.

    python tools/e2e_probe.py [config] [--reps N]
"""
import argparse
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_02165_b200 as wf  # noqa: E402
from bench import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c2")
ap.add_argument("--reps", type=int, default=30)
a = ap.parse_args()
ld = CONFIGS[a.config][0]
spec, x, w = ld.inputs()
dev = torch.device("cuda", 0)
pack = wf.transform_kernels(wf.Tensor4D(w), wf.make_basis(ld.tile))
cfg = wf.EngineConfig(kind="fused", tile=ld.tile, device=dev)
x_host = torch.from_numpy(x).pin_memory()
y_hosts = [torch.empty(spec.output_dims(), dtype=torch.float32, pin_memory=True) for _ in range(3)]
ref = None


def sync_mode(chunks, graph):
    pipe = wf.HostPipeline(spec, pack, cfg, chunks=chunks, graph=graph)
    for _ in range(3):
        pipe(x_host, y_hosts[0])
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        pipe(x_host, y_hosts[0])
        ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts), min(ts)


def stream_mode(chunks, depth):
    pipe = wf.HostPipeline(spec, pack, cfg, chunks=chunks, graph=False, depth=depth)
    for i in range(4):
        pipe.submit(x_host, y_hosts[i % depth])
    pipe.wait()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        for i in range(a.reps):
            pipe.submit(x_host, y_hosts[i % depth])
        pipe.wait()
        ts.append((time.perf_counter() - t0) * 1e3 / a.reps)
    return statistics.median(ts), min(ts)


for chunks in (2, 4, 8):
    for graph in (True, False):
        med, mn = sync_mode(chunks, graph)
        print(f"sync   chunks={chunks} graph={graph}: median {med:.3f} ms min {mn:.3f} ms", flush=True)
one = y_hosts[0].clone()
for depth in (2, 3):
    for chunks in (1, 2, 4, 8):
        med, mn = stream_mode(chunks, depth)
        ok = all(torch.equal(y_hosts[k], one) for k in range(depth))
        print(f"stream chunks={chunks} depth={depth}: median {med:.3f} ms/call min {mn:.3f}; bitwise equal {ok}", flush=True)
