"""Batch sharding host logic, including a real world_size=2 gloo run on CPU.

The per-rank compute here is the CPU oracle (the GPU path is the same
host logic with the CUDA engine as ``compute``; its bitwise shard property
is checked on the B200 in test_gpu_parity.py).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_1912_02165_b200 as wf
from paper_1912_02165_b200.sharding import run_sharded, shard_range, shard_spec


def test_shard_ranges_cover_batch_exactly():
    for batch in (1, 2, 7, 64, 256):
        for world in (1, 2, 4, 8):
            ranges = [shard_range(batch, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == batch
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [h - l for l, h in ranges]
            assert max(sizes) - min(sizes) <= 1
    assert shard_spec(wf.LayerSpec(1, 2, 2, 5, 5), 1, 2) is None
    with pytest.raises(wf.InvalidParameterError):
        shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, x, w, tile, q):
    import torch.distributed as dist
    from oracle import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = wf.LayerSpec(x.shape[0], x.shape[1], w.shape[0], x.shape[2], x.shape[3], 3, 1, 1)
    pack = O.transform_kernels(w, tile)
    full = run_sharded(x, spec, rank, world,
                       lambda xs, s: O.conv_fused(np.ascontiguousarray(xs), pack, s, tile, 24),
                       gather=dist.group.WORLD)
    q.put((rank, full.numpy()))
    dist.destroy_process_group()


def test_two_rank_gloo_sharding_is_bitwise():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((5, 6, 12, 10)).astype(np.float32)
    w = (rng.standard_normal((7, 6, 3, 3)) * 0.2).astype(np.float32)
    tile = 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, x, w, tile, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=60) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import oracle as O
    spec = wf.LayerSpec(5, 6, 7, 12, 10, 3, 1, 1)
    single = O.conv_fused(x, O.transform_kernels(w, tile), spec, tile, 24)
    for r in range(2):
        assert np.array_equal(results[r], single)
