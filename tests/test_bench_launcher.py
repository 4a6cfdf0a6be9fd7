"""bench.py's multi-GPU launcher on CPU: `--gpus N` without WORLD_SIZE
re-launches itself under torch.distributed.run with N ranks, each rank
checks WORLD_SIZE == N, works on its batch shard between barriers and rank
0 prints one line with n_gpus = N and the gathered output's checksum equal
to the single-rank run's (shards reassemble bitwise).  The compute is the
CPU oracle (--cpu-stub): the GPU path is the same protocol with the CUDA
engine."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(n):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--cpu-stub",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300, env=env,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_spawns_ranks_and_reassembles_shards():
    one = _run(1)
    two = _run(2)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2 and two["stub"]
    assert one["checksum"] == two["checksum"]
