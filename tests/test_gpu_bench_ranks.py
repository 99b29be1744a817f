"""bench.py under torchrun with 2 ranks sharing the one GPU (WL_BENCH_DEVICE=0,
gloo for the timing barrier): the multi-rank paths of the benchmark --
row-strip pyramid (configs[3]) with its cross-process halo exchange, batch
sharding (configs[4]) -- run, print one line from rank 0, and the strip
pyramid's checksum equals the single-rank run's (same deterministic image)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--size", "1024", "--steps", "2", "--warmup", "3", "--no-c3", "--e2e-steps", "0",
        "--no-cpu", "--no-unaligned", "--c4-size", "4096", "--c5-images", "16", "--c5-pool", "8"]


def _run(nproc):
    env = dict(os.environ, WL_BENCH_DEVICE="0", WL_BENCH_BACKEND="gloo")
    if nproc == 1:
        cmd = [sys.executable, "bench.py", *ARGS]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1", "--master-port",
               "29561", "bench.py", "--gpus", str(nproc), *ARGS]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_two_ranks_one_gpu():
    one, two = _run(1), _run(2)
    assert two["n_gpus"] == 2 and two["c4"]["ranks"] == 2 and one["c4"]["ranks"] == 1
    assert two["value"] > 0 and two["c5"]["value"] > 0
    a, b = one["c4"]["checksum"], two["c4"]["checksum"]
    assert abs(a - b) <= 1e-9 * max(abs(a), 1.0), (a, b)
