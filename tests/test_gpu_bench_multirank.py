"""bench.py's N > 1 path (torchrun, one pipeline per rank over its own shard
dataset, barrier + max-over-ranks timing, summed clouds, rank 0 prints one
line), run as 2 ranks on the one GPU of the test box with gloo collectives
(PCP_BENCH_SHARED_GPU): the plumbing, not a measurement."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("impl", ["ours", "reference"])
def test_two_rank_bench_line(impl):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--config", "shapenet_part",
           "--clouds-per-gpu", "256", "--no-cpu-baseline"]
    if impl == "reference":
        cmd += ["--impl", "reference"]
    env = dict(os.environ, PCP_BENCH_SHARED_GPU="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    d = json.loads(lines[0])
    assert d["value"] > 0
    if impl == "reference":
        assert d["impl"] == "reference"
        return
    assert d["n_gpus"] == 2 and d["steps"] == 2
    assert "record-sharded" in d["config"]["parallelism"]
    # both ranks' clouds are counted: 2 x 256 clouds per step
    assert abs(d["value"] * d["ms_per_step"] / 1e3 - 2 * 256) < 1e-6 * 512 + 1
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
