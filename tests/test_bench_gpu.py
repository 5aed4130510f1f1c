"""bench.py's multi-rank path (the one the driver's SCALE run uses) end to
end on one GPU: two ranks launched through torch.distributed.run, both on
cuda:0 with gloo collectives (LABS_BENCH_ONE_DEVICE=1). Checks the JSON
contract (n_gpus = 2, aggregate value, one line from rank 0), not speed."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


@pytest.mark.gpu
def test_bench_two_ranks_one_device():
    env = dict(os.environ, LABS_BENCH_ONE_DEVICE="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr", "127.0.0.1",
                        "--master-port", "29633", os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--quick", "--steps", "2", "--warmup", "1", "--epoch-ms", "20",
                        "--length", "40", "--replicas", "256"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["replicas_per_gpu"] == 256
    assert "rank 1/2" in r.stderr


@pytest.mark.gpu
def test_bench_refuses_missing_gpus():
    import torch
    n = torch.cuda.device_count() + 1
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n)],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 2 and "CUDA devices" in r.stderr
