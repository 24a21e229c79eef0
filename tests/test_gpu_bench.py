"""bench.py keeps the driver's contract: one JSON line with the required keys, at N=1 and (2 ranks
sharing one GPU over gloo, the validation mode) at N=2."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks",
        "gpu_launches"}


def _last_json(out):
    return json.loads(out.strip().splitlines()[-1])


def test_bench_n1_small():
    r = subprocess.run([sys.executable, "bench.py", "--config", "small", "--steps", "2",
                        "--warmup", "3", "--no-cpu"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d) and d["n_gpus"] == 1 and d["value"] > 0
    assert d["roofline"]["bound"] == "tensor" and 0 < d["roofline"]["frac"] < 1
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and d["backward"]["value"] > 0


def test_bench_two_ranks_same_gpu():
    env = dict(os.environ, CQS_SAME_DEVICE="1", CQS_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        "29533", "bench.py", "--gpus", "2", "--config", "small", "--steps", "2",
                        "--warmup", "3", "--no-cpu"], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d) and d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["parallelism"] == "task-sharded x2"
    assert d["e2e"]["value"] > 0 and d["backward"]["value"] > 0
