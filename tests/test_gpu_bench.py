"""GPU: bench.py runs and prints a well-formed JSON line; the NCCL gather /
merge path runs (world size 1 with a process group, --dist)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    r = subprocess.run([sys.executable] + args, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_line_small():
    d = _run(["bench.py", "--steps", "3", "--warmup", "3", "--scale", "0.02", "--no-cpu-baseline"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "e2e", "roofline",
              "clocks", "gpu_launches", "config"):
        assert k in d
    assert d["value"] > 0 and d["roofline"]["bound"] == "alu" and d["gpu_launches"] > 0
    # HBM as the non-binding limit: algorithmic bytes always, the committed ncu
    # traffic only for the default full-size workload (not this scaled one)
    hbm = d["roofline"]["hbm"]
    assert hbm["algorithmic_bytes"] > 0 and hbm["algorithmic_GBps"] > 0 and hbm["traffic_GBps"] is None


def test_bench_nccl_gather_path_world1():
    d = _run(["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr", "127.0.0.1",
              "--master-port", "29533", "bench.py", "--dist", "--steps", "3", "--warmup", "3", "--scale", "0.02",
              "--no-cpu-baseline"])
    assert d["value"] > 0 and d["n_gpus"] == 1
