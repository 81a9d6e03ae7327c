"""bench.py's N > 1 launch on a GPU box: a plain `python bench.py --gpus 2` (no torchrun
environment) re-launches itself with two ranks -- NCCL when two GPUs are visible, gloo with
the ranks sharing the GPU otherwise -- and prints one line for the whole job."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus_2_self_launch():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "cfg0",
                          "--steps", "2", "--warmup", "3", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and len(rec["per_rank"]) == 2, rec
    assert rec["value"] > 0 and rec["e2e"]["value"] > 0
    assert rec["gpu_launches"] > 0
