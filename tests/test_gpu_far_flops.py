"""Executed FP64 work per far-field pair, counted by ncu on a B200: k_far_pairs (one pair per
thread, no idle lanes) must execute bench.far_executed_flops(P) - 3 flops per pair
(2 DFMA + DMUL + DADD thread-instructions; the pair kernel receives dx, so the three dx
subtractions of the event loops are absent).  This pins the far roofline's flop count."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not shutil.which("ncu"), reason="ncu not installed")]

SNIPPET = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1811_12498_b200 as S
p, n = int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(1)
dx = rng.uniform(-1, 1, (n, 3)) + np.array([3.0, 0, 0])
E = (p + 1) * (p + 2) * (p + 3) // 6
S.farfield_pairs(dx, p, stok=rng.uniform(-1, 1, (n, E, 3)), strm=rng.uniform(-1, 1, (n, E, 9)))
"""


@pytest.mark.parametrize("p", [4, 8, 10])
def test_far_pair_executed_flops(p, tmp_path):
    sys.path.insert(0, ROOT)
    import bench
    n = 2048
    metrics = ",".join(f"smsp__sass_thread_inst_executed_op_{k}_pred_on.sum" for k in ("dfma", "dmul", "dadd"))
    log = tmp_path / "ncu.csv"
    out = subprocess.run(["ncu", "--metrics", metrics, "-k", "regex:k_far_pairs", "--csv", "--log-file", str(log),
                          sys.executable, "-c", SNIPPET, ROOT, str(p), str(n)],
                         capture_output=True, text=True, timeout=600)
    if out.returncode != 0 or not log.exists():
        pytest.skip("ncu could not profile here: " + (out.stderr or out.stdout)[-300:])
    import csv
    rows = list(csv.reader(log.read_text().splitlines()))
    h = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    ni, vi = rows[h].index("Metric Name"), rows[h].index("Metric Value")
    vals = {}
    for r in rows[h + 1:]:
        for k in ("dfma", "dmul", "dadd"):
            if len(r) > vi and f"op_{k}_pred_on" in r[ni]:
                vals[k] = vals.get(k, 0.0) + float(r[vi].replace(",", ""))
    assert set(vals) == {"dfma", "dmul", "dadd"}, log.read_text()[-2000:]
    per_pair = (2 * vals["dfma"] + vals["dmul"] + vals["dadd"]) / n
    assert per_pair == bench.far_executed_flops(p + 2) - 3, (p, per_pair, vals)
