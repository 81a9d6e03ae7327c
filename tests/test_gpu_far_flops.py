"""Executed FP64 work per far-field pair, counted by ncu on a B200, pins bench.py's far
roofline flop count (bench.far_executed_flops).  The case makes every event dense and
shared: 6,400 targets far from a compact source cloud each accept the root cluster only,
so k_far_list evaluates exactly one pair per target with every lane of both batches busy;
its 2 DFMA + DMUL + DADD thread-instructions divided by the far-field evaluations must
equal the formula.  k_far_list's epilogue also performs the combine (k_nreduce's sums,
fused): 3 DADD per target for far + near, which this case (no near entries, no deferred
events) executes once per target and which is subtracted."""
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
p = int(sys.argv[2])
rng = np.random.default_rng(1)
n = 5000
nu = rng.normal(size=(n, 3))
nu /= np.linalg.norm(nu, axis=1, keepdims=True)
ps = S.ParticleSet(rng.uniform(0, 0.01, (n, 3)), rng.uniform(-1, 1, (n, 3)), rng.uniform(-1, 1, (n, 3)), nu)
tg = rng.uniform(-1, 1, (6400, 3)) + np.array([10.0, 0, 0])
r = S.treecode_velocity_targets(ps, tg, S.TreecodeParams(order=p, theta=0.5, leaf_capacity=500))
assert r.stats.farfield_evals == 6400 and r.stats.direct_pairs == 0, r.stats
"""


@pytest.mark.parametrize("p", [4, 8, 10])
def test_far_pair_executed_flops(p, tmp_path):
    sys.path.insert(0, ROOT)
    import bench
    n = 6400
    metrics = ",".join(f"smsp__sass_thread_inst_executed_op_{k}_pred_on.sum" for k in ("dfma", "dmul", "dadd"))
    log = tmp_path / "ncu.csv"
    out = subprocess.run(["ncu", "--metrics", metrics, "-k", "regex:k_far_list", "--csv", "--log-file", str(log),
                          sys.executable, "-c", SNIPPET, ROOT, str(p)],
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
    per_pair = (2 * vals["dfma"] + vals["dmul"] + vals["dadd"] - 3 * n) / n
    assert per_pair == bench.far_executed_flops(p + 2), (p, per_pair, vals)
