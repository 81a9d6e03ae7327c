"""Time the moment pass alone (st_compute_moments over a prebuilt tree) for a config:
python scripts/moments_ab.py cfg4 [reps]; ST_MOMENTS_EPT selects entries per thread."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_12498_b200 as S  # noqa: E402
from bench import CONFIGS, make_inputs  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg1"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ps, _ = make_inputs(cfg)
T = S.build_tree(ps, cfg["n0"], True)
best = 1e9
for _ in range(reps):
    t0 = time.perf_counter()
    m = S.compute_moments(T, cfg["order"], S.KernelSelection.both())
    best = min(best, time.perf_counter() - t0)
print(f"{sys.argv[1]} EPT={os.environ.get('ST_MOMENTS_EPT', 'default')} moments wall {best * 1e3:.2f} ms")
