"""BASELINE cfg0 (10K cube, p 6, theta 0.5, N0 500, both kernels) through the host API, plus
a disjoint-target call, a sliced near field (ST_NEAR_MAX_ENTRIES) and the O(N^2) direct sum:
the workload compute-sanitizer's memcheck / racecheck / synccheck run on
(scripts/sanitize.sh).  No torch: only the library's own kernels run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1811_12498_b200 as S

ps = S.generate("cube", 10000, 12345, True)
prm = S.TreecodeParams(order=6, theta=0.5, leaf_capacity=500)
a = S.treecode_velocity(ps, prm, per_target=True)
tg = S.generate("points", 3000, 67890).position
b = S.treecode_velocity_targets(ps, tg, prm)
os.environ["ST_NEAR_MAX_ENTRIES"] = "200000"
c = S.treecode_velocity(ps, prm)
os.environ.pop("ST_NEAR_MAX_ENTRIES")
assert c.velocity.tobytes() == a.velocity.tobytes()
d = S.contracted_direct_velocity_at(ps, S.KernelSelection.both(), np.arange(0, 10000, 10))
print("E vs direct", S.relative_error(d, a.velocity[::10]), "stats", a.stats)
