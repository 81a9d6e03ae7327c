"""Quick timing probe of the device phases (not the bench contract)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1811_12498_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n0 = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
theta = float(sys.argv[4]) if len(sys.argv) > 4 else 0.5
ps = S.generate("cube", n, 12345, True)
prm = S.TreecodeParams(order=p, theta=theta, leaf_capacity=n0)
print("fp64 peak TF/s:", S.fp64_peak(0.3))
for it in range(3):
    t = time.time()
    r = S.treecode_velocity(ps, prm)
    w = time.time() - t
    print(f"wall {w:.3f}s total {r.time_total_s:.4f} build {r.time_build_s:.4f} mom {r.time_moments_s:.4f} "
          f"trav {r.time_traverse_s:.4f} far {r.time_far_s:.4f} near {r.time_near_s:.4f} h2d {r.time_h2d_s:.4f} "
          f"d2h {r.time_d2h_s:.4f} launches {r.gpu_launches} A/t {r.stats.farfield_evals/n:.1f} "
          f"D/t {r.stats.direct_pairs/n:.1f} V/t {r.stats.clusters_visited/n:.1f} targets/s {n/r.time_total_s:.3e}")
