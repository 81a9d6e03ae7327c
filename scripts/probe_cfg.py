"""Timing probe for any BASELINE config through the host API (not the bench contract)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_12498_b200 as S
from bench import CONFIGS, make_inputs
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = CONFIGS[name]
ps, tg = make_inputs(cfg)
prm = S.TreecodeParams(order=cfg["order"], theta=cfg["theta"], leaf_capacity=cfg["n0"])
nt = cfg["targets"] or cfg["n"]
for _ in range(reps):
    t = time.time()
    r = S.treecode_velocity_targets(ps, tg, prm)
    w = time.time() - t
    print(f"{name}: wall {w:.3f}s total {r.time_total_s:.4f} build {r.time_build_s:.4f} mom {r.time_moments_s:.4f} "
          f"far {r.time_far_s:.4f} near {r.time_near_s:.4f} other {r.time_traverse_s - r.time_far_s - r.time_near_s:.4f} "
          f"A/t {r.stats.farfield_evals/nt:.1f} D/t {r.stats.direct_pairs/nt:.1f} V/t {r.stats.clusters_visited/nt:.1f} "
          f"targets/s {nt/r.time_total_s:.3e}", flush=True)
