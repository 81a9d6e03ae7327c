"""Small self / disjoint-target treecode runs for compute-sanitizer (memcheck, racecheck):
python scripts/sanitize_near.py.  Exercises the near-field plan with one slab and with many
(ST_NEAR_MAX_ENTRIES), self regions with holes (leaves split across slabs), and checks that
every variant is bit-identical to the one-slab result."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1811_12498_b200 as S


def particles(n, seed):
    rng = np.random.default_rng(seed)
    nu = rng.normal(size=(n, 3))
    nu /= np.linalg.norm(nu, axis=1, keepdims=True)
    return S.ParticleSet(rng.uniform(-0.5, 0.5, (n, 3)), rng.uniform(-1, 1, (n, 3)),
                         rng.uniform(-1, 1, (n, 3)), nu)


def main():
    ps = particles(6000, 1)
    tg = np.random.default_rng(2).uniform(-0.6, 0.6, (3000, 3))
    for sel in (S.KernelSelection(), S.KernelSelection.stokeslet_only(), S.KernelSelection.stresslet_only()):
        prm = S.TreecodeParams(order=4, theta=0.6, leaf_capacity=150, kernels=sel)
        out = {}
        for cap in (None, "5000", "777"):
            if cap is None:
                os.environ.pop("ST_NEAR_MAX_ENTRIES", None)
            else:
                os.environ["ST_NEAR_MAX_ENTRIES"] = cap
            out[("self", cap)] = S.treecode_velocity(ps, prm).velocity
            out[("disjoint", cap)] = S.treecode_velocity_targets(ps, tg, prm).velocity
        os.environ.pop("ST_NEAR_MAX_ENTRIES", None)
        for kind in ("self", "disjoint"):
            for cap in ("5000", "777"):
                assert np.array_equal(out[(kind, None)], out[(kind, cap)]), (kind, cap)
        print("ok: slabs bit-identical", sel.stokeslet_enabled, sel.stresslet_enabled,
              {k[0]: float(np.abs(v).sum()) for k, v in out.items() if k[1] is None})


if __name__ == "__main__":
    main()
