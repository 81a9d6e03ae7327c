"""Regenerate the golden fixtures from the REFERENCE itself (oracle/_ref/libstref.so:
the unmodified headers of /root/reference compiled in place by oracle/Makefile).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The GPU box has no /root/reference; the committed .npz files pin the oracle there.

Inputs are the seeded generators of the product library (st_generate, DESIGN.md
"Synthetic inputs"); each fixture stores the SHA-256 of the input bytes so a
generator change is caught, and small cases also store the inputs themselves.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import paper_1811_12498_b200 as S  # noqa: E402  (host-side generator only)
from oracle import oracle as O  # noqa: E402


def digest(ps):
    h = hashlib.sha256()
    for a in (ps.position, ps.force_weight, ps.dipole_weight, ps.normal):
        if a is not None:
            h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def as_dict(ps):
    return dict(position=ps.position, force_weight=ps.force_weight, dipole_weight=ps.dipole_weight,
                normal=ps.normal)


def treecode_case(name, ps, order, theta, n0, shrink=True, sto=True, stre=True, targets=None,
                  store_inputs=False):
    d = as_dict(ps)
    ctx = O.RefContext(d, order, theta, n0, shrink, sto, stre, workers=os.cpu_count())
    T = ctx.tree()
    if targets is None:
        u, pt, st = ctx.eval(src_idx=np.arange(ps.size()), threads=os.cpu_count())
    else:
        u, pt, st = ctx.eval(xyz=targets, threads=os.cpu_count())
    out = dict(sha256=digest(ps), order=order, theta=theta, n0=n0, shrink=int(shrink), sto=int(sto),
               stre=int(stre), n=ps.size(), u=u, per_target=pt.astype(np.uint32),
               stats=np.array([st["farfield_evals"], st["direct_pairs"], st["clusters_visited"]], np.uint64),
               perm=T.to_original, be=np.stack([T.begin, T.end], 1), geom_bits=T.geom.view(np.uint64),
               children=T.children, meta=np.stack([T.n_children, T.is_leaf], 1))
    if targets is not None:
        out["targets"] = targets
    if store_inputs:
        for k, v in d.items():
            if v is not None:
                out["in_" + k] = v
    ctx.close()
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, st, "ncl", T.ncl)


def main():
    assert O.have_ref(), "needs oracle/_ref (make -C oracle with /root/reference mounted)"
    # BASELINE.json configs[0]
    treecode_case("cfg0", S.generate("cube", 10000, 12345, True), 6, 0.5, 500)
    # shrink off, stokeslet only / stresslet only, small
    treecode_case("small_noshrink", S.generate("unit", 3000, 5, True), 4, 0.6, 100, shrink=False,
                  store_inputs=True)
    treecode_case("small_sto", S.generate("unit", 2000, 62, False), 4, 0.6, 200, sto=True, stre=False,
                  store_inputs=True)
    treecode_case("small_str", S.generate("unit", 2000, 63, True), 5, 0.5, 150, sto=False, stre=True,
                  store_inputs=True)
    # configs[2] / configs[4] shapes, reduced
    treecode_case("sphere_small", S.generate("sphere", 8000, 12345, True), 10, 0.7, 400)
    treecode_case("mixture_disjoint", S.generate("mixture", 6000, 12345, True), 8, 0.6, 300,
                  targets=S.generate("points", 1500, 67890).position)
    # N0 = 1 stress tree
    treecode_case("unit_n0_1", S.generate("unit", 600, 3, True), 2, 0.5, 1, store_inputs=True)

    # moments (moments.hpp:140-175) of a small tree
    ps = S.generate("unit", 500, 9, True)
    ctx = O.RefContext(as_dict(ps), 3, 0.5, 64, True)
    m = ctx.moments()
    np.savez_compressed(os.path.join(HERE, "moments_p3.npz"), sha256=digest(ps), **m,
                        in_position=ps.position, in_force_weight=ps.force_weight,
                        in_dipole_weight=ps.dipole_weight, in_normal=ps.normal)
    ctx.close()

    # per-pair far field (farfield.hpp) and Coulomb coefficients (coulomb.hpp)
    rng = np.random.default_rng(2718)
    rows = []
    for p in (0, 2, 5, 8, 10):
        for pair in range(6):
            q = S.generate("unit", 20 + 5 * pair, 900 + pair, True)
            cx = O.RefContext(as_dict(q), p, 0.5, q.size() + 1, True)
            mm = cx.moments()
            T = cx.tree()
            dvec = rng.normal(size=3)
            dvec *= T.radius[0] * (1.5 + 2.5 * rng.uniform()) / np.linalg.norm(dvec)
            u = O.ref_farfield_pair(dvec, p, mm["stok"][0], mm["str"][0], mm["trace"][0], mm["sym"][0])
            rows.append((p, dvec, mm["stok"][0].copy(), mm["str"][0].copy(), mm["trace"][0].copy(),
                         mm["sym"][0].copy(), u))
            cx.close()
    np.savez_compressed(
        os.path.join(HERE, "farfield_pairs.npz"),
        p=np.array([r[0] for r in rows]), dx=np.array([r[1] for r in rows]),
        u=np.array([r[6] for r in rows]),
        **{f"stok_{i}": r[2] for i, r in enumerate(rows)}, **{f"str_{i}": r[3] for i, r in enumerate(rows)},
        **{f"trace_{i}": r[4] for i, r in enumerate(rows)}, **{f"sym_{i}": r[5] for i, r in enumerate(rows)})
    dxs = np.array([[1.0, 0, 0], [0, 2.0, 0], [0.3, -1.2, 0.4], [0.7, 0.2, -0.9]])
    np.savez_compressed(os.path.join(HERE, "coulomb.npz"), dx=dxs,
                        **{f"b{i}": O.ref_coulomb(d, 6) for i, d in enumerate(dxs)})

    # direct sums (kernels.hpp:89-150)
    ps = S.generate("unit", 400, 100, True)
    tg = np.arange(400)
    np.savez_compressed(os.path.join(HERE, "direct.npz"), sha256=digest(ps),
                        u_both=O.ref_direct_at(as_dict(ps), tg, True, True),
                        u_sto=O.ref_direct_at(as_dict(ps), tg, True, False),
                        u_str=O.ref_direct_at(as_dict(ps), tg, False, True),
                        u_naive=O.ref_naive_direct(as_dict(ps), True, True),
                        in_position=ps.position, in_force_weight=ps.force_weight,
                        in_dipole_weight=ps.dipole_weight, in_normal=ps.normal)
    taylor()
    print("golden fixtures written to", HERE)


def taylor():
    """Explicit Taylor coefficients (taylor_coeffs.hpp:13-46), grade <= 4 from b of depth 6."""
    dxs = np.array([[1.0, 0, 0], [1.0, 1, 1], [0.3, -1.2, 0.4], [-0.6, 0.25, 0.8]])
    out = {"dx": dxs}
    for i, d in enumerate(dxs):
        out[f"sto{i}"], out[f"str{i}"] = O.ref_taylor(d, 4, 6)
    np.savez_compressed(os.path.join(HERE, "taylor.npz"), **out)


if __name__ == "__main__":
    # `make_golden.py taylor` regenerates that fixture alone
    taylor() if sys.argv[1:] == ["taylor"] else main()
