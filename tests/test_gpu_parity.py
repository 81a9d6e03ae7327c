"""GPU parity: the CUDA path (through the C ABI) against the reference compiled in
place (oracle/_ref) and the C restatement (oracle/liboracle.so).

Bars (BASELINE.json north_star): tree and interaction lists bit-exact;
velocities within 1e-12 relative L2 of the reference treecode; error against
direct summation equal to the reference's within 1%."""
import numpy as np
import pytest

from conftest import as_dict

pytestmark = pytest.mark.gpu

REL_TOL = 1e-12  # north_star: fp64 velocities within 1e-12 relative L2 of the reference treecode


def tree_equal(T_gpu, T_ref):
    assert T_gpu.ncl == T_ref.ncl
    assert np.array_equal(T_gpu.to_original, T_ref.to_original)
    assert np.array_equal(T_gpu.begin, T_ref.begin) and np.array_equal(T_gpu.end, T_ref.end)
    assert np.array_equal(T_gpu.children, T_ref.children)
    assert np.array_equal(T_gpu.n_children, T_ref.n_children)
    assert np.array_equal(T_gpu.is_leaf, T_ref.is_leaf)
    # centre, radius and bbox bytes (cluster_tree.hpp:88-93)
    assert np.array_equal(T_gpu.geom.view(np.uint64), T_ref.geom.view(np.uint64))


@pytest.mark.parametrize("kind,n,n0,shrink", [
    ("cube", 10000, 500, True), ("cube", 10000, 500, False), ("unit", 3000, 1, True),
    ("sphere", 20000, 200, True), ("sphere", 20000, 200, False), ("mixture", 50000, 100, True),
    ("cube", 200000, 2000, True), ("unit", 7, 1, True),
    # > 64K splitting segments possible (n / (N0+1)): the keyed levels by the host loop, then
    # the partition passes below depth 10
    ("cube", 140000, 1, True),
])
def test_tree_bit_exact(S, need_ref, kind, n, n0, shrink):
    ps = S.generate(kind, n, 12345, True)
    T = S.build_tree(ps, n0, shrink)
    ctx = need_ref.RefContext(as_dict(ps), 0, 0.5, n0, shrink)
    tree_equal(T, ctx.tree())


def test_tree_coincident_points_reach_depth_64(S, need_ref):
    """3,000 copies of one point among 2,000 others: the reference splits them until its
    depth cap (leaf iff count <= N0 or depth >= 64, cluster_tree.hpp:96) -- 54 partition
    levels below the keyed ones."""
    rng = np.random.default_rng(5)
    pos = np.concatenate([rng.uniform(-1, 1, (2000, 3)), np.tile([[0.125, -0.25, 0.375]], (3000, 1))])
    pos = pos[rng.permutation(len(pos))]
    nu = rng.normal(size=pos.shape)
    nu /= np.linalg.norm(nu, axis=1, keepdims=True)
    ps = S.ParticleSet(pos, rng.uniform(-1, 1, pos.shape), rng.uniform(-1, 1, pos.shape), nu)
    T = S.build_tree(ps, 50, True)
    ctx = need_ref.RefContext(as_dict(ps), 0, 0.5, 50, True)
    R = ctx.tree()
    tree_equal(T, R)
    assert T.is_leaf.sum() > 0 and T.ncl > 64


_BUILD_SNIPPET = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1811_12498_b200 as S
kind, n, n0 = sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
T = S.build_tree(S.generate(kind, n, 12345, True), n0, True)
np.savez(sys.argv[5], to_original=T.to_original, begin=T.begin, end=T.end, children=T.children,
         geom=T.geom)
"""


@pytest.mark.parametrize("env", ["ST_TREE_PARTITION", "ST_TREE_LEVEL_LOOP"])
@pytest.mark.parametrize("kind,n,n0", [("cube", 50000, 100), ("mixture", 30000, 20), ("unit", 3000, 1)])
def test_tree_build_variants_bit_exact(S, need_ref, tmp_path, env, kind, n, n0):
    """The A/B switches of the build (partition passes from the root; the keyed levels by the
    host loop instead of the cooperative launch) give the same trees (env read once per
    process: a subprocess per variant)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "t.npz"
    r = subprocess.run([sys.executable, "-c", _BUILD_SNIPPET, root, kind, str(n), str(n0), str(out)],
                       env=dict(os.environ, **{env: "1"}), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = np.load(out)
    ps = S.generate(kind, n, 12345, True)
    R = need_ref.RefContext(as_dict(ps), 0, 0.5, n0, True).tree()
    assert np.array_equal(got["to_original"], R.to_original)
    assert np.array_equal(got["begin"], R.begin) and np.array_equal(got["end"], R.end)
    assert np.array_equal(got["children"], R.children)
    assert np.array_equal(got["geom"].view(np.uint64), R.geom.view(np.uint64))


def test_tree_corner_cases(S, need_ref):
    # eight cube corners with unit leaves (test_cluster_tree.cpp:63-83)
    pos = np.array([[x, y, z] for z in (0.0, 1.0) for y in (0.0, 1.0) for x in (0.0, 1.0)])
    ps = S.ParticleSet(pos, np.tile([1.0, 0, 0], (8, 1)))
    T = S.build_tree(ps, 1, True)
    assert T.ncl == 9 and T.n_children[0] == 8 and T.is_leaf.sum() == 8
    assert np.all(T.radius[T.is_leaf == 1] == 0.0)
    ctx = need_ref.RefContext(dict(position=pos, force_weight=ps.force_weight), 0, 0.5, 1, True,
                              sto=True, stre=False)
    tree_equal(T, ctx.tree())
    # single particle (:52-61)
    one = S.ParticleSet(np.array([[0.3, -0.2, 0.9]]), np.array([[1.0, 0, 0]]))
    T1 = S.build_tree(one, 2000, False)
    assert T1.ncl == 1 and T1.is_leaf[0] == 1 and T1.radius[0] == 0.0
    assert np.array_equal(T1.center[0], one.position[0])


def test_moments_match_reference(S, need_ref):
    ps = S.generate("cube", 20000, 7, True)
    T = S.build_tree(ps, 300, True)
    for p in (0, 3, 8):
        m = S.compute_moments(T, p, S.KernelSelection.both())
        ctx = need_ref.RefContext(as_dict(ps), p, 0.5, 300, True)
        r = ctx.moments()
        for key, mine in (("stok", m.stok), ("str", m.str), ("trace", m.trace), ("sym", m.sym)):
            ref = r[key].reshape(mine.shape)
            scale = np.abs(ref).max(axis=(1, 2), keepdims=True) + 1e-300
            # internal clusters come from the exact M2M shift of their children's moments,
            # so sums are reassociated relative to the reference's particle-order sum:
            # 1e-12 of the cluster's largest moment (observed <= 4e-13 at N = 20,000)
            assert np.max(np.abs(mine - ref) / scale) < 1e-12, (p, key)


def test_direct_matches_reference(S, need_ref):
    ps = S.generate("cube", 3000, 99, True)
    for sel in (S.KernelSelection.both(), S.KernelSelection.stokeslet_only(),
                S.KernelSelection.stresslet_only()):
        u = S.contracted_direct_velocity(ps, sel)
        ref = need_ref.ref_direct_at(as_dict(ps), np.arange(3000), sel.stokeslet_enabled, sel.stresslet_enabled)
        assert S.relative_error(ref, u) < 1e-14
    sub = S.contracted_direct_velocity(ps, S.KernelSelection.both(), 10, 25)
    full = S.contracted_direct_velocity(ps, S.KernelSelection.both())
    assert np.array_equal(sub, full[10:25])
    assert S.contracted_direct_velocity(ps, S.KernelSelection.both(), 5, 5).shape == (0, 3)
    at = S.contracted_direct_velocity_at(ps, S.KernelSelection.both(), [7, 3, 2999])
    assert np.array_equal(at, full[[7, 3, 2999]])


def test_naive_matches_contracted(S):
    # contracted == naive at <= 1e-13 (test_kernels.cpp:158-175)
    for n in (2, 10, 500):
        ps = S.generate("unit", n, 100 + n, True)
        for sel in (S.KernelSelection.both(), S.KernelSelection.stokeslet_only(),
                    S.KernelSelection.stresslet_only()):
            a = S.naive_direct_velocity(ps, sel)
            b = S.contracted_direct_velocity(ps, sel)
            num = np.linalg.norm(a - b, axis=1)
            den = np.maximum(np.linalg.norm(a, axis=1), np.linalg.norm(b, axis=1))
            assert np.all(num <= 1e-13 * np.maximum(den, 1e-300))


def test_naive_hand_cases(S):
    # test_kernels.cpp:130-156
    ps = S.ParticleSet(np.array([[0, 0, 0], [1, 0, 0.0]]), np.array([[1, 0, 0], [1, 0, 0.0]]))
    u = S.naive_direct_velocity(ps, S.KernelSelection.stokeslet_only())
    assert np.array_equal(u, [[2, 0, 0], [2, 0, 0]])
    ps = S.ParticleSet(np.array([[0, 0, 0], [1, 0, 0.0]]), np.zeros((2, 3)), np.array([[1, 0, 0], [1, 0, 0.0]]),
                       np.array([[1, 0, 0], [1, 0, 0.0]]))
    u = S.naive_direct_velocity(ps, S.KernelSelection.stresslet_only())
    assert np.array_equal(u, [[-1, 0, 0], [1, 0, 0]])


def test_coincident_points_raise_domain_error(S):
    # test_kernels.cpp:188-196
    ps = S.ParticleSet(np.array([[0, 0, 0], [1, 1, 1], [0, 0, 0.0]]), np.tile([1.0, 0, 0], (3, 1)))
    with pytest.raises(S.DomainError):
        S.contracted_direct_velocity(ps, S.KernelSelection.stokeslet_only())
    with pytest.raises(S.DomainError):
        S.naive_direct_velocity(ps, S.KernelSelection.stokeslet_only())
    with pytest.raises(S.DomainError):
        S.treecode_velocity(ps, S.TreecodeParams(kernels=S.KernelSelection.stokeslet_only()))


def random_cluster(S, rng, n, p):
    ps = S.generate("unit", n, int(rng.integers(1 << 30)), True)
    T = S.build_tree(ps, n + 1, True)
    return ps, T


@pytest.mark.parametrize("p", [0, 1, 2, 4, 6, 8, 10, 12, 16])
def test_farfield_pairs_match_reference(S, need_ref, p):
    rng = np.random.default_rng(p)
    dxs, stoks, strs, refs = [], [], [], []
    for pair in range(24):
        ps, T = random_cluster(S, rng, 20 + pair, p)
        m = S.compute_moments(T, p, S.KernelSelection.both())
        d = rng.normal(size=3)
        d *= T.radius[0] * (1.5 + 2.5 * rng.uniform()) / np.linalg.norm(d)
        stok, strm, tr, sy = m.stok[0], m.str[0], m.trace[0], m.sym[0]
        refs.append(need_ref.ref_farfield_pair(d, p, stok, strm, tr, sy))
        dxs.append(d)
        stoks.append(stok)
        strs.append(strm)
    u = S.farfield_pairs(np.array(dxs), p, np.array(stoks), np.array(strs))
    ref = np.array(refs)
    rel = np.linalg.norm(u - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert rel.max() < 1e-12, rel.max()


def test_coulomb_matches_reference(S, need_ref):
    rng = np.random.default_rng(3)
    dx = rng.normal(size=(50, 3))
    for pmax in (0, 3, 10):
        b = S.coulomb_coeffs(dx, pmax)
        for i in range(0, 50, 7):
            ref = need_ref.ref_coulomb(dx[i], pmax)[:-1]
            assert np.max(np.abs(b[i] - ref) / np.abs(ref).max()) < 1e-13
    # hand values (test_coulomb.cpp:11-25)
    b = S.coulomb_coeffs([[1, 0, 0], [0, 2, 0]], 3)
    assert b[0][0] == 1.0 and b[0][1 + 2] == 1.0  # b^0, b^(1,0,0)
    with pytest.raises(S.DomainError):
        S.coulomb_coeffs([[0, 0, 0]], 2)


def test_taylor_coeffs_match_oracle(S, O):
    # taylor_coeffs.hpp:13-46 on the device: b formed on the device, or the caller's b
    rng = np.random.default_rng(11)
    dx = rng.uniform(-2, 2, size=(40, 3))
    for order in (0, 1, 4, 8, 14):
        a, t = S.taylor_coeffs(dx, order)
        b = S.coulomb_coeffs(dx, order + 3)
        a2, t2 = S.taylor_coeffs(dx, order, b=b)
        for q in range(0, 40, 3):
            ao, to = O.or_taylor(dx[q], order, order + 2)
            for got, want in ((a[q], ao), (t[q], to), (a2[q], ao), (t2[q], to)):
                # device FMA contraction vs the reference's separate multiply/add
                assert np.max(np.abs(got - want)) <= 1e-13 * np.abs(want).max()
    # one kernel only: the other output is not formed
    a, t = S.taylor_coeffs(dx[:2], 3, stresslet=False)
    assert t is None and a.shape == (2, 20, 3, 3)


def test_taylor_coeffs_match_golden(S):
    import os
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "taylor.npz"))
    a, t = S.taylor_coeffs(g["dx"], 4, pmax_b=6)
    for i in range(len(g["dx"])):
        for got, want in ((a[i], g[f"sto{i}"]), (t[i], g[f"str{i}"])):
            assert np.max(np.abs(got - want)) <= 1e-13 * np.abs(want).max()


def test_taylor_coeffs_reference_tests(S, O):
    # test_taylor_coeffs.cpp:13-116 through the device entry point
    from test_oracle import check_taylor_fd, kernel_tensors, rel_diff, taylor_zeroth_cases
    for x, y in taylor_zeroth_cases(O):
        a, t = S.taylor_coeffs([x - y], 0, pmax_b=3)
        S_, T_ = kernel_tensors(x, y)
        assert rel_diff(a[0, 0], S_).max() < 1e-12 and rel_diff(t[0, 0], T_).max() < 5e-12
    a, _ = S.taylor_coeffs([[1.0, 0, 0], [0, 0, 1.0]], 0, stresslet=False)
    assert abs(a[0, 0, 0, 0] - 2.0) <= 1e-14 and a[1, 0, 0, 1] == 0.0
    _, t = S.taylor_coeffs([[1.0, 1, 1]], 0, stokeslet=False)
    assert abs(t[0, 0, 0, 0, 0] - 1 / (9 * np.sqrt(3))) <= 1e-13 * t[0, 0, 0, 0, 0]
    check_taylor_fd(O, lambda x, p: tuple(None if v is None else v[0] for v in S.taylor_coeffs([x], p)))


def run_pair(S, O, ps, order, theta, n0, shrink=True, sel=None):
    sel = sel or S.KernelSelection.both()
    prm = S.TreecodeParams(order=order, theta=theta, leaf_capacity=n0, shrink=shrink, kernels=sel)
    res = S.treecode_velocity(ps, prm, per_target=True)
    ctx = O.RefContext(as_dict(ps), order, theta, n0, shrink, sel.stokeslet_enabled, sel.stresslet_enabled)
    u_ref, pt_ref, st_ref = ctx.eval(src_idx=np.arange(ps.size()), threads=8)
    return res, u_ref, pt_ref, st_ref


@pytest.mark.parametrize("order,theta,n0", [(6, 0.5, 500), (2, 0.7, 200), (10, 0.5, 1000), (0, 0.3, 64)])
def test_treecode_cfg0_parity(S, need_ref, order, theta, n0):
    # BASELINE.json configs[0]: N = 10,000 cube, theta 0.5, p 6, N0 500
    ps = S.generate("cube", 10000, 12345, True)
    res, u_ref, pt_ref, st_ref = run_pair(S, need_ref, ps, order, theta, n0)
    # interaction lists: per-target (visited, accepted, direct pairs) bit-exact
    assert np.array_equal(res.per_target, pt_ref)
    assert res.stats.farfield_evals == st_ref["farfield_evals"]
    assert res.stats.direct_pairs == st_ref["direct_pairs"]
    assert res.stats.clusters_visited == st_ref["clusters_visited"]
    assert S.relative_error(u_ref, res.velocity) <= REL_TOL


@pytest.mark.parametrize("order,sel", [(12, "both"), (14, "stokeslet_only"), (16, "both"), (16, "stresslet_only")])
def test_treecode_high_orders(S, need_ref, order, sel):
    """The top of the order range (kMaxOrder = 16, engine.hpp:23): far kernels up to
    P = 18, where the harmonic recurrence's registers spill; still within 1e-12 of the
    reference, interaction lists bit-exact."""
    k = getattr(S.KernelSelection, sel)()
    ps = S.generate("cube", 6000, 4242, True)
    res, u_ref, pt_ref, st_ref = run_pair(S, need_ref, ps, order, 0.5, 250, sel=k)
    assert np.array_equal(res.per_target, pt_ref)
    assert res.stats.farfield_evals == st_ref["farfield_evals"]
    assert S.relative_error(u_ref, res.velocity) <= REL_TOL


def test_treecode_error_vs_direct_matches_reference(S, need_ref):
    ps = S.generate("cube", 10000, 12345, True)
    res, u_ref, _, _ = run_pair(S, need_ref, ps, 6, 0.5, 500)
    direct = S.contracted_direct_velocity(ps, S.KernelSelection.both())
    e_gpu = S.relative_error(direct, res.velocity)
    e_ref = S.relative_error(direct, u_ref)
    assert abs(e_gpu - e_ref) <= 0.01 * e_ref


@pytest.mark.parametrize("sel", ["stokeslet_only", "stresslet_only"])
def test_treecode_kernel_selection(S, need_ref, sel):
    k = getattr(S.KernelSelection, sel)()
    ps = S.generate("cube", 8000, 77, True)
    res, u_ref, pt_ref, _ = run_pair(S, need_ref, ps, 5, 0.6, 300, sel=k)
    assert np.array_equal(res.per_target, pt_ref)
    assert S.relative_error(u_ref, res.velocity) <= REL_TOL


def test_treecode_sphere_and_mixture(S, need_ref):
    for kind, order, theta, n0 in (("sphere", 10, 0.7, 500), ("mixture", 8, 0.6, 300)):
        ps = S.generate(kind, 30000, 12345, True)
        res, u_ref, pt_ref, _ = run_pair(S, need_ref, ps, order, theta, n0)
        assert np.array_equal(res.per_target, pt_ref)
        assert S.relative_error(u_ref, res.velocity) <= REL_TOL


def test_disjoint_targets(S, need_ref):
    # configs[4] shape, small: mixture sources, uniform disjoint targets
    ps = S.generate("mixture", 20000, 12345, True)
    tg = S.generate("points", 5000, 67890).position
    prm = S.TreecodeParams(order=8, theta=0.6, leaf_capacity=300)
    res = S.treecode_velocity_targets(ps, tg, prm, per_target=True)
    ctx = need_ref.RefContext(as_dict(ps), 8, 0.6, 300, True)
    u_ref, pt_ref, _ = ctx.eval(xyz=tg, threads=8)
    assert np.array_equal(res.per_target, pt_ref)
    assert S.relative_error(u_ref, res.velocity) <= REL_TOL


def test_vanishing_theta_is_direct(S):
    # test_engine.cpp:12-24
    ps = S.generate("unit", 3000, 9001, True)
    res = S.treecode_velocity(ps, S.TreecodeParams(order=5, theta=1e-9, leaf_capacity=100))
    direct = S.contracted_direct_velocity(ps, S.KernelSelection.both())
    assert res.stats.farfield_evals == 0
    assert S.relative_error(direct, res.velocity) <= 1e-13


def test_single_leaf_equals_direct(S):
    # test_engine.cpp:26-36 (bit-for-bit in the reference; same formula order here up to FMA)
    ps = S.generate("unit", 150, 404, True)
    res = S.treecode_velocity(ps, S.TreecodeParams(order=2, theta=0.5, leaf_capacity=2000))
    direct = S.contracted_direct_velocity(ps, S.KernelSelection.both())
    assert S.relative_error(direct, res.velocity) <= 1e-15
    assert res.stats.farfield_evals == 0


def test_single_particle_zero_velocity(S):
    ps = S.ParticleSet(np.array([[1.0, 2, 3]]), np.array([[4.0, 5, 6]]))
    res = S.treecode_velocity(ps, S.TreecodeParams(kernels=S.KernelSelection.stokeslet_only()))
    assert np.array_equal(res.velocity, [[0.0, 0, 0]])


def test_determinism_across_runs(S):
    ps = S.generate("cube", 50000, 5, True)
    prm = S.TreecodeParams(order=4, theta=0.5, leaf_capacity=400)
    a = S.treecode_velocity(ps, prm).velocity
    b = S.parallel_velocity(ps, S.TreecodeParams(order=4, theta=0.5, leaf_capacity=400, workers=4)).velocity
    assert a.tobytes() == b.tobytes()


def test_validation_errors(S):
    ps = S.generate("cube", 100, 1, True)
    bad = S.ParticleSet(ps.position.copy(), ps.force_weight, ps.dipole_weight, ps.normal.copy())
    bad.normal[17] *= 1.0 + 1e-9
    with pytest.raises(S.InvalidArgument, match="normal 17 is not unit length"):
        S.treecode_velocity(bad, S.TreecodeParams())
    bad2 = S.ParticleSet(ps.position.copy(), ps.force_weight)
    bad2.position[3, 1] = np.nan
    with pytest.raises(S.InvalidArgument, match="position"):
        S.treecode_velocity(bad2, S.TreecodeParams(kernels=S.KernelSelection.stokeslet_only()))
    with pytest.raises(S.InvalidArgument):
        S.treecode_velocity(S.ParticleSet(np.zeros((0, 3))), S.TreecodeParams())
    # validation precedes the coincident-pair domain error, as in run_treecode (engine.hpp:133-135)
    both = S.ParticleSet(ps.position.copy(), ps.force_weight, ps.dipole_weight, ps.normal.copy())
    both.position[5] = both.position[6]
    both.normal[9] *= 2.0
    with pytest.raises(S.InvalidArgument, match="normal 9"):
        S.treecode_velocity(both, S.TreecodeParams())
    with pytest.raises(S.InvalidArgument, match="targets"):
        S.treecode_velocity_targets(ps, np.array([[0.0, np.inf, 0.0]]), S.TreecodeParams())


@pytest.mark.parametrize("kind,n,n0,theta,shrink", [
    ("cube", 10000, 500, 0.5, True), ("sphere", 20000, 300, 0.7, True), ("mixture", 30000, 200, 0.6, False),
    ("cube", 200000, 2000, 0.5, True),
])
def test_interaction_lists_bit_exact(S, O, kind, n, n0, theta, shrink):
    """Full interaction lists (not just counts) equal the oracle's DFS lists."""
    ps = S.generate(kind, n, 12345, True)
    rng = np.random.default_rng(n)
    sel = rng.choice(n, 300, replace=False)
    prm = S.TreecodeParams(order=2, theta=theta, leaf_capacity=n0, shrink=shrink)
    far, near = S.interaction_lists(ps, prm, target_index=sel)
    T = O.or_build_tree(as_dict(ps), n0, shrink)
    to_tree = np.empty(n, np.uint32)
    to_tree[T.to_original] = np.arange(n, dtype=np.uint32)
    ofar, onear = O.or_lists(as_dict(ps), n0, shrink, theta, tree_idx=to_tree[sel], cap=4096)
    for i in range(len(sel)):
        assert np.array_equal(far[i], ofar[i]) and np.array_equal(near[i], onear[i]), i


def test_interaction_lists_disjoint_targets(S, O):
    ps = S.generate("mixture", 20000, 12345, True)
    pts = S.generate("points", 400, 67890).position
    prm = S.TreecodeParams(order=2, theta=0.6, leaf_capacity=300)
    far, near = S.interaction_lists(ps, prm, points=pts)
    ofar, onear = O.or_lists(as_dict(ps), 300, True, 0.6, xyz=pts, cap=4096)
    for i in range(len(pts)):
        assert np.array_equal(far[i], ofar[i]) and np.array_equal(near[i], onear[i]), i


@pytest.mark.parametrize("devices", [2, 3, 8])
def test_multi_device_bit_identical(S, devices):
    """params.devices > 1: shards on (logical) GPUs gathered over P2P; with one physical GPU
    the logical devices share it.  Results must be bit-identical to one device, the
    analogue of the reference's cross-worker identity (test_engine.cpp:48-70)."""
    for kind, tg in (("cube", None), ("mixture", S.generate("points", 7000, 67890).position)):
        ps = S.generate(kind, 30000, 5, True)
        one = S.treecode_velocity_targets(ps, tg, S.TreecodeParams(order=6, theta=0.5, leaf_capacity=400),
                                          per_target=True)
        many = S.treecode_velocity_targets(ps, tg, S.TreecodeParams(order=6, theta=0.5, leaf_capacity=400,
                                                                    devices=devices), per_target=True)
        assert many.velocity.tobytes() == one.velocity.tobytes()
        assert np.array_equal(many.per_target, one.per_target)
        assert many.stats == one.stats


def test_order_sweep_bit_identical_to_single_orders(S, need_ref):
    """One tree / moment pass / near pass for several orders == separate calls, bit for bit."""
    ps = S.generate("sphere", 20000, 12345, True)
    orders = [2, 0, 5, 8]
    prm = S.TreecodeParams(order=6, theta=0.7, leaf_capacity=400)
    u, fs, res = S.treecode_velocity_sweep(ps, prm, orders)
    assert np.all(fs > 0)
    for i, p in enumerate(orders):
        one = S.treecode_velocity(ps, S.TreecodeParams(order=p, theta=0.7, leaf_capacity=400))
        assert u[i].tobytes() == one.velocity.tobytes(), p
        assert res.stats == one.stats
    ctx = need_ref.RefContext(as_dict(ps), 8, 0.7, 400, True)
    u_ref, _, _ = ctx.eval(src_idx=np.arange(ps.size()), threads=8)
    assert S.relative_error(u_ref, u[3]) <= REL_TOL


def test_depth_64_chain_tree_matches_reference(S, need_ref):
    """Coincident points never separate: the reference recursion stops at depth 64
    (cluster_tree.hpp:72, 96).  The level-synchronous build must reproduce that chain."""
    ps = S.generate("unit", 500, 21, True)
    pos = ps.position.copy()
    pos[10] = pos[11] = pos[12] = pos[3]
    dup = S.ParticleSet(pos, ps.force_weight, ps.dipole_weight, ps.normal)
    T = S.build_tree(dup, 1, True)
    ctx = need_ref.RefContext(as_dict(dup), 0, 0.5, 1, True)
    tree_equal(T, ctx.tree())
    deepest = T.ncl
    assert deepest > 64 and T.is_leaf.sum() < 500  # a leaf holds the 4 coincident points
    with pytest.raises(S.DomainError):
        S.treecode_velocity(dup, S.TreecodeParams(order=2, leaf_capacity=1))


def test_large_leaves_multi_chunk_moments(S, need_ref):
    """Leaves above the 8,192-particle moment chunk use per-chunk partial sums."""
    ps = S.generate("cube", 100000, 3, True)
    T = S.build_tree(ps, 20000, True)
    assert (T.end - T.begin)[T.is_leaf == 1].max() > 8192
    m = S.compute_moments(T, 4, S.KernelSelection.both())
    r = need_ref.RefContext(as_dict(ps), 4, 0.5, 20000, True).moments()
    for key, mine in (("stok", m.stok), ("str", m.str)):
        ref = r[key].reshape(mine.shape)
        scale = np.abs(ref).max(axis=(1, 2), keepdims=True)
        assert np.max(np.abs(mine - ref) / scale) < 1e-12
    res = S.treecode_velocity(ps, S.TreecodeParams(order=4, theta=0.5, leaf_capacity=20000))
    u_ref, _, _ = need_ref.ref_parallel_velocity(as_dict(ps), 4, 0.5, 20000, workers=8)
    assert S.relative_error(u_ref, res.velocity) <= REL_TOL


def test_disjoint_target_on_a_source_is_a_domain_error(S):
    ps = S.generate("cube", 2000, 8, True)
    tg = np.vstack([S.generate("points", 10, 1).position, ps.position[17:18]])
    with pytest.raises(S.DomainError):
        S.treecode_velocity_targets(ps, tg, S.TreecodeParams(order=3, leaf_capacity=100))


def test_n0_one_full_tree_parity(S, need_ref):
    """Every leaf a single particle: all interactions are far field (test_cluster_tree)."""
    ps = S.generate("mixture", 3000, 4, True)
    res, u_ref, pt_ref, _ = run_pair(S, need_ref, ps, 3, 0.5, 1)
    assert np.array_equal(res.per_target, pt_ref)
    assert res.stats.direct_pairs == 0
    assert S.relative_error(u_ref, res.velocity) <= REL_TOL


def test_shard_device_slices_assemble_bit_exactly(S):
    """The one-rank-per-GPU entry: each shard's batch-order slice, assembled and unbatched,
    equals the single-GPU field bit for bit (shards run one after another on this GPU)."""
    import torch
    ps = S.generate("cube", 40000, 9, True)
    n = ps.size()
    src = torch.from_numpy(np.concatenate([ps.position, ps.force_weight, ps.dipole_weight, ps.normal])).cuda()
    b, stride = src.data_ptr(), n * 24
    ptrs = (b, b + stride, b + 2 * stride, b + 3 * stride)
    prm = S.TreecodeParams(order=6, theta=0.5, leaf_capacity=500)
    stream = torch.cuda.current_stream().cuda_stream
    full = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
    S.treecode_velocity_device(*ptrs, n, prm, full.data_ptr(), stream=stream)
    world = 3
    assembled = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
    torig = torch.empty(n, dtype=torch.int32, device="cuda")
    covered = 0
    for r in range(world):
        part = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
        t0, t1, _ = S.treecode_shard_device(*ptrs, n, prm, part.data_ptr(), torig.data_ptr(), shard=r,
                                            n_shards=world, stream=stream)
        assert t0 == covered
        covered = t1
        assembled[t0:t1] = part[t0:t1]
    assert covered == n
    out = torch.zeros_like(full)
    S.unbatch_device(n, torig.data_ptr(), assembled.data_ptr(), out.data_ptr(), stream=stream)
    torch.cuda.synchronize()
    assert torch.equal(out, full)


def test_near_field_slabs_are_bit_identical(S, monkeypatch):
    # the near field's per-entry buffers are cut into slabs of batch warps when they
    # would not fit; the cut points must not change a single bit
    ps = S.generate("cube", 30000, 7, True)
    prm = S.TreecodeParams(order=4, theta=0.5, leaf_capacity=300)
    a = S.treecode_velocity(ps, prm, per_target=True)
    for cap in ("5000", "777", "1"):
        monkeypatch.setenv("ST_NEAR_MAX_ENTRIES", cap)
        b = S.treecode_velocity(ps, prm, per_target=True)
        assert np.array_equal(a.velocity, b.velocity)
        assert np.array_equal(a.per_target, b.per_target)
        assert b.stats.direct_pairs == a.stats.direct_pairs


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_fused_gather(world):
    # bench.py's N>1 path: every rank's epilogue stores its shard into rank 0's buffer
    # through CUDA IPC (ranks share the one GPU here; they never wait on each other)
    import os
    import socket
    import subprocess
    import sys
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(here, "ipc_worker.py")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "IPC_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("world,case", [(2, ("cube", "30000", "6", "0.5", "300")),
                                        (3, ("sphere", "40000", "8", "0.7", "200")),
                                        (4, ("mixture", "30000", "5", "0.6", "100"))])
def test_split_moment_pass_ranks(world, case):
    """One process per rank, the moment pass split over the ranks and exchanged with
    torch.distributed (tests/split_worker.py): bit-identical to one GPU."""
    import os
    import socket
    import subprocess
    import sys
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(here, "split_worker.py"),
                        *case], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "SPLIT_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("devices", [2, 3, 8])
def test_split_moments_in_process_devices(S, devices):
    """TreecodeParams.devices > 1 splits the moment pass over the devices and exchanges the
    rows device to device (peer_exchange); deep trees (N0 = 20) so the split cuts below the
    root's children.  Bit-identical to one device."""
    for kind, n, n0, order in (("cube", 60000, 20, 6), ("sphere", 50000, 30, 10)):
        ps = S.generate(kind, n, 9, True)
        one = S.treecode_velocity(ps, S.TreecodeParams(order=order, theta=0.6, leaf_capacity=n0), per_target=True)
        many = S.treecode_velocity(ps, S.TreecodeParams(order=order, theta=0.6, leaf_capacity=n0, devices=devices),
                                   per_target=True)
        assert many.velocity.tobytes() == one.velocity.tobytes()
        assert np.array_equal(many.per_target, one.per_target)


def test_pageable_and_pinned_inputs_agree(S):
    # pageable host arrays go through the pinned staging ring in 4 MB chunks (an odd size
    # here: 3 full chunks + a tail per array); pinned arrays are copied directly
    import torch
    n = 175_001
    ps = S.generate("cube", n, 21, True)
    prm = S.TreecodeParams(order=3, theta=0.6, leaf_capacity=1000)
    a = S.treecode_velocity(ps, prm)
    pin = torch.empty((4 * n, 3), dtype=torch.float64).pin_memory().numpy()
    pin[:] = np.concatenate([ps.position, ps.force_weight, ps.dipole_weight, ps.normal])
    pps = S.ParticleSet(pin[:n], pin[n:2 * n], pin[2 * n:3 * n], pin[3 * n:])
    b = S.treecode_velocity(pps, prm)
    assert np.array_equal(a.velocity, b.velocity)
    d = S.contracted_direct_velocity_at(ps, S.KernelSelection.both(), np.arange(0, n, 997))
    e = S.contracted_direct_velocity_at(pps, S.KernelSelection.both(), np.arange(0, n, 997))
    assert np.array_equal(d, e)


def test_concurrent_calls_from_host_threads(S):
    # ctypes releases the GIL: four host threads call the library at once on one device
    # (shared per-device workspace, staging rings, copy pool); each result must equal the
    # sequential one bit for bit
    import threading
    cases = [(S.generate("cube", 60000 + 7000 * i, 50 + i, True),
              S.TreecodeParams(order=3 + i, theta=0.5, leaf_capacity=400)) for i in range(4)]
    want = [S.treecode_velocity(ps, prm).velocity for ps, prm in cases]
    got = [None] * 4
    errs = []

    def run(i):
        try:
            for _ in range(3):
                got[i] = S.treecode_velocity(*cases[i]).velocity
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for w, g in zip(want, got):
        assert np.array_equal(w, g)


def test_far_deferral_changes_rounding_only(S, need_ref, tmp_path):
    # sparse far events (accepted by <= 24 of a warp's lanes) are evaluated by the packed
    # pass and added after the dense ones; with ST_FAR_SPARSE=0 k_far evaluates every event.
    # Both orders agree to rounding and both match the reference treecode.
    import os
    import subprocess
    import sys
    ps = S.generate("mixture", 40000, 19, True)
    prm = S.TreecodeParams(order=6, theta=0.6, leaf_capacity=300)
    a = S.treecode_velocity(ps, prm).velocity
    out = tmp_path / "u0.npy"
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_1811_12498_b200 as S; "
            "ps = S.generate('mixture', 40000, 19, True); "
            "prm = S.TreecodeParams(order=6, theta=0.6, leaf_capacity=300); "
            "np.save(%r, S.treecode_velocity(ps, prm).velocity)" % (os.path.dirname(os.path.dirname(
                os.path.abspath(__file__))), str(out)))
    env = dict(os.environ, ST_FAR_SPARSE="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    b = np.load(out)
    assert S.relative_error(b, a) <= 1e-14
    ctx = need_ref.RefContext(as_dict(ps), 6, 0.6, 300, True)
    u_ref, _, _ = ctx.eval(src_idx=np.arange(ps.size()), threads=8)
    assert S.relative_error(u_ref, a) <= REL_TOL and S.relative_error(u_ref, b) <= REL_TOL


@pytest.mark.parametrize("n,n0,order,theta,sel", [
    (2, 1, 3, 0.5, "both"), (31, 1, 2, 0.9, "both"), (33, 2, 4, 0.5, "stokeslet_only"),
    (95, 3, 6, 0.7, "stresslet_only"), (257, 1, 1, 0.8, "both"), (1000, 7, 8, 0.4, "both"),
])
def test_ragged_sizes_match_reference(S, need_ref, n, n0, order, theta, sel):
    # batch boundaries (32 targets), one-particle leaves, every kernel selection: the
    # planned evaluation (near entries, dense far lists, deferred sparse far events)
    ksel = getattr(S.KernelSelection, sel)()
    ps = S.generate("unit", n, 1000 + n, ksel.stresslet_enabled)
    res, u_ref, pt_ref, st_ref = run_pair(S, need_ref, ps, order, theta, n0, sel=ksel)
    assert np.array_equal(res.per_target, pt_ref)
    assert res.stats.farfield_evals == st_ref["farfield_evals"]
    assert res.stats.direct_pairs == st_ref["direct_pairs"]
    assert S.relative_error(u_ref, res.velocity) <= REL_TOL


def test_near_plan_invariants_debug_checker():
    """ST_DEBUG_NEAR runs the bucket invariant kernels (every entry once, holes only in self
    regions, self entries at their record position) on self and disjoint targets, one slab
    and many, all three kernel selections; slab results must be bit-identical."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ST_DEBUG_NEAR="1")
    r = subprocess.run([sys.executable, os.path.join(root, "scripts", "sanitize_near.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("ok: slabs bit-identical") == 3
    assert "bucket invariant violated" not in r.stderr


@pytest.mark.parametrize("ept", ["1", "4"])
def test_moment_kernel_shapes_bit_identical(S, tmp_path, ept):
    # the moment kernel's multi-indices per thread (ST_MOMENTS_EPT; default 2) change only
    # which thread owns a multi-index, not the particle order of its sums: identical bits
    import os
    import subprocess
    import sys
    ps = S.generate("unit", 30000, 23, True)
    T = S.build_tree(ps, 700, True)
    m = S.compute_moments(T, 6, S.KernelSelection.both())
    out = tmp_path / "m.npz"
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_1811_12498_b200 as S; "
            "ps = S.generate('unit', 30000, 23, True); T = S.build_tree(ps, 700, True); "
            "m = S.compute_moments(T, 6, S.KernelSelection.both()); "
            "np.savez(%r, a=m.stok, b=m.str, c=m.trace, d=m.sym)" % (os.path.dirname(os.path.dirname(
                os.path.abspath(__file__))), str(out)))
    env = dict(os.environ, ST_MOMENTS_EPT=ept)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    g = np.load(out)
    for mine, other in ((m.stok, g["a"]), (m.str, g["b"]), (m.trace, g["c"]), (m.sym, g["d"])):
        assert mine.tobytes() == other.tobytes()


def test_device_call_with_weights_in_flight(S):
    # st_treecode_velocity_device_ev: the weight arrays arrive on another stream, the call
    # waits for their event after the tree build; the result equals the plain device call
    torch = pytest.importorskip("torch")
    ps = S.generate("cube", 60000, 29, True)
    n = ps.size()
    host = torch.from_numpy(np.concatenate([ps.position, ps.force_weight, ps.dipole_weight, ps.normal])).pin_memory()
    prm = S.TreecodeParams(order=6, theta=0.5, leaf_capacity=500)
    main = torch.cuda.current_stream()
    ref = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
    dsrc = host.cuda()
    b, st = dsrc.data_ptr(), n * 24
    S.treecode_velocity_device(b, b + st, b + 2 * st, b + 3 * st, n, prm, ref.data_ptr(), stream=main.cuda_stream)
    dsrc2 = torch.empty_like(dsrc)
    out = torch.zeros_like(ref)
    side = torch.cuda.Stream()
    ready = torch.cuda.Event()
    dsrc2[:n].copy_(host[:n], non_blocking=True)
    with torch.cuda.stream(side):
        torch.cuda._sleep(2_000_000)  # the weights arrive late
        dsrc2[n:].copy_(host[n:], non_blocking=True)
        ready.record(side)
    b2 = dsrc2.data_ptr()
    S.treecode_velocity_device(b2, b2 + st, b2 + 2 * st, b2 + 3 * st, n, prm, out.data_ptr(),
                               stream=main.cuda_stream, weights_event=ready.cuda_event)
    torch.cuda.synchronize()
    assert out.cpu().numpy().tobytes() == ref.cpu().numpy().tobytes()


@pytest.mark.parametrize("kind,n,n0,order,theta,world,disjoint", [
    ("cube", 20000, 300, 4, 0.5, 3, False), ("mixture", 12000, 200, 6, 0.6, 4, True),
    ("sphere", 9000, 150, 3, 0.7, 2, False),
])
def test_shard_plan_matches_host_model(S, O, kind, n, n0, order, theta, world, disjoint):
    """The batch order (octree keys) and the work-balanced shard ranges the library computes on the
    GPU equal tests/shard_model.py's host restatement (which tests/test_multirank.py uses for
    its gloo ranks): octree keys, k_count's integer cost model, st_shard_cuts."""
    import torch
    import shard_model as M
    ps = S.generate(kind, n, 21, True)
    tg = S.generate("points", 7000, 67890).position if disjoint else None
    nt = n if tg is None else len(tg)
    src = torch.from_numpy(np.concatenate([ps.position, ps.force_weight, ps.dipole_weight, ps.normal])).cuda()
    b, stride = src.data_ptr(), n * 24
    ptrs = (b, b + stride, b + 2 * stride, b + 3 * stride)
    dtg = torch.from_numpy(tg).cuda() if tg is not None else None
    prm = S.TreecodeParams(order=order, theta=theta, leaf_capacity=n0)
    stream = torch.cuda.current_stream().cuda_stream
    torig = torch.empty(nt, dtype=torch.int32, device="cuda")
    part = torch.zeros((nt, 3), dtype=torch.float64, device="cuda")
    ranges = []
    for r in range(world):
        t0, t1, _ = S.treecode_shard_device(*ptrs, n, prm, part.data_ptr(), torig.data_ptr(),
                                            targets_ptr=None if dtg is None else dtg.data_ptr(),
                                            n_targets=0 if dtg is None else nt, shard=r, n_shards=world,
                                            stream=stream)
        ranges.append((t0, t1))
    torch.cuda.synchronize()
    xyz = ps.position if tg is None else tg
    order_ = M.key_batch_order(xyz)
    assert np.array_equal(torig.cpu().numpy().astype(np.int64), order_)
    d = as_dict(ps)
    T = O.or_build_tree(d, n0, True)
    if tg is None:
        to_tree = np.empty(n, np.uint32)
        to_tree[T.to_original] = np.arange(n, dtype=np.uint32)
        far, near = O.or_lists(d, n0, True, theta, tree_idx=to_tree, cap=8192)
    else:
        far, near = O.or_lists(d, n0, True, theta, xyz=tg, cap=8192)
    cost = M.warp_costs(order_, far, near, (T.end - T.begin), order + 2)
    cuts = S.shard_cuts(cost, world)
    want = [(min(nt, 32 * int(cuts[r])), min(nt, 32 * int(cuts[r + 1]))) for r in range(world)]
    assert ranges == want
