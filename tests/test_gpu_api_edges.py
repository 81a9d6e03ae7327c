"""GPU edge cases of the drop-in API: error messages and their order (the reference's
throw order), empty shards, and the library's device-memory lifetime."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_naive_coincident_message_follows_kernel_selection(S):
    # naive_direct_velocity forms the Stokeslet first, so with stresslets only the
    # reference throws stresslet()'s message (kernels.hpp:17, 31, 98-112)
    pos = np.array([[0, 0, 0], [1, 1, 1], [0, 0, 0.0]])
    one = np.tile([1.0, 0, 0], (3, 1))
    ps = S.ParticleSet(pos, one, one, one)
    with pytest.raises(S.DomainError, match="^stokeslet: coincident points$"):
        S.naive_direct_velocity(ps, S.KernelSelection.both())
    with pytest.raises(S.DomainError, match="^stresslet: coincident points$"):
        S.naive_direct_velocity(ps, S.KernelSelection.stresslet_only())
    with pytest.raises(S.DomainError, match="^direct sum: coincident particles$"):
        S.contracted_direct_velocity(ps, S.KernelSelection.stresslet_only())


def test_direct_validates_values_before_the_target_range(S):
    # contracted_direct_velocity[_at] call validate(ps, sel) before the range / index
    # checks (kernels.hpp:125-127, 143-146)
    ps = S.generate("cube", 50, 3, True)
    bad = S.ParticleSet(ps.position.copy(), ps.force_weight, ps.dipole_weight, ps.normal.copy())
    bad.normal[4] *= 3.0
    with pytest.raises(S.InvalidArgument, match="normal 4 is not unit length"):
        S.contracted_direct_velocity(bad, S.KernelSelection.both(), 10, 5)
    with pytest.raises(S.InvalidArgument, match="normal 4 is not unit length"):
        S.contracted_direct_velocity_at(bad, S.KernelSelection.both(), [51])
    with pytest.raises(S.InvalidArgument, match="bad target range"):
        S.contracted_direct_velocity(ps, S.KernelSelection.both(), 10, 5)
    with pytest.raises(S.InvalidArgument, match="target out of range"):
        S.contracted_direct_velocity_at(ps, S.KernelSelection.both(), [51])


@pytest.mark.parametrize("nt", [1, 31, 100, 255])
def test_empty_shards_with_many_devices(S, nt):
    # fewer 32-target batch warps than shards: some shards are empty and must still order
    # their frees and timings after the moment pass (capi.cu run_treecode)
    ps = S.generate("cube", 20000, 11, True)
    tg = S.generate("points", nt, 67890).position
    prm1 = S.TreecodeParams(order=5, theta=0.5, leaf_capacity=300)
    one = S.treecode_velocity_targets(ps, tg, prm1, per_target=True)
    for dev in (3, 8):
        prm = S.TreecodeParams(order=5, theta=0.5, leaf_capacity=300, devices=dev)
        many = S.treecode_velocity_targets(ps, tg, prm, per_target=True)
        assert many.velocity.tobytes() == one.velocity.tobytes()
        assert np.array_equal(many.per_target, one.per_target)
        assert many.time_moments_s >= 0.0 and many.time_total_s > 0.0


def test_release_workspace_returns_memory_and_calls_still_work(S):
    import torch
    ps = S.generate("cube", 200000, 5, True)
    prm = S.TreecodeParams(order=4, theta=0.5, leaf_capacity=1000)
    a = S.treecode_velocity(ps, prm).velocity
    free_before, _ = torch.cuda.mem_get_info()
    S.release_workspace()
    free_after, _ = torch.cuda.mem_get_info()
    assert free_after >= free_before  # the pool and the near workspace were trimmed
    b = S.treecode_velocity(ps, prm).velocity
    assert a.tobytes() == b.tobytes()
    S.release_workspace()


def test_default_pool_is_not_reconfigured(S):
    # the library allocates from a private pool: the process's default pool keeps its
    # release threshold (0 unless the host application changed it)
    from cuda.bindings import runtime as rt
    ps = S.generate("cube", 5000, 5, True)
    S.treecode_velocity(ps, S.TreecodeParams(order=3, leaf_capacity=200))
    err, pool = rt.cudaDeviceGetDefaultMemPool(0)
    assert err == rt.cudaError_t.cudaSuccess
    err, thr = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold)
    assert err == rt.cudaError_t.cudaSuccess
    assert int(thr) == 0


DEBUG_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1811_12498_b200 as S
out = []
for kind, n, n0, theta, disjoint in (("cube", 30000, 200, 0.5, False), ("sphere", 20000, 1, 0.7, False),
                                     ("mixture", 30000, 100, 0.6, True), ("unit", 5000, 8, 0.9, False)):
    ps = S.generate(kind, n, 3, True)
    tg = S.generate("points", 4000, 67890).position if disjoint else None
    r = S.treecode_velocity_targets(ps, tg, S.TreecodeParams(order=4, theta=theta, leaf_capacity=n0))
    out.append(r.velocity)
np.save(sys.argv[2], np.concatenate(out))
"""


def test_debug_build_mac_containment_check(S, tmp_path):
    """`make debug` compiles the reference's MAC self-containment assert (engine.hpp:88-89) into
    the walk kernel (ST_DEBUG_CHECKS; a violation fails the call with ST_RUNTIME_ERROR).  The
    debug library runs clean on trees down to N0 = 1 and theta up to 0.9, bit-identical to
    the release library."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    dbg = os.path.join(root, "paper_1811_12498_b200", "libstokestree_b200_debug.so")
    if not os.path.exists(dbg):
        pytest.skip("debug library not built (make -C paper_1811_12498_b200 debug)")
    res = {}
    for tag, lib in (("release", None), ("debug", dbg)):
        env = dict(os.environ)
        if lib:
            env["ST_LIB_PATH"] = lib
        f = tmp_path / f"{tag}.npy"
        out = subprocess.run([sys.executable, "-c", DEBUG_SCRIPT, root, str(f)], env=env, capture_output=True,
                             text=True, timeout=600)
        assert out.returncode == 0, out.stderr
        res[tag] = np.load(f)
    assert res["debug"].tobytes() == res["release"].tobytes()


def _dict(ps):
    return dict(position=ps.position, force_weight=ps.force_weight, dipole_weight=ps.dipole_weight,
                normal=ps.normal)


def test_signed_zero_extremes_pinned(S, need_ref):
    """the device's order-free min/max puts -0.0 below +0.0, where the
    reference's tight_box keeps the first-seen of two equal extremes.  Pinned: the trees are
    identical except possibly in the sign of a zero bound (centre / bbox), and the
    velocities agree to 1e-12 (a signed zero never changes a distance)."""
    rng = np.random.default_rng(3)
    pos = rng.uniform(0.0, 1.0, (400, 3))
    pos[0] = [0.0, 0.3, 0.7]
    pos[1] = [-0.0, 0.6, 0.2]   # both signed zeros are the x extreme of the root
    pos[2] = [0.5, -0.0, 0.4]
    pos[3] = [0.2, 0.0, 0.9]    # and of y, in the other order
    f = rng.uniform(-1, 1, (400, 3))
    ps = S.ParticleSet(pos, f)
    sel = S.KernelSelection.stokeslet_only()
    for n0 in (1, 16, 500):
        T = S.build_tree(ps, n0, True)
        R = need_ref.RefContext(dict(position=pos, force_weight=f), 0, 0.5, n0, True, sto=True, stre=False).tree()
        assert np.array_equal(T.to_original, R.to_original)
        assert np.array_equal(T.begin, R.begin) and np.array_equal(T.end, R.end)
        assert np.array_equal(T.children, R.children)
        same_up_to_zero_sign = (T.geom == R.geom)  # -0.0 == +0.0 numerically
        assert same_up_to_zero_sign.all()
        differ = T.geom.view(np.uint64) != R.geom.view(np.uint64)
        assert np.all(T.geom[differ] == 0.0)  # only zero signs may differ
        prm = S.TreecodeParams(order=4, theta=0.5, leaf_capacity=n0, kernels=sel)
        u = S.treecode_velocity(ps, prm).velocity
        u_ref, _, _ = need_ref.ref_parallel_velocity(dict(position=pos, force_weight=f), 4, 0.5, n0, True,
                                                     sto=True, stre=False)
        assert S.relative_error(u_ref, u) <= 1e-12


def test_subnormal_distance_pinned(S, need_ref):
    """the near field tests the coincident-pair condition once per entry
    (its sums turn NaN), so a pair whose r^2 underflows to a subnormal raises domain_error on
    the device; the reference (which only tests r^2 == 0) returns inf / NaN velocities.
    Pinned on both sides."""
    rng = np.random.default_rng(4)
    pos = rng.uniform(0.0, 1.0, (50, 3))
    pos[3] = [0.0, 0.25, 0.75]
    pos[7] = [1e-160, 0.25, 0.75]  # r^2 = 1e-320: subnormal, not zero
    f = rng.uniform(-1, 1, (50, 3))
    ps = S.ParticleSet(pos, f)
    prm = S.TreecodeParams(order=3, theta=0.5, leaf_capacity=1000, kernels=S.KernelSelection.stokeslet_only())
    u_ref, _, _ = need_ref.ref_parallel_velocity(dict(position=pos, force_weight=f), 3, 0.5, 1000, True,
                                                 sto=True, stre=False)
    assert not np.isfinite(u_ref[[3, 7]]).all() and np.isfinite(np.delete(u_ref, [3, 7], axis=0)).all()
    with pytest.raises(S.DomainError):
        S.treecode_velocity(ps, prm)


OVERFLOW_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
rng = np.random.default_rng(4)
pos = rng.uniform(0.0, 1.0, (50, 3)); pos[7] = [1e155, 0.0, 0.0]   # |d|^2 = inf for every pair with it
f = rng.uniform(-1, 1, (50, 3))
if sys.argv[2] == "ref":
    from oracle import oracle as O
    O.ref_parallel_velocity(dict(position=pos, force_weight=f), 3, 0.5, 1000, True, sto=True, stre=False)
else:
    import paper_1811_12498_b200 as S
    S.treecode_velocity(S.ParticleSet(pos, f), S.TreecodeParams(order=3, theta=0.5, leaf_capacity=1000,
                                                                 kernels=S.KernelSelection.stokeslet_only()))
print("completed")
"""


def test_overflowing_distance_trips_the_mac_assert(S, need_ref):
    """|coordinates| ~ 1e155 make |d|^2 = inf, so the MAC (r_c^2 <= theta^2 |d|^2) accepts
    the root cluster, which holds the target: the reference's own assert (engine.hpp:88-89)
    aborts, and this library's debug build (ST_DEBUG_CHECKS) fails the call with the same
    message.  The release build does not check (the reference built with NDEBUG neither)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ref = subprocess.run([sys.executable, "-c", OVERFLOW_SCRIPT, root, "ref"], capture_output=True, text=True,
                         timeout=300)
    assert ref.returncode != 0 and "MAC accepted a cluster containing the target" in ref.stderr
    dbg = os.path.join(root, "paper_1811_12498_b200", "libstokestree_b200_debug.so")
    if not os.path.exists(dbg):
        pytest.skip("debug library not built")
    out = subprocess.run([sys.executable, "-c", OVERFLOW_SCRIPT, root, "gpu"], capture_output=True, text=True,
                         timeout=300, env=dict(os.environ, ST_LIB_PATH=dbg))
    assert out.returncode != 0 and "MAC accepted a cluster containing the target" in out.stderr, out.stderr
