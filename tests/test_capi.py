"""CPU: the C-ABI library loads, exports every symbol include/stokestree_c.h declares,
and its host-only logic (validation, generators, shard planning) behaves like the
reference -- no compute call needs a GPU here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stokestree_c.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(st_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_what_the_package_binds(S):
    assert sorted(S.EXPORTED_SYMBOLS) == declared_symbols()


def test_library_exports_every_declared_symbol(S):
    lib = C.CDLL(S.lib_path)
    missing = [name for name in declared_symbols() if not hasattr(lib, name)]
    assert not missing, missing
    assert lib.st_abi_version() == 1


def test_library_is_sm100a_only():
    # the product .so carries sm_100a SASS and no other architecture
    import subprocess
    lib = os.path.join(ROOT, "paper_1811_12498_b200", "libstokestree_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


@pytest.mark.parametrize("kw,msg", [
    (dict(theta=1.0), "theta must lie strictly in (0,1)"),
    (dict(theta=0.0), "theta must lie strictly in (0,1)"),
    (dict(order=-1), "order must be in [0, 16]"),
    (dict(order=17), "order must be in [0, 16]"),
    (dict(leaf_capacity=0), "leaf capacity must be >= 1"),
    (dict(workers=0), "workers must be >= 1"),
    (dict(devices=0), "devices must be >= 1"),
])
def test_params_validation_matches_reference(S, kw, msg):
    # engine.hpp:31-41 (test_engine.cpp:139-161)
    with pytest.raises(S.InvalidArgument, match=re.escape(msg)):
        S.TreecodeParams(**kw).validate()


def test_params_validation_kernel_selection(S):
    with pytest.raises(S.InvalidArgument, match="at least one kernel"):
        S.TreecodeParams(kernels=S.KernelSelection(False, False)).validate()
    S.TreecodeParams().validate()
    S.TreecodeParams(order=16, theta=0.999, leaf_capacity=1).validate()


def test_shape_validation_before_device(S):
    # particles.hpp:41-55: these checks happen on the host, before any device work
    with pytest.raises(S.InvalidArgument, match="particle set is empty"):
        S.treecode_velocity(S.ParticleSet(np.zeros((0, 3))), S.TreecodeParams())
    ps = S.ParticleSet(np.zeros((5, 3)), np.zeros((5, 3)))
    with pytest.raises(S.InvalidArgument, match="dipole_weight"):
        S.treecode_velocity(ps, S.TreecodeParams())  # stresslets on, h missing
    with pytest.raises(S.InvalidArgument, match="bad target range"):
        S.contracted_direct_velocity(ps, S.KernelSelection.stokeslet_only(), 3, 2)
    with pytest.raises(S.InvalidArgument, match="out of range"):
        S.contracted_direct_velocity_at(ps, S.KernelSelection.stokeslet_only(), [7])


def test_taylor_coeffs_validation_before_device(S):
    # taylor_coeffs.hpp:15-19, 32-36 (depth guards) and coulomb zero displacement
    with pytest.raises(S.InvalidArgument, match="not deep enough"):
        S.taylor_coeffs([[1.0, 1, 0]], 3, stokeslet=True, stresslet=False, pmax_b=3)
    with pytest.raises(S.InvalidArgument, match="not deep enough"):
        S.taylor_coeffs([[1.0, 1, 0]], 2, stokeslet=False, stresslet=True, pmax_b=3)
    with pytest.raises(S.DomainError):
        S.taylor_coeffs([[0.0, 0, 0]], 1)
    with pytest.raises(S.InvalidArgument):
        S.taylor_coeffs([[1.0, 0, 0]], 1, b=np.zeros((1, 7)))  # 7 is not E(p)


def test_compute_fails_loudly_without_gpu(S):
    if S.device_count() > 0:
        pytest.skip("a GPU is present")
    ps = S.generate("cube", 100, 1, True)
    with pytest.raises(S.StokesTreeError, match="no CPU fallback"):
        S.treecode_velocity(ps, S.TreecodeParams())
    with pytest.raises(S.StokesTreeError, match="no CPU fallback"):
        S.contracted_direct_velocity(ps, S.KernelSelection.both())
    with pytest.raises(S.StokesTreeError, match="no CPU fallback"):
        S.build_tree(ps, 10, True)
    with pytest.raises(S.StokesTreeError, match="no CPU fallback"):
        S.taylor_coeffs([[1.0, 0, 0]], 2)


def test_generators_follow_splitmix_recipe(S, O):
    # rng.hpp:10-29 + testutil::random_particles draw order (test_helpers.hpp:31-49)
    ps = S.generate("unit", 300, 7, True)
    py = O.random_particles_py(300, 7, True)
    for k in ("position", "force_weight", "dipole_weight", "normal"):
        assert np.array_equal(getattr(ps, k), py[k]), k
    cube = S.generate("cube", 300, 7, True)
    assert np.array_equal(cube.position, py["position"] - 0.5)
    assert np.array_equal(cube.normal, py["normal"])
    st = S.generate("unit", 50, 7, False)
    py2 = O.random_particles_py(50, 7, False)
    assert np.array_equal(st.position, py2["position"]) and st.dipole_weight is None


def test_generators_contracts(S):
    sph = S.generate("sphere", 2000, 3, True)
    assert np.allclose(np.linalg.norm(sph.position, axis=1), 1.0, atol=1e-15)
    assert np.array_equal(sph.position, sph.normal)
    mix = S.generate("mixture", 4000, 3, True)
    assert np.allclose(np.linalg.norm(mix.normal, axis=1), 1.0, atol=1e-14)
    pts = S.generate("points", 1000, 67890)
    assert pts.force_weight is None and pts.position.min() >= -0.5 and pts.position.max() < 0.5
    a = S.generate("mixture", 1000, 11, True)
    b = S.generate("mixture", 1000, 11, True)
    assert a.position.tobytes() == b.position.tobytes()


def test_shard_cuts(S):
    rng = np.random.default_rng(0)
    for n, k in ((1000, 8), (7, 3), (5, 8), (0, 2), (1, 1)):
        w = rng.uniform(0, 10, n)
        cuts = S.shard_cuts(w, k)
        assert cuts[0] == 0 and cuts[-1] == n and np.all(np.diff(cuts) >= 0)
        if n >= 100:
            parts = [w[cuts[i]:cuts[i + 1]].sum() for i in range(k)]
            assert max(parts) <= w.sum() / k + w.max()
    # identical on every call (ranks agree without communication)
    w = rng.uniform(0, 1, 5000)
    assert np.array_equal(S.shard_cuts(w, 4), S.shard_cuts(w.copy(), 4))


def test_relative_error_host(S):
    ref = np.array([[1, 0, 0], [0, 1, 0.0]])
    assert S.relative_error(ref, ref) == 0.0
    assert S.relative_error(ref, np.zeros((2, 3))) == 1.0
    with pytest.raises(S.DomainError):
        S.relative_error(np.zeros((1, 3)), np.ones((1, 3)))
    with pytest.raises(S.InvalidArgument):
        S.relative_error(ref[:1], ref)


def test_bench_relaunch_command_is_torchrun_with_n_ranks():
    """bench.py --gpus N (N > 1) without torchrun re-launches itself with N ranks."""
    import sys
    import bench
    cmd = bench.relaunch_command(["--gpus", "4", "--steps", "2"], 4, 29555)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[cmd.index(bench.__file__.replace(".pyc", ".py")) + 1:] == ["--gpus", "4", "--steps", "2"]


def test_bench_far_flop_conventions():
    import bench
    # SURVEY.md 8d table (reference-equivalent flops per accepted pair)
    assert [bench.f_far(p) for p in (2, 4, 6, 8, 10)] == [2278, 7527, 17640, 34209, 58826]
    # executed flops at P = 10 (p = 8 with stresslets), as counted in the SASS
    assert bench.far_executed_flops(10) == 1226
    assert bench.f_far(8) / bench.far_executed_flops(10) == pytest.approx(27.9, abs=0.05)


def test_nccl_unique_id_without_a_gpu():
    """NCCL inside the library is loaded at first use (dlopen): the id of a new communicator
    can be made on a host without a GPU."""
    import paper_1811_12498_b200 as S
    a, b = S.nccl_unique_id(), S.nccl_unique_id()
    assert len(a) == 128 and len(b) == 128 and a != b
