"""CPU: the paper's test geometries and the particle text format,
checked against the reference's own generators / reader / writer compiled in place."""
import os

import numpy as np
import pytest

from conftest import as_dict


@pytest.mark.parametrize("levels,seed", [(0, 5150), (2, 7), (4, 314159)])
def test_sphere_geometry_bit_identical(S, need_ref, levels, seed):
    mine = S.sphere_particles(levels, seed)
    ref = need_ref.ref_sphere_particles(levels, seed)
    assert mine.size() == 20 * 4 ** levels
    for k in ("position", "force_weight", "dipole_weight", "normal"):
        assert getattr(mine, k).tobytes() == ref[k].tobytes(), k
    # acceptance criterion 8 contracts (acceptance.cpp:269-305)
    assert np.abs(np.linalg.norm(mine.position, axis=1) - 1.0).max() <= 1e-14


@pytest.mark.parametrize("n,density,seed", [(12345, 2500.0, 99), (40000, 2500.0, 1618), (10, 1.0, 0)])
def test_cube_geometry_bit_identical(S, need_ref, n, density, seed):
    mine = S.cube_particles(n, density, seed)
    ref = need_ref.ref_cube_particles(n, density, seed)
    assert mine.position.tobytes() == ref["position"].tobytes()
    assert mine.force_weight.tobytes() == ref["force_weight"].tobytes()
    side = (n / density) ** (1 / 3)
    assert mine.position.min() >= 0 and mine.position.max() <= side
    assert mine.dipole_weight is None and mine.normal is None


def test_geometry_guards(S):
    with pytest.raises(S.InvalidArgument):
        S.sphere_particles(-1, 0)
    with pytest.raises(S.InvalidArgument):
        S.cube_particles(0)
    with pytest.raises(S.InvalidArgument):
        S.cube_particles(10, density=0.0)


@pytest.mark.parametrize("sel", ["both", "stokeslet_only", "stresslet_only"])
def test_particle_file_round_trip_and_reference_compat(S, need_ref, tmp_path, sel):
    # test_harness.cpp:62-118: bit-exact round trip, header per selection
    k = getattr(S.KernelSelection, sel)()
    ps = S.generate("unit", 64, 1234, True)
    mine_path, ref_path = tmp_path / "mine.txt", tmp_path / "ref.txt"
    S.write_particles(mine_path, ps, k)
    need_ref.ref_write_particles(ref_path, as_dict(ps), k.stokeslet_enabled, k.stresslet_enabled)
    assert mine_path.read_bytes() == ref_path.read_bytes()  # identical files
    back, ksel = S.read_particles(ref_path)
    assert ksel == k
    assert back.position.tobytes() == ps.position.tobytes()
    if k.stokeslet_enabled:
        assert back.force_weight.tobytes() == ps.force_weight.tobytes()
    else:
        assert back.force_weight is None
    if k.stresslet_enabled:
        assert back.dipole_weight.tobytes() == ps.dipole_weight.tobytes()
        assert back.normal.tobytes() == ps.normal.tobytes()
    ref_back = need_ref.ref_read_particles(mine_path, 64)
    assert ref_back["position"].tobytes() == ps.position.tobytes()


def test_particle_file_errors(S, tmp_path):
    # test_harness.cpp:122-161
    bad = tmp_path / "bad.txt"
    bad.write_text("x f\n0 0 0 1 1 1\n1 2 3 4 5\n")
    with pytest.raises(S.StokesTreeError, match="line 3"):
        S.read_particles(bad)
    with pytest.raises(S.StokesTreeError, match="cannot open"):
        S.read_particles(tmp_path / "missing.txt")
    hdr = tmp_path / "hdr.txt"
    hdr.write_text("x h\n0 0 0 1 1 1\n")
    with pytest.raises(S.StokesTreeError, match="must appear together"):
        S.read_particles(hdr)
    trail = tmp_path / "trail.txt"
    trail.write_text("x f\n0 0 0 1 1 1 7\n")
    with pytest.raises(S.StokesTreeError, match="trailing fields"):
        S.read_particles(trail)
    ps = S.generate("unit", 8, 5, True)
    ps.normal[2] *= 2
    with pytest.raises(S.InvalidArgument, match="normal 2"):
        S.write_particles(tmp_path / "w.txt", ps, S.KernelSelection.both())
