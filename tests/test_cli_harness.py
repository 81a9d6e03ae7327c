"""The reference's harness contract (bench.hpp run()/CSV, tools/stokestree_cli.cpp flags)
over the B200 path: argument handling on CPU, report rows on a B200."""
import csv
import io
import os
import subprocess

import numpy as np
import pytest

from conftest import as_dict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "stokestree")
HEADER = "N,p,theta,n0,workers,time_direct_s,time_tree_s,speedup,error_E,farfield_evals,direct_evals"


@pytest.fixture(scope="module")
def cli():
    out = subprocess.run(["make", "-C", os.path.join(ROOT, "tools")], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return CLI


def run(cli, *args, timeout=600):
    return subprocess.run([cli, *args], capture_output=True, text=True, timeout=timeout)


def test_cli_argument_errors_exit_1(cli):
    # the reference maps invalid_argument to exit 1 (stokestree_cli.cpp:109-115)
    for args in (["--testcase", "cube"], ["--testcase", "sphere"], ["--testcase", "bogus"],
                 ["--n", "10", "--theta", "1.0"], ["--n", "10", "--order", "17"], ["--n", "x"],
                 ["--unknown", "1"], ["--n"]):
        r = run(cli, *args)
        assert r.returncode == 1, (args, r.stdout, r.stderr)
        assert r.stderr.startswith("error: ")
    r = run(cli, "--help")
    assert r.returncode == 0 and "--direct-sample" in r.stdout


@pytest.mark.gpu
def test_cli_cube_csv_row_matches_reference(cli, S, need_ref):
    r = run(cli, "--testcase", "cube", "--n", "20000", "--seed", "5", "--order", "6", "--theta", "0.5",
            "--n0", "500", "--format", "csv")
    assert r.returncode == 0, r.stderr
    rows = list(csv.reader(io.StringIO(r.stdout)))
    assert ",".join(rows[0]) == HEADER and len(rows) == 2
    row = dict(zip(rows[0], rows[1]))
    # the same particles (testcases.hpp cube, Stokeslet only, shrink auto = off) on the reference
    ps = S.cube_particles(20000, 2500.0, 5)
    u_ref, st_ref, _ = need_ref.ref_parallel_velocity(as_dict(ps), 6, 0.5, 500, shrink=False, sto=True,
                                                      stre=False, workers=8)
    assert int(row["farfield_evals"]) == st_ref["farfield_evals"]
    assert int(row["direct_evals"]) == st_ref["direct_pairs"]
    direct = need_ref.ref_direct_at(as_dict(ps), np.arange(20000), True, False)
    e_ref = S.relative_error(direct, u_ref)
    assert abs(float(row["error_E"]) - e_ref) <= 0.01 * e_ref
    assert float(row["speedup"]) > 0 and float(row["time_tree_s"]) > 0


@pytest.mark.gpu
def test_cli_sphere_human_and_file_round_trip(cli, tmp_path):
    dump = tmp_path / "sphere.txt"
    r = run(cli, "--testcase", "sphere", "--levels", "4", "--seed", "11", "--order", "10", "--theta", "0.2",
            "--direct-sample", "500", "--dump-particles", str(dump))
    assert r.returncode == 0, r.stderr
    assert "extrapolated from 500 sampled targets" in r.stdout
    e = float([ln for ln in r.stdout.splitlines() if ln.startswith("error E")][0].split()[-1])
    assert e < 1e-9  # test_engine.cpp:95-105 (p = 10, theta = 0.2 on the L = 4 sphere)
    r2 = run(cli, "--testcase", "file", "--input", str(dump), "--order", "10", "--theta", "0.2", "--shrink", "on",
             "--direct-sample", "500", "--format", "csv", "--out", str(tmp_path / "o.csv"))
    assert r2.returncode == 0, r2.stderr
    rows = list(csv.reader(open(tmp_path / "o.csv")))
    assert abs(float(dict(zip(rows[0], rows[1]))["error_E"]) - e) <= 1e-5 * e  # human report: 6 digits


def _build_harness_bytes(tmp_path, include_dir, link_product):
    exe = tmp_path / ("hb_" + ("mine" if link_product else "ref"))
    cmd = ["g++", "-std=c++20", "-O1", "-I" + include_dir, "-o", str(exe),
           os.path.join(ROOT, "tests", "cpp", "harness_bytes.cpp")]
    if link_product:
        libdir = os.path.join(ROOT, "paper_1811_12498_b200")
        cmd += ["-L" + libdir, "-lstokestree_b200", "-Wl,-rpath," + libdir]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return str(exe)


def test_harness_renderings_match_reference_bytes(tmp_path):
    """write_csv / read_csv (incl. every error) / write_human of the drop-in harness produce
    the reference's bytes (golden: tests/cpp/harness_bytes.cpp compiled against the
    reference's bench.hpp, tests/golden/harness_bytes.txt).  Host-only."""
    exe = _build_harness_bytes(tmp_path, os.path.join(ROOT, "include"), True)
    mine = subprocess.run([exe], capture_output=True, check=True).stdout
    golden = open(os.path.join(ROOT, "tests", "golden", "harness_bytes.txt"), "rb").read()
    assert mine == golden
    ref_inc = "/root/reference/proj/include"
    if os.path.isdir(ref_inc):  # regenerate the golden from the reference itself
        ref = subprocess.run([_build_harness_bytes(tmp_path, ref_inc, False)], capture_output=True,
                             check=True).stdout
        assert ref == golden
