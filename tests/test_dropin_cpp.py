"""The C++ drop-in headers compile and link against the reference's call sites
(tests/cpp/dropin_test.cpp) -- host checks on CPU, the full program on a B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1811_12498_b200")


@pytest.fixture(scope="module")
def dropin_exe(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("cpp") / "dropin_test")
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp"), "-L", LIBDIR, "-lstokestree_b200",
           f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return exe


def test_dropin_compiles_and_host_checks_pass(dropin_exe):
    out = subprocess.run([dropin_exe, "host"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.gpu
def test_dropin_full_program_on_gpu(dropin_exe):
    out = subprocess.run([dropin_exe, "all"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
