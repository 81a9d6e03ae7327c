"""The C++ drop-in headers compile and link against the reference's call sites
(tests/cpp/dropin_test.cpp) and run the reference's unit tests restated case by case
(tests/cpp/reference_suite.cpp) -- host checks on CPU, the full programs on a B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1811_12498_b200")


def compile_cpp(tmp_path_factory, name):
    exe = str(tmp_path_factory.mktemp("cpp") / name)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", name + ".cpp"), "-L", LIBDIR, "-lstokestree_b200",
           f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return exe


@pytest.fixture(scope="module")
def dropin_exe(tmp_path_factory):
    return compile_cpp(tmp_path_factory, "dropin_test")


@pytest.fixture(scope="module")
def suite_exe(tmp_path_factory):
    return compile_cpp(tmp_path_factory, "reference_suite")


def test_dropin_compiles_and_host_checks_pass(dropin_exe):
    out = subprocess.run([dropin_exe, "host"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.gpu
def test_dropin_full_program_on_gpu(dropin_exe):
    out = subprocess.run([dropin_exe, "all"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr


def test_reference_suite_host_cases(suite_exe):
    out = subprocess.run([suite_exe, "host"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.gpu
def test_reference_suite_all_cases_on_gpu(suite_exe):
    out = subprocess.run([suite_exe, "all"], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout + out.stderr
