"""The C++ drop-in header (include/randla_b200/randla.hpp) compiles and links
against librandla_b200.so (CPU); the reference-style C++ test program runs
green on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_header_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_1406_5802_b200", "_lib")


def _build(tmp_path):
    exe = str(tmp_path / "test_header_api")
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "include", "randla_b200"),
           SRC, "-L", LIBDIR, "-lrandla_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_header_compiles_and_links(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_header_program_runs(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all passed" in r.stdout
