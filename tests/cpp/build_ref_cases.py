"""Compile the REFERENCE'S OWN C++ test cases for the hot path against the
B200 drop-in header, unchanged except for where their #includes resolve.

The cases are read at build time from /root/reference (nothing is copied into
this repository): the listed line ranges of the reference's test files (the
file prelude with its includes and helpers, then whole TEST_CASEs) are
concatenated under #line directives, so a failure reports the reference's
own file:line. Their `#include "randla/<x>.hpp"` resolve to
include/randla_dropin/randla/<x>.hpp, which forward to
include/randla_b200/randla.hpp; `#include <doctest.h>` resolves to our
harness in tests/cpp/doctest_shim (the reference keeps doctest out of tree).
The binaries land in tests/cpp/_build/ (git-ignored; they travel to the GPU
box with the tree) and tests/test_cpp_api.py runs them on the GPU.

Compiled: test_transforms.cpp (all but the text-fixture case, which needs
matrix_io.hpp's file format), test_lowrank.cpp (all but the three cases
built on the full SVD with singular vectors, svd(), which the device Jacobi
does not return: lines 77-112) and the whole of test_multipliers.cpp, whose
prelude includes the reference's own tests/support/exact_rank.hpp (read in
place with -I). test_elimination.cpp is left out: its prelude needs Eigen's
inverse(); its GENP / GEPP / block / refinement cases are restated in
tests/cpp/test_header_api.cpp instead.

Usage: python tests/cpp/build_ref_cases.py   (no-op when /root/reference is absent)
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.environ.get("RANDLA_REFERENCE", "/root/reference")
OUT = os.path.join(HERE, "_build")
LIBDIR = os.path.join(ROOT, "paper_1406_5802_b200", "_lib")

# binary -> (reference test file, inclusive 1-based line ranges)
CASES = {
    "ref_transforms": ("proj/tests/test_transforms.cpp", [(1, 29), (31, 211), (230, 239)]),
    "ref_lowrank": ("proj/tests/test_lowrank.cpp", [(1, 18), (20, 75), (114, 170), (172, 228), (230, 265)]),
    "ref_multipliers": ("proj/tests/test_multipliers.cpp", [(1, 262)]),
}


def assemble(rel, ranges):
    path = os.path.join(REF, rel)
    with open(path) as f:
        lines = f.read().split("\n")
    out = []
    for a, b in ranges:
        out.append(f'#line {a} "{path}"')
        out.extend(lines[a - 1:b])
    return "\n".join(out) + "\n"


def build(verbose=False):
    if not os.path.isdir(os.path.join(REF, "proj", "tests")):
        if verbose:
            print("reference tests not present: skipping the reference C++ cases")
        return []
    os.makedirs(OUT, exist_ok=True)
    built = []
    import tempfile
    tmp = tempfile.mkdtemp(prefix="randla_ref_cases_")  # the assembled source never lands in the tree
    for name, (rel, ranges) in CASES.items():
        src = os.path.join(tmp, name + ".cpp")
        with open(src, "w") as f:
            f.write(assemble(rel, ranges))
        exe = os.path.join(OUT, name)
        cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include", "randla_dropin"),
               "-I", os.path.join(ROOT, "include"), "-I", os.path.join(HERE, "doctest_shim"),
               # the reference's own test-support headers (support/exact_rank.hpp), read in place
               "-I", os.path.join(REF, "proj", "tests"), src,
               "-L", LIBDIR, "-lrandla_b200", "-Wl,-rpath,$ORIGIN/../../../paper_1406_5802_b200/_lib", "-o", exe]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"reference cases {name} do not compile against the drop-in:\n{r.stderr[-4000:]}")
        built.append(exe)
        os.remove(src)
    os.rmdir(tmp)
    return built


if __name__ == "__main__":
    print("\n".join(build(verbose=True)))
