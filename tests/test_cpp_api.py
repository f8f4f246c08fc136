"""The SPEC-named C++ API (include/stokesmg/solver.hpp) compiled with g++ against libsmg.so,
as a caller of the reference's stokesmg namespace would use it (SPEC:45, 121, 203, 212, 311,
361, 370, 422): host-side domain checks on CPU; on the GPU, BASELINE config 0 solved through
build_hierarchy / sqmr_solve and compared with the committed oracle golden bit for bit."""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_2312_10615_b200 as smg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    smg.lib()  # libsmg.so built
    out = str(tmp_path_factory.mktemp("cpp") / "solver_api_test")
    libdir = os.path.dirname(smg.LIB_PATH)
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                           "-o", out, os.path.join(ROOT, "tests", "cpp", "solver_api_test.cpp"), "-L", libdir, "-lsmg",
                           f"-Wl,-rpath,{libdir}"])
    return out


def test_cpp_api_host(binary):
    r = subprocess.run([binary], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "host checks ok" in r.stdout


@pytest.mark.gpu
def test_cpp_api_solves_cfg0_like_the_golden(binary):
    r = subprocess.run([binary, "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    got = json.loads(r.stdout.strip().splitlines()[-1])
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "cfg0_history.json")))
    assert got["status"] == g["status"] == 0
    assert got["history"] == g["history"]  # bit-identical (the oracle's canonical reductions)
    assert abs(got["u_norm"] - g["u_norm"]) <= 1e-12 * g["u_norm"]
    assert np.all(np.diff(np.log(got["history"])) < 1.5)


@pytest.mark.gpu
def test_cpp_api_labelled_domain(binary):
    """build_hierarchy on a CellGrid with Dirichlet and Exterior cells through the C++ API."""
    r = subprocess.run([binary, "gpu_labeled"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "labelled ok" in r.stdout
