"""The C++ drop-in shim (include/bitonic/gpu_sort.hpp) compiled with g++ and
run against the native library: the reference's call shapes and exception
types (test_engine.cpp:217-253, :439-449)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _compile(tmp_path, with_reference_headers):
    from paper_1506_01446_b200 import build
    lib = build.build()
    exe = str(tmp_path / ("shim_ref" if with_reference_headers else "shim"))
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include")]
    if with_reference_headers:
        cmd += ["-I", "/root/reference/proj/include"]
    cmd += [os.path.join(ROOT, "tests", "cpp", "test_gpu_sort.cpp"), lib,
            "-Wl,-rpath," + os.path.dirname(lib), "-o", exe]
    subprocess.run(cmd, check=True)
    return exe


def test_shim_compiles_standalone(tmp_path):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    _compile(tmp_path, False)


def test_shim_compiles_with_reference_error_types(tmp_path):
    if not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("reference headers not present")
    _compile(tmp_path, True)


@pytest.mark.gpu
def test_shim_runs_on_gpu(tmp_path):
    exe = _compile(tmp_path, False)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "OK" in r.stdout
