"""CPU: the static synchronisation / partition proof obligations of the
kernels (tests/cpp/check_sync.cu, the analogue of the reference's
disjointness check test_engine.cpp:395-437).  compute-sanitizer is not
available on this pool's GPUs (its runs are refused), so race freedom is
shown by construction: layouts are bijections onto distinct shared-memory
words, every __syncwarp-only transition keeps each warp's words, the cluster
exchange reads each key once, and every pass's cosets partition the array."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_layouts_transitions_and_cosets(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = str(tmp_path / "check_sync")
    subprocess.run([nvcc, "-std=c++17", "-O2", "--expt-relaxed-constexpr", "-diag-suppress", "128",
                    "-gencode", "arch=compute_100a,code=sm_100a", "-o", exe,
                    os.path.join(ROOT, "tests", "cpp", "check_sync.cu")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:])
    assert r.returncode == 0 and r.stdout.strip().splitlines()[-1].startswith("OK")
