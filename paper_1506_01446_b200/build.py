"""Build the in-tree sm_100a shared library (libb200_bitonic.so).

nvcc cross-compiles for sm_100a without a GPU; the .so is git-ignored but
travels to the GPU box with the repo snapshot.  The specialised kernels are
split over several translation units that compile in parallel.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# Experiment hooks: B200_BITONIC_OBJ / B200_BITONIC_LIBOUT redirect the object
# directory and the library; B200_BITONIC_EXTRA_NVCC adds flags (e.g. -D...).
OBJ = os.environ.get("B200_BITONIC_OBJ") or os.path.join(ROOT, "build", "obj")
LIB = os.environ.get("B200_BITONIC_LIBOUT") or os.path.join(HERE, "libb200_bitonic.so")
SOURCES = [os.path.join(CSRC, f) for f in
           ["bitonic_sort.cu", "k_tile.cu", "k_merge11.cu", "k_merge12.cu",
            "k_merge13.cu", "k_merge14.cu", "k_merge15.cu", "k_merge12r4.cu",
            "k_merge13r4.cu", "k_merge14r4.cu", "k_merge12kv.cu", "k_merge13kv.cu",
            "k_merge12k64.cu", "k_merge13k64.cu", "k_tile_k64.cu", "k_cluster.cu", "k_tile_tma.cu", "k_virt.cu",
            "host_entry.cu", "multi.cu"]]
HEADERS = [os.path.join(CSRC, f) for f in os.listdir(CSRC)
           if f.endswith((".cuh", ".hpp", ".h"))]
HEADERS.append(os.path.join(ROOT, "include", "b200_bitonic.h"))

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-diag-suppress", "128", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-warn-spills"] + os.environ.get("B200_BITONIC_EXTRA_NVCC", "").split()


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _obj(src: str) -> str:
    return os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def needs_build() -> bool:
    if not all(os.path.exists(_obj(s)) for s in SOURCES):
        return True
    return _stale(LIB, SOURCES + HEADERS + [_obj(s) for s in SOURCES])


# The race-stress variant (-DB200_JITTER: random sleeps at every shared-
# memory hand-off, bitonic_static.cuh jitter()) used by tests/test_gpu_jitter.py.
JITTER_OBJ = os.path.join(ROOT, "build", "obj_jitter")
JITTER_LIB = os.path.join(HERE, "libb200_bitonic_jitter.so")


def build_jitter(verbose: bool = False) -> str:
    global OBJ, LIB
    saved = (OBJ, LIB, list(NVCC_FLAGS))
    OBJ, LIB = JITTER_OBJ, JITTER_LIB
    NVCC_FLAGS.append("-DB200_JITTER")
    try:
        return build(verbose=verbose)
    finally:
        OBJ, LIB = saved[0], saved[1]
        NVCC_FLAGS[:] = saved[2]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    nv = nvcc()
    jobs = []
    for src in SOURCES:
        obj = _obj(src)
        if force or _stale(obj, [src] + HEADERS):
            jobs.append([nv, *NVCC_FLAGS, "-c", "-o", obj, src])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout + r.stderr, flush=True)

    with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4) or 1) as ex:
        list(ex.map(run, jobs))
    run([nv, *ARCH, "-shared", "-o", LIB, *[_obj(s) for s in SOURCES]])
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(LIB)
