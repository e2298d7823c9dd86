"""oracle -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

Two CPU checkers for the bitonic-sort hot path of arxiv/paper_1506_01446:

* ``Oracle``  -- ctypes view of ``oracle/liboracle.so``, a plain-C restatement
  of the reference algorithm (see bitonic_oracle.c for the file:line map).
* ``Reference`` -- ctypes view of ``oracle/_ref/libbitonic_ref.so``, the
  UNMODIFIED reference sources (/root/reference/proj/src) compiled in place by
  ``oracle/Makefile``.  Present wherever it was built (it travels to the GPU
  box as a built artefact); ``reference()`` returns None when it is absent.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package.  The product package
``paper_1506_01446_b200`` never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE_SO = os.path.join(_HERE, "liboracle.so")
_REF_SO = os.path.join(_HERE, "_ref", "libbitonic_ref.so")

_u32p = ctypes.POINTER(ctypes.c_uint32)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def build(with_reference: bool = True) -> None:
    """Compile the checkers (C restatement; the reference when its sources exist)."""
    targets = [os.path.join(_HERE, "liboracle.so")]
    subprocess.run(["make", "-s", "-C", _HERE, targets[0]], check=True)
    if with_reference and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)


def _ptr(a: np.ndarray, t):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(t)


class Oracle:
    """Plain-C restatement (bitonic_oracle.c)."""

    def __init__(self, path: str = _ORACLE_SO):
        if not os.path.exists(path):
            build(with_reference=False)
        lib = ctypes.CDLL(path)
        lib.oracle_generate_input.argtypes = [_u32p, ctypes.c_uint64, ctypes.c_uint64]
        lib.oracle_sequential_bitonic_i32.argtypes = [_i32p, ctypes.c_uint64]
        lib.oracle_bitonic_u32.argtypes = [_u32p, ctypes.c_uint64, ctypes.c_int]
        lib.oracle_bitonic_batched_u32.argtypes = [_u32p, ctypes.c_uint64,
                                                   ctypes.c_uint64, ctypes.c_int]
        lib.oracle_bitonic_pairs.argtypes = [_u32p, _u32p, ctypes.c_uint64, ctypes.c_int,
                                             ctypes.c_uint32]
        lib.oracle_bitonic_u64.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int,
                                           ctypes.c_uint64]
        lib.oracle_quicksort_i32.argtypes = [_i32p, ctypes.c_uint64]
        lib.oracle_quicksort_i32.restype = None
        lib.oracle_quicksort_u32.argtypes = [_u32p, ctypes.c_uint64, ctypes.c_int]
        lib.oracle_quicksort_u32.restype = None
        lib.oracle_predicted_counts.argtypes = [ctypes.c_uint, _u64p, _u64p]
        lib.oracle_fnv1a64.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        lib.oracle_fnv1a64.restype = ctypes.c_uint64
        lib.oracle_pad_to_pow2_i32.argtypes = [_i32p, ctypes.c_uint64, _i32p]
        lib.oracle_pad_to_pow2_i32.restype = ctypes.c_uint64
        lib.oracle_first_violation_u32.argtypes = [_u32p, ctypes.c_uint64, ctypes.c_int]
        lib.oracle_first_violation_u32.restype = ctypes.c_uint64
        self.lib = lib

    # generate_input (bench.cpp:354-364), as uint32 bits
    def generate_input(self, n: int, seed: int = 1) -> np.ndarray:
        out = np.empty(n, dtype=np.uint32)
        rc = self.lib.oracle_generate_input(_ptr(out, _u32p), n, seed)
        if rc:
            raise ValueError("invalid size")
        return out

    def sequential_bitonic_i32(self, keys: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(keys, dtype=np.int32).copy()
        if self.lib.oracle_sequential_bitonic_i32(_ptr(a, _i32p), a.size):
            raise ValueError("length must be a power of two >= 2")
        return a

    def bitonic_u32(self, keys: np.ndarray, descending: bool = False) -> np.ndarray:
        a = np.ascontiguousarray(keys, dtype=np.uint32).copy()
        if self.lib.oracle_bitonic_u32(_ptr(a, _u32p), a.size, int(descending)):
            raise ValueError("length must be a power of two >= 2")
        return a

    def bitonic_batched_u32(self, keys: np.ndarray, n_per: int,
                            descending: bool = False) -> np.ndarray:
        a = np.ascontiguousarray(keys, dtype=np.uint32).copy()
        if self.lib.oracle_bitonic_batched_u32(_ptr(a, _u32p), n_per,
                                               a.size // n_per, int(descending)):
            raise ValueError("length must be a power of two >= 2")
        return a

    def bitonic_pairs(self, keys: np.ndarray, values: np.ndarray, descending: bool = False):
        """The reference network with a payload moved on every swap.  keys may
        be int32 (signed order) or uint32."""
        kx = 0x80000000 if keys.dtype == np.int32 else 0
        k = np.ascontiguousarray(keys).view(np.uint32).copy()
        v = np.ascontiguousarray(values, dtype=np.uint32).copy()
        if self.lib.oracle_bitonic_pairs(_ptr(k, _u32p), _ptr(v, _u32p), k.size,
                                         int(descending), kx):
            raise ValueError("length must be a power of two >= 2")
        return k.view(keys.dtype), v

    def bitonic_64(self, keys: np.ndarray, descending: bool = False) -> np.ndarray:
        """The reference network on int64 / uint64 / float64 keys (float64 in
        IEEE totalOrder, -NaN < -inf < ... < -0.0 < +0.0 < ... < +NaN)."""
        dt = keys.dtype
        a = np.ascontiguousarray(keys).view(np.uint64).copy()
        kx = 0
        if dt == np.int64:
            kx = 1 << 63
        elif dt == np.float64:
            neg = (a >> np.uint64(63)).astype(bool)
            a = np.where(neg, ~a, a | np.uint64(1 << 63))
        elif dt != np.uint64:
            raise TypeError(f"64-bit keys expected, got {dt}")
        a = np.ascontiguousarray(a)
        if self.lib.oracle_bitonic_u64(a.ctypes.data, a.size, int(descending), kx):
            raise ValueError("length must be a power of two >= 2")
        if dt == np.float64:
            neg = ~(a >> np.uint64(63)).astype(bool)
            a = np.where(neg, ~a, a & np.uint64((1 << 63) - 1))
        return np.ascontiguousarray(a).view(dt)

    def quicksort_i32(self, keys: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(keys, dtype=np.int32).copy()
        self.lib.oracle_quicksort_i32(_ptr(a, _i32p), a.size)
        return a

    def quicksort_u32(self, keys: np.ndarray, descending: bool = False) -> np.ndarray:
        a = np.ascontiguousarray(keys, dtype=np.uint32).copy()
        self.lib.oracle_quicksort_u32(_ptr(a, _u32p), a.size, int(descending))
        return a

    def predicted_counts(self, k: int):
        r, c = ctypes.c_uint64(), ctypes.c_uint64()
        if self.lib.oracle_predicted_counts(k, ctypes.byref(r), ctypes.byref(c)):
            raise ValueError("k out of range")
        return r.value, c.value

    def pad_to_pow2_i32(self, keys: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(keys, dtype=np.int32)
        m = 2
        while m < a.size:
            m <<= 1
        out = np.empty(m, dtype=np.int32)
        got = self.lib.oracle_pad_to_pow2_i32(_ptr(a, _i32p), a.size, _ptr(out, _i32p))
        return out[:got]

    def fnv1a64(self, a: np.ndarray) -> int:
        a = np.ascontiguousarray(a)
        return int(self.lib.oracle_fnv1a64(a.ctypes.data, a.nbytes))

    def first_violation_u32(self, a: np.ndarray, descending: bool = False):
        a = np.ascontiguousarray(a, dtype=np.uint32)
        r = self.lib.oracle_first_violation_u32(_ptr(a, _u32p), a.size, int(descending))
        return None if r == 2**64 - 1 else int(r)


class Reference:
    """The reference's own code (oracle/_ref/libbitonic_ref.so)."""

    def __init__(self, path: str = _REF_SO):
        lib = ctypes.CDLL(path)
        lib.ref_sequential_bitonic_sort_i32.argtypes = [_i32p, ctypes.c_uint64]
        lib.ref_quicksort_i32.argtypes = [_i32p, ctypes.c_uint64]
        lib.ref_execute_i32.argtypes = [_i32p, ctypes.c_uint64, ctypes.c_int,
                                        ctypes.c_uint64, ctypes.c_uint, _u64p]
        lib.ref_execute_timed_i32.argtypes = [_i32p, ctypes.c_uint64, ctypes.c_int,
                                              ctypes.c_uint64, ctypes.c_uint,
                                              ctypes.POINTER(ctypes.c_double)]
        lib.ref_plan_counters.argtypes = [ctypes.c_uint, ctypes.c_int,
                                          ctypes.c_uint64, _u64p]
        lib.ref_predicted_counts.argtypes = [ctypes.c_uint, _u64p, _u64p]
        lib.ref_check_zero_one.argtypes = [ctypes.c_uint, ctypes.POINTER(ctypes.c_int)]
        lib.ref_has_bench.restype = ctypes.c_int
        self.has_bench = bool(lib.ref_has_bench())
        if self.has_bench:
            lib.ref_generate_input.argtypes = [_i32p, ctypes.c_uint64, ctypes.c_uint64]
            lib.ref_pad_to_pow2.argtypes = [_i32p, ctypes.c_uint64, _i32p, _u64p]
        self.lib = lib

    def sequential_bitonic_sort(self, keys: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(keys, dtype=np.int32).copy()
        rc = self.lib.ref_sequential_bitonic_sort_i32(_ptr(a, _i32p), a.size)
        if rc:
            raise ValueError(f"reference error {rc}")
        return a

    def sequential_bitonic_sort_inplace(self, a: np.ndarray) -> None:
        rc = self.lib.ref_sequential_bitonic_sort_i32(_ptr(a, _i32p), a.size)
        if rc:
            raise ValueError(f"reference error {rc}")

    def quicksort(self, keys: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(keys, dtype=np.int32).copy()
        self.lib.ref_quicksort_i32(_ptr(a, _i32p), a.size)
        return a

    def quicksort_inplace(self, a: np.ndarray) -> None:
        self.lib.ref_quicksort_i32(_ptr(a, _i32p), a.size)

    def execute(self, keys: np.ndarray, strategy: int = 2, cap: int = 1024,
                workers: int = 1):
        a = np.ascontiguousarray(keys, dtype=np.int32).copy()
        cnt = np.zeros(4, dtype=np.uint64)
        rc = self.lib.ref_execute_i32(_ptr(a, _i32p), a.size, strategy, cap,
                                      workers, _ptr(cnt, _u64p))
        if rc:
            raise ValueError(f"reference error {rc}")
        return a, tuple(int(x) for x in cnt)

    def execute_inplace(self, a: np.ndarray, strategy: int = 2, cap: int = 1024,
                        workers: int = 1) -> None:
        rc = self.lib.ref_execute_i32(_ptr(a, _i32p), a.size, strategy, cap,
                                      workers, None)
        if rc:
            raise ValueError(f"reference error {rc}")

    def execute_timed_inplace(self, a: np.ndarray, strategy: int = 2, cap: int = 1024,
                              workers: int = 1) -> float:
        """execute() in place, timed like run_cell (bench.cpp:92-107): plan
        build + execute on the clock, the vector copies off it.  Returns ms."""
        ms = ctypes.c_double(0.0)
        rc = self.lib.ref_execute_timed_i32(_ptr(a, _i32p), a.size, strategy, cap,
                                            workers, ctypes.byref(ms))
        if rc:
            raise ValueError(f"reference error {rc}")
        return ms.value

    def plan_counters(self, k: int, strategy: int, cap: int):
        cnt = np.zeros(4, dtype=np.uint64)
        rc = self.lib.ref_plan_counters(k, strategy, cap, _ptr(cnt, _u64p))
        if rc:
            raise ValueError(f"reference error {rc}")
        return tuple(int(x) for x in cnt)

    def predicted_counts(self, k: int):
        r, c = ctypes.c_uint64(), ctypes.c_uint64()
        rc = self.lib.ref_predicted_counts(k, ctypes.byref(r), ctypes.byref(c))
        if rc:
            raise ValueError(f"reference error {rc}")
        return r.value, c.value

    def check_zero_one(self, k: int) -> bool:
        ok = ctypes.c_int(0)
        rc = self.lib.ref_check_zero_one(k, ctypes.byref(ok))
        if rc:
            raise ValueError(f"reference error {rc}")
        return bool(ok.value)

    def generate_input(self, n: int, seed: int = 1) -> np.ndarray:
        out = np.empty(n, dtype=np.int32)
        rc = self.lib.ref_generate_input(_ptr(out, _i32p), n, seed)
        if rc:
            raise ValueError(f"reference error {rc}")
        return out

    def pad_to_pow2(self, keys: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(keys, dtype=np.int32)
        m = 2
        while m < a.size:
            m <<= 1
        out = np.empty(m, dtype=np.int32)
        got = ctypes.c_uint64()
        rc = self.lib.ref_pad_to_pow2(_ptr(a, _i32p), a.size, _ptr(out, _i32p),
                                      ctypes.byref(got))
        if rc:
            raise ValueError(f"reference error {rc}")
        return out[: got.value]


_oracle = None


def oracle() -> Oracle:
    global _oracle
    if _oracle is None:
        _oracle = Oracle()
    return _oracle


def reference():
    """The compiled reference, or None when oracle/_ref was not built."""
    if not os.path.exists(_REF_SO):
        return None
    return Reference()
