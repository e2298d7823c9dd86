"""paper_1506_01446_b200 -- B200-native (sm_100a) bitonic sort of 32-bit keys.

Python host mirror of the reference's sort entry points (namespace
``bitonic`` in /root/reference/proj/include/bitonic), calling the CUDA side
through the C ABI of include/b200_bitonic.h:

==============================================  ===============================
reference (C++)                                 here
==============================================  ===============================
sequential_bitonic_sort(span<int32_t>)          sequential_bitonic_sort(np.int32 array)
  engine.hpp:102-104, engine.cpp:248-266          (host array, in place, via GPU)
execute(build_plan(...), keys, workers)         sort_(tensor, descending)   (device, in place)
  engine.hpp:77-92
build_plan / account / Counters                 plan(n), counters(n)
  engine.hpp:44-84, engine.cpp:86-173
invalid_size_error (error.hpp:11-15)            InvalidSizeError  (a ValueError)
config_error       (error.hpp:19-23)            ConfigError       (a ValueError)
==============================================  ===============================

plus the north_star additions: ``descending``, uint32 keys, batched arrays
(``sort_batched_``), the partitioned multi-GPU sort (``sort_multi``) and the
merge-split building block (``merge_split_``).  There is no CPU fallback: the
native library must be present and a CUDA device must be visible.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _native

__all__ = [
    "InvalidSizeError", "ConfigError", "CudaError",
    "sort_", "sort_mergepath_", "sort_pairs_", "sort_planes_", "argsort", "sort_padded_", "sort_batched_", "run_pass_", "sequential_bitonic_sort", "sort_host",
    "merge_split_", "merge_", "sort_multi", "plan", "counters", "set_tuning",
    "PassPlan", "version", "library_path", "release_scratch", "generate_input",
]


class InvalidSizeError(ValueError):
    """Mirror of bitonic::invalid_size_error (std::invalid_argument)."""


class ConfigError(ValueError):
    """Mirror of bitonic::config_error (std::invalid_argument)."""


class CudaError(RuntimeError):
    """A CUDA runtime failure inside the native library."""


class NcclError(RuntimeError):
    """Reserved for the NCCL exchange path."""


_ERRORS = {1: InvalidSizeError, 2: ConfigError, 3: CudaError, 4: NcclError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = _native.lib().b200_bitonic_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RuntimeError)(msg)


def library_path() -> str:
    return _native.LIB_PATH


def version() -> str:
    return _native.lib().b200_bitonic_version().decode()


def _stream_ptr(stream) -> Optional[int]:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def _key_dtype(t):
    import torch
    if t.dtype == torch.int32:
        return "i32"
    if t.dtype == torch.uint32:
        return "u32"
    if t.dtype == torch.float32:
        return "f32"
    if t.dtype == torch.int64:
        return "i64"
    if t.dtype == torch.uint64:
        return "u64"
    if t.dtype == torch.float64:
        return "f64"
    raise ConfigError(f"keys must be int32, uint32, float32, int64, uint64 or float64, "
                      f"got {t.dtype}")


def _key_dtype32(t):
    kind = _key_dtype(t)
    if kind not in ("i32", "u32"):
        raise ConfigError(f"this entry point takes int32 or uint32 keys, got {t.dtype}")
    return kind


def _on_device(t):
    """Make t's device current for the native call (the library launches on
    the current device and uses that device's current stream)."""
    import torch
    return torch.cuda.device(t.device)


def _same_device(*ts) -> None:
    d = ts[0].device
    for t in ts[1:]:
        if t.device != d:
            raise ConfigError(f"tensors on different devices: {d} and {t.device}")


def _check_tensor(t) -> None:
    if not t.is_cuda:
        raise ConfigError("sort_ needs a CUDA tensor (use sort_host for host arrays)")
    if not t.is_contiguous():
        raise ConfigError("keys must be contiguous")


def sort_(t, descending: bool = False, stream=None):
    """Sort a 1-D CUDA tensor of int32 (signed order, the reference's key type),
    uint32, float32 (IEEE totalOrder), int64, uint64 or float64 keys in place;
    asynchronous on ``stream`` (default: current)."""
    _check_tensor(t)
    kind = _key_dtype(t)
    L = _native.lib()
    fn = {"i32": L.b200_bitonic_sort_i32, "u32": L.b200_bitonic_sort_u32,
          "f32": L.b200_bitonic_sort_f32, "i64": L.b200_bitonic_sort_i64,
          "u64": L.b200_bitonic_sort_u64, "f64": L.b200_bitonic_sort_f64}[kind]
    with _on_device(t):
        _check(fn(ctypes.c_void_p(t.data_ptr()), t.numel(), int(bool(descending)),
                  ctypes.c_void_p(_stream_ptr(stream))))
    return t


def sort_pairs_(keys, values, descending: bool = False, stream=None):
    """Key-value sort in place: ``values`` (a 32-bit payload tensor of the same
    length) moves with ``keys`` (int32 or uint32).  Same network and tie rule
    as the reference (swap only when strictly out of order): equal keys keep
    the reference network's payload order (not stable)."""
    import torch
    _check_tensor(keys)
    _check_tensor(values)
    if values.numel() != keys.numel() or values.element_size() != 4:
        raise ConfigError("values must be a 32-bit tensor with one entry per key")
    kind = _key_dtype32(keys)
    fn = (_native.lib().b200_bitonic_sort_pairs_i32 if kind == "i32"
          else _native.lib().b200_bitonic_sort_pairs_u32)
    _same_device(keys, values)
    with _on_device(keys):
        _check(fn(ctypes.c_void_p(keys.data_ptr()), ctypes.c_void_p(values.data_ptr()),
                  keys.numel(), int(bool(descending)), ctypes.c_void_p(_stream_ptr(stream))))
    return keys, values


def sort_planes_(hi, lo, descending: bool = False, stream=None):
    """64-bit keys held as two uint32/int32 word planes (key i = hi[i] << 32 |
    lo[i], unsigned), sorted in place with no scratch memory."""
    _check_tensor(hi)
    _check_tensor(lo)
    if hi.element_size() != 4 or lo.element_size() != 4 or hi.numel() != lo.numel():
        raise ConfigError("hi and lo must be 32-bit tensors of equal length")
    _same_device(hi, lo)
    with _on_device(hi):
        _check(_native.lib().b200_bitonic_sort_u64_planes(
            ctypes.c_void_p(hi.data_ptr()), ctypes.c_void_p(lo.data_ptr()), hi.numel(),
            int(bool(descending)), ctypes.c_void_p(_stream_ptr(stream))))
    return hi, lo


def release_scratch() -> None:
    """Return the library's retained scratch memory (all devices) to the driver."""
    _check(_native.lib().b200_bitonic_release_scratch())


def argsort(keys, descending: bool = False, stream=None):
    """Indices that sort ``keys`` (not modified), via the key-value network.
    int32 indices: up to 2^31 keys."""
    import torch
    if keys.numel() > (1 << 31):
        raise ConfigError("argsort returns int32 indices: at most 2^31 keys")
    k = keys.clone()
    idx = torch.arange(keys.numel(), dtype=torch.int32, device=keys.device)
    sort_pairs_(k, idx, descending=descending, stream=stream)
    return idx


def sort_padded_(t, descending: bool = False, stream=None):
    """Any-length sort: the reference's pad_to_pow2 + sort + truncate
    (bench.cpp:366-377) -- non-powers of two go through a padded scratch
    buffer (stream-ordered allocation); powers of two sort in place."""
    _check_tensor(t)
    kind = _key_dtype32(t)
    fn = (_native.lib().b200_bitonic_sort_padded_i32 if kind == "i32"
          else _native.lib().b200_bitonic_sort_padded_u32)
    with _on_device(t):
        _check(fn(ctypes.c_void_p(t.data_ptr()), t.numel(), int(bool(descending)),
                  ctypes.c_void_p(_stream_ptr(stream))))
    return t


def sort_mergepath_(t, descending: bool = False, stream=None):
    """The merge-path variant of ``sort_`` (uint32 / int32, power-of-two
    length): identical output, one pass per global phase (tile sort + co-rank
    partitioned bitonic tile merges through an n-key scratch buffer)."""
    _check_tensor(t)
    kind = _key_dtype32(t)
    fn = (_native.lib().b200_bitonic_sort_mergepath_i32 if kind == "i32"
          else _native.lib().b200_bitonic_sort_mergepath_u32)
    with _on_device(t):
        _check(fn(ctypes.c_void_p(t.data_ptr()), t.numel(), int(bool(descending)),
                  ctypes.c_void_p(_stream_ptr(stream))))
    return t


def sort_batched_(t, n_per_array: int, descending: bool = False, stream=None):
    """Sort ``t.numel() // n_per_array`` contiguous arrays independently."""
    _check_tensor(t)
    if n_per_array < 1 or t.numel() % n_per_array:
        raise ConfigError("numel must be a multiple of n_per_array")
    kind = _key_dtype32(t)
    fn = (_native.lib().b200_bitonic_sort_i32_batched if kind == "i32"
          else _native.lib().b200_bitonic_sort_u32_batched)
    with _on_device(t):
        _check(fn(ctypes.c_void_p(t.data_ptr()), n_per_array, t.numel() // n_per_array,
                  int(bool(descending)), ctypes.c_void_p(_stream_ptr(stream))))
    return t


def generate_input(n: int, seed: int = 1) -> np.ndarray:
    """The reference's benchmark keys, generate_input(size, seed)
    (bench.cpp:354-364): the low 32 bits of std::mt19937_64(seed), as a host
    uint32 array (the reference stores the same bits as int32)."""
    out = np.empty(int(n), dtype=np.uint32)
    _check(_native.lib().b200_bitonic_generate_input(
        ctypes.c_void_p(out.ctypes.data), int(n), int(seed)))
    return out


def sort_host(keys: np.ndarray, descending: bool = False) -> np.ndarray:
    """In-place sort of a host numpy int32/uint32 array (H2D, sort, D2H)."""
    if not isinstance(keys, np.ndarray) or not keys.flags["C_CONTIGUOUS"]:
        raise ConfigError("keys must be a C-contiguous numpy array")
    if not keys.flags["WRITEABLE"]:
        raise ConfigError("keys must be writeable (the sort is in place)")
    if keys.dtype == np.int32:
        fn = _native.lib().b200_bitonic_sort_host_i32
    elif keys.dtype == np.uint32:
        fn = _native.lib().b200_bitonic_sort_host_u32
    else:
        raise ConfigError(f"keys must be int32 or uint32, got {keys.dtype}")
    _check(fn(ctypes.c_void_p(keys.ctypes.data), keys.size, int(bool(descending))))
    return keys


def sequential_bitonic_sort(keys: np.ndarray) -> None:
    """Drop-in for bitonic::sequential_bitonic_sort(std::span<int32_t>)
    (engine.cpp:248-266): ascending, in place, power-of-two length >= 2,
    InvalidSizeError otherwise -- but the network runs on the GPU."""
    if not isinstance(keys, np.ndarray) or keys.dtype != np.int32:
        raise ConfigError("keys must be a numpy int32 array")
    sort_host(keys, descending=False)


def run_pass_(t, pass_index: int, n_per_array: Optional[int] = None,
              descending: bool = False, stream=None):
    """Run a single pass of the plan on uint32 keys (profiling aid)."""
    _check_tensor(t)
    n = n_per_array or t.numel()
    with _on_device(t):
        _check(_native.lib().b200_bitonic_run_pass_u32(
            ctypes.c_void_p(t.data_ptr()), n, t.numel() // n, int(bool(descending)),
            int(pass_index), ctypes.c_void_p(_stream_ptr(stream))))
    return t


def merge_split_(local, partner, out, keep_high: bool, key_xor: int = 0,
                 stream=None):
    """out <- the m smallest (keep_high=False) or largest keys of local U partner
    (both sorted in the order ``key_xor`` selects: 0 uint32, 0x80000000 int32,
    0xFFFFFFFF descending uint32)."""
    for x in (local, partner, out):
        _check_tensor(x)
    m = local.numel()
    if partner.numel() != m or out.numel() != m:
        raise ConfigError("local, partner and out must have the same length")
    _same_device(local, out)  # partner may live on a peer device (read over NVLink)
    with _on_device(out):
        _check(_native.lib().b200_bitonic_merge_split_u32(
            ctypes.c_void_p(local.data_ptr()), ctypes.c_void_p(partner.data_ptr()), m,
            int(bool(keep_high)), ctypes.c_uint32(key_xor & 0xFFFFFFFF),
            ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(_stream_ptr(stream))))
    return out


def merge_(a, b, out, key_xor: int = 0, stream=None):
    """out <- merge of the sorted tensors a and b (lengths may differ; order
    given by ``key_xor`` as in merge_split_)."""
    for x in (a, b, out):
        _check_tensor(x)
    if out.numel() != a.numel() + b.numel():
        raise ConfigError("out must hold a.numel() + b.numel() keys")
    with _on_device(out):
        _check(_native.lib().b200_bitonic_merge_u32(
            ctypes.c_void_p(a.data_ptr()), a.numel(), ctypes.c_void_p(b.data_ptr()), b.numel(),
            ctypes.c_uint32(key_xor & 0xFFFFFFFF), ctypes.c_void_p(out.data_ptr()),
            ctypes.c_void_p(_stream_ptr(stream))))
    return out


def sort_multi(shards: Sequence, descending: bool = False) -> None:
    """Partitioned sort: shards[r] (uint32, equal sizes, on any devices) are the
    contiguous slices of one array; afterwards shard r holds sorted positions
    [r*m, (r+1)*m).  Synchronous; one host thread drives every device."""
    import torch
    g = len(shards)
    ptrs = (ctypes.c_void_p * g)(*[ctypes.c_void_p(s.data_ptr()) for s in shards])
    devs = (ctypes.c_int * g)(*[s.device.index for s in shards])
    for s in shards:
        _check_tensor(s)
        if s.dtype != torch.uint32:
            raise ConfigError("sort_multi takes uint32 shards")
    n_total = sum(s.numel() for s in shards)
    if len({s.numel() for s in shards}) != 1:
        raise ConfigError("shards must have equal length")
    for s in shards:
        torch.cuda.synchronize(s.device)
    _check(_native.lib().b200_bitonic_sort_u32_multi(ptrs, devs, g, n_total,
                                                     int(bool(descending))))


@dataclass(frozen=True)
class PassPlan:
    tile_bits: int
    a: int
    y: int
    tile_sort: bool
    segA_hi: int
    pA: int
    segB_lo: int
    pB: int
    ctas: int
    compare_exchanges: int
    cluster: int = 1  # CTAs per cluster (2: a 2^15-key coset over a CTA pair)

    def step_bits(self) -> List[tuple]:
        """(phase, global bit) of every network step this pass runs, in order."""
        out = []
        C = self.tile_bits
        if self.tile_sort:
            for p in range(1, self.pA + 1):
                for b in range(p - 1, -1, -1):
                    out.append((p, b))
            return out

        def glob(l):
            return l if l < self.a else self.y + (l - self.a)

        if self.segA_hi >= 0:
            for l in range(self.segA_hi, -1, -1):
                out.append((self.pA, glob(l)))
        if self.segB_lo >= 0:
            for l in range(C - 1, self.segB_lo - 1, -1):
                out.append((self.pB, glob(l)))
        return out


def plan(n: int, batch: int = 1) -> List[PassPlan]:
    """The launch plan for ``batch`` arrays of ``n`` keys (host only)."""
    L = _native.lib()
    cnt = ctypes.c_int(0)
    _check(L.b200_bitonic_plan(n, batch, None, 0, ctypes.byref(cnt)))
    arr = (_native.PassInfo * max(cnt.value, 1))()
    _check(L.b200_bitonic_plan(n, batch, arr, cnt.value, ctypes.byref(cnt)))
    return [PassPlan(p.tile_bits, p.a, p.y, bool(p.tile_sort), p.segA_hi, p.pA,
                     p.segB_lo, p.pB, int(p.ctas), int(p.compare_exchanges), int(p.cluster))
            for p in arr[: cnt.value]]


def counters(n: int, batch: int = 1) -> dict:
    """Counters in the reference's model (engine.hpp:55-70): launches, key
    reads, key writes, compare-exchanges for one sort."""
    out = (ctypes.c_uint64 * 4)()
    _check(_native.lib().b200_bitonic_counters(n, batch, out))
    return {"kernel_launches": int(out[0]), "global_reads": int(out[1]),
            "global_writes": int(out[2]), "compare_exchanges": int(out[3])}


def set_tuning(tile_bits: int = 0, min_run_bits: int = 5) -> None:
    """tile_bits: 0 = automatic, else 6..15; min_run_bits: 2..10."""
    _check(_native.lib().b200_bitonic_set_tuning(tile_bits, min_run_bits))
