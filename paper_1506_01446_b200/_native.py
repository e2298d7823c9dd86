"""ctypes binding of the C ABI in include/b200_bitonic.h.

The shared library is the product: there is no Python or CPU fallback.  If
``libb200_bitonic.so`` is missing, every entry point raises immediately.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# B200_BITONIC_LIB overrides the library path (A/B performance experiments).
LIB_PATH = os.environ.get("B200_BITONIC_LIB") or os.path.join(HERE, "libb200_bitonic.so")

# Every symbol include/b200_bitonic.h declares (tests check the .so exports
# exactly these).
EXPORTED = (
    "b200_bitonic_sort_u32",
    "b200_bitonic_sort_i32",
    "b200_bitonic_sort_u32_batched",
    "b200_bitonic_sort_i32_batched",
    "b200_bitonic_sort_pairs_u32",
    "b200_bitonic_sort_pairs_i32",
    "b200_bitonic_sort_pairs_u32_batched",
    "b200_bitonic_sort_f32",
    "b200_bitonic_sort_u64",
    "b200_bitonic_sort_i64",
    "b200_bitonic_sort_f64",
    "b200_bitonic_sort_u64_planes",
    "b200_bitonic_release_scratch",
    "b200_bitonic_ipc_alloc",
    "b200_bitonic_ipc_free",
    "b200_bitonic_ipc_open",
    "b200_bitonic_ipc_close",
    "b200_bitonic_copy",
    "b200_bitonic_merge_split_u32_count",
    "b200_bitonic_ipc_event_create",
    "b200_bitonic_ipc_event_open",
    "b200_bitonic_event_destroy",
    "b200_bitonic_event_record",
    "b200_bitonic_stream_wait_event",
    "b200_bitonic_sort_padded_u32",
    "b200_bitonic_sort_padded_i32",
    "b200_bitonic_sort_mergepath_u32",
    "b200_bitonic_sort_mergepath_i32",
    "b200_bitonic_sort_host_i32",
    "b200_bitonic_sort_host_u32",
    "b200_bitonic_generate_input",
    "b200_bitonic_sort_u32_multi",
    "b200_bitonic_merge_split_u32",
    "b200_bitonic_merge_u32",
    "b200_bitonic_plan",
    "b200_bitonic_run_pass_u32",
    "b200_bitonic_counters",
    "b200_bitonic_set_tuning",
    "b200_bitonic_last_error",
    "b200_bitonic_version",
)


class IpcHandle(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_ubyte * 64)]


class PassInfo(ctypes.Structure):
    _fields_ = [
        ("tile_bits", ctypes.c_int),
        ("a", ctypes.c_int),
        ("y", ctypes.c_int),
        ("tile_sort", ctypes.c_int),
        ("segA_hi", ctypes.c_int),
        ("pA", ctypes.c_int),
        ("segB_lo", ctypes.c_int),
        ("pB", ctypes.c_int),
        ("ctas", ctypes.c_uint64),
        ("compare_exchanges", ctypes.c_uint64),
        ("cluster", ctypes.c_int),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """Load the native library (raises if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"native library {LIB_PATH} is missing: run "
            "`python -m paper_1506_01446_b200.build` (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, u64, i = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
    L.b200_bitonic_sort_u32.argtypes = [vp, u64, i, vp]
    L.b200_bitonic_sort_i32.argtypes = [vp, u64, i, vp]
    L.b200_bitonic_sort_u32_batched.argtypes = [vp, u64, u64, i, vp]
    L.b200_bitonic_sort_i32_batched.argtypes = [vp, u64, u64, i, vp]
    L.b200_bitonic_sort_f32.argtypes = [vp, u64, i, vp]
    L.b200_bitonic_sort_u64.argtypes = [vp, u64, i, vp]
    L.b200_bitonic_sort_i64.argtypes = [vp, u64, i, vp]
    L.b200_bitonic_sort_f64.argtypes = [vp, u64, i, vp]
    L.b200_bitonic_sort_u64_planes.argtypes = [vp, vp, u64, i, vp]
    L.b200_bitonic_release_scratch.argtypes = []
    L.b200_bitonic_ipc_alloc.argtypes = [u64, ctypes.POINTER(vp), ctypes.POINTER(IpcHandle)]
    L.b200_bitonic_ipc_free.argtypes = [vp]
    L.b200_bitonic_ipc_open.argtypes = [ctypes.POINTER(IpcHandle), ctypes.POINTER(vp)]
    L.b200_bitonic_ipc_close.argtypes = [vp]
    L.b200_bitonic_copy.argtypes = [vp, vp, u64, vp]
    L.b200_bitonic_merge_split_u32_count.argtypes = [vp, vp, u64, i, ctypes.c_uint32, vp, vp, vp]
    L.b200_bitonic_ipc_event_create.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(IpcHandle)]
    L.b200_bitonic_ipc_event_open.argtypes = [ctypes.POINTER(IpcHandle), ctypes.POINTER(vp)]
    L.b200_bitonic_event_destroy.argtypes = [vp]
    L.b200_bitonic_event_record.argtypes = [vp, vp]
    L.b200_bitonic_stream_wait_event.argtypes = [vp, vp]
    L.b200_bitonic_sort_pairs_u32.argtypes = [vp, vp, u64, i, vp]
    L.b200_bitonic_sort_pairs_i32.argtypes = [vp, vp, u64, i, vp]
    L.b200_bitonic_sort_pairs_u32_batched.argtypes = [vp, vp, u64, u64, i, vp]
    L.b200_bitonic_sort_padded_u32.argtypes = [vp, u64, i, vp]
    L.b200_bitonic_sort_padded_i32.argtypes = [vp, u64, i, vp]
    L.b200_bitonic_sort_mergepath_u32.argtypes = [vp, u64, i, vp]
    L.b200_bitonic_sort_mergepath_i32.argtypes = [vp, u64, i, vp]
    L.b200_bitonic_sort_host_i32.argtypes = [vp, u64, i]
    L.b200_bitonic_sort_host_u32.argtypes = [vp, u64, i]
    L.b200_bitonic_generate_input.argtypes = [vp, u64, u64]
    L.b200_bitonic_sort_u32_multi.argtypes = [ctypes.POINTER(vp),
                                              ctypes.POINTER(ctypes.c_int), i, u64, i]
    L.b200_bitonic_merge_split_u32.argtypes = [vp, vp, u64, i, ctypes.c_uint32, vp, vp]
    L.b200_bitonic_merge_u32.argtypes = [vp, u64, vp, u64, ctypes.c_uint32, vp, vp]
    L.b200_bitonic_plan.argtypes = [u64, u64, ctypes.POINTER(PassInfo), i,
                                    ctypes.POINTER(ctypes.c_int)]
    L.b200_bitonic_run_pass_u32.argtypes = [vp, u64, u64, i, i, vp]
    L.b200_bitonic_counters.argtypes = [u64, u64, ctypes.POINTER(ctypes.c_uint64)]
    L.b200_bitonic_set_tuning.argtypes = [i, i]
    L.b200_bitonic_last_error.argtypes = []
    L.b200_bitonic_version.argtypes = []
    L.b200_bitonic_last_error.restype = ctypes.c_char_p
    L.b200_bitonic_version.restype = ctypes.c_char_p
    for name in EXPORTED:
        getattr(L, name).restype = getattr(L, name).restype or ctypes.c_int
    L.b200_bitonic_last_error.restype = ctypes.c_char_p
    L.b200_bitonic_version.restype = ctypes.c_char_p
    _lib = L
    return L
