"""CPU: the C-ABI library loads, exports the header's symbols, plans the
network exactly, and refuses to run without a GPU (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1506_01446_b200 as b200
from paper_1506_01446_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "b200_bitonic.h")


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_1506_01446_b200 import build
    build.build()
    b200.set_tuning(0, 5)
    yield
    b200.set_tuning(0, 5)


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(b200_bitonic_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    decl = declared_symbols()
    assert decl, "header parse failed"
    assert sorted(_native.EXPORTED) == decl
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (b200_bitonic_\w+)", out))
    assert set(decl) <= exported
    L = _native.lib()
    for name in decl:
        assert getattr(L, name) is not None


def test_every_entry_has_argtypes():
    """ctypes would pass Python ints as 32-bit C ints without argtypes: every
    entry taking a 64-bit length (or any argument) must declare them."""
    L = _native.lib()
    missing = [name for name in _native.EXPORTED if getattr(L, name).argtypes is None]
    assert not missing, missing


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_kernel_spills():
    """Every kernel in the library runs without local-memory stack (ptxas
    spills): cuobjdump -res-usage reports STACK:0 for all of them."""
    out = subprocess.run(["cuobjdump", "-res-usage", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    stacks = re.findall(r"STACK:(\d+)", out)
    assert len(stacks) > 100
    names = re.findall(r"Function (\S+):", out)
    bad = [(n, st) for n, st in zip(names, stacks) if st != "0"]
    assert not bad, bad


def test_version():
    assert "sm_100a" in b200.version()


# ---- plan = the reference's schedule, regrouped ---------------------------

def schedule(k):
    """generate_schedule (schedule.cpp:20-36) as (phase, bit) pairs."""
    return [(p, s - 1) for p in range(1, k + 1) for s in range(p, 0, -1)]


@pytest.mark.parametrize("tile_bits,run_bits", [(0, 5), (14, 5), (15, 5), (13, 3),
                                                (12, 7), (10, 2), (6, 5), (11, 6)])
def test_plan_reproduces_schedule(tile_bits, run_bits):
    b200.set_tuning(tile_bits, run_bits)
    try:
        for k in list(range(1, 25)) + [28, 30, 32, 34]:
            n = 1 << k
            plan = b200.plan(n)
            steps = [s for p in plan for s in p.step_bits()]
            assert steps == schedule(k), (k, plan)
            rounds, ces = (k * (k + 1) // 2, (1 << (k - 1)) * (k * (k + 1) // 2))
            assert sum(p.compare_exchanges for p in plan) == ces
            for p in plan:
                C = p.tile_bits
                assert 1 <= C <= 15
                assert p.ctas == (n >> C) * p.cluster
                assert p.cluster == 1 or (tile_bits == 0 and k >= 24 and C == 15)
                if not p.tile_sort:
                    h = C - p.a
                    # coset bits: [0,a) and [y, y+h) disjoint, inside [0,k);
                    # the cluster plans' middle passes move 2^4-key runs
                    lo = min(run_bits, C, 4 if (tile_bits == 0 and k >= 24) else C)
                    assert p.a >= lo and p.a >= 2
                    assert h == 0 or p.y >= p.a
                    assert p.y + h <= k
                    # every step bit of the pass lies in the coset
                    for (_, bit) in p.step_bits():
                        assert bit < p.a or p.y <= bit < p.y + h
    finally:
        b200.set_tuning(0, 5)


def test_plan_batched():
    for k, batch in [(12, 4096), (3, 5), (10, 3), (16, 8), (20, 2)]:
        plan = b200.plan(1 << k, batch)
        steps = [s for p in plan for s in p.step_bits()]
        assert steps == schedule(k)
        total = (1 << k) * batch
        for p in plan:
            assert (p.ctas // p.cluster) << p.tile_bits == total


# The default plan's exact pass count per size (a regression in the planner
# shows up here, not as a slower bench).  P_min(k, 15) is the
# lower bound without the coalescing constraint.
PLAN_PASSES = {12: 1, 16: 7, 20: 15, 24: 20, 28: 29, 30: 34, 32: 40}
PMIN = {16: 3, 20: 7, 24: 13, 28: 21, 30: 24, 32: 29}


def test_pass_counts_pinned():
    got = {k: len(b200.plan(1 << k)) for k in PLAN_PASSES}
    assert got == PLAN_PASSES
    for k, pm in PMIN.items():
        assert got[k] >= pm


def test_generate_input_is_the_references(golden, orc):
    # product-side generate_input (bench.cpp:354-364) == the golden digests
    # made by the reference's own generator
    for c in golden["cases"][:12]:
        x = b200.generate_input(1 << c["k"], c["seed"])
        assert x.dtype == np.uint32
        assert "%016x" % orc.fnv1a64(x) == c["input_fnv"]
    assert [int(v) for v in b200.generate_input(3, 1)] == [0xbb686f68, 0x2318fa4e, 0x7ae6459a]
    with pytest.raises(b200.InvalidSizeError):
        b200.generate_input(0, 1)


def test_sort_host_rejects_read_only_buffers():
    a = np.frombuffer(bytes(64), dtype=np.int32)
    assert not a.flags["WRITEABLE"]
    with pytest.raises(b200.ConfigError):
        b200.sort_host(a)


def test_partitioned_sort_checks_the_shard():
    import torch
    from paper_1506_01446_b200 import dist as bdist
    for bad in [torch.zeros(16, dtype=torch.float32), torch.zeros(16, dtype=torch.int64),
                torch.zeros(32, dtype=torch.int32)[::2]]:
        with pytest.raises(b200.ConfigError):
            bdist.partitioned_sort_(bad, world=1, rank=0)
    with pytest.raises(b200.ConfigError):  # CPU shard without injected (test) ops
        bdist.partitioned_sort_(torch.zeros(16, dtype=torch.int32), world=1, rank=0)


def test_counters_match_reference_cost_model(ref):
    # engine.hpp:55-70: one pass = n reads + n writes; CEs = predicted_counts
    for k in range(1, 25):
        c = b200.counters(1 << k)
        r, ces = ref.predicted_counts(k)
        assert c["compare_exchanges"] == ces
        assert c["global_reads"] == c["kernel_launches"] << k
        assert c["global_writes"] == c["kernel_launches"] << k
    # fewer HBM round trips than the reference's own best plan (fused, 1024)
    for k in [16, 20, 22, 24]:
        ours = b200.counters(1 << k)["kernel_launches"]
        theirs = ref.plan_counters(k, 2, 1024)[0]
        assert ours < theirs


# ---- emulate each planned pass on the CPU (validates plan semantics) ------

def emulate_plan(x, k, batch=1, descending=False):
    """Apply every planned step with the reference's CE rule
    (compare_exchange engine.cpp:16-22; direction (i & 2^p) == 0)."""
    n = 1 << k
    a = x.copy().reshape(batch, n)
    idx = np.arange(n, dtype=np.int64)
    for p in b200.plan(n, batch):
        for (phase, bit) in p.step_bits():
            lo = idx[(idx >> bit) & 1 == 0]
            hi = lo + (1 << bit)
            asc = ((lo >> phase) & 1) == 0 if phase < k else np.ones(lo.size, bool)
            if descending:
                asc = ~asc
            u, v = a[:, lo], a[:, hi]
            mn, mx = np.minimum(u, v), np.maximum(u, v)
            a[:, lo] = np.where(asc, mn, mx)
            a[:, hi] = np.where(asc, mx, mn)
    return a.reshape(-1)


@pytest.mark.parametrize("k", [1, 2, 5, 9, 13, 16, 18])
def test_emulated_plan_sorts(orc, k):
    x = orc.generate_input(1 << k, 100 + k)
    assert (emulate_plan(x, k) == np.sort(x)).all()
    assert (emulate_plan(x, k, descending=True) == np.sort(x)[::-1]).all()


def test_emulated_plan_small_tiles(orc):
    b200.set_tuning(6, 2)
    try:
        for k in [7, 11, 15]:
            x = orc.generate_input(1 << k, k)
            assert (emulate_plan(x, k) == np.sort(x)).all()
    finally:
        b200.set_tuning(0, 5)


@pytest.mark.parametrize("tile,merge,k", [(12, 13, 16), (12, 14, 16), (12, 14, 18),
                                          (13, 14, 17), (13, 14, 18)])
def test_emulated_mixed_coset_plans(orc, monkeypatch, tile, merge, k):
    """Plans whose merge passes pick their coset size per pass (between the
    tile's and the merge override; the default from 2^24 keys) must still
    apply exactly the reference's step sequence: emulate them step by step
    on the CPU."""
    monkeypatch.setenv("B200_BITONIC_CMERGE", str(merge))
    monkeypatch.setenv("B200_BITONIC_WIDE_TAIL_COST", "0.2")
    b200.set_tuning(tile, 5)
    try:
        pl = b200.plan(1 << k)
        sizes = {p.tile_bits for p in pl[1:]}
        assert sizes <= set(range(tile, merge + 1)) and len(sizes) >= 2, sizes
        x = orc.generate_input(1 << k, 500 + k)
        assert (emulate_plan(x, k) == np.sort(x)).all(), (tile, merge, k)
        assert (emulate_plan(x, k, descending=True) == np.sort(x)[::-1]).all()
    finally:
        b200.set_tuning(0, 5)


def test_emulated_plan_batched(orc):
    x = orc.generate_input(8 * 1024, 3)
    out = emulate_plan(x, 10, batch=8)
    assert (out.reshape(8, -1) == np.sort(x.reshape(8, -1), axis=1)).all()


# ---- error contract -------------------------------------------------------

def test_plan_rejects_bad_sizes():
    for n in [0, 1, 3, 6, 1000]:
        with pytest.raises(b200.InvalidSizeError):
            b200.plan(n)
    with pytest.raises(b200.ConfigError):
        b200.plan(16, 0)


def test_set_tuning_rejects_bad_values():
    with pytest.raises(b200.ConfigError):
        b200.set_tuning(3, 5)
    with pytest.raises(b200.ConfigError):
        b200.set_tuning(0, 1)


def test_device_entry_validates_before_touching_the_gpu():
    L = _native.lib()
    assert L.b200_bitonic_sort_u32(None, 6, 0, None) == 1       # invalid size
    assert L.b200_bitonic_sort_u32(None, 16, 2, None) == 2      # bad direction
    assert L.b200_bitonic_sort_u32(None, 16, 0, None) == 2      # null pointer
    assert L.b200_bitonic_sort_u32(ctypes.c_void_p(8), 16, 0, None) == 2  # misaligned
    assert L.b200_bitonic_sort_u32_multi(None, None, 3, 16, 0) == 2  # ngpu


def test_no_cpu_fallback():
    """Without a GPU the product fails loudly (CudaError), never sorts on CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    x = np.arange(16, dtype=np.int32)[::-1].copy()
    with pytest.raises(b200.CudaError):
        b200.sequential_bitonic_sort(x)
    assert x.tolist() == list(range(16))[::-1]
    with pytest.raises(b200.ConfigError):
        b200.sort_(torch.arange(16, dtype=torch.int32))
    with pytest.raises(b200.InvalidSizeError):
        b200.sequential_bitonic_sort(np.zeros(6, np.int32))


def test_key_value_entry_validates():
    L = _native.lib()
    assert L.b200_bitonic_sort_pairs_u32(None, None, 16, 0, None) == 2
    assert L.b200_bitonic_sort_pairs_u32(None, None, 6, 0, None) in (1, 2)
