"""CPU: pin the oracle (plain-C restatement) to the reference.

The oracle is the checker for every GPU parity test, so it is validated here
against (a) the golden fixtures generated from the reference's own code
(tests/golden/make_golden.py) and (b) the compiled reference itself
(oracle/_ref) when present.
"""
import numpy as np
import pytest

FLIP = np.uint32(0x80000000)


def h(x):
    return "%016x" % x


def test_generate_input_matches_golden(orc, golden):
    for c in golden["cases"]:
        x = orc.generate_input(1 << c["k"], c["seed"])
        assert h(orc.fnv1a64(x)) == c["input_fnv"], c


def test_generate_input_first_values():
    # seed 1 starts bb686f68 2318fa4e 7ae6459a (as u32)
    import oracle
    x = oracle.oracle().generate_input(3, 1)
    assert [int(v) for v in x] == [0xbb686f68, 0x2318fa4e, 0x7ae6459a]


@pytest.mark.parametrize("kmax", [20])
def test_sequential_bitonic_matches_golden(orc, golden, kmax):
    for c in golden["cases"]:
        if c["k"] > kmax:
            continue
        x = orc.generate_input(1 << c["k"], c["seed"])
        i32 = orc.sequential_bitonic_i32(x.view(np.int32))
        assert h(orc.fnv1a64(i32)) == c["i32_asc_fnv"]
        u32 = orc.bitonic_u32(x)
        assert h(orc.fnv1a64(u32)) == c["u32_asc_fnv"]
        assert "%08x" % u32[0] == c["u32_first"] and "%08x" % u32[-1] == c["u32_last"]
        d32 = orc.bitonic_u32(x, descending=True)
        assert h(orc.fnv1a64(d32)) == c["u32_desc_fnv"]


def test_quicksort_port_matches_golden(orc, golden):
    for c in golden["cases"]:
        x = orc.generate_input(1 << c["k"], c["seed"])
        assert h(orc.fnv1a64(orc.quicksort_i32(x.view(np.int32)))) == c["i32_asc_fnv"]
        assert h(orc.fnv1a64(orc.quicksort_u32(x))) == c["u32_asc_fnv"]
        assert h(orc.fnv1a64(orc.quicksort_u32(x, True))) == c["u32_desc_fnv"]


def test_survey_appendix_a_first_last(orc):
    # First/last keys of SURVEY.md Appendix A (computed with the reference).
    table = {1: ("2318fa4e", "bb686f68", "bb686f68"),
             3: ("1bf14b09", "ecfc6738", "915bd1b4"),
             12: ("000f7c46", "fff4fd94", "800ece2c"),
             16: ("0001d22e", "fffdd246", "800107c2"),
             20: ("00003b70", "ffffe407", "80001c86")}
    for k, (f, l, i0) in table.items():
        x = orc.generate_input(1 << k, 1)
        u = orc.quicksort_u32(x)
        i = orc.quicksort_i32(x.view(np.int32)).view(np.uint32)
        assert ("%08x" % u[0], "%08x" % u[-1], "%08x" % i[0]) == (f, l, i0)


def test_batched_golden(orc, golden):
    b = golden["batched"]
    x = orc.generate_input(b["n_per"] * b["batch"], b["seed"])
    assert h(orc.fnv1a64(x)) == b["input_fnv"]
    s = np.sort(x.reshape(b["batch"], b["n_per"]), axis=1)
    assert h(orc.fnv1a64(s)) == b["u32_asc_fnv"]
    assert "%08x" % s[0, 0] == b["seg0_first"]
    # the C batched restatement on a slice (full size is covered by np.sort)
    part = orc.bitonic_batched_u32(x[: 64 * b["n_per"]], b["n_per"])
    assert (part.reshape(64, -1) == s[:64]).all()


def test_small_vectors_exact(orc, golden):
    for c in golden["small"]:
        x = np.array(c["input"], dtype=np.int32)
        assert (orc.generate_input(1 << c["k"], c["seed"]).view(np.int32) == x).all()
        assert orc.sequential_bitonic_i32(x).tolist() == c["i32_asc"]


def test_known_answers(orc, golden):
    for c in golden["kat"]:
        x = np.array(c["input"], dtype=np.int32)
        if x.size >= 2 and (x.size & (x.size - 1)) == 0:
            assert orc.sequential_bitonic_i32(x).tolist() == c["i32_asc"], c["name"]
        assert orc.quicksort_i32(x).tolist() == c["i32_asc"], c["name"]


def test_predicted_counts(orc, golden):
    for c in golden["counts"]:
        assert orc.predicted_counts(c["k"]) == (c["rounds"], c["compare_exchanges"])


def test_invalid_sizes(orc):
    with pytest.raises(ValueError):
        orc.sequential_bitonic_i32(np.zeros(6, np.int32))
    with pytest.raises(ValueError):
        orc.sequential_bitonic_i32(np.zeros(1, np.int32))


def test_all_permutations_of_8(orc):
    # test_verify.cpp:120-132: all 8! permutations sort through the network
    import itertools
    for p in itertools.permutations(range(1, 9)):
        assert orc.sequential_bitonic_i32(np.array(p, np.int32)).tolist() == list(range(1, 9))


def test_zero_one_exhaustive(orc):
    # verify.cpp:118-153: every binary vector of length <= 16 sorts
    for k in range(1, 5):
        n = 1 << k
        words = np.arange(1 << n, dtype=np.uint64)
        bits = ((words[:, None] >> np.arange(n, dtype=np.uint64)) & 1).astype(np.uint32)
        for row in bits[:: max(1, len(bits) // 4096)]:
            out = orc.bitonic_u32(row)
            assert (np.diff(out.astype(np.int64)) >= 0).all()


def test_bitonic_64_orders(orc):
    """64-bit oracle: uint64 / int64 orders equal a sort; float64 equals
    IEEE totalOrder (bit patterns, so -0.0 < +0.0 and NaNs at the ends)."""
    rng = np.random.default_rng(64)
    for k in (1, 2, 5, 10):
        for dt in (np.uint64, np.int64):
            info = np.iinfo(dt)
            x = rng.integers(info.min, info.max, size=1 << k, dtype=dt, endpoint=True)
            x[: x.size // 2] = x[x.size // 2:]  # ties
            for desc in (False, True):
                want = np.sort(x)[::-1] if desc else np.sort(x)
                assert (orc.bitonic_64(x, desc) == want).all()
        f = rng.standard_normal(1 << k)
        sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, -np.nan, 5e-324, -5e-324])
        f[: min(f.size, sp.size)] = sp[: min(f.size, sp.size)]
        u = f.view(np.uint64)
        tok = np.where(u >> np.uint64(63) == 1, ~u, u | np.uint64(1 << 63))
        want = f[np.argsort(tok, kind="stable")]
        assert (orc.bitonic_64(f).view(np.uint64) == want.view(np.uint64)).all()
    with pytest.raises(ValueError):
        orc.bitonic_64(np.zeros(3, np.uint64))


# ---- cross-check against the compiled reference itself -------------------

def test_oracle_vs_reference_random(orc, ref):
    rng = np.random.default_rng(7)
    for k in range(1, 15):
        for _ in range(3):
            x = rng.integers(-2**31, 2**31, size=1 << k, dtype=np.int64).astype(np.int32)
            assert (orc.sequential_bitonic_i32(x) == ref.sequential_bitonic_sort(x)).all()
            assert (orc.quicksort_i32(x) == ref.quicksort(x)).all()


def test_oracle_generate_input_vs_reference(orc, ref):
    if not ref.has_bench:
        pytest.skip("reference bench.cpp not compiled")
    for n, seed in [(1, 0), (7, 3), (1000, 0x5EED), (1 << 16, 42)]:
        assert (orc.generate_input(n, seed).view(np.int32) == ref.generate_input(n, seed)).all()


def test_pad_to_pow2_vs_reference(orc, ref):
    if not ref.has_bench:
        pytest.skip("reference bench.cpp not compiled")
    for n in [1, 2, 3, 5, 8, 1000]:
        x = np.arange(n, dtype=np.int32)[::-1].copy()
        assert (orc.pad_to_pow2_i32(x) == ref.pad_to_pow2(x)).all()


def test_reference_zero_one_and_counts(ref, orc):
    for k in range(1, 7):
        assert ref.check_zero_one(k)
    for k in range(1, 30):
        assert ref.predicted_counts(k) == orc.predicted_counts(k)


def test_oracle_at_2_24_matches_reference_digest(orc, golden):
    """The large fixture (reference sequential_bitonic_sort at 2^24) pins the
    oracle's generator and sort at the top of the CPU-checkable range."""
    c = [c for c in golden["large"] if c["k"] == 24][0]
    x = orc.generate_input(1 << 24, 1)
    assert h(orc.fnv1a64(x)) == c["input_fnv"]
    assert h(orc.fnv1a64(orc.quicksort_u32(x))) == c["u32_asc_fnv"]


def _network_virtual(x, k, nreal, X=None):
    """The bitonic network on 2^k slots with slots >= nreal virtual (+inf)
    and the virtual plans' direction rule (phase p descending iff bit p of
    i ^ (nreal - 1) is set).  Returns the output and whether any
    compare-exchange moved a real key into a virtual slot."""
    n = 1 << k
    a = np.full(n, 0xFFFFFFFF, dtype=np.uint64)
    a[:nreal] = x
    X = nreal - 1 if X is None else X
    leaked = False
    idx = np.arange(n)
    for p in range(1, k + 1):
        for s in range(p - 1, -1, -1):
            lo = idx[(idx >> s) & 1 == 0]
            hi = lo | (1 << s)
            desc = ((lo ^ X) >> p) & 1 if p < k else np.zeros_like(lo)
            x0, x1 = a[lo], a[hi]
            mn, mx = np.minimum(x0, x1), np.maximum(x0, x1)
            new_lo = np.where(desc == 1, mx, mn)
            new_hi = np.where(desc == 1, mn, mx)
            # a real key (index < nreal) must never land on a virtual slot
            moved = (hi >= nreal) & (new_hi != 0xFFFFFFFF)
            leaked |= bool(moved.any())
            a[lo], a[hi] = new_lo, new_hi
    return a[:nreal].astype(np.uint32), leaked


@pytest.mark.parametrize("k", [3, 5, 8, 11])
def test_virtual_padding_direction_rule(k):
    """Virtual padding (no padded copy) is exact: with the direction rule of
    the virtual plans, no compare-exchange ever moves a real key into a
    virtual slot, for every length 2^(k-1) < n <= 2^k, and the real prefix
    comes out sorted (bench.cpp:366-377's pad + sort + truncate)."""
    rng = np.random.default_rng(k)
    ns = range((1 << (k - 1)) + 1, (1 << k) + 1) if k <= 8 else \
        sorted(set(rng.integers((1 << (k - 1)) + 1, (1 << k) + 1, 40).tolist()))
    for n in ns:
        x = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
        x[: n // 5] = 0xFFFFFFFF  # real keys equal to the padding value
        got, leaked = _network_virtual(x, k, n)
        assert not leaked, n
        assert (got == np.sort(x)).all(), n
    # with the standard rule (X = 0) real keys do leak into the padding:
    # the direction rule is what makes the copy unnecessary
    n = (1 << k) - 3
    x = rng.integers(0, 2**31, n, dtype=np.uint64).astype(np.uint32)
    _, leaked = _network_virtual(x, k, n, X=0)
    assert leaked
