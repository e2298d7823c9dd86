"""CPU model of the merge-path variant (b200_bitonic_sort_mergepath_*,
csrc/merge_split.cuh mergepath_* kernels): the claim it rests on, checked
with numpy at small sizes.

Phase p of the bitonic network merges run pairs with the bitonic merger.
Its first p - C half-cleaner steps only move keys between 2^C-key windows,
and afterwards window t of a pair holds exactly the keys of ranks
[t 2^C, (t+1) 2^C) of the pair's merge.  The variant computes that routing
with a co-rank search per window (A first on ties, as corank_global) and
runs the merger's last C steps on each window laid out as A part ascending
+ B part reversed.  Pure test infrastructure (no GPU, no product code)."""
import numpy as np
import pytest


def corank(d, A, B):
    """Keys of A among the first d of merge(A, B), A first on ties."""
    lo, hi = max(0, d - len(B)), min(d, len(A))
    while lo < hi:
        mid = (lo + hi) // 2
        if A[mid] <= B[d - mid - 1]:
            lo = mid + 1
        else:
            hi = mid
    return lo


def half_cleaners(x, bits):
    """Ascending bitonic-merger steps on the given bits, in order."""
    x = x.copy()
    idx = np.arange(x.size)
    for b in bits:
        lo = idx[(idx >> b) & 1 == 0]
        hi = lo | (1 << b)
        a, c = x[lo], x[hi]
        x[lo], x[hi] = np.minimum(a, c), np.maximum(a, c)
    return x


def mergepath_sort(x, tile_bits, C):
    n = x.size
    k = n.bit_length() - 1
    N = 1 << C
    cur = np.concatenate([np.sort(t) for t in x.reshape(-1, 1 << tile_bits)])
    for p in range(tile_bits + 1, k + 1):
        half = 1 << (p - 1)
        out = np.empty_like(cur)
        for t in range(n // N):
            o = t * N
            base = o & ~((half << 1) - 1)
            d = o - base
            A, B = cur[base:base + half], cur[base + half:base + 2 * half]
            i0 = corank(d, A, B)
            i1 = half if d + N == 2 * half else corank(d + N, A, B)
            j1 = d + N - i1
            j0 = j1 - (N - (i1 - i0))
            window = np.concatenate([A[i0:i1], B[j0:j1][::-1]])  # bitonic
            out[o:o + N] = half_cleaners(window, range(C - 1, -1, -1))
        cur = out
    return cur


@pytest.mark.parametrize("k,tile_bits,C", [(6, 3, 2), (8, 4, 3), (9, 4, 3), (10, 5, 3), (10, 4, 4)])
@pytest.mark.parametrize("kind", ["random", "few_values", "sorted", "reversed", "equal"])
def test_mergepath_model_sorts(k, tile_bits, C, kind):
    rng = np.random.default_rng(k * 31 + C)
    n = 1 << k
    x = {"random": rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32),
         "few_values": rng.integers(0, 4, n).astype(np.uint32),
         "sorted": np.arange(n, dtype=np.uint32),
         "reversed": np.arange(n, dtype=np.uint32)[::-1].copy(),
         "equal": np.full(n, 7, dtype=np.uint32)}[kind]
    assert (mergepath_sort(x, tile_bits, C) == np.sort(x)).all()


@pytest.mark.parametrize("p,C", [(5, 2), (6, 3), (7, 3), (8, 4)])
def test_windows_match_the_network_half_cleaners(p, C):
    """After the first p - C half-cleaner steps of the network's merger (on A
    ascending + B descending), each 2^C window holds the same multiset as the
    co-rank window of merge(A, B) -- the routing the variant computes."""
    rng = np.random.default_rng(p * 7 + C)
    for trial in range(20):
        half = 1 << (p - 1)
        vals = 3 if trial % 2 else 2**32
        A = np.sort(rng.integers(0, vals, half).astype(np.uint64))
        B = np.sort(rng.integers(0, vals, half).astype(np.uint64))
        net = half_cleaners(np.concatenate([A, B[::-1]]), range(p - 1, C - 1, -1))
        N = 1 << C
        for t in range(2 * half // N):
            d = t * N
            i0, i1 = corank(d, A, B), corank(d + N, A, B)
            j0, j1 = d - i0, d + N - i1
            want = np.sort(np.concatenate([A[i0:i1], B[j0:j1]]))
            assert (np.sort(net[d:d + N]) == want).all(), (p, C, trial, t)
