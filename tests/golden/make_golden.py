"""Generate tests/golden/golden.json from the REFERENCE's own code.

Run in the dev container (needs oracle/_ref/libbitonic_ref.so, built by
`make -C oracle` from /root/reference/proj/src).  Every expected output here
comes from the reference library, never from the code under test:

* inputs: bitonic::generate_input(n, seed) (bench.cpp:354-364)
* "i32_asc": bitonic::sequential_bitonic_sort (engine.cpp:248-266)
* "u32_asc": sequential_bitonic_sort on the sign-flipped keys, flipped back
  (u32 order of x == i32 order of x ^ 0x80000000)
* "quicksort": bitonic::reference_quicksort (verify.cpp:109-116)
* digest: FNV-1a 64 over the little-endian key bytes.

Also records the known-answer vectors of the reference's tests
(test_engine.cpp:217-235, :289-293; test_verify.cpp:16-20) with the
reference's outputs, and the launch/CE closed forms it checks.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

FLIP = np.uint32(0x80000000)


def fnv(a):
    a = np.ascontiguousarray(a)
    h = 0xcbf29ce484222325
    b = a.tobytes()
    # numpy-vectorised FNV is awkward; use the C oracle for speed when present
    return oracle.oracle().fnv1a64(a) if len(b) > 4096 else _fnv_py(b, h)


def _fnv_py(b, h):
    for x in b:
        h ^= x
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def main():
    ref = oracle.reference()
    assert ref is not None and ref.has_bench, "build oracle/_ref first (make -C oracle)"
    out = {"generator": "tests/golden/make_golden.py (reference code via oracle/_ref)",
           "digest": "fnv1a64 over little-endian uint32/int32 key bytes",
           "cases": [], "kat": [], "small": [], "counts": []}
    for k in [1, 2, 3, 4, 8, 12, 16, 20, 22]:
        n = 1 << k
        for seed in ([1, 2] if k <= 20 else [1]):
            x = ref.generate_input(n, seed)             # int32 bits
            u = x.view(np.uint32)
            i32 = ref.sequential_bitonic_sort(x)
            u32 = (ref.sequential_bitonic_sort((u ^ FLIP).view(np.int32)).view(np.uint32) ^ FLIP)
            qs = ref.quicksort(x)
            assert (qs == i32).all()
            out["cases"].append({
                "k": k, "seed": seed,
                "input_fnv": "%016x" % fnv(u),
                "i32_asc_fnv": "%016x" % fnv(i32),
                "u32_asc_fnv": "%016x" % fnv(u32),
                "u32_desc_fnv": "%016x" % fnv(u32[::-1].copy()),
                "i32_desc_fnv": "%016x" % fnv(i32[::-1].copy()),
                "u32_first": "%08x" % u32[0], "u32_last": "%08x" % u32[-1],
                "i32_first": "%08x" % (int(i32[0]) & 0xFFFFFFFF),
            })
    # batched: generate_input(2^24, 1) as 4096 arrays of 2^12, each u32-ascending
    x = ref.generate_input(1 << 24, 1).view(np.uint32).reshape(4096, 4096)
    segs = np.empty_like(x)
    for r in range(4096):
        segs[r] = ref.sequential_bitonic_sort((x[r] ^ FLIP).view(np.int32)).view(np.uint32) ^ FLIP
    out["batched"] = {"n_per": 4096, "batch": 4096, "seed": 1,
                      "input_fnv": "%016x" % fnv(x),
                      "u32_asc_fnv": "%016x" % fnv(segs),
                      "seg0_first": "%08x" % segs[0, 0]}
    # small explicit vectors (input + reference output) for exact comparison
    for k, seed in [(5, 11), (7, 12), (10, 13)]:
        x = ref.generate_input(1 << k, seed)
        out["small"].append({"k": k, "seed": seed,
                             "input": [int(v) for v in x],
                             "i32_asc": [int(v) for v in ref.sequential_bitonic_sort(x)]})
    # known-answer tests from the reference's own suites
    kat = [
        ("canonical bitonic sequence (test_engine.cpp:217-227)", [1, 5, 9, 10, 12, 8, 7, 2]),
        ("reversed quad (test_engine.cpp:289-293)", [4, 3, 2, 1]),
        ("iota(-12) fixed point (test_engine.cpp:229-235)", list(range(-12, 52))),
        ("all equal", [7] * 16),
        ("extremes", [2**31 - 1, -2**31, 0, -1, 1, 2**31 - 1, -2**31, 5]),
    ]
    for name, v in kat:
        a = np.array(v, dtype=np.int32)
        out["kat"].append({"name": name, "input": v,
                           "i32_asc": [int(t) for t in ref.sequential_bitonic_sort(a)]})
    for k in range(1, 33):
        r, c = ref.predicted_counts(k)
        out["counts"].append({"k": k, "rounds": r, "compare_exchanges": c})
    out["large"] = large_cases(ref)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


def large_cases(ref):
    """Digests at north_star's upper sizes: 2^24 through the reference's
    sequential_bitonic_sort, 2^28 through reference_quicksort (the bitonic
    network would take minutes on one core; any correct sort of payload-free
    keys gives the same bytes)."""
    cases = []
    for k, how in [(24, "sequential_bitonic_sort"), (28, "reference_quicksort")]:
        x = ref.generate_input(1 << k, 1)
        u = x.view(np.uint32)
        sort = ref.sequential_bitonic_sort if how == "sequential_bitonic_sort" else ref.quicksort
        i32 = sort(x)
        u32 = sort((u ^ FLIP).view(np.int32)).view(np.uint32) ^ FLIP
        cases.append({"k": k, "seed": 1, "reference_function": how,
                      "input_fnv": "%016x" % fnv(u),
                      "i32_asc_fnv": "%016x" % fnv(i32),
                      "u32_asc_fnv": "%016x" % fnv(u32),
                      "u32_desc_fnv": "%016x" % fnv(u32[::-1].copy()),
                      "u32_first": "%08x" % u32[0], "u32_last": "%08x" % u32[-1],
                      "u32_median": "%08x" % u32[u32.size // 2]})
        print("large case", k, "done", flush=True)
    return cases


if __name__ == "__main__":
    if sys.argv[1:] == ["--large-only"]:
        # add / refresh only the large digests in the existing fixture
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
        with open(path) as f:
            cur = json.load(f)
        cur["large"] = large_cases(oracle.reference())
        with open(path, "w") as f:
            json.dump(cur, f, indent=1)
        print("updated", path)
    else:
        main()
