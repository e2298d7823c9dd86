/*
 * oracle/bitonic_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's CPU algorithm for the hot path
 * (arxiv/paper_1506_01446 artifact, /root/reference/proj).  It is the CHECKER
 * for the CUDA sort, never the thing measured or shipped: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product path (paper_1506_01446_b200) never links it.
 *
 * Parity is pinned: tests/test_oracle.py checks every function here against
 * (a) the golden digests in tests/golden/ (generated from the reference's own
 * code compiled into oracle/_ref by oracle/Makefile), and (b) the reference
 * library itself when oracle/_ref is present.
 *
 * Restated functions (reference file:line):
 *   oracle_mt19937_64_*       std::mt19937_64 as used by generate_input,
 *                             proj/src/bench.cpp:354-364 and
 *                             proj/tests/oracles.hpp:34-42 (C++11 [rand.eng.mers])
 *   oracle_generate_input     proj/src/bench.cpp:354-364
 *   oracle_pad_to_pow2_i32    proj/src/bench.cpp:366-377
 *   oracle_sequential_bitonic_i32
 *                             proj/src/engine.cpp:248-266 (+ pair_base :26-29,
 *                             compare_exchange :16-22)
 *   oracle_bitonic_u32        same network, uint32 order, with the new
 *                             `descending` argument north_star asks for
 *   oracle_bitonic_u64        same network on 64-bit keys (int64 via key_xor)
 *   oracle_quicksort_i32      proj/src/verify.cpp:17-75, :109-116
 *   oracle_predicted_counts   proj/src/schedule.cpp:71-78
 *   oracle_fnv1a64            digest used for the golden fixtures (SURVEY.md
 *                             Appendix A)
 */
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_INVALID_SIZE 1

/* ---------------------------------------------------------------------- */
/* std::mt19937_64 (w=64, n=312, m=156, r=31).  The C++ standard pins the   */
/* algorithm and its seeding, so the reference's generate_input is fully    */
/* determined by (size, seed).                                              */
/* ---------------------------------------------------------------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
} oracle_mt64;

static void mt64_seed(oracle_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i) {
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) +
               (uint64_t)i;
  }
  s->idx = 312;
}

static uint64_t mt64_next(oracle_mt64* s) {
  static const uint64_t kUpper = 0xFFFFFFFF80000000ULL;
  static const uint64_t kLower = 0x7FFFFFFFULL;
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (s->mt[i] & kUpper) | (s->mt[(i + 1) % 312] & kLower);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* generate_input (bench.cpp:354-364): key_i = low 32 bits of the i-th draw. */
int oracle_generate_input(uint32_t* out, uint64_t n, uint64_t seed) {
  if (n < 1) return ORACLE_INVALID_SIZE;
  oracle_mt64 s;
  mt64_seed(&s, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = (uint32_t)mt64_next(&s);
  return ORACLE_OK;
}

/* pad_to_pow2 (bench.cpp:366-377): append INT32_MAX up to max(2, bit_ceil).
 * Writes into out (capacity >= returned length); returns padded length. */
uint64_t oracle_pad_to_pow2_i32(const int32_t* in, uint64_t n, int32_t* out) {
  if (n < 1) return 0;
  uint64_t m = 2;
  while (m < n) m <<= 1;
  memcpy(out, in, n * sizeof(int32_t));
  for (uint64_t i = n; i < m; ++i) out[i] = INT32_MAX;
  return m;
}

static int is_pow2_ge2(uint64_t n) { return n >= 2 && (n & (n - 1)) == 0; }

/* pair_base (engine.cpp:26-29): t with a zero bit inserted at the stride. */
static inline uint64_t pair_base(uint64_t t, uint64_t stride) {
  const uint64_t low = stride - 1;
  return ((t & ~low) << 1) | (t & low);
}

/* sequential_bitonic_sort (engine.cpp:248-266): phase p = 1..k, step s = p..1,
 * stride 2^(s-1), direction ascending iff (i & 2^p) == 0, swap only when
 * strictly out of order (compare_exchange, engine.cpp:16-22). */
int oracle_sequential_bitonic_i32(int32_t* a, uint64_t n) {
  if (!is_pow2_ge2(n)) return ORACLE_INVALID_SIZE;
  unsigned k = 0;
  while ((1ULL << k) < n) ++k;
  for (unsigned phase = 1; phase <= k; ++phase) {
    const uint64_t span = 1ULL << phase;
    for (unsigned step = phase; step >= 1; --step) {
      const uint64_t stride = 1ULL << (step - 1);
      for (uint64_t t = 0; t < n / 2; ++t) {
        const uint64_t i = pair_base(t, stride);
        const int asc = (i & span) == 0;
        int32_t x = a[i], y = a[i + stride];
        if (asc ? (x > y) : (x < y)) {
          a[i] = y;
          a[i + stride] = x;
        }
      }
    }
  }
  return ORACLE_OK;
}

/* Same network on uint32 keys with an overall direction.  Descending output
 * equals std::sort(..., std::greater<>()) (the direction
 * argument is new; the reference is ascending-only). */
int oracle_bitonic_u32(uint32_t* a, uint64_t n, int descending) {
  if (!is_pow2_ge2(n)) return ORACLE_INVALID_SIZE;
  unsigned k = 0;
  while ((1ULL << k) < n) ++k;
  for (unsigned phase = 1; phase <= k; ++phase) {
    const uint64_t span = 1ULL << phase;
    for (unsigned step = phase; step >= 1; --step) {
      const uint64_t stride = 1ULL << (step - 1);
      for (uint64_t t = 0; t < n / 2; ++t) {
        const uint64_t i = pair_base(t, stride);
        int asc = (i & span) == 0;
        if (descending) asc = !asc;
        uint32_t x = a[i], y = a[i + stride];
        if (asc ? (x > y) : (x < y)) {
          a[i] = y;
          a[i + stride] = x;
        }
      }
    }
  }
  return ORACLE_OK;
}

/* Key-value: the same network (engine.cpp:248-266) with a 32-bit payload
 * moved alongside every key swap.  compare_exchange swaps only when strictly
 * out of order (engine.cpp:16-22), so the payload order of equal keys is the
 * network's own (not stable) -- the GPU kernels must reproduce it exactly.
 * key_xor: 0 = uint32 order, 0x80000000 = int32 order. */
int oracle_bitonic_pairs(uint32_t* k, uint32_t* v, uint64_t n, int descending,
                         uint32_t key_xor) {
  if (!is_pow2_ge2(n)) return ORACLE_INVALID_SIZE;
  unsigned lg = 0;
  while ((1ULL << lg) < n) ++lg;
  for (unsigned phase = 1; phase <= lg; ++phase) {
    const uint64_t span = 1ULL << phase;
    for (unsigned step = phase; step >= 1; --step) {
      const uint64_t stride = 1ULL << (step - 1);
      for (uint64_t t = 0; t < n / 2; ++t) {
        const uint64_t i = pair_base(t, stride);
        int asc = (i & span) == 0;
        if (descending) asc = !asc;
        const uint32_t x = k[i] ^ key_xor, y = k[i + stride] ^ key_xor;
        if (asc ? (x > y) : (x < y)) {
          uint32_t tk = k[i];
          k[i] = k[i + stride];
          k[i + stride] = tk;
          uint32_t tv = v[i];
          v[i] = v[i + stride];
          v[i + stride] = tv;
        }
      }
    }
  }
  return ORACLE_OK;
}

/* 64-bit keys (the paper's future-work types): the same
 * network (engine.cpp:248-266) on uint64 keys compared after XOR with
 * key_xor (1 << 63 = int64 order).  float64 order is the caller's totalOrder
 * bit map (oracle/__init__.py) onto this uint64 order. */
int oracle_bitonic_u64(uint64_t* a, uint64_t n, int descending, uint64_t key_xor) {
  if (!is_pow2_ge2(n)) return ORACLE_INVALID_SIZE;
  unsigned k = 0;
  while ((1ULL << k) < n) ++k;
  for (unsigned phase = 1; phase <= k; ++phase) {
    const uint64_t span = 1ULL << phase;
    for (unsigned step = phase; step >= 1; --step) {
      const uint64_t stride = 1ULL << (step - 1);
      for (uint64_t t = 0; t < n / 2; ++t) {
        const uint64_t i = pair_base(t, stride);
        int asc = (i & span) == 0;
        if (descending) asc = !asc;
        const uint64_t x = a[i] ^ key_xor, y = a[i + stride] ^ key_xor;
        if (asc ? (x > y) : (x < y)) {
          const uint64_t tk = a[i];
          a[i] = a[i + stride];
          a[i + stride] = tk;
        }
      }
    }
  }
  return ORACLE_OK;
}

/* Batched: `batch` contiguous arrays of n_per keys, each sorted on its own. */
int oracle_bitonic_batched_u32(uint32_t* a, uint64_t n_per, uint64_t batch,
                               int descending) {
  if (!is_pow2_ge2(n_per)) return ORACLE_INVALID_SIZE;
  for (uint64_t b = 0; b < batch; ++b) {
    int rc = oracle_bitonic_u32(a + b * n_per, n_per, descending);
    if (rc) return rc;
  }
  return ORACLE_OK;
}

/* ---------------------------------------------------------------------- */
/* reference_quicksort (verify.cpp:17-75, :109-116): median-of-three Hoare  */
/* partition, recurse into the smaller side, insertion sort at <= 16        */
/* elements, heapsort once the depth budget 2*log2(n) runs out.             */
/* ---------------------------------------------------------------------- */
static void insertion_sort_i32(int32_t* first, int32_t* last) {
  for (int32_t* it = first + 1; it < last; ++it) {
    const int32_t v = *it;
    int32_t* pos = it;
    while (pos > first && pos[-1] > v) {
      pos[0] = pos[-1];
      --pos;
    }
    *pos = v;
  }
}

static int32_t median3(int32_t a, int32_t b, int32_t c) {
  if (a < b) {
    if (b < c) return b;
    return a < c ? c : a;
  }
  if (a < c) return a;
  return b < c ? c : b;
}

static void sift_down_i32(int32_t* h, ptrdiff_t start, ptrdiff_t len) {
  ptrdiff_t root = start;
  for (;;) {
    ptrdiff_t child = 2 * root + 1;
    if (child >= len) return;
    if (child + 1 < len && h[child] < h[child + 1]) ++child;
    if (h[root] >= h[child]) return;
    int32_t t = h[root];
    h[root] = h[child];
    h[child] = t;
    root = child;
  }
}

/* make_heap + sort_heap fallback (verify.cpp:42-46).  Any correct heapsort
 * yields the same (unique) sorted keys. */
static void heapsort_i32(int32_t* first, int32_t* last) {
  const ptrdiff_t len = last - first;
  for (ptrdiff_t s = len / 2 - 1; s >= 0; --s) sift_down_i32(first, s, len);
  for (ptrdiff_t end = len - 1; end > 0; --end) {
    int32_t t = first[0];
    first[0] = first[end];
    first[end] = t;
    sift_down_i32(first, 0, end);
  }
}

static void quicksort_rec_i32(int32_t* first, int32_t* last, int depth) {
  while (last - first > 16) {
    if (depth-- == 0) {
      heapsort_i32(first, last);
      return;
    }
    const int32_t pivot = median3(*first, first[(last - first) / 2], last[-1]);
    int32_t* lo = first - 1;
    int32_t* hi = last;
    for (;;) {
      do ++lo; while (*lo < pivot);
      do --hi; while (*hi > pivot);
      if (lo >= hi) break;
      int32_t t = *lo;
      *lo = *hi;
      *hi = t;
    }
    int32_t* mid = hi + 1;
    if (mid - first < last - mid) {
      quicksort_rec_i32(first, mid, depth);
      first = mid;
    } else {
      quicksort_rec_i32(mid, last, depth);
      last = mid;
    }
  }
  insertion_sort_i32(first, last);
}

void oracle_quicksort_i32(int32_t* a, uint64_t n) {
  if (n < 2) return;
  unsigned bw = 0;
  while (bw < 64 && (n >> bw) != 0) ++bw; /* std::bit_width */
  quicksort_rec_i32(a, a + n, 2 * ((int)bw - 1));
}

/* uint32 order through the exact sign-flip bridge:
 * u32 order of x == i32 order of (x ^ 0x80000000). */
void oracle_quicksort_u32(uint32_t* a, uint64_t n, int descending) {
  const uint32_t flip = 0x80000000u;
  for (uint64_t i = 0; i < n; ++i) a[i] ^= flip;
  oracle_quicksort_i32((int32_t*)a, n);
  for (uint64_t i = 0; i < n; ++i) a[i] ^= flip;
  if (descending) {
    for (uint64_t i = 0, j = n ? n - 1 : 0; i < j; ++i, --j) {
      uint32_t t = a[i];
      a[i] = a[j];
      a[j] = t;
    }
  }
}

/* predicted_counts (schedule.cpp:71-78). */
int oracle_predicted_counts(unsigned k, uint64_t* rounds, uint64_t* ces) {
  if (k < 1 || k > 48) return ORACLE_INVALID_SIZE;
  *rounds = (uint64_t)k * (k + 1) / 2;
  *ces = (1ULL << (k - 1)) * *rounds;
  return ORACLE_OK;
}

/* FNV-1a 64 over raw bytes (SURVEY.md Appendix A digest). */
uint64_t oracle_fnv1a64(const void* data, uint64_t nbytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ULL;
  for (uint64_t i = 0; i < nbytes; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* Sortedness check in uint32 or int32 order; returns first violation index
 * or UINT64_MAX (validate, verify.cpp:155-165). */
uint64_t oracle_first_violation_u32(const uint32_t* a, uint64_t n,
                                    int descending) {
  for (uint64_t i = 0; i + 1 < n; ++i) {
    if (descending ? (a[i] < a[i + 1]) : (a[i] > a[i + 1])) return i;
  }
  return UINT64_MAX;
}
