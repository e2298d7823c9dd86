/*
 * b200_bitonic.h -- C ABI of the B200-native bitonic sort (sm_100a).
 *
 * Drop-in boundary for the hot path of arxiv/paper_1506_01446's artifact:
 * the reference's C++ entry points (namespace bitonic, /root/reference/proj)
 * sort a power-of-two array of 32-bit keys in place on the CPU.  These C
 * functions replace them with CUDA kernels; C++ callers use the thin shim
 * include/bitonic/gpu_sort.hpp, which maps the status codes below back onto
 * the reference's exception types.  No torch types cross this boundary.
 *
 * Status codes (returned by every function):
 *   0 B200_OK
 *   1 B200_INVALID_SIZE   -> bitonic::invalid_size_error  (error.hpp:11-15):
 *                            n < 2, n not a power of two, n too large
 *   2 B200_CONFIG         -> bitonic::config_error        (error.hpp:19-23):
 *                            bad argument (null pointer, misaligned pointer,
 *                            ngpu not in {1,2,4,8}, bad batch, ...)
 *   3 B200_CUDA_ERROR     CUDA runtime failure (message in last_error)
 *   4 B200_NCCL_ERROR     reserved for the NCCL exchange path
 * There is no CPU fallback: a missing/unsupported GPU is B200_CUDA_ERROR.
 *
 * Device-pointer entry points are stream-ordered and asynchronous: they
 * enqueue kernels on `stream` and return.  The power-of-two 32-bit sorts
 * (u32/i32/f32, batched, pairs) and u64_planes are in place and allocate
 * nothing; the interleaved 64-bit entries, the padded entries (non-power-
 * of-two lengths) and merge / merge_split take scratch from a retained
 * per-device pool (b200_bitonic_release_scratch returns it).  They are
 * reentrant per stream.
 */
#ifndef B200_BITONIC_H
#define B200_BITONIC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Compatible with the CUDA runtime's own typedef. */
struct CUstream_st;
typedef struct CUstream_st* b200_stream_t;

enum {
  B200_OK = 0,
  B200_INVALID_SIZE = 1,
  B200_CONFIG = 2,
  B200_CUDA_ERROR = 3,
  B200_NCCL_ERROR = 4
};

/* In-place sort of n uint32 keys at device pointer d_keys.
 * Replaces bitonic::sequential_bitonic_sort(std::span<int32_t>)
 * (proj/include/bitonic/engine.hpp:102-104, proj/src/engine.cpp:248-266)
 * and bitonic::execute(build_plan(...), keys, workers) (engine.hpp:77-92),
 * with the uint32 key order BASELINE.json's metric uses and a new
 * `descending` flag (0 = ascending, the reference's only order; 1 =
 * std::greater order).  n must be a power of two >= 2 (same contract as
 * engine.cpp:250-253); d_keys must be 16-byte aligned when n >= 4. */
int b200_bitonic_sort_u32(uint32_t* d_keys, uint64_t n, int descending,
                          b200_stream_t stream);

/* Same with the reference's own key type and order (signed int32,
 * engine.hpp:13-15).  Bit-identical to sequential_bitonic_sort's output. */
int b200_bitonic_sort_i32(int32_t* d_keys, uint64_t n, int descending,
                          b200_stream_t stream);

/* Merge-path variant of the same sort (keys only; identical output bytes):
 * the tile sort leaves every 2^13-key tile ascending, then each global phase
 * p = 14..log2(n) is ONE pass -- a co-rank partition of every run pair's
 * merge into 2^13-key output tiles (the keys the phase's large-stride
 * half-cleaner steps would route to each tile) and the bitonic merger's last
 * 13 steps on each tile -- ping-ponging through an n-key scratch buffer from
 * the retained pool (log2(n) - 12 passes; 2^28: 16 against the network's
 * 29).  n a power of two >= 2; n <= 2^13 runs the network sort.  Not part of
 * the reference's interface: an option for callers that only need the
 * sorted keys. */
int b200_bitonic_sort_mergepath_u32(uint32_t* d_keys, uint64_t n, int descending,
                                    b200_stream_t stream);
int b200_bitonic_sort_mergepath_i32(int32_t* d_keys, uint64_t n, int descending,
                                    b200_stream_t stream);

/* `batch` independent contiguous arrays of n_per_array keys each, every one
 * sorted on its own (BASELINE config "4096 arrays of 2^12").  n_per_array
 * must be a power of two >= 2; batch >= 1. */
int b200_bitonic_sort_u32_batched(uint32_t* d_keys, uint64_t n_per_array,
                                  uint64_t batch, int descending,
                                  b200_stream_t stream);
int b200_bitonic_sort_i32_batched(int32_t* d_keys, uint64_t n_per_array,
                                  uint64_t batch, int descending,
                                  b200_stream_t stream);

/* Key-value sort: d_vals[i] (a 32-bit payload) moves with d_keys[i].  The
 * network is the reference's exactly (same compare-exchange pairs and
 * directions, swap only when strictly out of order, engine.cpp:16-22), so
 * the payload order of equal keys is the reference network's own -- not
 * stable, but bit-identical to sequential_bitonic_sort carrying a payload.
 * n must be a power of two >= 2; both pointers 16-byte aligned. */
int b200_bitonic_sort_pairs_u32(uint32_t* d_keys, uint32_t* d_vals, uint64_t n,
                                int descending, b200_stream_t stream);
int b200_bitonic_sort_pairs_i32(int32_t* d_keys, uint32_t* d_vals, uint64_t n,
                                int descending, b200_stream_t stream);
int b200_bitonic_sort_pairs_u32_batched(uint32_t* d_keys, uint32_t* d_vals,
                                        uint64_t n_per_array, uint64_t batch,
                                        int descending, b200_stream_t stream);

/* float32 keys (the paper's future-work key types): sorted
 * by IEEE-754 totalOrder -- -NaN < -inf < ... < -0.0 < +0.0 < ... < +inf <
 * +NaN -- via the order-preserving bit map f -> f ^ (sign ? ~0 : 0x80000000)
 * applied before and undone after the uint32 network (two elementwise
 * passes).  n must be a power of two >= 2; use b200_bitonic_sort_padded_*
 * semantics via the Python sort_padded_ for other lengths. */
int b200_bitonic_sort_f32(float* d_keys, uint64_t n, int descending,
                          b200_stream_t stream);

/* 64-bit keys (the paper's other future-work key types, PAPER.md:125:
 * 64-bit integers and doubles).  The network runs on two word planes (hi,
 * lo) compared lexicographically, 16 keys per thread; the interleaved entry
 * points split the array into a stream-ordered scratch pair of planes, sort
 * and join back (float64: IEEE totalOrder like b200_bitonic_sort_f32).
 * b200_bitonic_sort_u64_planes sorts keys already held as planes
 * (key i = hi[i] << 32 | lo[i]) in place with no scratch.  n must be a
 * power of two >= 2; pointers 16-byte aligned. */
int b200_bitonic_sort_u64(uint64_t* d_keys, uint64_t n, int descending,
                          b200_stream_t stream);
int b200_bitonic_sort_i64(int64_t* d_keys, uint64_t n, int descending,
                          b200_stream_t stream);
int b200_bitonic_sort_f64(double* d_keys, uint64_t n, int descending,
                          b200_stream_t stream);
int b200_bitonic_sort_u64_planes(uint32_t* d_hi, uint32_t* d_lo, uint64_t n,
                                 int descending, b200_stream_t stream);

/* Scratch buffers (padded copies, 64-bit word planes, merge coranks, host
 * staging) come from a library-owned stream-ordered pool per device that
 * retains freed memory for the next call; this returns it to the driver.
 * Call only when no sort is in flight. */
int b200_bitonic_release_scratch(void);

/* Any length n >= 1 (the reference's pad_to_pow2 + sort + truncate,
 * bench.cpp:366-377, acceptance.cpp:114-156): when n is not a power of two
 * the keys are copied into a stream-ordered scratch buffer of bit_ceil(n)
 * keys padded with the order's maximum (INT32_MAX for ascending int32, as
 * pad_to_pow2 does), sorted, and the first n keys are copied back.  Powers
 * of two sort in place with no allocation.  From 2^20 keys, lengths up to
 * 1.5 x a power of two 2^j sort the 2^j-key prefix in place, the rest
 * recursively, and merge the two runs through a scratch buffer (same
 * result, about 1.5 instead of 2.2 sorts' work). */
int b200_bitonic_sort_padded_u32(uint32_t* d_keys, uint64_t n, int descending,
                                 b200_stream_t stream);
int b200_bitonic_sort_padded_i32(int32_t* d_keys, uint64_t n, int descending,
                                 b200_stream_t stream);

/* Host-memory convenience entries: H2D copy, sort, D2H copy, synchronous.
 * Mirror sequential_bitonic_sort(std::span<int32_t>) exactly (in place on
 * caller-owned host memory).  Device buffers: one block of 8 bytes per key
 * per pipeline context, grown on demand and kept for later calls (after a
 * 2^30-key sort that is 8 GiB); concurrent callers on one device get their
 * own context (up to 4, then they queue); b200_bitonic_release_scratch
 * frees the blocks. */
int b200_bitonic_sort_host_i32(int32_t* h_keys, uint64_t n, int descending);
int b200_bitonic_sort_host_u32(uint32_t* h_keys, uint64_t n, int descending);

/* Partitioned sort over ngpu GPUs driven from one host thread.
 * d_shards[r] is a device pointer on device devices[r] holding the
 * contiguous slice r (work_slice rule, worker_pool.hpp:22-25) of an array of
 * n_total keys; each shard holds n_total/ngpu keys.  On return rank r holds
 * global sorted positions [r*m, (r+1)*m).  ngpu in {1,2,4,8}; devices may
 * repeat (then the "ranks" share one GPU and exchange through its memory).
 * Each rank sorts locally, then a rank-level bitonic network of merge-split
 * steps runs; the merge kernel reads the partner's shard directly through
 * CUDA peer memory (NVLink).  Synchronous (waits for prior work on the
 * shards' devices).  One scratch shard per rank, the streams and events are
 * kept for the next call with the same devices and size
 * (b200_bitonic_release_scratch frees them); peer access is enabled once per
 * device pair. */
int b200_bitonic_sort_u32_multi(uint32_t* const* d_shards, const int* devices,
                                int ngpu, uint64_t n_total, int descending);

/* One merge-split step (the building block of the partitioned sort, exposed
 * for multi-process drivers that move shards with NCCL): local and partner
 * are sorted (ascending in the order given by key_xor: 0 = uint32,
 * 0x80000000 = int32, ~0 = descending uint32); out receives the m smallest
 * (keep_high = 0) or m largest (keep_high = 1) keys of their union, sorted
 * in the same order.  out must not alias either input.  partner may be a
 * peer-device pointer. */
int b200_bitonic_merge_split_u32(const uint32_t* local, const uint32_t* partner,
                                 uint64_t m, int keep_high, uint32_t key_xor,
                                 uint32_t* out, b200_stream_t stream);

/* General two-way merge of sorted a[0..la) and b[0..lb) (same order
 * convention as merge_split) into out[0..la+lb).  Used by the half-shard
 * exchange of the NCCL partitioned sort: each rank merges the part of its
 * own shard it keeps with the part of the partner shard it received. */
int b200_bitonic_merge_u32(const uint32_t* a, uint64_t la, const uint32_t* b,
                           uint64_t lb, uint32_t key_xor, uint32_t* out,
                           b200_stream_t stream);

/* ---- cross-process peer memory (one process per GPU) ---------------------
 * The fused merge-split of the multi-process partitioned sort reads the
 * partner rank's shard directly over NVLink: each rank allocates its shard
 * buffers with b200_bitonic_ipc_alloc, exchanges the 64-byte handles (any
 * host transport, e.g. torch.distributed), and maps the partner's buffers
 * with b200_bitonic_ipc_open; b200_bitonic_merge_split_u32 then takes the
 * mapped pointer as `partner`.  Handles name whole allocations (offset 0). */
typedef struct {
  unsigned char bytes[64];
} b200_ipc_handle;

int b200_bitonic_ipc_alloc(uint64_t bytes, void** d_ptr, b200_ipc_handle* handle);
int b200_bitonic_ipc_free(void* d_ptr);
int b200_bitonic_ipc_open(const b200_ipc_handle* handle, void** d_ptr);
int b200_bitonic_ipc_close(void* d_ptr);
/* merge_split that also adds, on the stream, the number of keys of `out`
 * taken from `partner` (the keys that crossed the link) to the device
 * counter *d_partner_keys (may be null). */
int b200_bitonic_merge_split_u32_count(const uint32_t* local, const uint32_t* partner,
                                       uint64_t m, int keep_high, uint32_t key_xor,
                                       uint32_t* out, b200_stream_t stream,
                                       uint64_t* d_partner_keys);

/* Device-side ordering between processes: interprocess CUDA events (one per
 * rank and network step, handles exchanged once).  A rank records its event
 * after its merge of a step; the partner's stream waits on it before its
 * next merge -- no host synchronisation of the GPU between steps. */
int b200_bitonic_ipc_event_create(void** event, b200_ipc_handle* handle);
int b200_bitonic_ipc_event_open(const b200_ipc_handle* handle, void** event);
int b200_bitonic_event_destroy(void* event);
int b200_bitonic_event_record(void* event, b200_stream_t stream);
int b200_bitonic_stream_wait_event(b200_stream_t stream, void* event);

/* Stream-ordered device-to-device copy (moves a shard into / out of the
 * IPC buffers). */
int b200_bitonic_copy(void* dst, const void* src, uint64_t bytes, b200_stream_t stream);

/* The reference's benchmark input, generate_input(size, seed)
 * (proj/src/bench.cpp:354-364): key i = the low 32 bits of the i-th output
 * of std::mt19937_64(seed), written to host memory h_out[0..n).  Host only
 * (no GPU needed); n >= 1 else B200_INVALID_SIZE. */
int b200_bitonic_generate_input(uint32_t* h_out, uint64_t n, uint64_t seed);

/* ---- plan introspection (host only, no GPU needed) ----------------------
 * One entry per kernel launch of the sort of `batch` arrays of n keys. */
typedef struct {
  int tile_bits;  /* C: keys per CTA = 2^C                                  */
  int a;          /* low local bits = global bits [0, a)                    */
  int y;          /* high local bits = global bits [y, y + C - a)           */
  int tile_sort;  /* 1 = phases 1..C in one pass                           */
  int segA_hi;    /* tail CE bits segA_hi..0 of phase pA (-1 = none)        */
  int pA;
  int segB_lo;    /* head CE bits C-1..segB_lo (local) of phase pB (-1 = none) */
  int pB;
  uint64_t ctas;  /* grid size                                              */
  uint64_t compare_exchanges; /* CEs executed by this launch               */
  int cluster;    /* CTAs per thread-block cluster (2: the coset is split over */
                  /* two CTAs that exchange keys through DSMEM; else 1)      */
} b200_pass_info;

/* Fills up to max_passes entries; *n_passes receives the plan length. */
int b200_bitonic_plan(uint64_t n, uint64_t batch, b200_pass_info* out,
                      int max_passes, int* n_passes);

/* Runs only pass `pass_index` of the plan for (n_per_array, batch) on
 * uint32 keys (profiling aid: running every index in order equals
 * b200_bitonic_sort_u32_batched).  Returns B200_CONFIG for an index outside
 * the plan. */
int b200_bitonic_run_pass_u32(uint32_t* d_keys, uint64_t n_per_array,
                              uint64_t batch, int descending, int pass_index,
                              b200_stream_t stream);

/* Counters in the reference's cost model (engine.hpp:55-70, account() in
 * engine.cpp:147-173): {kernel_launches, global_reads, global_writes,
 * compare_exchanges}; reads/writes count keys (x4 for bytes). */
int b200_bitonic_counters(uint64_t n, uint64_t batch, uint64_t out[4]);

/* Tuning knobs (process-wide; for benchmarks and tests).  tile_bits in
 * [6, 15] caps the CTA tile (default chosen per n); min_run_bits in [2, 10]
 * is the minimum contiguous run (2^bits keys) every merge pass moves. */
int b200_bitonic_set_tuning(int tile_bits, int min_run_bits);

/* Thread-local message for the last non-zero status. */
const char* b200_bitonic_last_error(void);

/* Library version string. */
const char* b200_bitonic_version(void);

#ifdef __cplusplus
}
#endif

#endif /* B200_BITONIC_H */
