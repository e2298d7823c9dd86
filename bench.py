#!/usr/bin/env python3
"""bench.py -- device-timed Gkeys/s of the B200 bitonic sort (BASELINE.json metric).

Default (N=1): BASELINE.json configs[2]'s 2^28 point -- the largest
single-GPU configuration, north_star's primary HBM-bound size and the
paper's largest Table-1 row: 2^28 keys from the reference's
own ``generate_input(n, seed=1)`` (bench.cpp:354-364: low 32 bits of
std::mt19937_64(1)), sorted ascending as uint32.  The GPU arm, its
``cpu_baseline`` leg and ``--impl reference`` all sort that same buffer (the
reference's CPU code sorts it as int32 after x ^ 0x80000000, the exact
uint32-order bridge), and both arms print the same ``config`` dict.

One "step" = one full in-place sort of the array.  The unsorted input is
restored (device-to-device copy) and L2 is flushed (a 256 MiB write, larger
than the 126 MB L2; the 1 GiB array is itself 8x L2) before every step,
outside the timed region; each step is timed with CUDA events on the sorting
stream.  Under torchrun (N>1) every rank owns a 2^(32 - log2 N)-key shard of
one 2^32-key array (BASELINE configs[4]) and the partitioned sort (local sort
+ merge-split network, paper_1506_01446_b200/dist.py) is timed, max over
ranks ("strong").  ``--log2n`` / ``--batched`` select the other configs.

Extra JSON keys (see the task contract): e2e (host pinned buffers, H2D + sort
+ D2H inside the timed region, through the reference-facing host entry),
roofline (dominant kernel family, measured live with CUDA events), sort_roofline
(north_star's whole-sort definition: P_min x 8 bytes x n / HBM BW),
cpu_baseline (the reference's own CPU code from oracle/_ref on this host,
with its output compared key for key with the GPU's), clocks (NVML sampled
during the timed region), gpu_launches.

``--impl reference`` times the reference's CPU implementation of the path
(oracle/_ref: generate_schedule + build_plan(fused, 1024) + execute on all
host threads, run_cell's timing discipline, bench.cpp:68-116) on the same
workload and prints the same line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback
METRIC = "Gkeys/s sorting uint32 (device-timed) vs HBM roofline; speedup vs CPU quicksort"
SEED = 1  # generate_input's default seed (bench.cpp:354, BenchConfig)
# The paper's published numbers for this path (Table 1
# "GPU Optimized", Kepler K10), as Gkeys/s per log2 size.
PAPER_GKEYS = {17: 0.364, 18: 0.397, 19: 0.400, 20: 0.375, 21: 0.357, 22: 0.341,
               23: 0.318, 24: 0.298, 25: 0.278, 26: 0.259, 27: 0.243, 28: 0.227}
# P_min(k, c=15): minimum HBM round trips of the network.
PMIN = {16: 3, 20: 7, 24: 13, 28: 21, 29: 22, 30: 24, 31: 27, 32: 29}


def pmin(k: int, c: int = 15) -> int:
    if k in PMIN:
        return PMIN[k]
    bits, passes = set(), 1
    for p in range(1, k + 1):
        for s in range(p, 0, -1):
            nb = bits | {s - 1}
            if len(nb) > c:
                passes += 1
                nb = {s - 1}
            bits = nb
    return passes


def peaks():
    try:
        with open(MEASURED) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured", d
    except Exception:
        return HBM_FALLBACK, "fallback", {}


def host_info():
    """CPU model and core count of this host (the GPU box's, when run there)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except Exception:
        usable = os.cpu_count() or 1
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "usable_cpus": usable}


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled during the timed
    region: NVML every ~5 ms when pynvml is importable, else nvidia-smi."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int, interval: float = 0.005):
        # multi-rank steps synchronise the host several times per step: a
        # 5 ms sampler there costs ~10 ms per step (measured), so N > 1 samples
        # every 100 ms
        self.index = index
        self.interval = float(os.environ.get("B200_BENCH_CLOCK_INTERVAL", interval))
        self.samples = []  # (sm_mhz, max_mhz, set of reason names)
        self._stop = threading.Event()
        self._t = None
        self.source = None

    def _nvml_open(self):
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))

        def sample():
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.samples.append((float(sm), mx, {n for n, b in bits.items() if r & b}))
        self._sample = sample
        self.source = "nvml"

    def _nvml(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(self.interval)

    def _smi(self):
        self.source = "nvidia-smi"
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                f = [x.strip() for x in out.split(",")]
                if len(f) >= 7 and f[0].replace(".", "").isdigit():
                    self.samples.append((float(f[0]), float(f[1]) if f[1].replace(".", "").isdigit()
                                         else None,
                                         {n for n, v in zip(self.NAMES, f[3:7])
                                          if v.lower() == "active"}))
            except Exception:
                pass
            self._stop.wait(0.2)

    def _run(self):
        try:
            if self._sample is None:
                raise RuntimeError("no NVML")
            self._nvml()
        except Exception:
            if not self.samples:
                self._smi()

    def __enter__(self):
        self._sample = None
        try:  # open NVML and take the first sample before the timed region
            self._nvml_open()
            self._sample()
        except Exception:
            self._sample = None
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if self._sample is not None:
            try:
                self._sample()  # and the last one right after it
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = sorted(x[0] for x in self.samples)
        mx = max((x[1] for x in self.samples if x[1]), default=None)
        reasons = set()
        for x in self.samples:
            reasons |= x[2]
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "sm_min_mhz": sm[0],
                "reasons": sorted(reasons), "samples": len(self.samples), "source": self.source}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# the workload (identical in both arms)
# ---------------------------------------------------------------------------
def resolve_args(args):
    """Fill in log2n / scaling from the config the flags select."""
    world = dist_env()[0]
    args.scaling = "weak"
    if args.log2n is None:
        if args.batched:
            args.log2n = 24
        elif world > 1:
            args.log2n = 32 - (world.bit_length() - 1)
            args.scaling = "strong"  # 2^32 keys in all, whatever N
        else:
            args.log2n = 28
    return args


def workload_config(args, world):
    """The config dict both arms print (the driver compares them)."""
    n = 1 << args.log2n
    total = n * world
    if args.batched:
        return {"workload": (f"batched: {n // args.batched} arrays of {args.batched} keys, "
                             f"each sorted independently, ascending uint32; keys = "
                             f"generate_input({n}, seed={SEED}) (bench.cpp:354-364)"),
                "keys_total": total, "n_per_array": args.batched,
                "arrays": n // args.batched, "seed": SEED}
    if world > 1:
        return {"workload": (f"2^{total.bit_length() - 1} keys, one array partitioned over "
                             f"{world} GPUs (2^{args.log2n} per rank; shard r = "
                             f"generate_input(2^{args.log2n}, seed={SEED}+r), "
                             f"bench.cpp:354-364), ascending uint32"),
                "keys_total": total, "keys_per_gpu": n, "seed": SEED}
    return {"workload": (f"2^{args.log2n} keys = generate_input(2^{args.log2n}, seed={SEED}) "
                         f"(bench.cpp:354-364: low 32 bits of std::mt19937_64), one array, "
                         f"ascending uint32"),
            "keys_total": total, "keys_per_gpu": n, "seed": SEED}


# ---------------------------------------------------------------------------
# reference arm (CPU): the reference's own code from oracle/_ref
# ---------------------------------------------------------------------------
def reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0  # rank 0 alone runs and prints the reference arm
    import oracle
    ref = oracle.reference()
    cfg = workload_config(args, world)
    info = host_info()
    cores = info["usable_cpus"]
    if args.batched:
        return reference_arm_batched(args, ref, cfg, info)
    n_cfg = cfg["keys_total"]
    # N=1: the whole workload.  N>1: the 2^32-key workload would take ~2 min
    # per step on the CPU; a 2^28-key sample of it (rank 0's generator
    # stream) keeps the run within minutes.
    n = n_cfg if world == 1 else min(n_cfg, 1 << 28)
    if ref is not None and ref.has_bench:
        kind = "reference"
        x = ref.generate_input(n, SEED)  # the reference's own generator (int32 bits)
        x ^= np.int32(-2**31)            # u32 order == i32 order of x ^ 0x80000000
        work = x.copy()

        def run():
            return ref.execute_timed_inplace(work, 2, min(1024, n), cores) * 1e-3
        what = (f"bitonic::execute(build_plan(generate_schedule({n.bit_length() - 1}), fused, "
                f"{min(1024, n)}), keys, {cores} workers), timed as run_cell does "
                f"(bench.cpp:92-107)")
        if n < n_cfg:
            what += (f", on a 2^{n.bit_length() - 1}-key sample of the "
                     f"2^{n_cfg.bit_length() - 1}-key workload")
    else:  # pragma: no cover - oracle port when the reference was not built
        kind = "port"
        o = oracle.oracle()
        x = (o.generate_input(n, SEED) ^ np.uint32(0x80000000)).view(np.int32)
        work = x.copy()

        def run():
            t0 = time.perf_counter()
            work[:] = o.sequential_bitonic_i32(work)
            return time.perf_counter() - t0
        what = "oracle sequential_bitonic_i32 (1 core)"
        cores = 1
    warm = args.warmup
    for _ in range(warm):
        work[:] = x
        run()
    times = []
    for _ in range(args.steps):
        work[:] = x
        times.append(run())
    assert (np.diff(work.astype(np.int64)) >= 0).all(), "reference output not sorted"
    ms = 1e3 * sum(times) / len(times)
    value = n / (ms * 1e-3) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gkeys/s",
        "n_gpus": world, "steps": args.steps, "warmup": warm,
        "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": "Gkeys/s", "cores": cores,
                         "kind": kind, "sample": what, "sample_keys": n, **info},
        "e2e": {"value": value, "unit": "Gkeys/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _per_array_parallel(fn, arrays, cores):
    """fn on every row, rows spread over `cores` threads (the ctypes calls
    release the GIL, so the reference code runs on all cores)."""
    from concurrent.futures import ThreadPoolExecutor
    rows = list(arrays)
    if cores <= 1:
        for r in rows:
            fn(r)
        return
    with ThreadPoolExecutor(cores) as ex:
        list(ex.map(fn, rows))


def reference_arm_batched(args, ref, cfg, info):
    """Reference arm for the batched config: the reference's own
    sequential_bitonic_sort on every array of the workload, arrays spread
    over all host cores (the reference has no batched entry; one array per
    call is its API)."""
    n_per = args.batched
    n = cfg["keys_total"]
    cores = info["usable_cpus"]
    if ref is not None and ref.has_bench:
        x = (ref.generate_input(n, SEED) ^ np.int32(-2**31)).reshape(-1, n_per)
        kind, fn = "reference", ref.sequential_bitonic_sort_inplace
        what = (f"bitonic::sequential_bitonic_sort on each of the {x.shape[0]} arrays of "
                f"{n_per} keys, {cores} threads")
    else:  # pragma: no cover
        import oracle
        o = oracle.oracle()
        x = (o.generate_input(n, SEED) ^ np.uint32(0x80000000)).view(np.int32).reshape(-1, n_per)
        kind = "port"
        fn = lambda a: a.__setitem__(slice(None), o.sequential_bitonic_i32(a))
        what = f"oracle sequential_bitonic_i32 on {x.shape[0]} arrays, {cores} threads"
    work = x.copy()
    for _ in range(args.warmup):
        work[:] = x
        _per_array_parallel(fn, work, cores)
    times = []
    for _ in range(args.steps):
        work[:] = x
        t0 = time.perf_counter()
        _per_array_parallel(fn, work, cores)
        times.append(time.perf_counter() - t0)
    assert (np.diff(work.astype(np.int64), axis=1) >= 0).all()
    ms = 1e3 * sum(times) / len(times)
    value = work.size / (ms * 1e-3) / 1e9
    world, _, _ = dist_env()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gkeys/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": value, "unit": "Gkeys/s", "cores": cores,
                         "kind": kind, "sample": what, "sample_keys": int(work.size), **info},
        "e2e": {"value": value, "unit": "Gkeys/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# cpu_baseline leg of our arm (rank 0, N=1): the same buffer on the host
# ---------------------------------------------------------------------------
def cpu_baseline(x_u32: np.ndarray, gpu_sorted_u32: np.ndarray, info):
    """The paper's CPU quicksort (1 core, the paper's speedup baseline,
    verify.cpp:109-116) and the reference's CPU bitonic sorts on the SAME keys
    the GPU sorted; the reference fused engine's output is compared key for
    key with the GPU's (run_cell's check, bench.cpp:68-116)."""
    import oracle
    ref = oracle.reference()
    n = x_u32.size
    x = (x_u32 ^ np.uint32(0x80000000)).view(np.int32)  # int32 order == u32 order of x
    cores = info["usable_cpus"]
    out = {}
    if ref is None:  # pragma: no cover
        o = oracle.oracle()
        kind = "port"
        t0 = time.perf_counter()
        qs = o.quicksort_i32(x)
        out["quicksort_ms"] = (time.perf_counter() - t0) * 1e3
        ref_sorted = qs
    else:
        kind = "reference"
        w = x.copy()
        t0 = time.perf_counter()
        ref.quicksort_inplace(w)  # one rep: ~25 s at 2^28 on one core
        out["quicksort_ms"] = (time.perf_counter() - t0) * 1e3
        w = x.copy()
        out["fused_engine_ms"] = ref.execute_timed_inplace(w, 2, min(1024, n), cores)
        out["fused_engine_cores"] = cores
        ref_sorted = w
        # sequential bitonic (1 core) costs ~2 min at 2^28: time it on the
        # first 2^min(k,24) keys and say so
        ns = min(n, 1 << 24)
        w = x[:ns].copy()
        t0 = time.perf_counter()
        ref.sequential_bitonic_sort_inplace(w)
        out["sequential_bitonic_ms"] = (time.perf_counter() - t0) * 1e3
        out["sequential_bitonic_keys"] = ns
    got = gpu_sorted_u32 ^ np.uint32(0x80000000)
    out["gpu_output_equals_reference"] = bool(np.array_equal(got.view(np.int32), ref_sorted))
    return kind, cores, out


def cpu_baseline_batched(x_u32: np.ndarray, n_per: int, info):
    """Batched workload on the host: the paper's quicksort per array (1 core)
    on a bounded sample of the arrays, and the reference's sequential bitonic
    on every array over all cores."""
    import oracle
    ref = oracle.reference()
    arrays = (x_u32 ^ np.uint32(0x80000000)).view(np.int32).reshape(-1, n_per)
    cores = info["usable_cpus"]
    sample = arrays[: max(1, min(arrays.shape[0], (1 << 22) // n_per))]
    if ref is None:  # pragma: no cover
        o = oracle.oracle()
        kind = "port"
        qs = lambda a: a.__setitem__(slice(None), o.quicksort_i32(a))
        seq = lambda a: a.__setitem__(slice(None), o.sequential_bitonic_i32(a))
    else:
        kind, qs, seq = "reference", ref.quicksort_inplace, ref.sequential_bitonic_sort_inplace
    out = {"sample_arrays": int(sample.shape[0]), "sample_keys": int(sample.size)}
    w = sample.copy()
    t0 = time.perf_counter()
    _per_array_parallel(qs, w, 1)
    out["quicksort_ms"] = (time.perf_counter() - t0) * 1e3
    w = arrays.copy()
    t0 = time.perf_counter()
    _per_array_parallel(seq, w, cores)
    out["sequential_bitonic_all_cores_ms"] = (time.perf_counter() - t0) * 1e3
    out["all_keys"] = int(arrays.size)
    return kind, cores, out, w


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--log2n", type=int, default=None,
                    help="keys per GPU = 2^log2n.  Default: 28 at N=1 (BASELINE "
                         "configs[2], the largest single-GPU config); 32 - log2(N) at N>1 "
                         "(configs[4]: 2^32 keys partitioned over the N GPUs); 24 with "
                         "--batched (configs[3])")
    ap.add_argument("--batched", type=int, default=0,
                    help="n_per_array for the batched config (e.g. 4096)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip the merge-path variant measurement")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    resolve_args(args)

    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import torch.distributed as dist
    import paper_1506_01446_b200 as b200

    world, rank, local = dist_env()
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    # Functional test hook (never a measurement): B200_BENCH_SHARED_GPU=1 runs
    # every rank on cuda:0 with gloo, to exercise the N>1 code path on a
    # one-GPU box.  The ranks' kernels never wait on each other (the peer
    # exchange is ordered by host-side events).
    shared_gpu = world > 1 and os.environ.get("B200_BENCH_SHARED_GPU") == "1"
    if shared_gpu:
        local = 0
    if world > 1:
        torch.cuda.set_device(local)
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    info = host_info()
    cfg = workload_config(args, world)

    n = 1 << args.log2n
    hbm, peak_kind, peaks_json = peaks()
    # the reference's generate_input bits (product host function, same
    # algorithm as bench.cpp:354-364), generated outside any timing
    x_host = b200.generate_input(n, SEED + (rank if world > 1 else 0))
    src = torch.from_numpy(x_host.view(np.int32)).to(dev).view(torch.uint32)
    work = src.clone()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    batched = args.batched
    dist_stats = {}
    if world > 1:
        from paper_1506_01446_b200 import dist as bdist
        exchange = os.environ.get("B200_BITONIC_EXCHANGE", "peer")

        def sort_step():
            bdist.partitioned_sort_(work, exchange=exchange, stats=dist_stats)
        plan = b200.plan(n)
        # local sort + one fused merge-split (partition + merge kernels) per
        # network step (the two shard copies are memcpys, not kernels)
        launches_per_step = len(plan) + 2 * len(bdist.network_steps(world))
    elif batched:
        def sort_step():
            b200.sort_batched_(work, batched)
        plan = b200.plan(batched, n // batched)
        launches_per_step = len(plan)
    else:
        def sort_step():
            b200.sort_(work)
        plan = b200.plan(n)
        launches_per_step = len(plan)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- warm-up -------------------------------------------------------------
    for _ in range(args.warmup):
        work.copy_(src)
        sort_step()
    torch.cuda.synchronize()

    # ---- correctness of the timed configuration (outside timing) -----------
    if world == 1:
        ref = src.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        if batched:
            ref = torch.sort(ref.view(-1, batched), dim=1).values.view(-1)
        else:
            ref = torch.sort(ref).values
        got = work.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        ok = torch.equal(got, ref)
        del ref, got
        torch.cuda.empty_cache()
        if not ok:
            print(json.dumps({"error": "sort output mismatch"}), flush=True)
            return 1
    gpu_sorted = work.view(torch.int32).cpu().numpy().view(np.uint32) if world == 1 else None

    # ---- timed region ----------------------------------------------------------
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    sampler = ClockSampler(torch.cuda.current_device() if world == 1 else local,
                           0.005 if world == 1 else 0.1)
    barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    with sampler:
        for i in range(args.steps):
            work.copy_(src)      # restore the unsorted input (not timed)
            flush.zero_()        # evict L2 (not timed)
            # ~50 us device-side delay so the host has enqueued every pass of
            # the sort before the start event fires: the events then bracket
            # the device execution of the sort, not host launch overhead
            # (which e2e below does include).
            torch.cuda._sleep(100_000)
            evs[i][0].record(stream)
            sort_step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    barrier()
    wall = time.perf_counter() - wall0
    ms_steps = [a.elapsed_time(b) for a, b in evs]
    ms = sum(ms_steps) / len(ms_steps)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    keys_total = n * world
    value = keys_total / (ms * 1e-3) / 1e9

    # ---- per-kernel timing: dominant kernel family -----------------------------
    roofline = None
    sort_roof = None
    if world == 1:
        # Per-pass durations inside the pass chain: the plan's passes are
        # enqueued back to back (after an L2 flush and a device sleep that
        # keeps host launch latency out), with an event between consecutive
        # passes on the sort stream; pass i lasts e[i+1] - e[i].  (The events
        # break the programmatic-dependent-launch overlap, so these durations
        # are slightly longer than inside the graph-launched sort.)
        fam_t, fam_n = {}, {}
        reps = 10
        for _ in range(reps):
            work.copy_(src)
            flush.zero_()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(plan) + 1)]
            torch.cuda._sleep(4_000_000)  # ~2 ms: every pass is enqueued before the first runs
            ev[0].record(stream)
            for i in range(len(plan)):
                b200.run_pass_(work, i, n_per_array=(batched or n))
                ev[i + 1].record(stream)
            torch.cuda.synchronize()
            for i, p in enumerate(plan):
                fam = "tile_sort" if p.tile_sort else "merge"
                fam_t[fam] = fam_t.get(fam, 0.0) + ev[i].elapsed_time(ev[i + 1])
                fam_n[fam] = fam_n.get(fam, 0) + 1
        dom = max(fam_t, key=lambda f: fam_t[f])
        share = {f: fam_t[f] / sum(fam_t.values()) for f in fam_t}
        # Average launch of the dominant family inside the timed (graph-
        # launched) sort: its share of the event-bracketed chain applied to
        # the measured step time.  The event-bracketed per-pass mean itself
        # (kept as avg_launch_ms_bracketed) adds ~4 us of per-event launch
        # overhead, which dominates passes of a few microseconds.
        avg_bracketed = fam_t[dom] / fam_n[dom]
        avg_ms = ms * share[dom] / (fam_n[dom] / reps)
        alg_bytes = 8 * n  # one read + one write of every key per launch
        achieved = alg_bytes / (avg_ms * 1e-3) / 1e9
        traffic = None
        for fname in ("traffic.json", "r1_traffic.json"):
            try:  # measured DRAM bytes per launch from the committed ncu capture
                with open(os.path.join(ROOT, "profiles", fname)) as f:
                    tr = json.load(f)
                key = f"batched{batched}" if batched else str(args.log2n)
                traffic = tr.get(key, {}).get(dom)
                if traffic is not None:
                    break
            except Exception:
                pass
        roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm,
                    "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm,
                    "traffic": traffic,
                    "algorithmic_bytes_per_launch": alg_bytes,
                    "avg_launch_ms": avg_ms,
                    "avg_launch_ms_bracketed": avg_bracketed,
                    "method": ("step time x the family's share of an event-bracketed "
                               "replay of the same plan on the same stream, / launches "
                               "per step"),
                    "share_of_step": share}
        if achieved > hbm and traffic:
            roofline["note"] = (f"frac > 1: part of the array stays L2-resident between passes "
                                f"(DRAM bytes per launch {traffic} < algorithmic {alg_bytes})")
        k = args.log2n if not batched else (batched.bit_length() - 1)
        pm = 1 if batched else pmin(k)
        t_roof = pm * 8 * n / (hbm * 1e9)
        sort_roof = {"p_min": pm, "p_design": len(plan), "t_roof_us": t_roof * 1e6,
                     "frac": t_roof / (ms * 1e-3),
                     "definition": "P_min(k,15) x 8 B x n / measured HBM BW (SURVEY 8d)"}

    # ---- the merge-path variant on the same keys (single array, k > 13) -------
    # b200_bitonic_sort_mergepath_u32: same output bytes, one HBM pass per
    # global phase (co-rank partitioned bitonic tile merges) instead of the
    # network's fused half-cleaner passes.  Reported beside the headline (which
    # stays the network, the reference's algorithm), same timing discipline.
    variant = None
    if world == 1 and not batched and args.log2n > 14 and not args.no_variants:
        try:
            vt = []
            for i in range(args.warmup + args.steps):
                work.copy_(src)
                flush.zero_()
                torch.cuda._sleep(100_000)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                b200.sort_mergepath_(work)
                e1.record(stream)
                torch.cuda.synchronize()
                if i >= args.warmup:
                    vt.append(e0.elapsed_time(e1))
            same = bool(np.array_equal(work.view(torch.int32).cpu().numpy().view(np.uint32),
                                       gpu_sorted))
            vms = sum(vt) / len(vt)
            tile_bits = 14  # the variant's default tile (B200_BITONIC_MERGEPATH_TILE)
            t_roof = pmin(args.log2n) * 8 * n / (hbm * 1e9)
            variant = {
                "mergepath": {
                    "value": n / (vms * 1e-3) / 1e9, "unit": "Gkeys/s", "ms_per_step": vms,
                    "steps": len(vt), "output_equals_network_output": same,
                    "passes": 1 + args.log2n - tile_bits,
                    "kernels": (f"tile_sort_kernel<{tile_bits},5> + per phase "
                                "mergepath_partition_kernel + mergepath_merge_kernel<13,6>"),
                    "sort_roofline_frac": t_roof / (vms * 1e-3),
                    "sort_roofline_definition": "the network's P_min(k,15) x 8 B x n / HBM BW, "
                                                "as for the headline",
                    "api": "b200_bitonic_sort_mergepath_u32 (device pointer, in place, "
                           "n-key scratch from the pool)",
                }}
        except Exception as ex:  # pragma: no cover - report, do not fail the bench
            variant = {"mergepath": {"error": repr(ex)[:200]}}

    # ---- end to end through the public API with host buffers ---------------
    # Single array: the reference-facing host entry (sort_host ->
    # b200_bitonic_sort_host_u32, the drop-in for sequential_bitonic_sort),
    # synchronous, timed on the host clock around the call; it copies H2D,
    # sorts and copies D2H (chunk-pipelined) inside the call.  Batched: the
    # device entry between explicit pinned copies, CUDA-event timed.
    e2e = None
    if world == 1:
        h_src = torch.from_numpy(x_host.view(np.int32)).pin_memory()
        h_out = torch.empty_like(h_src).pin_memory()
        dwork = torch.empty_like(src)
        tt = []
        h_src_np = h_src.numpy()
        arr = h_out.numpy().view(np.uint32)
        for i in range(args.warmup + args.steps):
            flush.zero_()
            if not batched:
                torch.cuda.synchronize()
                # restore the unsorted input (untimed) with a single-threaded
                # copy: torch's multi-threaded CPU copy leaves its worker
                # threads spinning, which delays the host thread's CUDA calls
                np.copyto(arr, h_src_np.view(np.uint32))
                c0 = time.perf_counter()
                b200.sort_host(arr)
                t_ms = (time.perf_counter() - c0) * 1e3
            else:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                dwork.copy_(h_src.view(torch.uint32), non_blocking=True)
                b200.sort_batched_(dwork, batched)
                h_out.view(torch.uint32).copy_(dwork, non_blocking=True)
                e1.record(stream)
                torch.cuda.synchronize()
                t_ms = e0.elapsed_time(e1)
            if i >= args.warmup:
                tt.append(t_ms)
        if not np.array_equal(arr, gpu_sorted):
            raise SystemExit("e2e output differs from the device-entry output")
        ems = sum(tt) / len(tt)
        e2e = {"value": n / (ems * 1e-3) / 1e9, "unit": "Gkeys/s",
               "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4 * n,
               "ms_per_step": ems, "host_buffers": "pinned",
               "api": ("b200_bitonic_sort_host_u32 (host clock)" if not batched
                       else "H2D + b200_bitonic_sort_u32_batched + D2H (CUDA events)")}
        del dwork, h_src, h_out

    if world > 1:
        # Each rank: H2D of its shard from pinned host memory, the partitioned
        # sort, D2H of its sorted shard; host clock, max over ranks.  Few
        # steps (restoring GiB-sized pinned buffers on the host is slow).
        err = None
        try:
            h_src = torch.from_numpy(x_host.view(np.int32)).pin_memory()
            h_work = torch.empty_like(h_src).pin_memory()
        except Exception as ex:  # pragma: no cover
            err = repr(ex)[:200]
        okf = torch.tensor([0 if err else 1], device=dev, dtype=torch.int32)
        dist.all_reduce(okf, op=dist.ReduceOp.MIN)  # every rank agrees before timing
        if int(okf.item()) == 1:
            tt = []
            e_steps = min(args.steps, 3)
            for i in range(1 + e_steps):
                h_work.copy_(h_src)
                torch.cuda.synchronize()
                barrier()
                c0 = time.perf_counter()
                work.view(torch.int32).copy_(h_work, non_blocking=True)
                sort_step()
                h_work.copy_(work.view(torch.int32), non_blocking=True)
                torch.cuda.synchronize()
                t_ms = (time.perf_counter() - c0) * 1e3
                t = torch.tensor([t_ms], device=dev, dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                if i >= 1:
                    tt.append(float(t.item()))
            ems = sum(tt) / len(tt)
            e2e = {"value": keys_total / (ems * 1e-3) / 1e9, "unit": "Gkeys/s",
                   "h2d_bytes_per_step": 4 * keys_total, "d2h_bytes_per_step": 4 * keys_total,
                   "ms_per_step": ems, "steps": e_steps, "host_buffers": "pinned, one per rank",
                   "api": "H2D + paper_1506_01446_b200.dist.partitioned_sort_ + D2H per rank "
                          "(host clock, max over ranks)"}
        else:  # pragma: no cover - report instead of failing the bench
            e2e = {"value": None, "unit": "Gkeys/s", "h2d_bytes_per_step": 4 * keys_total,
                   "d2h_bytes_per_step": 4 * keys_total,
                   "error": err or "pinned host buffers unavailable on some rank"}

    # ---- CPU baseline (rank 0, N=1 only), on the same buffer -----------------
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline and batched:
        try:
            kind, cores, c, ref_sorted = cpu_baseline_batched(x_host, batched, info)
            qs_gk = c["sample_keys"] / (c["quicksort_ms"] * 1e-3) / 1e9
            same = bool(np.array_equal((gpu_sorted ^ np.uint32(0x80000000)).view(np.int32),
                                       ref_sorted.reshape(-1)))
            cpu = {"value": qs_gk, "unit": "Gkeys/s", "cores": 1, "kind": kind,
                   "sample": f"bitonic::reference_quicksort on each of the first "
                             f"{c['sample_arrays']} of the {n // batched} arrays of "
                             f"{batched} keys (1 core)",
                   "quicksort_ms": c["quicksort_ms"],
                   "sequential_bitonic_all_cores_ms": c["sequential_bitonic_all_cores_ms"],
                   "sequential_bitonic_all_cores_gkeys": c["all_keys"] / (
                       c["sequential_bitonic_all_cores_ms"] * 1e-3) / 1e9,
                   "all_cores": cores, "gpu_output_equals_reference": same,
                   "speedup_vs_quicksort": value / qs_gk, **info}
        except Exception as e:  # pragma: no cover - report, do not fail the bench
            cpu = {"value": None, "unit": "Gkeys/s", "cores": 0, "kind": "unavailable",
                   "sample": f"cpu baseline failed: {e}"}
    if world == 1 and rank == 0 and not args.no_cpu_baseline and not batched:
        try:
            kind, cores, c = cpu_baseline(x_host, gpu_sorted, info)
            qs_gk = n / (c["quicksort_ms"] * 1e-3) / 1e9
            cpu = {"value": qs_gk, "unit": "Gkeys/s", "cores": 1, "kind": kind,
                   "sample": (f"bitonic::reference_quicksort (the paper's CPU baseline, "
                              f"verify.cpp:109-116) on the same 2^{args.log2n} keys, one rep, "
                              f"1 core"),
                   "quicksort_ms": c["quicksort_ms"],
                   "fused_engine_ms": c.get("fused_engine_ms"),
                   "fused_engine_cores": c.get("fused_engine_cores"),
                   "sequential_bitonic_ms": c.get("sequential_bitonic_ms"),
                   "sequential_bitonic_keys": c.get("sequential_bitonic_keys"),
                   "gpu_output_equals_reference": c["gpu_output_equals_reference"],
                   "speedup_vs_quicksort": c["quicksort_ms"] / ms,
                   **info}
            if c.get("fused_engine_ms"):
                cpu["speedup_vs_fused_engine"] = c["fused_engine_ms"] / ms
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "error": str(e)}

    # ---- N>1: NVLink bytes and the 1-GPU time of the same total -------------
    multi = None
    if world > 1:
        multi = {}
        pk = dist_stats.pop("partner_keys", None)
        if pk is not None:
            per_step = [4 * int(x) for x in pk.tolist()]  # bytes this rank read over NVLink
            t = torch.tensor(per_step, device=dev, dtype=torch.int64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            multi["nvlink_bytes_per_rank_per_step_max"] = t.tolist()
            multi["nvlink_bytes_per_step_all_ranks"] = None
            tsum = torch.tensor(per_step, device=dev, dtype=torch.int64)
            dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
            multi["nvlink_bytes_per_step_all_ranks"] = tsum.tolist()
            multi["nvlink_floor_us_per_step"] = [b / 900e9 * 1e6 for b in t.tolist()]
            multi["nvlink_link_gbs_assumed"] = 900.0
        # strong-scaling reference: rank 0 sorts the whole 2^k-key array alone
        # (same kernels, one GPU), so efficiency is self-contained in the line
        barrier()
        if rank == 0 and not shared_gpu:
            try:
                del work
                torch.cuda.empty_cache()
                big = torch.empty(keys_total, dtype=torch.uint32, device=dev)
                gi = torch.Generator(device=dev)
                gi.manual_seed(SEED)
                ts = []
                for i in range(3):
                    big.view(torch.int32).random_(generator=gi)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    b200.sort_(big)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    if i:
                        ts.append(e0.elapsed_time(e1))
                one_ms = sum(ts) / len(ts)
                multi["one_gpu_ms_same_total"] = one_ms
                multi["one_gpu_gkeys_same_total"] = keys_total / (one_ms * 1e-3) / 1e9
                multi["speedup_vs_one_gpu"] = one_ms / ms
                del big
                torch.cuda.empty_cache()
            except Exception as ex:  # pragma: no cover - report, do not fail
                multi["one_gpu_error"] = repr(ex)[:200]
        barrier()

    # vs_baseline: the paper's own Table-1 GPU number for this exact size (K10)
    vs_base = None
    if world == 1 and not batched and args.log2n in PAPER_GKEYS:
        vs_base = value / PAPER_GKEYS[args.log2n]
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gkeys/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": vs_base,
            "vs_baseline_source": ("paper Table 1, GPU Optimized on a Kepler K10 at this size "
                                   "(BASELINE.md section 1, PAPER.md:96-107)"
                                   if vs_base is not None else None),
            "dtype": "u32", "data": "synthetic", "config": cfg,
            "timing": {"l2_flush": "256 MiB write before every step (outside timing)",
                       "input_restore": "D2D copy before every step (outside timing)",
                       "events": "CUDA events on the sort stream around each step; a device "
                                 "sleep before the start event keeps host launch overhead out",
                       "passes": len(plan),
                       **({"exchange": ("half (peer unavailable)"
                                        if dist_stats.get("peer_fallback") else exchange),
                           **{k: v for k, v in dist_stats.items() if k != "peer_fallback"}}
                          if world > 1 else {})},
            "e2e": e2e, "roofline": roofline, "sort_roofline": sort_roof,
            **({"variants": variant} if variant is not None else {}),
            "cpu_baseline": cpu, "clocks": sampler.summary(),
            **({"multi_gpu": multi} if multi is not None else {}),
            "gpu_launches": launches_per_step * args.steps,
            "wall_s": wall,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
