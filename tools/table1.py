"""table1.py -- the paper's Table 1 on B200, as a separate tool.

SURVEY.md 8(f) item 4: emit the reference's Table-1 shape for the GPU rows
without touching the reference's own parser (``parse_strategies("gpu")`` must
keep throwing, test_bench.cpp:346).  For each size:

* ``qs_ms``          bitonic::reference_quicksort, 1 core (the paper's CPU
                     baseline; oracle/_ref, verify.cpp:109-116)
* ``bitonic_seq_ms`` bitonic::sequential_bitonic_sort, 1 core (engine.cpp:248)
                     -- skipped (empty) above --seq-max-log2
* ``gpu_ms``         this repo's sm_100a sort, device-timed with CUDA events
                     (input restored and L2 flushed outside the timing)
* ``ratio``          qs_ms / gpu_ms  (the paper's "acceleration ratio",
                     PAPER.md:115, bench.cpp:435-438)
* ``launches_gpu``, ``gmem_gpu`` the GPU plan's counters in the reference's
                     cost model (engine.hpp:55-70): launches and global key
                     reads + writes.

Formats follow the reference's emit_report (bench.cpp:185-290): an aligned
table, RFC-4180 CSV with one header row, or a JSON array.  The size grammar is
the reference's parse_sizes (bench.cpp:460-484): ``8,2^4,2^17..2^24``.

    python tools/table1.py --sizes 2^17..2^24 --format csv

A report tool beside bench.py (it times the reference's CPU code through the
oracle/_ref checker), kept outside the product package.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import math
import sys
import time
from typing import Dict, List, Optional
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

MAX_LOG2 = 48  # kMaxLog2Length, schedule.hpp:15

COLUMNS = ["size", "qs_ms", "bitonic_seq_ms", "gpu_ms", "gpu_gkeys", "ratio",
           "launches_gpu", "gmem_gpu", "roofline_frac"]


class ConfigError(ValueError):
    """Mirror of bitonic::config_error for the CLI grammar."""


def _size_token(tok: str) -> int:
    try:
        if tok.startswith("2^"):
            e = int(tok[2:])
            if e > MAX_LOG2:
                raise ConfigError(f"size exponent too large: {tok}")
            if tok[2:] != str(e):
                raise ValueError
            return 1 << e
        if not tok.isdigit():
            raise ValueError
        return int(tok)
    except ConfigError:
        raise
    except Exception:
        raise ConfigError(f"bad size token: '{tok}'")


def parse_sizes(text: str) -> List[int]:
    """The reference's size grammar (bench.cpp:460-484; test_bench.cpp:321-331)."""
    sizes: List[int] = []
    for raw in text.split(","):
        tok = raw.strip()
        if not tok:
            raise ConfigError(f"empty size token in '{text}'")
        if ".." not in tok:
            sizes.append(_size_token(tok))
            continue
        lo_s, hi_s = tok.split("..", 1)
        lo, hi = _size_token(lo_s), _size_token(hi_s)
        if lo < 1 or lo > hi:
            raise ConfigError(f"bad size range: '{tok}'")
        v = lo
        while True:
            sizes.append(v)
            if v > hi // 2:
                break
            v *= 2
    return sizes


def emit(records: List[Dict], fmt: str) -> str:
    if not records:
        raise ConfigError("no records to report")
    if fmt == "json":
        return json.dumps(records, indent=1) + "\n"
    if fmt == "csv":
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(COLUMNS)
        for r in records:
            w.writerow(["" if r.get(c) is None else r[c] for c in COLUMNS])
        return buf.getvalue()
    if fmt == "table":
        def cell(v):
            if v is None:
                return "-"
            if isinstance(v, float):
                return f"{v:.4g}"
            return str(v)
        rows = [COLUMNS] + [[cell(r.get(c)) for c in COLUMNS] for r in records]
        width = [max(len(row[i]) for row in rows) for i in range(len(COLUMNS))]
        return "\n".join("  ".join(x.rjust(width[i]) for i, x in enumerate(row))
                         for row in rows) + "\n"
    raise ConfigError(f"unknown format '{fmt}' (expected table, csv, or json)")


def measure(sizes: List[int], seed: int = 1, reps: int = 5, seq_max_log2: int = 22,
            qs_max_log2: int = 28) -> List[Dict]:
    """Time every cell on this host / GPU (needs oracle/_ref and a CUDA device)."""
    import numpy as np
    import torch
    import oracle
    import paper_1506_01446_b200 as b200

    ref = oracle.reference()
    if ref is None:
        raise RuntimeError("oracle/_ref (the reference library) was not built")
    dev = torch.device("cuda", torch.cuda.current_device())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    hbm = 6556.5
    try:
        import os
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"])
    except Exception:
        pass
    out = []
    for n in sizes:
        keys = ref.generate_input(n, seed)  # the reference's generator (int32)
        rec: Dict[str, Optional[float]] = {"size": n}
        k = n.bit_length() - 1
        if k <= qs_max_log2:
            best = math.inf
            for _ in range(reps if k <= 24 else 1):
                w = keys.copy()
                t0 = time.perf_counter()
                ref.quicksort_inplace(w)
                best = min(best, time.perf_counter() - t0)
            rec["qs_ms"] = best * 1e3
        else:
            rec["qs_ms"] = None
        if k <= seq_max_log2 and n >= 2 and n & (n - 1) == 0:
            best = math.inf
            for _ in range(max(1, reps // 2)):
                w = keys.copy()
                t0 = time.perf_counter()
                ref.sequential_bitonic_sort_inplace(w)
                best = min(best, time.perf_counter() - t0)
            rec["bitonic_seq_ms"] = best * 1e3
        else:
            rec["bitonic_seq_ms"] = None
        src = torch.from_numpy(keys.copy()).to(dev)
        work = src.clone()
        sort = b200.sort_ if n & (n - 1) == 0 else b200.sort_padded_
        for _ in range(3):
            work.copy_(src)
            sort(work)
        ts = []
        for _ in range(reps):
            work.copy_(src)
            flush.zero_()
            torch.cuda._sleep(100_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sort(work)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        got = work.cpu().numpy()
        if not (np.diff(got.astype(np.int64)) >= 0).all():
            raise RuntimeError(f"validation failed: size={n}")
        gpu_ms = min(ts)
        rec["gpu_ms"] = gpu_ms
        rec["gpu_gkeys"] = n / (gpu_ms * 1e-3) / 1e9
        rec["ratio"] = rec["qs_ms"] / gpu_ms if rec["qs_ms"] else None
        if n & (n - 1) == 0 and n >= 2:
            c = b200.counters(n)
            rec["launches_gpu"] = c["kernel_launches"]
            rec["gmem_gpu"] = c["global_reads"] + c["global_writes"]
            pm = _pmin(k)
            rec["roofline_frac"] = (pm * 8 * n / (hbm * 1e9)) / (gpu_ms * 1e-3)
        else:
            rec["launches_gpu"] = rec["gmem_gpu"] = rec["roofline_frac"] = None
        out.append(rec)
    return out


def _pmin(k: int, c: int = 15) -> int:
    bits, passes = set(), 1
    for p in range(1, k + 1):
        for s in range(p, 0, -1):
            nb = bits | {s - 1}
            if len(nb) > c:
                passes += 1
                nb = {s - 1}
            bits = nb
    return passes


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--sizes", default="2^17..2^24")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--format", default="table")
    ap.add_argument("--seq-max-log2", type=int, default=22)
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    try:
        sizes = parse_sizes(a.sizes)
        emit([{"size": 1}], a.format)  # validate the format before timing
    except ConfigError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    text = emit(measure(sizes, a.seed, a.reps, a.seq_max_log2), a.format)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
