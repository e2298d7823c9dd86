"""The Table-1 report tool: the reference's size grammar and report formats
(test_bench.cpp:226-354) on the GPU rows; the GPU run itself is gpu-marked."""
import csv
import io
import json

import pytest

import importlib.util
import os

_spec = importlib.util.spec_from_file_location(
    "table1", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "tools", "table1.py"))
t1 = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(t1)


def test_parse_sizes_like_the_reference():
    # test_bench.cpp:321-331
    assert t1.parse_sizes("8,2^4,100") == [8, 16, 100]
    assert t1.parse_sizes("2^17..2^20") == [131072, 262144, 524288, 1048576]
    assert t1.parse_sizes("3..20") == [3, 6, 12]
    assert t1.parse_sizes("2^3..2^3") == [8]
    for bad in ["", "abc", "2^99", "16..8", "8,,16"]:
        with pytest.raises(t1.ConfigError):
            t1.parse_sizes(bad)


RECS = [{"size": 1 << 17, "qs_ms": 7.5, "bitonic_seq_ms": 20.0, "gpu_ms": 0.02,
         "gpu_gkeys": 6.5, "ratio": 375.0, "launches_gpu": 7, "gmem_gpu": 1835008,
         "roofline_frac": 0.05},
        {"size": 1 << 18, "qs_ms": 16.0, "bitonic_seq_ms": None, "gpu_ms": 0.03,
         "gpu_gkeys": 8.7, "ratio": 533.3, "launches_gpu": 10, "gmem_gpu": 5242880,
         "roofline_frac": 0.06}]


def test_csv_round_trip():
    text = t1.emit(RECS, "csv")
    rows = list(csv.reader(io.StringIO(text)))
    assert rows[0] == t1.COLUMNS and len(rows) == 3
    assert float(rows[1][t1.COLUMNS.index("ratio")]) == 375.0
    assert rows[2][t1.COLUMNS.index("bitonic_seq_ms")] == ""


def test_table_and_json():
    lines = t1.emit(RECS, "table").splitlines()
    assert len(lines) == 3 and lines[0].split()[0] == "size"
    assert json.loads(t1.emit(RECS, "json"))[1]["size"] == 1 << 18
    with pytest.raises(t1.ConfigError):
        t1.emit([], "csv")
    with pytest.raises(t1.ConfigError):
        t1.emit(RECS, "xml")


@pytest.mark.gpu
def test_table1_runs_on_gpu():
    recs = t1.measure([1 << 12, 3000, 1 << 16], reps=2, seq_max_log2=16)
    assert [r["size"] for r in recs] == [4096, 3000, 65536]
    assert all(r["gpu_ms"] > 0 and r["ratio"] > 0 for r in recs)
