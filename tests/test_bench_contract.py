"""The bench.py contract (the driver parses its last JSON line): the reference
arm on CPU, and (on a GPU) our arm with every key the contract names, the
same config dict in both arms, and the merge-path variant's output check."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                       capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, r.stdout[-2000:]
    return json.loads(lines[-1])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--log2n", "16", "--steps", "1", "--warmup", "3")
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["higher_is_better"] is True
    assert d["unit"] == "Gkeys/s" and d["value"] > 0 and d["warmup"] >= 3
    assert abs(d["value"] - (1 << 16) / (d["ms_per_step"] * 1e-3) / 1e9) < 1e-9
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["config"]["keys_total"] == 1 << 16


@pytest.mark.gpu
def test_our_arm_line_matches_the_contract():
    ours = run_bench("--log2n", "20", "--steps", "3", "--warmup", "3")
    ref = run_bench("--impl", "reference", "--log2n", "20", "--steps", "1", "--warmup", "3")
    assert ours["config"] == ref["config"] and ours["metric"] == ref["metric"]
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "e2e", "roofline", "cpu_baseline", "clocks", "gpu_launches"):
        assert key in ours, key
    n = 1 << 20
    assert abs(ours["value"] - n / (ours["ms_per_step"] * 1e-3) / 1e9) < 1e-6 * ours["value"]
    assert ours["e2e"]["h2d_bytes_per_step"] == 4 * n and ours["e2e"]["d2h_bytes_per_step"] == 4 * n
    rf = ours["roofline"]
    assert rf["bound"] == "hbm" and rf["peak"] > 0 and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert ours["gpu_launches"] > 0 and ours["clocks"]["sm_mhz"] > 0
    assert ours["cpu_baseline"]["gpu_output_equals_reference"] is True
    v = ours["variants"]["mergepath"]
    assert v["output_equals_network_output"] is True and v["value"] > 0
