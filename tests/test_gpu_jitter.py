"""GPU race stress: the whole kernel set rebuilt with -DB200_JITTER (random
0..1 us sleeps per lane at every shared-memory hand-off and cluster
exchange, bitonic_static.cuh jitter()), run on every kernel family and
compared with numpy.  compute-sanitizer is refused on this pool, so this
(plus the static proof in tests/test_sync_check.py) is the race evidence."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
JITTER_LIB = os.path.join(ROOT, "paper_1506_01446_b200", "libb200_bitonic_jitter.so")


def _run(extra_env, timeout=900):
    if not os.path.exists(JITTER_LIB):
        pytest.fail("jitter build missing: run __graft_entry__.build()")
    env = dict(os.environ, B200_BITONIC_LIB=JITTER_LIB, **extra_env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "race_workload.py")],
                       capture_output=True, text=True, timeout=timeout, env=env)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0 and "race_workload: OK" in r.stdout


def test_race_workload_under_jitter():
    _run({"SAN_KS": "10,12,13,14,16,18,20,22"})


def test_race_workload_under_jitter_cluster_and_tma():
    # the off-by-default kernels too: 2-CTA cluster passes and the TMA tile
    _run({"SAN_KS": "16,20,24", "B200_BITONIC_CLUSTER": "1", "B200_BITONIC_TMA": "1"})
