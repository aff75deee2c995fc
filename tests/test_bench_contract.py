"""bench.py's reference arm (CPU, runs here): the JSON line the driver reads.

The reference arm times the compiled reference (oracle/_ref) on the host;
it must print one JSON line with impl = "reference", the base contract keys,
a cpu_baseline describing the run (kind, cores, sample) and an e2e block
whose value equals the line's own, and exit 0. Non-zero torchrun ranks exit
without work.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, env=None):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=300, env=dict(os.environ, CUDA_VISIBLE_DEVICES="", **(env or {})))


@pytest.fixture(scope="module")
def ref_line():
    from oracle.pyoracle import available
    if not available("ref"):
        pytest.skip("oracle/_ref not built")
    r = _run("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


def test_reference_line_contract(ref_line):
    d = ref_line
    assert d["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["metric"] == "pca_rows_per_sec" and d["unit"] == "rows/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["dtype"] == "f64"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_reference_arm_nonzero_rank_exits_quietly():
    r = _run("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0", env={"RANK": "1"})
    assert r.returncode == 0
    assert not [x for x in r.stdout.splitlines() if x.startswith("{")]
