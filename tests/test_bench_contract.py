"""bench.py's JSON contract, checked on CPU through the reference arm
(`--impl reference` times the reference's own pfac_scan + verify_hits from
oracle/_ref on host cores, so it runs without a GPU), plus the argument
surface the driver uses."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libref_logtrawl.so")


def _run(*args, timeout=600):
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # ONE JSON line
    return json.loads(lines[0])


def test_help_lists_driver_flags():
    out = subprocess.run([sys.executable, "bench.py", "--help"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0
    for flag in ("--gpus", "--steps", "--warmup", "--impl", "--config"):
        assert flag in out.stdout


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built (build() compiles it)")
@pytest.mark.parametrize("config", ["pfac", "kmp"])
def test_reference_arm_line(config):
    d = _run("--impl", "reference", "--config", config, "--steps", "1", "--warmup", "0",
             "--bytes-per-gpu", "2e6")
    assert d["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["unit"] == "Gbps" and d["higher_is_better"] is True and d["n_gpus"] == 1
    assert d["value"] > 0 and d["steps"] == 1
    assert d["metric"].startswith({"pfac": "PFAC log-scan Gbps", "kmp": "KMP log-scan Gbps"}[config])
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built (build() compiles it)")
def test_reference_arm_never_maps_libglop():
    """The reference arm generates its corpus and rules through oracle/_ref:
    with GLOP_LIB pointing nowhere, importing the product binding would fail."""
    env = dict(os.environ, GLOP_LIB="/nonexistent/libglop.so")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                          "--bytes-per-gpu", "1e6", "--no-configs"], cwd=ROOT, capture_output=True, text=True,
                         timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    assert d["parity"]["sha"] and d["cpu_baseline"]["cpu_model"]
