"""The logtrawl CLI over the B200 path: the reference's
CLI contract (tests/cli_test.sh:20-87 of the reference) restated, and the
JSONL byte-for-byte equal to the reference's own rendering
(render_alerts_jsonl, jsonl.hpp:14-34, produced by oracle/gen_jsonl.cpp from
the unmodified reference into tests/golden/cli_*)."""
import gzip
import hashlib
import os
import re
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
BIN = os.path.join(ROOT, "paper_1704_02278_b200", "logtrawl")
GOLD = os.path.join(HERE, "golden")
ENGINES = ["pfac_compact", "pfac_dense", "kmp", "ac_chunked"]


@pytest.fixture(scope="module")
def cli():
    if not os.path.exists(BIN):
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "paper_1704_02278_b200", "cli")])
    return BIN


def run(args, cwd, env=None):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run(args, cwd=cwd, capture_output=True, timeout=300, env=e)
    return r.returncode, r.stdout


def golden(name):
    with gzip.open(os.path.join(GOLD, name + ".gz"), "rb") as f:
        return f.read()


def test_gen_contract(cli, tmp_path):  # cli_test.sh:63-72
    rc, out = run([cli, "gen", "--size", "1048576", "--seed", "7", "-o", "gen.log"], tmp_path)
    assert rc == 0
    data = (tmp_path / "gen.log").read_bytes()
    assert len(data) == 1048576
    line = out.decode()
    assert re.match(r"^sha256  [0-9a-f]{64} .* 1048576$", line.strip())
    assert line.split()[1] == hashlib.sha256(data).hexdigest()
    rc2, out2 = run([cli, "gen", "--size", "1048576", "--seed", "7", "-o", "gen2.log"], tmp_path)
    assert out2.split()[1] == out.split()[1]


def test_error_exits(cli, tmp_path):  # cli_test.sh:35-44: exit 2 before any device work
    (tmp_path / "empty_rules.txt").write_text("# only comments\n")
    (tmp_path / "rules.txt").write_text("his-rule : HIS\nshe-rule : SHE\n")
    (tmp_path / "hit.log").write_text("SHIS\n")
    assert run([cli, "scan", "-r", "empty_rules.txt", "hit.log"], tmp_path)[0] == 2
    assert run([cli, "scan", "-r", "rules.txt", "missing.log"], tmp_path)[0] == 2
    assert run([cli, "scan", "-r", "rules.txt", "--format", "xml", "hit.log"], tmp_path)[0] == 2
    assert run([cli, "bogus"], tmp_path)[0] == 2


@pytest.mark.gpu
def test_scan_jsonl_equals_reference(cli, tmp_path):
    """Every engine, the reference's alert stream byte for byte."""
    (tmp_path / "hit.log").write_bytes(b"SHIS\n")
    (tmp_path / "clean.log").write_bytes(b"nothing to see\n")
    rc, out = run([cli, "gen", "--size", "200000", "--seed", "42", "--line-len", "80", "-o", "big.log"], tmp_path)
    assert rc == 0
    for case in ("hit", "big"):
        (tmp_path / f"{case}.rules").write_bytes(golden(f"cli_{case}.rules"))
        for eng in ENGINES:
            rc, out = run([cli, "scan", "-r", f"{case}.rules", "--engine", eng, f"{case}.log"], tmp_path)
            assert rc == 1, (case, eng)
            assert out == golden(f"cli_{case}_{eng}.jsonl"), (case, eng)
    rc, out = run([cli, "scan", "-r", "hit.rules", "clean.log"], tmp_path)
    assert rc == 0 and b'"total_matches":0' in out
    rc, out = run([cli, "scan", "-r", "hit.rules", "--format", "summary", "hit.log"], tmp_path)
    assert rc == 1 and b"total_matches=1" in out
    # the pfac engines read the log in windows through the device stream:
    # small reads (feed boundaries) and small device windows give the same bytes
    for eng in ("pfac_compact", "pfac_dense"):
        rc, out = run([cli, "scan", "-r", "big.rules", "--engine", eng, "big.log"], tmp_path,
                      {"LOGTRAWL_READ_WINDOW": "4093", "GLOP_STREAM_WINDOW": "997"})
        assert rc == 1 and out == golden(f"cli_big_{eng}.jsonl"), eng
    w1 = run([cli, "scan", "-r", "big.rules", "--workers", "1", "big.log"], tmp_path)[1]
    w8 = run([cli, "scan", "-r", "big.rules", "--workers", "8", "big.log"], tmp_path)[1]
    we = run([cli, "scan", "-r", "big.rules", "big.log"], tmp_path, {"LOGTRAWL_WORKERS": "3"})[1]
    assert w1 == w8 == we


@pytest.mark.gpu
def test_bench_csv(cli, tmp_path):  # cli_test.sh:74-80
    run([cli, "gen", "--size", "1048576", "--seed", "7", "-o", "gen.log"], tmp_path)
    for eng in ("kmp", "pfac_compact"):
        rc, _ = run([cli, "bench", "-i", "gen.log", "--engine", eng, "--patterns", "10,100", "--runs", "1",
                     "-o", "bench.csv"], tmp_path)
        assert rc == 0
        lines = (tmp_path / "bench.csv").read_text().splitlines()
        assert lines[0] == "engine,backend,patterns,bytes,runs,mean_seconds,throughput_bps"
        assert len(lines) == 3 and lines[1].split(",")[2:5] == ["10", "1048576", "1"]
