"""Multi-GPU inside libglop (glop_group): N contexts -- on one
device here, one per GPU on an 8-GPU box -- split the text into halo'd
shards and merge in rank order.  Results must be byte-identical to one
context and to the oracle for every N (the worker-determinism property of
test_scan.cpp:80-88 / acceptance.cpp:183-206), KMP comparison counts
included (each shard recovers the KMP state from m-1 bytes of left context).
Also the drop-in C++ API (tests/cpp/dropin_test) run on a 3-member group.
Run on the B200: pytest -m gpu."""
import os
import subprocess

import numpy as np
import pytest

import oracle_ffi as O
from paper_1704_02278_b200 import glop
from paper_1704_02278_b200.parity import alerts16

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ctx():
    return glop.Context(0)


def group(n, monkeypatch, min_shard=1 << 16):
    monkeypatch.setenv("GLOP_GROUP_MIN_SHARD", str(min_shard))
    return glop.Group([0] * n)


@pytest.mark.parametrize("members", [1, 2, 3, 4, 8])
def test_group_pfac_and_pipeline_equal_single(ctx, members, monkeypatch):
    g = group(members, monkeypatch)
    assert g.size == members
    text = glop.gen_syslog_host(3 << 20, seed=31)
    pats, _ = glop.gen_rules(1000, 606)
    pats = list(pats) + [b"Failed password for invalid user", b"session opened for user root by"]
    a = glop.build_failureless_trie(pats, 8)
    ref_hits = O.pfac_scan(text, O.Trie(pats, 8))
    assert g.pfac_scan(g.upload(a), text).tobytes() == ref_hits.tobytes()
    assert ctx.pfac_scan(ctx.upload(a), text).tobytes() == ref_hits.tobytes()
    ref_alerts = O.verify_hits(text, ref_hits, pats, 8, with_lines=True)
    alerts, counts, s1, lines, line_count = g.run_pfac_pipeline(g.upload(a), g.upload_rules(pats, 8), text,
                                                                lines=True)
    assert s1 == len(ref_hits)
    assert np.array_equal(alerts16(alerts), alerts16(ref_alerts))
    assert np.array_equal(lines, ref_alerts["line"])
    assert line_count == 1 + int(np.count_nonzero(text == 10))
    assert np.array_equal(counts, np.bincount(ref_alerts["rule_id"].astype(np.int64),
                                              minlength=len(pats)).astype(np.uint64))


@pytest.mark.parametrize("members", [2, 5, 8])
def test_group_kmp_exact_comparisons(members, monkeypatch):
    """Shard boundaries inside runs of a self-overlapping pattern: the KMP
    state at a boundary is not 0, so the shard must recover it."""
    g = group(members, monkeypatch, min_shard=4096)
    rng = np.random.default_rng(members)
    text = np.full(1 << 18, 97, dtype=np.uint8)  # 'a' ...
    text[rng.integers(0, text.size, 2000)] = 98  # ... with a few 'b'
    for p in (b"aaaa", b"aab", b"abaab", b"Failed password"):
        offs, cmp_ = g.kmp_search(p, text)
        r_offs, r_cmp = O.kmp_search(text, p)
        assert np.array_equal(offs, r_offs), p
        assert cmp_ == r_cmp, (p, cmp_, r_cmp)


def test_group_uses_fewer_members_on_small_text(monkeypatch):
    g = group(4, monkeypatch, min_shard=1 << 20)
    text = glop.gen_syslog_host(1 << 19, seed=2)  # below one min shard: one member works
    pats, _ = glop.gen_rules(100, 606)
    a = glop.build_failureless_trie(pats, 8)
    assert g.pfac_scan(g.upload(a), text).tobytes() == O.pfac_scan(text, O.Trie(pats, 8)).tobytes()


def test_dropin_cpp_on_three_member_group():
    """The drop-in C++ API (pfac_scan, verify_hits, run_engine_scan with lines,
    kmp, chunked AC) on a 3-context group: GLOP_DEVICES=0,0,0."""
    exe = os.path.join(ROOT, "tests", "cpp", "dropin_test")
    if not os.path.exists(exe):
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")])
    env = dict(os.environ, GLOP_DEVICES="0,0,0", GLOP_GROUP_MIN_SHARD="512")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout + r.stderr


def test_group_pipeline_pageable_shards_over_one_chunk(monkeypatch):
    """Two members each scanning a > 256 MiB shard of PAGEABLE text: both
    members' streamed pipelines stage their chunks through the shared host
    copy pool at the same time; the merge equals the reference."""
    g = group(2, monkeypatch)
    n = (600 << 20) + 12345
    text = glop.gen_syslog_host(n, seed=77)
    pats, _ = glop.gen_rules(1000, 606)
    alerts, counts, s1, lines, line_count = g.run_pfac_pipeline(
        g.upload(glop.build_failureless_trie(pats, 8)), g.upload_rules(pats, 8), text, lines=True)
    if O.ref() is not None:
        r_hits, r_alerts = O.ref_pfac_verify(text, pats, 8, compact=True, workers=0, with_lines=True)
    else:
        r_hits, r_alerts = O.pfac_verify(text, pats, 8, with_lines=True)
    assert s1 == len(r_hits)
    assert np.array_equal(alerts16(alerts), alerts16(r_alerts))
    assert np.array_equal(lines, r_alerts["line"])
    assert np.array_equal(counts, np.bincount(r_alerts["rule_id"].astype(np.int64),
                                              minlength=len(pats)).astype(np.uint64))
