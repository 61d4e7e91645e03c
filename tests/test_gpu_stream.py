"""Streaming ingest (glop_stream_begin/feed/end): a text fed
in pieces of any size gives exactly the whole-text result (alerts, counts,
stage-1 hits, LineIndex lines) -- the reference's semantics over the
concatenation (pfac_scan + verify_hits, scan.hpp:177-202, verify.hpp:69-105;
SPEC.md:290's max_len-1 windowing), including matches that straddle a feed()
boundary and a window boundary.  Run on the B200: pytest -m gpu."""
import numpy as np
import pytest

import oracle_ffi as O
from paper_1704_02278_b200 import glop
from paper_1704_02278_b200.parity import alerts16

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return glop.Context(0)


def reference(text, pats, with_lines=True):
    if O.ref() is not None:
        return O.ref_pfac_verify(text, pats, 8, compact=True, workers=0, with_lines=with_lines)
    return O.pfac_verify(text, pats, 8, with_lines=with_lines)


def check(result, text, pats):
    alerts, counts, s1, lines, line_count, nbytes = result
    r_hits, r_alerts = reference(text, pats)
    assert nbytes == text.size
    assert s1 == len(r_hits)
    assert np.array_equal(alerts16(alerts), alerts16(r_alerts))
    assert np.array_equal(lines, r_alerts["line"])
    assert line_count == 1 + int(np.count_nonzero(text == 10))
    assert np.array_equal(counts, np.bincount(r_alerts["rule_id"].astype(np.int64),
                                              minlength=len(pats)).astype(np.uint64))
    return alerts


def test_stream_700mb_random_pieces_vs_reference(ctx):
    """700 MB in random pieces (crossing two 256 MiB windows), occurrences of
    8-byte and 32-byte rules spliced across feed boundaries and window
    boundaries."""
    rng = np.random.default_rng(4)
    n = 700_000_000
    text = glop.gen_syslog_host(n, 21)
    pats, _ = glop.gen_rules(1000, 606)
    pats = list(pats) + [b"Failed password for invalid user", b"straddling-the-window-boundary!!"]
    cuts = np.sort(rng.integers(1, n, 40))
    win = 256 << 20
    splices = [(int(c) - 3, pats[7]) for c in cuts[:10]] + [(int(c) - 17, pats[-1]) for c in cuts[10:20]] + \
              [(win - 5, pats[-1]), (2 * win - 4, pats[3])]
    for at, p in splices:
        text[at:at + len(p)] = np.frombuffer(p, np.uint8)
    trie = ctx.upload(glop.build_failureless_trie(pats, 8))
    rules = ctx.upload_rules(pats, 8)
    st = glop.Stream(ctx, trie, rules, lines=True)
    lo = 0
    for c in list(cuts) + [n]:
        st.feed(text[lo:int(c)])
        lo = int(c)
    alerts = check(st.end(), text, pats)
    got = set(int(o) for o in alerts["offset"])
    for at, _ in splices:
        assert at in got


@pytest.mark.parametrize("window", [64, 4096, 1 << 20])
def test_stream_small_windows_tiny_feeds(ctx, monkeypatch, window):
    """Windows far smaller than the patterns' spans (DPI contents up to 24
    bytes, a 64-byte window) and feeds of 1..300 bytes: every window boundary
    and feed boundary is crossed by some match."""
    monkeypatch.setenv("GLOP_STREAM_WINDOW", str(window))
    rng = np.random.default_rng(window)
    text = glop.gen_payload_host(1 << 20 if window > 64 else 1 << 16, seed=window)
    pats = glop.gen_dpi_rules(2000, 606, 8, 24)
    for at in rng.integers(0, text.size - 32, 300):
        p = pats[int(rng.integers(0, len(pats)))]
        text[int(at):int(at) + len(p)] = np.frombuffer(p, np.uint8)
    trie = ctx.upload(glop.build_failureless_trie(pats, 8))
    rules = ctx.upload_rules(pats, 8)
    st = glop.Stream(ctx, trie, rules, lines=True)
    lo = 0
    while lo < text.size:
        step = int(rng.integers(1, 300)) if window <= 4096 else int(rng.integers(1, 200_000))
        st.feed(text[lo:lo + step])
        lo += step
    check(st.end(), text, pats)


def test_stream_empty_and_without_lines(ctx):
    pats, _ = glop.gen_rules(10, 606)
    trie = ctx.upload(glop.build_failureless_trie(pats, 8))
    rules = ctx.upload_rules(pats, 8)
    st = glop.Stream(ctx, trie, rules)
    alerts, counts, s1, lines, lc, nb = st.end()
    assert len(alerts) == 0 and s1 == 0 and nb == 0 and not counts.any() and lines is None
    st = glop.Stream(ctx, trie, rules)
    text = glop.gen_syslog_host(3 << 20, 5)
    st.feed(text[:12345])
    st.feed(b"")
    st.feed(text[12345:])
    alerts, counts, s1, lines, lc, nb = st.end()
    r_hits, r_alerts = reference(text, pats, with_lines=False)
    assert np.array_equal(alerts16(alerts), alerts16(r_alerts)) and s1 == len(r_hits) and nb == text.size


@pytest.mark.parametrize("members,window", [(1, 1 << 20), (3, 1 << 16), (4, 997)])
def test_group_stream_vs_reference(ctx, members, window):
    """glop_group_stream_*: windows round-robin over the group's members (on
    one GPU here), random feed pieces; the merged result equals the reference's
    over the concatenation, lines included."""
    rng = np.random.default_rng(members * 7 + window)
    text = glop.gen_syslog_host(5 << 20, 31 + members)
    pats, _ = glop.gen_rules(1000, 606)
    pats = list(pats) + [b"Failed password for invalid user", b"session opened for user root by (uid=0)"]
    g = glop.Group([0] * members)
    st = glop.GroupStream(g, g.upload(glop.build_failureless_trie(pats, 8)), g.upload_rules(pats, 8), lines=True,
                          window=window)
    lo = 0
    while lo < text.size:
        step = int(rng.integers(1, 300_000))
        st.feed(text[lo:lo + step])
        lo += step
    check(st.end(), text, pats)
