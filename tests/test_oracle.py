"""Pins the CPU oracle (oracle/pfac_oracle.c) to the reference.

Every check here compares the C restatement with what the UNMODIFIED
reference computed (tests/golden/, written by oracle/gen_golden.cpp) or with
the reference's own known-answer tests (cited file:line).  CPU only.
"""
import numpy as np
import pytest

import golden_io as G
import oracle_ffi as O


def _hits_key(h):
    return [(int(x["offset"]), int(x["pattern_id"]), int(x["matched_len"])) for x in h]


# ---------------------------------------------------------------- known answers
def test_pfac_shis():  # test_scan.cpp:57-63
    hits = O.pfac_scan(b"SHIS", O.Trie([b"HIS", b"SHE"], 8))
    assert _hits_key(hits) == [(1, 0, 3)]


def test_pfac_intermediate_outputs():  # test_scan.cpp:65-70
    hits = O.pfac_scan(b"ABAB", O.Trie([b"AB", b"ABC"], 8))
    assert _hits_key(hits) == [(0, 0, 2), (2, 0, 2)]


def test_pfac_empty_text():  # test_scan.cpp:72-78
    assert len(O.pfac_scan(b"", O.Trie([b"A"], 8))) == 0


def test_trie_shapes():  # test_automaton.cpp:55-102
    t = O.Trie([b"HIS", b"SHE"], 8)
    assert t.state_count == 7
    assert O.Trie([b"AB", b"ABC"], 8).state_count == 4
    assert O.Trie([], 8).state_count == 1
    with pytest.raises(O.OracleError) as e:
        O.Trie([b"ABCDEFGH"], 8, max_states=4)
    assert e.value.code == 2
    with pytest.raises(O.OracleError):
        O.Trie([b"A"], 0)  # rules.hpp:192-193


def test_trie_bfs_numbering():  # automaton.hpp:198-212 (root 0, BFS, ascending byte)
    t = O.Trie([b"HIS", b"SHE"], 8)
    assert t.table[0, ord("H")] == 1 and t.table[0, ord("S")] == 2
    assert t.table[1, ord("I")] == 3 and t.table[2, ord("H")] == 4
    assert list(t.depth) == [0, 1, 1, 2, 2, 3, 3]


def test_verify_known_answers():  # test_verify.cpp:26-65
    r = [b"GETPASSWORDFILE"]
    a = O.verify_hits(b"0123456789GETPASSWORDFILE....", np.array([(10, 0, 8)], G.HIT_DTYPE), r, 8)
    assert len(a) == 1 and a[0]["offset"] == 10 and a[0]["pattern_len"] == 15
    assert len(O.verify_hits(b"0123456789GETPASSWXYZ..........", np.array([(10, 0, 8)], G.HIT_DTYPE), r, 8)) == 0
    assert len(O.verify_hits(b"rootkit", np.array([(0, 0, 4)], G.HIT_DTYPE), [b"root"], 8)) == 1
    assert len(O.verify_hits(b"..GETPASSW", np.array([(2, 0, 8)], G.HIT_DTYPE), r, 8)) == 0
    with pytest.raises(O.OracleError) as e:
        O.verify_hits(b"ab", np.array([(1, 0, 4)], G.HIT_DTYPE), [b"root"], 8)
    assert e.value.code == 3


def test_line_of():  # test_verify.cpp:114-124
    t = b"abc\ndef\n\nxyz"
    assert [O.line_of(t, o) for o in (0, 3, 4, 8, 9)] == [1, 1, 2, 3, 4]


def test_kmp_known_answers():  # test_kmp.cpp:29-74
    assert list(O.kmp_failure(b"ABAB")) == [0, 0, 1, 2]
    assert list(O.kmp_failure(b"AAAA")) == [0, 1, 2, 3]
    assert list(O.kmp_failure(b"X")) == [0]
    assert list(O.kmp_search(b"AABAABAAB", b"AAB")[0]) == [0, 3, 6]
    assert list(O.kmp_search(b"SHIS", b"HIS")[0]) == [1]
    assert len(O.kmp_search(b"AB", b"HIS")[0]) == 0
    assert list(O.kmp_search(b"AAAA", b"AA")[0]) == [0, 1, 2]


# ---------------------------------------------------------------- golden families
@pytest.mark.parametrize("family", ["known_answer", "loggen_evil", "scan_workers"])
def test_full_records(family):
    for c in G.load(family):
        hits, alerts = O.pfac_verify(c.text, c.patterns, c.L, with_lines=True)
        assert G.pack_hits(hits) == G.pack_hits(c.hits)
        if family == "scan_workers":
            alerts["line"] = 0
        assert G.pack_alerts(alerts) == G.pack_alerts(c.alerts)


def _digest_family(name, gen):
    recs = G.load(name)
    n = 0
    for rec, (pats, text, L, _w) in zip(recs, gen()):
        assert G.sha(G.pack_inputs(pats, text)) == rec.inputs_sha, "regenerator drifted"
        hits, alerts = O.pfac_verify(text, pats, L)
        assert len(hits) == rec.n_hits and G.sha(G.pack_hits(hits)) == rec.hits_sha
        assert len(alerts) == rec.n_alerts and G.sha(G.pack_alerts(alerts)) == rec.alerts_sha
        # the core invariant (acceptance.cpp:72-74): verify(pfac) == naive
        naive = O.naive_scan(text, pats)
        assert np.array_equal(alerts["offset"], naive["offset"])
        assert np.array_equal(alerts["rule_id"], naive["pattern_id"])
        n += 1
    assert n == len(recs)


def test_acceptance_exactness():  # acceptance.cpp:42-78, all 1000 trials
    _digest_family("acceptance_exactness", G.acceptance_exactness_inputs)


def test_scan_superset():  # test_scan.cpp:157-176
    _digest_family("scan_superset", G.scan_superset_inputs)


def test_kmp_families():  # test_kmp.cpp:76-93, acceptance.cpp:209-229
    recs = G.load("kmp_naive")
    digests = [r for r in recs if r.inputs_sha]
    full = [r for r in recs if not r.inputs_sha]
    for rec, (p, text) in zip(digests, G.kmp_naive_inputs()):
        assert G.sha(G.pack_kmp_inputs(p, text)) == rec.inputs_sha
        offs, cmp_ = O.kmp_search(text, p)
        assert len(offs) == rec.n_offsets and G.sha(offs.astype("<u8").tobytes()) == rec.offsets_sha
        assert cmp_ == rec.comparisons and cmp_ <= 2 * len(text)
    for rec in full:
        offs, cmp_ = O.kmp_search(rec.text, rec.pattern)
        assert list(offs) == list(rec.offsets) and cmp_ == rec.comparisons
        assert list(O.kmp_failure(rec.pattern)) == list(rec.table)
    for rec, (p, text) in zip(G.load("kmp_bound"), G.kmp_bound_inputs()):
        assert G.sha(G.pack_kmp_inputs(p, text)) == rec.inputs_sha
        offs, cmp_ = O.kmp_search(text, p)
        assert cmp_ == rec.comparisons and len(offs) == rec.n_offsets


def test_reference_shim_agrees_when_built():
    """Where the reference was compiled (oracle/_ref), the oracle equals it on
    a syslog-like random case too (not just the fixtures)."""
    if O.ref() is None:
        pytest.skip("oracle/_ref not built on this box")
    rng = np.random.default_rng(3)
    text = bytes(rng.integers(65, 70, 20000, dtype=np.uint8))
    pats = list({bytes(rng.integers(65, 70, int(rng.integers(1, 12)), dtype=np.uint8)) for _ in range(40)})
    for L in (3, 8):
        h1, a1 = O.pfac_verify(text, pats, L, with_lines=True)
        for compact in (False, True):
            h2, a2 = O.ref_pfac_verify(text, pats, L, compact=compact, workers=3, with_lines=True)
            assert G.pack_hits(h1) == G.pack_hits(h2)
            assert G.pack_alerts(a1) == G.pack_alerts(a2)
