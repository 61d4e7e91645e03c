"""CPU-side checks of the C ABI library (no kernel launches): it loads,
exports every entry point include/glop.h declares, and its host-side pieces
(automaton builder, workload generators) agree with the oracle / reference."""
import os
import re

import numpy as np
import pytest

import golden_io as G
import oracle_ffi as O
from paper_1704_02278_b200 import glop

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "glop.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(glop_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    names = _declared()
    assert len(names) >= 25
    lib = glop.lib_handle()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_no_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(glop.CudaError):
        glop.Context(0)


def _cmp_trie(pats, L):
    a = glop.build_failureless_trie(pats, L)
    o = O.Trie(pats, L)
    assert a.state_count == o.state_count
    assert np.array_equal(a.dense_table, o.table)
    assert np.array_equal(a.out_offsets, o.out_offsets)
    assert np.array_equal(a.out_flat, o.out_flat)


def test_trie_builder_matches_oracle():
    # automaton.hpp:147-212: BFS numbering, children by ascending byte,
    # merged-prefix outputs in id order
    _cmp_trie([b"HIS", b"SHE"], 8)
    _cmp_trie([b"AB", b"ABC"], 8)
    _cmp_trie([b"ABCDEFGHX", b"ABCDEFGHY", b"ABC"], 8)
    rng = np.random.default_rng(5)
    for trial in range(200):
        full = trial % 2 == 1
        k = int(rng.integers(1, 40))
        pats = list({bytes(rng.integers(0, 256 if full else 4, int(rng.integers(1, 17)), dtype=np.uint8) +
                            (0 if full else 65)) for _ in range(k)})
        _cmp_trie(pats, int(rng.choice([1, 2, 4, 8, 64])))


def test_trie_builder_errors():
    with pytest.raises(glop.CapacityError):  # test_automaton.cpp:96-102
        glop.build_failureless_trie([b"ABCDEFGH"], 8, max_states=4)
    with pytest.raises(glop.InvalidArgument):  # rules.hpp:192-193
        glop.build_failureless_trie([b"A"], 0)
    assert glop.build_failureless_trie([], 8).state_count == 1


def test_host_corpus_matches_golden():
    recs = {r.name: r for r in G.load("syslog")}
    t = glop.gen_syslog_host(recs["syslog_k10"].n, seed=1)
    assert G.sha(t.tobytes()) == recs["syslog_k10"].text_sha
    mid = glop.gen_syslog_host(100000, seed=1, begin=123457)
    assert G.sha(mid.tobytes()) == recs["syslog_mid"].text_sha
    # ranges compose: [0, a) + [a, n) == [0, n)
    a = glop.gen_syslog_host(5000, seed=9)
    b = glop.gen_syslog_host(7000, seed=9, begin=5000)
    assert np.array_equal(np.concatenate([a, b]), glop.gen_syslog_host(12000, seed=9))
    assert t[4095] == 10 and t[8191] == 10  # every block ends with LF


def test_reference_generators():
    # loggen.hpp:44-57 via the loggen_evil fixture (generate_log(10000,77,40)
    # with EVILEVL spliced at 4321)
    (c,) = G.load("loggen_evil")
    t = glop.gen_reference_log(10000, 77, 40).tobytes()
    assert t[:4321] == c.text[:4321] and t[4328:] == c.text[4328:]
    pats, vocab = glop.gen_rules(1000, 7)
    recs = {r.name: r for r in G.load("syslog")}
    assert pats == recs["syslog_k1000"].patterns
    assert len(set(pats)) == 1000 and all(len(p) == 8 for p in pats)
    assert 400 <= int(vocab.sum()) <= 500


def test_kmp_failure_table():  # test_kmp.cpp:29-36
    assert list(glop.kmp_failure_table(b"ABAB")) == [0, 0, 1, 2]
    assert list(glop.kmp_failure_table(b"AAAA")) == [0, 1, 2, 3]
    for p in (b"Failed password", b"ABABCABAB", b"x"):
        assert list(glop.kmp_failure_table(p)) == list(O.kmp_failure(p))


def test_engine_library_exports_and_fails_loudly_without_gpu():
    """libglop_engine.so (run_engine_scan behind a C ABI): loads, exports its
    entry points, builds a RuleSet on the host, and -- with no sm_100 device --
    reports the failure instead of falling back to the host."""
    import torch

    eng = glop.Engine([b"Failed password", b"root"])
    for n in ("glop_engine_rules_create", "glop_engine_rules_destroy", "glop_engine_run", "glop_engine_last_error"):
        assert hasattr(eng.lib, n)
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    text = np.frombuffer(b"x Failed password for root\n", np.uint8).copy()
    with pytest.raises(glop.GlopError):
        eng.run(text.ctypes.data, text.size)
    eng.close()
