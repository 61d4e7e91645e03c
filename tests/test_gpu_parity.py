"""GPU parity: the sm_100a kernels (through the C ABI) against the reference's
golden vectors and the CPU oracle.  Bit-exact for every hit, alert, offset
and comparison count.  Run on the B200: pytest -m gpu."""
import os
import subprocess

import numpy as np
import pytest

import golden_io as G
import oracle_ffi as O
from paper_1704_02278_b200 import glop

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# AUTO runs the PREFIX8 kernel whenever every output lies at depth >= 8
KERNELS = [glop.PFAC_AUTO, glop.PFAC_FILTERED, glop.PFAC_DIRECT]


@pytest.fixture(scope="module")
def ctx():
    return glop.Context(0)


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    assert torch.cuda.is_available(), "-m gpu tests need the B200"
    return torch


def dev_scan(ctx, torch, trie, text: np.ndarray, kernel, own=None, base=0, offset=0):
    """pfac_scan_device over text[offset:] resident in HBM."""
    n = text.size - offset
    d = torch.from_numpy(np.array(text, dtype=np.uint8, copy=True)).cuda() if text.size else torch.zeros(1, dtype=torch.uint8).cuda()
    cap = max(1 << 16, 4 * n)
    out = torch.empty(cap * 16, dtype=torch.uint8, device="cuda")
    nh = ctx.pfac_scan_device(trie, d.data_ptr() + offset, n, out.data_ptr(), cap, own=own, base=base, kernel=kernel)
    ctx.synchronize()
    return out[: nh * 16].cpu().numpy().view(glop.HIT_DTYPE).copy()


def alerts_as_golden(a, lines=None):
    out = np.zeros(len(a), dtype=G.ALERT_DTYPE)
    out["offset"], out["rule_id"], out["pattern_len"] = a["offset"], a["rule_id"], a["pattern_len"]
    if lines is not None:
        out["line"] = lines
    return out


def line_numbers(text: np.ndarray, offsets) -> np.ndarray:
    """LineIndex::line_of (verify.hpp:48-53) for test bookkeeping."""
    nl = np.flatnonzero(text == 10)
    return np.searchsorted(nl + 1, np.asarray(offsets, dtype=np.int64), side="right") + 1


def run_case(ctx, pats, text, L, kernel):
    trie = ctx.upload(glop.build_failureless_trie(pats, L))
    hits = ctx.pfac_scan(trie, text) if kernel is None else dev_scan(ctx, __import__("torch"), trie,
                                                                     np.frombuffer(text, np.uint8), kernel)
    rules = ctx.upload_rules(pats, L)
    alerts = ctx.verify_hits(rules, text, hits)
    return hits, alerts


# ------------------------------------------------------------------ known answers
def test_known_answers(ctx):
    """test_scan.cpp:57-78, test_verify.cpp:26-65 via the golden records."""
    for c in G.load("known_answer") + G.load("loggen_evil") + G.load("scan_workers"):
        for kernel in (None, *KERNELS):
            hits, alerts = run_case(ctx, c.patterns, c.text, c.L, kernel)
            assert G.pack_hits(hits) == G.pack_hits(c.hits)
            t = np.frombuffer(c.text, np.uint8)
            lines = line_numbers(t, alerts["offset"]) if c.alerts["line"].any() else None
            assert G.pack_alerts(alerts_as_golden(alerts, lines)) == G.pack_alerts(c.alerts)


def test_errors_map_to_reference_exceptions(ctx):
    rules = ctx.upload_rules([b"root"], 8)
    with pytest.raises(glop.LogicError):  # verify.hpp:76-77
        ctx.verify_hits(rules, b"ab", np.array([(1, 0, 4)], dtype=glop.HIT_DTYPE))
    a = glop.build_failureless_trie([b"AB"], 8)
    bad = glop.Automaton(a.dense_table.copy(), a.out_offsets, a.out_flat)
    bad.dense_table[1, ord("Z")] = 0  # edge back to the root: not a trie
    with pytest.raises(glop.InvalidArgument):
        ctx.upload(bad)


# ------------------------------------------------------------------ randomized families
@pytest.mark.parametrize("family,gen", [("acceptance_exactness", G.acceptance_exactness_inputs),
                                        ("scan_superset", G.scan_superset_inputs)])
def test_randomized_families(ctx, torch_cuda, family, gen):
    """acceptance.cpp:42-78 (1000 trials) and test_scan.cpp:157-176: both
    kernels bit-identical to the reference (hit and alert digests)."""
    for rec, (pats, text, L, _w) in zip(G.load(family), gen()):
        assert G.sha(G.pack_inputs(pats, text)) == rec.inputs_sha
        trie = ctx.upload(glop.build_failureless_trie(pats, L))
        rules = ctx.upload_rules(pats, L)
        t = np.frombuffer(text, np.uint8)
        for kernel in KERNELS:
            hits = dev_scan(ctx, torch_cuda, trie, t, kernel)
            assert len(hits) == rec.n_hits and G.sha(G.pack_hits(hits)) == rec.hits_sha, (family, kernel)
        alerts = ctx.verify_hits(rules, text, hits)
        assert len(alerts) == rec.n_alerts
        assert G.sha(G.pack_alerts(alerts_as_golden(alerts))) == rec.alerts_sha


def test_kmp_families(ctx):
    """test_kmp.cpp:58-93, acceptance.cpp:209-229: offsets and the exact
    sequential comparison count."""
    recs = G.load("kmp_naive")
    for rec, (p, text) in zip([r for r in recs if r.inputs_sha], G.kmp_naive_inputs()):
        offs, cmp_ = ctx.kmp_search(p, text)
        assert len(offs) == rec.n_offsets and G.sha(offs.astype("<u8").tobytes()) == rec.offsets_sha
        assert cmp_ == rec.comparisons
    for rec in [r for r in recs if not r.inputs_sha]:
        offs, cmp_ = ctx.kmp_search(rec.pattern, rec.text)
        assert list(offs) == list(rec.offsets) and cmp_ == rec.comparisons
    for rec, (p, text) in zip(G.load("kmp_bound"), G.kmp_bound_inputs()):
        offs, cmp_ = ctx.kmp_search(p, text)
        assert cmp_ == rec.comparisons and len(offs) == rec.n_offsets and cmp_ <= 2 * len(text)


# ------------------------------------------------------------------ large texts
def test_reference_corpus_fixtures(ctx, torch_cuda):
    """acceptance.cpp:165-206: 10 MB reference corpora (determinism with 50
    spliced patterns; stage-1 false-positive rate)."""
    for name in ("determinism", "fp_rate"):
        (rec,) = G.load(name)
        if name == "determinism":
            text = bytearray(glop.gen_reference_log(10_000_000, 1111, 80).tobytes())
            rng = G.MT19937(1313)
            for _ in range(50):
                p = rec.patterns[rng() % len(rec.patterns)]
                pos = rng() % (len(text) - len(p))
                text[pos:pos + len(p)] = p
            text = bytes(text)
        else:
            text = glop.gen_reference_log(10_000_000, 909, 80).tobytes()
        assert G.sha(text) == rec.text_sha
        t = np.frombuffer(text, np.uint8)
        trie = ctx.upload(glop.build_failureless_trie(rec.patterns, rec.L))
        rules = ctx.upload_rules(rec.patterns, rec.L)
        for kernel in KERNELS:
            hits = dev_scan(ctx, torch_cuda, trie, t, kernel)
            assert len(hits) == rec.n_hits
            alerts = ctx.verify_hits(rules, text, hits)
            got = alerts_as_golden(alerts, line_numbers(t, alerts["offset"]))
            assert G.pack_alerts(got) == G.pack_alerts(rec.alerts)


def test_syslog_golden(ctx, torch_cuda):
    """The synthetic RFC 5424 corpus scanned by the reference pipeline."""
    recs = {r.name: r for r in G.load("syslog")}
    for name in ("syslog_k10", "syslog_k1000", "syslog_mid"):
        rec = recs[name]
        t = glop.gen_syslog_host(rec.n, seed=1, begin=123457 if name == "syslog_mid" else 0)
        assert G.sha(t.tobytes()) == rec.text_sha
        trie = ctx.upload(glop.build_failureless_trie(rec.patterns, rec.L))
        rules = ctx.upload_rules(rec.patterns, rec.L)
        for kernel in KERNELS:
            hits = dev_scan(ctx, torch_cuda, trie, t, kernel)
            assert len(hits) == rec.n_hits
            alerts = ctx.verify_hits(rules, t, hits)
            assert G.pack_alerts(alerts_as_golden(alerts, line_numbers(t, alerts["offset"]))) == G.pack_alerts(rec.alerts)


def test_device_corpus_equals_host(ctx, torch_cuda):
    for begin, n in ((0, 1 << 20), (123457, 300001), (4095, 2), (1 << 30, 70000)):
        d = torch_cuda.empty(n, dtype=torch_cuda.uint8, device="cuda")
        ctx.gen_syslog_device(d.data_ptr(), n, seed=5, begin=begin)
        ctx.synchronize()
        assert np.array_equal(d.cpu().numpy(), glop.gen_syslog_host(n, seed=5, begin=begin))


@pytest.mark.parametrize("k", [10, 1000])
def test_large_syslog_vs_oracle(ctx, torch_cuda, k):
    """64 MB device-generated syslog: both kernels == oracle, hit for hit."""
    n = 64 << 20
    d = torch_cuda.empty(n, dtype=torch_cuda.uint8, device="cuda")
    ctx.gen_syslog_device(d.data_ptr(), n, seed=42)
    ctx.synchronize()
    text = d.cpu().numpy()
    pats, _ = glop.gen_rules(k, seed=606)
    trie = ctx.upload(glop.build_failureless_trie(pats, 8))
    ref = O.pfac_scan(text, O.Trie(pats, 8))
    assert len(ref) > 0
    assert trie.info.min_depth >= 8
    for kernel in KERNELS + [glop.PFAC_PREFIX8]:
        assert dev_scan(ctx, torch_cuda, trie, text, kernel).tobytes() == ref.tobytes()


# level-1 table layouts of the PREFIX8 kernel (pfac8.cuh): the host picks
# lane-replicated bits, one-byte d-mask buckets or one-bit buckets (+ a second
# level-2 bit, + two level-1 bits) by gram count; force each
P8_LAYOUTS = {"auto": {}, "bytes": {"GLOP_P8_BITS_MIN": "1000000000", "GLOP_P8_LANE_MAX": "0"},
              "lane": {"GLOP_P8_LANE_MAX": "1000000000"},
              "bits": {"GLOP_P8_BITS_MIN": "0", "GLOP_P8_BLOOM2_MIN": "1000000000", "GLOP_P8_LANE_MAX": "0"},
              "bits+bloom2": {"GLOP_P8_BITS_MIN": "0", "GLOP_P8_BLOOM2_MIN": "0", "GLOP_P8_LANE_MAX": "0"},
              "two-bit": {"GLOP_P8_BITS_MIN": "0", "GLOP_P8_BLOOM2_MIN": "0", "GLOP_P8_BITS2_MIN": "0",
                          "GLOP_P8_LANE_MAX": "0"}}


@pytest.mark.parametrize("layout", list(P8_LAYOUTS))
def test_prefix8_shards_and_dense(ctx, torch_cuda, layout, monkeypatch):
    """PREFIX8 kernel: shards with halo == whole == oracle; colliding
    prefixes (several ids per state); a hit-dense text (exact fallback)."""
    for k, v in P8_LAYOUTS[layout].items():
        monkeypatch.setenv(k, v)
    text = glop.gen_syslog_host(6 << 20, seed=31)
    pats, _ = glop.gen_rules(300, seed=5)
    pats += [b"Failed password", b"Failed passwd", b"<38>1 2026-", b"\n<38>1 20"]
    trie = ctx.upload(glop.build_failureless_trie(pats, 8))
    assert trie.info.min_depth == 8
    ref = O.pfac_scan(text, O.Trie(pats, 8))
    whole = dev_scan(ctx, torch_cuda, trie, text, glop.PFAC_PREFIX8)
    assert whole.tobytes() == ref.tobytes()
    for shards in (2, 7):
        S = -(-text.size // shards)
        parts = []
        for g in range(shards):
            lo, hi = g * S, min((g + 1) * S, text.size)
            rd = min(hi + 7, text.size)
            parts.append(dev_scan(ctx, torch_cuda, trie, text[lo:rd], glop.PFAC_PREFIX8, own=hi - lo, base=lo))
        assert np.concatenate(parts).tobytes() == whole.tobytes()
    dense = np.frombuffer(b"A" * 70000 + b"AAAAAAAAB" + b"A" * 3001, np.uint8)
    dp = [b"AAAAAAAAx", b"AAAAAAAAy", b"AAAAAAAB", b"AAAAAAAAB"]
    dtrie = ctx.upload(glop.build_failureless_trie(dp, 8))
    dref = O.pfac_scan(dense, O.Trie(dp, 8))
    assert len(dref) > 100000
    assert dev_scan(ctx, torch_cuda, dtrie, dense, glop.PFAC_PREFIX8).tobytes() == dref.tobytes()
    with pytest.raises(glop.InvalidArgument):  # PREFIX8 needs depth >= 8 outputs
        dev_scan(ctx, torch_cuda, ctx.upload(glop.build_failureless_trie([b"AB"], 8)), dense, glop.PFAC_PREFIX8)


def test_shards_with_halo_equal_whole(ctx, torch_cuda):
    """Contiguous shards reporting only owned starts, reading an
    (lmax-1)-byte halo, concatenate to the whole-text result."""
    text = glop.gen_syslog_host(8 << 20, seed=3)
    pats, _ = glop.gen_rules(1000, seed=17)
    pats += [b"\n<38>1 2026", b"Fa", b"ssh2\n<"]  # short + line-crossing prefixes
    trie = ctx.upload(glop.build_failureless_trie(pats, 8))
    whole = dev_scan(ctx, torch_cuda, trie, text, glop.PFAC_FILTERED)
    lmax = trie.info.max_depth
    for shards in (2, 3, 8):
        S = -(-text.size // shards)
        parts = []
        for g in range(shards):
            lo, hi = g * S, min((g + 1) * S, text.size)
            rd = min(hi + lmax - 1, text.size)
            parts.append(dev_scan(ctx, torch_cuda, trie, text[lo:rd], glop.PFAC_FILTERED, own=hi - lo, base=lo))
        assert np.concatenate(parts).tobytes() == whole.tobytes()


def test_unaligned_text(ctx, torch_cuda):
    text = glop.gen_syslog_host(1 << 20, seed=8)
    pats, _ = glop.gen_rules(100, seed=2)
    trie = ctx.upload(glop.build_failureless_trie(pats, 8))
    for off in (1, 3, 7, 13):
        ref = O.pfac_scan(text[off:], O.Trie(pats, 8))
        for kernel in KERNELS:
            assert dev_scan(ctx, torch_cuda, trie, text, kernel, offset=off).tobytes() == ref.tobytes()


def test_hit_dense_fallback(ctx):
    """More hits than a tile's shared-memory buffer: exact global fallback."""
    text = b"A" * 100000 + b"B" + b"A" * 5000
    pats = [b"A", b"AA", b"AAA", b"AB"]
    trie = ctx.upload(glop.build_failureless_trie(pats, 8))
    ref = O.pfac_scan(text, O.Trie(pats, 8))
    assert ctx.pfac_scan(trie, text).tobytes() == ref.tobytes()
    offs, cmp_ = ctx.kmp_search(b"AA", text)
    r_offs, r_cmp = O.kmp_search(text, b"AA")
    assert np.array_equal(offs, r_offs) and cmp_ == r_cmp


def test_kmp_large(ctx, torch_cuda):
    n = 32 << 20
    text = glop.gen_syslog_host(n, seed=21)
    for p in (b"Failed password", b"session opened for user root", b"x"):
        offs, cmp_ = ctx.kmp_search(p, text)
        r_offs, r_cmp = O.kmp_search(text, p)
        assert np.array_equal(offs, r_offs) and cmp_ == r_cmp


def test_verify_unsorted_and_counts(ctx):
    text = b"xxGETPASSWORDFILExxGETPASSWxx root"
    pats = [b"GETPASSWORDFILE", b"root"]
    rules = ctx.upload_rules(pats, 8)
    hits = np.array([(30, 1, 4), (2, 0, 8), (19, 0, 8)], dtype=glop.HIT_DTYPE)
    alerts, counts = ctx.verify_hits(rules, text, hits, counts=True)
    assert [(int(a["offset"]), int(a["rule_id"])) for a in alerts] == [(2, 0), (30, 1)]
    assert list(counts) == [1, 1]


def test_dropin_cpp_binary():
    """The reference's C++ call sites compiled against include/logtrawl."""
    exe = os.path.join(ROOT, "tests", "cpp", "dropin_test")
    if not os.path.exists(exe):
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("k,L,lens", [(10000, 8, (8, 8)), (300, 16, (12, 16)), (200, 64, (9, 40)),
                                      (500, 8, (1, 8)), (64, 4096, (2, 30))])
def test_kernel_variants_vs_oracle(ctx, torch_cuda, k, L, lens):
    """Jump table in global memory (k=10000), lmin > 8 (jump depth 8 then a
    table walk), stride-1 sampling (1-byte patterns), long prefixes."""
    rng = np.random.default_rng(k + L)
    text = glop.gen_syslog_host(4 << 20, seed=k)
    vocab = [text[o:o + int(rng.integers(lens[0], lens[1] + 1))].tobytes()
             for o in rng.integers(0, text.size - 64, k // 2)]
    rand = [bytes(rng.integers(32, 127, int(rng.integers(lens[0], lens[1] + 1)), dtype=np.uint8))
            for _ in range(k - k // 2)]
    pats = list(dict.fromkeys(vocab + rand))
    trie = ctx.upload(glop.build_failureless_trie(pats, L))
    ref = O.pfac_scan(text, O.Trie(pats, L))
    for kernel in KERNELS:
        got = dev_scan(ctx, torch_cuda, trie, text, kernel)
        assert got.tobytes() == ref.tobytes(), (kernel, len(got), len(ref))
    if k == 10000:
        assert not trie.info.jump_in_smem


def test_streamed_host_pipeline(ctx, torch_cuda):
    """Host-text pipeline (chunked H2D overlapped with scan + verify, SURVEY
    §8f row 2) == the device-resident pipeline: alerts, counts, stage-1 hits,
    across chunk boundaries, with a shard's own/base and a halo."""
    n = (256 << 20) * 2 + 12345  # > 2 streaming chunks
    d = torch_cuda.empty(n + 64, dtype=torch_cuda.uint8, device="cuda")
    ctx.gen_syslog_device(d.data_ptr(), n, seed=77)
    ctx.synchronize()
    host = d[:n].cpu().numpy()
    pats, _ = glop.gen_rules(1000, seed=606)
    pats += [b"Failed password for invalid user", b"session opened for user root by"]
    trie = ctx.upload(glop.build_failureless_trie(pats, 8))
    rules = ctx.upload_rules(pats, 8)
    for own, base in ((n, 0), (n - 1000, 5 << 30)):
        ref = ctx.run_pfac_pipeline(trie, rules, d.data_ptr(), n, True, own=own, base=base)
        got = ctx.run_pfac_pipeline(trie, rules, host.ctypes.data, n, False, own=own, base=base)
        assert got[2] == ref[2] and len(ref[0]) > 1000
        assert got[0].tobytes() == ref[0].tobytes()
        assert np.array_equal(got[1], ref[1])
    # and both equal the oracle on a window that straddles the first chunk boundary
    lo = (256 << 20) - 5000
    win = host[lo: lo + 20000]
    w_alerts = ctx.run_pfac_pipeline(trie, rules, win.ctypes.data, win.size, False)[0]
    ref_alerts = O.verify_hits(win, O.pfac_scan(win, O.Trie(pats, 8)), pats, 8)
    assert np.array_equal(w_alerts["offset"], ref_alerts["offset"])
    assert np.array_equal(w_alerts["rule_id"], ref_alerts["rule_id"])


def test_dpi_payloads_vs_oracle(ctx, torch_cuda):
    """DPI configuration (configs[4]): 10,000 Snort-style contents of 8..24
    bytes over full-byte packet payloads -- 8-byte-prefix scan (u32 table,
    > 32K states) + stage-2 suffix verification == the oracle; device
    payload generator == host."""
    n = 8 << 20
    d = torch_cuda.empty(n + 64, dtype=torch_cuda.uint8, device="cuda")
    ctx.gen_payload_device(d.data_ptr(), n, seed=1, begin=3 << 20)
    ctx.synchronize()
    text = d[:n].cpu().numpy()
    assert np.array_equal(text, glop.gen_payload_host(n, seed=1, begin=3 << 20))
    pats = glop.gen_dpi_rules(10000, seed=606, min_len=8, max_len=24)
    trie = ctx.upload(glop.build_failureless_trie(pats, 8))
    assert trie.info.state_count > 32768 and trie.info.min_depth == 8
    rules = ctx.upload_rules(pats, 8)
    ref_hits = O.pfac_scan(text, O.Trie(pats, 8))
    for kernel in (glop.PFAC_PREFIX8, glop.PFAC_FILTERED):
        hits = dev_scan(ctx, torch_cuda, trie, text, kernel)
        assert hits.tobytes() == ref_hits.tobytes()
    ref_alerts = O.verify_hits(text, ref_hits, pats, 8)
    alerts, counts, s1 = ctx.run_pfac_pipeline(trie, rules, d.data_ptr(), n, True)
    assert s1 == len(ref_hits) and len(alerts) < s1  # some prefix hits fail stage 2
    assert np.array_equal(alerts["offset"], ref_alerts["offset"])
    assert np.array_equal(alerts["rule_id"], ref_alerts["rule_id"])
    assert counts.sum() == len(alerts)


def test_device_line_index(ctx, torch_cuda):
    """Device LineIndex == LineIndex::line_of
    (verify.hpp:40-64, via the oracle) and == the reference's golden alert
    lines; offsets at LFs, block edges, 0 and n; unaligned text; the device
    form on alert records with a shard base."""
    t = glop.gen_syslog_host(3_000_017, seed=12)
    rng = np.random.default_rng(4)
    nl = np.flatnonzero(t == 10)
    offs = np.concatenate([[0, t.size, 4095, 4096, 4097], nl[:50], nl[:50] + 1,
                           rng.integers(0, t.size, 5000)]).astype(np.uint64)
    want = (np.searchsorted(nl, offs.astype(np.int64), side="left") + 1).astype(np.uint64)
    assert [O.line_of(t, int(o)) for o in offs[:60]] == want[:60].tolist()  # the oracle pins the rule
    assert np.array_equal(ctx.line_numbers(t, offs), want)
    t3 = t[3:]
    o3 = offs[offs <= t3.size]
    assert np.array_equal(ctx.line_numbers(t3, o3),
                          np.searchsorted(np.flatnonzero(t3 == 10), o3.astype(np.int64), side="left") + 1)
    # the reference's own alert lines (acceptance.cpp:183-206 fixture)
    (rec,) = G.load("determinism")
    text = bytearray(glop.gen_reference_log(10_000_000, 1111, 80).tobytes())
    rng2 = G.MT19937(1313)
    for _ in range(50):
        p = rec.patterns[rng2() % len(rec.patterns)]
        pos = rng2() % (len(text) - len(p))
        text[pos:pos + len(p)] = p
    text = np.frombuffer(bytes(text), np.uint8)
    assert len(rec.alerts) > 0 and rec.alerts["line"].all()
    assert np.array_equal(ctx.line_numbers(text, rec.alerts["offset"]), rec.alerts["line"])
    # device form over alert records (stride 16) of a shard at global base
    base = 7 << 30
    pats, _ = glop.gen_rules(300, seed=9)
    trie = ctx.upload(glop.build_failureless_trie(pats, 8))
    rules = ctx.upload_rules(pats, 8)
    d = torch_cuda.from_numpy(t.copy()).cuda()
    alerts, _, _ = ctx.run_pfac_pipeline(trie, rules, d.data_ptr(), t.size, True, base=base)
    assert len(alerts) > 100
    da = torch_cuda.from_numpy(alerts.view(np.uint8).copy()).cuda()
    dl = torch_cuda.zeros(len(alerts), dtype=torch_cuda.int64, device="cuda")
    ctx.line_numbers_device(d.data_ptr(), t.size, da.data_ptr(), 16, len(alerts), dl.data_ptr(), base=base)
    ctx.synchronize()
    ref = [O.line_of(t, int(o) - base) for o in alerts["offset"]]
    assert dl.cpu().numpy().tolist() == ref


def test_kmp_shards_equal_whole(ctx, torch_cuda):
    """KMP shard form: starts [0, own) with an (m-1)-byte halo; offsets and
    comparison counts of the shards sum to the whole-text reference."""
    text = glop.gen_syslog_host(3_000_000, seed=41)
    for p in (b"Failed password", b"ab", b"session opened for user root by (uid=0)"):
        r_offs, r_cmp = O.kmp_search(text, p)
        m = len(p)
        for shards in (2, 5):
            S = -(-text.size // shards)
            offs, cmp_total = [], 0
            for g in range(shards):
                lo, hi = g * S, min((g + 1) * S, text.size)
                rd = min(hi + m - 1, text.size)
                d = torch_cuda.from_numpy(text[lo:rd].copy()).cuda()
                out = torch_cuda.empty(1 << 16, dtype=torch_cuda.int64, device="cuda")
                n, c = ctx.kmp_search_device(p, d.data_ptr(), rd - lo, out.data_ptr(), 1 << 16, own=hi - lo, base=lo)
                ctx.synchronize()
                offs.append(out[:n].cpu().numpy())
                cmp_total += c
            assert np.array_equal(np.concatenate(offs), r_offs), (p, shards)
            assert cmp_total == r_cmp, (p, shards)


@pytest.mark.parametrize("layout", ["auto", "bits", "bits+bloom2"])
def test_prefix8_small_and_ragged(ctx, torch_cuda, layout, monkeypatch):
    """PREFIX8 on the edge cases the big inputs do not reach: texts of 0..5000
    bytes (< 8, one tile, a tile + a few bytes), unaligned starts, shards
    with tiny owned ranges, full-byte alphabets, prefixes colliding on their
    first 8 bytes, patterns longer than the prefix (the deeper trie walk)."""
    for k, v in P8_LAYOUTS[layout].items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(2024)
    for trial in range(120):
        alpha = 4 if trial % 3 == 0 else 256
        n = int(rng.choice([0, 1, 7, 8, 9, 100, 2047, 2048, 2049, 2063, 4096 + 5, int(rng.integers(0, 5000))]))
        text = (rng.integers(0, alpha, n) + (65 if alpha == 4 else 0)).astype(np.uint8)
        k = int(rng.integers(1, 24))
        pats = []
        for _ in range(k):
            ln = int(rng.integers(8, 17))
            if n >= ln and rng.random() < 0.6:  # a window of the text: guaranteed hits
                o = int(rng.integers(0, n - ln + 1))
                pats.append(text[o:o + ln].tobytes())
            else:
                pats.append((rng.integers(0, alpha, ln) + (65 if alpha == 4 else 0)).astype(np.uint8).tobytes())
        pats = list(dict.fromkeys(pats))
        L = 8 if trial % 4 else 12
        trie = ctx.upload(glop.build_failureless_trie(pats, L))
        assert trie.info.min_depth >= 8
        ref = O.pfac_scan(text, O.Trie(pats, L)) if n else np.zeros(0, dtype=glop.HIT_DTYPE)
        off = int(rng.integers(0, 16))
        padded = np.concatenate([np.zeros(off, np.uint8), text])
        got = dev_scan(ctx, torch_cuda, trie, padded, glop.PFAC_PREFIX8, offset=off)
        assert got.tobytes() == ref.tobytes(), (trial, n, k, L, off)
        if n > 20:  # a shard: starts [lo, hi) of the text, reading an lmax-1 halo
            lo = int(rng.integers(0, n - 10))
            hi = int(rng.integers(lo + 1, n + 1))
            rd = min(hi + trie.info.max_depth - 1, n)
            part = dev_scan(ctx, torch_cuda, trie, text[lo:rd], glop.PFAC_PREFIX8, own=hi - lo, base=lo + (1 << 33))
            want = ref[(ref["offset"] >= lo) & (ref["offset"] < hi)].copy()
            want["offset"] += 1 << 33
            assert part.tobytes() == want.tobytes(), (trial, lo, hi)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_pipeline_shards_1_2_4_8(ctx, torch_cuda, world):
    """SURVEY §8e parity: the per-rank pipeline (glop_run_pfac_pipeline_shard
    on shards.plan_shards ranges with the halo bench.py uses) concatenated in
    rank order, counts summed, equals the single-GPU result -- for 1, 2, 4
    and 8 ranks (run here one after another on one GPU)."""
    from paper_1704_02278_b200.shards import plan_shards

    n = 24 << 20
    d = torch_cuda.empty(n + 64, dtype=torch_cuda.uint8, device="cuda")
    ctx.gen_syslog_device(d.data_ptr(), n, seed=99)
    ctx.synchronize()
    pats, _ = glop.gen_rules(1000, seed=606)
    pats += [b"Failed password for invalid user", b"pam_unix(sshd:session): session opened"]
    trie = ctx.upload(glop.build_failureless_trie(pats, 8))
    rules = ctx.upload_rules(pats, 8)
    whole = ctx.run_pfac_pipeline(trie, rules, d.data_ptr(), n, True)
    halo = max(trie.info.max_depth, max(len(p) for p in pats)) - 1
    alerts, counts, s1 = [], np.zeros(len(pats), np.uint64), 0
    for sh in plan_shards(n, world, halo):
        a, c, h = ctx.run_pfac_pipeline(trie, rules, d.data_ptr() + sh.lo, sh.read, True, own=sh.own, base=sh.lo)
        alerts.append(a)
        counts += c
        s1 += h
    assert np.concatenate(alerts).tobytes() == whole[0].tobytes()
    assert np.array_equal(counts, whole[1]) and s1 == whole[2]


@pytest.mark.parametrize("layout", list(P8_LAYOUTS))
def test_prefix8_hit_density_sweep(ctx, torch_cuda, layout, monkeypatch):
    """PREFIX8 over 4-letter texts where most 8-byte windows are patterns:
    hit densities from sparse to several per word, several ids per prefix,
    so the hit buffer's in-order batches, the out-of-order sort, the
    overflow replay and the staging-region growth all run -- each result
    bit-exact with the oracle."""
    for k, v in P8_LAYOUTS[layout].items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(77)
    for trial, (n, k) in enumerate([(1 << 20, 50), (1 << 20, 2000), (3 << 19, 20000)]):
        text = (rng.integers(0, 4, n) + 65).astype(np.uint8)
        starts = rng.integers(0, n - 16, k)
        pats = [text[s:s + int(rng.integers(8, 13))].tobytes() for s in starts]
        pats += [p[:8] + b"Z" for p in pats[:k // 4]]  # colliding 8-byte prefixes
        pats = list(dict.fromkeys(pats))
        trie = ctx.upload(glop.build_failureless_trie(pats, 8))
        ref = O.pfac_scan(text, O.Trie(pats, 8))
        got = dev_scan(ctx, torch_cuda, trie, text, glop.PFAC_PREFIX8)
        assert got.tobytes() == ref.tobytes(), (layout, trial, len(got), len(ref))


@pytest.mark.parametrize("seed", range(8))
def test_prefix8_byte_layout_carried_rounds(ctx, torch_cuda, seed):
    """Small rule sets (<= 64 grams: the byte layout, whose partial drain
    rounds are carried in registers from tile to tile): random texts with
    the patterns spliced at random places (every tile edge, the halo, the
    last bytes), random shards (own / base / misaligned start) == oracle."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 600_000))
    text = (rng.integers(0, 4, n) + 65).astype(np.uint8) if seed % 2 else glop.gen_syslog_host(n, seed)
    k = int(rng.integers(1, 15))
    pats = [bytes((rng.integers(0, 4, int(rng.integers(8, 13))) + 65).astype(np.uint8)) for _ in range(k)]
    for _ in range(int(rng.integers(0, 400))):  # occurrences, several per 2 KB tile
        p = pats[int(rng.integers(0, k))]
        at = int(rng.integers(0, max(1, n - len(p))))
        text[at:at + len(p)] = np.frombuffer(p, np.uint8)[: n - at]
    trie = ctx.upload(glop.build_failureless_trie(pats, 8))
    ref = O.pfac_scan(text, O.Trie(pats, 8))
    assert dev_scan(ctx, torch_cuda, trie, text, glop.PFAC_PREFIX8).tobytes() == ref.tobytes()
    off = int(rng.integers(0, 16))
    if n > off + 64:
        own = int(rng.integers(1, n - off))
        r = ref[(ref["offset"] >= off) & (ref["offset"] < off + own)].copy()
        r["offset"] -= off
        got = dev_scan(ctx, torch_cuda, trie, text, glop.PFAC_PREFIX8, own=own, offset=off)
        assert got.tobytes() == r.tobytes()
