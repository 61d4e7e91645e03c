"""GPU parity of the fused device pipeline (glop_run_pfac_pipeline_device,
csrc/pipeline.cuh): scan -> ordered hits -> stage-2 verify -> alerts +
per-pattern counts with one host wait, against the oracle's pfac_scan +
verify_hits (scan.hpp:177-202, verify.hpp:69-105), and against the general
(unfused) path.  Also the pfac8 hit-buffer replay: a replayed lane starts
with an empty buffer, so only a lane that alone overflows it takes the
exact fallback.  Run on the B200: pytest -m gpu."""
import numpy as np
import pytest

import oracle_ffi as O
from paper_1704_02278_b200 import glop
from paper_1704_02278_b200.parity import alerts16

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return glop.Context(0)


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    assert torch.cuda.is_available(), "-m gpu tests need the B200"
    return torch


def fused(ctx, torch, pats, text: np.ndarray, L=8, own=None, base=0, alert_cap=None, with_hits=True):
    trie = ctx.upload(glop.build_failureless_trie(pats, L))
    rules = ctx.upload_rules(pats, L)
    n = text.size
    d = torch.from_numpy(np.concatenate([text, np.zeros(64, np.uint8)])).cuda()
    cap = max(1 << 16, 2 * n)
    d_hits = torch.empty(cap * 16, dtype=torch.uint8, device="cuda")
    acap = cap if alert_cap is None else alert_cap
    d_alerts = torch.empty(max(acap, 1) * 16, dtype=torch.uint8, device="cuda")
    d_counts = torch.full((len(pats),), 7, dtype=torch.int64, device="cuda")  # overwritten, not accumulated
    nh, na = ctx.run_pfac_pipeline_device(trie, rules, d.data_ptr(), n, d_alerts.data_ptr(), acap,
                                          d_counts.data_ptr(), own=own, base=base,
                                          d_hits=d_hits.data_ptr() if with_hits else None,
                                          hit_cap=cap if with_hits else 0)
    ctx.synchronize()
    hits = d_hits[: nh * 16].cpu().numpy().view(glop.HIT_DTYPE).copy() if with_hits else None
    alerts = d_alerts[: na * 16].cpu().numpy().view(glop.ALERT_DTYPE).copy()
    return hits, alerts, d_counts.cpu().numpy().astype(np.uint64)


def oracle(pats, text, L=8, own=None, base=0):
    hits = O.pfac_scan(text, O.Trie(pats, L))
    alerts = O.verify_hits(text, hits, pats, L)
    if own is not None:
        hits, alerts = hits[hits["offset"] < own].copy(), alerts[alerts["offset"] < own].copy()
    hits["offset"] += base
    alerts["offset"] += base
    counts = np.bincount(alerts["rule_id"].astype(np.int64), minlength=len(pats)).astype(np.uint64)
    return hits, alerts, counts


def corpus_case(seed, k, extra=()):
    text = glop.gen_syslog_host(6 << 20, seed=seed)
    pats, _ = glop.gen_rules(k, seed=606)
    return list(pats) + list(extra), text


@pytest.mark.parametrize("unfused", [False, True])
@pytest.mark.parametrize("case", ["prefix8", "stage2", "dpi", "shard"])
def test_fused_pipeline_vs_oracle(ctx, torch_cuda, case, unfused, monkeypatch):
    if unfused:
        monkeypatch.setenv("GLOP_NO_FUSED", "1")
    own, base = None, 0
    if case == "prefix8":
        pats, text = corpus_case(5, 1000)
    elif case == "stage2":  # longer patterns sharing 8-byte prefixes: verify rejects some hits
        pats, text = corpus_case(6, 1000, [b"Failed password for invalid user", b"Failed password for root",
                                           b"session opened for user root by", b"session opened for user nobody"])
    elif case == "dpi":
        text = glop.gen_payload_host(6 << 20, seed=3)
        pats = glop.gen_dpi_rules(10000, 606, 8, 24)
    else:  # a shard: starts [0, own) of a text with a halo, global offsets past 2^32
        pats, text = corpus_case(8, 1000, [b"Failed password for invalid user"])
        own, base = text.size - 31, (5 << 30) + 3
    hits, alerts, counts = fused(ctx, torch_cuda, pats, text, own=own, base=base)
    r_hits, r_alerts, r_counts = oracle(pats, text, own=own, base=base)
    assert len(r_alerts) > 100
    assert hits.tobytes() == r_hits.tobytes()
    assert np.array_equal(alerts16(alerts), alerts16(r_alerts))
    assert np.array_equal(counts, r_counts)
    if case in ("stage2", "dpi"):
        assert len(r_alerts) < len(r_hits)


def test_fused_pipeline_without_hits_and_capacity(ctx, torch_cuda):
    pats, text = corpus_case(9, 1000, [b"Failed password for invalid user"])
    r_hits, r_alerts, r_counts = oracle(pats, text)
    _, alerts, counts = fused(ctx, torch_cuda, pats, text, with_hits=False)
    assert np.array_equal(alerts16(alerts), alerts16(r_alerts)) and np.array_equal(counts, r_counts)
    with pytest.raises(glop.CapacityError):
        fused(ctx, torch_cuda, pats, text, alert_cap=len(r_alerts) - 1)
    _, alerts, _ = fused(ctx, torch_cuda, pats, text, alert_cap=len(r_alerts))  # exactly enough
    assert np.array_equal(alerts16(alerts), alerts16(r_alerts))


def test_fused_pipeline_empty_and_tiny(ctx, torch_cuda):
    pats, _ = glop.gen_rules(10, seed=606)
    for text in (np.zeros(0, np.uint8), np.frombuffer(pats[3], np.uint8).copy(),
                 np.frombuffer(b"x" + pats[3] + pats[3][:7], np.uint8).copy()):
        hits, alerts, counts = fused(ctx, torch_cuda, pats, text)
        r_hits, r_alerts, r_counts = oracle(pats, text)
        assert hits.tobytes() == r_hits.tobytes()
        assert np.array_equal(alerts16(alerts), alerts16(r_alerts)) and np.array_equal(counts, r_counts)


def test_replay_lane_starts_with_empty_buffer(ctx, torch_cuda):
    """one drain round whose candidates emit 16 + 20 ids (> the
    32-key warp buffer) is replayed lane by lane; the second lane's 20 ids
    must not see the first lane's 16 still buffered -- exact, and no
    global-key fallback."""
    rng = np.random.default_rng(5)
    p1 = b"QWERTYUI"
    p2 = b"ZXCVBNM,"
    pats = [p1 + bytes([65 + j]) for j in range(16)] + [p2 + bytes([97 + j]) for j in range(20)]
    text = rng.integers(48, 58, 1 << 16).astype(np.uint8)  # digits only: no other candidates
    for t0 in range(0, text.size - 4096, 4096):
        text[t0 + 64:t0 + 73] = np.frombuffer(pats[3], np.uint8)
        text[t0 + 700:t0 + 709] = np.frombuffer(pats[30], np.uint8)
    before = ctx.fallbacks
    hits, alerts, counts = fused(ctx, torch_cuda, pats, text)
    r_hits, r_alerts, r_counts = oracle(pats, text)
    assert len(r_hits) == 36 * (text.size // 4096 - 1)
    assert hits.tobytes() == r_hits.tobytes()
    assert np.array_equal(alerts16(alerts), alerts16(r_alerts)) and np.array_equal(counts, r_counts)
    assert ctx.fallbacks == before, "a replayed lane took the global-key fallback"


@pytest.mark.parametrize("engine", ["pfac_compact", "pfac_dense", "ac_chunked"])
def test_dropin_engine_pageable_with_lines(engine):
    """The drop-in run_engine_scan (libglop_engine.so) on PAGEABLE host text
    past the 256 MiB streaming chunk (the staged copy path), with a LineIndex:
    alerts and their line numbers equal the reference's run over the same
    bytes (pipeline.hpp:49-100, verify.hpp:40-64)."""
    n = (256 << 20) + (40 << 20)
    text = glop.gen_syslog_host(n, 12)
    pats, _ = glop.gen_rules(1000, 606)
    pats = list(pats) + [b"Failed password for invalid user", b"session opened for user root by"]
    eng = glop.Engine(pats)
    alerts, lines, s1 = eng.run(text.ctypes.data, n, engine=engine, lines=True)
    if O.ref() is not None:
        r_hits, r_alerts = O.ref_pfac_verify(text, pats, 8, compact=True, workers=0, with_lines=True)
    else:
        r_hits, r_alerts = O.pfac_verify(text, pats, 8, with_lines=True)
    assert np.array_equal(alerts16(alerts), alerts16(r_alerts))
    assert np.array_equal(lines, r_alerts["line"])
    if engine != "ac_chunked":
        assert s1 == len(r_hits)
    else:
        assert s1 == len(r_alerts)  # ac_chunked matches full patterns: every hit is an alert


def test_async_pipeline_tickets(ctx, torch_cuda):
    """glop_run_pfac_pipeline_device_async: several submissions back to back,
    each ticket read after one synchronize equals the synchronous call; a
    hit-dense input that overflows a warp's buffer reports Again (its outputs
    are not valid) and the synchronous call then gives the exact result."""
    torch = torch_cuda
    pats, text = corpus_case(11, 1000, [b"Failed password for invalid user"])
    trie = ctx.upload(glop.build_failureless_trie(pats, 8))
    rules = ctx.upload_rules(pats, 8)
    d = torch.from_numpy(np.concatenate([text, np.zeros(64, np.uint8)])).cuda()
    cap = 1 << 20
    d_alerts = torch.empty(cap * 16, dtype=torch.uint8, device="cuda")
    d_counts = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    r_hits, r_alerts, r_counts = oracle(pats, text)
    tickets = ctx.host_alloc(glop.TICKET_BYTES * 4)
    try:
        for i in range(4):
            ctx.run_pfac_pipeline_device_async(trie, rules, d.data_ptr(), text.size, d_alerts.data_ptr(), cap,
                                               d_counts.data_ptr(), tickets + glop.TICKET_BYTES * i)
        ctx.synchronize()
        for i in range(4):
            assert glop.ticket_result(tickets + glop.TICKET_BYTES * i) == (len(r_hits), len(r_alerts))
        alerts = d_alerts[: len(r_alerts) * 16].cpu().numpy().view(glop.ALERT_DTYPE)
        assert np.array_equal(alerts16(alerts), alerts16(r_alerts))
        assert np.array_equal(d_counts.cpu().numpy().astype(np.uint64), r_counts)
        # hit-dense: every position of an 'A' run matches several patterns
        dense = np.full(1 << 16, 65, np.uint8)
        dpats = [b"AAAAAAAA" + bytes([66 + j]) for j in range(40)]
        dt = ctx.upload(glop.build_failureless_trie(dpats, 8))
        dr = ctx.upload_rules(dpats, 8)
        dd = torch.from_numpy(np.concatenate([dense, np.zeros(64, np.uint8)])).cuda()
        dcap = 1 << 23
        da = torch.empty(dcap * 16, dtype=torch.uint8, device="cuda")
        dc = torch.zeros(len(dpats), dtype=torch.int64, device="cuda")
        ctx.run_pfac_pipeline_device_async(dt, dr, dd.data_ptr(), dense.size, da.data_ptr(), dcap, dc.data_ptr(),
                                           tickets)
        ctx.synchronize()
        with pytest.raises(glop.Again):
            glop.ticket_result(tickets)
        nh, na = ctx.run_pfac_pipeline_device(dt, dr, dd.data_ptr(), dense.size, da.data_ptr(), dcap, dc.data_ptr())
        h, a, c = oracle(dpats, dense)
        assert (nh, na) == (len(h), len(a)) and nh > 0
    finally:
        ctx.host_free(tickets)


@pytest.mark.parametrize("chunk,overlap", [(0, 0), (1 << 16, None), (4096, 3), (997, 0), (64, 20), (1 << 20, 1)])
def test_chunked_ac_vs_reference(ctx, chunk, overlap):
    """glop_chunked_ac_scan against the reference's chunked_ac_scan
    (scan.hpp:207-243, oracle/_ref) on 8 MB of syslog with patterns of 3..24
    bytes: lossless overlaps (max_len - 1, None here) and lossy ones (the
    reference loses the matches its chunk cannot reach; so must we)."""
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(chunk + 7)
    text = glop.gen_syslog_host(8 << 20, seed=17)
    pats = list(dict.fromkeys(text[o:o + int(rng.integers(3, 25))].tobytes() for o in rng.integers(0, text.size - 32, 300)))
    max_len = max(len(p) for p in pats)
    ov = max_len - 1 if overlap is None else overlap
    ac = ctx.upload(glop.build_failureless_trie(pats, max_len))
    got = ctx.chunked_ac_scan(ac, text, chunk, ov)
    ref = O.ref_chunked_ac_scan(text, pats, chunk, ov)
    assert len(ref) > 1000
    assert np.array_equal(got["offset"], ref["offset"]) and np.array_equal(got["pattern_id"], ref["pattern_id"])


def test_async_kmp_tickets(ctx, torch_cuda):
    """glop_kmp_search_device_async: back-to-back submissions, each ticket equal
    to the synchronous call and the oracle; a match-dense input (every
    position of an 'A' run) reports Again and the synchronous call is exact."""
    torch = torch_cuda
    text = glop.gen_syslog_host(3 << 20, 5)
    pat = b"Failed password"
    d = torch.from_numpy(np.concatenate([text, np.zeros(64, np.uint8)])).cuda()
    cap = 1 << 20
    d_out = torch.empty(cap * 8, dtype=torch.uint8, device="cuda")
    r_offs, r_cmp = O.kmp_search(text, pat)
    tickets = ctx.host_alloc(glop.TICKET_BYTES * 3)
    try:
        for i in range(3):
            ctx.kmp_search_device_async(pat, d.data_ptr(), text.size, d_out.data_ptr(), cap,
                                        tickets + glop.TICKET_BYTES * i)
        ctx.synchronize()
        for i in range(3):
            assert glop.kmp_ticket_result(tickets + glop.TICKET_BYTES * i) == (len(r_offs), r_cmp)
        assert np.array_equal(d_out[: len(r_offs) * 8].cpu().numpy().view("<u8"), r_offs)
        dense = np.full(1 << 20, 65, np.uint8)
        dd = torch.from_numpy(np.concatenate([dense, np.zeros(64, np.uint8)])).cuda()
        ctx.kmp_search_device_async(b"AA", dd.data_ptr(), dense.size, d_out.data_ptr(), cap, tickets)
        ctx.synchronize()
        with pytest.raises(glop.Again):
            glop.kmp_ticket_result(tickets)
        nm, cmp_ = ctx.kmp_search_device(b"AA", dd.data_ptr(), dense.size, d_out.data_ptr(), cap)
        o, c = O.kmp_search(dense, b"AA")
        assert (nm, cmp_) == (len(o), c)
        assert np.array_equal(d_out[: nm * 8].cpu().numpy().view("<u8"), o)
    finally:
        ctx.host_free(tickets)
