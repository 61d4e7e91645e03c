"""Randomised cross-checks of every device entry point against the reference
(oracle/_ref where built, else the C restatement): random texts (4-letter,
syslog, full-byte), random rule sets (1..40-byte patterns, shared prefixes,
duplicate bytes under different ids), prefix lengths 4 / 8 / 16, through the
fused device pipeline (with and without the hit list, synchronous and
asynchronous), the streamed host pipeline, the windowed stream with random
pieces, the multi-context group, and chunked AC with random chunk / overlap.
Seeded; every trial bit-exact.  Run on the B200: pytest -m gpu."""
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


def trial_inputs(seed):
    rng = np.random.default_rng(seed)
    kind = seed % 3
    n = int(rng.integers(1, 3 << 20))
    if kind == 0:
        text = (rng.integers(0, 4, n) + 65).astype(np.uint8)
    elif kind == 1:
        text = glop.gen_syslog_host(n, seed)
    else:
        text = rng.integers(0, 256, n).astype(np.uint8)
    k = int(rng.integers(1, 300))
    pats = []
    for _ in range(k):
        m = int(rng.integers(1, 41))
        if rng.random() < 0.6 and n > 64:  # a window of the text: real matches
            at = int(rng.integers(0, max(1, n - m)))
            p = text[at:at + m].tobytes()
        else:
            p = bytes(rng.integers(0, 256 if kind == 2 else 128, m).astype(np.uint8))
        if p:
            pats.append(p)
    if pats and rng.random() < 0.5:  # shared prefixes and a duplicate under another id
        base = pats[0]
        pats += [base + bytes([c]) for c in b"xyz"] + [base]
    L = int(rng.choice([4, 8, 16]))
    return rng, text, pats, L


def reference(text, pats, L, lines=False):
    if O.ref() is not None:
        return O.ref_pfac_verify(text, pats, L, compact=True, workers=0, with_lines=lines)
    return O.pfac_verify(text, pats, L, with_lines=lines)


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_pipelines(ctx, torch_cuda, seed, monkeypatch):
    torch = torch_cuda
    rng, text, pats, L = trial_inputs(seed)
    r_hits, r_alerts = reference(text, pats, L, lines=True)
    r_counts = np.bincount(r_alerts["rule_id"].astype(np.int64), minlength=len(pats)).astype(np.uint64)
    trie = ctx.upload(glop.build_failureless_trie(pats, L))
    rules = ctx.upload_rules(pats, L)
    # fused device pipeline, with and without the hit list, sync and async
    d = torch.from_numpy(np.concatenate([text, np.zeros(64, np.uint8)])).cuda()
    cap = max(1 << 16, 2 * len(r_hits) + 16)
    d_hits = torch.empty(cap * 16, dtype=torch.uint8, device="cuda")
    d_alerts = torch.empty(cap * 16, dtype=torch.uint8, device="cuda")
    d_counts = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    for with_hits in (True, False):
        nh, na = ctx.run_pfac_pipeline_device(trie, rules, d.data_ptr(), text.size, d_alerts.data_ptr(), cap,
                                              d_counts.data_ptr(), d_hits=d_hits.data_ptr() if with_hits else None,
                                              hit_cap=cap if with_hits else 0)
        ctx.synchronize()
        assert (nh, na) == (len(r_hits), len(r_alerts)), (seed, with_hits)
        a = d_alerts[: na * 16].cpu().numpy().view(glop.ALERT_DTYPE)
        assert np.array_equal(alerts16(a), alerts16(r_alerts)), seed
        assert np.array_equal(d_counts.cpu().numpy().astype(np.uint64), r_counts)
        if with_hits:
            assert d_hits[: nh * 16].cpu().numpy().tobytes() == r_hits.tobytes()
    ticket = ctx.host_alloc(glop.TICKET_BYTES)
    try:
        ctx.run_pfac_pipeline_device_async(trie, rules, d.data_ptr(), text.size, d_alerts.data_ptr(), cap,
                                           d_counts.data_ptr(), ticket)
        ctx.synchronize()
        try:
            assert glop.ticket_result(ticket) == (len(r_hits), len(r_alerts))
        except glop.Again:  # hit-dense input: the synchronous call above is the answer
            pass
    finally:
        ctx.host_free(ticket)
    # host-text pipeline with lines, and the windowed stream in random pieces
    alerts, counts, s1 = ctx.run_pfac_pipeline(trie, rules, text.ctypes.data, text.size, False)
    assert s1 == len(r_hits) and np.array_equal(alerts16(alerts), alerts16(r_alerts))
    monkeypatch.setenv("GLOP_STREAM_WINDOW", str(int(rng.integers(64, 1 << 18))))
    st = glop.Stream(ctx, trie, rules, lines=True)
    lo = 0
    while lo < text.size:
        step = int(rng.integers(1, 1 << 17))
        st.feed(text[lo:lo + step])
        lo += step
    alerts, counts, s1, lines, line_count, nb = st.end()
    assert nb == text.size and s1 == len(r_hits)
    assert np.array_equal(alerts16(alerts), alerts16(r_alerts)) and np.array_equal(counts, r_counts)
    assert np.array_equal(lines, r_alerts["line"])
    # a group of random size on this device, small shards
    monkeypatch.setenv("GLOP_GROUP_MIN_SHARD", str(int(rng.integers(1, 1 << 16))))
    g = glop.Group([0] * int(rng.integers(1, 6)))
    alerts, counts, s1, lines, line_count = g.run_pfac_pipeline(g.upload(glop.build_failureless_trie(pats, L)),
                                                                g.upload_rules(pats, L), text, lines=True)
    assert s1 == len(r_hits) and np.array_equal(alerts16(alerts), alerts16(r_alerts))
    assert np.array_equal(lines, r_alerts["line"]) and np.array_equal(counts, r_counts)


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_chunked_ac_and_kmp(ctx, seed):
    rng, text, pats, L = trial_inputs(100 + seed)
    max_len = max(len(p) for p in pats)
    if O.ref() is not None:
        chunk = int(rng.integers(0, 1 << 15))
        overlap = int(rng.integers(0, 2 * max_len))
        ac = ctx.upload(glop.build_failureless_trie(pats, max_len))
        got = ctx.chunked_ac_scan(ac, text, chunk, overlap)
        ref = O.ref_chunked_ac_scan(text, pats, chunk, overlap)
        assert np.array_equal(got["offset"], ref["offset"]) and np.array_equal(got["pattern_id"], ref["pattern_id"])
    for p in pats[:3]:
        offs, cmp_ = ctx.kmp_search(p, text)
        r_offs, r_cmp = O.kmp_search(text, p)
        assert np.array_equal(offs, r_offs) and cmp_ == r_cmp
