"""GPU parity at the sizes the bench measures (BASELINE.json configs).

The parity tests in test_gpu_parity.py pin every semantic corner at small
sizes; these rerun the bench's own workloads at full size and compare the
complete result with the unmodified reference (oracle/_ref, all host threads;
the C restatement when _ref was never built):

* configs[2]: PFAC, 1,000 rules, 8e9 bytes of syslog in ONE launch -- device
  offsets pass 2^32 -- hits, alerts and per-pattern counts;
* configs[0]: PFAC, 10 rules, 256e6 bytes;
* configs[1]: KMP "Failed password" over 1e9 bytes, offsets and the exact
  comparison count;
* configs[4] per GPU: DPI, 10,000 contents (8..24 bytes, stage-2 verify) over
  a 4e9-byte payload shard;
* the host-text streamed pipeline at 868 MiB (crosses its 256 MiB chunks)
  with occurrences spliced across every chunk boundary.

Reference semantics: scan.hpp:177-202 (pfac_scan), verify.hpp:69-105
(verify_hits), kmp.hpp:41-69 (kmp_search).  Run on the B200: pytest -m gpu.
"""
import numpy as np
import pytest

import oracle_ffi as O
from paper_1704_02278_b200 import glop
from paper_1704_02278_b200.parity import alerts16, digest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return glop.Context(0)


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    assert torch.cuda.is_available(), "-m gpu tests need the B200"
    return torch


def reference_pfac(text: np.ndarray, pats, L=8):
    """(hits, alerts) of the unmodified reference, else the C restatement."""
    if O.ref() is not None:
        return O.ref_pfac_verify(text, pats, L, compact=True, workers=0)
    return O.pfac_verify(text, pats, L)


def device_pfac(ctx, torch, d_text, n, pats, L=8, base=0):
    trie = ctx.upload(glop.build_failureless_trie(pats, L))
    rules = ctx.upload_rules(pats, L)
    cap = max(1 << 20, n // 256)
    d_hits = torch.empty(cap * 16, dtype=torch.uint8, device="cuda")
    d_alerts = torch.empty(cap * 16, dtype=torch.uint8, device="cuda")
    d_counts = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    nh = ctx.pfac_scan_device(trie, d_text.data_ptr(), n, d_hits.data_ptr(), cap, base=base)
    na = ctx.verify_hits_device(rules, d_text.data_ptr(), n, d_hits.data_ptr(), nh, d_alerts.data_ptr(),
                                d_counts.data_ptr(), base=base)
    ctx.synchronize()
    hits = d_hits[: nh * 16].cpu().numpy().view(glop.HIT_DTYPE).copy()
    alerts = d_alerts[: na * 16].cpu().numpy().view(glop.ALERT_DTYPE).copy()
    counts = d_counts.cpu().numpy().astype(np.uint64)
    del d_hits, d_alerts, d_counts
    return hits, alerts, counts


def check_same(hits, alerts, counts, ref_hits, ref_alerts, k):
    assert len(hits) == len(ref_hits), (len(hits), len(ref_hits))
    assert np.array_equal(hits, ref_hits)
    assert len(alerts) == len(ref_alerts), (len(alerts), len(ref_alerts))
    assert np.array_equal(alerts16(alerts), alerts16(ref_alerts))
    ref_counts = np.bincount(ref_alerts["rule_id"].astype(np.int64), minlength=k).astype(np.uint64)
    assert np.array_equal(counts, ref_counts)
    assert digest(hits, alerts, k)["sha"] == digest(ref_hits, ref_alerts, k)["sha"]


def _free(torch):
    import gc

    gc.collect()
    torch.cuda.empty_cache()


def test_pfac_8gb_k1000_one_launch(ctx, torch_cuda):
    """configs[2] exactly as bench.py runs it: 8e9 bytes, gen_rules(1000, 606),
    corpus seed 1, one scan launch whose offsets pass 2^32."""
    torch = torch_cuda
    S = 8_000_000_000
    pats, _ = glop.gen_rules(1000, 606)
    d_text = torch.empty(S + 64, dtype=torch.uint8, device="cuda")
    ctx.gen_syslog_device(d_text.data_ptr(), S, 1)
    hits, alerts, counts = device_pfac(ctx, torch, d_text, S, pats)
    host = d_text[:S].cpu().numpy()
    del d_text
    _free(torch)
    assert int(hits["offset"].max()) > 1 << 32 and len(hits) > 1_000_000
    ref_hits, ref_alerts = reference_pfac(host, pats)
    check_same(hits, alerts, counts, ref_hits, ref_alerts, len(pats))


def test_pfac_256mb_k10(ctx, torch_cuda):
    """configs[0]: 10 rules over 256e6 bytes."""
    torch = torch_cuda
    S = 256_000_000
    pats, _ = glop.gen_rules(10, 606)
    d_text = torch.empty(S + 64, dtype=torch.uint8, device="cuda")
    ctx.gen_syslog_device(d_text.data_ptr(), S, 1)
    hits, alerts, counts = device_pfac(ctx, torch, d_text, S, pats)
    host = d_text[:S].cpu().numpy()
    del d_text
    assert len(alerts) > 0
    ref_hits, ref_alerts = reference_pfac(host, pats)
    check_same(hits, alerts, counts, ref_hits, ref_alerts, len(pats))


def test_kmp_1gb(ctx, torch_cuda):
    """configs[1]: 'Failed password' over 1e9 bytes -- offsets and the exact
    number of byte comparisons of the sequential scan (kmp.hpp:41-69)."""
    torch = torch_cuda
    S = 1_000_000_000
    p = b"Failed password"
    d_text = torch.empty(S + 64, dtype=torch.uint8, device="cuda")
    ctx.gen_syslog_device(d_text.data_ptr(), S, 1)
    cap = 1 << 24
    d_out = torch.empty(cap * 8, dtype=torch.uint8, device="cuda")
    nm, cmp_ = ctx.kmp_search_device(p, d_text.data_ptr(), S, d_out.data_ptr(), cap)
    ctx.synchronize()
    offs = d_out[: nm * 8].cpu().numpy().view(np.uint64).copy()
    host = d_text[:S].cpu().numpy()
    del d_text, d_out
    assert nm > 1000
    if O.ref() is not None:
        import ctypes as C

        r = O.ref()
        op, no, rc = C.c_void_p(), C.c_uint64(), C.c_uint64()
        pa = np.frombuffer(p, np.uint8).copy()
        r.ref_kmp_search(host.ctypes.data_as(O.u8p), S, pa.ctypes.data_as(O.u8p), len(p), C.byref(op), C.byref(no),
                         C.byref(rc))
        ref_offs = O._take(op, no.value, np.uint64, r.ref_free)
        ref_cmp = rc.value
    else:
        ref_offs, ref_cmp = O.kmp_search(host, p)
    assert np.array_equal(offs, ref_offs)
    assert cmp_ == ref_cmp


def test_dpi_4gb_shard(ctx, torch_cuda):
    """configs[4] per GPU: 10,000 Snort-style contents (8..24 bytes, so
    stage-2 verification rejects some hits) over 4e9 payload bytes."""
    torch = torch_cuda
    S = 4_000_000_000
    pats = glop.gen_dpi_rules(10000, 606, 8, 24)
    d_text = torch.empty(S + 64, dtype=torch.uint8, device="cuda")
    ctx.gen_payload_device(d_text.data_ptr(), S, 1)
    hits, alerts, counts = device_pfac(ctx, torch, d_text, S, pats)
    host = d_text[:S].cpu().numpy()
    del d_text
    _free(torch)
    assert len(alerts) < len(hits), "stage 2 must reject some hits"
    ref_hits, ref_alerts = reference_pfac(host, pats)
    check_same(hits, alerts, counts, ref_hits, ref_alerts, len(pats))


def test_streamed_pipeline_868mb_vs_reference(ctx):
    """The host-text pipeline (glop_run_pfac_pipeline, 256 MiB chunks on a
    copy stream) at 868 MiB against the reference, with pattern occurrences
    spliced across every chunk boundary (a match that starts in chunk i and
    ends in chunk i+1 must be found exactly once)."""
    chunk = 256 << 20
    n = 3 * chunk + (100 << 20)
    pats, _ = glop.gen_rules(1000, 606)
    long_pats = pats[:990] + [b"BOUNDARY-straddling-" + bytes([65 + i]) * 9 for i in range(10)]
    text = glop.gen_syslog_host(n, 7)
    # boundary 1: a 29-byte pattern 12 bytes before it (stage 2 reads the halo);
    # boundary 2: an 8-byte rule 4 bytes before it; boundary 3: a 29-byte
    # pattern starting on the chunk's last byte
    for at, p in ((chunk - 12, long_pats[990]), (2 * chunk - 4, pats[5]), (3 * chunk - 1, long_pats[993])):
        text[at:at + len(p)] = np.frombuffer(p, np.uint8)
    trie = ctx.upload(glop.build_failureless_trie(long_pats, 8))
    rules = ctx.upload_rules(long_pats, 8)
    alerts, counts, s1 = ctx.run_pfac_pipeline(trie, rules, text.ctypes.data, n, False)
    ref_hits, ref_alerts = reference_pfac(text, long_pats)
    assert s1 == len(ref_hits)
    assert np.array_equal(alerts16(alerts), alerts16(ref_alerts))
    assert np.array_equal(counts, np.bincount(ref_alerts["rule_id"].astype(np.int64),
                                              minlength=len(long_pats)).astype(np.uint64))
    for at in (chunk - 12, 2 * chunk - 4, 3 * chunk - 1):
        assert at in set(int(o) for o in alerts["offset"])


def test_streamed_pipeline_long_pattern_after_short(ctx):
    """The same context's pageable-text pipeline first with a short halo,
    then with a 20,000-byte pattern straddling the 256 MiB chunk boundary:
    the pinned staging ring must grow with the halo (max pattern length - 1)."""
    chunk = 256 << 20
    n = chunk + (1 << 20)
    text = glop.gen_syslog_host(n, 11)
    short, _ = glop.gen_rules(100, 606)
    at = chunk - 10_000
    long_pat = text[at:at + 20_000].tobytes()
    for pats in (short, short + [long_pat]):
        trie = ctx.upload(glop.build_failureless_trie(pats, 8))
        rules = ctx.upload_rules(pats, 8)
        alerts, counts, s1 = ctx.run_pfac_pipeline(trie, rules, text.ctypes.data, n, False)
        ref_hits, ref_alerts = reference_pfac(text, pats)
        assert s1 == len(ref_hits)
        assert np.array_equal(alerts16(alerts), alerts16(ref_alerts))
    assert (at, len(pats) - 1) in set(zip(alerts["offset"].tolist(), alerts["rule_id"].tolist()))
