"""Result digests for parity at bench scale.

A scan's observable result (SURVEY.md §8a parity semantics) is the sorted
hit list (offset, pattern_id, matched_len), the sorted alert list (offset,
rule_id, pattern_len) and the per-pattern alert counts.  Full-size results
(millions of records) are compared as SHA-256 digests of their packed
little-endian 16-byte records, so the bench's GPU arm and the reference arm
(bench.py --impl reference) can print the same `parity` block and the driver
can check them for equality.  Pure hashlib/numpy: no device, no oracle.
"""
from __future__ import annotations

import hashlib

import numpy as np

HIT_DTYPE = np.dtype([("offset", "<u8"), ("pattern_id", "<u4"), ("matched_len", "<u4")])
ALERT16_DTYPE = np.dtype([("offset", "<u8"), ("rule_id", "<u4"), ("pattern_len", "<u4")])


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def alerts16(alerts: np.ndarray) -> np.ndarray:
    """Any alert record array with offset/rule_id/pattern_len fields as the
    packed 16-byte glop_alert layout."""
    out = np.empty(len(alerts), dtype=ALERT16_DTYPE)
    for f in ALERT16_DTYPE.names:
        out[f] = alerts[f]
    return out


def digest(hits: np.ndarray | None, alerts: np.ndarray, n_patterns: int) -> dict:
    """{hits, hits_sha, alerts, alerts_sha, counts_sha, sha}: `sha` covers all
    three, i.e. the whole observable result of pfac_scan + verify_hits."""
    a = alerts16(alerts)
    counts = np.bincount(a["rule_id"].astype(np.int64), minlength=n_patterns).astype("<u8") if len(a) else \
        np.zeros(n_patterns, "<u8")
    d = {"alerts": int(len(a)), "alerts_sha": _sha(a), "counts_sha": _sha(counts)}
    if hits is not None:
        h = np.ascontiguousarray(hits).view(HIT_DTYPE) if hits.dtype != HIT_DTYPE else hits
        d["hits"] = int(len(h))
        d["hits_sha"] = _sha(h)
    d["sha"] = hashlib.sha256("|".join(d.get(k, "") for k in ("hits_sha", "alerts_sha", "counts_sha"))
                              .encode()).hexdigest()
    return d


def offsets_digest(offsets: np.ndarray, comparisons: int | None = None) -> dict:
    """KMP result: ascending u64 start offsets (+ the comparison count)."""
    o = np.ascontiguousarray(offsets, dtype="<u8")
    d = {"matches": int(len(o)), "offsets_sha": _sha(o)}
    if comparisons is not None:
        d["comparisons"] = int(comparisons)
    d["sha"] = hashlib.sha256(f"{d['offsets_sha']}|{d.get('comparisons', '')}".encode()).hexdigest()
    return d
