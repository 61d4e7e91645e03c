"""Golden fixtures (tests/golden/*.bin.gz) and the seeded trial regenerators.

The fixtures are written by oracle/gen_golden.cpp, i.e. by the unmodified
reference replaying its own seeded tests.  Randomized families store only
digests; their inputs are regenerated here with the same std::mt19937 call
sequence (numpy's MT19937 with legacy seeding is bit-identical to
std::mt19937), and each record carries sha256(inputs) so a drifting
regenerator is caught, not silently compared.
"""
from __future__ import annotations

import gzip
import hashlib
import os
import struct
from dataclasses import dataclass, field

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

HIT_DTYPE = np.dtype([("offset", "<u8"), ("pattern_id", "<u4"), ("matched_len", "<u4")])
# packed alert layout used by the fixture digests
ALERT_DTYPE = np.dtype([("offset", "<u8"), ("line", "<u8"), ("rule_id", "<u4"), ("pattern_len", "<u4")])


class MT19937:
    """std::mt19937 call-by-call (buffered raw outputs)."""

    def __init__(self, seed: int):
        self._bg = np.random.MT19937()
        self._bg._legacy_seeding(seed)
        self._buf: list[int] = []
        self._i = 0

    def __call__(self) -> int:
        if self._i >= len(self._buf):
            self._buf = self._bg.random_raw(4096).tolist()
            self._i = 0
        v = self._buf[self._i]
        self._i += 1
        return v


@dataclass
class PfacCase:
    L: int
    patterns: list
    text: bytes
    hits: np.ndarray | None = None       # HIT_DTYPE
    alerts: np.ndarray | None = None     # ALERT_DTYPE
    n_hits: int = 0
    n_alerts: int = 0
    hits_sha: str = ""
    alerts_sha: str = ""
    inputs_sha: str = ""
    workers: int = 1


@dataclass
class KmpCase:
    pattern: bytes
    text: bytes
    offsets: np.ndarray | None = None
    table: list = field(default_factory=list)
    n_offsets: int = 0
    offsets_sha: str = ""
    inputs_sha: str = ""
    comparisons: int = 0


@dataclass
class Summary:
    name: str
    text_sha: str
    n: int
    L: int
    patterns: list
    n_hits: int
    n_alerts: int
    alerts: np.ndarray | None


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def pack_inputs(patterns, text: bytes) -> bytes:
    out = bytearray()
    for p in patterns:
        out += struct.pack("<I", len(p)) + p
    out += struct.pack("<Q", len(text)) + text
    return bytes(out)


def pack_kmp_inputs(p: bytes, text: bytes) -> bytes:
    return struct.pack("<I", len(p)) + p + struct.pack("<Q", len(text)) + text


class _Reader:
    def __init__(self, raw: bytes):
        self.b = raw
        self.i = 8
        assert raw[:8] == b"GLOPGLD1"

    def u32(self):
        v = struct.unpack_from("<I", self.b, self.i)[0]
        self.i += 4
        return v

    def u64(self):
        v = struct.unpack_from("<Q", self.b, self.i)[0]
        self.i += 8
        return v

    def raw(self, n):
        v = self.b[self.i:self.i + n]
        self.i += n
        return bytes(v)

    def arr(self, dtype, n):
        a = np.frombuffer(self.b, dtype=dtype, count=n, offset=self.i).copy()
        self.i += n * np.dtype(dtype).itemsize
        return a

    def done(self):
        return self.i >= len(self.b)


def load(name: str) -> list:
    with gzip.open(os.path.join(GOLDEN, name + ".bin.gz"), "rb") as f:
        r = _Reader(f.read())
    out = []
    while not r.done():
        tag = r.u32()
        if tag == 1:
            L = r.u64()
            pats = [r.raw(r.u32()) for _ in range(r.u32())]
            text = r.raw(r.u64())
            hits = r.arr(HIT_DTYPE, r.u64())
            alerts = r.arr(ALERT_DTYPE, r.u64())
            out.append(PfacCase(L, pats, text, hits, alerts, len(hits), len(alerts)))
        elif tag == 4:
            L = r.u64()
            c = PfacCase(L, [], b"")
            c.inputs_sha = r.raw(64).decode()
            c.n_hits = r.u64()
            c.hits_sha = r.raw(64).decode()
            c.n_alerts = r.u64()
            c.alerts_sha = r.raw(64).decode()
            out.append(c)
        elif tag == 2:
            m = r.u32()
            p = r.raw(m)
            text = r.raw(r.u64())
            table = list(r.arr("<u4", m))
            offs = r.arr("<u8", r.u64())
            cmp_ = r.u64()
            out.append(KmpCase(p, text, offs, table, len(offs), comparisons=cmp_))
        elif tag == 5:
            k = KmpCase(b"", b"")
            k.inputs_sha = r.raw(64).decode()
            k.n_offsets = r.u64()
            k.offsets_sha = r.raw(64).decode()
            k.comparisons = r.u64()
            out.append(k)
        elif tag == 3:
            name_ = r.raw(r.u32()).decode()
            tsha = r.raw(64).decode()
            n = r.u64()
            L = r.u64()
            pats = [r.raw(r.u32()) for _ in range(r.u32())]
            n_hits = r.u64()
            n_keep = r.u64()
            n_alerts = r.u64()
            alerts = r.arr(ALERT_DTYPE, n_keep)
            out.append(Summary(name_, tsha, n, L, pats, n_hits, n_alerts, alerts))
        else:
            raise ValueError(f"bad tag {tag}")
    return out


# --------------------------------------------------------------------------
# Seeded regenerators: Python restatements of the reference tests' input
# loops, call-for-call.
# --------------------------------------------------------------------------
def _rand_patterns(rng, max_count, max_len, full_byte, skip_dup_continue=True):
    used, pats = set(), []
    count = 1 + rng() % max_count
    while len(pats) < count:
        ln = 1 + rng() % max_len
        b = bytes((rng() & 0xFF) if full_byte else (65 + rng() % 4) for _ in range(ln))
        if b in used:
            continue
        used.add(b)
        pats.append(b)
    return pats


def _rand_text(rng, max_len, full_byte):
    n = rng() % max_len
    return bytes((rng() & 0xFF) if full_byte else (65 + rng() % 4) for _ in range(n))


def acceptance_exactness_inputs():
    """acceptance.cpp:42-78 (seed 2024, 1000 trials)."""
    rng = MT19937(2024)
    for trial in range(1000):
        fb = trial % 2 == 1
        pats = _rand_patterns(rng, 32, 16, fb)
        text = _rand_text(rng, 4096, fb)
        L = 4 if trial % 3 == 0 else (8 if trial % 3 == 1 else 4096)
        workers = 1 + rng() % 4
        yield pats, text, L, workers


def scan_superset_inputs():
    """test_scan.cpp:157-176 (seed 29, 100 trials)."""
    rng = MT19937(29)
    for trial in range(100):
        fb = trial % 2 == 1
        pats = _rand_patterns(rng, 16, 16, fb)
        L = 4 if trial % 3 == 0 else (8 if trial % 3 == 1 else 64)
        text = _rand_text(rng, 4096, fb)
        workers = 1 + rng() % 4
        yield pats, text, L, workers


def kmp_naive_inputs():
    """test_kmp.cpp:76-93 (seed 9, 500 trials)."""
    rng = MT19937(9)
    for trial in range(500):
        n = rng() % 4096
        m = 1 + rng() % 32
        alpha = 2 if trial % 2 else 4
        text = bytes(65 + rng() % alpha for _ in range(n))
        p = bytes(65 + rng() % alpha for _ in range(m))
        yield p, text


def kmp_bound_inputs(count=2000):
    """acceptance.cpp:209-229 (seed 1414)."""
    rng = MT19937(1414)
    for _ in range(count):
        n = rng() % 1024
        m = 1 + rng() % 32
        alpha = 1 + rng() % 4
        text = bytes(65 + rng() % alpha for _ in range(n))
        p = bytes(65 + rng() % alpha for _ in range(m))
        yield p, text


def pack_hits(h: np.ndarray) -> bytes:
    return np.ascontiguousarray(h, dtype=HIT_DTYPE).tobytes()


def pack_alerts(a: np.ndarray) -> bytes:
    return np.ascontiguousarray(a, dtype=ALERT_DTYPE).tobytes()
