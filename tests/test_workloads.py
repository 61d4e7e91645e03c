"""Synthetic-input generators (bench / parity infrastructure, not the path):
the packet-payload stream for the DPI configuration (BASELINE.json
configs[4]) is block-parallel and range-consistent, and the Snort-style
content sets are distinct and within their length bounds."""
import numpy as np

from paper_1704_02278_b200 import glop


def test_payload_ranges_are_consistent():
    whole = glop.gen_payload_host(1 << 20, seed=9)
    assert len(np.unique(whole)) == 256  # full byte alphabet
    for begin, n in ((0, 1), (4095, 2), (12345, 70001), (1 << 19, 1 << 19)):
        part = glop.gen_payload_host(n, seed=9, begin=begin, threads=3)
        assert np.array_equal(part, whole[begin:begin + n])
    assert not np.array_equal(glop.gen_payload_host(4096, seed=10), whole[:4096])


def test_payload_has_protocol_text():
    p = glop.gen_payload_host(4 << 20, seed=1).tobytes()
    for tok in (b"HTTP/1.1", b"User-Agent: ", b"/etc/passwd", b"\x16\x03", b"<script>alert("):
        assert tok in p


def test_dpi_rules():
    r = glop.gen_dpi_rules(2000, seed=3, min_len=8, max_len=24)
    assert len(r) == len(set(r)) == 2000
    assert min(map(len, r)) >= 8 and max(map(len, r)) <= 24
    assert r == glop.gen_dpi_rules(2000, seed=3, min_len=8, max_len=24)
    sample = glop.gen_payload_host(4 << 20, seed=1).tobytes()
    windows = [x for i, x in enumerate(r) if 10 <= i % 20 < 19][:200]
    assert sum(x in sample for x in windows) > len(windows) // 2  # payload windows occur
    prefixes = {}
    for x in r:
        prefixes[x[:8]] = prefixes.get(x[:8], 0) + 1
    assert max(prefixes.values()) <= 3
