"""ctypes bindings to the CPU oracle (oracle/liboracle.so) and, when built,
the unmodified reference (oracle/_ref/libref_logtrawl.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg.  Never by the product path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from golden_io import ALERT_DTYPE, HIT_DTYPE

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libref_logtrawl.so")

_ORACLE_ALERT = np.dtype([("offset", "<u8"), ("rule_id", "<u4"), ("pattern_len", "<u4"), ("line", "<u8")])

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


class OracleError(Exception):
    def __init__(self, code: int):
        super().__init__({1: "invalid_argument", 2: "capacity", 3: "logic_error"}.get(code, str(code)))
        self.code = code


def _load(path):
    if not os.path.exists(path):
        return None
    return C.CDLL(path)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load(ORACLE_SO)
        if _lib is None:
            raise RuntimeError(f"{ORACLE_SO} not built (make -C oracle)")
        vp = C.c_void_p
        _lib.or_build_trie.argtypes = [u8p, u64p, C.c_uint32, C.c_uint64, C.c_uint64, C.POINTER(vp)]
        _lib.or_pfac_scan.argtypes = [u8p, C.c_uint64, vp, C.POINTER(vp), u64p]
        _lib.or_naive_scan.argtypes = [u8p, C.c_uint64, u8p, u64p, C.c_uint32, C.POINTER(vp), u64p]
        _lib.or_verify_hits.argtypes = [u8p, C.c_uint64, vp, C.c_uint64, u8p, u64p, C.c_uint32,
                                        C.c_uint64, C.c_int, C.POINTER(vp), u64p]
        _lib.or_kmp_failure.argtypes = [u8p, C.c_uint32, u32p]
        _lib.or_kmp_search.argtypes = [u8p, C.c_uint64, u8p, C.c_uint32, u32p, C.POINTER(vp), u64p, u64p]
        _lib.or_free.argtypes = [vp]
        _lib.or_trie_free.argtypes = [vp]
        for f in ("or_trie_table", "or_trie_out_offsets", "or_trie_out_flat", "or_trie_depth"):
            getattr(_lib, f).argtypes = [vp]
            getattr(_lib, f).restype = vp
        _lib.or_trie_state_count.argtypes = [vp]
        _lib.or_trie_state_count.restype = C.c_uint32
        _lib.or_line_of.argtypes = [u8p, C.c_uint64, C.c_uint64]
        _lib.or_line_of.restype = C.c_uint64
    return _lib


def ref():
    """The unmodified reference (None where it was never built)."""
    global _ref
    if _ref is None:
        _ref = _load(REF_SO)
        if _ref is not None:
            vp = C.c_void_p
            _ref.ref_pfac_scan_verify.argtypes = [u8p, C.c_uint64, u8p, u64p, C.c_uint32, C.c_uint64, C.c_int,
                                                  C.c_uint, C.c_int, C.POINTER(vp), u64p, C.POINTER(vp), u64p]
            _ref.ref_measure.argtypes = [u8p, C.c_uint64, u8p, u64p, C.c_uint32, C.c_uint64, C.c_int, C.c_uint,
                                         C.c_uint64, C.POINTER(C.c_double), C.POINTER(C.c_double)]
            _ref.ref_kmp_search.argtypes = [u8p, C.c_uint64, u8p, C.c_uint32, C.POINTER(vp), u64p, u64p]
            _ref.ref_free.argtypes = [vp]
            _ref.ref_time_pfac.argtypes = [u8p, C.c_uint64, u8p, u64p, C.c_uint32, C.c_uint64, C.c_int, C.c_uint,
                                           C.c_uint32, C.c_uint32, C.POINTER(C.c_double), u64p]
            _ref.ref_time_kmp.argtypes = [u8p, C.c_uint64, u8p, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.POINTER(C.c_double), u64p]
            _ref.ref_default_workers.restype = C.c_uint
    return _ref


def _buf(b) -> "u8p":
    if isinstance(b, np.ndarray):
        return b.ctypes.data_as(u8p)
    return C.cast(C.c_char_p(bytes(b)), u8p) if len(b) else C.cast(C.create_string_buffer(1), u8p)


class _Keep:
    """Holds the bytes objects whose pointers are handed to C."""

    def __init__(self, *objs):
        self.objs = objs


def pack_patterns(patterns):
    blob = b"".join(patterns)
    off = np.zeros(len(patterns) + 1, dtype=np.uint64)
    np.cumsum([len(p) for p in patterns], out=off[1:]) if patterns else None
    arr = np.frombuffer(blob, dtype=np.uint8).copy() if blob else np.zeros(1, np.uint8)
    return arr, off


def _text_arr(text):
    if isinstance(text, np.ndarray):
        return text if len(text) else np.zeros(1, np.uint8), len(text)
    return (np.frombuffer(text, dtype=np.uint8).copy() if len(text) else np.zeros(1, np.uint8)), len(text)


def _take(ptr, n, dtype, free):
    if n == 0:
        free(ptr)
        return np.zeros(0, dtype=dtype)
    a = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), shape=(n * np.dtype(dtype).itemsize,))
    out = a.view(dtype).copy()
    free(ptr)
    return out


class Trie:
    def __init__(self, patterns, L, max_states=1 << 22):
        pat, off = pack_patterns(patterns)
        h = C.c_void_p()
        rc = lib().or_build_trie(pat.ctypes.data_as(u8p), off.ctypes.data_as(u64p), len(patterns), L,
                                 max_states, C.byref(h))
        if rc:
            raise OracleError(rc)
        self.h = h
        q = lib().or_trie_state_count(h)
        self.state_count = q
        self.table = np.ctypeslib.as_array(C.cast(lib().or_trie_table(h), C.POINTER(C.c_int32)),
                                           shape=(q * 256,)).reshape(q, 256).copy()
        self.out_offsets = np.ctypeslib.as_array(C.cast(lib().or_trie_out_offsets(h), u32p),
                                                 shape=(q + 1,)).copy()
        no = int(self.out_offsets[-1])
        flat = np.ctypeslib.as_array(C.cast(lib().or_trie_out_flat(h), u32p), shape=(max(2 * no, 1),)).copy()
        self.out_flat = flat[:2 * no].reshape(no, 2)
        self.depth = np.ctypeslib.as_array(C.cast(lib().or_trie_depth(h), u32p), shape=(q,)).copy()

    def __del__(self):
        try:
            lib().or_trie_free(self.h)
        except Exception:
            pass


def pfac_scan(text, trie: Trie) -> np.ndarray:
    t, n = _text_arr(text)
    p, nh = C.c_void_p(), C.c_uint64()
    rc = lib().or_pfac_scan(t.ctypes.data_as(u8p), n, trie.h, C.byref(p), C.byref(nh))
    if rc:
        raise OracleError(rc)
    return _take(p, nh.value, HIT_DTYPE, lib().or_free)


def naive_scan(text, patterns) -> np.ndarray:
    t, n = _text_arr(text)
    pat, off = pack_patterns(patterns)
    p, nh = C.c_void_p(), C.c_uint64()
    lib().or_naive_scan(t.ctypes.data_as(u8p), n, pat.ctypes.data_as(u8p), off.ctypes.data_as(u64p),
                        len(patterns), C.byref(p), C.byref(nh))
    return _take(p, nh.value, HIT_DTYPE, lib().or_free)


def verify_hits(text, hits: np.ndarray, patterns, L, with_lines=False) -> np.ndarray:
    """Alerts as ALERT_DTYPE (offset, line, rule_id, pattern_len)."""
    t, n = _text_arr(text)
    pat, off = pack_patterns(patterns)
    h = np.ascontiguousarray(hits, dtype=HIT_DTYPE)
    if len(h) == 0:
        h = np.zeros(1, dtype=HIT_DTYPE)
    p, na = C.c_void_p(), C.c_uint64()
    rc = lib().or_verify_hits(t.ctypes.data_as(u8p), n, h.ctypes.data_as(C.c_void_p), len(hits),
                              pat.ctypes.data_as(u8p), off.ctypes.data_as(u64p), len(patterns), L,
                              1 if with_lines else 0, C.byref(p), C.byref(na))
    if rc:
        raise OracleError(rc)
    a = _take(p, na.value, _ORACLE_ALERT, lib().or_free)
    out = np.zeros(len(a), dtype=ALERT_DTYPE)
    for f in ("offset", "line", "rule_id", "pattern_len"):
        out[f] = a[f]
    return out


def kmp_failure(p: bytes) -> np.ndarray:
    t = np.zeros(max(len(p), 1), dtype=np.uint32)
    pa = np.frombuffer(p, dtype=np.uint8).copy() if p else np.zeros(1, np.uint8)
    lib().or_kmp_failure(pa.ctypes.data_as(u8p), len(p), t.ctypes.data_as(u32p))
    return t[:len(p)]


def kmp_search(text, p: bytes):
    """(offsets, comparisons)"""
    t, n = _text_arr(text)
    pa = np.frombuffer(p, dtype=np.uint8).copy() if p else np.zeros(1, np.uint8)
    tab = kmp_failure(p)
    tab_ = tab if len(tab) else np.zeros(1, np.uint32)
    o, no, cmp_ = C.c_void_p(), C.c_uint64(), C.c_uint64(0)
    lib().or_kmp_search(t.ctypes.data_as(u8p), n, pa.ctypes.data_as(u8p), len(p), tab_.ctypes.data_as(u32p),
                        C.byref(o), C.byref(no), C.byref(cmp_))
    return _take(o, no.value, np.uint64, lib().or_free), cmp_.value


def line_of(text, offset):
    t, n = _text_arr(text)
    return lib().or_line_of(t.ctypes.data_as(u8p), n, offset)


def pfac_verify(text, patterns, L, with_lines=False):
    trie = Trie(patterns, L)
    hits = pfac_scan(text, trie)
    return hits, verify_hits(text, hits, patterns, L, with_lines)


# ------------------------------------------------------------------ reference
def ref_pfac_verify(text, patterns, L, compact=True, workers=1, with_lines=False):
    r = ref()
    if r is None:
        raise RuntimeError("reference shim not built")
    t, n = _text_arr(text)
    pat, off = pack_patterns(patterns)
    hp, nh, ap, na = C.c_void_p(), C.c_uint64(), C.c_void_p(), C.c_uint64()
    rc = r.ref_pfac_scan_verify(t.ctypes.data_as(u8p), n, pat.ctypes.data_as(u8p), off.ctypes.data_as(u64p),
                                len(patterns), L, 1 if compact else 0, workers, 1 if with_lines else 0,
                                C.byref(hp), C.byref(nh), C.byref(ap), C.byref(na))
    if rc:
        raise OracleError(rc)
    hits = _take(hp, nh.value, HIT_DTYPE, r.ref_free)
    a = _take(ap, na.value, _ORACLE_ALERT, r.ref_free)
    out = np.zeros(len(a), dtype=ALERT_DTYPE)
    for f in ("offset", "line", "rule_id", "pattern_len"):
        out[f] = a[f]
    return hits, out


def ref_measure(text, patterns, L, engine=2, workers=0, runs=3):
    """The reference's measure() (bench.hpp:64-113): (mean_seconds, bps)."""
    r = ref()
    t, n = _text_arr(text)
    pat, off = pack_patterns(patterns)
    ms, bps = C.c_double(), C.c_double()
    rc = r.ref_measure(t.ctypes.data_as(u8p), n, pat.ctypes.data_as(u8p), off.ctypes.data_as(u64p),
                       len(patterns), L, engine, workers, runs, C.byref(ms), C.byref(bps))
    if rc:
        raise OracleError(rc)
    return ms.value, bps.value


def ref_time_pfac(text, patterns, L, warmup=1, runs=3, workers=0, compact=True):
    """Reference pfac_scan + verify_hits timed per run (the body of
    bench.hpp:103-109).  Returns (run_seconds list, n_alerts)."""
    r = ref()
    t, n = _text_arr(text)
    pat, off = pack_patterns(patterns)
    secs = (C.c_double * max(runs, 1))()
    na = C.c_uint64()
    rc = r.ref_time_pfac(t.ctypes.data_as(u8p), n, pat.ctypes.data_as(u8p), off.ctypes.data_as(u64p),
                         len(patterns), L, 1 if compact else 0, workers, warmup, runs, secs, C.byref(na))
    if rc:
        raise OracleError(rc)
    return list(secs)[:runs], na.value


def ref_time_kmp(text, p: bytes, warmup=1, runs=3):
    r = ref()
    t, n = _text_arr(text)
    pa = np.frombuffer(p, dtype=np.uint8).copy()
    secs = (C.c_double * max(runs, 1))()
    nm = C.c_uint64()
    r.ref_time_kmp(t.ctypes.data_as(u8p), n, pa.ctypes.data_as(u8p), len(p), warmup, runs, secs, C.byref(nm))
    return list(secs)[:runs], nm.value


def port_time_pfac(text, patterns, L, warmup=1, runs=3):
    """The C restatement (oracle/liboracle.so) timed the same way, single
    thread -- the CPU baseline when oracle/_ref was never built."""
    import time

    trie = Trie(patterns, L)
    secs, na = [], 0
    for i in range(warmup + runs):
        t0 = time.perf_counter()
        hits = pfac_scan(text, trie)
        na = len(verify_hits(text, hits, patterns, L))
        if i >= warmup:
            secs.append(time.perf_counter() - t0)
    return secs, na


# ------------------------------------------------------------------ workloads (reference arm)
# The same header-only generators libglop exports (csrc/workload.hpp), built
# into oracle/_ref/libref_logtrawl.so so the reference arm of bench.py never
# maps the product library.
def _ref_gen():
    r = ref()
    if r is None:
        raise RuntimeError("reference shim not built")
    if not getattr(r, "_gen_sigs", False):
        r.ref_gen_syslog.argtypes = [u8p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint]
        r.ref_gen_payload.argtypes = [u8p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint]
        r.ref_gen_rules.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, u8p, u8p]
        r.ref_gen_dpi_rules.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, u8p, u64p]
        r.ref_cpu_model.argtypes = [C.c_char_p, C.c_uint64]
        r._gen_sigs = True
    return r


def ref_gen_syslog(n: int, seed: int, begin: int = 0, threads: int = 0) -> np.ndarray:
    out = np.empty(max(n, 1), dtype=np.uint8)
    _ref_gen().ref_gen_syslog(out.ctypes.data_as(u8p), begin, n, seed, threads)
    return out[:n]


def ref_gen_payload(n: int, seed: int, begin: int = 0, threads: int = 0) -> np.ndarray:
    out = np.empty(max(n, 1), dtype=np.uint8)
    _ref_gen().ref_gen_payload(out.ctypes.data_as(u8p), begin, n, seed, threads)
    return out[:n]


def ref_gen_rules(k: int, seed: int, length: int = 8) -> list[bytes]:
    b = np.zeros(max(k * length, 1), dtype=np.uint8)
    _ref_gen().ref_gen_rules(k, seed, length, b.ctypes.data_as(u8p), None)
    return [bytes(b[i * length:(i + 1) * length]) for i in range(k)]


def ref_gen_dpi_rules(k: int, seed: int, min_len: int = 8, max_len: int = 24) -> list[bytes]:
    b = np.zeros(max(k * max_len, 1), dtype=np.uint8)
    off = np.zeros(k + 1, dtype=np.uint64)
    _ref_gen().ref_gen_dpi_rules(k, seed, min_len, max_len, b.ctypes.data_as(u8p), off.ctypes.data_as(u64p))
    return [bytes(b[int(off[i]):int(off[i + 1])]) for i in range(k)]


def cpu_model() -> str:
    r = ref()
    if r is not None:
        buf = C.create_string_buffer(256)
        _ref_gen().ref_cpu_model(buf, 256)
        return buf.value.decode(errors="replace")
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ref_chunked_ac_scan(text, patterns, chunk_size, overlap, workers=0):
    """The reference's chunked_ac_scan (scan.hpp:207-243) over
    build_ac_automaton(patterns): HIT_DTYPE records (offset, pattern_id, 0)."""
    r = ref()
    if not getattr(r, "_ac_sig", False):
        r.ref_chunked_ac_scan.argtypes = [u8p, C.c_uint64, u8p, u64p, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint,
                                          C.POINTER(C.c_void_p), u64p]
        r._ac_sig = True
    t, n = _text_arr(text)
    pat, off = pack_patterns(patterns)
    p, nm = C.c_void_p(), C.c_uint64()
    rc = r.ref_chunked_ac_scan(t.ctypes.data_as(u8p), n, pat.ctypes.data_as(u8p), off.ctypes.data_as(u64p),
                               len(patterns), chunk_size, overlap, workers, C.byref(p), C.byref(nm))
    if rc:
        raise OracleError(rc)
    return _take(p, nm.value, HIT_DTYPE, r.ref_free)
