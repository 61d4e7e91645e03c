"""ctypes binding to libglop.so (include/glop.h) -- the Python face of the
B200 matching path, used by the tests, bench.py and the multi-GPU driver.

Names follow the reference API (logtrawl::build_failureless_trie, pfac_scan,
verify_hits, kmp_search, ...).  There is no CPU fallback: if libglop.so is
missing this module raises on import, and device calls raise CudaError on a
machine without an sm_100 GPU.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GLOP_LIB") or os.path.join(HERE, "libglop.so")  # GLOP_LIB: experiment builds

HIT_DTYPE = np.dtype([("offset", "<u8"), ("pattern_id", "<u4"), ("matched_len", "<u4")])
ALERT_DTYPE = np.dtype([("offset", "<u8"), ("rule_id", "<u4"), ("pattern_len", "<u4")])

PFAC_AUTO, PFAC_FILTERED, PFAC_DIRECT, PFAC_PREFIX8 = 0, 1, 2, 3


class GlopError(RuntimeError):
    code = -1


class InvalidArgument(GlopError, ValueError):  # std::invalid_argument
    code = 1


class CapacityError(GlopError):  # logtrawl::CapacityError
    code = 2


class LogicError(GlopError):  # std::logic_error
    code = 3


class CudaError(GlopError):
    code = 4


class OutOfMemory(GlopError, MemoryError):
    code = 5


class Again(GlopError):  # an asynchronous call must be redone synchronously
    code = 6


_ERRORS = {c.code: c for c in (InvalidArgument, CapacityError, LogicError, CudaError, OutOfMemory, Again)}

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
_lib = C.CDLL(LIB_PATH)

vp = C.c_void_p
u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)


class TrieInfo(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("state_count", "classes", "min_depth", "max_depth", "q", "stride",
                                          "entry_bytes", "table_in_smem")] + [("table_bytes", C.c_uint64)] + \
        [(n, C.c_uint32) for n in ("jump_depth", "jump_in_smem", "jump_slots", "reserved")]


def _sig(name, *args):
    f = getattr(_lib, name)
    f.argtypes = list(args)
    f.restype = C.c_int
    return f


_lib.glop_last_error.restype = C.c_char_p
_lib.glop_version.restype = C.c_char_p
_lib.glop_ctx_stream.argtypes = [vp]
_lib.glop_ctx_stream.restype = vp
_lib.glop_free.argtypes = [vp]
_lib.glop_free.restype = None
_sig("glop_ctx_create", C.c_int, C.POINTER(vp))
_sig("glop_ctx_destroy", vp)
_sig("glop_ctx_synchronize", vp)
_sig("glop_trie_upload", vp, i32p, C.c_uint32, u32p, vp, C.POINTER(vp))
_sig("glop_trie_destroy", vp)
_sig("glop_trie_get_info", vp, C.POINTER(TrieInfo))
_sig("glop_pfac_scan", vp, vp, vp, C.c_uint64, C.c_int, C.POINTER(vp), u64p)
_sig("glop_pfac_scan_device", vp, vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, vp, C.c_uint64, u64p)
_sig("glop_run_pfac_pipeline", vp, vp, vp, vp, C.c_uint64, C.c_int, C.POINTER(vp), u64p, u64p, u64p)
_sig("glop_run_pfac_pipeline_shard", vp, vp, vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(vp), u64p,
     u64p, u64p)
_sig("glop_last_kernel_ms", vp, C.POINTER(C.c_float))
_lib.glop_ctx_launch_count.argtypes = [vp]
_lib.glop_ctx_launch_count.restype = C.c_uint64
_lib.glop_ctx_fallback_count.argtypes = [vp]
_lib.glop_ctx_fallback_count.restype = C.c_uint64
_sig("glop_run_pfac_pipeline_device", vp, vp, vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, vp, C.c_uint64, vp,
     C.c_uint64, vp, u64p, u64p)
_sig("glop_run_pfac_pipeline_device_async", vp, vp, vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, vp, C.c_uint64, vp,
     C.c_uint64, vp, vp)
_sig("glop_pipeline_ticket_result", vp, u64p, u64p)
_sig("glop_kmp_search_device_async", vp, u8p, C.c_uint32, u32p, vp, C.c_uint64, C.c_uint64, C.c_uint64, vp,
     C.c_uint64, vp)
_sig("glop_kmp_ticket_result", vp, u64p, u64p)


def kmp_ticket_result(ticket_ptr: int):
    """(n_offsets, comparisons) of an asynchronous KMP call, once its
    context's stream is synchronized; raises Again when it must be redone."""
    no, cmp_ = C.c_uint64(), C.c_uint64(0)
    _check(_lib.glop_kmp_ticket_result(ticket_ptr, C.byref(no), C.byref(cmp_)), "kmp_ticket_result")
    return no.value, cmp_.value
_sig("glop_chunked_ac_scan", vp, vp, vp, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.POINTER(vp), u64p)
TICKET_BYTES = 8 * 8 + 3 * 8 + 2 * 4  # glop_pipeline_ticket
# peer exchange (CUDA IPC + copy engines; glop.h "peer exchange", peer.py)
_sig("glop_peer_alloc", vp, C.c_uint64, C.POINTER(vp), vp)
_sig("glop_peer_free", vp, vp)
_sig("glop_peer_open", vp, vp, C.POINTER(vp))
_sig("glop_peer_close", vp, vp)
_sig("glop_peer_event", vp, C.POINTER(vp), vp)
_sig("glop_peer_event_open", vp, vp, C.POINTER(vp))
_sig("glop_peer_event_destroy", vp, vp)
_sig("glop_peer_record", vp, vp, vp)
_sig("glop_peer_wait", vp, vp, vp)
_sig("glop_peer_copy", vp, vp, vp, C.c_uint64, vp)


def ticket_result(ticket_ptr: int):
    """(n_hits, n_alerts) of an asynchronous pipeline call, once its context's
    stream is synchronized; raises Again when it must be redone synchronously."""
    nh, na = C.c_uint64(), C.c_uint64()
    _check(_lib.glop_pipeline_ticket_result(ticket_ptr, C.byref(nh), C.byref(na)), "pipeline_ticket_result")
    return nh.value, na.value
_sig("glop_rules_upload", vp, u8p, u64p, C.c_uint32, C.c_uint64, C.POINTER(vp))
_sig("glop_rules_destroy", vp)
_sig("glop_verify_hits", vp, vp, vp, C.c_uint64, C.c_int, vp, C.c_uint64, C.c_int, C.POINTER(vp), u64p, u64p)
_sig("glop_verify_hits_device", vp, vp, vp, C.c_uint64, C.c_uint64, vp, C.c_uint64, vp, u64p, vp)
_sig("glop_kmp_search", vp, u8p, C.c_uint32, u32p, vp, C.c_uint64, C.c_int, C.POINTER(vp), u64p, u64p)
_sig("glop_kmp_search_device", vp, u8p, C.c_uint32, u32p, vp, C.c_uint64, C.c_uint64, C.c_uint64, vp,
     C.c_uint64, u64p, u64p)
_sig("glop_device_alloc", vp, C.c_uint64, C.POINTER(vp))
_sig("glop_device_free", vp, vp)
_sig("glop_host_alloc", C.c_uint64, C.POINTER(vp))
_sig("glop_host_free", vp)
_sig("glop_memcpy", vp, vp, vp, C.c_uint64, C.c_int)
_sig("glop_gen_syslog_device", vp, vp, C.c_uint64, C.c_uint64, C.c_uint64)
_sig("glop_gen_syslog_host", vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint)
_sig("glop_gen_reference_log", vp, C.c_uint64, C.c_uint32, C.c_uint64)
_sig("glop_gen_payload_device", vp, vp, C.c_uint64, C.c_uint64, C.c_uint64)
_sig("glop_line_numbers", vp, vp, C.c_uint64, C.c_int, u64p, C.c_uint64, u64p)
_sig("glop_line_numbers_device", vp, vp, C.c_uint64, C.c_uint64, vp, C.c_uint32, C.c_uint64, vp)
_sig("glop_gen_payload_host", vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint)
_sig("glop_gen_dpi_rules", C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, u8p, u64p)
_sig("glop_gen_rules", C.c_uint32, C.c_uint32, C.c_uint32, u8p, u8p)
_sig("glop_build_failureless_trie", u8p, u64p, C.c_uint32, C.c_uint64, C.c_uint64, C.POINTER(i32p),
     u32p, C.POINTER(u32p), C.POINTER(vp))


def _check(rc: int, what: str):
    if rc:
        msg = (_lib.glop_last_error() or b"").decode(errors="replace")
        raise _ERRORS.get(rc, GlopError)(f"{what}: {msg}")


def version() -> str:
    return _lib.glop_version().decode()


def lib_handle():
    return _lib


def _u8(b) -> np.ndarray:
    if isinstance(b, np.ndarray):
        return np.ascontiguousarray(b, dtype=np.uint8)
    return np.frombuffer(bytes(b), dtype=np.uint8) if len(b) else np.zeros(0, np.uint8)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(vp) if a.size else None


def pack_patterns(patterns):
    blob = b"".join(patterns)
    off = np.zeros(len(patterns) + 1, dtype=np.uint64)
    if patterns:
        np.cumsum([len(p) for p in patterns], out=off[1:])
    arr = np.frombuffer(blob, dtype=np.uint8).copy() if blob else np.zeros(1, np.uint8)
    return arr, off


def _take(ptr: vp, n: int, dtype) -> np.ndarray:
    """numpy view of a library-owned result array; large results are not
    copied -- the buffer is released by glop_free once the last view is
    gone."""
    if not n:
        _lib.glop_free(ptr)
        return np.zeros(0, dtype=dtype)
    nbytes = n * np.dtype(dtype).itemsize
    if nbytes < (1 << 20):
        raw = np.ctypeslib.as_array(C.cast(ptr, u8p), shape=(nbytes,))
        out = raw.view(dtype).copy()
        _lib.glop_free(ptr)
        return out
    buf = (C.c_uint8 * nbytes).from_address(ptr.value)
    weakref.finalize(buf, _lib.glop_free, C.c_void_p(ptr.value))
    return np.frombuffer(buf, dtype=dtype)


# ----------------------------------------------------------------- host side
@dataclass
class Automaton:
    """The reference's dense failureless trie (automaton.hpp:51-141)."""

    dense_table: np.ndarray  # (Q, 256) int32, -1 = no edge
    out_offsets: np.ndarray  # Q + 1 uint32
    out_flat: np.ndarray     # (n_out, 2) uint32: (pattern_id, matched_len)

    @property
    def state_count(self) -> int:
        return self.dense_table.shape[0]


def build_failureless_trie(patterns, prefix_len: int = 8, max_states: int = 1 << 22) -> Automaton:
    """truncate_prefixes + build_failureless_trie (rules.hpp:190, automaton.hpp:283),
    run by the drop-in C++ host code inside libglop."""
    pat, off = pack_patterns(list(patterns))
    d, q, o, f = i32p(), C.c_uint32(), u32p(), vp()
    _check(_lib.glop_build_failureless_trie(pat.ctypes.data_as(u8p), off.ctypes.data_as(u64p), len(patterns),
                                            prefix_len, max_states, C.byref(d), C.byref(q), C.byref(o),
                                            C.byref(f)), "build_failureless_trie")
    Q = q.value
    dense = np.ctypeslib.as_array(d, shape=(Q * 256,)).reshape(Q, 256).copy()
    offs = np.ctypeslib.as_array(o, shape=(Q + 1,)).copy()
    n_out = int(offs[-1])
    flat = np.ctypeslib.as_array(C.cast(f, u32p), shape=(max(2 * n_out, 1),)).copy()[:2 * n_out].reshape(n_out, 2)
    for p in (C.cast(d, vp), C.cast(o, vp), f):
        _lib.glop_free(p)
    return Automaton(dense, offs, flat)


def gen_syslog_host(n: int, seed: int, begin: int = 0, threads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    buf = np.empty(n, dtype=np.uint8) if out is None else out
    if n:
        _check(_lib.glop_gen_syslog_host(buf.ctypes.data_as(vp), begin, n, seed, threads), "gen_syslog_host")
    return buf


def gen_payload_host(n: int, seed: int, begin: int = 0, threads: int = 0) -> np.ndarray:
    """Bytes [begin, begin+n) of the synthetic packet-payload stream (DPI config)."""
    buf = np.empty(n, dtype=np.uint8)
    if n:
        _check(_lib.glop_gen_payload_host(buf.ctypes.data_as(vp), begin, n, seed, threads), "gen_payload_host")
    return buf


def gen_dpi_rules(k: int, seed: int, min_len: int = 8, max_len: int = 24) -> list[bytes]:
    """Snort-style content set for the DPI config (see csrc/workload.hpp)."""
    b = np.zeros(max(k * max_len, 1), dtype=np.uint8)
    off = np.zeros(k + 1, dtype=np.uint64)
    _check(_lib.glop_gen_dpi_rules(k, seed, min_len, max_len, b.ctypes.data_as(u8p), off.ctypes.data_as(u64p)),
           "gen_dpi_rules")
    raw = b.tobytes()
    return [raw[int(off[i]):int(off[i + 1])] for i in range(k)]


def gen_reference_log(size: int, seed: int, line_len: int = 80) -> np.ndarray:
    buf = np.empty(size, dtype=np.uint8)
    _check(_lib.glop_gen_reference_log(buf.ctypes.data_as(vp), size, seed, line_len), "generate_log")
    return buf


def gen_rules(k: int, seed: int, length: int = 8):
    """(patterns, is_vocab): the bench rule sets (see csrc/workload.hpp)."""
    b = np.zeros(max(k * length, 1), dtype=np.uint8)
    v = np.zeros(max(k, 1), dtype=np.uint8)
    _check(_lib.glop_gen_rules(k, seed, length, b.ctypes.data_as(u8p), v.ctypes.data_as(u8p)), "gen_rules")
    raw = b.tobytes()
    return [raw[i * length:(i + 1) * length] for i in range(k)], v[:k].astype(bool)


def kmp_failure_table(p: bytes) -> np.ndarray:
    """build_failure_table (kmp.hpp:25-36), host side like the reference."""
    t = np.zeros(len(p), dtype=np.uint32)
    k = 0
    for i in range(1, len(p)):
        while k and p[i] != p[k]:
            k = int(t[k - 1])
        if p[i] == p[k]:
            k += 1
        t[i] = k
    return t


# ----------------------------------------------------------------- device side
class DeviceTrie:
    def __init__(self, ctx: "Context", h: vp):
        self._ctx, self.h = ctx, h

    @property
    def info(self) -> TrieInfo:
        i = TrieInfo()
        _check(_lib.glop_trie_get_info(self.h, C.byref(i)), "trie_info")
        return i

    def close(self):
        if self.h:
            _lib.glop_trie_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceRules:
    def __init__(self, h: vp, n_patterns: int):
        self.h, self.n_patterns = h, n_patterns

    def close(self):
        if self.h:
            _lib.glop_rules_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """One CUDA device + stream + scratch (glop_ctx)."""

    def __init__(self, device: int = 0):
        h = vp()
        _check(_lib.glop_ctx_create(device, C.byref(h)), "glop_ctx_create")
        self.h, self.device = h, device

    def close(self):
        if getattr(self, "h", None):
            _lib.glop_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return _lib.glop_ctx_stream(self.h) or 0

    def synchronize(self):
        _check(_lib.glop_ctx_synchronize(self.h), "synchronize")

    # -- automaton / rules
    def upload(self, a: Automaton) -> DeviceTrie:
        dense = np.ascontiguousarray(a.dense_table, dtype=np.int32)
        offs = np.ascontiguousarray(a.out_offsets, dtype=np.uint32)
        flat = np.ascontiguousarray(a.out_flat, dtype=np.uint32).reshape(-1)
        if flat.size == 0:
            flat = np.zeros(2, np.uint32)
        h = vp()
        _check(_lib.glop_trie_upload(self.h, dense.ctypes.data_as(i32p), dense.shape[0], offs.ctypes.data_as(u32p),
                                     flat.ctypes.data_as(vp), C.byref(h)), "glop_trie_upload")
        return DeviceTrie(self, h)

    def upload_rules(self, patterns, prefix_len: int) -> DeviceRules:
        pat, off = pack_patterns(list(patterns))
        h = vp()
        _check(_lib.glop_rules_upload(self.h, pat.ctypes.data_as(u8p), off.ctypes.data_as(u64p), len(patterns),
                                      prefix_len, C.byref(h)), "glop_rules_upload")
        return DeviceRules(h, len(patterns))

    # -- PFAC
    def pfac_scan(self, trie: DeviceTrie, text) -> np.ndarray:
        t = _u8(text)
        p, n = vp(), C.c_uint64()
        _check(_lib.glop_pfac_scan(self.h, trie.h, _ptr(t), t.size, 0, C.byref(p), C.byref(n)), "pfac_scan")
        return _take(p, n.value, HIT_DTYPE)

    def pfac_scan_device(self, trie: DeviceTrie, d_text: int, n: int, d_out: int, cap: int, own: int | None = None,
                         base: int = 0, kernel: int = PFAC_AUTO) -> int:
        nh = C.c_uint64()
        _check(_lib.glop_pfac_scan_device(self.h, trie.h, d_text, n, n if own is None else own, base, kernel, d_out,
                                          cap, C.byref(nh)), "pfac_scan_device")
        return nh.value

    # -- end-to-end pipeline (run_engine_scan's PFAC branch)
    def run_pfac_pipeline(self, trie: DeviceTrie, rules: DeviceRules, text_ptr: int, n: int, on_device: bool,
                          own: int | None = None, base: int = 0):
        """(alerts, counts, stage1_hits) for text at a raw host or device pointer
        covering global offsets [base, base+n); starts [base, base+own) reported."""
        p, na, s1 = vp(), C.c_uint64(), C.c_uint64()
        cnt = np.zeros(max(rules.n_patterns, 1), dtype=np.uint64)
        _check(_lib.glop_run_pfac_pipeline_shard(self.h, trie.h, rules.h, text_ptr, n, n if own is None else own, base,
                                                 1 if on_device else 0, C.byref(p), C.byref(na),
                                                 cnt.ctypes.data_as(u64p), C.byref(s1)), "run_pfac_pipeline")
        return _take(p, na.value, ALERT_DTYPE), cnt[:rules.n_patterns], s1.value

    def run_pfac_pipeline_device(self, trie: DeviceTrie, rules: DeviceRules, d_text: int, n: int, d_alerts: int,
                                 alert_cap: int, d_counts: int | None = None, own: int | None = None, base: int = 0,
                                 d_hits: int | None = None, hit_cap: int = 0):
        """Device-resident scan + verify + counts (one host wait): returns
        (n_hits, n_alerts); alerts / counts / optional hits stay on the device."""
        nh, na = C.c_uint64(), C.c_uint64()
        _check(_lib.glop_run_pfac_pipeline_device(self.h, trie.h, rules.h, d_text, n, n if own is None else own, base,
                                                  d_hits, hit_cap, d_alerts, alert_cap, d_counts, C.byref(nh),
                                                  C.byref(na)), "run_pfac_pipeline_device")
        return nh.value, na.value

    def run_pfac_pipeline_device_async(self, trie: DeviceTrie, rules: DeviceRules, d_text: int, n: int,
                                       d_alerts: int, alert_cap: int, d_counts: int | None, ticket: int,
                                       own: int | None = None, base: int = 0, d_hits: int | None = None,
                                       hit_cap: int = 0):
        """Enqueue the device pipeline without waiting; `ticket` (pinned host
        memory, TICKET_BYTES) receives the status -- read it with
        ticket_result() after synchronize()."""
        _check(_lib.glop_run_pfac_pipeline_device_async(self.h, trie.h, rules.h, d_text, n, n if own is None else own,
                                                        base, d_hits, hit_cap, d_alerts, alert_cap, d_counts, ticket),
               "run_pfac_pipeline_device_async")

    def chunked_ac_scan(self, ac_trie: DeviceTrie, text, chunk_size: int, overlap: int) -> np.ndarray:
        """chunked_ac_scan (scan.hpp:207-243): `ac_trie` is the goto trie of the
        full patterns (build_failureless_trie(patterns, max_len)); sorted
        (offset, pattern_id, matched_len) records of the owned, reached matches."""
        t = _u8(text)
        p, n = vp(), C.c_uint64()
        _check(_lib.glop_chunked_ac_scan(self.h, ac_trie.h, _ptr(t), t.size, 0, chunk_size, overlap, C.byref(p),
                                         C.byref(n)), "chunked_ac_scan")
        return _take(p, n.value, HIT_DTYPE)

    @property
    def fallbacks(self) -> int:
        """Scans on this context that took the exact global-key fallback."""
        return int(_lib.glop_ctx_fallback_count(self.h))

    def line_numbers(self, text, offsets) -> np.ndarray:
        """LineIndex(text).line_of(o) for every o (verify.hpp:40-64), on the device."""
        t = _u8(text)
        o = np.ascontiguousarray(offsets, dtype=np.uint64)
        out = np.zeros(o.size, dtype=np.uint64)
        _check(_lib.glop_line_numbers(self.h, _ptr(t), t.size, 0, o.ctypes.data_as(u64p), o.size,
                                      out.ctypes.data_as(u64p)), "line_numbers")
        return out

    def line_numbers_device(self, d_text: int, n: int, d_records: int, stride: int, count: int, d_lines: int,
                            base: int = 0):
        _check(_lib.glop_line_numbers_device(self.h, d_text, n, base, d_records, stride, count, d_lines),
               "line_numbers_device")

    def last_kernel_ms(self) -> float:
        ms = C.c_float()
        _check(_lib.glop_last_kernel_ms(self.h, C.byref(ms)), "last_kernel_ms")
        return ms.value

    @property
    def launches(self) -> int:
        return int(_lib.glop_ctx_launch_count(self.h))

    # -- verify
    def verify_hits(self, rules: DeviceRules, text, hits: np.ndarray, counts: bool = False):
        t = _u8(text)
        h = np.ascontiguousarray(hits, dtype=HIT_DTYPE)
        p, n = vp(), C.c_uint64()
        cnt = np.zeros(max(rules.n_patterns, 1), dtype=np.uint64)
        _check(_lib.glop_verify_hits(self.h, rules.h, _ptr(t), t.size, 0, _ptr(h), h.size, 0, C.byref(p),
                                     C.byref(n), cnt.ctypes.data_as(u64p) if counts else None), "verify_hits")
        a = _take(p, n.value, ALERT_DTYPE)
        return (a, cnt[:rules.n_patterns]) if counts else a

    def verify_hits_device(self, rules: DeviceRules, d_text: int, n: int, d_hits: int, n_hits: int, d_out: int,
                           d_counts: int | None = None, base: int = 0) -> int:
        na = C.c_uint64()
        _check(_lib.glop_verify_hits_device(self.h, rules.h, d_text, n, base, d_hits, n_hits, d_out, C.byref(na),
                                            d_counts), "verify_hits_device")
        return na.value

    # -- KMP
    def kmp_search(self, pattern: bytes, text, failure: np.ndarray | None = None):
        """(offsets, comparisons)"""
        t = _u8(text)
        p = _u8(pattern)
        f = np.ascontiguousarray(kmp_failure_table(pattern) if failure is None else failure, dtype=np.uint32)
        o, n, cmp_ = vp(), C.c_uint64(), C.c_uint64(0)
        pp = p if p.size else np.zeros(1, np.uint8)
        ff = f if f.size else np.zeros(1, np.uint32)
        _check(_lib.glop_kmp_search(self.h, pp.ctypes.data_as(u8p), p.size, ff.ctypes.data_as(u32p), _ptr(t), t.size,
                                    0, C.byref(o), C.byref(n), C.byref(cmp_)), "kmp_search")
        return _take(o, n.value, np.uint64), cmp_.value

    def kmp_search_device(self, pattern: bytes, d_text: int, n: int, d_out: int, cap: int, own: int | None = None,
                          base: int = 0):
        """(n_offsets, comparisons)"""
        p = _u8(pattern)
        f = kmp_failure_table(pattern)
        no, cmp_ = C.c_uint64(), C.c_uint64(0)
        _check(_lib.glop_kmp_search_device(self.h, p.ctypes.data_as(u8p), p.size, f.ctypes.data_as(u32p), d_text, n,
                                           n if own is None else own, base, d_out, cap, C.byref(no), C.byref(cmp_)),
               "kmp_search_device")
        return no.value, cmp_.value

    def kmp_search_device_async(self, pattern: bytes, d_text: int, n: int, d_out: int, cap: int, ticket: int,
                                own: int | None = None, base: int = 0):
        """Enqueue the device KMP without waiting (result via kmp_ticket_result)."""
        p = _u8(pattern)
        f = kmp_failure_table(pattern)
        self._kmp_keep = (p, f)  # alive until the call returns (the DFA is built from them on the host)
        _check(_lib.glop_kmp_search_device_async(self.h, p.ctypes.data_as(u8p), p.size, f.ctypes.data_as(u32p),
                                                 d_text, n, n if own is None else own, base, d_out, cap, ticket),
               "kmp_search_device_async")

    # -- memory / workloads
    def host_alloc(self, nbytes: int) -> int:
        """Pinned host buffer (cudaMallocHost); free with host_free."""
        h = vp()
        _check(_lib.glop_host_alloc(nbytes, C.byref(h)), "host_alloc")
        return h.value

    def host_free(self, ptr: int):
        _check(_lib.glop_host_free(ptr), "host_free")

    def memcpy(self, dst: int, src: int, nbytes: int, kind: int):
        """kind: 1 h2d, 2 d2h, 3 d2d (on the context stream)."""
        _check(_lib.glop_memcpy(self.h, dst, src, nbytes, kind), "memcpy")

    def gen_syslog_device(self, d_out: int, n: int, seed: int, begin: int = 0):
        _check(_lib.glop_gen_syslog_device(self.h, d_out, begin, n, seed), "gen_syslog_device")

    def gen_payload_device(self, d_out: int, n: int, seed: int, begin: int = 0):
        _check(_lib.glop_gen_payload_device(self.h, d_out, begin, n, seed), "gen_payload_device")


# ---------------------------------------------------------------- drop-in engine
class Engine:
    """The drop-in C++ run_engine_scan (include/logtrawl/pipeline.hpp) through
    libglop_engine.so -- the call a reference C++ caller makes, for bench.py's
    e2e_dropin leg and FFI callers.  engine: "kmp", "pfac_dense",
    "pfac_compact" (default), "ac_chunked"."""

    ENGINES = {"kmp": 0, "pfac_dense": 1, "pfac_compact": 2, "ac_chunked": 3}

    def __init__(self, patterns):
        path = os.path.join(HERE, "libglop_engine.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} is not built (make -C paper_1704_02278_b200/cli)")
        self.lib = C.CDLL(path)
        self.lib.glop_engine_rules_create.restype = vp
        self.lib.glop_engine_rules_create.argtypes = [u8p, u64p, C.c_uint32]
        self.lib.glop_engine_rules_destroy.argtypes = [vp]
        self.lib.glop_engine_last_error.restype = C.c_char_p
        self.lib.glop_engine_run.argtypes = [vp, vp, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.c_int,
                                             C.POINTER(vp), C.POINTER(vp), u64p, u64p]
        pat, off = pack_patterns(list(patterns))
        self.h = self.lib.glop_engine_rules_create(pat.ctypes.data_as(u8p), off.ctypes.data_as(u64p), len(patterns))

    def run(self, text_ptr: int, n: int, engine: str = "pfac_compact", prefix_len: int = 8, chunk_size: int = 0,
            lines: bool = False):
        """(alerts ALERT_DTYPE, lines or None, stage1_hits) of run_engine_scan
        over the host bytes at text_ptr (pageable or pinned)."""
        a, ln, na, s1 = vp(), vp(), C.c_uint64(), C.c_uint64()
        rc = self.lib.glop_engine_run(self.h, text_ptr, n, self.ENGINES[engine], prefix_len, chunk_size,
                                      1 if lines else 0, C.byref(a), C.byref(ln), C.byref(na), C.byref(s1))
        if rc:
            raise _ERRORS.get({1: 1, 2: 2, 3: 3}.get(rc, 4), GlopError)(
                "run_engine_scan: " + (self.lib.glop_engine_last_error() or b"").decode())
        alerts = _take(a, na.value, ALERT_DTYPE)
        return alerts, (_take(ln, na.value, np.uint64) if lines else None), s1.value

    def close(self):
        if getattr(self, "h", None):
            self.lib.glop_engine_rules_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- multi-GPU group
_sig("glop_group_create", vp, C.c_int, C.POINTER(vp))
_sig("glop_group_destroy", vp)
_lib.glop_group_size.argtypes = [vp]
_lib.glop_group_size.restype = C.c_int
_sig("glop_group_trie_upload", vp, i32p, C.c_uint32, u32p, vp, C.POINTER(vp))
_sig("glop_group_trie_destroy", vp)
_sig("glop_group_rules_upload", vp, u8p, u64p, C.c_uint32, C.c_uint64, C.POINTER(vp))
_sig("glop_group_rules_destroy", vp)
_sig("glop_group_pfac_scan", vp, vp, vp, C.c_uint64, C.POINTER(vp), u64p)
_sig("glop_group_run_pfac_pipeline", vp, vp, vp, vp, C.c_uint64, C.POINTER(vp), u64p, u64p, u64p, C.POINTER(vp), u64p)
_sig("glop_group_kmp_search", vp, u8p, C.c_uint32, u32p, vp, C.c_uint64, C.POINTER(vp), u64p, u64p)
_sig("glop_plan_shards", C.c_uint64, C.c_uint32, C.c_uint64, u64p, u64p, u64p)


def plan_shards_c(n: int, parts: int, halo: int):
    """glop_plan_shards (host only): [(lo, own, read)] per shard."""
    lo, own, rd = (np.zeros(parts, np.uint64) for _ in range(3))
    _check(_lib.glop_plan_shards(n, parts, halo, lo.ctypes.data_as(u64p), own.ctypes.data_as(u64p),
                                 rd.ctypes.data_as(u64p)), "plan_shards")
    return [(int(a), int(b), int(c)) for a, b, c in zip(lo, own, rd)]


class Group:
    """A glop_group: one context per member device (devices may repeat);
    every call splits the text into halo'd shards across the members and
    merges the results in rank order."""

    def __init__(self, devices=None):
        h = vp()
        if devices is None:
            _check(_lib.glop_group_create(None, 0, C.byref(h)), "glop_group_create")
        else:
            d = (C.c_int * len(devices))(*devices)
            _check(_lib.glop_group_create(d, len(devices), C.byref(h)), "glop_group_create")
        self.h = h

    @property
    def size(self) -> int:
        return int(_lib.glop_group_size(self.h))

    def close(self):
        if getattr(self, "h", None):
            _lib.glop_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, a: Automaton):
        dense = np.ascontiguousarray(a.dense_table, dtype=np.int32)
        offs = np.ascontiguousarray(a.out_offsets, dtype=np.uint32)
        flat = np.ascontiguousarray(a.out_flat, dtype=np.uint32).reshape(-1)
        if flat.size == 0:
            flat = np.zeros(2, np.uint32)
        h = vp()
        _check(_lib.glop_group_trie_upload(self.h, dense.ctypes.data_as(i32p), dense.shape[0],
                                           offs.ctypes.data_as(u32p), flat.ctypes.data_as(vp), C.byref(h)),
               "glop_group_trie_upload")
        return _GroupHandle(h, _lib.glop_group_trie_destroy)

    def upload_rules(self, patterns, prefix_len: int):
        pat, off = pack_patterns(list(patterns))
        h = vp()
        _check(_lib.glop_group_rules_upload(self.h, pat.ctypes.data_as(u8p), off.ctypes.data_as(u64p), len(patterns),
                                            prefix_len, C.byref(h)), "glop_group_rules_upload")
        r = _GroupHandle(h, _lib.glop_group_rules_destroy)
        r.n_patterns = len(patterns)
        return r

    def pfac_scan(self, trie, text) -> np.ndarray:
        t = _u8(text)
        p, n = vp(), C.c_uint64()
        _check(_lib.glop_group_pfac_scan(self.h, trie.h, _ptr(t), t.size, C.byref(p), C.byref(n)), "group_pfac_scan")
        return _take(p, n.value, HIT_DTYPE)

    def run_pfac_pipeline(self, trie, rules, text, lines: bool = False):
        """(alerts, counts, stage1_hits, lines or None, line_count or None)"""
        t = _u8(text)
        p, na, s1, lp, lc = vp(), C.c_uint64(), C.c_uint64(), vp(), C.c_uint64()
        cnt = np.zeros(max(rules.n_patterns, 1), dtype=np.uint64)
        _check(_lib.glop_group_run_pfac_pipeline(self.h, trie.h, rules.h, _ptr(t), t.size, C.byref(p), C.byref(na),
                                                 cnt.ctypes.data_as(u64p), C.byref(s1),
                                                 C.byref(lp) if lines else None, C.byref(lc) if lines else None),
               "group_run_pfac_pipeline")
        alerts = _take(p, na.value, ALERT_DTYPE)
        return (alerts, cnt[:rules.n_patterns], s1.value, _take(lp, na.value, np.uint64) if lines else None,
                lc.value if lines else None)

    def kmp_search(self, pattern: bytes, text, failure: np.ndarray | None = None):
        t = _u8(text)
        p = _u8(pattern)
        f = np.ascontiguousarray(kmp_failure_table(pattern) if failure is None else failure, dtype=np.uint32)
        o, n, cmp_ = vp(), C.c_uint64(), C.c_uint64(0)
        pp = p if p.size else np.zeros(1, np.uint8)
        ff = f if f.size else np.zeros(1, np.uint32)
        _check(_lib.glop_group_kmp_search(self.h, pp.ctypes.data_as(u8p), p.size, ff.ctypes.data_as(u32p), _ptr(t),
                                          t.size, C.byref(o), C.byref(n), C.byref(cmp_)), "group_kmp_search")
        return _take(o, n.value, np.uint64), cmp_.value


class _GroupHandle:
    def __init__(self, h, destroy):
        self.h, self._destroy = h, destroy

    def close(self):
        if getattr(self, "h", None):
            self._destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- streaming ingest
_sig("glop_stream_begin", vp, vp, vp, C.c_int, C.POINTER(vp))
_sig("glop_stream_feed", vp, vp, C.c_uint64)
_sig("glop_stream_end", vp, C.POINTER(vp), u64p, u64p, u64p, C.POINTER(vp), u64p, u64p)


class Stream:
    """glop_stream_*: the PFAC pipeline over a text fed in pieces of any size
    (the result equals run_pfac_pipeline over the concatenation)."""

    def __init__(self, ctx: "Context", trie: "DeviceTrie", rules: "DeviceRules", lines: bool = False):
        h = vp()
        _check(_lib.glop_stream_begin(ctx.h, trie.h, rules.h, 1 if lines else 0, C.byref(h)), "stream_begin")
        self.h, self.lines, self.n_patterns = h, lines, rules.n_patterns
        self._keep = (ctx, trie, rules)

    def feed(self, data):
        t = _u8(data)
        _check(_lib.glop_stream_feed(self.h, _ptr(t), t.size), "stream_feed")

    def end(self):
        """(alerts, counts, stage1_hits, lines or None, line_count or None, bytes)"""
        p, na, s1, lp, lc, nb = vp(), C.c_uint64(), C.c_uint64(), vp(), C.c_uint64(), C.c_uint64()
        cnt = np.zeros(max(self.n_patterns, 1), dtype=np.uint64)
        h, self.h = self.h, None
        _check(_lib.glop_stream_end(h, C.byref(p), C.byref(na), cnt.ctypes.data_as(u64p), C.byref(s1),
                                    C.byref(lp) if self.lines else None, C.byref(lc) if self.lines else None,
                                    C.byref(nb)), "stream_end")
        alerts = _take(p, na.value, ALERT_DTYPE)
        return (alerts, cnt[:self.n_patterns], s1.value, _take(lp, na.value, np.uint64) if self.lines else None,
                lc.value if self.lines else None, nb.value)


_sig("glop_group_stream_begin", vp, vp, vp, C.c_int, C.c_uint64, C.POINTER(vp))
_sig("glop_group_stream_feed", vp, vp, C.c_uint64)
_sig("glop_group_stream_end", vp, C.POINTER(vp), u64p, u64p, u64p, C.POINTER(vp), u64p, u64p)


class GroupStream(Stream):
    """glop_group_stream_*: windows handed round-robin to the group's members."""

    def __init__(self, group: Group, trie, rules, lines: bool = False, window: int = 0):
        h = vp()
        _check(_lib.glop_group_stream_begin(group.h, trie.h, rules.h, 1 if lines else 0, window, C.byref(h)),
               "group_stream_begin")
        self.h, self.lines, self.n_patterns = h, lines, rules.n_patterns
        self._keep = (group, trie, rules)
        self._feed, self._end = _lib.glop_group_stream_feed, _lib.glop_group_stream_end

    def feed(self, data):
        t = _u8(data)
        _check(self._feed(self.h, _ptr(t), t.size), "group_stream_feed")

    def end(self):
        p, na, s1, lp, lc, nb = vp(), C.c_uint64(), C.c_uint64(), vp(), C.c_uint64(), C.c_uint64()
        cnt = np.zeros(max(self.n_patterns, 1), dtype=np.uint64)
        h, self.h = self.h, None
        _check(self._end(h, C.byref(p), C.byref(na), cnt.ctypes.data_as(u64p), C.byref(s1),
                         C.byref(lp) if self.lines else None, C.byref(lc) if self.lines else None, C.byref(nb)),
               "group_stream_end")
        alerts = _take(p, na.value, ALERT_DTYPE)
        return (alerts, cnt[:self.n_patterns], s1.value, _take(lp, na.value, np.uint64) if self.lines else None,
                lc.value if self.lines else None, nb.value)
