"""Scratch: a few small calls of every device path, for compute-sanitizer."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1704_02278_b200 import glop
ctx = glop.Context(0)
text = glop.gen_syslog_host((3 << 20) + 13, 5)
for k, L in ((10, 8), (100, 8), (1000, 8), (300, 4)):
    pats = glop.gen_rules(k, 606)[0] + [b"Failed password for", b"Failed passwd"]
    trie = ctx.upload(glop.build_failureless_trie(pats, L))
    rules = ctx.upload_rules(pats, L)
    h = ctx.pfac_scan(trie, text)
    a, c, s1 = ctx.run_pfac_pipeline(trie, rules, text.ctypes.data, text.size, False)
    print(k, L, len(h), len(a), s1, flush=True)
pay = glop.gen_payload_host(2 << 20, 3)
pats = glop.gen_dpi_rules(10000, 606, 8, 24)
trie = ctx.upload(glop.build_failureless_trie(pats, 8)); rules = ctx.upload_rules(pats, 8)
a, c, s1 = ctx.run_pfac_pipeline(trie, rules, pay.ctypes.data, pay.size, False)
print("dpi", len(a), s1, flush=True)
offs, cmp_ = ctx.kmp_search(b"Failed password", text)
print("kmp", len(offs), cmp_, flush=True)
dense = np.full(1 << 16, 65, np.uint8)
dp = [b"AAAAAAAA" + bytes([66 + j]) for j in range(40)] + [b"AAAAAAAA"]
t2 = ctx.upload(glop.build_failureless_trie(dp, 8))
print("dense", len(ctx.pfac_scan(t2, dense)), flush=True)
ac = ctx.upload(glop.build_failureless_trie(pats[:50], max(len(p) for p in pats[:50])))
print("chunked", len(ctx.chunked_ac_scan(ac, pay[:1 << 20], 4096, 30)), flush=True)
