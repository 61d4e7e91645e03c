"""Where the drop-in e2e time goes: pinned vs pageable text through the C ABI
pipeline and through run_engine_scan (libglop_engine.so)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1704_02278_b200 import glop
S = int(float(sys.argv[1])) if len(sys.argv) > 1 else 8_000_000_000
ctx = glop.Context(0)
pats, _ = glop.gen_rules(1000, 606)
trie = ctx.upload(glop.build_failureless_trie(pats, 8)); rules = ctx.upload_rules(pats, 8)
d = torch.empty(S + 64, dtype=torch.uint8, device="cuda"); ctx.gen_syslog_device(d.data_ptr(), S, 1); ctx.synchronize()
page = d[:S].cpu().numpy()
pin = ctx.host_alloc(S); ctx.memcpy(pin, d.data_ptr(), S, 2); ctx.synchronize()
def t(f, n=3):
    f(); t0 = time.perf_counter()
    for _ in range(n): r = f()
    return (time.perf_counter() - t0) / n * 1e3
print("abi pinned   ms", t(lambda: ctx.run_pfac_pipeline(trie, rules, pin, S, False)))
print("abi pageable ms", t(lambda: ctx.run_pfac_pipeline(trie, rules, page.ctypes.data, S, False)))
eng = glop.Engine(pats)
print("engine pinned   ms", t(lambda: eng.run(pin, S)))
print("engine pageable ms", t(lambda: eng.run(page.ctypes.data, S)))
print("engine pageable +lines ms", t(lambda: eng.run(page.ctypes.data, S, lines=True)))
