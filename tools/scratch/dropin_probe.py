"""Scratch: split of the drop-in run_engine_scan time on pageable text."""
import os, sys, time
os.environ.setdefault("GLOP_ENGINE_TIMING", "1")
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1704_02278_b200 import glop
N = int(float(sys.argv[1])) if len(sys.argv) > 1 else 8_000_000_000
pats = glop.gen_rules(1000, 606)[0]
ctx = glop.Context(0)
import torch
d = torch.empty(N + 64, dtype=torch.uint8, device="cuda")
ctx.gen_syslog_device(d.data_ptr(), N, 1); ctx.synchronize()
host = d[:N].cpu().numpy()
eng = glop.Engine(pats)
eng.run(host.ctypes.data, N)
for _ in range(3):
    t = time.perf_counter(); a, _, s1 = eng.run(host.ctypes.data, N); dt = time.perf_counter() - t
    print("total %.1f ms  %.1f Gbps  alerts %d" % (dt * 1e3, 8 * N / dt / 1e9, len(a)), flush=True)
