import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1704_02278_b200 import glop
ctx = glop.Context(0)
n = 1 << 30
pats = glop.gen_dpi_rules(10000, 606, 8, 24)
trie = ctx.upload(glop.build_failureless_trie(pats, 8)); rules = ctx.upload_rules(pats, 8)
d = torch.empty(n + 64, dtype=torch.uint8, device='cuda'); ctx.gen_payload_device(d.data_ptr(), n, 1); ctx.synchronize()
h = ctx.host_alloc(n); ctx.memcpy(h, d.data_ptr(), n, 2); ctx.synchronize()
for i in range(3):
    t = time.perf_counter(); a, c, s1 = ctx.run_pfac_pipeline(trie, rules, h, n, False); dt = time.perf_counter() - t
    print(f"e2e {dt*1e3:.1f} ms {8*n/dt/1e9:.0f} Gbps hits {s1} alerts {len(a)}", flush=True)
t = time.perf_counter(); ctx.memcpy(d.data_ptr(), h, n, 1); ctx.synchronize(); print("h2d only", (time.perf_counter()-t)*1e3, "ms")
