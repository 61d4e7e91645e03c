import sys, numpy as np, torch
sys.path.insert(0,'.')
from paper_1704_02278_b200 import glop
ctx=glop.Context(0)
pats,_=glop.gen_rules(1000, seed=606)
trie=ctx.upload(glop.build_failureless_trie(pats,8))
for n in (1<<20, 4<<20, 16<<20, 64<<20, 256<<20):
    d=torch.empty(n+64,dtype=torch.uint8,device='cuda')
    ctx.gen_syslog_device(d.data_ptr(), n, 1)
    out=torch.empty((n//64+(1<<16))*16,dtype=torch.uint8,device='cuda')
    l0=ctx.launches
    nh=ctx.pfac_scan_device(trie, d.data_ptr(), n, out.data_ptr(), n//64+(1<<16), kernel=glop.PFAC_PREFIX8)
    ctx.synchronize()
    print(n, nh, ctx.launches-l0, flush=True)
