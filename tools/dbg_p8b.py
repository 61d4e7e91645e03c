import sys, numpy as np, torch
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
from paper_1704_02278_b200 import glop
import oracle_ffi as O
ctx=glop.Context(0)
def scan(trie, text, kernel):
    d=torch.from_numpy(text.copy()).cuda()
    cap=max(1<<16, 4*text.size)
    out=torch.empty(cap*16,dtype=torch.uint8,device='cuda')
    nh=ctx.pfac_scan_device(trie, d.data_ptr(), text.size, out.data_ptr(), cap, kernel=kernel)
    ctx.synchronize()
    return out[:nh*16].cpu().numpy().view(glop.HIT_DTYPE).copy()
def cmp(name, got, ref):
    if got.tobytes()==ref.tobytes(): print(name, "OK", len(ref)); return
    print(name, "MISMATCH got", len(got), "ref", len(ref))
    g=set(map(tuple,np.stack([got['offset'],got['pattern_id']],1).tolist())); r=set(map(tuple,np.stack([ref['offset'],ref['pattern_id']],1).tolist()))
    print("  extra", sorted(g-r)[:10], "missing", sorted(r-g)[:10], "dups", len(got)-len(g))
    if not (g-r) and not (r-g): 
        k=np.argmax(got['offset']!=ref['offset']) if len(got)==len(ref) else 0
        print("  order differs near", k, got[max(0,k-3):k+3], ref[max(0,k-3):k+3])
text=glop.gen_syslog_host(6<<20, seed=31)
pats,_=glop.gen_rules(300, seed=5)
pats+=[b"Failed password", b"Failed passwd", b"<38>1 2026-", b"\n<38>1 20"]
trie=ctx.upload(glop.build_failureless_trie(pats,8))
cmp("syslog", scan(trie,text,glop.PFAC_PREFIX8), O.pfac_scan(text,O.Trie(pats,8)))
dense=np.frombuffer(b"A"*70000+b"AAAAAAAAB"+b"A"*3001,np.uint8)
dp=[b"AAAAAAAAx", b"AAAAAAAAy", b"AAAAAAAB", b"AAAAAAAAB"]
dt=ctx.upload(glop.build_failureless_trie(dp,8))
cmp("dense", scan(dt,dense,glop.PFAC_PREFIX8), O.pfac_scan(dense,O.Trie(dp,8)))
pats,_=glop.gen_rules(1000, seed=606)
t2=glop.gen_syslog_host(16<<20, seed=1)
trie=ctx.upload(glop.build_failureless_trie(pats,8))
cmp("k1000", scan(trie,t2,glop.PFAC_PREFIX8), O.pfac_scan(t2,O.Trie(pats,8)))
