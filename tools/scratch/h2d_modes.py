"""Host->device modes for pageable text (scratch probe): driver pageable copy,
cudaHostRegister in place, threaded staging memcpy bandwidth."""
import ctypes, os, sys, time, threading
import numpy as np, torch

N = int(float(sys.argv[1])) if len(sys.argv) > 1 else 8_000_000_000
host = np.empty(N, np.uint8); host[::4096] = 1; host[:] = 7  # touched, pageable
dev = torch.empty(N, dtype=torch.uint8, device="cuda")
rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
def tm(f, reps=2):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter(); f(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    return best
src = torch.from_numpy(host)
print("pageable copy_ : %.1f GB/s" % (N / tm(lambda: dev.copy_(src)) / 1e9), flush=True)
cr = torch.cuda.cudart()
def reg():
    assert cr.cudaHostRegister(host.ctypes.data, N, 0) == 0
def unreg():
    assert cr.cudaHostUnregister(host.ctypes.data) == 0
t = time.perf_counter(); reg(); t1 = time.perf_counter(); print("register: %.1f ms (%.1f GB/s)" % ((t1-t)*1e3, N/(t1-t)/1e9), flush=True)
print("registered copy: %.1f GB/s" % (N / tm(lambda: dev.copy_(src, non_blocking=True)) / 1e9), flush=True)
t = time.perf_counter(); unreg(); print("unregister: %.1f ms" % ((time.perf_counter()-t)*1e3), flush=True)
pin = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True).numpy()
for nt in (1, 4, 8, 16):
    per = (1 << 30) // nt
    def job(i):
        for r in range(N // (1 << 30)):
            np.copyto(pin[i*per:(i+1)*per], host[r*(1<<30)+i*per: r*(1<<30)+(i+1)*per])
    def run():
        ts = [threading.Thread(target=job, args=(i,)) for i in range(nt)]
        [x.start() for x in ts]; [x.join() for x in ts]
    print("staging memcpy %2d threads: %.1f GB/s" % (nt, (N // (1<<30)) * (1<<30) / tm(run, 1) / 1e9), flush=True)
