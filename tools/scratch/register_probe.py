"""Scratch: cudaHostRegister throughput of a pageable buffer, sliced over T threads."""
import ctypes, glob, sys, threading, time
import numpy as np, torch

N = int(float(sys.argv[1])) if len(sys.argv) > 1 else 4_000_000_000
torch.cuda.init()
lib = ctypes.CDLL(sorted(glob.glob("/usr/local/cuda/lib64/libcudart.so*"))[0])
host = np.empty(N, np.uint8); host[:] = 7
base = host.ctypes.data
for T in (1, 4, 8, 16):
    per = (N // T) & ~4095
    rc = [0] * T
    def reg(i):
        lo = i * per; n = per if i < T - 1 else N - lo
        rc[i] = lib.cudaHostRegister(ctypes.c_void_p(base + lo), ctypes.c_size_t(n), 0)
    def unreg(i):
        lib.cudaHostUnregister(ctypes.c_void_p(base + i * per))
    t = time.perf_counter(); ths = [threading.Thread(target=reg, args=(i,)) for i in range(T)]
    [x.start() for x in ths]; [x.join() for x in ths]; dt = time.perf_counter() - t
    t = time.perf_counter(); ths = [threading.Thread(target=unreg, args=(i,)) for i in range(T)]
    [x.start() for x in ths]; [x.join() for x in ths]; du = time.perf_counter() - t
    print("T=%2d register %.1f GB/s (rc %s) unregister %.1f GB/s" % (T, N / dt / 1e9, set(rc), N / du / 1e9), flush=True)
