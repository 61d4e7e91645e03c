"""H2D bandwidth probe: pinned host -> device, 1 vs 2 streams, chunk sizes."""
import torch, time
n = 4 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = [torch.cuda.Stream() for _ in range(4)]
for ns in (1, 2, 4):
    for chunk in (64 << 20, 256 << 20):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i, off in enumerate(range(0, n, chunk)):
            with torch.cuda.stream(s[i % ns]):
                d[off:off + chunk].copy_(h[off:off + chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(f"streams={ns} chunk={chunk>>20}MB {n/dt/1e9:.1f} GB/s", flush=True)
