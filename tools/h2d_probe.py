"""PCIe H2D throughput from pinned memory: one stream vs several concurrent streams."""
import time

import torch

N = 64 << 20  # 64 MB chunks (bf16 elements x2 bytes below)
chunks = 36
host = [torch.empty(N // 2, dtype=torch.bfloat16).pin_memory() for _ in range(4)]
dev = [torch.empty(N // 2, dtype=torch.bfloat16, device="cuda") for _ in range(4)]
for ns in (1, 2, 3, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(chunks):
            s = streams[i % ns]
            with torch.cuda.stream(s):
                dev[i % 4].copy_(host[i % 4], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"streams {ns}: {chunks * N / dt / 1e9:.1f} GB/s")
# D2H concurrently with H2D
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
hout = torch.empty(N // 2, dtype=torch.bfloat16).pin_memory()
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(chunks):
    with torch.cuda.stream(s1):
        dev[i % 4].copy_(host[i % 4], non_blocking=True)
    if i % 7 == 0:
        with torch.cuda.stream(s2):
            hout.copy_(dev[(i + 1) % 4], non_blocking=True)
torch.cuda.synchronize()
print(f"H2D with concurrent D2H: {chunks * N / (time.perf_counter() - t0) / 1e9:.1f} GB/s (H2D bytes only)")
