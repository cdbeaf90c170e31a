"""Pinned host -> device copy bandwidth of one large buffer by chunking and stream count
(is one cudaMemcpyAsync of 16 GB the fastest way to upload C3's A?)."""
import time

import torch

GB = 4
n = GB * (1 << 30) // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for streams, chunk_mb in [(1, 0), (1, 256), (2, 256), (4, 256), (2, 64), (4, 1024), (8, 64)]:
    ss = [torch.cuda.Stream() for _ in range(streams)]
    best = 1e9
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if chunk_mb == 0:
            d.copy_(h, non_blocking=True)
        else:
            ce = chunk_mb * (1 << 20) // 8
            for i, off in enumerate(range(0, n, ce)):
                with torch.cuda.stream(ss[i % streams]):
                    d[off:off + ce].copy_(h[off:off + ce], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"{streams} stream(s), chunks of {chunk_mb or GB * 1024} MB: {GB * (1 << 30) / best / 1e9:.2f} GB/s")
