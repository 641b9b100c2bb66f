"""Pinned host->device copy bandwidth for an 80 MB buffer (the e2e leg's
per-step logits upload) with 1-8 concurrent chunks on separate streams."""
import torch, time
n = 80_000_000
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for chunks in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(chunks)]
    torch.cuda.synchronize()
    for it in range(3):
        t0 = time.perf_counter()
        for r in range(20):
            for i, s in enumerate(streams):
                with torch.cuda.stream(s):
                    a, b = i * n // chunks, (i + 1) * n // chunks
                    d[a:b].copy_(h[a:b], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"chunks={chunks}: {20 * n / dt / 1e9:.1f} GB/s")
