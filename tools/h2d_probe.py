"""Pinned host->device / device->host copy bandwidth with k concurrent streams (diagnostics)."""
import torch, time
n = 28 << 20
h = torch.empty(n // 4, dtype=torch.float32).pin_memory()
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
hy = torch.empty(n // 4, dtype=torch.float32).pin_memory()
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    parts = [(i * (n // 4) // k, (i + 1) * (n // 4) // k) for i in range(k)]
    for direction in ("h2d", "d2h", "both"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for rep in range(20):
            for s, (a, b) in zip(streams, parts):
                with torch.cuda.stream(s):
                    if direction in ("h2d", "both"):
                        d[a:b].copy_(h[a:b], non_blocking=True)
                    if direction in ("d2h", "both"):
                        hy[a:b].copy_(d[a:b], non_blocking=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 20
        mult = 2 if direction == "both" else 1
        print(f"streams={k} {direction}: {mult * n / dt / 1e9:.1f} GB/s", flush=True)
