import time
import torch
n = 1 << 30   # 1 GiB
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    chunk = n // streams
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.perf_counter()
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"H2D pinned, {streams} stream(s): {n / dt / 1e9:.1f} GB/s")
t0 = time.perf_counter(); h.copy_(d); torch.cuda.synchronize(); print(f"D2H pinned: {n / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
