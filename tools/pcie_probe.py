import torch, time
torch.cuda.set_device(0)
n = 256 << 20  # floats = 1 GiB
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for ns in (1, 2, 4, 8):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    for _ in range(2):
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i * n // ns:(i + 1) * n // ns].copy_(h[i * n // ns:(i + 1) * n // ns], non_blocking=True)
        torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i * n // ns:(i + 1) * n // ns].copy_(h[i * n // ns:(i + 1) * n // ns], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    print(f"H2D streams={ns}: {4 * n / dt / 1e9:.1f} GB/s")
# D2H
t = time.perf_counter()
for _ in range(3):
    h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
print(f"D2H: {4 * n * 3 / (time.perf_counter() - t) / 1e9:.1f} GB/s")
