import torch, time
for nb in (409600, 819200, 8 << 20):
    h = torch.empty(nb, dtype=torch.uint8).pin_memory(); d = torch.empty(nb, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for name, fn in (("D2H", lambda: h.copy_(d, non_blocking=True)), ("H2D", lambda: d.copy_(h, non_blocking=True))):
        with torch.cuda.stream(s1):
            for _ in range(10): fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            for _ in range(200): fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 200
        print(f"{name} {nb/1024:.0f} KiB: {dt*1e6:.1f} us, {nb/dt/1e9:.1f} GB/s")

# concurrent: H2D 400 KiB on one stream and D2H 800 KiB on another (the headline e2e pattern)
hi = torch.empty(409600, dtype=torch.uint8).pin_memory(); di = torch.empty(409600, dtype=torch.uint8, device="cuda")
ho = torch.empty(819200, dtype=torch.uint8).pin_memory(); do = torch.empty(819200, dtype=torch.uint8, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    with torch.cuda.stream(sa): di.copy_(hi, non_blocking=True)
    with torch.cuda.stream(sb): ho.copy_(do, non_blocking=True)
torch.cuda.synchronize()
print(f"concurrent H2D 400 KiB + D2H 800 KiB: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us per pair")
