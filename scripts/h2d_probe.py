import torch, time
n = 320_000_000 // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True); h.normal_()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        k = n // streams
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i*k:(i+1)*k].copy_(h[i*k:(i+1)*k], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"H2D {streams} streams: {dt*1e3:.2f} ms {n*8/dt/1e9:.1f} GB/s")
torch.cuda.synchronize(); t = time.perf_counter(); h.copy_(d); torch.cuda.synchronize(); dt = time.perf_counter()-t
print(f"D2H: {dt*1e3:.2f} ms {n*8/dt/1e9:.1f} GB/s")
