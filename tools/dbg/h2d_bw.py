import torch, time
n = 2 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for chunks, nstreams in [(1, 1), (8, 1), (8, 2), (16, 4)]:
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize()
    for rep in range(2):
        t = time.perf_counter()
        cs = n // chunks
        for c in range(chunks):
            with torch.cuda.stream(streams[c % nstreams]):
                d[c * cs:(c + 1) * cs].copy_(h[c * cs:(c + 1) * cs], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"chunks {chunks} streams {nstreams}: {n / dt / 1e9:.1f} GB/s")
