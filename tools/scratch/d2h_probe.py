import torch, time
dev = torch.empty(65_000_000, dtype=torch.uint8, device="cuda")
host = torch.empty(65_000_000, dtype=torch.uint8, pin_memory=True)
def run(chunk, nstreams):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize()
    best = 1e9
    for rep in range(5):
        t0 = time.perf_counter()
        i = 0
        for lo in range(0, dev.numel(), chunk):
            hi = min(lo + chunk, dev.numel())
            with torch.cuda.stream(streams[i % nstreams]):
                host[lo:hi].copy_(dev[lo:hi], non_blocking=True)
            i += 1
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return dev.numel() / best / 1e9
for chunk in (1_200_000, 1_572_864, 3_145_728, 6_291_456, 65_000_000):
    print(chunk, "1 stream %.1f GB/s" % run(chunk, 1), "2 streams %.1f GB/s" % run(chunk, 2), "3 streams %.1f GB/s" % run(chunk, 3))
