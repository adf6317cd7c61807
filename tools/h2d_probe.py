import torch, time
n = 590 * 1024 * 1024
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for chunk in (8 << 20, 64 << 20, n):
    for streams in (1, 2, 4):
        ss = [torch.cuda.Stream() for _ in range(streams)]
        torch.cuda.synchronize()
        t = time.perf_counter()
        for rep in range(3):
            for i, off in enumerate(range(0, n, chunk)):
                st = ss[i % streams]
                with torch.cuda.stream(st):
                    d[off:off + chunk].copy_(h[off:off + chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 3
        print(f"chunk {chunk>>20} MB streams {streams}: {n/dt/1e9:.1f} GB/s")
