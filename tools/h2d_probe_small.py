import torch, time
dev = torch.device("cuda:0")
s = torch.cuda.Stream(dev)
for mb in (1, 2, 4, 8.7, 16, 64, 256):
    n = int(mb * (1 << 20)) // 4
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device=dev)
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(20): d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{mb:7.1f} MB one copy: {ms*1e3:8.1f} us  {mb*(1<<20)/ms/1e6:6.1f} GB/s")
    # three pieces (1/6, 1/3, 1/2 ... like mu/cov/nrm 12/24/12 of 48)
    parts = [n // 4, n // 2, n - n // 4 - n // 2]
    e0.record()
    for _ in range(20):
        o = 0
        for p in parts:
            d[o:o+p].copy_(h[o:o+p], non_blocking=True); o += p
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{mb:7.1f} MB three copies: {ms*1e3:8.1f} us  {mb*(1<<20)/ms/1e6:6.1f} GB/s")
