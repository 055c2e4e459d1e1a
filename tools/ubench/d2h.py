import torch, time
d = torch.randn(6647296, device="cuda")
for pin in (True,):
    h = torch.empty(6647296, pin_memory=pin)
    for sz in (1<<20, 8<<20, 26588):
        pass
    for i in range(3):
        torch.cuda.synchronize(); t=time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
        print("d2h 26.6MB", dt*1e3, "ms", d.numel()*4/dt/1e9, "GB/s")
    for i in range(3):
        torch.cuda.synchronize(); t=time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
        print("h2d 26.6MB", dt*1e3, "ms", d.numel()*4/dt/1e9, "GB/s")
    # chunked on 2 streams
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    n = d.numel(); k = n // 4
    for i in range(3):
        torch.cuda.synchronize(); t=time.perf_counter()
        for j in range(4):
            with torch.cuda.stream(s1 if j % 2 == 0 else s2):
                h[j*k:(j+1)*k].copy_(d[j*k:(j+1)*k], non_blocking=True)
        torch.cuda.synchronize(); dt=time.perf_counter()-t
        print("d2h 4 chunks 2 streams", dt*1e3, "ms", n*4/dt/1e9, "GB/s")
