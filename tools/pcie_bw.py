import torch, time
for n in (6_220_800, 24_883_200, 99_532_800):
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True); d = torch.empty(n, dtype=torch.uint8, device='cuda')
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True); d2 = torch.empty(n, dtype=torch.uint8, device='cuda')
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3): d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    h2d = n*10/e0.elapsed_time(e1)/1e6
    e0.record()
    for _ in range(10): h2.copy_(d2, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    d2h = n*10/e0.elapsed_time(e1)/1e6
    torch.cuda.synchronize(); t=time.perf_counter()
    with torch.cuda.stream(s1):
        for _ in range(10): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        for _ in range(10): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); both = n*10/(time.perf_counter()-t)/1e9
    print(f"{n/1e6:.1f} MB: h2d {h2d:.1f} GB/s d2h {d2h:.1f} GB/s concurrent each {both:.1f} GB/s")
