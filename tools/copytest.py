import torch, time
for mb in (256, 1024, 4096):
    n = mb * 2**20 // 4
    a = torch.rand(n, device="cuda"); b = torch.empty_like(a)
    for _ in range(3): b.copy_(a)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(50):
        (b.copy_(a) if i % 2 == 0 else a.copy_(b))
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 50
    print(mb, "MB copy:", round(2 * n * 4 / t / 1e6, 1), "GB/s", round(t*1e3,1), "us")
