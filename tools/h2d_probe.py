import torch, time
for mb in (0.2, 1.25, 4, 32):
    n = int(mb * 1e6 / 8)
    h = torch.randn(n, dtype=torch.float64).pin_memory()
    d = torch.empty(n, dtype=torch.float64, device='cuda')
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); R = 50
    for _ in range(R): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / R
    print(f"H2D {mb} MB: {dt*1e6:.1f} us  {mb*1e6/dt/1e9:.1f} GB/s")
