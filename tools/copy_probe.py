"""GPU-side cost of the e2e copies (development helper): 3 H2D + 4 D2H vs merged."""
import torch, numpy as np
s = torch.cuda.Stream()
def pin(n, dt): return torch.empty(n, dtype=dt).pin_memory()
h_nn, h_nb, h_dp = pin(2000, torch.int32), pin(52000, torch.int32), pin(156000, torch.float64)
d_nn, d_nb, d_dp = (t.cuda() for t in (h_nn, h_nb, h_dp))
h_f, h_e, h_t, h_r = pin(6000, torch.float64), pin(2000, torch.float64), pin(1, torch.float64), pin(1, torch.int32)
d_f, d_e, d_t, d_r = (t.cuda() for t in (h_f, h_e, h_t, h_r))
h_all, d_all = pin(8002, torch.float64), torch.zeros(8002, dtype=torch.float64, device='cuda')
def t(fn, R=200):
    with torch.cuda.stream(s):
        for _ in range(5): fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(R): fn()
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / R * 1e3
h2d = lambda: (d_nn.copy_(h_nn, non_blocking=True), d_nb.copy_(h_nb, non_blocking=True), d_dp.copy_(h_dp, non_blocking=True))
d2h4 = lambda: (h_r.copy_(d_r, non_blocking=True), h_f.copy_(d_f, non_blocking=True), h_e.copy_(d_e, non_blocking=True), h_t.copy_(d_t, non_blocking=True))
d2h1 = lambda: h_all.copy_(d_all, non_blocking=True)
print(f"3 H2D (1.46 MB): {t(h2d):.1f} us   4 D2H (64 KB): {t(d2h4):.1f} us   1 D2H (64 KB): {t(d2h1):.1f} us")
