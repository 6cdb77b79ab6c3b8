"""GPU-side vs wall time of one end-to-end step (development helper)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2011_12875_b200 as snap

p = snap.bcc_problem(10, 10, 10, 8)
eng = snap.SnapEngine.for_problem(p)
s = torch.cuda.Stream()
eng.set_stream(s.cuda_stream)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
nn, nb, dp = pin(p.numneigh), pin(p.nbr), pin(p.disp)
f = pin(np.zeros((p.natoms, 3))); e = pin(np.zeros(p.natoms)); t = pin(np.zeros(1))
for _ in range(10): eng.step(nn, nb, dp, forces=f, eatom=e, etotal=t)
R = 200
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(R)]
w = []
for r in range(R):
    t0 = time.perf_counter()
    ev[r][0].record(s)
    eng.step(nn, nb, dp, forces=f, eatom=e, etotal=t)
    ev[r][1].record(s)
    w.append(time.perf_counter() - t0)
torch.cuda.synchronize()
g = [a.elapsed_time(b) * 1e3 for a, b in ev]
print(f"wall {np.median(w)*1e6:.1f} us  gpu(events around step) {np.median(g):.1f} us")
t0 = time.perf_counter()
for r in range(R): eng.step(nn, nb, dp, forces=f, eatom=e, etotal=t)
print(f"loop wall per step {(time.perf_counter()-t0)/R*1e6:.1f} us")
# decomposition on the engine stream: torch copies + graph replay
d_nn = torch.from_numpy(nn).cuda(); d_nb = torch.from_numpy(nb).cuda(); d_dp = torch.from_numpy(dp).cuda()
h_nn, h_nb, h_dp = (torch.from_numpy(a) for a in (nn, nb, dp))
def seq():
    with torch.cuda.stream(s):
        d_nn.copy_(h_nn, non_blocking=True); d_nb.copy_(h_nb, non_blocking=True); d_dp.copy_(h_dp, non_blocking=True)
    eng.run()
for name, fn in (("graph only", lambda: eng.run()), ("3 H2D + graph", seq)):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(R): fn()
    b.record(s)
    torch.cuda.synchronize()
    print(f"{name}: {a.elapsed_time(b) / R * 1e3:.1f} us per step (GPU)")
