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
