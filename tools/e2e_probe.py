"""Break down the host-side cost of one end-to-end step (development helper)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2011_12875_b200 as snap

p = snap.bcc_problem(10, 10, 10, 8)
eng = snap.SnapEngine.for_problem(p)
nn = torch.from_numpy(np.ascontiguousarray(p.numneigh)).pin_memory().numpy()
nb = torch.from_numpy(np.ascontiguousarray(p.nbr)).pin_memory().numpy()
dp = torch.from_numpy(np.ascontiguousarray(p.disp)).pin_memory().numpy()
f = torch.zeros((p.natoms, 3), dtype=torch.float64).pin_memory().numpy()
eng.set_neighbors(nn, nb, dp); eng.run(); eng.synchronize()
def t(fn, n=200):
    fn(); eng.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    eng.synchronize()
    return (time.perf_counter() - t0) / n * 1e6
print("set_neighbors   us", t(lambda: eng.set_neighbors(nn, nb, dp)))
print("run (graph)     us", t(lambda: eng.run()))
print("forces D2H      us", t(lambda: eng.forces(f)))
print("energy          us", t(lambda: eng.energy()))
def full():
    eng.set_neighbors(nn, nb, dp); eng.run(); eng.forces(f); eng.energy()
print("full e2e step   us", t(full))
ff=np.zeros((p.natoms,3)); ee=np.zeros(p.natoms); tt=np.zeros(1)
print("step() one call us", t(lambda: eng.step(nn, nb, dp, forces=f, eatom=ee, etotal=tt)))
print("sync only       us", t(lambda: eng.synchronize()))
