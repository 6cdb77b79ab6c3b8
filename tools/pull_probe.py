"""One-call steps from pinned host lists (the compute_U pull path), for
ncu launch lists (development helper): pull_probe.py [NX] [reps]."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2011_12875_b200 as snap

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 10
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
p = snap.bcc_problem(nx, nx, nx, 8)
eng = snap.SnapEngine.for_problem(p)
keep = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (p.numneigh, p.nbr, p.disp)]
args = [t.numpy() for t in keep]
f = torch.zeros((p.natoms, 3), dtype=torch.float64).pin_memory().numpy()
e = torch.zeros(p.natoms, dtype=torch.float64).pin_memory().numpy()
t = torch.zeros(1, dtype=torch.float64).pin_memory().numpy()
for _ in range(reps):
    eng.step(*args, forces=f, eatom=e, etotal=t)
print("ok", t[0])
