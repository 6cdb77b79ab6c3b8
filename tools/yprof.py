"""Per-row cycle profile of k_compute_Y_cwin (SNAP_Y_PROFILE build) vs the plan's cost model."""
import ctypes as C, sys
import numpy as np
sys.path.insert(0, '.')
import paper_2011_12875_b200 as snap
if len(sys.argv) > 1 and sys.argv[1].startswith("--lib="):  # the SNAP_Y_PROFILE build
    snap.LIB_PATH = sys.argv.pop(1)[6:]

nx, ny, nz = (int(x) for x in sys.argv[1:4])
parts = int(sys.argv[4]) if len(sys.argv) > 4 else 0
T = 8
p = snap.bcc_problem(nx, ny, nz, twojmax=T)
eng = snap.SnapEngine.for_problem(p)
eng.set_problem(p)
if parts: eng.tune(parts)
eng.enable_stage_timing(True)  # direct launches (the profile buffer is allocated lazily)
eng.run(); eng.synchronize()
L = snap.library()
buf = (C.c_longlong * 64)()
L.snapgpu_debug_yprof(buf, 64)          # reset after warm-up
reps = 3
for _ in range(reps):
    eng.run()
eng.synchronize()
L.snapgpu_debug_yprof(buf, 64)
ntiles = (p.natoms + 31) // 32
rows = [(j, mb) for j in range(T + 1) for mb in range(j // 2 + 1)]
cyc = np.array(buf[:len(rows)], dtype=float) / (reps * ntiles)
# model (tables.cpp ycoop_pair_plan)
tuples = [(j1, j2, j) for j1 in range(T + 1) for j2 in range(j1 + 1) for j in range(j1 - j2, min(j1 + j2, T) + 1, 2)]
model, units, steps = [], [], []
for (j, mb) in rows:
    nout = j // 2 + 1 if 2 * mb == j else j + 1
    c = 0.0; nu = 0; ns = 0
    for (j1, j2, jj) in tuples:
        if jj != j: continue
        D = (j1 + j2 - j) // 2
        lo, hi = max(0, mb + D - j2), min(j1, mb + D)
        for mb1 in range(lo, hi + 1, 2):
            g = 2 if mb1 + 1 <= hi else 1
            c += (j2 + 1) * ((10 if g == 2 else 6) * nout + 8) + (60 if g == 2 else 40)
            nu += 1; ns += j2 + 1
    model.append(c); units.append(nu); steps.append(ns)
model = np.array(model)
print("row   cycles/tile  model  ratio  units steps")
for (j, mb), cy, m, u, s in zip(rows, cyc, model, units, steps):
    print(f"({j},{mb})  {cy:10.0f} {m:8.0f} {cy/m:6.2f} {u:4d} {s:4d}")
# least squares: cycles ~ a*model + b*units + c
A = np.stack([model, np.array(units, float), np.ones(len(rows))], 1)
coef, *_ = np.linalg.lstsq(A, cyc, rcond=None)
print("fit cycles = %.3f*model + %.1f*units + %.1f" % tuple(coef))
print("total cycles per tile (all groups)", cyc.sum())
nct = buf[61]
print("CTAs", nct / reps, "prologue cycles/CTA", buf[60] / max(1, nct), "CTA total cycles/CTA", buf[62] / max(1, nct))
ph = np.array(buf[40:44], dtype=float)
print("row phases (warp-cycles, share): units %.1f%%  wait1 %.1f%%  reduce+store %.1f%%  wait2 %.1f%%" %
      tuple(100 * ph / ph.sum()))
