"""compute_Y stage time vs the y_parts knob (development helper): tune_time.py [--lib=...] NX NY NZ P..."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2011_12875_b200 as snap
if len(sys.argv) > 1 and sys.argv[1].startswith("--lib="):
    snap.LIB_PATH = sys.argv.pop(1)[6:]
nx, ny, nz = (int(x) for x in sys.argv[1:4])
p = snap.bcc_problem(nx, ny, nz, twojmax=8)
eng = snap.SnapEngine.for_problem(p)
eng.set_problem(p)
for yp in [int(x) for x in sys.argv[4:]]:
    eng.tune(y_parts=yp)
    eng.enable_stage_timing(True)
    for _ in range(3): eng.run()
    ys = []
    for _ in range(10):
        eng.run(); ys.append(eng.stage_times()["Y"])
    print(f"N={p.natoms} y_parts={yp} Y {np.median(ys)*1e3:.1f} us", flush=True)
