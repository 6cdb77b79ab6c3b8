"""Quick device timing of the force step (development helper)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_2011_12875_b200 as snap
if len(sys.argv) > 1 and sys.argv[1].startswith("--lib="):  # A/B builds (make OUT=... EXTRA=...)
    snap.LIB_PATH = sys.argv.pop(1)[6:]

def run(nx, ny, nz, T=8, reps=10, tune=None):
    p = snap.bcc_problem(nx, ny, nz, twojmax=T)
    eng = snap.SnapEngine.for_problem(p)
    eng.set_problem(p)
    if tune: eng.tune(*tune)
    eng.enable_stage_timing(True)
    for _ in range(3): eng.run()
    st = {k: [] for k in ("U", "Y", "dE", "forces")}
    for _ in range(reps):
        eng.run()
        for k, v in eng.stage_times().items(): st[k].append(v)
    med = {k: float(np.median(v)) for k, v in st.items()}
    eng.enable_stage_timing(False)
    eng.run(); eng.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): eng.run()
    eng.synchronize()
    dt = (time.perf_counter() - t0) / reps * 1e3
    n = p.natoms
    print(f"T={T} N={n} tune={tune} stages(ms)={ {k: round(v,4) for k,v in med.items()} } step {dt:.4f} ms -> {n/dt:.1f} Katom-steps/s, {dt*1e6/n:.2f} ns/atom", flush=True)
    eng.close()

if __name__ == "__main__":
    for spec in sys.argv[1:]:
        f = [int(x) for x in spec.split(",")]
        tune = (f[4],) if len(f) > 4 else None
        run(f[0], f[1], f[2], T=f[3], reps=10 if f[0]*f[1]*f[2] < 50000 else 3, tune=tune)
