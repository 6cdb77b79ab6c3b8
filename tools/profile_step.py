"""Run the force step a few times for ncu captures: profile_step.py NX NY NZ [T] [reps]."""
import sys
sys.path.insert(0, '.')
import paper_2011_12875_b200 as snap

nx, ny, nz = (int(x) for x in sys.argv[1:4])
T = int(sys.argv[4]) if len(sys.argv) > 4 else 8
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
p = snap.bcc_problem(nx, ny, nz, twojmax=T)
eng = snap.SnapEngine.for_problem(p)
eng.set_problem(p)
eng.enable_stage_timing(True)   # direct launches (no graph) so ncu sees each kernel
for _ in range(reps):
    eng.run()
eng.synchronize()
print("stage ms", eng.stage_times())
