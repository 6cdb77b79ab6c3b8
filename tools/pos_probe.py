"""Per-kernel times of the one-call positions step (run under ncu --metrics gpu__time_duration.sum)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2011_12875_b200 as snap
if len(sys.argv) > 1 and sys.argv[1].startswith("--lib="):  # A/B builds
    snap.LIB_PATH = sys.argv.pop(1)[6:]

p = snap.bcc_problem(10, 10, 10, twojmax=8)
with snap.SnapEngine.for_problem(p) as eng:
    for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
        eng.step_positions(p.positions, p.box)
