"""Bounds-checked build vs the product build (compute-sanitizer is closed on
the GPU pool): run small problems through a build made with
`make OUT=../_build_bc EXTRA=-DSNAP_BOUNDS_CHECK` (device asserts on every
shared-memory / C' index range of the item-pair compute_Y quad units) and
save forces / energies; a second run with the product build must give the
same bits.
    python tools/bounds_check.py _build_bc out_bc.npz
    python tools/bounds_check.py _build out.npz
    python tools/bounds_check.py --compare out_bc.npz out.npz"""
import sys

import numpy as np

sys.path.insert(0, ".")
if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print("bounds_check: %d arrays, %d differ %s" % (len(a.files), len(bad), bad))
    sys.exit(1 if bad else 0)
import paper_2011_12875_b200 as snap

snap.LIB_PATH = "paper_2011_12875_b200/%s/libsnapgpu.so" % sys.argv[1]
out = {}
for T in range(9, 15):
    for cells in ((3, 3, 3), (4, 4, 4), (4, 4, 7)):
        p = snap.bcc_problem(*cells, twojmax=T)
        r = snap.run_pipeline(p, device=0)
        key = "T%d_%d%d%d" % ((T,) + cells)
        out[key + "_f"] = r.forces
        out[key + "_e"] = np.asarray([r.etotal])
        print(key, r.etotal, flush=True)
np.savez(sys.argv[2], **out)
print("bounds_check: done")
