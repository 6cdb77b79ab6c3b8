"""Every engine kernel once, small problems, for compute-sanitizer
(tests/test_sanitizers.py): memcheck / racecheck / synccheck / initcheck."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2011_12875_b200 as snap  # noqa: E402


def log(*a):
    print("sanitize_step:", *a, flush=True)


def exercise(p, parts=(0,)):
    with snap.SnapEngine.for_problem(p) as eng:
        eng.set_problem(p)
        eng.compute_U()
        eng.compute_Y()
        eng.compute_fused_dE()
        eng.scatter_forces()
        f = eng.forces()
        log("staged")
        for yp in parts:
            eng.tune(y_parts=yp)
            eng.run()
            eng.synchronize()
            log("graph run, y_parts", yp)
        eng.virial()
        eng.descriptors()
        log("virial, descriptors")
        f2, e, t = eng.step(p.numneigh, p.nbr, p.disp)
        log("one-call step")
        assert np.isfinite(f).all() and np.isfinite(f2).all() and np.isfinite(t)
        if p.positions is not None:
            eng.set_positions(p.positions, p.box)
            eng.run()


exercise(snap.bcc_problem(3, 3, 3, twojmax=8), parts=(1, 2))
exercise(snap.bcc_problem(3, 3, 3, twojmax=14))
exercise(snap.bcc_problem(3, 3, 3, twojmax=5))
print("sanitize_step: done")
