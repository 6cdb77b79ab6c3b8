"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Every array here comes out of oracle/_ref/libsnapref.so, i.e. the reference's
own code compiled from /root/reference/proj/include by oracle/Makefile:
problem generators (harness.hpp:230-262 generate_synthetic,
tests/test_support.hpp:21-64 make_cluster, harness.hpp:119-202
build_neighborlist) and the deterministic pipeline stages
(snap_core.hpp compute_U / compute_B_from_U+compute_energy / compute_Y /
compute_fused_dE / scatter_forces, the `fused` variant of
exec_variants.hpp:153-167).  The BCC lattice positions are our generator
(oracle/snap_oracle.c orc_bcc) -- the reference has none -- but the neighbor
lists and every output are the reference's.

The fixtures are small (<1 MB total) so they travel with the repo to the GPU
box, where /root/reference does not exist.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

FULL = ("forces", "eatom", "etotal", "ulisttot", "ylist", "delist")
LIGHT = ("forces", "eatom", "etotal", "delist")


def save(name, prob, res, extra=None):
    d = dict(
        twojmax=prob.twojmax, rcut=prob.rcut, rmin0=prob.rmin0, rfac0=prob.rfac0,
        wself=prob.wself, self_flag=prob.self_flag, beta=prob.beta,
        weights=np.asarray(prob.weights, np.float64),
        numneigh=prob.numneigh, nbr=prob.nbr, disp=prob.disp,
    )
    if getattr(prob, "types", None) is not None:
        d["types"] = prob.types
    if getattr(prob, "positions", None) is not None:
        d["positions"] = prob.positions
    if getattr(prob, "box", None) is not None:
        d["box"] = prob.box
    for k, v in res.items():
        d["out_" + k] = np.asarray(v)
    if extra:
        d.update(extra)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)


def main():
    oracle.build()
    R = oracle.Ref()
    P = oracle.Port()

    # BCC tungsten 3x3x3 cells (54 atoms, exactly 26 neighbors), 2J=8.
    pos, beta, box = P.bcc(3, 3, 3, 8)
    numneigh, nbr, disp = R.neighborlist(pos, box[0], 4.7)
    bcc = oracle.SimpleNamespace(twojmax=8, rcut=4.7, rmin0=0.0, rfac0=0.99363,
                                 wself=1.0, self_flag=1, beta=beta, weights=np.ones(1),
                                 types=None, positions=pos, box=box, numneigh=numneigh,
                                 nbr=nbr, disp=disp)
    save("bcc54_2j8", bcc, R.run(bcc, "fused", True, 4, FULL))

    # Same lattice at 2J=14 (forces / energies / dElist only: keeps it small).
    pos14, beta14, _ = P.bcc(3, 3, 3, 14)
    bcc14 = oracle.SimpleNamespace(**{**vars(bcc), "twojmax": 14, "beta": beta14})
    save("bcc54_2j14", bcc14, R.run(bcc14, "fused", True, 8, LIGHT))

    # Ragged all-pairs clusters (tests/test_support.hpp), several band limits,
    # including a two-type weight table.
    for (n, T, seed, nt) in [(6, 8, 910, 1), (4, 6, 905, 2), (5, 4, 906, 1),
                             (5, 2, 908, 1), (3, 0, 903, 1), (4, 14, 914, 1),
                             (7, 5, 915, 3)]:
        c = R.make_cluster(n, T, seed, nt)
        save(f"cluster_n{n}_2j{T}_s{seed}_t{nt}", c, R.run(c, "fused", True, 2, FULL))

    # Fixed-shape synthetic lists (harness.hpp:230-262), non-mirrored.
    s = R.synthetic(40, 26, 8, seed=12345)
    save("synthetic_n40_k26_2j8", s, R.run(s, "fused", True, 4, FULL))

    # The acceptance gate's determinism problem (acceptance.cpp:249-275):
    # 64 atoms x 14 synthetic neighbors, 2J=8, seed 600; the reference's
    # staged-ladder force checksum is dd6d6cc7a1c2e358.
    s6 = R.synthetic(64, 14, 8, seed=600)
    save("synthetic_n64_k14_2j8_s600", s6, R.run(s6, "v1", True, 4, LIGHT),
         extra={"fnv_checksum": np.array("dd6d6cc7a1c2e358")})

    # Problem files written by the reference's own save_problem
    # (harness.hpp:698-780, schema 1): the BCC lattice with positions and
    # its cubic box, and a typed ragged cluster.
    R.save_problem(bcc, os.path.join(HERE, "bcc54_2j8.problem.json"), seed=2011,
                   box_length=float(box[0]))
    c7 = R.make_cluster(7, 5, 915, 3)
    R.save_problem(c7, os.path.join(HERE, "cluster_n7_2j5_s915_t3.problem.json"), seed=915)

    # Known-answer tables.
    tabs = {}
    for T in (0, 2, 4, 8, 14):
        tabs[f"counts_{T}"] = np.array(R.counts(T), np.int32)
    tabs["cg_8"] = R.cg_table(8)
    rng = np.random.default_rng(5)
    dirs = rng.normal(size=(16, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    disps = dirs * (4.7 * rng.uniform(0.3, 0.95, size=(16, 1)))
    tabs["wigner_disp"] = disps
    tabs["wigner_u8"] = np.stack([R.wigner_u_half(d, 8) for d in disps])
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **tabs)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
