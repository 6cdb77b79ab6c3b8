"""Full-size parity for BASELINE.json configs C3 (2J=8, 262,144 atoms) and C4
(2J=14, 32,768 atoms), through checks whose cost does not grow with the size:

* sampled atoms: the per-atom energy E_i and the pair gradients dE(i, k)
  depend only on atom i's own neighbor list (compute_U snap_core.hpp:369-489,
  compute_Y :1085-1200, compute_fused_dE :1274-1406), so the oracle run on a
  sub-problem made of the sampled atoms' lists must reproduce the full-size
  GPU values (every tile position, including the padded last tile);
* Newton's third law on the closed periodic lattice: sum_i F_i = 0
  (oracle.hpp:224-237);
* determinism: a second run is bitwise identical (ordered reductions);
* rotation invariance (oracle.hpp:175-203): energies invariant, forces
  co-rotate with the displacements.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FTOL, ETOL = 1e-10, 1e-12


def normerr(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def snap():
    import paper_2011_12875_b200 as snap

    return snap


def _sample(n, k=48, seed=5):
    rng = np.random.default_rng(seed)
    idx = set(rng.choice(n, size=k - 4, replace=False).tolist())
    idx.update([0, 31, n - 1, (n // 32) * 32 - 1])  # tile edges and the last atom
    return np.array(sorted(i for i in idx if 0 <= i < n))


def _subproblem(p, idx):
    """The sampled atoms' own lists as a standalone problem (neighbor indices
    remapped to valid non-self atoms: E_i and dE(i, k) do not depend on them)."""
    from types import SimpleNamespace

    m = len(idx)
    S = p.nbr.shape[1]
    nbr = (np.arange(m)[:, None] + 1 + np.arange(S)[None, :]) % m
    return SimpleNamespace(twojmax=p.twojmax, rcut=p.rcut, rmin0=p.rmin0, rfac0=p.rfac0,
                           wself=p.wself, self_flag=p.self_flag, beta=p.beta,
                           weights=np.ones(1), numneigh=np.ascontiguousarray(p.numneigh[idx]),
                           nbr=np.ascontiguousarray(nbr.astype(np.int32)),
                           disp=np.ascontiguousarray(p.disp[idx]), types=None)


@pytest.mark.parametrize("cells,T", [((64, 64, 32), 8), ((32, 32, 16), 14)],
                         ids=["C3_2j8_262144", "C4_2j14_32768"])
def test_full_size_sampled_atoms_vs_oracle(snap, port, cells, T):
    p = snap.bcc_problem(*cells, twojmax=T)
    n = p.natoms
    eng = snap.SnapEngine.for_problem(p)
    eng.set_problem(p)
    eng.run()
    f = eng.forces()
    eatom, etot = eng.energy()
    dedr = eng.dedr()
    idx = _sample(n)
    ref = port.run(_subproblem(p, idx), want=("eatom", "delist"))
    assert normerr(eatom[idx], ref["eatom"]) <= ETOL
    assert normerr(dedr[idx], ref["delist"]) <= FTOL
    # closed periodic lattice: Newton's third law
    assert np.abs(f.sum(axis=0)).max() <= 1e-12 * np.abs(f).max() * np.sqrt(n)
    # total energy is the ordered sum of the per-atom energies
    assert abs(etot - float(np.sum(eatom))) <= 1e-12 * abs(etot)
    # determinism: bitwise equal forces and energies on a second run
    eng.run()
    eatom2, etot2 = eng.energy()
    assert etot2 == etot
    assert np.array_equal(eatom2, eatom)
    assert np.array_equal(eng.forces(), f)
    eng.close()


@pytest.mark.parametrize("cells,T", [((64, 64, 32), 8), ((32, 32, 16), 14)],
                         ids=["C3_2j8_262144", "C4_2j14_32768"])
def test_full_size_full_vectors_vs_reference(snap, cells, T):
    """BASELINE.json configs C3 / C4 at full size: the whole force vector,
    every per-atom energy and the total against the UNMODIFIED reference
    (oracle/_ref, run_pipeline fused-det on all host threads)."""
    import os

    import oracle

    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    p = snap.bcc_problem(*cells, twojmax=T)
    r = snap.run_pipeline(p)
    ref = oracle.Ref().run(p, "fused", True, os.cpu_count() or 1,
                           want=("forces", "eatom", "etotal"))
    assert normerr(r.forces, ref["forces"]) <= FTOL
    assert normerr(r.eatom, ref["eatom"]) <= ETOL
    assert abs(r.etotal - ref["etotal"]) <= ETOL * abs(ref["etotal"])


def test_rotation_invariance_bcc2000(snap):
    p = snap.bcc_problem(10, 10, 10, twojmax=8)
    base = snap.run_pipeline(p)
    rng = np.random.default_rng(7)
    q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    pr = snap.Problem.from_any(p)
    pr.disp = np.ascontiguousarray(p.disp @ q.T)
    rot = snap.run_pipeline(pr)
    assert normerr(rot.eatom, base.eatom) <= 1e-10
    assert normerr(rot.forces, base.forces @ q.T) <= 1e-10


def test_virial_from_delist_vs_oracle(snap, port):
    """W_ab = sum_{i,k} r_ik,a (-dE_ik,b) from the device dElist
    equals the same contraction of the oracle's dElist."""
    from conftest import load_golden

    for name in ("bcc54_2j8", "cluster_n6_2j8_s910_t1", "bcc54_2j14"):
        p, out, _ = load_golden(name)
        eng = snap.SnapEngine.for_problem(p)
        eng.set_problem(snap.Problem.from_any(p))
        eng.run()
        w = eng.virial()
        nn = np.asarray(p.numneigh)
        mask = (np.arange(p.nbr.shape[1])[None, :] < nn[:, None])[..., None]
        r = np.asarray(p.disp) * mask
        d = np.asarray(out["delist"]) * mask
        ref = -np.array([(r[..., 0] * d[..., 0]).sum(), (r[..., 1] * d[..., 1]).sum(),
                         (r[..., 2] * d[..., 2]).sum(), (r[..., 0] * d[..., 1]).sum(),
                         (r[..., 0] * d[..., 2]).sum(), (r[..., 1] * d[..., 2]).sum()])
        assert normerr(w, ref) <= FTOL, name
        eng.close()


@pytest.mark.parametrize("cells,jitter,seed", [((3, 3, 3), 0.05, 1), ((10, 10, 10), 0.05, 2011),
                                               ((5, 4, 3), 0.3, 9), ((64, 64, 32), 0.05, 2011)])
def test_device_neighbor_lists_bitwise_and_forces(snap, cells, jitter, seed):
    """lists built on the GPU from positions equal the host
    builder's (harness.hpp:119-202 restatement) bit for bit, and the force
    step on them matches the step on uploaded lists."""
    p = snap.bcc_problem(*cells, twojmax=8, seed=seed, jitter=jitter)
    eng = snap.SnapEngine.for_problem(p)
    eng.set_positions(p.positions, p.box)
    nn, nbr, disp = eng.neighbors()
    S = p.nbr.shape[1]
    assert nbr.shape[1] == S
    assert np.array_equal(nn, p.numneigh)
    mask = np.arange(S)[None, :] < nn[:, None]
    assert np.array_equal(np.where(mask, nbr, 0), np.where(mask, p.nbr, 0))
    assert np.array_equal(np.where(mask[..., None], disp, 0.0),
                          np.where(mask[..., None], p.disp, 0.0))
    if p.natoms <= 20000:
        eng.run()
        ref = snap.run_pipeline(p)
        assert np.array_equal(eng.forces(), ref.forces)  # same lists: bitwise
        assert eng.energy()[1] == ref.etotal
    eng.close()


def test_descriptors_vs_oracle_blist(snap, port):
    """B_l(i) (compute_B_from_U, snap_core.hpp:642-681) from
    the one-pass k_compute_B equals the oracle's blist at 2J = 4, 5, 8, 14
    (typed clusters included) and satisfies E_i = sum_l beta_l B_l."""
    from conftest import load_golden

    for name in ("cluster_n6_2j8_s910_t1", "bcc54_2j8", "cluster_n5_2j4_s906_t1",
                 "bcc54_2j14", "cluster_n7_2j5_s915_t3", "cluster_n4_2j14_s914_t1"):
        p, out, _ = load_golden(name)
        pr = snap.Problem.from_any(p)
        eng = snap.SnapEngine.for_problem(pr)
        eng.set_problem(pr)
        b = eng.descriptors()
        ref = port.run(pr, want=("blist",))["blist"]
        assert normerr(b, ref) <= 1e-11, name
        assert np.array_equal(eng.descriptors(), b)  # deterministic
        # energy identity E_i = sum_l beta_l B_l (compute_energy, snap_core.hpp:684-701)
        eng.run()
        e, _ = eng.energy()
        assert normerr(b @ np.asarray(pr.beta), e) <= 1e-11, name
        assert normerr(eng.forces(), out["forces"]) <= FTOL
        eng.close()


def test_report_row_schema_and_checksum(snap, port):
    """a gpu row in the reference RunReport schema; the
    checksum is the reference's (acceptance gate value on the oracle forces)."""
    from paper_2011_12875_b200 import report

    q = port.synthetic(64, 14, 8, seed=600)
    assert report.checksum_hex(port.run(q, want=("forces",))["forces"]) == "dd6d6cc7a1c2e358"
    p = snap.bcc_problem(4, 4, 4, twojmax=8)
    row = report.gpu_row(p, steps=3)
    csv = report.write_report_csv([row])
    head = csv.splitlines()[0]
    assert head.startswith(report.CSV_HEADER)
    assert csv.splitlines()[1].startswith("gpu-b200,128,")
    assert row["ok"] and row["katom_steps_per_s"] > 0 and len(row["force_checksum"]) == 16
