"""Deterministic forces and finite-difference forces on the GPU.

* scatter_forces' deterministic mode (snap_core.hpp:889-899; pipeline.hpp
  :269-272) walks the pairs serially, F_i += dE(i,k), F_nbr -= dE(i,k).  The
  engine's force gather pulls the same terms in the same order, so its forces
  must equal that serialized sum of the engine's own dElist BITWISE, and be
  bitwise stable run to run and context to context (README.md:111-118: "the
  force checksum is bitwise stable across runs").
* finite differences (oracle.hpp:133-172, tests/test_oracle.cpp:137-144):
  forces are -dE_total/dx by central differences of the GPU total energy,
  step h = 1e-6 Rcut (tolerances.hpp:32), elementwise rel_err <= 1e-5
  (tolerances.hpp:41, floor 1e-14 :83), neighbor displacements rebuilt per
  evaluation keeping the original pairs inside Rcut (oracle.hpp:101-122).
"""
import numpy as np
import pytest

from conftest import fnv1a

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def snap():
    import paper_2011_12875_b200 as snap

    return snap


def serialized_scatter(nbr, numneigh, dedr, natoms):
    """snap_core.hpp:889-899 in the same floating-point order."""
    f = np.zeros((natoms, 3))
    for i in range(numneigh.shape[0]):
        for k in range(int(numneigh[i])):
            de = dedr[i, k]
            j = nbr[i, k]
            for d in range(3):
                f[i, d] += de[d]
                f[j, d] -= de[d]
    return f


@pytest.mark.parametrize("cells,T", [((10, 10, 10), 8), ((3, 3, 3), 14), ((4, 4, 4), 5)])
def test_forces_are_the_serialized_scatter_of_dedr(snap, cells, T):
    p = snap.bcc_problem(*cells, twojmax=T)
    with snap.SnapEngine.for_problem(p) as eng:
        eng.set_problem(p)
        eng.run()
        f = eng.forces()
        ref = serialized_scatter(p.nbr, p.numneigh, eng.dedr(), p.natoms)
    assert np.array_equal(f, ref)


def test_synthetic_lists_serialized_scatter(snap, port):
    """Non-symmetric lists (harness.hpp:230-262): the reverse index is general."""
    p = port.synthetic(64, 14, 8, seed=600)
    with snap.SnapEngine.for_problem(p) as eng:
        eng.set_problem(p)
        eng.compute_U()
        eng.compute_Y()
        eng.compute_fused_dE()
        eng.scatter_forces()
        f = eng.forces()
        ref = serialized_scatter(p.nbr, p.numneigh, eng.dedr(), 64)
    assert np.array_equal(f, ref)


def test_forces_bitwise_stable_across_runs_and_contexts(snap):
    p = snap.bcc_problem(10, 10, 10, twojmax=8)
    sums = set()
    for _ in range(2):
        with snap.SnapEngine.for_problem(p) as eng:
            eng.set_problem(p)
            for _ in range(3):
                eng.run()
                sums.add(fnv1a(eng.forces()))
            f, e, t = eng.step(p.numneigh, p.nbr, p.disp)  # one-call path too
            sums.add(fnv1a(f))
    assert len(sums) == 1, sums


def _lists_from_positions(pos, nbr0, numneigh0, rcut):
    n = pos.shape[0]
    S = nbr0.shape[1]
    nbr = np.zeros((n, S), np.int32)
    disp = np.zeros((n, S, 3))
    nn = np.zeros(n, np.int32)
    for i in range(n):
        m = 0
        for k in range(int(numneigh0[i])):
            j = nbr0[i, k]
            d = pos[j] - pos[i]
            if d @ d < rcut * rcut:
                nbr[i, m] = j
                disp[i, m] = d
                m += 1
        nn[i] = m
    return nn, nbr, disp


@pytest.mark.parametrize("T", [4, 8])
def test_forces_match_finite_differences(snap, port, T):
    """tests/test_oracle.cpp:137-144 on the GPU path (make_cluster(8, T, 23+T))."""
    p = port.make_cluster(8, T, 23 + T)
    pos = p.positions.copy()
    h = 1e-6 * p.rcut
    with snap.SnapEngine.for_problem(p) as eng:
        f, _, _ = eng.step(p.numneigh, p.nbr, p.disp, p.types)
        fd = np.zeros_like(f)
        for i in range(pos.shape[0]):
            for d in range(3):
                e = []
                for s in (+1.0, -1.0):
                    q = pos.copy()
                    q[i, d] += s * h
                    nn, nbr, disp = _lists_from_positions(q, p.nbr, p.numneigh, p.rcut)
                    e.append(eng.step(nn, nbr, disp, p.types)[2])
                fd[i, d] = -(e[0] - e[1]) / (2.0 * h)
    denom = np.maximum(np.maximum(np.abs(f), np.abs(fd)), 1e-14)
    assert float(np.max(np.abs(f - fd) / denom)) <= 1e-5


def test_one_call_positions_step(snap):
    """snapgpu_run_positions (lists rebuilt on the device inside one graph,
    partner slots instead of the CSR) equals the host-list step bitwise on
    the same lists, stays exact when the atoms move, and re-plans when a
    list outgrows the stride."""
    p = snap.bcc_problem(10, 10, 10, twojmax=8)
    ref = snap.run_pipeline(p)
    with snap.SnapEngine.for_problem(p) as eng:
        for _ in range(3):  # slow path, then graph replays
            f, e, t = eng.step_positions(p.positions, p.box)
            assert np.array_equal(f, ref.forces) and np.array_equal(e, ref.eatom)
            assert t == ref.etotal
        rng = np.random.default_rng(3)
        for it in range(3):  # moving atoms: lists rebuilt every step
            q = p.positions + rng.uniform(-0.02, 0.02, p.positions.shape)
            f, e, t = eng.step_positions(q, p.box)
            nn, nbr, disp = snap.build_neighborlist(q, p.box, p.rcut)
            pr = snap.Problem.from_any(p)
            pr.numneigh, pr.nbr, pr.disp = nn, nbr, disp
            r = snap.run_pipeline(pr)
            assert np.array_equal(f, r.forces) and t == r.etotal
        # a list outgrowing the stride inside the graph: expand the lattice
        # (14 neighbors, stride 14), then the original spacing in that box
        box2 = p.box * 1.05
        eng.step_positions(p.positions * 1.05, box2)
        f, e, t = eng.step_positions(p.positions, box2)
        nn, nbr, disp = snap.build_neighborlist(p.positions, box2, p.rcut)
        assert nn.max() > 14
        pr = snap.Problem.from_any(p)
        pr.numneigh, pr.nbr, pr.disp = nn, nbr, disp
        r = snap.run_pipeline(pr)
        assert np.array_equal(f, r.forces) and t == r.etotal


@pytest.mark.parametrize("cells", [(10, 10, 10), (16, 16, 16), (3, 3, 3)])
def test_y_to_de_overlap_bitwise(snap, cells):
    """The per-tile compute_Y -> compute_fused_dE hand-off (dE CTAs start on
    a tile's flag while other tiles still run) gives bitwise the results of
    waiting for the whole compute_Y grid, run after run, and through the
    one-call path; the automatic plan (tiles with one part more) stays
    within round-off of the uniform two-part split."""
    p = snap.bcc_problem(*cells, twojmax=8)
    with snap.SnapEngine.for_problem(p) as eng:
        eng.set_problem(p)
        eng.set_overlap(False)
        eng.run()
        f0, (e0, t0) = eng.forces().copy(), eng.energy()
        d0 = eng.dedr()
        eng.set_overlap(True)
        for _ in range(5):
            eng.run()
            assert np.array_equal(eng.forces(), f0) and np.array_equal(eng.dedr(), d0)
            e1, t1 = eng.energy()
            assert np.array_equal(e1, e0) and t1 == t0
        f2, e2, t2 = eng.step(p.numneigh, p.nbr, p.disp)
        assert np.array_equal(f2, f0) and t2 == t0
        eng.tune(2)
        eng.run()
        f3 = eng.forces()
        assert np.abs(f3 - f0).max() <= 1e-12 * np.abs(f0).max()


def test_positions_step_pinned_and_box_change(snap):
    """snapgpu_run_positions with pinned positions and outputs (the copy-free
    graph: binning reads the positions over PCIe, the kernels write the
    results in place) equals the pageable path bitwise; a box change that
    keeps the list stride re-plans the graphs (cells, minimum image)."""
    import torch

    p = snap.bcc_problem(10, 10, 10, twojmax=8)
    keep = []

    def pin(a):
        t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        keep.append(t)
        return t.numpy()

    with snap.SnapEngine.for_problem(p) as eng:
        f0, e0, t0 = eng.step_positions(p.positions, p.box)
        pos = pin(p.positions)
        outs = [pin(np.zeros(x)) for x in ((p.natoms, 3), p.natoms, 1)]
        for _ in range(3):
            f1, e1, t1 = eng.step_positions(pos, p.box, *outs)
            assert np.array_equal(f1, f0) and np.array_equal(e1, e0) and t1 == t0
        rng = np.random.default_rng(5)
        q = p.positions + rng.uniform(-0.02, 0.02, p.positions.shape)
        pos[:] = q
        f2, _, t2 = eng.step_positions(pos, p.box, *outs)
        fr, _, tr = eng.step_positions(q, p.box)  # pageable path on the same positions
        assert np.array_equal(f2, fr) and t2 == tr
        box2 = p.box * 1.002  # same neighbor count, new cells / minimum image
        f3, _, t3 = eng.step_positions(pos, box2, *outs)
        nn, nbr, disp = snap.build_neighborlist(q, box2, p.rcut)
        pr = snap.Problem.from_any(p)
        pr.numneigh, pr.nbr, pr.disp = nn, nbr, disp
        r = snap.run_pipeline(pr)
        assert np.array_equal(f3, r.forces) and t3 == r.etotal


@pytest.mark.parametrize("n,tune", [(40, 0), (97, 3), (300, 0), (1000, 5)])
def test_y_to_de_overlap_ragged(snap, port, n, tune):
    """The per-tile hand-off on ragged typed clusters (a partial last tile,
    several part counts, forced splits): bitwise the grid-wide wait, and
    within the parity bar of the oracle."""
    p = port.make_cluster(n, 8, 1000 + n, ntypes=2)
    with snap.SnapEngine.for_problem(p) as eng:
        eng.set_problem(p)
        if tune:
            eng.tune(tune)
        eng.set_overlap(False)
        eng.run()
        f0, d0 = eng.forces().copy(), eng.dedr()
        eng.set_overlap(True)
        for _ in range(3):
            eng.run()
            assert np.array_equal(eng.forces(), f0) and np.array_equal(eng.dedr(), d0)
    ref = port.run(p, want=("forces",))
    assert np.abs(f0 - ref["forces"]).max() <= 1e-10 * np.abs(ref["forces"]).max()
