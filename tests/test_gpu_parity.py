"""GPU parity: the CUDA path through the C-ABI vs the oracle and golden fixtures.

Tolerances (BASELINE.json north_star):
  forces        max|dF| / max|F|   <= 1e-10   (norm-wise; the reference's own
                                               reordered variants miss 1e-10
                                               elementwise against itself)
  total energy  |dE| / |E|         <= 1e-12
  per-atom E    max|dE_i| / max|E_i| <= 1e-12
  ulisttot / ylist / dElist        norm-wise <= 1e-12 / 1e-11 / 1e-10
"""
import numpy as np
import pytest

from conftest import golden_names, load_golden

pytestmark = pytest.mark.gpu

FTOL, ETOL = 1e-10, 1e-12


def normerr(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    scale = max(np.abs(b).max(), 1e-300)
    return float(np.abs(a - b).max() / scale)


@pytest.fixture(scope="module")
def snap():
    import paper_2011_12875_b200 as snap

    return snap


def _engine_run(snap, p, staged=False):
    eng = snap.SnapEngine.for_problem(p)
    eng.set_problem(p)
    if staged:
        eng.compute_U()
        eng.compute_Y()
        eng.compute_fused_dE()
        eng.scatter_forces()
    else:
        eng.run()
    return eng


@pytest.mark.parametrize("name", golden_names())
def test_golden_fixture(snap, name):
    p, out, _ = load_golden(name)
    eng = _engine_run(snap, p, staged=True)
    f = eng.forces()
    e, et = eng.energy()
    assert normerr(f, out["forces"]) <= FTOL
    assert abs(et - out["etotal"]) <= ETOL * abs(out["etotal"])
    assert normerr(e, out["eatom"]) <= ETOL
    if "ulisttot" in out:
        u = eng.ulisttot()
        assert normerr(u, out["ulisttot"]) <= 1e-12
    if "ylist" in out:
        y = eng.ylist()
        assert normerr(y, out["ylist"]) <= 1e-11
    if "delist" in out:
        assert normerr(eng.dedr(), out["delist"]) <= FTOL
    eng.close()


def test_graph_run_matches_staged(snap):
    p, out, _ = load_golden("bcc54_2j8")
    a = _engine_run(snap, p, staged=True)
    b = _engine_run(snap, p, staged=False)
    fa, fb = a.forces(), b.forces()
    assert normerr(fb, fa) <= 1e-13
    # replaying the captured graph gives the same answer again
    b.run()
    assert normerr(b.forces(), fa) <= 1e-13
    a.close()
    b.close()


def test_bcc2000_vs_oracle_port(snap, port):
    p = snap.bcc_problem(10, 10, 10, twojmax=8)
    assert p.natoms == 2000 and int(p.numneigh.min()) == 26 and int(p.numneigh.max()) == 26
    ref = port.run(p, want=("forces", "eatom", "etotal"))
    r = snap.run_pipeline(p)
    assert normerr(r.forces, ref["forces"]) <= FTOL
    assert abs(r.etotal - ref["etotal"]) <= ETOL * abs(ref["etotal"])
    assert normerr(r.eatom, ref["eatom"]) <= ETOL


@pytest.mark.parametrize("T", list(range(15)))
def test_every_band_limit_vs_oracle(snap, port, T):
    p = port.make_cluster(7, T, 1000 + T, ntypes=2)
    ref = port.run(p, want=("forces", "eatom", "etotal", "ulisttot", "ylist", "delist"))
    eng = _engine_run(snap, p, staged=True)
    assert normerr(eng.ulisttot(), ref["ulisttot"]) <= 1e-12
    assert normerr(eng.ylist(), ref["ylist"]) <= 1e-11
    assert normerr(eng.dedr(), ref["delist"]) <= FTOL
    assert normerr(eng.forces(), ref["forces"]) <= FTOL
    e, et = eng.energy()
    assert abs(et - ref["etotal"]) <= ETOL * max(abs(ref["etotal"]), 1e-300)
    eng.close()


def test_bcc_2j14_vs_golden(snap):
    p, out, _ = load_golden("bcc54_2j14")
    r = snap.run_pipeline(p)
    assert normerr(r.forces, out["forces"]) <= FTOL
    assert abs(r.etotal - out["etotal"]) <= ETOL * abs(out["etotal"])


def test_newton_sum_and_checksum_problem(snap):
    # acceptance.cpp:249-275 problem; Newton sum is not zero for synthetic
    # (non-mirrored) lists, so only parity is checked here.
    p, out, extra = load_golden("synthetic_n64_k14_2j8_s600")
    r = snap.run_pipeline(p)
    assert normerr(r.forces, out["forces"]) <= FTOL
    # closed periodic lists: forces sum to zero (oracle.hpp:224-237)
    q = snap.bcc_problem(4, 4, 4, twojmax=8)
    rq = snap.run_pipeline(q)
    assert np.abs(rq.forces.sum(axis=0)).max() / np.abs(rq.forces).max() <= 1e-10


def test_partition_sum_equals_full(snap):
    """Atom partition: per-shard partial forces sum to the full result."""
    p = snap.bcc_problem(4, 4, 4, twojmax=8)
    full = snap.run_pipeline(p)
    n = p.natoms
    cuts = [0, 37, 90, n]
    acc = np.zeros_like(full.forces)
    etot = 0.0
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        eng = snap.SnapEngine.for_problem(p)
        eng.set_neighbors_partition(n, lo, p.numneigh[lo:hi], p.nbr[lo:hi], p.disp[lo:hi])
        eng.run()
        acc += eng.forces()
        e, et = eng.energy()
        assert normerr(e, full.eatom[lo:hi]) <= 1e-12
        etot += et
        eng.close()
    assert normerr(acc, full.forces) <= 1e-12
    assert abs(etot - full.etotal) <= 1e-12 * abs(full.etotal)


def test_set_beta_and_one_hot(snap, port):
    p = port.make_cluster(5, 4, 911)
    eng = snap.SnapEngine.for_problem(p)
    eng.set_problem(p)
    for l in range(0, len(p.beta), 3):
        b = np.zeros_like(p.beta)
        b[l] = 1.0
        p.beta = b
        eng.set_beta(b)
        eng.run()
        ref = port.run(p, want=("forces",))
        assert normerr(eng.forces(), ref["forces"]) <= FTOL
    eng.close()


def test_errors_map_to_reference_exceptions(snap):
    p = snap.bcc_problem(3, 3, 3, twojmax=8)
    eng = snap.SnapEngine.for_problem(p)
    with pytest.raises(snap.StateError):
        eng.compute_Y()  # compute_Y: no Ulisttot (snap_core.hpp:1089)
    bad = p.disp.copy()
    bad[0, 0] = [5.0, 0.0, 0.0]  # beyond Rcut (snap_core.hpp:112)
    with pytest.raises(snap.InvalidArgument, match="Rcut"):
        eng.set_neighbors(p.numneigh, p.nbr, bad)
    nbr = p.nbr.copy()
    nbr[1, 0] = 1  # self neighbor (snap_core.hpp:108)
    with pytest.raises(snap.InvalidArgument, match="self"):
        eng.set_neighbors(p.numneigh, nbr, p.disp)
    with pytest.raises(snap.InvalidArgument, match="beta"):
        snap.SnapEngine(8, beta=np.zeros(3))
    eng.close()


_PINNED_KEEP = []


def _pinned(a):
    """A page-locked (hence device-mapped) copy of `a` as a numpy array."""
    import torch

    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    _PINNED_KEEP.append(t)
    return t.numpy()


@pytest.mark.parametrize("T", [2, 5, 8, 10])
def test_one_call_pinned_lists_pull(snap, port, T):
    """snapgpu_run_host with pinned host lists: compute_U pulls them over PCIe
    (2J <= 8; 2J > 8 uploads them) -- bitwise the result of the pageable-list
    upload path, and within the parity bar of the oracle, on a ragged typed
    cluster and on BCC lattices; the device copies it leaves serve a
    following graph run."""
    for p in (port.make_cluster(12, T, 91 + T), snap.bcc_problem(4, 4, 4, twojmax=T)):
        p = snap.Problem.from_any(p)
        ty = p.types
        with snap.SnapEngine.for_problem(p) as eng:
            f0, e0, t0 = eng.step(p.numneigh, p.nbr, p.disp, ty)
            args = [_pinned(x) for x in (p.numneigh, p.nbr, p.disp)]
            outs = [_pinned(np.full(x.shape, np.nan)) for x in (f0, e0, np.zeros(1))]
            for it in range(3):  # pageable outputs (read back), then pinned (written in place)
                o = {} if it == 0 else dict(zip(("forces", "eatom", "etotal"), outs))
                f1, e1, t1 = eng.step(*args, ty, **o)
                assert np.array_equal(f1, f0) and np.array_equal(e1, e0) and t1 == t0
                if it:
                    assert f1 is outs[0] and e1 is outs[1]
            eng.run()  # graph run on the lists the pull left on the device
            assert np.array_equal(eng.forces(), f0)
            nn, nbr, disp = eng.neighbors()
            assert np.array_equal(nn, p.numneigh) and np.array_equal(disp, p.disp)
        ref = port.run(p, want=("forces", "etotal"))
        assert np.abs(f1 - ref["forces"]).max() <= 1e-10 * np.abs(ref["forces"]).max()
        assert abs(t1 - ref["etotal"]) <= 1e-12 * abs(ref["etotal"])


def test_one_call_partition_slab_pinned(snap):
    """snapgpu_run_host on a rank's slab (atom_lo > 0, nlocal < natoms_total:
    set_neighbors_partition semantics) with pinned lists: the partial forces
    equal the pageable-upload path bitwise, and the slabs' partial forces sum
    to the single-GPU forces (to round-off: the sum order differs)."""
    p = snap.bcc_problem(6, 6, 6, twojmax=8)
    ref = snap.run_pipeline(p)
    n = p.natoms
    tot = np.zeros((n, 3))
    etot = 0.0
    for lo, hi in ((0, n // 3), (n // 3, n)):
        sl = [np.ascontiguousarray(x[lo:hi]) for x in (p.numneigh, p.nbr, p.disp)]
        with snap.SnapEngine.for_problem(p) as eng:
            f0, e0, t0 = eng.step(*sl, natoms_total=n, atom_lo=lo)
            f0 = f0.copy()
            f1, e1, t1 = eng.step(*[_pinned(x) for x in sl], natoms_total=n, atom_lo=lo)
        assert np.array_equal(f1, f0) and np.array_equal(e1, e0) and t1 == t0
        assert np.abs(e1 - ref.eatom[lo:hi]).max() <= 1e-12 * np.abs(ref.eatom).max()
        tot += f1
        etot += t1
    assert normerr(tot, ref.forces) <= 1e-12
    assert abs(etot - ref.etotal) <= 1e-12 * abs(ref.etotal)


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("case", ["cut", "self", "index", "zero", "count", "type"])
def test_one_call_step_validates_on_device(snap, case, pinned):
    """snapgpu_run_host defers Problem::validate (snap_core.hpp:89-118) to the
    U kernel: every violation still raises InvalidArgument with the host
    message, nothing is scattered, and the next valid step is exact."""
    p = snap.bcc_problem(3, 3, 3, twojmax=8)
    ref = snap.run_pipeline(p)
    nn, nbr, disp = p.numneigh.copy(), p.nbr.copy(), p.disp.copy()
    types = np.zeros(p.natoms, np.int32)
    match = {"cut": "Rcut", "self": "self", "index": "index", "zero": "zero-length",
             "count": "count", "type": "type"}[case]
    if case == "cut":
        disp[3, 2] = [5.0, 0.0, 0.0]
    elif case == "self":
        nbr[4, 1] = 4
    elif case == "index":
        nbr[5, 0] = p.natoms
    elif case == "zero":
        disp[6, 0] = 0.0
    elif case == "count":
        nn[7] = nbr.shape[1] + 1
    else:
        types[8] = 3
    if pinned:  # the compute_U pull path
        nn, nbr, disp = (_pinned(x) for x in (nn, nbr, disp))
    o = {}
    if pinned:  # pinned outputs too: written in place by the kernels
        o = dict(zip(("forces", "eatom", "etotal"),
                     (_pinned(np.zeros(x)) for x in ((p.natoms, 3), p.natoms, 1))))
    with snap.SnapEngine.for_problem(p) as eng:
        with pytest.raises(snap.InvalidArgument, match=match):
            eng.step(nn, nbr, disp, types, **o)
        f, e, t = eng.step(p.numneigh, p.nbr, p.disp, **o)
        # deterministic force gather and energy reductions: bitwise equal
        assert np.array_equal(f, ref.forces)
        assert np.array_equal(e, ref.eatom)
        assert t == ref.etotal


def test_empty_and_isolated_atoms(snap, port):
    p = port.make_cluster(6, 8, 77)
    p.numneigh = p.numneigh.copy()
    p.numneigh[2] = 0  # an isolated atom: only the self term
    ref = port.run(p, want=("forces", "etotal", "eatom"))
    r = snap.run_pipeline(p)
    assert normerr(r.forces, ref["forces"]) <= FTOL
    assert normerr(r.eatom, ref["eatom"]) <= ETOL


def test_stage_timing_and_tuning_knobs(snap):
    """Every compute_Y row split gives the same forces and energies to
    round-off, and each split is bitwise reproducible (the energy epilogue
    sums the parts of a tile in part order whichever CTA finishes last)."""
    p = snap.bcc_problem(6, 6, 6, twojmax=8)
    base = snap.run_pipeline(p)
    eng = snap.SnapEngine.for_problem(p)
    eng.set_problem(p)
    for yp in [1, 2, 3, 0, 7, 8]:
        eng.tune(y_parts=yp)
        eng.enable_stage_timing(True)
        eng.run()
        st = eng.stage_times()
        assert all(v > 0 for v in st.values())
        f1 = eng.forces()
        e1, et1 = eng.energy()
        assert normerr(f1, base.forces) <= 1e-13
        assert normerr(e1, base.eatom) <= 1e-13
        eng.run()
        e2, et2 = eng.energy()
        assert np.array_equal(eng.forces(), f1)
        assert np.array_equal(e2, e1) and et2 == et1
    with pytest.raises(snap.InvalidArgument):
        eng.tune(y_parts=9)
    with pytest.raises(snap.InvalidArgument):
        eng.tune(y_parts=-1)
    eng.close()
