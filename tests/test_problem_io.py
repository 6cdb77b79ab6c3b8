"""Problem files in the reference schema (harness.hpp:698-780).

The fixtures under tests/golden/*.problem.json were written by the
reference's own harness::save_problem (tests/golden/make_golden.py).  Loading
them must give exactly the arrays of the matching golden .npz; our writer's
files must load bit for bit in the reference (harness::load_problem, which
validates) and in our reader; a reference re-save of our file must read back
identically.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden


@pytest.fixture(scope="module")
def pio():
    from paper_2011_12875_b200 import problem_io

    return problem_io


def _same(a, b):
    assert a.twojmax == b.twojmax
    for k in ("rcut", "rmin0", "rfac0", "wself"):
        assert float(getattr(a, k)) == float(getattr(b, k)), k
    assert int(a.self_flag) == int(b.self_flag)
    for k in ("beta", "weights"):
        assert np.array_equal(np.asarray(getattr(a, k), np.float64),
                              np.asarray(getattr(b, k), np.float64)), k
    n = np.asarray(a.numneigh).shape[0]
    assert np.array_equal(np.asarray(a.numneigh), np.asarray(b.numneigh))
    for i in range(n):
        k = int(a.numneigh[i])
        assert np.array_equal(np.asarray(a.nbr)[i, :k], np.asarray(b.nbr)[i, :k])
        assert np.array_equal(np.asarray(a.disp)[i, :k], np.asarray(b.disp)[i, :k])


@pytest.mark.parametrize("name", ["bcc54_2j8", "cluster_n7_2j5_s915_t3"])
def test_reference_written_file_loads_bitwise(pio, name):
    p = pio.load_problem(os.path.join(GOLDEN, name + ".problem.json"))
    g, _, _ = load_golden(name)
    _same(p, g)
    if g.positions is not None:
        assert np.array_equal(p.positions, g.positions)
    if g.types is not None:
        assert np.array_equal(p.types, g.types)


def test_writer_matches_reference_schema_and_roundtrips(pio, tmp_path):
    import oracle

    src = os.path.join(GOLDEN, "bcc54_2j8.problem.json")
    p = pio.load_problem(src)
    ours = tmp_path / "ours.json"
    pio.save_problem(p, str(ours))
    # same keys, order and values as the reference writer's file
    assert json.load(open(ours)) == json.load(open(src))
    assert list(json.load(open(ours)).keys()) == list(json.load(open(src)).keys())
    _same(pio.load_problem(str(ours)), p)
    if oracle.ref_available():
        back = tmp_path / "ref_resaved.json"
        oracle.Ref().resave_problem(str(ours), str(back))  # validates in the reference
        _same(pio.load_problem(str(back)), p)


def test_loader_rejects_bad_files(pio, tmp_path):
    from paper_2011_12875_b200 import InvalidArgument

    j = json.load(open(os.path.join(GOLDEN, "cluster_n7_2j5_s915_t3.problem.json")))
    bad = dict(j, schema=2)
    f = tmp_path / "bad.json"
    f.write_text(json.dumps(bad))
    with pytest.raises(InvalidArgument, match="schema"):
        pio.load_problem(str(f))
    far = json.loads(json.dumps(j))
    far["neighbors"][0][0]["disp"] = [5.0, 0.0, 0.0]  # beyond Rcut (snap_core.hpp:112)
    f.write_text(json.dumps(far))
    with pytest.raises(InvalidArgument, match="Rcut"):
        pio.load_problem(str(f))
    with pytest.raises(InvalidArgument, match="cannot open"):
        pio.load_problem(str(tmp_path / "missing.json"))


@pytest.mark.gpu
def test_engine_on_reference_problem_file(pio):
    import paper_2011_12875_b200 as snap

    p = pio.load_problem(os.path.join(GOLDEN, "bcc54_2j8.problem.json"))
    _, out, _ = load_golden("bcc54_2j8")
    r = snap.run_pipeline(p)
    f = out["forces"]
    assert np.abs(r.forces - f).max() <= 1e-10 * np.abs(f).max()
    assert abs(r.etotal - out["etotal"]) <= 1e-12 * abs(out["etotal"])
