"""The oracle is pinned before it is trusted (CPU only).

1. our C restatement (oracle/_build/liboracle.so) reproduces the golden
   fixtures generated from the unmodified reference bitwise;
2. it reproduces the reference acceptance gate's force checksum
   dd6d6cc7a1c2e358 (tests/acceptance.cpp:249-275);
3. the reference's own known-answer values (tests/test_halfint_index.cpp,
   tests/test_angular_basis.cpp) hold;
4. where oracle/_ref exists, port == reference bitwise on fresh problems.
"""
import numpy as np
import pytest

import oracle
from conftest import fnv1a, golden_names, load_golden

import os

TABLES = np.load(os.path.join(os.path.dirname(__file__), "golden", "tables.npz"))


@pytest.mark.parametrize("name", golden_names())
def test_port_reproduces_golden_bitwise(port, name):
    p, out, _ = load_golden(name)
    want = tuple(k for k in ("forces", "eatom", "etotal", "ulisttot", "ylist", "delist")
                 if k in out)
    got = port.run(p, want=want)
    for k in want:
        g, r = np.asarray(got[k]), np.asarray(out[k])
        assert g.shape == r.shape and g.dtype == r.dtype, k
        assert g.tobytes() == r.tobytes(), k  # bitwise


def test_acceptance_checksum(port):
    p = port.synthetic(64, 14, 8, seed=600)
    assert fnv1a(port.run(p, want=("forces",))["forces"]) == "dd6d6cc7a1c2e358"


def test_known_counts(port):
    # test_halfint_index.cpp:47-68, 115-139
    assert port.counts(0)[0] == 1
    assert port.counts(2)[0] == 5
    assert port.counts(8)[0] == 55
    assert port.counts(14)[0] == 204
    assert port.counts(8)[2] == 285 and port.counts(14)[2] == 1240
    assert port.counts(8)[3] == 155
    assert port.counts(8)[1] == 125 and port.counts(8)[4] == 2386
    for T in (0, 2, 4, 8, 14):
        assert tuple(TABLES[f"counts_{T}"]) == port.counts(T)


def test_cg_table_and_closed_forms(port):
    cg = port.cg_table(8)
    assert np.array_equal(cg, TABLES["cg_8"])
    tup = port.tuples(2)
    # (j1,j2,j) = (1,1,0): CG(1/2 m1 1/2 m2 | 0 0) = +-1/sqrt(2)  (test_angular_basis.cpp:138-154)
    cg2 = port.cg_table(2)
    q = [i for i, t in enumerate(tup) if tuple(t[:3]) == (1, 1, 0)][0]
    blk = cg2[tup[q, 4]: tup[q, 4] + 4]
    assert np.allclose(sorted(np.abs(blk[[1, 2]])), [2 ** -0.5] * 2, atol=1e-15)
    assert blk[1] == -blk[2]
    # (0,0,0): 1
    assert cg2[0] == 1.0


def test_wigner_half_stack_vs_reference(port):
    for d, ref in zip(TABLES["wigner_disp"], TABLES["wigner_u8"]):
        assert np.array_equal(port.wigner_u_half(d, 8), ref)


def test_level01_blocks(port):
    # test_angular_basis.cpp:156-171: level 1 = [[conj a, -conj b], [b, a]]
    d = np.array([0.7, -1.1, 1.9])
    m = np.zeros(19)
    port.L.orc_map_to_3sphere(d, 4.7, 0.0, 0.99363, m)
    a = m[1] + 1j * m[2]
    b = m[3] + 1j * m[4]
    u = port.wigner_u_half(d, 1)
    assert u[0] == 1.0
    assert np.allclose(u[1:3], [np.conj(a), -np.conj(b)], rtol=0, atol=1e-15)
    assert abs(abs(a) ** 2 + abs(b) ** 2 - 1.0) < 1e-14


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built here")
@pytest.mark.parametrize("T,n,seed,nt", [(8, 9, 31, 2), (4, 6, 32, 1), (14, 4, 33, 1),
                                         (3, 5, 34, 3)])
def test_port_equals_reference_bitwise(port, T, n, seed, nt):
    R = oracle.Ref()
    p = R.make_cluster(n, T, seed, nt)
    q = port.make_cluster(n, T, seed, nt)
    for k in ("positions", "types", "weights", "numneigh", "nbr", "disp", "beta"):
        assert np.array_equal(getattr(p, k), getattr(q, k)), k
    a = port.run(q)
    b = R.run(p, "fused", True, 2)
    c = R.run(p, "v1", True, 2)
    for k in a:
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k
    assert np.array_equal(a["forces"], c["forces"])


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built here")
def test_port_neighborlist_and_synthetic_equal_reference(port):
    R = oracle.Ref()
    pos, beta, box = port.bcc(4, 4, 4, 8)
    a = port.neighborlist(pos, box, 4.7)
    b = R.neighborlist(pos, box[0], 4.7)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    s1 = port.synthetic(30, 26, 8, seed=99)
    s2 = R.synthetic(30, 26, 8, seed=99)
    for k in ("numneigh", "nbr", "disp", "beta"):
        assert np.array_equal(getattr(s1, k), getattr(s2, k))


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built here")
def test_reference_oracle_suite_on_bcc(port):
    # oracle.hpp:175-237: rotation invariance, Newton sum, cross-pipeline
    R = oracle.Ref()
    p = port.bcc_problem(3, 3, 3, 4)
    chk = R.oracle_checks(p)
    assert chk["rotation"] <= 1e-9
    assert chk["newton"] <= 1e-10
    assert chk["cross_pipeline"] <= 1e-10
