"""C-ABI library checks that need no GPU.

* libsnapgpu.so loads and exports every entry point include/snapgpu.h declares;
* the context-free host utilities (table sizes, neighbor lists, BCC lattice)
  agree with the oracle / reference bitwise;
* without a CUDA device, creating a context fails loudly (no CPU fallback).
"""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2011_12875_b200 as snap
from conftest import ROOT, gpu_available


def header_symbols():
    src = open(os.path.join(ROOT, "include", "snapgpu.h")).read()
    return sorted(set(re.findall(r"\b(snapgpu_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = snap.library()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    assert b"sm_100a" in L.snapgpu_version()


def test_library_is_sm100a_cubin():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", snap.LIB_PATH], capture_output=True,
                         text=True)
    assert "sm_100a" in out.stdout


def test_counts_match_reference_known_answers(port):
    for T in (0, 2, 4, 8, 14):
        c = snap.counts(T)
        assert tuple(c.values()) == port.counts(T)
    assert snap.counts(8)["n_triples"] == 55 and snap.counts(14)["n_triples"] == 204


@pytest.mark.parametrize("cells", [(3, 3, 3), (4, 4, 4), (5, 4, 3), (6, 3, 4)])
def test_bcc_and_neighborlist_match_oracle_bitwise(port, cells):
    nx, ny, nz = cells
    p = snap.bcc_problem(nx, ny, nz, twojmax=8)
    pos, beta, box = port.bcc(nx, ny, nz, 8)
    assert np.array_equal(p.positions, pos) and np.array_equal(p.beta, beta)
    if min(cells) * 3.1803 >= 2 * 4.7:
        nn, nb, dp = port.neighborlist(pos, box, 4.7)
        assert np.array_equal(p.numneigh, nn)
        assert np.array_equal(p.nbr, nb)
        assert np.array_equal(p.disp, dp)
        assert int(p.numneigh.min()) == 26 and int(p.numneigh.max()) == 26


def test_neighborlist_errors():
    with pytest.raises(snap.InvalidArgument, match="box/2"):
        snap.build_neighborlist(np.zeros((2, 3)), [5.0, 5.0, 5.0], 4.7)


def test_neighborlist_brute_force_random(port):
    rng = np.random.default_rng(3)
    box = np.array([11.0, 12.5, 10.0])
    pos = rng.uniform(-5, 20, size=(150, 3))
    a = snap.build_neighborlist(pos, box, 4.7)
    b = port.neighborlist(pos, box, 4.7)  # direct O(n^2) scan
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly():
    with pytest.raises(snap.PipelineError):
        snap.SnapEngine(8, beta=np.zeros(55))


def _y_plan(T, ntiles, nsm, parts=0):
    L = snap.library()
    cta = np.zeros(4 * 20000, np.int32)
    tasks = np.zeros(1 << 16, np.int32)
    fn = L.snapgpu_debug_y_plan
    fn.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    n = fn(T, ntiles, nsm, parts, cta.ctypes.data, cta.size, tasks.ctypes.data, tasks.size)
    assert n > 0, snap.library().snapgpu_last_error(None)
    return cta[: 4 * n].reshape(n, 4), tasks


@pytest.mark.parametrize("ntiles", [1, 7, 63, 73, 74, 147, 148, 200, 8192])
def test_y_launch_plan_covers_every_row_once(ntiles):
    """compute_Y's launch plan (tables.cpp y_cta_plan): every 32-atom tile
    is split into parts 0..P-1 exactly once; each (part, group) row list of
    a tile's part count together covers the tile's 25 target rows (2J=8)
    exactly once; one wave (CTAs <= SMs) when the tiles are fewer than the
    SMs, with part counts floor/ceil(SMs / tiles) and an even number of
    base-count tiles; part-major order (consecutive CTAs share a TPC and run
    the same row lists)."""
    nsm, T, groups = 148, 8, 3
    cta, tasks = _y_plan(T, ntiles, nsm)
    tile, part, parts = cta[:, 0], cta[:, 1] & 0xFF, cta[:, 1] >> 8
    rows = sorted(j * 64 + mb for j in range(T + 1) for mb in range(j // 2 + 1))
    for t in range(ntiles):
        sel = tile == t
        P = set(parts[sel])
        assert len(P) == 1
        q = P.pop()
        assert sorted(part[sel]) == list(range(q))
        got = []
        for k in np.nonzero(sel)[0]:
            for g in range(groups):
                base = cta[k, 2] + g * cta[k, 3]
                lst = tasks[base: base + cta[k, 3]]
                got += [int(x) for x in lst[: list(lst).index(-1)]]
        assert sorted(got) == rows
    order = list(zip(parts, part, tile))
    assert order == sorted(order)
    if ntiles < nsm:
        assert len(cta) <= nsm
        base = max(1, min(8, nsm // ntiles))
        assert set(parts) <= {base, base + 1}
        if base < 8 and len(set(parts)) == 2:
            assert (parts[part == 0] == base).sum() % 2 == 0
    else:
        assert set(parts) == {1}
    # a forced part count (snapgpu_tune) is uniform
    cta2, _ = _y_plan(T, ntiles, nsm, parts=2)
    assert set(cta2[:, 1] >> 8) == {2} and len(cta2) == 2 * ntiles


def test_step_argument_reuse():
    """SnapEngine._arg: an argument that is already a C-contiguous array of the
    wanted type is passed as it is and its pointer is reused when the same
    object comes back; converted copies are rebuilt every call (the source may
    have changed)."""
    class _E:
        _args = {}
    e = _E()
    arg = snap.SnapEngine._arg.__get__(e)
    a = np.zeros((5, 3), np.float64)
    x, p = arg(0, a, np.float64)
    assert x is a and p == a.ctypes.data
    a[0, 0] = 7.0  # in-place changes stay visible through the same buffer
    x2, p2 = arg(0, a, np.float64)
    assert x2 is a and p2 == p and x2[0, 0] == 7.0
    b = np.zeros(4, np.float32)  # converted: never reused
    y, _ = arg(1, b, np.float64)
    assert y is not b and y.dtype == np.float64 and e._args[1] is None
    b[0] = 3.0
    y2, _ = arg(1, b, np.float64)
    assert y2[0] == 3.0
    c = np.zeros((4, 6))[:, ::2]  # non-contiguous: converted
    z, _ = arg(2, c, np.float64)
    assert z.flags.c_contiguous and z is not c
