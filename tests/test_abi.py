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
