"""Multi-rank host logic on CPU (gloo, world_size 2): slab partition,
partial-force scatter, force reduce-scatter and energy all-reduce give the
single-process result.  The per-rank compute is the oracle
(dE per pair); the GPU kernels' partition path is covered by
tests/test_gpu_parity.py::test_partition_sum_equals_full."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2011_12875_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2011_12875_b200 as snap

        port_ = oracle.Port()
        p = snap.bcc_problem(4, 4, 3 * world, twojmax=4)
        ref = port_.run(p, want=("forces", "eatom", "etotal", "delist"))
        n = p.natoms
        lo, hi = D.slab_bounds(n, world, rank)
        part = D.partial_forces_host(p.nbr[lo:hi], p.numneigh[lo:hi], ref["delist"][lo:hi], lo, n)
        rows = D.padded_rows(n, world)
        buf = torch.zeros(rows * 3, dtype=torch.float64)
        buf[: n * 3] = torch.from_numpy(part.reshape(-1))
        own = D.reduce_forces(buf, world, rank, n).numpy().reshape(-1, 3)
        k = rows // world
        glo = np.arange(rank * k, min((rank + 1) * k, n))
        ferr = np.abs(own[: len(glo)] - ref["forces"][glo]).max() / np.abs(ref["forces"]).max()
        e = torch.tensor([ref["eatom"][lo:hi].sum()], dtype=torch.float64)
        D.reduce_energy(e)
        eerr = abs(float(e[0]) - ref["etotal"]) / abs(ref["etotal"])
        q.put((rank, ferr, eerr, lo, hi))
    finally:
        dist.destroy_process_group()


def test_slab_bounds_cover_all_atoms():
    for n, w in [(2000, 1), (2000, 2), (2001, 4), (16000, 8), (7, 3)]:
        got = [D.slab_bounds(n, w, r) for r in range(w)]
        assert got[0][0] == 0 and got[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(got[:-1], got[1:]))
        assert max(h - l for l, h in got) - min(h - l for l, h in got) <= 1
        assert D.padded_rows(n, w) % w == 0 and D.padded_rows(n, w) >= n


@pytest.mark.parametrize("world", [2])
def test_gloo_partitioned_forces_and_energy(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, ferr, eerr, lo, hi in res:
        assert ferr <= 1e-13, (rank, ferr)
        assert eerr <= 1e-13, (rank, eerr)
