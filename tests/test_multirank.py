"""Multi-rank host logic on CPU (gloo, world_size 2): slab partition, the
chunked partial-force layout with its energy slots, and the single
reduce-scatter give the single-process forces and total energy (SURVEY.md
§8(e)).  The per-rank compute is the oracle (dE per pair); the engine's
partition path runs in tests/test_gpu_multirank.py (two ranks on one GPU)."""
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

        port_ = oracle.Port()
        p = port_.bcc_problem(4, 4, 3 * world, 4)
        ref = port_.run(p, want=("forces", "eatom", "etotal", "delist"))
        n = p.numneigh.shape[0]
        lo, hi = D.slab_bounds(n, world, rank)
        e_own = float(ref["eatom"][lo:hi].sum())
        part = D.chunked_partial_host(p.nbr[lo:hi], p.numneigh[lo:hi], ref["delist"][lo:hi],
                                      lo, n, world, e_own)
        chunk = D.reduce_chunks(torch.from_numpy(part), world, rank).numpy()
        k = D.chunk_rows(n, world)
        own = chunk[: 3 * (hi - lo)].reshape(-1, 3)
        ferr = np.abs(own - ref["forces"][lo:hi]).max() / np.abs(ref["forces"]).max()
        eerr = abs(float(chunk[3 * k]) - ref["etotal"]) / abs(ref["etotal"])
        q.put((rank, ferr, eerr, lo, hi))
    finally:
        dist.destroy_process_group()


def test_slab_bounds_cover_all_atoms():
    for n, w in [(2000, 1), (2000, 2), (2001, 4), (16000, 8), (7, 3), (10, 4)]:
        got = [D.slab_bounds(n, w, r) for r in range(w)]
        assert got[0][0] == 0 and got[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(got[:-1], got[1:]))
        k = D.chunk_rows(n, w)
        # the owned slab of rank r is exactly the atoms of force chunk r
        assert all(lo == min(n, r * k) and hi == min(n, (r + 1) * k)
                   for r, (lo, hi) in enumerate(got))
        assert D.chunk_stride(n, w) == 3 * k + 1


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
