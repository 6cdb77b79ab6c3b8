"""The engine's partitioned multi-GPU step, as W ranks sharing one GPU.

Each rank is a process with its own PartitionedEngine (owned slab, chunked
partial-force buffer filled by the force gather, energy slots) and the
collective runs over gloo on CUDA tensors (NCCL refuses two ranks on one
device; gloo's all_reduce + slice path stands in for the reduce-scatter and
gives the same sums).  The owned forces and the total energy must equal the
single-GPU step (the coupling replaced is scatter_forces
snap_core.hpp:889-898 and the energy sum :692-699).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cells, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2011_12875_b200 as snap
        from paper_2011_12875_b200.distributed import PartitionedEngine

        torch.cuda.set_device(0)
        p = snap.bcc_problem(*cells, twojmax=8)
        pe = PartitionedEngine(p, world, rank, 0)
        for _ in range(2):  # the second step replays the captured graph
            f_own, e_tot = pe.step()
        torch.cuda.synchronize()
        f_dev, e_dev = f_own.cpu().numpy().copy(), float(e_tot.cpu()[0])
        # the end-to-end call on pinned host lists (compute_U reads them)
        pin = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in pe.own]
        for _ in range(2):
            f_own, e_tot = pe.step_host(*[x.numpy() for x in pin])
        torch.cuda.synchronize()
        if not (np.array_equal(f_own.cpu().numpy(), f_dev) and float(e_tot.cpu()[0]) == e_dev):
            raise AssertionError("step_host differs from step")
        q.put((rank, pe.lo, pe.hi, f_own.cpu().numpy().copy(), float(e_tot.cpu()[0])))
        pe.close()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, -1, -1, repr(e), 0.0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cells", [(2, (6, 6, 6)), (3, (5, 5, 5))])
def test_partitioned_engine_matches_single_gpu(world, cells):
    import torch.multiprocessing as mp

    import paper_2011_12875_b200 as snap

    p = snap.bcc_problem(*cells, twojmax=8)
    full = snap.run_pipeline(p)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cells, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda x: x[0])
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    covered = 0
    fmax = np.abs(full.forces).max()
    for rank, lo, hi, f_own, e_tot in res:
        assert lo >= 0, f_own
        covered += hi - lo
        own = f_own.reshape(-1, 3)
        assert own.shape[0] == hi - lo
        assert np.abs(own - full.forces[lo:hi]).max() <= 1e-12 * fmax
        assert abs(e_tot - full.etotal) <= 1e-12 * abs(full.etotal)
    assert covered == p.natoms
