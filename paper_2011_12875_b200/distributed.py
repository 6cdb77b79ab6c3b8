"""Atom-partitioned multi-GPU force step.

One process per GPU.  Positions / neighbor displacements are replicated;
rank r owns a contiguous slab of atoms [lo, hi) (the BCC generator is
z-major, so contiguous indices are spatial z-slabs) and uploads only the
owned atoms' neighbor lists.  U, Y and the fused dU/dE run on owned atoms
and pairs; the scatter F_nbr -= dE(i,k) reaches atoms owned elsewhere, so
every rank produces a PARTIAL natoms_total x 3 force buffer.  The only
exchange steps are the ones the reference path implies
(snap_core.hpp:889-898 scatter, :692-699 energy sum):

    forces  : reduce-scatter (sum) of the partial buffers -> owned slices
    energy  : all-reduce (sum) of the owned-atom totals

over NCCL (NVLink/NVSwitch).  gloo has no reduce_scatter, so the CPU test
path uses all_reduce + slice; the result is the same.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np


def slab_bounds(natoms: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous owned range of `rank`; equal sizes when world divides natoms."""
    base, extra = divmod(natoms, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def padded_rows(natoms: int, world: int) -> int:
    """Atom rows of the reduce-scatter buffer: natoms rounded up to world * k."""
    return ((natoms + world - 1) // world) * world


def reduce_forces(partial, world: int, rank: int, natoms: int, out=None):
    """Sum the ranks' partial (padded_rows x 3, flattened) force buffers and
    return this rank's owned rows [rank*k, (rank+1)*k), k = padded_rows/world."""
    import torch
    import torch.distributed as dist

    k = padded_rows(natoms, world) // world
    if out is None:
        out = torch.empty(k * 3, dtype=partial.dtype, device=partial.device)
    if dist.get_backend() == "nccl":
        dist.reduce_scatter_tensor(out, partial)
    else:  # gloo: no reduce_scatter
        full = partial.clone()
        dist.all_reduce(full)
        out.copy_(full[rank * k * 3:(rank + 1) * k * 3])
    return out


def reduce_energy(local_total):
    import torch.distributed as dist

    dist.all_reduce(local_total)
    return local_total


def partial_forces_host(nbr, numneigh, dedr, lo: int, natoms_total: int) -> np.ndarray:
    """Host statement of what one rank's scatter produces (scatter_forces,
    snap_core.hpp:889-898, restricted to owned pairs): used by the CPU tests."""
    f = np.zeros((natoms_total, 3))
    n = numneigh.shape[0]
    for i in range(n):
        for k in range(int(numneigh[i])):
            f[lo + i] += dedr[i, k]
            f[nbr[i, k]] -= dedr[i, k]
    return f


class PartitionedEngine:
    """SnapEngine bound to this rank's slab with the NCCL reductions attached."""

    def __init__(self, problem, world: int, rank: int, device: int, stream=None):
        import torch

        from . import Problem, SnapEngine

        p = Problem.from_any(problem)
        self.world, self.rank = world, rank
        self.natoms = p.natoms
        self.lo, self.hi = slab_bounds(p.natoms, world, rank)
        self.eng = SnapEngine.for_problem(p, device=device)
        if stream is not None:
            self.eng.set_stream(stream.cuda_stream)
        self.own = (np.ascontiguousarray(p.numneigh[self.lo:self.hi]),
                    np.ascontiguousarray(p.nbr[self.lo:self.hi]),
                    np.ascontiguousarray(p.disp[self.lo:self.hi]))
        self.types = p.types
        self.upload(*self.own)
        rows = padded_rows(p.natoms, world)
        self.f_full = torch.zeros(rows * 3, dtype=torch.float64, device=device)
        self.f_own = torch.zeros(rows // world * 3, dtype=torch.float64, device=device)
        self.e_tot = torch.zeros(1, dtype=torch.float64, device=device)

    def upload(self, numneigh, nbr, disp):
        if self.world == 1:
            self.eng.set_neighbors(numneigh, nbr, disp, self.types)
        else:
            self.eng.set_neighbors_partition(self.natoms, self.lo, numneigh, nbr, disp,
                                             self.types)

    def step(self):
        """One force step; returns (owned force rows (flattened), total energy) on device."""
        self.eng.run()
        if self.world == 1:
            self.eng.forces_to_device(self.f_full.data_ptr())
            self.eng.energy_to_device(self.e_tot.data_ptr())
            return self.f_full, self.e_tot
        self.eng.forces_to_device(self.f_full.data_ptr())
        self.eng.energy_to_device(self.e_tot.data_ptr())
        reduce_forces(self.f_full, self.world, self.rank, self.natoms, out=self.f_own)
        reduce_energy(self.e_tot)
        return self.f_own, self.e_tot

    def close(self):
        self.eng.close()
