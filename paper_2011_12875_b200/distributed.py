"""Atom-partitioned multi-GPU force step.

One process per GPU.  Positions / neighbor displacements are replicated;
rank r owns a contiguous slab of atoms (the BCC generator is z-major, so
contiguous indices are spatial z-slabs) and uploads only the owned atoms'
neighbor lists.  U, Y and the fused dU/dE run on owned atoms and pairs; the
scatter F_nbr -= dE(i,k) reaches atoms owned elsewhere, so every rank
produces a PARTIAL force array for all atoms.  The only exchange steps are
the ones the reference path implies (snap_core.hpp:889-898 scatter,
:692-699 energy sum), and they travel in ONE collective:

    the engine writes its partial forces straight into a caller-owned
    buffer of `world` chunks, chunk r = the k = ceil(N / world) atoms of
    rank r (3k doubles) followed by one energy slot that holds this rank's
    owned-atom energy in every chunk (snapgpu_set_force_layout);
    a reduce-scatter (sum) of that buffer hands rank r its owned forces
    and, in its energy slot, the total energy.

NCCL over NVLink/NVSwitch on GPUs; gloo has no reduce_scatter, so the CPU /
single-GPU test path uses all_reduce + slice, which gives the same numbers.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np


def chunk_rows(natoms: int, world: int) -> int:
    """Atoms per rank chunk: ceil(natoms / world)."""
    return max(1, -(-natoms // world))


def slab_bounds(natoms: int, world: int, rank: int) -> Tuple[int, int]:
    """Owned atoms [lo, hi) of `rank`: exactly the atoms of its force chunk."""
    k = chunk_rows(natoms, world)
    lo = min(natoms, rank * k)
    return lo, min(natoms, lo + k)


def chunk_stride(natoms: int, world: int) -> int:
    """Doubles per chunk: 3 per atom + the energy slot."""
    return 3 * chunk_rows(natoms, world) + 1


def chunked_partial_host(nbr, numneigh, dedr, lo: int, natoms: int, world: int,
                         energy: float) -> np.ndarray:
    """Host statement of one rank's chunked partial buffer (what
    k_gather_forces writes under snapgpu_set_force_layout): the serialized
    scatter (snap_core.hpp:889-898) of the owned pairs, atom a at
    (a // k) * (3k+1) + (a % k) * 3, this rank's energy in every chunk's
    last slot.  Used by the CPU tests of the collective logic."""
    k = chunk_rows(natoms, world)
    cs = 3 * k + 1
    f = np.zeros((natoms, 3))
    for i in range(numneigh.shape[0]):
        for kk in range(int(numneigh[i])):
            f[lo + i] += dedr[i, kk]
            f[nbr[i, kk]] -= dedr[i, kk]
    buf = np.zeros(world * cs)
    for r in range(world):
        a0, a1 = min(natoms, r * k), min(natoms, (r + 1) * k)
        buf[r * cs: r * cs + 3 * (a1 - a0)] = f[a0:a1].reshape(-1)
        buf[r * cs + 3 * k] = energy
    return buf


def reduce_chunks(partial, world: int, rank: int, out=None):
    """Sum the ranks' chunked partial buffers; returns this rank's chunk
    (3k owned-force doubles + the total energy)."""
    import torch
    import torch.distributed as dist

    cs = partial.numel() // world
    if out is None:
        out = torch.empty(cs, dtype=partial.dtype, device=partial.device)
    if dist.get_backend() == "nccl":
        dist.reduce_scatter_tensor(out, partial)
    else:  # gloo: no reduce_scatter
        full = partial.clone()
        dist.all_reduce(full)
        out.copy_(full[rank * cs:(rank + 1) * cs])
    return out


class _DevView:
    """__cuda_array_interface__ over an engine-owned device pointer."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3}


class PartitionedEngine:
    """SnapEngine bound to this rank's slab, writing its partial forces into
    the reduce-scatter buffer, on one stream shared with the collective."""

    def __init__(self, problem, world: int, rank: int, device: int, stream=None):
        import torch

        from . import Problem, SnapEngine

        p = Problem.from_any(problem)
        self.world, self.rank = world, rank
        self.natoms = p.natoms
        self.lo, self.hi = slab_bounds(p.natoms, world, rank)
        self.k = chunk_rows(p.natoms, world)
        # the engine and the collectives run on ONE stream, so the
        # reduce-scatter is ordered after the force gather that fills it
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        self.eng = SnapEngine.for_problem(p, device=device)
        self.eng.set_stream(self.stream.cuda_stream)
        self.own = (np.ascontiguousarray(p.numneigh[self.lo:self.hi]),
                    np.ascontiguousarray(p.nbr[self.lo:self.hi]),
                    np.ascontiguousarray(p.disp[self.lo:self.hi]))
        self.types = p.types
        if world > 1:
            cs = chunk_stride(p.natoms, world)
            self.f_part = torch.zeros(world * cs, dtype=torch.float64, device=device)
            self.chunk = torch.zeros(cs, dtype=torch.float64, device=device)
            self.eng.set_force_layout(world, self.f_part.data_ptr())
        self.upload(*self.own)
        f, _, e = self.eng.device_outputs()
        if world == 1:
            self.f_own = torch.as_tensor(_DevView(f, 3 * p.natoms), device=f"cuda:{device}")
            self.e_tot = torch.as_tensor(_DevView(e, 1), device=f"cuda:{device}")
        else:
            self.f_own = self.chunk[: 3 * (self.hi - self.lo)]
            self.e_tot = self.chunk[3 * self.k:]

    def upload(self, numneigh, nbr, disp):
        if self.world == 1:
            self.eng.set_neighbors(numneigh, nbr, disp, self.types)
        else:
            self.eng.set_neighbors_partition(self.natoms, self.lo, numneigh, nbr, disp,
                                             self.types)

    def step(self):
        """One force step; returns (owned force rows, flattened; total
        energy), both device tensors, ready on self.stream."""
        import torch

        with torch.cuda.stream(self.stream):
            self.eng.run()
            if self.world > 1:
                reduce_chunks(self.f_part, self.world, self.rank, out=self.chunk)
        return self.f_own, self.e_tot

    def step_host(self, numneigh, nbr, disp):
        """One force step from this rank's host lists (the end-to-end call):
        snapgpu_run_host on the slab -- page-locked lists are read by
        compute_U over PCIe, validated on the device -- then the
        reduce-scatter; returns like step()."""
        import torch

        with torch.cuda.stream(self.stream):
            self.eng.step(numneigh, nbr, disp, self.types, natoms_total=self.natoms,
                          atom_lo=self.lo, forces=None, eatom=None, etotal=None, readback=False)
            if self.world > 1:
                reduce_chunks(self.f_part, self.world, self.rank, out=self.chunk)
        return self.f_own, self.e_tot

    def close(self):
        self.eng.close()
