"""Algorithmic work of the SNAP force step.

Exact trip counts of the reference loop nests, mul and add counted
separately, complex multiply = 6 (the pipeline.hpp:36-40 CounterModel
convention):

    F_U  per pair = 18 E_U + 4 N_half          compute_U   snap_core.hpp:369-489
    F_Y  per atom = 10 MAC + 4 NB + 4 NZ       compute_Y   snap_core.hpp:1085-1200
    F_dE per pair = 18 E_U + 102 E_U + 33 E_C  compute_fused_dE :1274-1406

with MAC / NB / NZ the z_element trip counts (z_loop_bounds,
halfint_index.hpp:257-276), E_U = sum_t (t/2+1) t Wigner element updates and
E_C the contracted elements.  2J=8: 2,960 / 465,246 / 20,385; 2J=14:
13,192 / 11,991,616 / 91,152.
"""
from __future__ import annotations

from functools import lru_cache

FP64_SPEC_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # B200: 148 SM x 64 DFMA/clk x 2 x 1.965 GHz


@lru_cache(maxsize=None)
def flop_model(T: int) -> dict:
    def zlb(j1, j2, j, mb, ma):
        t = 2 * ma - j
        ma1 = 0 if t + j1 - j2 < 0 else (t + j1 - j2) // 2
        na = min(j1, (t + j2 + j1) // 2) - ma1 + 1
        t = 2 * mb - j
        mb1 = 0 if t + j1 - j2 < 0 else (t + j1 - j2) // 2
        nb = min(j1, (t + j2 + j1) // 2) - mb1 + 1
        return na, nb

    mac = nb_sum = nz = 0
    for j1 in range(T + 1):
        for j2 in range(j1 + 1):
            for j in range(j1 - j2, min(j1 + j2, T) + 1, 2):
                for mb in range(j // 2 + 1):
                    for ma in range(j + 1):
                        na, nb = zlb(j1, j2, j, mb, ma)
                        mac += na * nb
                        nb_sum += nb
                        nz += 1
    nhalf = sum((t // 2 + 1) * (t + 1) for t in range(T + 1))
    e_u = sum((t // 2 + 1) * t for t in range(1, T + 1))
    e_c = 1 + sum((t + 1) * ((t + 1) // 2) + ((t // 2 + 1) if t % 2 == 0 else 0)
                  for t in range(1, T + 1))
    f_u = 18 * e_u + 4 * nhalf
    f_y = 10 * mac + 4 * nb_sum + 4 * nz
    f_de = 18 * e_u + 102 * e_u + 33 * e_c
    return {"U_per_pair": f_u, "Y_per_atom": f_y, "dE_per_pair": f_de,
            "per_atom_step_26": f_y + 26 * (f_u + f_de)}


def step_flops(twojmax: int, npairs: int, natoms: int) -> float:
    """Algorithmic FLOPs of one force step."""
    fm = flop_model(twojmax)
    return fm["U_per_pair"] * npairs + fm["Y_per_atom"] * natoms + fm["dE_per_pair"] * npairs
