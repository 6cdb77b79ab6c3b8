"""B200-native SNAP force engine (TestSNAP workload of arXiv 2011.12875).

Host-side mirror of the reference's stage interface (snapforge,
/root/reference/proj/include/snapforge) over the C-ABI in include/snapgpu.h,
implemented by hand-written sm_100a FP64 kernels in csrc/.

    Problem            <- snapforge::Problem / SnapParams   (snap_core.hpp:48-119)
    SnapEngine         <- DescriptorState + stage functions (snap_core.hpp:130-1406)
      .compute_U()            compute_U            :369
      .compute_Y()            compute_Y            :1085  (+ per-atom energy)
      .compute_fused_dE()     compute_fused_dE     :1274  (compute_dU + compute_deidrj)
      .scatter_forces()       scatter_forces       :872
    run_pipeline()     <- run_pipeline (pipeline.hpp:206), adjoint `fused` branch
    build_neighborlist <- harness::build_neighborlist (harness.hpp:119)
    bcc_problem        TestSNAP BCC tungsten generator (new; not in the reference)

There is no CPU fallback: if the CUDA extension is missing or no GPU is
present, engine construction raises.  Errors map onto the reference's
exception types (common.hpp:21-42): InvalidArgument, PipelineError.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "InvalidArgument", "PipelineError", "CudaError", "StateError", "Problem",
    "PipelineResult", "SnapEngine", "run_pipeline", "build_neighborlist", "bcc_problem",
    "counts", "library", "LIB_PATH",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libsnapgpu.so")


class InvalidArgument(ValueError):
    """snapforge::InvalidArgument (common.hpp:21-25)."""


class PipelineError(RuntimeError):
    """snapforge::PipelineError (common.hpp:28-31)."""


class CudaError(PipelineError):
    """CUDA runtime failure inside the engine."""


class StateError(PipelineError):
    """A stage was called before its inputs exist."""


_ERRS = {1: InvalidArgument, 2: PipelineError, 3: CudaError, 4: StateError}

_lib = None


def library() -> C.CDLL:
    """Load libsnapgpu.so (built by __graft_entry__.build()); fail loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} missing: the CUDA extension is not built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`). "
            "There is no CPU fallback.")
    L = C.CDLL(LIB_PATH)
    vp, ip, dp = C.c_void_p, C.c_int, C.c_double
    L.snapgpu_last_error.restype = C.c_char_p
    L.snapgpu_last_error.argtypes = [vp]
    L.snapgpu_version.restype = C.c_char_p
    L.snapgpu_create.argtypes = [ip, ip, dp, dp, dp, dp, ip, vp, ip, vp, ip, C.POINTER(vp)]
    L.snapgpu_destroy.argtypes = [vp]
    L.snapgpu_set_beta.argtypes = [vp, vp, ip]
    L.snapgpu_set_stream.argtypes = [vp, vp]
    L.snapgpu_set_neighbors.argtypes = [vp, ip, ip, vp, vp, vp, vp]
    L.snapgpu_set_neighbors_partition.argtypes = [vp, ip, ip, ip, ip, vp, vp, vp, vp]
    for f in ("compute_U", "compute_Y", "compute_dU_deidrj", "scatter_forces", "run",
              "synchronize"):
        getattr(L, "snapgpu_" + f).argtypes = [vp]
    L.snapgpu_run_host.argtypes = [vp, ip, ip, ip, ip, vp, vp, vp, vp, vp, vp, vp]
    L.snapgpu_get_forces.argtypes = [vp, vp]
    L.snapgpu_get_energy.argtypes = [vp, vp, vp]
    L.snapgpu_get_ulisttot.argtypes = [vp, vp]
    L.snapgpu_get_ylist.argtypes = [vp, vp]
    L.snapgpu_get_dedr.argtypes = [vp, vp]
    L.snapgpu_get_virial.argtypes = [vp, vp]
    L.snapgpu_compute_descriptors.argtypes = [vp, vp]
    L.snapgpu_set_positions.argtypes = [vp, ip, vp, vp]
    L.snapgpu_run_positions.argtypes = [vp, ip, vp, vp, vp, vp, vp]
    L.snapgpu_get_neighbors.argtypes = [vp, vp, vp, vp]
    L.snapgpu_device_outputs.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]
    L.snapgpu_get_forces_device.argtypes = [vp, vp]
    L.snapgpu_get_energy_device.argtypes = [vp, vp, vp]
    L.snapgpu_fp64_peak.argtypes = [ip, ip, vp, vp]
    L.snapgpu_enable_stage_timing.argtypes = [vp, ip]
    L.snapgpu_stage_times.argtypes = [vp, vp]
    L.snapgpu_tune.argtypes = [vp, ip]
    L.snapgpu_set_overlap.argtypes = [vp, ip]
    L.snapgpu_set_force_layout.argtypes = [vp, ip, vp]
    L.snapgpu_counts.argtypes = [ip, vp]
    L.snapgpu_build_neighborlist.argtypes = [vp, ip, vp, dp, ip, vp, vp, vp]
    L.snapgpu_bcc_lattice.argtypes = [ip, ip, ip, dp, dp, C.c_uint64, ip, vp, vp]
    _lib = L
    return L


def _check(rc: int, ctx=None) -> None:
    if rc != 0:
        L = library()
        msg = L.snapgpu_last_error(ctx).decode()
        raise _ERRS.get(rc, PipelineError)(msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def counts(twojmax: int) -> dict:
    """Index-map sizes (HalfIntIndexMaps, halfint_index.hpp:85-98)."""
    out = np.zeros(6, np.int32)
    _check(library().snapgpu_counts(int(twojmax), out.ctypes.data))
    keys = ("n_triples", "n_tuples", "u_full_total", "u_half_total", "z_total_elements",
            "cg_total")
    return dict(zip(keys, (int(x) for x in out)))


@dataclass
class Problem:
    """snapforge::Problem + SnapParams (snap_core.hpp:48-119), flattened.

    numneigh[i] neighbors of atom i live in slots k < numneigh[i] of
    nbr[i, k] (int32) and disp[i, k, :] (float64, center -> neighbor).
    """

    twojmax: int = 8
    rcut: float = 4.7
    rmin0: float = 0.0
    rfac0: float = 0.99363
    wself: float = 1.0
    self_flag: int = 1
    beta: np.ndarray = field(default_factory=lambda: np.zeros(0))
    weights: np.ndarray = field(default_factory=lambda: np.ones(1))
    numneigh: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    nbr: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.int32))
    disp: np.ndarray = field(default_factory=lambda: np.zeros((0, 0, 3)))
    types: Optional[np.ndarray] = None
    positions: Optional[np.ndarray] = None
    box: Optional[np.ndarray] = None
    seed: int = 0             # Problem::seed (snap_core.hpp:70)
    synthetic: bool = False   # Problem::synthetic (:71)
    box_length: float = 0.0   # Problem::box_length (:69): cubic edge, 0 if not periodic

    @property
    def natoms(self) -> int:
        return int(np.asarray(self.numneigh).shape[0])

    @property
    def stride(self) -> int:
        nbr = np.asarray(self.nbr)
        return int(nbr.shape[1]) if nbr.ndim == 2 else int(nbr.size // max(self.natoms, 1))

    @property
    def npairs(self) -> int:
        return int(np.asarray(self.numneigh).sum())

    @classmethod
    def from_any(cls, p) -> "Problem":
        if isinstance(p, cls):
            return p
        kw = {k: getattr(p, k) for k in ("twojmax", "rcut", "rmin0", "rfac0", "wself",
                                          "self_flag", "beta", "numneigh", "nbr", "disp")}
        for k in ("weights", "types", "positions", "box", "seed", "synthetic", "box_length"):
            if getattr(p, k, None) is not None:
                kw[k] = getattr(p, k)
        return cls(**kw)

    def validate(self) -> "Problem":
        """Problem::validate (snap_core.hpp:89-118) on the host arrays."""
        n = self.natoms
        nb = counts(self.twojmax)["n_triples"]
        if not (self.rcut > self.rmin0):
            raise InvalidArgument("problem: Rcut must exceed rmin0")
        if np.asarray(self.beta).size != nb:
            raise InvalidArgument("problem: beta length must match the triple count")
        w = np.asarray(self.weights)
        if w.size == 0:
            raise InvalidArgument("problem: empty weight table")
        if self.types is not None:
            t = np.asarray(self.types)
            if t.size != n or (n and (t.min() < 0 or t.max() >= w.size)):
                raise InvalidArgument("problem: atom type outside weight table")
        if self.positions is not None and np.asarray(self.positions).shape[0] not in (0, n):
            raise InvalidArgument("problem: positions/neighbors size mismatch")
        nn = np.asarray(self.numneigh)
        S = self.stride
        if n and (nn.min() < 0 or nn.max() > S):
            raise InvalidArgument("problem: neighbor count outside stride")
        mask = np.arange(S)[None, :] < nn[:, None]
        nbr = np.asarray(self.nbr).reshape(n, S)
        disp = np.asarray(self.disp).reshape(n, S, 3)
        if np.any(mask & ((nbr < 0) | (nbr >= n))):
            raise InvalidArgument("problem: neighbor index out of range")
        if np.any(mask & (nbr == np.arange(n)[:, None])):
            raise InvalidArgument("problem: self neighbor")
        r2 = (disp * disp).sum(-1)
        if np.any(mask & ~(r2 > 0.0)):
            raise InvalidArgument("problem: zero-length neighbor displacement")
        if np.any(mask & ~(r2 < self.rcut * self.rcut)):
            raise InvalidArgument("problem: neighbor at or beyond Rcut")
        return self


@dataclass
class PipelineResult:
    """The parts of snapforge::PipelineResult (pipeline.hpp:47-70) the GPU path fills."""

    forces: np.ndarray
    eatom: np.ndarray
    etotal: float
    stage_ms: Optional[dict] = None


class SnapEngine:
    """A device context: tables uploaded once, stages launched stream-ordered.

    Mirrors the reference's DescriptorState + stage functions; the arrays
    live in HBM and are read back only through the getters.
    """

    def __init__(self, twojmax=8, rcut=4.7, rmin0=0.0, rfac0=0.99363, wself=1.0,
                 self_flag=1, beta=None, weights=(1.0,), device=0):
        L = library()
        self._L = L
        self.twojmax = int(twojmax)
        self._beta = np.ascontiguousarray(beta, np.float64)
        self._weights = np.ascontiguousarray(weights, np.float64)
        h = C.c_void_p()
        _check(L.snapgpu_create(int(device), self.twojmax, float(rcut), float(rmin0),
                                float(rfac0), float(wself), int(self_flag),
                                self._beta.ctypes.data, int(self._beta.size),
                                self._weights.ctypes.data, int(self._weights.size),
                                C.byref(h)))
        self._h = h
        self.natoms_total = 0
        self.nlocal = 0
        self.stride = 0
        self._keep = ()
        self._args = {}  # per-argument (object, array, pointer) of the last step call

    @classmethod
    def for_problem(cls, p, device=0) -> "SnapEngine":
        p = Problem.from_any(p)
        return cls(p.twojmax, p.rcut, p.rmin0, p.rfac0, p.wself, p.self_flag, p.beta,
                   p.weights, device)

    # -- lifetime ----------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._L.snapgpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    def _c(self, rc):
        _check(rc, self._h)

    # -- inputs ------------------------------------------------------------
    def set_stream(self, cuda_stream_handle: int | None):
        """Run on a caller stream (e.g. torch.cuda.current_stream().cuda_stream).

        Handle 0 is CUDA's legacy default stream, which the C-ABI spells
        cudaStreamLegacy (0x1); None restores the engine's own stream."""
        if cuda_stream_handle == 0:
            cuda_stream_handle = 1  # cudaStreamLegacy
        self._c(self._L.snapgpu_set_stream(self._h, cuda_stream_handle))

    def set_beta(self, beta):
        b = np.ascontiguousarray(beta, np.float64)
        self._c(self._L.snapgpu_set_beta(self._h, b.ctypes.data, int(b.size)))
        self._beta = b

    def set_neighbors(self, numneigh, nbr, disp, types=None):
        nn = np.ascontiguousarray(numneigh, np.int32)
        nb = np.ascontiguousarray(nbr, np.int32)
        dp = np.ascontiguousarray(disp, np.float64)
        ty = None if types is None else np.ascontiguousarray(types, np.int32)
        n = int(nn.shape[0])
        stride = int(nb.shape[1]) if nb.ndim == 2 else int(nb.size // max(n, 1))
        self._c(self._L.snapgpu_set_neighbors(self._h, n, stride, nn.ctypes.data,
                                              nb.ctypes.data, dp.ctypes.data, _ptr(ty)))
        self.natoms_total, self.nlocal, self.stride = n, n, stride
        self._keep = (nn, nb, dp, ty)

    def set_problem(self, p):
        p = Problem.from_any(p)
        self.set_neighbors(p.numneigh, p.nbr, p.disp, p.types)

    def set_neighbors_partition(self, natoms_total, atom_lo, numneigh, nbr, disp, types=None):
        nn = np.ascontiguousarray(numneigh, np.int32)
        nb = np.ascontiguousarray(nbr, np.int32)
        dp = np.ascontiguousarray(disp, np.float64)
        ty = None if types is None else np.ascontiguousarray(types, np.int32)
        n = int(nn.shape[0])
        stride = int(nb.shape[1]) if nb.ndim == 2 else int(nb.size // max(n, 1))
        self._c(self._L.snapgpu_set_neighbors_partition(
            self._h, int(natoms_total), int(atom_lo), n, stride, nn.ctypes.data,
            nb.ctypes.data, dp.ctypes.data, _ptr(ty)))
        self.natoms_total, self.nlocal, self.stride = int(natoms_total), n, stride
        self._keep = (nn, nb, dp, ty)

    # -- stages (snap_core.hpp) ---------------------------------------------
    def compute_U(self):
        self._c(self._L.snapgpu_compute_U(self._h))

    def compute_Y(self):
        self._c(self._L.snapgpu_compute_Y(self._h))

    def compute_fused_dE(self):
        self._c(self._L.snapgpu_compute_dU_deidrj(self._h))

    compute_dU_deidrj = compute_fused_dE

    def scatter_forces(self):
        self._c(self._L.snapgpu_scatter_forces(self._h))

    def run(self):
        self._c(self._L.snapgpu_run(self._h))

    def _arg(self, slot, a, dtype):
        """(array, data pointer) of a step argument.  An argument that is
        already a C-contiguous `dtype` array is passed as it is, and the same
        object passed again (an MD loop reusing its pinned buffers) skips the
        conversion and the pointer lookup: the slot holds a reference, so the
        buffer cannot move.  Converted copies are never reused (the caller may
        change the source between calls)."""
        c = self._args.get(slot)
        if c is not None and c[0] is a:
            return c[1], c[2]
        arr = np.ascontiguousarray(a, dtype)
        ptr = arr.ctypes.data
        self._args[slot] = (a, arr, ptr) if arr is a else None
        return arr, ptr

    def step(self, numneigh, nbr, disp, types=None, forces=None, eatom=None, etotal=None,
             natoms_total=None, atom_lo=0, readback=True):
        """One end-to-end force step from host arrays (snapgpu_run_host): upload,
        run, read back; outputs are written into the given (ideally pinned)
        arrays when provided.  Returns (forces, eatom, etotal).  With
        readback=False nothing is read back (the results stay on the device,
        e.g. for the partitioned step's reduce-scatter) and None is returned."""
        nn, pn = self._arg(0, numneigh, np.int32)
        nb, pb = self._arg(1, nbr, np.int32)
        dp, pd = self._arg(2, disp, np.float64)
        ty, pt = (None, None) if types is None else self._arg(3, types, np.int32)
        n = int(nn.shape[0])
        stride = int(nb.shape[1]) if nb.ndim == 2 else int(nb.size // max(n, 1))
        ntot = n if natoms_total is None else int(natoms_total)
        if not readback:
            self._c(self._L.snapgpu_run_host(self._h, ntot, int(atom_lo), n, stride,
                                             pn, pb, pd, pt, None, None, None))
            self.natoms_total, self.nlocal, self.stride = ntot, n, stride
            self._keep = (nn, nb, dp, ty)
            return None
        f, pf = self._arg(4, forces if forces is not None else np.zeros((ntot, 3), np.float64),
                          np.float64)
        e, pe = self._arg(5, eatom if eatom is not None else np.zeros(n, np.float64), np.float64)
        t, ptt = self._arg(6, etotal if etotal is not None else np.zeros(1, np.float64),
                           np.float64)
        self._c(self._L.snapgpu_run_host(self._h, ntot, int(atom_lo), n, stride, pn, pb, pd, pt,
                                         pf, pe, ptt))
        self.natoms_total, self.nlocal, self.stride = ntot, n, stride
        self._keep = (nn, nb, dp, ty)
        return f, e, float(t[0])

    def synchronize(self):
        self._c(self._L.snapgpu_synchronize(self._h))

    def tune(self, y_parts=0):
        """compute_Y CTAs per 32-atom tile, 1..8 (0 = automatic)."""
        self._c(self._L.snapgpu_tune(self._h, int(y_parts)))

    def set_overlap(self, on=True):
        """compute_fused_dE starting per tile while compute_Y runs (2J <= 8;
        default on, off under ncu / compute-sanitizer)."""
        self._c(self._L.snapgpu_set_overlap(self._h, int(bool(on))))

    def set_force_layout(self, nchunks=1, ext_forces_ptr=None):
        """Chunked force output for the partitioned multi-GPU step
        (snapgpu_set_force_layout): one chunk of ceil(natoms/nchunks) atoms
        plus an energy slot per rank, optionally written straight into a
        caller-owned device buffer.  Takes effect at the next list upload."""
        self._c(self._L.snapgpu_set_force_layout(self._h, int(nchunks), ext_forces_ptr))
        self._nchunks = int(nchunks)

    def enable_stage_timing(self, on=True):
        self._c(self._L.snapgpu_enable_stage_timing(self._h, int(bool(on))))

    def stage_times(self) -> dict:
        out = np.zeros(4, np.float32)
        self._c(self._L.snapgpu_stage_times(self._h, out.ctypes.data))
        return dict(zip(("U", "Y", "dE", "forces"), (float(x) for x in out)))

    # -- outputs -------------------------------------------------------------
    def forces(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        """natoms_total x 3 forces (with a chunked layout: the raw chunks)."""
        nch = getattr(self, "_nchunks", 1)
        if nch > 1:
            k = -(-self.natoms_total // nch)
            f = out if out is not None else np.zeros(nch * (3 * k + 1), np.float64)
        else:
            f = out if out is not None else np.zeros((self.natoms_total, 3), np.float64)
        self._c(self._L.snapgpu_get_forces(self._h, f.ctypes.data))
        return f

    def energy(self):
        e = np.zeros(self.nlocal, np.float64)
        t = np.zeros(1, np.float64)
        self._c(self._L.snapgpu_get_energy(self._h, e.ctypes.data, t.ctypes.data))
        return e, float(t[0])

    def ulisttot(self) -> np.ndarray:
        nh = counts(self.twojmax)["u_half_total"]
        o = np.zeros((self.nlocal, nh, 2), np.float64)
        self._c(self._L.snapgpu_get_ulisttot(self._h, o.ctypes.data))
        return o.view(np.complex128)[..., 0]

    def ylist(self) -> np.ndarray:
        nh = counts(self.twojmax)["u_half_total"]
        o = np.zeros((self.nlocal, nh, 2), np.float64)
        self._c(self._L.snapgpu_get_ylist(self._h, o.ctypes.data))
        return o.view(np.complex128)[..., 0]

    def set_positions(self, positions, box):
        """Build the neighbor lists on the GPU from positions (
        harness.hpp:119-202, bitwise the host builder's lists)."""
        pos = np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
        bx = np.ascontiguousarray(np.broadcast_to(np.asarray(box, np.float64), (3,)))
        self._c(self._L.snapgpu_set_positions(self._h, int(pos.shape[0]), pos.ctypes.data,
                                              bx.ctypes.data))
        self.nlocal = self.natoms_total = int(pos.shape[0])
        self.stride = int(self.neighbors(counts_only=True).max(initial=0))
        return self

    def step_positions(self, positions, box, forces=None, eatom=None, etotal=None):
        """One end-to-end force step from host positions (snapgpu_run_positions):
        one graph uploads them, rebuilds the neighbor lists on the device,
        runs the force step and reads the results back.  Returns
        (forces, eatom, etotal)."""
        pos, pp = self._arg(7, positions, np.float64)
        if pos.size % 3:
            raise ValueError("positions: expected (natoms, 3) coordinates")
        n = int(pos.size // 3)
        if isinstance(box, np.ndarray) and box.shape == (3,):
            bx, pbx = self._arg(8, box, np.float64)
        else:
            bx = np.ascontiguousarray(np.broadcast_to(np.asarray(box, np.float64), (3,)))
            pbx = bx.ctypes.data
        f, pf = self._arg(4, forces if forces is not None else np.zeros((n, 3), np.float64),
                          np.float64)
        e, pe = self._arg(5, eatom if eatom is not None else np.zeros(n, np.float64), np.float64)
        t, ptt = self._arg(6, etotal if etotal is not None else np.zeros(1, np.float64),
                           np.float64)
        self._c(self._L.snapgpu_run_positions(self._h, n, pp, pbx, pf, pe, ptt))
        self.natoms_total = self.nlocal = n
        return f, e, float(t[0])

    def neighbors(self, counts_only=False):
        """(numneigh, nbr, disp) of the current lists, read back from the device."""
        nn = np.zeros(self.nlocal, np.int32)
        if counts_only:
            self._c(self._L.snapgpu_get_neighbors(self._h, nn.ctypes.data, None, None))
            return nn
        nbr = np.zeros((self.nlocal, self.stride), np.int32)
        disp = np.zeros((self.nlocal, self.stride, 3), np.float64)
        self._c(self._L.snapgpu_get_neighbors(self._h, nn.ctypes.data, nbr.ctypes.data,
                                              disp.ctypes.data))
        return nn, nbr, disp

    def descriptors(self) -> np.ndarray:
        """B_l(i), shape (nlocal, ntriples) (compute_B_from_U)."""
        nt = counts(self.twojmax)["n_triples"]
        o = np.zeros((self.nlocal, nt), np.float64)
        self._c(self._L.snapgpu_compute_descriptors(self._h, o.ctypes.data))
        return o

    def virial(self) -> np.ndarray:
        """W_xx, W_yy, W_zz, W_xy, W_xz, W_yz = sum_pairs r_ik (x) (-dE_ik)."""
        o = np.zeros(6, np.float64)
        self._c(self._L.snapgpu_get_virial(self._h, o.ctypes.data))
        return o

    def dedr(self) -> np.ndarray:
        o = np.zeros((self.nlocal, self.stride, 3), np.float64)
        self._c(self._L.snapgpu_get_dedr(self._h, o.ctypes.data))
        return o

    def forces_to_device(self, dst_ptr: int):
        """Stream-ordered D2D copy of the force buffer into device memory dst_ptr."""
        self._c(self._L.snapgpu_get_forces_device(self._h, dst_ptr))

    def energy_to_device(self, etotal_ptr: int, eatom_ptr: int | None = None):
        """Stream-ordered D2D copy of the owned total energy (and per-atom energies)."""
        self._c(self._L.snapgpu_get_energy_device(self._h, eatom_ptr, etotal_ptr))

    def device_outputs(self):
        f, e, t = C.c_void_p(), C.c_void_p(), C.c_void_p()
        self._c(self._L.snapgpu_device_outputs(self._h, C.byref(f), C.byref(e), C.byref(t)))
        return f.value, e.value, t.value


def run_pipeline(problem, device=0, stage_timing=False) -> PipelineResult:
    """run_pipeline (pipeline.hpp:206-303) for the fused adjoint path on the GPU."""
    p = Problem.from_any(problem)
    with SnapEngine.for_problem(p, device) as eng:
        if stage_timing:
            eng.enable_stage_timing(True)
        f, e, t = eng.step(p.numneigh, p.nbr, p.disp, p.types)
        st = eng.stage_times() if stage_timing else None
    return PipelineResult(forces=f, eatom=e, etotal=t, stage_ms=st)


def fp64_peak(device=0, iters=200000):
    """Measured FP64 DFMA throughput (TFLOP/s) of `device` (diagnostic probe)."""
    t = np.zeros(1)
    ms = np.zeros(1)
    _check(library().snapgpu_fp64_peak(int(device), int(iters), t.ctypes.data, ms.ctypes.data))
    return float(t[0]), float(ms[0])


def build_neighborlist(positions, box, rcut):
    """harness::build_neighborlist (harness.hpp:119-202), orthorhombic boxes."""
    L = library()
    pos = np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
    n = pos.shape[0]
    bx = np.ascontiguousarray(np.broadcast_to(np.asarray(box, np.float64), (3,)))
    numneigh = np.zeros(n, np.int32)
    mx = L.snapgpu_build_neighborlist(pos.ctypes.data, n, bx.ctypes.data, float(rcut), 0,
                                      numneigh.ctypes.data, None, None)
    if mx < 0:
        _check(-mx)
    s = max(mx, 1)
    nbr = np.zeros((n, s), np.int32)
    disp = np.zeros((n, s, 3), np.float64)
    mx = L.snapgpu_build_neighborlist(pos.ctypes.data, n, bx.ctypes.data, float(rcut), s,
                                      numneigh.ctypes.data, nbr.ctypes.data, disp.ctypes.data)
    if mx < 0:
        _check(-mx)
    return numneigh, nbr, disp


def bcc_problem(nx, ny, nz, twojmax=8, seed=2011, a=3.1803, jitter=0.05, rcut=4.7) -> Problem:
    """TestSNAP BCC tungsten: nx*ny*nz cells (2 atoms each), 26 neighbors per atom."""
    L = library()
    n = 2 * nx * ny * nz
    pos = np.zeros((n, 3), np.float64)
    beta = np.zeros(counts(twojmax)["n_triples"], np.float64)
    rc = L.snapgpu_bcc_lattice(int(nx), int(ny), int(nz), float(a), float(jitter),
                               int(seed), int(twojmax), pos.ctypes.data, beta.ctypes.data)
    if rc < 0:
        _check(-rc)
    box = np.array([nx * a, ny * a, nz * a])
    numneigh, nbr, disp = build_neighborlist(pos, box, rcut)
    return Problem(twojmax=int(twojmax), rcut=float(rcut), beta=beta, numneigh=numneigh,
                   nbr=nbr, disp=disp, positions=pos, box=box, seed=int(seed),
                   box_length=float(box[0]) if nx == ny == nz else 0.0)
