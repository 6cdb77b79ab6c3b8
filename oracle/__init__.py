"""Parity oracle for the B200 SNAP engine -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package, and only as
the checker or the timed CPU baseline.  The product package
``paper_2011_12875_b200`` never imports it.

Two CPU implementations are exposed through ctypes:

* ``port``  -- ``_build/liboracle.so``: our C99 restatement of the reference's
  deterministic ``fused`` path (``snap_oracle.c``; every function cites the
  reference file:line it follows).
* ``ref``   -- ``_ref/libsnapref.so``: the unmodified reference library
  (``/root/reference/proj/include/snapforge``) compiled in place through our
  ``ref_driver.cpp`` shim.  Absent on machines without ``/root/reference``
  unless the prebuilt ``.so`` travelled with the repo snapshot.

Problems are duck-typed: any object with the attributes of
``paper_2011_12875_b200.Problem`` (twojmax, rcut, rmin0, rfac0, wself,
self_flag, beta, weights, numneigh, nbr, disp, types) works.
"""
from __future__ import annotations

import ctypes as C
import os
from types import SimpleNamespace  # noqa: F401  (re-exported)

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(_HERE, "_build", "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libsnapref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def build(quiet: bool = True) -> None:
    """Compile the oracle port (and the reference shim when /root/reference exists)."""
    import subprocess

    subprocess.run(["make", "-C", _HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


class _Problem(C.Structure):
    _fields_ = [
        ("twojmax", C.c_int), ("rcut", C.c_double), ("rmin0", C.c_double),
        ("rfac0", C.c_double), ("wself", C.c_double), ("self_flag", C.c_int),
        ("beta", C.c_void_p), ("nbeta", C.c_int), ("weights", C.c_void_p),
        ("nweights", C.c_int), ("natoms", C.c_int), ("stride", C.c_int),
        ("numneigh", C.c_void_p), ("nbr", C.c_void_p), ("disp", C.c_void_p),
        ("types", C.c_void_p),
    ]


def _ptr(a):
    return None if a is None else a.ctypes.data


def _arrays(p):
    """Normalise a problem's arrays to contiguous numpy (kept alive by caller)."""
    d = SimpleNamespace()
    d.beta = np.ascontiguousarray(p.beta, dtype=np.float64)
    d.weights = np.ascontiguousarray(getattr(p, "weights", [1.0]), dtype=np.float64)
    d.numneigh = np.ascontiguousarray(p.numneigh, dtype=np.int32)
    d.nbr = np.ascontiguousarray(p.nbr, dtype=np.int32)
    d.disp = np.ascontiguousarray(p.disp, dtype=np.float64)
    t = getattr(p, "types", None)
    d.types = None if t is None else np.ascontiguousarray(t, dtype=np.int32)
    d.natoms = int(d.numneigh.shape[0])
    d.stride = int(d.nbr.shape[1]) if d.nbr.ndim == 2 else (int(d.nbr.size // max(d.natoms, 1)))
    return d


class Port:
    """ctypes view of our C restatement (oracle/_build/liboracle.so)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        L.orc_last_error.restype = C.c_char_p
        L.orc_run.argtypes = [C.POINTER(_Problem)] + [C.c_void_p] * 7
        L.orc_bcc.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                              C.c_uint64, C.c_int, _dp, _dp]
        L.orc_build_neighborlist.argtypes = [_dp, C.c_int, _dp, C.c_double, C.c_int,
                                             C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_make_cluster.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, _dp, _ip,
                                       _dp, _ip, _ip, _dp, _dp]
        L.orc_generate_synthetic.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double,
                                             C.c_uint64, _ip, _ip, _dp, _dp]
        L.orc_cg_table.argtypes = [C.c_int, _dp]
        L.orc_wigner_u_half.argtypes = [_dp, C.c_double, C.c_double, C.c_double,
                                        C.c_int, _dp]
        L.orc_map_to_3sphere.argtypes = [_dp, C.c_double, C.c_double, C.c_double, _dp]
        L.orc_rng_stream.argtypes = [C.c_uint64, C.c_int, _dp]
        for f in ("orc_n_triples", "orc_n_tuples", "orc_u_half_total", "orc_u_full_total",
                  "orc_z_total_elements", "orc_cg_total"):
            getattr(L, f).argtypes = [C.c_int]
        L.orc_triples.argtypes = [C.c_int, _ip]
        L.orc_tuples.argtypes = [C.c_int, _ip]

    def err(self):
        return self.L.orc_last_error().decode()

    # -- counts / tables --------------------------------------------------
    def counts(self, T):
        L = self.L
        return (L.orc_n_triples(T), L.orc_n_tuples(T), L.orc_u_full_total(T),
                L.orc_u_half_total(T), L.orc_z_total_elements(T), L.orc_cg_total(T))

    def cg_table(self, T):
        out = np.zeros(self.L.orc_cg_total(T), np.float64)
        self.L.orc_cg_table(T, out)
        return out

    def tuples(self, T):
        out = np.zeros((self.L.orc_n_tuples(T), 5), np.int32)
        self.L.orc_tuples(T, out.reshape(-1))
        return out

    def triples(self, T):
        out = np.zeros((self.L.orc_n_triples(T), 3), np.int32)
        self.L.orc_triples(T, out.reshape(-1))
        return out

    def wigner_u_half(self, disp, T, rcut=4.7, rmin0=0.0, rfac0=0.99363):
        out = np.zeros(2 * self.L.orc_u_half_total(T), np.float64)
        if self.L.orc_wigner_u_half(np.ascontiguousarray(disp, np.float64), rcut, rmin0,
                                    rfac0, T, out):
            raise ValueError(self.err())
        return out.view(np.complex128)

    def rng_stream(self, seed, n):
        out = np.zeros(n, np.float64)
        self.L.orc_rng_stream(seed, n, out)
        return out

    # -- pipeline ---------------------------------------------------------
    def run(self, p, want=("forces", "eatom", "etotal", "ulisttot", "ylist", "delist")):
        d = _arrays(p)
        T = int(p.twojmax)
        nh = self.L.orc_u_half_total(T)
        nt = self.L.orc_n_triples(T)
        N, S = d.natoms, d.stride
        out = {}
        shapes = {"forces": (N, 3), "eatom": (N,), "ulisttot": (N, nh, 2),
                  "ylist": (N, nh, 2), "delist": (N, S, 3), "blist": (N, nt)}
        for k, shp in shapes.items():
            out[k] = np.zeros(shp, np.float64) if (k in want) else None
        et = np.zeros(1, np.float64) if "etotal" in want else None
        prob = _Problem(T, float(p.rcut), float(p.rmin0), float(p.rfac0), float(p.wself),
                        int(p.self_flag), d.beta.ctypes.data, int(d.beta.size),
                        d.weights.ctypes.data, int(d.weights.size), N, S,
                        d.numneigh.ctypes.data, d.nbr.ctypes.data, d.disp.ctypes.data,
                        _ptr(d.types))
        rc = self.L.orc_run(C.byref(prob), _ptr(out["forces"]), _ptr(out["eatom"]),
                            _ptr(et), _ptr(out["ulisttot"]), _ptr(out["ylist"]),
                            _ptr(out["delist"]), _ptr(out["blist"]))
        if rc:
            raise ValueError(self.err())
        res = {k: v for k, v in out.items() if v is not None}
        for k in ("ulisttot", "ylist"):
            if k in res:
                res[k] = res[k].view(np.complex128)[..., 0]
        if et is not None:
            res["etotal"] = float(et[0])
        return res

    # -- generators -------------------------------------------------------
    def bcc(self, nx, ny, nz, T, a=3.1803, jitter=0.05, seed=2011):
        n = 2 * nx * ny * nz
        pos = np.zeros(n * 3, np.float64)
        beta = np.zeros(self.L.orc_n_triples(T), np.float64)
        self.L.orc_bcc(nx, ny, nz, a, jitter, seed, T, pos, beta)
        return pos.reshape(n, 3), beta, np.array([nx * a, ny * a, nz * a])

    def neighborlist(self, pos, box, rcut):
        pos = np.ascontiguousarray(pos, np.float64).reshape(-1)
        n = pos.size // 3
        box = np.ascontiguousarray(np.broadcast_to(np.asarray(box, np.float64), (3,)))
        numneigh = np.zeros(n, np.int32)
        mx = self.L.orc_build_neighborlist(pos, n, box, rcut, 0, numneigh.ctypes.data,
                                           None, None)
        if mx < 0:
            raise ValueError(self.err())
        nbr = np.zeros((n, max(mx, 1)), np.int32)
        disp = np.zeros((n, max(mx, 1), 3), np.float64)
        self.L.orc_build_neighborlist(pos, n, box, rcut, max(mx, 1), numneigh.ctypes.data,
                                      nbr.ctypes.data, disp.ctypes.data)
        return numneigh, nbr, disp

    def make_cluster(self, natoms, T, seed, ntypes=1):
        pos = np.zeros(natoms * 3, np.float64)
        types = np.zeros(natoms, np.int32)
        weights = np.zeros(ntypes, np.float64)
        numneigh = np.zeros(natoms, np.int32)
        nbr = np.zeros(natoms * natoms, np.int32)
        disp = np.zeros(natoms * natoms * 3, np.float64)
        beta = np.zeros(self.L.orc_n_triples(T), np.float64)
        self.L.orc_make_cluster(natoms, T, seed, ntypes, pos, types, weights, numneigh,
                                nbr, disp, beta)
        return SimpleNamespace(twojmax=T, rcut=4.7, rmin0=0.0, rfac0=0.99363, wself=1.0,
                               self_flag=1, beta=beta, weights=weights, types=types,
                               positions=pos.reshape(natoms, 3), numneigh=numneigh,
                               nbr=nbr.reshape(natoms, natoms),
                               disp=disp.reshape(natoms, natoms, 3))

    def synthetic(self, natoms, nnbor, T, seed=12345, rcut=4.7):
        numneigh = np.zeros(natoms, np.int32)
        nbr = np.zeros(natoms * nnbor, np.int32)
        disp = np.zeros(natoms * nnbor * 3, np.float64)
        beta = np.zeros(self.L.orc_n_triples(T), np.float64)
        self.L.orc_generate_synthetic(natoms, nnbor, T, rcut, seed, numneigh, nbr, disp,
                                      beta)
        return SimpleNamespace(twojmax=T, rcut=rcut, rmin0=0.0, rfac0=0.99363, wself=1.0,
                               self_flag=1, beta=beta, weights=np.ones(1), types=None,
                               numneigh=numneigh, nbr=nbr.reshape(natoms, nnbor),
                               disp=disp.reshape(natoms, nnbor, 3))

    def bcc_problem(self, nx, ny, nz, T, seed=2011, rcut=4.7):
        pos, beta, box = self.bcc(nx, ny, nz, T, seed=seed)
        numneigh, nbr, disp = self.neighborlist(pos, box, rcut)
        return SimpleNamespace(twojmax=T, rcut=rcut, rmin0=0.0, rfac0=0.99363, wself=1.0,
                               self_flag=1, beta=beta, weights=np.ones(1), types=None,
                               positions=pos, box=box, numneigh=numneigh, nbr=nbr,
                               disp=disp)


def ref_available(path: str = REF_SO) -> bool:
    return os.path.exists(path)


class Ref:
    """ctypes view of the unmodified reference (oracle/_ref/libsnapref.so)."""

    _PROB = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
             C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
             C.c_void_p, C.c_void_p, C.c_void_p]

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_run.argtypes = self._PROB + [C.c_char_p, C.c_int, C.c_int] + [C.c_void_p] * 7
        L.ref_time.argtypes = self._PROB + [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p]
        L.ref_build_neighborlist.argtypes = [_dp, C.c_int, C.c_double, C.c_double, C.c_int,
                                             C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_cg_table.argtypes = [C.c_int, _dp]
        L.ref_counts.argtypes = [C.c_int, _ip]
        L.ref_wigner_u_half.argtypes = [_dp, C.c_double, C.c_double, C.c_double, C.c_int,
                                        _dp]
        L.ref_make_cluster.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, _dp, _ip, _dp,
                                       _ip, _ip, _dp, _dp]
        L.ref_generate_synthetic.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double,
                                             C.c_uint64, _ip, _ip, _dp, _dp]
        L.ref_oracle_checks.argtypes = self._PROB + [C.c_uint64, _dp]
        L.ref_save_problem.argtypes = self._PROB + [C.c_uint64, C.c_int, C.c_double,
                                                    C.c_void_p, C.c_char_p]
        L.ref_resave_problem.argtypes = [C.c_char_p, C.c_char_p]

    def err(self):
        return self.L.ref_last_error().decode()

    def _pargs(self, p, d):
        return [int(p.twojmax), float(p.rcut), float(p.rmin0), float(p.rfac0),
                float(p.wself), int(p.self_flag), d.beta.ctypes.data, int(d.beta.size),
                d.weights.ctypes.data, int(d.weights.size), d.natoms, d.stride,
                d.numneigh.ctypes.data, d.nbr.ctypes.data, d.disp.ctypes.data,
                _ptr(d.types)]

    def counts(self, T):
        out = np.zeros(6, np.int32)
        if self.L.ref_counts(T, out):
            raise ValueError(self.err())
        return tuple(int(x) for x in out)

    def cg_table(self, T):
        n = self.counts(T)[5]
        out = np.zeros(n, np.float64)
        self.L.ref_cg_table(T, out)
        return out

    def wigner_u_half(self, disp, T, rcut=4.7, rmin0=0.0, rfac0=0.99363):
        n = self.counts(T)[3]
        out = np.zeros(2 * n, np.float64)
        if self.L.ref_wigner_u_half(np.ascontiguousarray(disp, np.float64), rcut, rmin0,
                                    rfac0, T, out):
            raise ValueError(self.err())
        return out.view(np.complex128)

    def run(self, p, variant="fused", deterministic=True, workers=1,
            want=("forces", "eatom", "etotal", "ulisttot", "ylist", "delist")):
        d = _arrays(p)
        T = int(p.twojmax)
        ntrip, _, _, nh, _, _ = self.counts(T)
        N, S = d.natoms, d.stride
        shapes = {"forces": (N, 3), "eatom": (N,), "ulisttot": (N, nh, 2),
                  "ylist": (N, nh, 2), "delist": (N, S, 3), "blist": (N, ntrip)}
        out = {k: (np.zeros(s, np.float64) if k in want else None) for k, s in shapes.items()}
        et = np.zeros(1, np.float64) if "etotal" in want else None
        rc = self.L.ref_run(*self._pargs(p, d), variant.encode(), int(deterministic),
                            int(workers), _ptr(out["forces"]), _ptr(out["eatom"]), _ptr(et),
                            _ptr(out["ulisttot"]), _ptr(out["ylist"]), _ptr(out["delist"]),
                            _ptr(out["blist"]))
        if rc:
            raise ValueError(self.err())
        res = {k: v for k, v in out.items() if v is not None}
        for k in ("ulisttot", "ylist"):
            if k in res:
                res[k] = res[k].view(np.complex128)[..., 0]
        if et is not None:
            res["etotal"] = float(et[0])
        return res

    def time(self, p, variant="fused", deterministic=True, workers=1, warmup=1, steps=5,
             with_energy=False, wall=False):
        """Per-step times (ms) of run_pipeline in the harness protocol
        (harness.hpp:534-556): PipelineResult::total_ms, the stage-time sum;
        with wall=True also the wall clock around each call."""
        d = _arrays(p)
        ms = np.zeros(steps, np.float64)
        wms = np.zeros(steps, np.float64)
        forces = np.zeros((d.natoms, 3), np.float64)
        et = np.zeros(1, np.float64)
        rc = self.L.ref_time(*self._pargs(p, d), variant.encode(), int(deterministic),
                             int(workers), int(warmup), int(steps), int(with_energy),
                             ms.ctypes.data, wms.ctypes.data, forces.ctypes.data,
                             et.ctypes.data)
        if rc:
            raise ValueError(self.err())
        if wall:
            return ms, wms, forces, float(et[0])
        return ms, forces, float(et[0])

    def neighborlist(self, pos, box, rcut):
        pos = np.ascontiguousarray(pos, np.float64).reshape(-1)
        n = pos.size // 3
        numneigh = np.zeros(n, np.int32)
        mx = self.L.ref_build_neighborlist(pos, n, float(box), rcut, 0,
                                           numneigh.ctypes.data, None, None)
        if mx < 0:
            raise ValueError(self.err())
        nbr = np.zeros((n, max(mx, 1)), np.int32)
        disp = np.zeros((n, max(mx, 1), 3), np.float64)
        self.L.ref_build_neighborlist(pos, n, float(box), rcut, max(mx, 1),
                                      numneigh.ctypes.data, nbr.ctypes.data,
                                      disp.ctypes.data)
        return numneigh, nbr, disp

    def make_cluster(self, natoms, T, seed, ntypes=1):
        pos = np.zeros(natoms * 3, np.float64)
        types = np.zeros(natoms, np.int32)
        weights = np.zeros(ntypes, np.float64)
        numneigh = np.zeros(natoms, np.int32)
        nbr = np.zeros(natoms * natoms, np.int32)
        disp = np.zeros(natoms * natoms * 3, np.float64)
        beta = np.zeros(self.counts(T)[0], np.float64)
        if self.L.ref_make_cluster(natoms, T, seed, ntypes, pos, types, weights, numneigh,
                                   nbr, disp, beta) < 0:
            raise ValueError(self.err())
        return SimpleNamespace(twojmax=T, rcut=4.7, rmin0=0.0, rfac0=0.99363, wself=1.0,
                               self_flag=1, beta=beta, weights=weights, types=types,
                               positions=pos.reshape(natoms, 3), numneigh=numneigh,
                               nbr=nbr.reshape(natoms, natoms),
                               disp=disp.reshape(natoms, natoms, 3))

    def synthetic(self, natoms, nnbor, T, seed=12345, rcut=4.7):
        numneigh = np.zeros(natoms, np.int32)
        nbr = np.zeros(natoms * nnbor, np.int32)
        disp = np.zeros(natoms * nnbor * 3, np.float64)
        beta = np.zeros(self.counts(T)[0], np.float64)
        if self.L.ref_generate_synthetic(natoms, nnbor, T, rcut, seed, numneigh, nbr, disp,
                                         beta):
            raise ValueError(self.err())
        return SimpleNamespace(twojmax=T, rcut=rcut, rmin0=0.0, rfac0=0.99363, wself=1.0,
                               self_flag=1, beta=beta, weights=np.ones(1), types=None,
                               numneigh=numneigh, nbr=nbr.reshape(natoms, nnbor),
                               disp=disp.reshape(natoms, nnbor, 3))

    def save_problem(self, p, path, seed=0, synthetic=False, box_length=0.0):
        """harness::save_problem (harness.hpp:770-775) of problem p."""
        d = _arrays(p)
        pos = getattr(p, "positions", None)
        pos = None if pos is None else np.ascontiguousarray(pos, np.float64)
        if self.L.ref_save_problem(*self._pargs(p, d), int(seed), int(bool(synthetic)),
                                   float(box_length), _ptr(pos), str(path).encode()):
            raise ValueError(self.err())

    def resave_problem(self, in_path, out_path):
        """harness::load_problem (validating) then harness::save_problem."""
        if self.L.ref_resave_problem(str(in_path).encode(), str(out_path).encode()):
            raise ValueError(self.err())

    def oracle_checks(self, p, seed=77):
        d = _arrays(p)
        out = np.zeros(3, np.float64)
        if self.L.ref_oracle_checks(*self._pargs(p, d), seed, out):
            raise ValueError(self.err())
        return {"rotation": out[0], "newton": out[1], "cross_pipeline": out[2]}
