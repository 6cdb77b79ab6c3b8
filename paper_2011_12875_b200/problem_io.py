"""Problem files in the reference schema.

harness::problem_to_json / problem_from_json (harness.hpp:698-780): a
versioned JSON snapshot (``"schema": 1``) of one Problem with the keys, key
order and nesting of the reference writer, doubles in shortest round-trip
form (Python's float repr, like nlohmann's dump), so a save/load cycle
reproduces the problem bit for bit and the CPU reference and this engine can
share inputs in both directions.  ``load_problem`` ends with
Problem::validate (snap_core.hpp:89-118) like problem_from_json (:766).
"""
from __future__ import annotations

import json
from typing import Any

import numpy as np

from . import InvalidArgument, Problem


def problem_to_json(p) -> dict:
    """harness.hpp:701-727, same key order."""
    p = Problem.from_any(p)
    n = p.natoms
    nn = np.asarray(p.numneigh)
    nbr = np.asarray(p.nbr).reshape(n, -1) if n else np.zeros((0, 0), np.int32)
    disp = np.asarray(p.disp).reshape(n, -1, 3) if n else np.zeros((0, 0, 3))
    pos = [] if p.positions is None else [[float(c) for c in x] for x in np.asarray(p.positions)]
    types = [] if p.types is None else [int(t) for t in np.asarray(p.types)]
    neighbors = []
    for i in range(n):
        neighbors.append([{"index": int(nbr[i, k]),
                           "disp": [float(disp[i, k, 0]), float(disp[i, k, 1]),
                                    float(disp[i, k, 2])]}
                          for k in range(int(nn[i]))])
    return {
        "schema": 1,
        "seed": int(p.seed),
        "synthetic": bool(p.synthetic),
        "box_length": float(p.box_length),
        "params": {"twojmax": int(p.twojmax), "rcut": float(p.rcut),
                   "rmin0": float(p.rmin0), "rfac0": float(p.rfac0),
                   "weights": [float(w) for w in np.asarray(p.weights)],
                   "wself": float(p.wself), "self_contribution": bool(p.self_flag),
                   "beta": [float(b) for b in np.asarray(p.beta)]},
        "positions": pos,
        "types": types,
        "neighbors": neighbors,
    }


def problem_from_json(j: Any) -> Problem:
    """harness.hpp:729-767: schema check, then the flattened Problem."""
    if not isinstance(j, dict) or j.get("schema", 0) != 1:
        raise InvalidArgument("problem file: unsupported schema")
    prm = j["params"]
    lists = j["neighbors"]
    n = len(lists)
    stride = max((len(l) for l in lists), default=0)
    numneigh = np.array([len(l) for l in lists], np.int32)
    nbr = np.zeros((n, stride), np.int32)
    disp = np.zeros((n, stride, 3), np.float64)
    for i, l in enumerate(lists):
        for k, e in enumerate(l):
            nbr[i, k] = int(e["index"])
            d = e["disp"]
            disp[i, k] = (float(d[0]), float(d[1]), float(d[2]))
    pos = j.get("positions") or []
    types = j.get("types") or []
    if pos and len(pos) != n:
        raise InvalidArgument("problem: positions/neighbors size mismatch")
    if types and len(types) != n:
        raise InvalidArgument("problem: types/neighbors size mismatch")
    bl = float(j["box_length"])
    return Problem(
        twojmax=int(prm["twojmax"]), rcut=float(prm["rcut"]), rmin0=float(prm["rmin0"]),
        rfac0=float(prm["rfac0"]), wself=float(prm["wself"]),
        self_flag=int(bool(prm["self_contribution"])),
        beta=np.array(prm["beta"], np.float64), weights=np.array(prm["weights"], np.float64),
        numneigh=numneigh, nbr=nbr, disp=disp,
        types=np.array(types, np.int32) if types else None,
        positions=np.array(pos, np.float64) if pos else None,
        box=np.array([bl, bl, bl]) if bl > 0 else None,
        seed=int(j["seed"]), synthetic=bool(j["synthetic"]), box_length=bl).validate()


def save_problem(p, path: str) -> None:
    """harness::save_problem (harness.hpp:769-775): indented JSON + newline."""
    with open(path, "w") as f:
        f.write(json.dumps(problem_to_json(p), indent=2))
        f.write("\n")


def load_problem(path: str) -> Problem:
    """harness::load_problem (harness.hpp:777-783)."""
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError as e:
        raise InvalidArgument(f"load_problem: cannot open '{path}'") from e
    return problem_from_json(j)
