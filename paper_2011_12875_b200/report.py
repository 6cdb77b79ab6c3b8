"""Run reports in the reference harness schema.

The reference harness writes one RunReport row per variant (harness.hpp:
510-675): CSV with the header `kCsvHeader` (harness.hpp:621-623) or JSON with
stage times, array bytes and counters (:640-672).  `gpu_row()` times the B200
engine on a problem and returns a row in that schema, variant "gpu-b200",
plus roofline columns appended after the reference's (algorithmic FP64
TFLOP/s of the step and its fraction of the B200 FP64 peak).  The force
checksum is the reference's FNV-1a over the IEEE bytes (common.hpp:81-99).
"""
from __future__ import annotations

import io
import json
import time

import numpy as np

from .flops import FP64_SPEC_TFLOPS as FP64_PEAK_TFLOPS
from .flops import step_flops

CSV_HEADER = ("variant,natoms,nnbor,twojmax,steps,wall_ms_per_step,katom_steps_per_s,"
              "speedup_vs_baseline,peak_bytes_total,force_checksum")  # harness.hpp:621-623
ROOFLINE_COLUMNS = ("step_tflops", "fp64_peak_frac")


def checksum_hex(x) -> str:
    """fnv1a_bits + checksum_hex (common.hpp:81-99) over the IEEE-754 bytes."""
    b = np.frombuffer(np.ascontiguousarray(x, np.float64).tobytes(), np.uint8)
    h = 0xcbf29ce484222325
    for v in b.tolist():
        h ^= v
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


def _fmt(v: float) -> str:  # detail::fmt_double: shortest round-trip text
    return repr(float(v))


def gpu_row(problem, steps: int = 20, baseline_ms: float | None = None, device: int = 0) -> dict:
    """Time `steps` force steps of the engine (graph replay, device resident
    lists) and return a RunReport row (harness.hpp:640-672 field names)."""
    import paper_2011_12875_b200 as snap

    p = snap.Problem.from_any(problem)
    eng = snap.SnapEngine.for_problem(p, device)
    try:
        eng.set_problem(p)
        eng.run()
        eng.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            eng.run()
        eng.synchronize()
        ms = (time.perf_counter() - t0) * 1e3 / steps
        eng.enable_stage_timing(True)
        eng.run()
        st = eng.stage_times()
        eng.enable_stage_timing(False)
        eng.run()
        f = eng.forces()
        _, etot = eng.energy()
    finally:
        eng.close()
    n, npairs = p.natoms, p.npairs
    nh = snap.counts(p.twojmax)["u_half_total"]
    array_bytes = {"ulisttot": n * nh * 16, "ylist": n * nh * 16,
                   "delist": n * p.stride * 24, "forces": n * 24,
                   "neighbors": n * p.stride * 28 + n * 4}
    flops = step_flops(p.twojmax, npairs, n)
    tflops = flops / (ms * 1e-3) / 1e12
    return {
        "variant": "gpu-b200", "natoms": n, "nnbor": int(p.stride), "twojmax": int(p.twojmax),
        "steps": steps, "wall_ms_per_step": ms, "katom_steps_per_s": n / ms,
        "speedup_vs_baseline": (baseline_ms / ms) if baseline_ms else 1.0,
        "peak_bytes_total": int(sum(array_bytes.values())),
        "force_checksum": checksum_hex(f), "energy_total": float(etot),
        "ok": True, "error": "", "unstable": False,
        "stage_ms": {"compute_U": st["U"], "compute_Y": st["Y"], "compute_fused_dE": st["dE"],
                     "scatter_forces": st["forces"]},
        "array_bytes": array_bytes,
        "counters": {"flops": flops, "bytes_loaded": 0, "bytes_stored": 0},
        "step_tflops": tflops, "fp64_peak_frac": tflops / FP64_PEAK_TFLOPS,
    }


def write_report_csv(rows, out=None) -> str:
    """CSV in the reference column order (write_report_csv, harness.hpp:625-634),
    roofline columns appended."""
    s = io.StringIO() if out is None else out
    s.write(CSV_HEADER + "," + ",".join(ROOFLINE_COLUMNS) + "\n")
    for r in rows:
        s.write(",".join([r["variant"], str(r["natoms"]), str(r["nnbor"]), str(r["twojmax"]),
                          str(r["steps"]), _fmt(r["wall_ms_per_step"]),
                          _fmt(r["katom_steps_per_s"]), _fmt(r["speedup_vs_baseline"]),
                          str(r["peak_bytes_total"]), r["force_checksum"],
                          _fmt(r["step_tflops"]), _fmt(r["fp64_peak_frac"])]) + "\n")
    return s.getvalue() if out is None else ""


def write_report_json(rows, config: dict) -> str:
    """JSON like write_report_json (harness.hpp:636-673)."""
    return json.dumps({"config": config, "rows": list(rows)}, indent=2)
