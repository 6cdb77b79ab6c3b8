"""Executed vs algorithmic FP64 rate per kernel from an ncu report
(the hardware analogue of the reference's analytic CounterModel,
pipeline.hpp:36-45).

    python tools/fp64_report.py REPORT.ncu-rep NATOMS NPAIRS TWOJMAX

Executed FLOPs = 2 DFMA + DMUL + DADD thread instructions
(sm__sass_thread_inst_executed_op_{dfma,dmul,dadd}_pred_on.sum; capture with
those metrics added to --set full).  Algorithmic FLOPs: the reference loop
nests (paper_2011_12875_b200/flops.py).  Durations are ncu's (cold cache,
serialised): the rates are per kernel under the profiler, not bench values.
"""
import csv
import io
import json
import subprocess
import sys

sys.path.insert(0, ".")
from paper_2011_12875_b200.flops import FP64_SPEC_TFLOPS, flop_model  # noqa: E402


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        yield {h: (v, u) for h, v, u in zip(hdr, row, units)}


def num(d, k):
    v, u = d.get(k, ("0", ""))
    v = float(str(v).replace(",", "") or 0)
    scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
             "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
             "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    return v * scale.get(u, 1.0)


def main():
    path, natoms, npairs, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    fm = flop_model(T)
    algo = {"k_compute_U": fm["U_per_pair"] * npairs, "k_compute_Y": fm["Y_per_atom"] * natoms,
            "k_fused_dE": fm["dE_per_pair"] * npairs}
    out = []
    for d in rows(path):
        name = d["Kernel Name"][0]
        t = num(d, "gpu__time_duration.sum")
        ex = (2 * num(d, "sm__sass_thread_inst_executed_op_dfma_pred_on.sum") +
              num(d, "sm__sass_thread_inst_executed_op_dmul_pred_on.sum") +
              num(d, "sm__sass_thread_inst_executed_op_dadd_pred_on.sum"))
        key = next((k for k in algo if k in name), None)
        rec = {"kernel": name.split("(")[0], "ncu_time_us": t * 1e6,
               "executed_flop": ex, "executed_tflops": ex / t / 1e12 if t else None,
               "executed_frac": ex / t / 1e12 / FP64_SPEC_TFLOPS if t else None,
               "fp64_pipe_pct": num(d, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
               "dram_bytes": num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum")}
        if key:
            rec.update({"algorithmic_flop": algo[key],
                        "algorithmic_tflops": algo[key] / t / 1e12 if t else None,
                        "algorithmic_frac": algo[key] / t / 1e12 / FP64_SPEC_TFLOPS if t else None,
                        "executed_over_algorithmic": ex / algo[key] if algo[key] else None})
        out.append(rec)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
