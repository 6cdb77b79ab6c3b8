"""Summarise an ncu --set full report: key throughput / stall metrics per kernel."""
import csv, io, subprocess, sys, json

KEYS = [
    ("gpu__time_duration.sum", "duration_ns"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_pct"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_pct_active"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_cycles_pct_active"),
    ("sm__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("dram__bytes_read.sum", "dram_read_B"),
    ("dram__bytes_write.sum", "dram_write_B"),
    ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "dfma_thread_inst"),
    ("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "dmul_thread_inst"),
    ("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "dadd_thread_inst"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active_threads_per_inst"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock_hz"),
]
STALLS = "smsp__average_warp_latency_issue_stalled_"

def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        k = {"kernel": d.get("Kernel Name", "")[:40], "id": d.get("ID")}
        for m, name in KEYS:
            v = d.get(m)
            try:
                k[name] = float(v.replace(",", "")) if v not in (None, "") else None
            except ValueError:
                k[name] = v
        st = {}
        for m, v in d.items():
            if m.startswith("smsp__average_warp_latency_issue_stalled_") and m.endswith(".ratio"):
                try:
                    st[m[len("smsp__average_warp_latency_issue_stalled_"):-6]] = float(v)
                except ValueError:
                    pass
        if not st:
            for m, v in d.items():
                if m.startswith("smsp__pcsamp_warps_issue_stalled_") and not m.endswith("not_issued"):
                    try:
                        st[m[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(v.replace(",", ""))
                    except ValueError:
                        pass
        tot = sum(st.values()) or 1.0
        k["top_stalls"] = sorted(((s, round(v / tot, 3)) for s, v in st.items()), key=lambda x: -x[1])[:6]
        res.append(k)
    return res

if __name__ == "__main__":
    for path in sys.argv[1:]:
        print("==", path)
        for k in load(path):
            print(json.dumps(k))
