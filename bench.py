#!/usr/bin/env python
"""Benchmark of the B200 SNAP force step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2|C3|C4|C5]

Workloads (BASELINE.json configs; TestSNAP tungsten BCC, a = 3.1803 A, seeded
jitter, exactly 26 neighbors per atom, random beta, synthetic data):
    C2 (default, the metric's headline config[1]): 2J=8, 2000 atoms per GPU
        (10x10x10 cells per GPU, stacked along z for N GPUs: weak scaling)
    C3: 2J=8, 262,144 atoms (64x64x32 cells), 1 B200 (saturation study)
    C4: 2J=14, 32,768 atoms (32x32x16 cells), 1 B200 (high-J)
    C5: 2J=8, 262,144 atoms per GPU (64x64x32 cells per GPU along z), weak
        scaling with the NCCL force reduce-scatter
With --gpus N > 1 and no torchrun environment, bench.py re-launches itself
under torch.distributed.run with N ranks (one per GPU, 127.0.0.1).

A step is one full force evaluation in the reference stage order
(run_pipeline adjoint branch, pipeline.hpp:234-272): compute_U, compute_Y
(+ per-atom energy), fused compute_dU/compute_deidrj, deterministic force
scatter; with N > 1 also the one NCCL reduce-scatter that sums the partial
forces and the energy.

value    : whole-job Katom-steps/s (harness.hpp:443-447 grind definition),
           device-timed with CUDA events per step on the engine stream, L2
           flushed (256 MiB write) before every timed step, max over ranks.
e2e      : the same metric through the public one-call API with HOST
           buffers (wall clock, synced every call): every step moves that
           step's neighbor lists from pinned host memory to the GPU --
           compute_U reads them over PCIe while it computes and leaves the
           device copies (zero-copy; h2d_bytes_per_step counts them) --,
           validates them on the device, rebuilds the reverse index beside
           Y / dE, and lands forces and energies in the caller's pinned
           arrays (d2h_bytes_per_step).  e2e.positions: positions in, lists
           rebuilt on the device inside the step graph.
roofline : FP64 SIMT (the CG contraction is sparse FP64; no tensor-core path):
           algorithmic FLOPs of the dominant kernel (paper_2011_12875_b200.
           flops, reference loop nests, mul and add counted separately) / its
           CUDA-event launch time, against the B200 FP64 spec peak.
cpu_baseline : the unmodified reference (oracle/_ref/libsnapref.so, fused
           variant, deterministic, WorkerPool over all host threads) timed on
           this box on a bounded sample of the same workload (rank 0, N=1).
--impl reference : the same reference alone, with this arm's metric/config.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grind time µs/atom-step (Katom-steps/s), 2J=8 W, vs FP64 roofline"
FP64_SPEC_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 37.2: 148 SM x 64 DFMA/clk x 2 flop
CONFIGS = {
    "C2": {"cells": (10, 10, 10), "twojmax": 8,
           "desc": "2J=8 tungsten, 2000 atoms/GPU (paper headline, BASELINE.json configs[1])"},
    "C3": {"cells": (64, 64, 32), "twojmax": 8,
           "desc": "2J=8 tungsten, 262144 atoms, 1 B200 (saturation, configs[2])"},
    "C4": {"cells": (32, 32, 16), "twojmax": 14,
           "desc": "2J=14 tungsten, 32768 atoms, 1 B200 (high-J, configs[3])"},
    "C5": {"cells": (64, 64, 32), "twojmax": 8,
           "desc": "2J=8 tungsten weak scaling, 262144 atoms/GPU (configs[4])"},
}


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock + throttle reasons sampled (NVML, every ~2 ms) during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N

            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
            self.bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
                         "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
                         "sw_power_cap": 0x4}
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.N = None
        return self

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.samples.append(float(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.bits.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *exc):
        self._stop.set()
        if getattr(self, "t", None):
            self.t.join(timeout=2)

    def summary(self) -> dict:
        s = self.samples
        return {"sm_mhz": statistics.median(s) if s else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s), "source": "nvml"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload_cells(cfg: str, n_gpus: int):
    nx, ny, nz = CONFIGS[cfg]["cells"]
    return nx, ny, nz * n_gpus


def workload_config(args, n_gpus: int) -> dict:
    """The `config` object of both arms (identical, so the driver can pair them)."""
    c = CONFIGS[args.config]
    nx, ny, nz = c["cells"]
    per = 2 * nx * ny * nz
    return {"workload": f"{args.config}: TestSNAP {c['desc']}; {per} atoms/GPU x 26 neighbors "
                        f"({nx}x{ny}x{nz} BCC cells per GPU along z), {n_gpus} GPU(s)",
            "config_id": args.config, "twojmax": c["twojmax"], "natoms_per_gpu": per,
            "natoms_total": per * n_gpus, "neighbors_per_atom": 26,
            "parallelism": f"atom-partition x{n_gpus}" + (
                " + one NCCL reduce-scatter (forces + energy)" if n_gpus > 1 else ""),
            "l2": "flushed by a 256 MiB write before every timed step"}


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_distributed(args) -> int:
    """--gpus N without a torchrun environment: run N ranks under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------
# the reference (unmodified, oracle/_ref) on the host cores
# ---------------------------------------------------------------------------
def reference_problem(cells, T):
    """The workload built with the oracle generators only (no product code):
    BCC positions + beta (TestSNAP generator restated in oracle/snap_oracle.c)
    and the reference's own neighbor builder (harness.hpp:119-202, cubic)."""
    import oracle

    port = oracle.Port()
    pos, beta, box = port.bcc(*cells, T)
    if cells[0] == cells[1] == cells[2]:
        numneigh, nbr, disp = oracle.Ref().neighborlist(pos, float(box[0]), 4.7)
    else:  # the reference builder is cubic-only: its orthorhombic restatement
        numneigh, nbr, disp = port.neighborlist(pos, box, 4.7)
    from types import SimpleNamespace

    return SimpleNamespace(twojmax=T, rcut=4.7, rmin0=0.0, rfac0=0.99363, wself=1.0,
                           self_flag=1, beta=beta, weights=np.ones(1), types=None,
                           numneigh=numneigh, nbr=nbr, disp=disp)


def reference_sample_cells(cfg: str, n_gpus: int):
    """Bounded sample of the workload for the CPU arm: the workload itself
    when small, else a cubic lattice of the same material and band limit."""
    cells = workload_cells(cfg, n_gpus)
    natoms = 2 * cells[0] * cells[1] * cells[2]
    T = CONFIGS[cfg]["twojmax"]
    cap = 16000 if T <= 8 else 2000
    if natoms <= cap:
        return cells, ""
    side = 20 if T <= 8 else 10
    return (side, side, side), (f" (bounded sample: {2 * side ** 3} atoms of the same "
                                f"workload; grind is per atom)")


def cpu_reference_time(cfg: str, budget_s=12.0, steps_cap=40) -> dict:
    """cpu_baseline of our arm: the reference fused-det force path."""
    import oracle

    cells, note = reference_sample_cells(cfg, 1)
    T = CONFIGS[cfg]["twojmax"]
    p = reference_problem(cells, T)
    n = int(p.numneigh.shape[0])
    R = oracle.Ref()
    workers = os.cpu_count() or 1
    ms, _, _ = R.time(p, "fused", True, workers, warmup=1, steps=1)
    steps = int(max(2, min(steps_cap, budget_s / max(ms[0] * 1e-3, 1e-3))))
    ms, _, _ = R.time(p, "fused", True, workers, warmup=0, steps=steps)
    secs = float(np.sum(ms)) * 1e-3
    return {"value": n * steps / secs / 1000.0, "unit": "Katom-steps/s",
            "cores": workers, "kind": "reference", "cpu_model": cpu_model(),
            "sample": f"{n}-atom BCC W, 2J={T}, reference run_pipeline (fused, "
                      f"deterministic, force path; harness protocol: stage-time sum) x "
                      f"{steps} steps after 1 warm-up, WorkerPool({workers}){note}",
            "ms_per_step": secs * 1e3 / steps}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle

    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libsnapref.so not built (needs /root/reference)"}))
        return 0
    n_gpus = max(ws, args.gpus)
    cells, note = reference_sample_cells(args.config, n_gpus)
    T = CONFIGS[args.config]["twojmax"]
    p = reference_problem(cells, T)
    n = int(p.numneigh.shape[0])
    R = oracle.Ref()
    workers = os.cpu_count() or 1
    # harness protocol (harness.hpp:534-556): warm-up with energy, then the
    # force path; W warm-ups like our arm
    R.time(p, "fused", True, workers, warmup=args.warmup, steps=1)
    t_all, w_all = [], []
    for _ in range(args.steps):
        ms, wms, _, _ = R.time(p, "fused", True, workers, warmup=0, steps=1, wall=True)
        t_all.append(ms[0])
        w_all.append(wms[0])
    secs = float(np.sum(t_all)) * 1e-3
    value = n * len(t_all) / secs / 1000.0
    # the oracle path (v1, deterministic): BASELINE.md §3
    v1_steps = max(1, min(3, args.steps))
    ms1, _, _ = R.time(p, "v1", True, workers, warmup=1, steps=v1_steps)
    v1 = n * v1_steps / (float(np.sum(ms1)) * 1e-3) / 1000.0
    line = {
        "metric": METRIC, "value": value, "unit": "Katom-steps/s", "n_gpus": n_gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3 / len(t_all),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": workload_config(args, n_gpus),
        "cpu_baseline": {"value": value, "unit": "Katom-steps/s", "cores": workers,
                         "kind": "reference", "cpu_model": cpu_model(),
                         "sample": f"{n}-atom BCC W, 2J={T}, reference run_pipeline fused-det "
                                   f"force path (harness protocol: stage-time sum), "
                                   f"{len(t_all)} steps after {args.warmup} warm-ups, "
                                   f"WorkerPool({workers}){note}",
                         "wall_ms_per_step": float(np.mean(w_all)),
                         "v1_det_katom_steps_s": v1},
        "e2e": {"value": value, "unit": "Katom-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch

    ws, rank, local = dist_env()
    dist = None
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    import paper_2011_12875_b200 as snap
    from paper_2011_12875_b200.distributed import PartitionedEngine
    from paper_2011_12875_b200.flops import flop_model

    n_gpus = ws
    T = CONFIGS[args.config]["twojmax"]
    p = snap.bcc_problem(*workload_cells(args.config, n_gpus), twojmax=T)
    N = p.natoms
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    pe = PartitionedEngine(p, n_gpus, rank, dev, stream)
    eng = pe.eng
    lo, hi = pe.lo, pe.hi
    own = pe.own
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        if n_gpus == 1:
            eng.run()  # forces / energy stay resident; read back in the e2e leg
        else:
            pe.step()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(dev if ws == 1 else local) as clk:
        for s in range(args.steps):
            flush.fill_(float(s))  # evict L2 (> 126 MB) outside the timed window
            evs[s][0].record(stream)
            step()
            evs[s][1].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    t_local = float(np.sum(step_ms))
    if dist:
        tt = torch.tensor([t_local], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total = float(tt.item())
    else:
        t_total = t_local
    value = N * args.steps / (t_total * 1e-3) / 1000.0

    # ---- per-stage device times (events inside the engine, same stream) ----
    eng.enable_stage_timing(True)
    st = {"U": [], "Y": [], "dE": [], "forces": []}
    for s in range(args.steps):
        flush.fill_(float(s))
        eng.run()
        for k, v in eng.stage_times().items():
            st[k].append(v)
    eng.enable_stage_timing(False)
    stage_ms = {k: float(np.mean(v)) for k, v in st.items()}
    fm = flop_model(T)
    npairs_local = int(own[0].sum())
    natoms_local = hi - lo
    stage_flops = {"U": fm["U_per_pair"] * npairs_local,
                   "Y": fm["Y_per_atom"] * natoms_local,
                   "dE": fm["dE_per_pair"] * npairs_local}
    dom = max(("U", "Y", "dE"), key=lambda k: stage_ms[k])
    achieved = stage_flops[dom] / (stage_ms[dom] * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config, {}).get(f"{dom}_bytes_per_launch")
        except Exception:
            traffic = None
    step_flops = sum(stage_flops.values())
    whole_tflops = step_flops * n_gpus / (t_total * 1e-3 / args.steps) / 1e12

    # ---- end to end through the public API with host buffers ----------------
    e2e = None
    if not args.no_e2e:
        pin = [torch.from_numpy(a).pin_memory() for a in own]
        host_np = [t.numpy() for t in pin]
        if n_gpus == 1:
            f_host = torch.zeros((N, 3), dtype=torch.float64).pin_memory().numpy()
            e_host = torch.zeros(natoms_local, dtype=torch.float64).pin_memory().numpy()
            t_host = torch.zeros(1, dtype=torch.float64).pin_memory().numpy()
            d2h = f_host.nbytes + e_host.nbytes + 8
        else:
            c_host = torch.zeros(pe.chunk.numel(), dtype=torch.float64).pin_memory()
            d2h = c_host.numel() * 8
        h2d = sum(a.nbytes for a in host_np)

        def e2e_step():
            if n_gpus == 1:  # the public one-call API: upload, run, read back
                eng.step(*host_np, forces=f_host, eatom=e_host, etotal=t_host)
            else:  # the slab's lists in (read by compute_U), step, reduce-scatter, chunk out
                pe.step_host(*host_np)
                c_host.copy_(pe.chunk, non_blocking=True)
                stream.synchronize()

        for _ in range(max(1, args.warmup // 2)):
            e2e_step()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        t_e2e = time.perf_counter() - t0
        if dist:
            tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = float(tt.item())
        e2e = {"value": N * args.steps / t_e2e / 1000.0, "unit": "Katom-steps/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": t_e2e * 1e3 / args.steps,
               "path": "snapgpu_run_host: pinned neighbor lists in (read over PCIe by "
                       "compute_U), forces/energies out into pinned arrays"}
        if n_gpus == 1:
            # the MD-loop call: positions in (neighbor lists rebuilt on the
            # device every step inside the same graph), forces/energies out
            pos_h = torch.from_numpy(np.ascontiguousarray(p.positions)).pin_memory().numpy()
            for _ in range(max(1, args.warmup // 2)):
                eng.step_positions(pos_h, p.box, forces=f_host, eatom=e_host, etotal=t_host)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                eng.step_positions(pos_h, p.box, forces=f_host, eatom=e_host, etotal=t_host)
            t_pos = time.perf_counter() - t0
            e2e["positions"] = {"value": N * args.steps / t_pos / 1000.0,
                                "unit": "Katom-steps/s", "h2d_bytes_per_step": int(pos_h.nbytes),
                                "d2h_bytes_per_step": int(d2h),
                                "ms_per_step": t_pos * 1e3 / args.steps,
                                "path": "snapgpu_run_positions: positions in, lists rebuilt "
                                        "on the device in the step graph, forces/energies out"}

    # ---- FP64 issue-rate probe on this box --------------------------------
    probe = None
    if rank == 0 and not args.no_probe:
        try:
            probe, _ = snap.fp64_peak(dev, 400000)
        except Exception:
            probe = None

    cpu = None
    if rank == 0 and n_gpus == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_time(args.config)
        except Exception as e:  # oracle/_ref absent on this box
            cpu = {"value": None, "unavailable": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Katom-steps/s", "n_gpus": n_gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "grind_us_per_atom_step": 1000.0 / value,
            "config": workload_config(args, n_gpus),
            "stages_ms": stage_ms,
            "roofline": {"bound": "fp64", "kernel": dom, "achieved": achieved,
                         "peak": FP64_SPEC_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP64_SPEC_TFLOPS, "traffic": traffic,
                         "peak_source": "B200 FP64 spec (148 SM x 64 DFMA/clk x 2 x 1.965 GHz); "
                                        "MEASURED_PEAKS.json has no FP64 entry",
                         "peak_measured_dfma_probe": probe,
                         "algorithmic_flops_per_launch": stage_flops[dom],
                         "whole_step_tflops": whole_tflops,
                         "whole_step_frac": whole_tflops / (FP64_SPEC_TFLOPS * n_gpus)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk.summary(),
            # our kernels per timed step: U, Y (+energy), fused dU/dE, force gather
            "gpu_launches": 4 * args.steps,
            "reference_points": {"v100_kokkos_baseline_katom_steps_s": 32.8,
                                 "v100_final_lammps_derived_katom_steps_s": 643},
        }
        print(json.dumps(line))
    pe.close()
    if dist:
        dist.destroy_process_group()
    return 0


def run_dry(args):
    """Launch check without a GPU: each rank reports its place in the job."""
    ws, rank, local = dist_env()
    print(json.dumps({"dry_run": True, "rank": rank, "world": ws, "local_rank": local,
                      "config": workload_config(args, max(ws, 1))}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-probe", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ws, _, _ = dist_env()
    if ws == 1 and args.gpus > 1 and "LOCAL_RANK" not in os.environ:
        return relaunch_distributed(args)
    if ws > 1:
        args.gpus = ws
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
