#!/usr/bin/env python
"""Benchmark of the B200 SNAP force step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], the metric's headline config): TestSNAP
2J=8 tungsten, BCC a = 3.1803 A, 2000 atoms per GPU (10x10x10 cells per GPU,
stacked along z for N GPUs: weak scaling), exactly 26 neighbors per atom,
synthetic positions (seeded jitter) and random beta (no checkpoints exist).

A step is one full force evaluation through the reference stage order
(run_pipeline adjoint branch, pipeline.hpp:234-272): compute_U, compute_Y
(+ per-atom energy), fused compute_dU/compute_deidrj, force scatter; with
N > 1 also the NCCL force reduce-scatter and energy all-reduce.

value    : whole-job Katom-steps/s (harness.hpp:443-447 grind definition),
           device-timed with CUDA events per step on the engine stream, L2
           flushed (256 MiB write) before every timed step, max over ranks.
e2e      : the same metric through the public API with HOST buffers: every
           step uploads that step's neighbor lists from pinned memory
           (snapgpu_set_neighbors, incl. Problem::validate) and reads forces
           and energies back (wall clock, synchronized).
roofline : FP64 SIMT (the CG contraction is sparse FP64; no tensor-core path):
           algorithmic FLOPs of the dominant kernel (SURVEY.md §8(d) counts,
           reference loop nests, mul and add counted separately) / its
           CUDA-event launch time, against the B200 FP64 spec peak.
cpu_baseline : the unmodified reference (oracle/_ref/libsnapref.so, fused
           variant, deterministic, WorkerPool over all host threads) timed on
           this box on a bounded sample of the same workload (rank 0, N=1).
"""
from __future__ import annotations

import argparse
import json
import os
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
CELLS_PER_GPU = (10, 10, 10)


# ---------------------------------------------------------------------------
# algorithmic work (exact trip counts of the reference nests)
# ---------------------------------------------------------------------------
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


def build_problem(snap, ngpus: int, twojmax: int):
    nx, ny, nz = CELLS_PER_GPU
    return snap.bcc_problem(nx, ny, nz * ngpus, twojmax=twojmax)


def cpu_reference_time(p, steps_cap=40, budget_s=12.0) -> dict:
    """Time the unmodified reference (oracle/_ref) fused-det run_pipeline."""
    import oracle

    R = oracle.Ref()
    workers = os.cpu_count() or 1
    ms, _, _ = R.time(p, "fused", True, workers, warmup=1, steps=1, with_energy=False)
    steps = int(max(2, min(steps_cap, budget_s / max(ms[0] * 1e-3, 1e-3))))
    ms, _, _ = R.time(p, "fused", True, workers, warmup=0, steps=steps, with_energy=False)
    secs = float(np.sum(ms)) * 1e-3
    return {"value": p.natoms * steps / secs / 1000.0, "unit": "Katom-steps/s",
            "cores": workers, "kind": "reference",
            "sample": f"{p.natoms}-atom BCC W, 2J={p.twojmax}, reference run_pipeline "
                      f"(fused, deterministic, force path) x {steps} steps after 1 warm-up, "
                      f"WorkerPool({workers})",
            "ms_per_step": secs * 1e3 / steps}


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle

    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libsnapref.so not built (needs /root/reference)"}))
        return 0
    import paper_2011_12875_b200 as snap  # problem generation only (host C++)

    n_gpus = args.gpus
    p = build_problem(snap, n_gpus, args.twojmax)
    sample_note = ""
    if p.natoms > 16000:  # bounded sample: same lattice, 16000 atoms
        p = snap.bcc_problem(20, 20, 20, twojmax=args.twojmax)
        sample_note = " (16000-atom sample of the workload; grind is per atom)"
    R = oracle.Ref()
    workers = os.cpu_count() or 1
    t_all = []
    R.time(p, "fused", True, workers, warmup=min(args.warmup, 1), steps=1)
    for _ in range(args.steps):
        ms, _, _ = R.time(p, "fused", True, workers, warmup=0, steps=1, with_energy=False)
        t_all.append(ms[0])
    secs = float(np.sum(t_all)) * 1e-3
    value = p.natoms * len(t_all) / secs / 1000.0
    line = {
        "metric": METRIC, "value": value, "unit": "Katom-steps/s", "n_gpus": n_gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3 / len(t_all),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": f"TestSNAP 2J={args.twojmax} tungsten BCC, "
                               f"{2000 * n_gpus} atoms x 26 neighbors{sample_note}",
                   "twojmax": args.twojmax, "natoms_timed": p.natoms},
        "cpu_baseline": {"value": value, "unit": "Katom-steps/s", "cores": workers,
                         "kind": "reference",
                         "sample": f"{p.natoms}-atom BCC, reference run_pipeline fused-det "
                                   f"force path, {len(t_all)} steps, WorkerPool({workers})"},
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

    n_gpus = ws
    T = args.twojmax
    p = build_problem(snap, n_gpus, T)
    N = p.natoms
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    from paper_2011_12875_b200.distributed import PartitionedEngine

    pe = PartitionedEngine(p, n_gpus, rank, dev, stream)
    eng = pe.eng
    lo, hi = pe.lo, pe.hi
    per = hi - lo
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
                   "dE": fm["dE_per_pair"] * npairs_local, "forces": 6 * npairs_local}
    dom = max(("U", "Y", "dE"), key=lambda k: stage_ms[k])
    achieved = stage_flops[dom] / (stage_ms[dom] * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"{dom}_bytes_per_launch")
        except Exception:
            traffic = None
    step_flops = sum(v for k, v in stage_flops.items() if k != "forces")
    whole_tflops = step_flops * n_gpus / (t_total * 1e-3 / args.steps) / 1e12

    # ---- end to end through the public API with host buffers ----------------
    e2e = None
    if not args.no_e2e:
        pin = [torch.from_numpy(a).pin_memory() for a in own]
        host_np = [t.numpy() for t in pin]
        f_host = torch.zeros((N, 3), dtype=torch.float64).pin_memory()
        e_host = torch.zeros(natoms_local, dtype=torch.float64).pin_memory().numpy()
        t_host = torch.zeros(1, dtype=torch.float64).pin_memory().numpy()
        h2d = sum(a.nbytes for a in host_np)
        d2h = (pe.f_own.numel() if n_gpus > 1 else N * 3) * 8 + natoms_local * 8 + 8

        def e2e_step():
            if n_gpus == 1:  # the public one-call API: upload, run, read back
                eng.step(*host_np, forces=f_host.numpy(), eatom=e_host, etotal=t_host)
            else:
                pe.upload(*host_np)
                step()
                f_host.view(-1)[: pe.f_own.numel()].copy_(pe.f_own, non_blocking=False)
                eng.energy()

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
               "ms_per_step": t_e2e * 1e3 / args.steps}

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
            cpu = cpu_reference_time(p)
        except Exception as e:  # oracle/_ref absent on this box
            cpu = {"value": None, "unavailable": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Katom-steps/s", "n_gpus": n_gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "grind_us_per_atom_step": 1000.0 / value,
            "config": {"workload": f"TestSNAP 2J={T} tungsten BCC, {per} atoms/GPU x 26 "
                                   f"neighbors (10x10x{10 * n_gpus} cells)",
                       "twojmax": T, "natoms_per_gpu": per, "natoms_total": N,
                       "neighbors_per_atom": 26,
                       "parallelism": f"atom-partition x{n_gpus}" + (
                           " + NCCL reduce-scatter(forces) + all-reduce(energy)"
                           if n_gpus > 1 else ""),
                       "l2": "flushed by a 256 MiB write before every timed step"},
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
            # our kernels per step: U, Y (+energy), fused dU/dE (+scatter when fused)
            "gpu_launches": (3 if per * p.stride <= (1 << 18) else 4) * args.steps,
            "reference_points": {"v100_kokkos_baseline_katom_steps_s": 32.8,
                                 "v100_final_lammps_derived_katom_steps_s": 643},
        }
        print(json.dumps(line))
    pe.close()
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--twojmax", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-probe", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ws, _, _ = dist_env()
    if ws > 1 and args.gpus != ws:
        args.gpus = ws
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
