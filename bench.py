#!/usr/bin/env python
"""Benchmark of the B200 EAM hot path (BASELINE.json metric: atom-steps/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one velocity-Verlet MD step (sim.cpp:248-273) -- kick/drift,
wrap + rehash + ghosts, density, embedding, force, kick + measure -- of
BASELINE config 2 (BCC Fe 50^3 = 250,000 atoms, 600 K + U(+-0.05 A)
displacements, dt = 1 fs), the configuration the metric is quoted on that
fits one GPU.  Inputs are synthetic (seeded, host-generated).

* value: device-resident steps, CUDA events per step on the library's stream,
  L2 evicted (512 MB write) before every timed step (the whole state is
  ~40 MB < 126 MB L2), max over ranks.
* e2e: the same steps through the reference-facing C ABI with HOST buffers:
  cbx_upload_store -> K x cbx_step(dt, 1) (StepState read on the host each
  step) -> cbx_download_store, transfers inside the timed region and
  amortised over the run; e2e.per_call re-uploads and downloads the whole
  store around every step.
* roofline: dominant kernel (force pass) against the measured fp64 peak.
* cpu_baseline / --impl reference: the reference core (oracle/_ref, built from
  /root/reference) on all host cores; the C restatement if that is absent.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "atom-steps/sec (fp64 EAM, 1/2/4/8 B200) and fraction of HBM/FP64 roofline"
UNIT = "atom-steps/s"
# canonical algorithmic work: per half-list candidate 8 flop,
# per in-cutoff pair 14 (density) / 44 (force), per atom 16 (embedding);
# compulsory fp64 SoA bytes per owned atom: density 32, embedding 16, force 56
FLOP_CAND, FLOP_DENS, FLOP_FORCE, FLOP_EMB = 8, 14, 44, 16
BYTES_DENS, BYTES_EMB, BYTES_FORCE = 32, 16, 56


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region"""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def table_path():
    from paper_2107_07866_b200.potential import write_baseline_table
    d = tempfile.mkdtemp(prefix="cbx_bench_")
    return write_baseline_table(os.path.join(d, "baseline.eam"))


# ------------------------------------------------------------- CPU arms
def reference_sim(w, path, workers):
    """the workload's initial state in the reference (oracle/_ref) or, where
    that was not built, the C restatement"""
    from oracle import oracle
    from paper_2107_07866_b200.workloads import displacements
    kind = "ref" if os.path.exists(oracle.REF_LIB) else "oracle"
    s = oracle.Sim(path, box=w.cells, temperature=w.temperature, seed=w.seed,
                   workers=workers, kind=kind)
    if w.displacement > 0:
        s.displace_interior(displacements(w, w.atoms))
        s.rehash()
        s.refresh_forces()
    return s, kind


def time_reference(w, path, steps, warmup, budget_s=None):
    cores = os.cpu_count() or 1
    s, kind = reference_sim(w, path, cores)
    s.step(w.dt, max(warmup, 1))
    t0 = time.perf_counter()
    done = 0
    while done < steps:
        s.step(w.dt, 1)
        done += 1
        if budget_s and time.perf_counter() - t0 > budget_s:
            break
    el = time.perf_counter() - t0
    # the reference colouring caps usable workers at box_z / 6 (forces.cpp:349-351)
    usable = min(cores, max(1, w.cells[2] // 6)) if kind == "ref" else 1
    return {"value": w.atoms * done / el, "unit": UNIT, "cores": usable if kind == "ref" else 1,
            "kind": "reference" if kind == "ref" else "port",
            "sample": f"{done} steps of {w.name} ({w.atoms} atoms) after {max(warmup, 1)} "
                      f"warm-up; {cores} host cores requested, WorkerPool uses "
                      f"{usable} (colouring cap box_z/6)",
            "seconds": el, "steps": done}


# -------------------------------------------------------------- our arm
def run_ours(args, w, path, ws, rank, local):
    from paper_2107_07866_b200 import EamPotential, _lib
    from paper_2107_07866_b200.workloads import build_device_state
    import ctypes as C

    lib = _lib.load()
    pot = EamPotential.load(path)
    slab = ws > 1 or args.slab
    if slab:
        # z-slab decomposition: rank r owns cells[2] planes of a box stacked
        # ws times along z; halos, migrants and the StepState reduction go
        # through NCCL inside each rank's step graph
        from paper_2107_07866_b200.workloads import build_slab_state
        dev, n = build_slab_state(w, pot, rank, ws, device=local, stencil=args.stencil,
                                  transport=args.transport)
    else:
        dev, n = build_device_state(w, pot, device=local, stencil=args.stencil)
    cand, pairs = dev.count_pairs()  # candidates / in-cutoff pairs of one half-list pass
    peak = C.c_double()
    mhz = C.c_double()
    _lib.check(lib.cbx_fp64_peak(local, C.byref(peak), C.byref(mhz)))

    out = (C.c_double * 8)()
    _lib.check(lib.cbx_bench_steps(dev.h, w.dt, args.warmup, args.flush_mb, out), dev.h)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    l0 = dev.kernel_launches()
    with ClockSampler(local) as clocks:
        _lib.check(lib.cbx_bench_steps(dev.h, w.dt, args.steps, args.flush_mb, out), dev.h)
    launches = dev.kernel_launches() - l0
    # per-phase breakdown: a separate short run whose graph carries event
    # nodes between the phases (diagnostic; not part of the timed region)
    ph = (C.c_double * 8)()
    nph = max(5, min(args.steps, 20))
    _lib.check(lib.cbx_bench_phases(dev.h, 1), dev.h)
    _lib.check(lib.cbx_bench_steps(dev.h, w.dt, nph, args.flush_mb, ph), dev.h)
    _lib.check(lib.cbx_bench_phases(dev.h, 0), dev.h)
    t = {"step": out[5], "force_kernel": out[7]}
    phases = {"density": ph[0] / nph, "embed": ph[1] / nph, "force": ph[2] / nph,
              "store": ph[3] / nph, "integrate": ph[4] / nph, "step": ph[5] / nph,
              "force_kernel": ph[7] / nph}
    total_ms = t["step"]
    if ws > 1:
        import torch
        import torch.distributed as dist
        x = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        total_ms = float(x.item())
    value = ws * n * args.steps / (total_ms * 1e-3)

    # roofline of the dominant kernel (force pass), canonical flops per launch
    K = args.steps
    f_force = FLOP_CAND * cand + FLOP_FORCE * pairs
    f_dens = FLOP_CAND * cand + FLOP_DENS * pairs
    t_force = t["force_kernel"] / K * 1e-3  # the force kernel launch alone
    t_dens = phases["density"] * 1e-3  # density phase (kernel + its memsets), diagnostic run
    ach_force = f_force / t_force / 1e12
    prof = load_profile_traffic()
    roofline = {"bound": "fp64",
                "kernel": "force pass: k_force_lean_smem<Newton-3> (clash records in the same "
                          "launch); CUDA events around the launch inside the step graph",
                "achieved": ach_force, "peak": peak.value, "unit": "TFLOP/s",
                "frac": ach_force / peak.value,
                "peak_source": "measured fp64 DFMA stream (cbx_fp64_peak) on this GPU; "
                               "MEASURED_PEAKS.json has no fp64 entry",
                "traffic": prof.get("force_traffic"),
                "algorithmic_flop_per_launch": f_force,
                "candidates_per_launch": cand, "pairs_per_launch": pairs,
                "density_kernel": {"achieved": f_dens / t_dens / 1e12,
                                   "frac": f_dens / t_dens / 1e12 / peak.value},
                "eam_passes": {"achieved": (f_force + f_dens + FLOP_EMB * n) /
                               ((phases["force"] + phases["density"] + phases["embed"]) * 1e-3)
                               / 1e12},
                # the resource that binds the stencil passes (ncu, profiles/)
                "binding_resource": prof.get("binding_resource")}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm = peaks.get("hbm_gbs")
        roofline["hbm"] = {"achieved_gbs": BYTES_FORCE * n / t_force / 1e9, "peak_gbs": hbm,
                           "frac": BYTES_FORCE * n / t_force / 1e9 / hbm}
    except (OSError, ValueError):
        pass

    # e2e through the C ABI with host buffers
    e2e = run_e2e(dev, w, args.e2e_steps, ws, local)
    res = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded host-generated BCC lattice, MB velocities, displacements)",
           "config": {"workload": w.note, "atoms_per_gpu": n, "dt_ps": w.dt,
                      "stencil": args.stencil,
                      "l2": f"flushed before every timed step ({args.flush_mb:.0f} MB buffer written, then read back so the step starts on clean lines)",
                      "parallelism": (f"z-slab x{ws}, {getattr(dev, 'transport', args.transport)} halo/migrant "
                                      f"exchange + reduction inside the step graph"
                                      + (", density/force partials added into the neighbours' "
                                         "memory by the passes" if getattr(dev, "fused", False)
                                         else "")) if slab
                                     else "single-gpu",
                      "global_cells": [w.cells[0], w.cells[1], w.cells[2] * ws]},
           "roofline": roofline, "e2e": e2e, "gpu_launches": launches,
           "clocks": clocks.summary(),
           "kernels_ms_per_step": {k: v / K for k, v in t.items()},
           "phases_ms_per_step": phases,
           "fp64_peak_probe": {"tflops": peak.value, "sm_mhz_est": mhz.value},
           "engine": dev.describe()}
    return res


def _max_over_ranks(el, ws, local):
    if ws > 1:
        import torch
        import torch.distributed as dist
        x = torch.tensor([el], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        el = float(x.item())
    return el


def run_e2e(dev, w, steps, ws=1, local=0, per_call_steps=5):
    """End to end through the reference-facing C ABI with page-locked HOST
    buffers (every rank; the slowest rank's time counts).

    Run (the headline `e2e`): the way Simulation::step is driven -- the host
    store is uploaded (cbx_upload_store), `steps` x cbx_step(dt, 1), each
    returning the step's StepState to the host (sim.h:11-21: energies, KE,
    max speed), then the store is downloaded (cbx_download_store); all of it
    inside the timed region, the transfers amortised over the run.

    Per call (`per_call`): upload -> one step -> download every step (the
    parity-test boundary of a per-call eval_forces drop-in)."""
    import ctypes
    from paper_2107_07866_b200 import _lib
    from paper_2107_07866_b200.engine import pinned_store
    s = dev.download(out=pinned_store(dev.n_slots))  # page-locked host buffers
    nbytes_in = sum(getattr(s, k).nbytes for k in ("pos", "vel", "force", "rho", "df", "tag",
                                                   "valid", "ghost"))
    state_bytes = ctypes.sizeof(_lib.State)

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    barrier()
    t0 = time.perf_counter()
    dev.upload(s)
    energies = 0.0
    for _ in range(steps):
        st = dev.step(w.dt, 1)
        energies += st["kinetic"]  # the step's result read on the host
    s = dev.download(out=s)
    el = _max_over_ranks(time.perf_counter() - t0, ws, local)
    nbytes_out = sum(getattr(s, k).nbytes for k in ("pos", "vel", "force", "rho", "df", "tag",
                                                    "valid", "ghost", "clash_key", "clash_pos"))
    n = int((s.valid.astype(bool) & ~s.ghost.astype(bool)).sum()) * ws
    run = {"value": n * steps / el, "unit": UNIT,
           "h2d_bytes_per_step": int(nbytes_in / steps),
           "d2h_bytes_per_step": int(nbytes_out / steps + state_bytes), "steps": steps,
           "path": "cbx_upload_store -> %d x cbx_step(dt,1) (StepState to the host every step) "
                   "-> cbx_download_store, pinned host buffers, reference-id AoS layout "
                   "converted on the device" % steps}

    barrier()
    t0 = time.perf_counter()
    for _ in range(per_call_steps):
        dev.upload(s)
        dev.step(w.dt, 1)
        s = dev.download(out=s)
    el = _max_over_ranks(time.perf_counter() - t0, ws, local)
    run["per_call"] = {"value": n * per_call_steps / el, "unit": UNIT,
                       "h2d_bytes_per_step": int(nbytes_in),
                       "d2h_bytes_per_step": int(nbytes_out), "steps": per_call_steps,
                       "path": "cbx_upload_store -> cbx_step(dt,1) -> cbx_download_store "
                               "every step"}
    return run


def load_profile_traffic():
    p = os.path.join(ROOT, "profiles", "latest_traffic.json")
    try:
        return json.load(open(p))
    except (OSError, ValueError):
        return {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--stencil", default="newton3", choices=["newton3", "full"])
    ap.add_argument("--flush-mb", type=float, default=512.0)
    ap.add_argument("--e2e-steps", type=int, default=100)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="slab exchange: peer-memory kernels or NCCL send/recv")
    ap.add_argument("--slab", action="store_true",
                    help="use the slab path (NCCL self-exchange) also at N=1")
    args = ap.parse_args()
    ws, rank, local = dist_env()
    from paper_2107_07866_b200.workloads import CONFIGS
    w = CONFIGS[args.config]
    path = table_path()

    if args.impl == "reference":
        if rank != 0:
            return
        r = time_reference(w, path, args.steps, args.warmup)
        line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": ws,
                "steps": r["steps"], "warmup": args.warmup,
                "ms_per_step": r["seconds"] / r["steps"] * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": w.note, "atoms": w.atoms, "dt_ps": w.dt},
                "impl": "reference",
                "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    res = run_ours(args, w, path, ws, rank, local)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cb = time_reference(w, path, 10_000, 1, budget_s=args.cpu_budget)
        res["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(res), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
