#!/usr/bin/env python
"""Benchmark of the B200 EAM hot path (BASELINE.json metric: atom-steps/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--scaling weak|strong] [--config c1..c5]

A "step" is one velocity-Verlet MD step (sim.cpp:248-273) -- kick/drift,
wrap + rehash + ghosts, density, embedding, force, kick + measure.

Workloads (BASELINE.json configs, synthetic seeded inputs):
* --scaling weak (default): config 5, BCC Fe 256^3 cells = 33,554,432 atoms
  PER GPU, 600 K, one 20 keV PKA per GPU subdomain, dt = 1 fs.  At N = 1 this
  is the configuration the metric is quoted on; at N > 1 the global box stacks
  N subdomains along z (z-slab decomposition, one rank per GPU).
* --scaling strong: config 4, BCC Fe 200^3 = 16,000,000 atoms in total, one
  5 keV PKA at the centre, dt = 0.2 fs, split into N z-slabs.

* value: device-resident steps, CUDA events per step on the library's stream,
  max over ranks.  The state (>= 2.5 GB per GPU) is larger than the 126 MB
  L2, so no flush is needed between steps (configs 1-3 flush a 512 MB buffer).
* e2e: the same steps through the reference-facing C ABI with HOST buffers:
  cbx_upload_store -> K x cbx_step(dt, 1) (StepState read on the host each
  step) -> cbx_download_store, transfers inside the timed region and
  amortised over the run; e2e.per_call re-uploads and downloads the whole
  store around every step.
* roofline: dominant kernel (force pass) against the measured fp64 peak, with
  the flops it executes (52 per in-cutoff pair: the replayed mask skips the
  out-of-cutoff candidates).
* cpu_baseline / --impl reference: the reference core (oracle/_ref, built from
  /root/reference) on all host cores, a bounded number of steps of the same
  workload (one GPU subdomain); the C restatement if _ref is absent.
* --gpus N without a torchrun environment spawns the N ranks itself
  (torch.distributed.run, 127.0.0.1); under torchrun WORLD_SIZE must equal N.
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
L2_BYTES = 126 * 2 ** 20


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
                 "--format=csv,noheader,nounits", "-lms", "20"],
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
    that was not built, the C restatement: init_bcc, the displacements of
    config 2, the PKA of configs 3-5 (Simulation::inject_pka, sim.cpp:163-186)"""
    from oracle import oracle
    from paper_2107_07866_b200.workloads import displacements
    kind = "ref" if os.path.exists(oracle.REF_LIB) else "oracle"
    centre = tuple(c // 2 for c in w.cells)
    s = oracle.Sim(path, box=w.cells, temperature=w.temperature, seed=w.seed,
                   workers=workers, kind=kind, pka_energy_kev=w.pka_kev, pka_site=centre,
                   pka_dir=tuple(w.pka_dir))
    if w.displacement > 0:
        s.displace_interior(displacements(w, w.atoms))
        s.rehash()
        s.refresh_forces()
    if w.pka_kev > 0:
        s.inject_pka()
    return s, kind


def time_reference(w, path, steps, warmup, budget_s=None):
    """the reference's step loop on the host cores: `warmup` untimed steps
    (at most 1 when a budget is set), then timed steps until `steps` or the
    budget (a bounded sample of the workload; the line says how many)"""
    cores = os.cpu_count() or 1
    s, kind = reference_sim(w, path, cores)
    nw = max(1, min(warmup, 1) if budget_s else warmup)
    s.step(w.dt, nw)
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
            "sample": f"{done} steps of {w.name} ({w.atoms} atoms, one GPU subdomain"
                      f"{', %g keV PKA' % w.pka_kev if w.pka_kev else ''}) after {nw} "
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
        # z-slab decomposition: halos, migrants and the StepState reduction go
        # through the peer-memory (or NCCL) transport inside each rank's step
        # graph; weak: rank r owns cells[2] planes of a box stacked ws times
        # along z, one PKA per subdomain; strong: the box split ws ways
        from paper_2107_07866_b200.workloads import build_slab_state
        dev, n = build_slab_state(w, pot, rank, ws, device=local, stencil=args.stencil,
                                  transport=args.transport, scaling=args.scaling)
    else:
        dev, n = build_device_state(w, pot, device=local, stencil=args.stencil)
    n_total = n * ws if args.scaling == "weak" else w.atoms
    state_bytes = dev.memory_report()["slots"]
    flush_mb = args.flush_mb if args.flush_mb is not None else (
        0.0 if state_bytes > 4 * L2_BYTES else 512.0)
    cand, pairs = dev.count_pairs()  # candidates / in-cutoff pairs of one half-list pass
    peak = C.c_double()
    mhz = C.c_double()
    _lib.check(lib.cbx_fp64_peak(local, C.byref(peak), C.byref(mhz)))

    out = (C.c_double * 8)()
    _lib.check(lib.cbx_bench_steps(dev.h, w.dt, args.warmup, flush_mb, out), dev.h)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    l0 = dev.kernel_launches()
    with ClockSampler(local) as clocks:
        _lib.check(lib.cbx_bench_steps(dev.h, w.dt, args.steps, flush_mb, out), dev.h)
    launches = dev.kernel_launches() - l0
    st_end = dev.state()
    # the pair counts after the timed steps (the cascade changes them)
    cand2, pairs2 = dev.count_pairs()
    cand, pairs = (cand + cand2) / 2.0, (pairs + pairs2) / 2.0
    # per-phase breakdown: a separate short run whose graph carries event
    # nodes between the phases (diagnostic; not part of the timed region)
    ph = (C.c_double * 8)()
    nph = max(3, min(args.steps, 10))
    _lib.check(lib.cbx_bench_phases(dev.h, 1), dev.h)
    _lib.check(lib.cbx_bench_steps(dev.h, w.dt, nph, flush_mb, ph), dev.h)
    _lib.check(lib.cbx_bench_phases(dev.h, 0), dev.h)
    t = {"step": out[5], "force_kernel": out[7]}
    phases = {"density": ph[0] / nph, "embed": ph[1] / nph, "force": ph[2] / nph,
              "store": ph[3] / nph, "integrate": ph[4] / nph, "step": ph[5] / nph,
              "force_kernel": ph[7] / nph}
    total_ms = _max_over_ranks(t["step"], ws, local)
    value = n_total * args.steps / (total_ms * 1e-3)

    # roofline of the dominant kernel (force pass): the flops it executes --
    # the distance of each in-cutoff pair (8) and the pair arithmetic (44);
    # the mask replayed from the density pass skips the out-of-cutoff ones
    K = args.steps
    f_force = (FLOP_CAND + FLOP_FORCE) * pairs
    f_dens = FLOP_CAND * cand + FLOP_DENS * pairs
    t_force = t["force_kernel"] / K * 1e-3  # the force kernel launch alone
    t_dens = phases["density"] * 1e-3  # density phase (kernel + its memsets), diagnostic run
    ach_force = f_force / t_force / 1e12
    prof = load_profile_traffic(w.name)
    roofline = {"bound": "fp64",
                "kernel": "force pass: k_force_lean_smem<Newton-3> (clash records in the same "
                          "launch); CUDA events around the launch inside the step graph",
                "achieved": ach_force, "peak": peak.value, "unit": "TFLOP/s",
                "frac": ach_force / peak.value,
                "peak_source": "measured fp64 DFMA stream (cbx_fp64_peak) on this GPU; "
                               "MEASURED_PEAKS.json has no fp64 entry",
                "traffic": prof.get("force_traffic"),
                "traffic_source": prof.get("source"),
                "algorithmic_flop_per_launch": f_force,
                "flop_per_pair": FLOP_CAND + FLOP_FORCE,
                "candidates_per_launch": cand, "pairs_per_launch": pairs,
                "density_kernel": {"achieved": f_dens / t_dens / 1e12,
                                   "frac": f_dens / t_dens / 1e12 / peak.value,
                                   "traffic": prof.get("density_traffic")},
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
        t_emb = phases["embed"] * 1e-3
        roofline["embed_kernel"] = {"bound": "hbm",
                                    "achieved_gbs": BYTES_EMB * n / t_emb / 1e9,
                                    "frac": BYTES_EMB * n / t_emb / 1e9 / hbm}
    except (OSError, ValueError, ZeroDivisionError):
        pass

    # e2e through the C ABI with host buffers
    e2e = run_e2e(dev, w, args.e2e_steps, ws, local)
    if slab:
        par = (f"z-slab x{ws} ({args.scaling} scaling), {getattr(dev, 'transport', args.transport)} "
               f"halo/migrant exchange + reduction inside the step graph"
               + (", density/force partials added into the neighbours' memory by the passes"
                  if getattr(dev, "fused", False) else ""))
    else:
        par = "single-gpu"
    gz = w.cells[2] * ws if args.scaling == "weak" else w.cells[2]
    res = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
           "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
           "dtype": "f64",
           "data": "synthetic (seeded host-generated BCC lattice, MB velocities"
                   + (", PKA" if w.pka_kev else "") + ")",
           "config": {"workload": w.note, "atoms_total": n_total, "atoms_this_rank": n,
                      "dt_ps": w.dt, "stencil": args.stencil,
                      "l2": (f"flushed before every timed step ({flush_mb:.0f} MB buffer written, "
                             "then read back)") if flush_mb > 0 else
                            f"no flush: inputs larger than L2 ({state_bytes / 1e9:.2f} GB of "
                            "slot arrays per GPU vs 126 MB L2)",
                      "parallelism": par,
                      "global_cells": [w.cells[0], w.cells[1], gz],
                      "pka_kev": w.pka_kev,
                      "pka_per": ("subdomain" if args.scaling == "weak" else "box")
                      if w.pka_kev else None},
           "roofline": roofline, "e2e": e2e, "gpu_launches": launches,
           "clocks": clocks.summary(),
           "kernels_ms_per_step": {k: v / K for k, v in t.items()},
           "phases_ms_per_step": phases,
           "state_after_timed_steps": dict(
               {k: st_end[k] for k in ("step", "t", "kinetic", "pair", "embedding",
                                       "max_speed")},
               clash_records=int(dev.lib.cbx_clash_count(dev.h)),
               defects=_defects(dev)),
           "fp64_peak_probe": {"tflops": peak.value, "sm_mhz_est": mhz.value},
           "engine": dev.describe()}
    return res


def _defects(dev):
    """Wigner-Seitz (vacancies, interstitials, Frenkel pairs) of this rank's store"""
    try:
        return list(dev.count_defects())
    except Exception:  # noqa: BLE001 -- informational only
        return None


def _sum_over_ranks(v, ws, local):
    if ws > 1:
        import torch
        import torch.distributed as dist
        x = torch.tensor([float(v)], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(x, op=dist.ReduceOp.SUM)
        v = float(x.item())
    return v


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
    t1 = time.perf_counter()
    energies = 0.0
    for _ in range(steps):
        st = dev.step(w.dt, 1)
        energies += st["kinetic"]  # the step's result read on the host
    t2 = time.perf_counter()
    s = dev.download(out=s)
    t3 = time.perf_counter()
    el = _max_over_ranks(t3 - t0, ws, local)
    nbytes_out = sum(getattr(s, k).nbytes for k in ("pos", "vel", "force", "rho", "df", "tag",
                                                    "valid", "ghost", "clash_key", "clash_pos"))
    # atoms of the whole job: slot atoms + interior clash records of every rank
    n = int((s.valid.astype(bool) & ~s.ghost.astype(bool)).sum() + (s.clash_ghost == 0).sum())
    n = int(_sum_over_ranks(n, ws, local))
    run = {"value": n * steps / el, "unit": UNIT,
           "h2d_bytes_per_step": int(nbytes_in / steps),
           "d2h_bytes_per_step": int(nbytes_out / steps + state_bytes), "steps": steps,
           "path": "cbx_upload_store -> %d x cbx_step(dt,1) (StepState to the host every step) "
                   "-> cbx_download_store, pinned host buffers, reference-id AoS layout "
                   "converted on the device" % steps,
           "seconds": {"upload": t1 - t0, "steps": t2 - t1, "download": t3 - t2}}

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


def load_profile_traffic(config: str):
    """ncu dram bytes per launch of the force / density kernels measured on
    this configuration (profiles/traffic_<config>.json, written from a
    committed `ncu --set full` capture); {} when that config has none"""
    p = os.path.join(ROOT, "profiles", f"traffic_{config}.json")
    try:
        return json.load(open(p))
    except (OSError, ValueError):
        return {}


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: launch the N ranks (one per GPU)
    with torch.distributed.run on 127.0.0.1 and return its exit code"""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="ranks (one per GPU); spawns them when not under torchrun")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: config 5 per GPU (default); strong: config 4 split over N")
    ap.add_argument("--config", default=None, help="c1..c5 (default: c5 weak / c4 strong)")
    ap.add_argument("--stencil", default="newton3", choices=["newton3", "full"])
    ap.add_argument("--flush-mb", type=float, default=None,
                    help="L2 flush before each timed step (default: 512 MB when the state "
                         "fits in 4x L2, else none)")
    ap.add_argument("--e2e-steps", type=int, default=100)
    ap.add_argument("--cpu-budget", type=float, default=30.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="slab exchange: peer-memory kernels or NCCL send/recv")
    ap.add_argument("--slab", action="store_true",
                    help="use the slab path (self-exchange) also at N=1")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    ws, rank, local = dist_env()
    if args.gpus is not None and args.gpus != ws:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    from paper_2107_07866_b200.workloads import CONFIGS
    name = args.config or ("c5" if args.scaling == "weak" else "c4")
    w = CONFIGS[name]
    path = table_path()

    if args.impl == "reference":
        if rank != 0:
            return
        # a bounded sample of the workload: one GPU subdomain (weak) or the
        # whole box (strong), 1 warm-up step, timed steps within the budget
        budget = args.cpu_budget if w.atoms > 1_000_000 else None
        r = time_reference(w, path, args.steps, args.warmup, budget_s=budget)
        gz = w.cells[2] * ws if args.scaling == "weak" else w.cells[2]
        line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": ws,
                "steps": r["steps"], "warmup": args.warmup,
                "ms_per_step": r["seconds"] / r["steps"] * 1e3, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": w.note, "atoms_sampled": w.atoms, "dt_ps": w.dt,
                           "global_cells": [w.cells[0], w.cells[1], gz],
                           "pka_kev": w.pka_kev},
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
