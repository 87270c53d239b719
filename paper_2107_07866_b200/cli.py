"""Command-line front end: tools/src/main.cpp:1-200 restated over the device.

    python -m paper_2107_07866_b200 run --config FILE [--set key=value ...] [--quiet]
    python -m paper_2107_07866_b200 bench-mem --config FILE [--set key=value ...]
    python -m paper_2107_07866_b200 gen-potential [--output PATH] [--nrho N] [--nr N]
    python -m paper_2107_07866_b200 check --config FILE [--set key=value ...]

Same subcommands, options, config layering (config.py) and report lines as
the reference's ``cascademd`` tool.  Where the reference reports its CPU
worker partition, this front end reports the device (the B200 the context
runs on and the brick decomposition of the stencil passes); ``bench-mem``
reports the device structures instead of the 104-byte AoS records.
Errors print ``error: <what>`` on stderr and exit 1, as main.cpp:187-192.
"""
from __future__ import annotations

import argparse
import ctypes as C
import math
import sys
import time

from . import _lib
from .config import load_config, nrt_displacements


def _csv_time(t: float) -> str:  # analysis.cpp:67-76
    s = "%.9g" % t
    if not any(c in s for c in ".eE") and all(c in "-0123456789" for c in s):
        s += ".0"
    return s


def _flush_c_stdout():
    C.CDLL(None).fflush(None)


def cmd_run(cfg_path: str, overrides, quiet: bool) -> int:  # main.cpp:18-71
    from .engine import Simulation
    cfg = load_config(cfg_path, overrides)
    sim = Simulation(cfg)
    if not quiet:
        print("box %dx%dx%d cells, %d atoms, device cuda:%d (sm_100a, fp64)"
              % (cfg.box_x, cfg.box_y, cfg.box_z, sim.n_atoms, cfg.device))
    sys.stdout.flush()
    t0 = time.perf_counter()
    try:
        sim.run("" if quiet else "-")
    except _lib.CbxError as e:
        _flush_c_stdout()
        print(f"error: {e}", file=sys.stderr)
        dump = sim.post_mortem_path()
        if dump:
            print(f"post-mortem snapshot: {dump}", file=sys.stderr)
        return 1
    _flush_c_stdout()
    wall = time.perf_counter() - t0
    st = sim.state
    ts, d = sim.series
    peak, peak_t = 0, 0.0
    for t, row in zip(ts, d):
        if row[2] > peak:
            peak, peak_t = int(row[2]), float(t)
    print("done: %d steps, %s ps simulated, %.2f s wall" % (st["step"], _csv_time(st["t"]), wall))
    print("frenkel pairs: peak %d at %s ps, final %d"
          % (peak, _csv_time(peak_t), int(d[-1][2]) if len(d) else 0))
    if cfg.pka.energy_kev > 0.0:
        print("nrt estimate: %.3g displacements (Ed=%g eV)"
              % (nrt_displacements(cfg.pka.energy_kev * 1000.0, cfg.displacement_energy),
                 cfg.displacement_energy))
    if cfg.output.timeseries:
        print(f"timeseries: {cfg.output.timeseries}")
    if cfg.output.snapshot_prefix:
        print(f"final snapshot: {cfg.output.snapshot_prefix}_final.xyz")
    return 0


def cmd_bench_mem(cfg_path: str, overrides) -> int:  # main.cpp:73-118
    from .engine import Simulation
    cfg = load_config(cfg_path, overrides)
    sim = Simulation(cfg)
    m = sim.dev.memory_report()
    atoms = sim.atom_count()
    s = sim.store()
    n_clash = len(s.clash_key)
    buckets = len(set(s.clash_key.tolist()))
    S = m["n_slots"]
    structure = m["slots"] + m["clash"] + m["ghosts"] + m["offset_bytes"]
    print(f"atoms: {atoms}")
    print("record: %d bytes per slot across the SoA arrays (reference AoS 104, budget 128)"
          % (m["slots"] // S))
    print(f"slots: {S} records, {m['slots']} bytes")
    print(f"clash: {n_clash} atoms in {buckets} buckets, capacity {m['clash_capacity']}, "
          f"{m['clash']} bytes")
    print(f"ghost links: {m['ghost_links']} entries, {m['ghosts']} bytes")
    print(f"offset lists: {m['offset_bytes']} bytes")
    print(f"total structure bytes: {structure}")
    print("bytes/atom: %.1f" % (structure / atoms if atoms else 0.0))
    print(f"device working set: rehash {m['rehash']}, tables {m['tables']}, "
          f"reduction {m['reduction']}, staging {m['staging']}, exchange {m['exchange']} bytes")
    total = sum(m[k] for k in sim.dev.MEM_CATEGORIES) + m["offset_bytes"]
    print("device total bytes: %d (%.1f bytes/atom)" % (total, total / atoms if atoms else 0.0))
    return 0


def cmd_gen_potential(out_path: str, nrho: int, nr: int) -> int:  # main.cpp:120-126
    from .engine import EamPotential
    _lib.check(_lib.load().cbx_write_synthetic_table(out_path.encode(), nrho, nr))
    pot = EamPotential.load(out_path)
    print("wrote %s (Nrho=%d, Nr=%d, cutoff %g A); parse check OK"
          % (out_path, nrho, nr, pot.cutoff))
    return 0


def cmd_check(cfg_path: str, overrides) -> int:  # main.cpp:128-160
    from .engine import EamPotential, build_offsets
    cfg = load_config(cfg_path, overrides)
    pot = EamPotential.load(cfg.potential_path)
    a0 = cfg.a0 if cfg.a0 > 0.0 else pot.lattice_const
    index_cutoff = pot.cutoff + 0.3 * a0
    gw = cfg.ghost_width if cfg.ghost_width > 0 else int(math.ceil(index_cutoff / a0))
    if not (cfg.box_x > 0 and cfg.box_y > 0 and cfg.box_z > 0 and a0 > 0.0 and gw >= 0):
        raise _lib.CbxInvalidArgument("box: invalid dimensions")
    idx = build_offsets((cfg.box_x, cfg.box_y, cfg.box_z, a0, gw), index_cutoff)
    print("config OK: box %dx%dx%d cells, %d atoms"
          % (cfg.box_x, cfg.box_y, cfg.box_z, 2 * cfg.box_x * cfg.box_y * cfg.box_z))
    print("potential: Z=%d, %.4g amu, cutoff %g A, a0 %g A"
          % (pot.atomic_number, pot.mass, pot.cutoff, a0))
    print("ghost width: %d cells; index cutoff %.4g A" % (gw, index_cutoff))
    print("offsets per site: even %d (half %d), odd %d (half %d)"
          % (len(idx["even_full"]), len(idx["even_half"]), len(idx["odd_full"]),
             len(idx["odd_half"])))
    strips = -(-cfg.box_x * cfg.box_y // 32)
    units = strips * -(-cfg.box_z // 4)
    print("partition: device cuda:%d, %d units of 32-cell strips x 4 z planes per pass "
          "(CPU workers %d unused)" % (cfg.device, units, cfg.workers))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(
        prog="python -m paper_2107_07866_b200",
        description="collision-cascade molecular dynamics on a lattice-hash store (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    run = sub.add_parser("run", help="run a cascade simulation")
    run.add_argument("--config", required=True, help="config file (key = value lines)")
    run.add_argument("--set", action="append", default=[], dest="overrides",
                     help="override a config key (key=value)")
    run.add_argument("--quiet", action="store_true", help="suppress per-interval log lines")
    bm = sub.add_parser("bench-mem", help="report data-structure bytes per atom")
    bm.add_argument("--config", required=True, help="config file")
    bm.add_argument("--set", action="append", default=[], dest="overrides",
                    help="override a config key (key=value)")
    gen = sub.add_parser("gen-potential",
                         help="write the synthetic single-element potential table")
    gen.add_argument("--output", default="Fe-synthetic.eam", help="output path")
    gen.add_argument("--nrho", type=int, default=5000, help="embedding knot count")
    gen.add_argument("--nr", type=int, default=5000, help="radial knot count")
    chk = sub.add_parser("check", help="validate config, potential, and derived structures")
    chk.add_argument("--config", required=True, help="config file")
    chk.add_argument("--set", action="append", default=[], dest="overrides",
                     help="override a config key (key=value)")
    a = ap.parse_args(argv)
    try:
        if a.cmd == "run":
            return cmd_run(a.config, a.overrides, a.quiet)
        if a.cmd == "bench-mem":
            return cmd_bench_mem(a.config, a.overrides)
        if a.cmd == "gen-potential":
            return cmd_gen_potential(a.output, a.nrho, a.nr)
        return cmd_check(a.config, a.overrides)
    except (_lib.CbxError, ValueError, RuntimeError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
