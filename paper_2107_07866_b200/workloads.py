"""The BASELINE.json configurations as seeded synthetic workloads.

BASELINE.json quotes five configurations (restated in SURVEY.md §8(d)).  No
public dataset is involved: every initial state is generated on the host by
the reference-compatible lattice/RNG code (init_bcc, sim.cpp:100-130) from a
seed, plus -- for config 2 -- per-component uniform +-0.05 A displacements
drawn with numpy's PCG64 (seed 12345) in interior-site order.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Workload:
    name: str
    cells: tuple
    temperature: float
    dt: float
    steps: int
    displacement: float = 0.0
    pka_kev: float = 0.0
    pka_dir: tuple = (1, 3, 5)
    seed: int = 12345
    note: str = ""

    @property
    def atoms(self) -> int:
        return 2 * self.cells[0] * self.cells[1] * self.cells[2]


CONFIGS = {
    "c1": Workload("c1", (20, 20, 20), 600.0, 1e-3, 100,
                   note="BCC Fe 20^3 cells (16,000 atoms), 600 K, 100 x 1 fs"),
    "c2": Workload("c2", (50, 50, 50), 600.0, 1e-3, 200, displacement=0.05,
                   note="BCC Fe 50^3 cells (250,000 atoms), 600 K + U(-0.05,0.05) A, 200 x 1 fs"),
    "c3": Workload("c3", (100, 100, 100), 600.0, 1e-4, 1000, pka_kev=10.0,
                   note="BCC Fe 100^3 (2,000,000 atoms), 600 K, 10 keV PKA (1,3,5), 1000 x 0.1 fs"),
    "c4": Workload("c4", (200, 200, 200), 600.0, 2e-4, 500, pka_kev=5.0,
                   note="BCC Fe 200^3 (16,000,000 atoms), 600 K, 5 keV PKA, 500 x 0.2 fs"),
    "c5": Workload("c5", (256, 256, 256), 600.0, 1e-3, 100, pka_kev=20.0,
                   note="BCC Fe 256^3 per GPU (33,554,432 atoms), 600 K, 20 keV PKA, 100 x 1 fs"),
}


def displacements(w: Workload, n_atoms: int) -> np.ndarray:
    """config 2's random displacements, one row per atom in interior-id order"""
    if w.displacement <= 0.0:
        return np.zeros((n_atoms, 3))
    rng = np.random.Generator(np.random.PCG64(w.seed))
    return rng.uniform(-w.displacement, w.displacement, size=(n_atoms, 3))


def pka_site_id(w: Workload, ghost_width: int) -> int:
    """corner site of the centre cell (sim.cpp:165-170)"""
    bx, by, bz = w.cells
    g = ghost_width
    tx, ty = bx + 2 * g, by + 2 * g
    cx, cy, cz = bx // 2, by // 2, bz // 2
    return ((g + cz) * ty + (g + cy)) * 2 * tx + 2 * (g + cx)


def pka_velocity(w: Workload, mass: float):
    """Simulation::inject_pka's velocity (sim.cpp:172-185): pka_speed(E, m)
    along the direction normalised on the host, as the reference computes it"""
    from .engine import pka_speed
    d = [float(x) for x in w.pka_dir]
    ln = math.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])
    s = pka_speed(w.pka_kev * 1000.0, mass) / ln
    return (d[0] * s, d[1] * s, d[2] * s)


def slab_site_id(info, cx: int, cy: int, cz_global: int) -> int:
    """local reference id of the corner site of global cell (cx, cy, cz) on a
    slab rank (cbx_slab_info: zoff, bz, g, tx, ty); -1 if another rank owns it"""
    zoff, bz, g, tx, ty = info[2], info[3], info[4], info[5], info[6]
    zl = cz_global - zoff
    if not 0 <= zl < bz:
        return -1
    return ((g + zl) * ty + (g + cy)) * 2 * tx + 2 * (g + cx)


def build_device_state(w: Workload, potential, device: int = 0, stencil: str = "newton3"):
    """A DeviceStore in the workload's initial state: lattice + MB velocities,
    displacements, rehash, forces, measure (the Simulation constructor path)."""
    from .engine import DeviceStore, SimConfig, make_box
    cfg = SimConfig(box_x=w.cells[0], box_y=w.cells[1], box_z=w.cells[2],
                    temperature=w.temperature, seed=w.seed)
    box, _ = make_box(cfg, potential)
    dev = DeviceStore(box, potential, device=device, stencil=stencil)
    n = dev.init_bcc(w.temperature, w.seed, potential.atomic_number)
    if w.displacement > 0.0:
        s = dev.download()
        m = s.valid.astype(bool) & ~s.ghost.astype(bool)
        s.pos[m] += displacements(w, n)
        dev.upload(s)
        dev.rehash()
    dev.eval_forces()
    if w.pka_kev > 0.0:  # the configuration's PKA (sim.cpp:163-186; measures)
        dev.inject_pka(pka_site_id(w, box.ghost_width), pka_velocity(w, potential.mass))
    dev.measure()
    return dev, n


def build_slab_state(w: Workload, potential, rank: int, nranks: int, device: int = 0,
                     stencil: str = "newton3", transport: str = "p2p",
                     scaling: str = "weak"):
    """Rank `rank` of a z-slab run over `nranks` GPUs.

    weak:   the global box stacks `nranks` copies of the workload's cells
            along z (cells[2] planes per rank) with one PKA at the centre cell
            of every rank's subdomain (BASELINE config 5);
    strong: the workload's box itself is split into `nranks` slabs with the
            one PKA at the global centre (BASELINE config 4).
    The slab holds exactly its planes of the single-box initial state of the
    global box (same lattice RNG stream and displacement rows).  The ranks
    connect through torch.distributed (P2P handles or the NCCL id); forces
    and the kinetic energy are evaluated collectively."""
    from .engine import SimConfig, make_box
    from .slab import SlabRank
    bx, by, bz = w.cells
    gz = bz * nranks if scaling == "weak" else bz
    cfg = SimConfig(box_x=bx, box_y=by, box_z=gz, temperature=w.temperature, seed=w.seed)
    gbox, _ = make_box(cfg, potential)
    r = SlabRank(gbox, potential, rank, nranks, device=device, stencil=stencil)
    n = r.init_bcc(w.temperature, w.seed, potential.atomic_number)
    if w.displacement > 0.0:
        per_plane = 2 * bx * by
        z0 = r.info[2]
        d = displacements(w, per_plane * gz)[z0 * per_plane:(z0 + r.info[3]) * per_plane]
        s = r.download()
        m = s.valid.astype(bool) & ~s.ghost.astype(bool)
        s.pos[m] += d
        r.upload(s)
    r.connect(transport)
    r.eval_forces()
    if w.pka_kev > 0.0:
        centres = ([bz * q + bz // 2 for q in range(nranks)] if scaling == "weak" else [gz // 2])
        v = pka_velocity(w, potential.mass)
        for cz in centres:
            site = slab_site_id(r.info, bx // 2, by // 2, cz)
            if site >= 0:
                r.inject_pka(site, v)
    r.measure()
    return r, n
