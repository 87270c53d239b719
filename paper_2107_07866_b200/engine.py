"""Host-side mirror of the reference simulation API over the C ABI.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/core/include/cascademd/*.h):

* ``SimConfig``      -- config.h:36-53 (the fields the hot path consumes)
* ``EamPotential``   -- potential.h:33-69 (``EamPotential.load`` = parse_potential_file)
* ``DeviceStore``    -- a LatticeStore (store.h:45-78) resident on one B200,
                        with the force engine (forces.h:42-67) and the step
* ``Simulation``     -- sim.h:38-91

Every compute call runs the sm_100a kernels of libcascade_b200.so.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check

# units.h:17-24
ACCEL_FACTOR = (1.602176634e-19 / 1e-10 / 1.66053906660e-27) * (1e-12 * 1e-12) / 1e-10
SPEED_FACTOR = 98.22694750253277
MV2_TO_EV = 1.0 / ACCEL_FACTOR
BOLTZMANN_EV = 1.380649e-23 / 1.602176634e-19


@dataclass
class PkaSpec:  # config.h:9-15
    site: tuple = (-1, -1, -1)
    energy_kev: float = 0.0
    direction: tuple = (1, 3, 5)


@dataclass
class ThermostatSpec:  # config.h:16-20
    enabled: bool = False
    interval: int = 10
    boundary_cells: int = 0


@dataclass
class OutputSpec:  # config.h:22-27
    timeseries: str = ""
    snapshot_prefix: str = ""
    snapshot_interval: int = 0
    defect_interval: int = 10


@dataclass
class SimConfig:  # config.h:36-53
    box_x: int = 10
    box_y: int = 10
    box_z: int = 10
    a0: float = 0.0
    ghost_width: int = 0
    temperature: float = 0.0
    potential_path: str = ""
    pka: PkaSpec = field(default_factory=PkaSpec)
    steps: int = 0
    max_time: float = 0.0
    dt_max: float = 1e-3
    max_disp: float = 0.05
    thermostat: ThermostatSpec = field(default_factory=ThermostatSpec)
    output: OutputSpec = field(default_factory=OutputSpec)
    workers: int = 1
    seed: int = 12345
    equilibration_steps: int = 0
    displacement_energy: float = 40.0  # eV, NRT threshold (analysis.cpp:58-65)
    device: int = 0
    stencil: str = "newton3"


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class EamPotential:
    """parse_potential_file + build_spline (potential.cpp:134-185), host side."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def load(cls, path: str) -> "EamPotential":
        lib = _lib.load()
        out = C.POINTER(_lib.Potential)()
        check(lib.cbx_potential_load(path.encode(), C.byref(out)))
        return cls(out)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.load().cbx_potential_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    cutoff = property(lambda self: self._h.contents.cutoff)
    mass = property(lambda self: self._h.contents.mass)
    lattice_const = property(lambda self: self._h.contents.lattice_const)
    atomic_number = property(lambda self: self._h.contents.atomic_number)

    def table(self, which: str):
        s = getattr(self._h.contents, which)
        seg = np.ctypeslib.as_array(s.seg, shape=(s.nseg * 7,)).reshape(s.nseg, 7).copy()
        return s.x0, s.h, seg


def make_box(cfg: SimConfig, pot: EamPotential):
    """make_box + index cutoff (sim.cpp:62-84)."""
    lib = _lib.load()
    box = _lib.Box()
    ic = C.c_double()
    check(lib.cbx_make_box(cfg.box_x, cfg.box_y, cfg.box_z, cfg.a0, cfg.ghost_width,
                           cfg.max_disp, pot.handle, C.byref(box), C.byref(ic)))
    return box, ic.value


def build_offsets(box, cutoff: float) -> dict:
    """build_offsets (neighbors.cpp:11-87) -> dict of numpy lists."""
    lib = _lib.load()
    out = C.POINTER(_lib.Offsets)()
    b = box if isinstance(box, _lib.Box) else _lib.Box(*box)
    check(lib.cbx_offsets_build(C.byref(b), cutoff, C.byref(out)))
    o = out.contents
    res = {
        "cutoff": o.cutoff, "z_reach": o.z_reach,
        "even_full": np.ctypeslib.as_array(o.even_full, (o.n_even_full,)).copy(),
        "odd_full": np.ctypeslib.as_array(o.odd_full, (o.n_odd_full,)).copy(),
        "even_half": np.ctypeslib.as_array(o.even_half, (o.n_even_half,)).copy(),
        "odd_half": np.ctypeslib.as_array(o.odd_half, (o.n_odd_half,)).copy(),
    }
    lib.cbx_offsets_free(out)
    return res


def pka_speed(energy_ev: float, mass_amu: float) -> float:
    """sim.cpp:88-92"""
    if not mass_amu > 0.0:
        raise ValueError("mass must be positive")
    if energy_ev < 0.0:
        raise ValueError("energy cannot be negative")
    return _lib.load().cbx_pka_speed(energy_ev, mass_amu)


def adaptive_dt(max_speed: float, cfg: SimConfig) -> float:
    """sim.cpp:94-98"""
    return _lib.load().cbx_adaptive_dt(max_speed, cfg.dt_max, cfg.max_disp)


@dataclass
class StoreArrays:
    """A LatticeStore snapshot: slot arrays by reference site id, clash
    records in (key, bucket index) order (store.h:16-78)."""
    pos: np.ndarray
    vel: np.ndarray
    force: np.ndarray
    rho: np.ndarray
    df: np.ndarray
    tag: np.ndarray
    valid: np.ndarray
    ghost: np.ndarray
    clash_key: np.ndarray
    clash_idx: np.ndarray
    clash_pos: np.ndarray
    clash_vel: np.ndarray
    clash_force: np.ndarray
    clash_rho: np.ndarray
    clash_df: np.ndarray
    clash_tag: np.ndarray
    clash_ghost: np.ndarray


def pinned_store(n_slots: int) -> StoreArrays:
    """slot arrays in page-locked host memory (DMA at full PCIe / C2C rate);
    clash arrays are small and stay pageable"""
    import torch

    def pin(shape, dtype):
        return torch.empty(shape, dtype=dtype, pin_memory=True).numpy()
    S = n_slots
    return StoreArrays(pos=pin((S, 3), torch.float64), vel=pin((S, 3), torch.float64),
                       force=pin((S, 3), torch.float64), rho=pin((S,), torch.float64),
                       df=pin((S,), torch.float64), tag=pin((S,), torch.int64).view(np.uint64),
                       valid=pin((S,), torch.uint8), ghost=pin((S,), torch.uint8),
                       clash_key=np.zeros(0, np.int64), clash_idx=np.zeros(0, np.int32),
                       clash_pos=np.zeros((0, 3)), clash_vel=np.zeros((0, 3)),
                       clash_force=np.zeros((0, 3)), clash_rho=np.zeros(0),
                       clash_df=np.zeros(0), clash_tag=np.zeros(0, np.uint64),
                       clash_ghost=np.zeros(0, np.uint8))


class DeviceStore:
    """A LatticeStore + force engine resident on one GPU (one cbx_ctx)."""

    def __init__(self, box, potential: EamPotential, offsets: Optional[dict] = None,
                 device: int = 0, stencil: str = "newton3"):
        lib = _lib.load()
        self.lib = lib
        self.potential = potential
        self.box = box if isinstance(box, _lib.Box) else _lib.Box(*box)
        keep = None
        idx_p = None
        if offsets is not None:
            arrs = [np.ascontiguousarray(offsets[k], dtype=np.int64)
                    for k in ("even_full", "odd_full", "even_half", "odd_half")]
            idx = _lib.Offsets(offsets["cutoff"], offsets.get("z_reach", 0),
                               *[a.ctypes.data_as(C.POINTER(C.c_int64)) for a in arrs],
                               *[len(a) for a in arrs])
            keep = arrs
            idx_p = C.byref(idx)
        h = C.c_void_p()
        check(lib.cbx_create(C.byref(self.box), potential.handle, idx_p, device, C.byref(h)))
        del keep
        self.h = h
        self.n_slots = lib.cbx_slot_count(h)
        if stencil != "newton3":
            self.set_stencil(stencil)

    def close(self):
        if getattr(self, "h", None):
            self.lib.cbx_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def _check(self, rc):
        check(rc, self.h)

    def set_stencil(self, mode: str):
        self._check(self.lib.cbx_set_stencil(self.h, {"newton3": 0, "full": 1, "reference": 2}[mode]))

    # --- store transfer ----------------------------------------------------
    def upload(self, s) -> None:
        """upload a store snapshot (any object with StoreArrays' fields)."""
        S = self.n_slots
        f64 = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64)
        pos, vel, force = f64(s.pos), f64(getattr(s, "vel", None)), f64(getattr(s, "force", None))
        rho, df = f64(getattr(s, "rho", None)), f64(getattr(s, "df", None))
        tag = np.ascontiguousarray(s.tag, dtype=np.uint64)
        valid = np.ascontiguousarray(s.valid, dtype=np.uint8)
        ghost = np.ascontiguousarray(getattr(s, "ghost", np.zeros(S, np.uint8)), dtype=np.uint8)
        ck = np.ascontiguousarray(getattr(s, "clash_key", np.zeros(0, np.int64)), dtype=np.int64)
        n = len(ck)
        cp = f64(getattr(s, "clash_pos", np.zeros((0, 3))))
        cv = f64(getattr(s, "clash_vel", np.zeros((n, 3))))
        cf = f64(getattr(s, "clash_force", np.zeros((n, 3))))
        cr = f64(getattr(s, "clash_rho", np.zeros(n)))
        cd = f64(getattr(s, "clash_df", np.zeros(n)))
        ct = np.ascontiguousarray(getattr(s, "clash_tag", np.zeros(n, np.uint64)), dtype=np.uint64)
        cg = np.ascontiguousarray(getattr(s, "clash_ghost", np.zeros(n, np.uint8)), dtype=np.uint8)
        st = _lib.Store(S, _ptr(pos), _ptr(vel), _ptr(force), _ptr(rho), _ptr(df), _ptr(tag),
                        _ptr(valid), _ptr(ghost), n, _ptr(ck), None, _ptr(cp), _ptr(cv),
                        _ptr(cf), _ptr(cr), _ptr(cd), _ptr(ct), _ptr(cg))
        self._check(self.lib.cbx_upload_store(self.h, C.byref(st)))

    def download(self, out: Optional["StoreArrays"] = None) -> StoreArrays:
        """the store snapshot; `out` (e.g. from pinned_store()) is reused for
        the slot arrays when given"""
        S = self.n_slots
        if out is not None and len(out.tag) == S:
            a = {k: getattr(out, k) for k in ("pos", "vel", "force", "rho", "df", "tag", "valid",
                                               "ghost")}
        else:
            a = dict(pos=np.zeros((S, 3)), vel=np.zeros((S, 3)), force=np.zeros((S, 3)),
                     rho=np.zeros(S), df=np.zeros(S), tag=np.zeros(S, np.uint64),
                     valid=np.zeros(S, np.uint8), ghost=np.zeros(S, np.uint8))
        n = self.lib.cbx_clash_count(self.h)
        c = dict(clash_key=np.zeros(n, np.int64), clash_idx=np.zeros(n, np.int32),
                 clash_pos=np.zeros((n, 3)), clash_vel=np.zeros((n, 3)),
                 clash_force=np.zeros((n, 3)), clash_rho=np.zeros(n), clash_df=np.zeros(n),
                 clash_tag=np.zeros(n, np.uint64), clash_ghost=np.zeros(n, np.uint8))
        st = _lib.Store(S, *[_ptr(a[k]) for k in ("pos", "vel", "force", "rho", "df", "tag",
                                                   "valid", "ghost")],
                        n, *[_ptr(c[k]) for k in ("clash_key", "clash_idx", "clash_pos",
                                                   "clash_vel", "clash_force", "clash_rho",
                                                   "clash_df", "clash_tag", "clash_ghost")])
        self._check(self.lib.cbx_download_store(self.h, C.byref(st)))
        return StoreArrays(**a, **c)

    def init_bcc(self, temperature: float, seed: int, species: int = 26) -> int:
        n = C.c_long()
        self._check(self.lib.cbx_init_bcc(self.h, species, temperature, seed, C.byref(n)))
        return n.value

    # --- store ops ---------------------------------------------------------
    def rehash(self):
        self._check(self.lib.cbx_rehash(self.h))

    def fill_ghosts(self):
        self._check(self.lib.cbx_fill_ghosts(self.h))

    # --- force engine ------------------------------------------------------
    def eval_forces(self):
        e1, e2 = C.c_double(), C.c_double()
        self._check(self.lib.cbx_eval_forces(self.h, C.byref(e1), C.byref(e2)))
        return e1.value, e2.value

    def compute_density(self):
        self._check(self.lib.cbx_compute_density(self.h))

    def compute_embedding_derivative(self) -> float:
        e = C.c_double()
        self._check(self.lib.cbx_compute_embedding_derivative(self.h, C.byref(e)))
        return e.value

    def compute_pair_forces(self) -> float:
        e = C.c_double()
        self._check(self.lib.cbx_compute_pair_forces(self.h, C.byref(e)))
        return e.value

    def guards(self):
        g = (C.c_uint64 * 2)()
        self._check(self.lib.cbx_guards(self.h, g))
        return int(g[0]), int(g[1])

    # --- integrator --------------------------------------------------------
    def set_adaptive(self, dt_max: float, max_disp: float):
        self._check(self.lib.cbx_set_adaptive(self.h, dt_max, max_disp))

    def step(self, dt: float = -1.0, n: int = 1) -> dict:
        st = _lib.State()
        self._check(self.lib.cbx_step(self.h, dt, n, C.byref(st)))
        return {k: getattr(st, k) for k, _ in _lib.State._fields_}

    def measure(self):
        self._check(self.lib.cbx_measure(self.h))

    def state(self) -> dict:
        st = _lib.State()
        self._check(self.lib.cbx_get_state(self.h, C.byref(st)))
        return {k: getattr(st, k) for k, _ in _lib.State._fields_}

    def set_state(self, d: dict):
        st = _lib.State(*[d.get(k, 0) for k, _ in _lib.State._fields_])
        self._check(self.lib.cbx_set_state(self.h, C.byref(st)))

    def inject_pka(self, site: int, v):
        vv = (C.c_double * 3)(*v)
        self._check(self.lib.cbx_inject_pka(self.h, site, vv))

    def count_defects(self):
        out = (C.c_long * 3)()
        self._check(self.lib.cbx_count_defects(self.h, out))
        return tuple(out)

    def thermostat_rescale(self, temperature: float, boundary_cells: int = 0):
        self._check(self.lib.cbx_thermostat_rescale(self.h, temperature, boundary_cells))

    def write_snapshot(self, path: str, t_ps: Optional[float] = None):
        t = self.state()["t"] if t_ps is None else t_ps
        self._check(self.lib.cbx_write_snapshot(self.h, path.encode(), t))

    def write_snapshot_async(self, path: str, t_ps: Optional[float] = None):
        """pack now, copy and write in the background (snapshot_wait joins)"""
        t = self.state()["t"] if t_ps is None else t_ps
        self._check(self.lib.cbx_write_snapshot_async(self.h, path.encode(), t))

    def snapshot_wait(self):
        self._check(self.lib.cbx_snapshot_wait(self.h))

    def run(self, spec: "_lib.RunSpec", log_path: str = ""):
        self._spec = spec  # keep the strings alive
        self._check(self.lib.cbx_run(self.h, C.byref(spec), log_path.encode()))

    def series(self):
        n = self.lib.cbx_run_series(self.h, None, None)
        t = np.zeros(n)
        d = np.zeros(3 * n, dtype=np.int64)
        self.lib.cbx_run_series(self.h, t.ctypes.data_as(C.POINTER(C.c_double)),
                                d.ctypes.data_as(C.POINTER(C.c_long)))
        return t, d.reshape(n, 3)

    # --- instrumentation ---------------------------------------------------
    def enable_timing(self, on: bool = True):
        self._check(self.lib.cbx_enable_timing(self.h, 1 if on else 0))

    def timings(self) -> dict:
        t = (C.c_double * 8)()
        self._check(self.lib.cbx_last_timings(self.h, t))
        return {"density_ms": t[0], "embed_ms": t[1], "force_ms": t[2], "store_ms": t[3],
                "integrate_ms": t[4], "step_ms": t[5], "steps": t[6]}

    def skin_stats(self, enable: bool):
        """(skin candidates examined, skin candidates listed) of the density
        passes since counting was enabled; enable=True restarts the count"""
        out = (C.c_uint64 * 2)()
        self._check(self.lib.cbx_skin_stats(self.h, 1 if enable else 0, out))
        return int(out[0]), int(out[1])

    def count_pairs(self):
        out = (C.c_uint64 * 2)()
        self._check(self.lib.cbx_count_pairs(self.h, out))
        return int(out[0]), int(out[1])

    def describe(self) -> dict:
        import json
        buf = C.create_string_buffer(1024)
        self._check(self.lib.cbx_describe(self.h, buf, 1024))
        return json.loads(buf.value.decode())

    MEM_CATEGORIES = ("slots", "clash", "ghosts", "rehash", "tables", "reduction",
                      "staging", "exchange")

    def memory_report(self) -> dict:
        """device bytes by structure (cbx_memory_report) plus the slot, clash
        capacity, ghost-link and offset-list counts"""
        n = len(self.MEM_CATEGORIES)
        out = (C.c_longlong * (n + 4))()
        self._check(self.lib.cbx_memory_report(self.h, out))
        r = {k: int(out[i]) for i, k in enumerate(self.MEM_CATEGORIES)}
        r.update(n_slots=int(out[n]), clash_capacity=int(out[n + 1]),
                 ghost_links=int(out[n + 2]), offset_bytes=int(out[n + 3]))
        return r

    def kernel_launches(self) -> int:
        n = C.c_uint64()
        self._check(self.lib.cbx_kernel_launches(self.h, C.byref(n)))
        return n.value


class Simulation:
    """sim.h:38-91 over the device: the constructor builds the box, offsets
    and lattice, fills ghosts, evaluates forces and measures (sim.cpp:135-148)."""

    def __init__(self, cfg: SimConfig, potential: Optional[EamPotential] = None):
        if potential is None:
            if not cfg.potential_path:
                raise ValueError("potential: no potential file configured")
            potential = EamPotential.load(cfg.potential_path)
        self.cfg = cfg
        self.pot = potential
        self.box, self.index_cutoff = make_box(cfg, potential)
        self.dev = DeviceStore(self.box, potential, device=cfg.device, stencil=cfg.stencil)
        self.dev.set_adaptive(cfg.dt_max, cfg.max_disp)
        self.n_atoms = self.dev.init_bcc(cfg.temperature, cfg.seed, potential.atomic_number)
        self.refresh_forces()
        self.dev.measure()

    def refresh_forces(self):
        self.dev.eval_forces()

    @property
    def state(self) -> dict:
        return self.dev.state()

    def total_energy(self) -> float:
        s = self.dev.state()
        return s["kinetic"] + s["pair"] + s["embedding"]

    def temperature(self) -> float:
        n = self.atom_count()
        return 0.0 if n == 0 else 2.0 * self.dev.state()["kinetic"] / (3.0 * n * BOLTZMANN_EV)

    def atom_count(self) -> int:
        s = self.dev.download()
        interior = (s.valid.astype(bool) & ~s.ghost.astype(bool)).sum()
        return int(interior + (s.clash_ghost == 0).sum())

    def total_momentum(self):
        s = self.dev.download()
        m = s.valid.astype(bool) & ~s.ghost.astype(bool)
        p = s.vel[m].sum(axis=0) + s.clash_vel[s.clash_ghost == 0].sum(axis=0)
        return self.pot.mass * p

    def store(self) -> StoreArrays:
        return self.dev.download()

    def step(self, dt: Optional[float] = None, n: int = 1) -> dict:
        if dt is not None and not dt > 0.0:
            raise ValueError("dt must be positive")
        return self.dev.step(dt if dt is not None else -1.0, n)

    def pka_site_id(self) -> int:
        b, p = self.box, self.cfg.pka
        cx = p.site[0] if p.site[0] >= 0 else self.cfg.box_x // 2
        cy = p.site[1] if p.site[1] >= 0 else self.cfg.box_y // 2
        cz = p.site[2] if p.site[2] >= 0 else self.cfg.box_z // 2
        g = b.ghost_width
        tx = b.box_x + 2 * g
        ty = b.box_y + 2 * g
        return ((g + cz) * ty + (g + cy)) * 2 * tx + 2 * (g + cx)

    def inject_pka(self):
        """sim.cpp:163-186: velocity of magnitude pka_speed along the
        normalised direction, computed on the host like the reference."""
        p = self.cfg.pka
        d = [float(x) for x in p.direction]
        ln = math.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])
        if not ln > 0.0:
            raise ValueError("pka.direction: must not be the zero vector")
        v = pka_speed(p.energy_kev * 1000.0, self.pot.mass)
        s = v / ln
        self.dev.inject_pka(self.pka_site_id(), (d[0] * s, d[1] * s, d[2] * s))

    def count_defects(self):
        return self.dev.count_defects()

    def thermostat_rescale(self):
        """sim.cpp:188-221: toward cfg.temperature in cfg.thermostat.boundary_cells"""
        self.dev.thermostat_rescale(self.cfg.temperature, self.cfg.thermostat.boundary_cells)

    def run_spec(self) -> "_lib.RunSpec":
        c = self.cfg
        return _lib.RunSpec(
            c.steps, c.max_time, c.equilibration_steps, 1 if c.thermostat.enabled else 0,
            c.thermostat.interval, c.thermostat.boundary_cells, c.temperature,
            c.output.timeseries.encode(), c.output.snapshot_prefix.encode(),
            c.output.snapshot_interval, c.output.defect_interval,
            (C.c_long * 3)(*c.pka.site), c.pka.energy_kev, (C.c_long * 3)(*c.pka.direction))

    def post_mortem_path(self) -> str:
        """sim.cpp:284-287: the snapshot a failed step leaves behind"""
        p = self.cfg.output.snapshot_prefix
        return p + "_postmortem.xyz" if p else ""

    def run(self, log: str = ""):
        """Simulation::run (sim.cpp:289-360); log: path, "-" for stdout, "" none"""
        self.dev.run(self.run_spec(), log)

    @property
    def series(self):
        """(t_ps, [[vacancies, interstitials, frenkel_pairs], ...]) of the last run"""
        return self.dev.series()
