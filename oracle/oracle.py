"""ctypes front end for the CPU checkers (TEST INFRASTRUCTURE ONLY).

Two libraries implement the same C API (oracle/cascade_oracle.h):

* ``lib/libcascade_oracle.so`` -- the plain-C restatement of the reference
  hot path (oracle/cascade_oracle.c), always buildable with gcc;
* ``_ref/libcascade_ref.so`` -- the real reference core compiled from
  /root/reference plus oracle/ref_harness.cpp (present only where it was built).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
``--impl reference``) import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "lib", "libcascade_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libcascade_ref.so")

ERRORS = {1: ValueError, 2: RuntimeError, 3: ArithmeticError, 4: AssertionError}


class OrcConfig(C.Structure):
    _fields_ = [
        ("box_x", C.c_long), ("box_y", C.c_long), ("box_z", C.c_long),
        ("a0", C.c_double), ("ghost_width", C.c_long), ("temperature", C.c_double),
        ("seed", C.c_ulonglong), ("workers", C.c_int),
        ("pka_site", C.c_long * 3), ("pka_energy_kev", C.c_double), ("pka_dir", C.c_long * 3),
        ("dt_max", C.c_double), ("max_disp", C.c_double),
        ("thermostat_boundary_cells", C.c_long),
    ]


class OrcRunSpec(C.Structure):  # orc_run_spec
    _fields_ = [
        ("steps", C.c_long), ("max_time", C.c_double), ("equilibration_steps", C.c_long),
        ("thermostat_enabled", C.c_int), ("thermostat_interval", C.c_long),
        ("thermostat_boundary_cells", C.c_long), ("timeseries", C.c_char_p),
        ("snapshot_prefix", C.c_char_p), ("snapshot_interval", C.c_long),
        ("defect_interval", C.c_long),
    ]


def run_spec(steps=0, max_time=0.0, equilibration_steps=0, thermostat=False,
             thermostat_interval=10, boundary_cells=0, timeseries="", snapshot_prefix="",
             snapshot_interval=0, defect_interval=10) -> OrcRunSpec:
    return OrcRunSpec(steps, max_time, equilibration_steps, 1 if thermostat else 0,
                      thermostat_interval, boundary_cells, timeseries.encode(),
                      snapshot_prefix.encode(), snapshot_interval, defect_interval)


class OrcState(C.Structure):
    _fields_ = [
        ("step", C.c_long), ("t", C.c_double), ("dt", C.c_double), ("kinetic", C.c_double),
        ("pair", C.c_double), ("embedding", C.c_double), ("max_speed", C.c_double),
        ("r_underflow", C.c_ulonglong), ("rho_clamp", C.c_ulonglong),
    ]


def build(ref: bool = True) -> None:
    """make the checker libraries (the reference one only where its sources exist)."""
    targets = ["lib/libcascade_oracle.so"]
    if ref and os.path.isdir("/root/reference/proj/core/src"):
        targets.append("_ref/libcascade_ref.so")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


_LIBS: dict = {}


def _load(kind: str):
    if kind in _LIBS:
        return _LIBS[kind]
    path = ORACLE_LIB if kind == "oracle" else REF_LIB
    if not os.path.exists(path):
        if kind == "oracle":
            build(ref=False)
        else:
            raise FileNotFoundError(f"reference harness not built: {path}")
    lib = C.CDLL(path)
    P = C.c_void_p
    D = C.c_double
    dp = C.POINTER(C.c_double)
    lib.orc_create.restype = P
    lib.orc_create.argtypes = [C.c_char_p, C.POINTER(OrcConfig), C.c_int]
    lib.orc_create_error.restype = C.c_char_p
    lib.orc_error.restype = C.c_char_p
    lib.orc_error.argtypes = [P]
    lib.orc_destroy.argtypes = [P]
    for name in ["orc_canonicalize", "orc_update_hash", "orc_fill_ghosts", "orc_rehash",
                 "orc_compute_density", "orc_refresh_forces", "orc_measure", "orc_inject_pka"]:
        getattr(lib, name).argtypes = [P]
    lib.orc_box.argtypes = [P, C.POINTER(C.c_long), dp]
    for name in ["orc_index_cutoff", "orc_potential_cutoff", "orc_mass"]:
        getattr(lib, name).argtypes = [P]
        getattr(lib, name).restype = D
    lib.orc_insert.argtypes = [P, dp, dp, C.c_ulonglong]
    lib.orc_displace_interior.argtypes = [P, P, C.c_long]
    lib.orc_displace_interior.restype = C.c_long
    lib.orc_set_atom.argtypes = [P, C.c_longlong, C.c_int, dp, dp]
    lib.orc_atom_count.argtypes = [P]
    lib.orc_atom_count.restype = C.c_long
    lib.orc_nearest_site.argtypes = [P, dp]
    lib.orc_nearest_site.restype = C.c_longlong
    lib.orc_eval_forces.argtypes = [P, dp, dp]
    lib.orc_compute_embedding.argtypes = [P, dp]
    lib.orc_compute_pair.argtypes = [P, dp]
    lib.orc_guards.argtypes = [P, C.POINTER(C.c_ulonglong)]
    lib.orc_step.argtypes = [P, D, C.c_long]
    lib.orc_get_state.argtypes = [P, C.POINTER(OrcState)]
    lib.orc_count_defects.argtypes = [P, C.POINTER(C.c_long)]
    lib.orc_slot_count.argtypes = [P]
    lib.orc_slot_count.restype = C.c_long
    lib.orc_get_slots.argtypes = [P] + [P] * 8
    lib.orc_clash_count.argtypes = [P]
    lib.orc_clash_count.restype = C.c_long
    lib.orc_get_clash.argtypes = [P] + [P] * 9
    lib.orc_offsets.argtypes = [P, C.POINTER(C.c_long), P, P, P, P, C.POINTER(C.c_long)]
    lib.orc_potential_eval.argtypes = [P, C.c_int, D, dp]
    lib.orc_spline.argtypes = [P, C.c_int, dp, dp, P]
    lib.orc_spline.restype = C.c_long
    lib.orc_pka_speed.argtypes = [D, D]
    lib.orc_pka_speed.restype = D
    lib.orc_adaptive_dt.argtypes = [D, D, D]
    lib.orc_adaptive_dt.restype = D
    lib.orc_write_synthetic_table.argtypes = [C.c_char_p, C.c_long, C.c_long]
    lib.orc_thermostat_rescale.argtypes = [P]
    lib.orc_write_snapshot.argtypes = [P, C.c_char_p]
    lib.orc_write_timeseries.argtypes = [C.c_char_p, C.c_long, dp, C.POINTER(C.c_long)]
    lib.orc_run.argtypes = [P, C.POINTER(OrcRunSpec), C.c_char_p]
    lib.orc_series.argtypes = [P, dp, C.POINTER(C.c_long)]
    lib.orc_series.restype = C.c_long
    _LIBS[kind] = lib
    return lib


def available(kind: str) -> bool:
    return os.path.exists(ORACLE_LIB if kind == "oracle" else REF_LIB) or kind == "oracle"


def lib(kind: str = "oracle"):
    return _load(kind)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _dp(vals):
    a = (C.c_double * len(vals))(*vals)
    return C.cast(a, C.POINTER(C.c_double)), a


@dataclass
class Store:
    """Store dump: slot arrays by site id, clash records in (key, index) order."""
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


class Sim:
    """One oracle (or reference) simulation context."""

    def __init__(self, potential_path: str, box=(10, 10, 10), a0=0.0, ghost_width=0,
                 temperature=0.0, seed=12345, workers=1, init_lattice=True,
                 pka_site=(-1, -1, -1), pka_energy_kev=0.0, pka_dir=(1, 3, 5),
                 dt_max=1e-3, max_disp=0.05, kind="oracle", boundary_cells=0):
        self.kind = kind
        self.lib = _load(kind)
        cfg = OrcConfig()
        cfg.box_x, cfg.box_y, cfg.box_z = box
        cfg.a0, cfg.ghost_width, cfg.temperature = a0, ghost_width, temperature
        cfg.seed, cfg.workers = seed, workers
        cfg.pka_site[:] = list(pka_site)
        cfg.pka_energy_kev = pka_energy_kev
        cfg.pka_dir[:] = list(pka_dir)
        cfg.dt_max, cfg.max_disp = dt_max, max_disp
        cfg.thermostat_boundary_cells = boundary_cells
        self.cfg = cfg
        h = self.lib.orc_create(potential_path.encode(), C.byref(cfg), 1 if init_lattice else 0)
        if not h:
            raise RuntimeError(self.lib.orc_create_error().decode())
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.lib.orc_destroy(h)
            self.h = None

    def _check(self, rc):
        if rc:
            raise ERRORS.get(rc, RuntimeError)(self.lib.orc_error(self.h).decode())

    # geometry -----------------------------------------------------------
    @property
    def box(self):
        d = (C.c_long * 4)()
        a0 = C.c_double()
        self.lib.orc_box(self.h, d, C.byref(a0))
        return tuple(d[:3]), a0.value, d[3]

    @property
    def index_cutoff(self):
        return self.lib.orc_index_cutoff(self.h)

    @property
    def mass(self):
        return self.lib.orc_mass(self.h)

    def offsets(self):
        cnt = (C.c_long * 4)()
        zr = C.c_long()
        self.lib.orc_offsets(self.h, cnt, None, None, None, None, C.byref(zr))
        arrs = [np.zeros(cnt[i], dtype=np.int64) for i in range(4)]
        self.lib.orc_offsets(self.h, cnt, *[_ptr(a) for a in arrs], C.byref(zr))
        return {"even_full": arrs[0], "odd_full": arrs[1], "even_half": arrs[2],
                "odd_half": arrs[3], "z_reach": zr.value}

    def spline(self, which: int):
        x0, h = C.c_double(), C.c_double()
        n = self.lib.orc_spline(self.h, which, C.byref(x0), C.byref(h), None)
        seg = np.zeros((n, 7))
        self.lib.orc_spline(self.h, which, C.byref(x0), C.byref(h), _ptr(seg))
        return x0.value, h.value, seg

    # store ops ----------------------------------------------------------
    def insert(self, pos, tag, vel=(0.0, 0.0, 0.0)):
        p, _a = _dp(pos)
        v, _b = _dp(vel)
        self._check(self.lib.orc_insert(self.h, p, v, tag))

    def set_atom(self, site, clash_idx=-1, pos=None, vel=None):
        p = _dp(pos) if pos is not None else (None, None)
        v = _dp(vel) if vel is not None else (None, None)
        self._check(self.lib.orc_set_atom(self.h, site, clash_idx, p[0], v[0]))

    def displace_interior(self, disp: np.ndarray) -> int:
        d = np.ascontiguousarray(disp, dtype=np.float64)
        return self.lib.orc_displace_interior(self.h, _ptr(d), len(d))

    def rehash(self):
        self._check(self.lib.orc_rehash(self.h))

    def fill_ghosts(self):
        self._check(self.lib.orc_fill_ghosts(self.h))

    def nearest_site(self, p):
        q, _a = _dp(p)
        r = self.lib.orc_nearest_site(self.h, q)
        if r < 0:
            raise ArithmeticError(self.lib.orc_error(self.h).decode())
        return r

    def atom_count(self):
        return self.lib.orc_atom_count(self.h)

    # forces -------------------------------------------------------------
    def eval_forces(self):
        e1, e2 = C.c_double(), C.c_double()
        self._check(self.lib.orc_eval_forces(self.h, C.byref(e1), C.byref(e2)))
        return e1.value, e2.value

    def compute_density(self):
        self._check(self.lib.orc_compute_density(self.h))

    def compute_embedding(self):
        e = C.c_double()
        self._check(self.lib.orc_compute_embedding(self.h, C.byref(e)))
        return e.value

    def compute_pair(self):
        e = C.c_double()
        self._check(self.lib.orc_compute_pair(self.h, C.byref(e)))
        return e.value

    def guards(self):
        g = (C.c_ulonglong * 2)()
        self.lib.orc_guards(self.h, g)
        return int(g[0]), int(g[1])

    def potential_eval(self, which, x):
        out = (C.c_double * 2)()
        self._check(self.lib.orc_potential_eval(self.h, which, x, out))
        return out[0], out[1]

    # simulation ---------------------------------------------------------
    def step(self, dt=1e-3, n=1):
        self._check(self.lib.orc_step(self.h, dt, n))

    def inject_pka(self):
        self._check(self.lib.orc_inject_pka(self.h))

    def refresh_forces(self):
        self._check(self.lib.orc_refresh_forces(self.h))

    def state(self):
        st = OrcState()
        self.lib.orc_get_state(self.h, C.byref(st))
        return {k: getattr(st, k) for k, _ in OrcState._fields_}

    def count_defects(self):
        out = (C.c_long * 3)()
        self.lib.orc_count_defects(self.h, out)
        return tuple(out)

    # run loop (sim.cpp:188-360, analysis.cpp:66-116) -------------------
    def thermostat_rescale(self):
        self._check(self.lib.orc_thermostat_rescale(self.h))

    def write_snapshot(self, path: str):
        self._check(self.lib.orc_write_snapshot(self.h, path.encode()))

    def run(self, spec: OrcRunSpec, log_path: str = ""):
        self._spec = spec  # keep the strings alive
        self._check(self.lib.orc_run(self.h, C.byref(spec), log_path.encode()))

    def series(self):
        n = self.lib.orc_series(self.h, None, None)
        t = np.zeros(n)
        d = np.zeros(3 * n, dtype=np.int64)
        self.lib.orc_series(self.h, t.ctypes.data_as(C.POINTER(C.c_double)),
                            d.ctypes.data_as(C.POINTER(C.c_long)))
        return t, d.reshape(n, 3)

    def store(self) -> Store:
        n = self.lib.orc_slot_count(self.h)
        pos, vel, force = (np.zeros((n, 3)) for _ in range(3))
        rho, df = np.zeros(n), np.zeros(n)
        tag = np.zeros(n, dtype=np.uint64)
        valid, ghost = np.zeros(n, dtype=np.uint8), np.zeros(n, dtype=np.uint8)
        self.lib.orc_get_slots(self.h, _ptr(pos), _ptr(vel), _ptr(force), _ptr(rho), _ptr(df),
                               _ptr(tag), _ptr(valid), _ptr(ghost))
        m = self.lib.orc_clash_count(self.h)
        key = np.zeros(m, dtype=np.int64)
        idx = np.zeros(m, dtype=np.int32)
        cpos, cvel, cforce = (np.zeros((m, 3)) for _ in range(3))
        crho, cdf = np.zeros(m), np.zeros(m)
        ctag = np.zeros(m, dtype=np.uint64)
        cghost = np.zeros(m, dtype=np.uint8)
        if m:
            self.lib.orc_get_clash(self.h, _ptr(key), _ptr(idx), _ptr(cpos), _ptr(cvel),
                                   _ptr(cforce), _ptr(crho), _ptr(cdf), _ptr(ctag), _ptr(cghost))
        return Store(pos, vel, force, rho, df, tag, valid, ghost, key, idx, cpos, cvel, cforce,
                     crho, cdf, ctag, cghost)


def pka_speed(e_ev, mass, kind="oracle"):
    return _load(kind).orc_pka_speed(e_ev, mass)


def adaptive_dt(vmax, dt_max=1e-3, max_disp=0.05, kind="oracle"):
    return _load(kind).orc_adaptive_dt(vmax, dt_max, max_disp)


def write_synthetic_table(path, nrho=5000, nr=5000, kind="oracle"):
    rc = _load(kind).orc_write_synthetic_table(path.encode(), nrho, nr)
    if rc:
        raise RuntimeError(f"write_synthetic_table failed ({rc})")
