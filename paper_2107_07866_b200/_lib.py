"""ctypes binding of libcascade_b200.so (include/cascade_b200.h).

The library is the product: every compute call goes to the sm_100a kernels
in it.  There is no CPU fallback -- if the shared object is missing or no
CUDA device is present, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CBX_LIB") or os.path.join(HERE, "libcascade_b200.so")

STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "RUNTIME", 3: "DOMAIN", 4: "LOGIC", 5: "CUDA",
          6: "NCCL"}


class CbxError(RuntimeError):
    """base of the errors raised for a non-OK cbx_status"""
    code = 2


class CbxInvalidArgument(CbxError, ValueError):
    code = 1


class CbxRuntimeError(CbxError):
    code = 2


class CbxDomainError(CbxError, ArithmeticError):
    code = 3


class CbxLogicError(CbxError):
    code = 4


class CbxCudaError(CbxError):
    code = 5


ERRORS = {1: CbxInvalidArgument, 2: CbxRuntimeError, 3: CbxDomainError, 4: CbxLogicError,
          5: CbxCudaError, 6: CbxError}


class Box(C.Structure):
    _fields_ = [("box_x", C.c_long), ("box_y", C.c_long), ("box_z", C.c_long),
                ("a0", C.c_double), ("ghost_width", C.c_long)]


class Spline(C.Structure):
    _fields_ = [("x0", C.c_double), ("h", C.c_double), ("nseg", C.c_long),
                ("seg", C.POINTER(C.c_double))]


class Potential(C.Structure):
    _fields_ = [("atomic_number", C.c_int), ("mass", C.c_double),
                ("lattice_const", C.c_double), ("cutoff", C.c_double),
                ("embed", Spline), ("zr", Spline), ("dens", Spline)]


class Offsets(C.Structure):
    _fields_ = [("cutoff", C.c_double), ("z_reach", C.c_long),
                ("even_full", C.POINTER(C.c_int64)), ("odd_full", C.POINTER(C.c_int64)),
                ("even_half", C.POINTER(C.c_int64)), ("odd_half", C.POINTER(C.c_int64)),
                ("n_even_full", C.c_long), ("n_odd_full", C.c_long),
                ("n_even_half", C.c_long), ("n_odd_half", C.c_long)]


class Store(C.Structure):
    _fields_ = [("n_slots", C.c_long),
                ("pos", C.c_void_p), ("vel", C.c_void_p), ("force", C.c_void_p),
                ("rho", C.c_void_p), ("df", C.c_void_p), ("tag", C.c_void_p),
                ("valid", C.c_void_p), ("ghost", C.c_void_p),
                ("n_clash", C.c_long), ("clash_key", C.c_void_p), ("clash_idx", C.c_void_p),
                ("clash_pos", C.c_void_p), ("clash_vel", C.c_void_p),
                ("clash_force", C.c_void_p), ("clash_rho", C.c_void_p),
                ("clash_df", C.c_void_p), ("clash_tag", C.c_void_p),
                ("clash_ghost", C.c_void_p)]


class RunSpec(C.Structure):  # cbx_run_spec
    _fields_ = [("steps", C.c_long), ("max_time", C.c_double),
                ("equilibration_steps", C.c_long), ("thermostat_enabled", C.c_int),
                ("thermostat_interval", C.c_long), ("thermostat_boundary_cells", C.c_long),
                ("temperature", C.c_double), ("timeseries", C.c_char_p),
                ("snapshot_prefix", C.c_char_p), ("snapshot_interval", C.c_long),
                ("defect_interval", C.c_long), ("pka_site", C.c_long * 3),
                ("pka_energy_kev", C.c_double), ("pka_dir", C.c_long * 3)]


class State(C.Structure):
    _fields_ = [("step", C.c_long), ("t", C.c_double), ("dt", C.c_double),
                ("kinetic", C.c_double), ("pair", C.c_double), ("embedding", C.c_double),
                ("max_speed", C.c_double), ("r_underflow", C.c_uint64),
                ("rho_clamp", C.c_uint64)]


# every symbol include/cascade_b200.h declares: (name, restype, argtypes)
_P = C.c_void_p
_D = C.c_double
SIGNATURES = [
    ("cbx_abi_version", C.c_int, []),
    ("cbx_build_info", C.c_char_p, []),
    ("cbx_last_error", C.c_char_p, [_P]),
    ("cbx_potential_load", C.c_int, [C.c_char_p, C.POINTER(C.POINTER(Potential))]),
    ("cbx_potential_free", None, [C.POINTER(Potential)]),
    ("cbx_offsets_build", C.c_int, [C.POINTER(Box), _D, C.POINTER(C.POINTER(Offsets))]),
    ("cbx_offsets_free", None, [C.POINTER(Offsets)]),
    ("cbx_make_box", C.c_int, [C.c_long, C.c_long, C.c_long, _D, C.c_long, _D,
                               C.POINTER(Potential), C.POINTER(Box), C.POINTER(C.c_double)]),
    ("cbx_pka_speed", _D, [_D, _D]),
    ("cbx_write_synthetic_table", C.c_int, [C.c_char_p, C.c_long, C.c_long]),
    ("cbx_adaptive_dt", _D, [_D, _D, _D]),
    ("cbx_create", C.c_int, [C.POINTER(Box), C.POINTER(Potential), C.POINTER(Offsets), C.c_int,
                             C.POINTER(_P)]),
    ("cbx_destroy", None, [_P]),
    ("cbx_set_stencil", C.c_int, [_P, C.c_int]),
    ("cbx_slot_count", C.c_long, [_P]),
    ("cbx_upload_store", C.c_int, [_P, C.POINTER(Store)]),
    ("cbx_download_store", C.c_int, [_P, C.POINTER(Store)]),
    ("cbx_clash_count", C.c_long, [_P]),
    ("cbx_init_bcc", C.c_int, [_P, C.c_int, _D, C.c_uint64, C.POINTER(C.c_long)]),
    ("cbx_rehash", C.c_int, [_P]),
    ("cbx_fill_ghosts", C.c_int, [_P]),
    ("cbx_eval_forces", C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("cbx_compute_density", C.c_int, [_P]),
    ("cbx_compute_embedding_derivative", C.c_int, [_P, C.POINTER(C.c_double)]),
    ("cbx_compute_pair_forces", C.c_int, [_P, C.POINTER(C.c_double)]),
    ("cbx_guards", C.c_int, [_P, C.POINTER(C.c_uint64)]),
    ("cbx_step", C.c_int, [_P, _D, C.c_long, C.POINTER(State)]),
    ("cbx_set_adaptive", C.c_int, [_P, _D, _D]),
    ("cbx_refresh_forces", C.c_int, [_P]),
    ("cbx_measure", C.c_int, [_P]),
    ("cbx_get_state", C.c_int, [_P, C.POINTER(State)]),
    ("cbx_set_state", C.c_int, [_P, C.POINTER(State)]),
    ("cbx_inject_pka", C.c_int, [_P, C.c_int64, C.POINTER(C.c_double)]),
    ("cbx_count_defects", C.c_int, [_P, C.POINTER(C.c_long)]),
    ("cbx_last_timings", C.c_int, [_P, C.POINTER(C.c_double)]),
    ("cbx_enable_timing", C.c_int, [_P, C.c_int]),
    ("cbx_count_pairs", C.c_int, [_P, C.POINTER(C.c_uint64)]),
    ("cbx_skin_stats", C.c_int, [_P, C.c_int, C.POINTER(C.c_uint64)]),
    ("cbx_kernel_launches", C.c_int, [_P, C.POINTER(C.c_uint64)]),
    ("cbx_describe", C.c_int, [_P, C.c_char_p, C.c_long]),
    ("cbx_slab_p2p_fused", C.c_int, [_P]),
    ("cbx_slab_p2p_set_fused", C.c_int, [_P, C.c_int]),
    ("cbx_slab_p2p_close", C.c_int, [_P]),
    ("cbx_memory_report", C.c_int, [_P, C.POINTER(C.c_longlong)]),
    ("cbx_bench_steps", C.c_int, [_P, _D, C.c_long, _D, C.POINTER(C.c_double)]),
    ("cbx_fp64_peak", C.c_int, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("cbx_create_slab", C.c_int, [C.POINTER(Box), C.POINTER(Potential), C.POINTER(Offsets),
                                  C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    ("cbx_slab_info", C.c_int, [_P, C.POINTER(C.c_long)]),
    ("cbx_slab_buffer_bytes", C.c_long, [_P, C.c_int]),
    ("cbx_slab_phase", C.c_int, [_P, C.c_int, _D]),
    ("cbx_slab_p2p_send", C.c_int, [_P, C.c_int]),
    ("cbx_slab_p2p_recv", C.c_int, [_P, C.c_int]),
    ("cbx_slab_pack", C.c_int, [_P, C.c_int, C.c_int, _P, C.c_long, C.POINTER(C.c_long)]),
    ("cbx_slab_unpack", C.c_int, [_P, C.c_int, C.c_int, _P, C.c_long]),
    ("cbx_slab_local_state", C.c_int, [_P, C.POINTER(C.c_double)]),
    ("cbx_slab_commit", C.c_int, [_P, C.POINTER(C.c_double)]),
    ("cbx_bench_phases", C.c_int, [_P, C.c_int]),
    ("cbx_run", C.c_int, [_P, C.POINTER(RunSpec), C.c_char_p]),
    ("cbx_run_series", C.c_long, [_P, C.POINTER(C.c_double), C.POINTER(C.c_long)]),
    ("cbx_thermostat_rescale", C.c_int, [_P, _D, C.c_long]),
    ("cbx_write_snapshot", C.c_int, [_P, C.c_char_p, _D]),
    ("cbx_write_snapshot_async", C.c_int, [_P, C.c_char_p, _D]),
    ("cbx_snapshot_wait", C.c_int, [_P]),
    ("cbx_write_timeseries", C.c_int, [C.c_char_p, C.c_long, C.POINTER(C.c_double),
                                       C.POINTER(C.c_long)]),
    ("cbx_nccl_unique_id", C.c_int, [_P, C.c_long]),
    ("cbx_slab_comm_init", C.c_int, [_P, _P, C.c_long]),
    ("cbx_slab_p2p_handle", C.c_int, [_P, _P, C.c_long]),
    ("cbx_slab_p2p_init", C.c_int, [_P, _P, C.c_long]),
    ("cbx_upload_store_global", C.c_int, [_P, C.POINTER(Store)]),
    ("cbx_download_store_global", C.c_int, [_P, C.POINTER(Store), C.POINTER(C.c_long)]),
]

_lib = None


def load(path: str = LIB_PATH):
    """load the shared object (building it first if it is absent and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        from . import build as _build
        _build.build()
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(rc: int, ctx=None) -> None:
    if rc:
        lib = load()
        msg = lib.cbx_last_error(ctx).decode()
        raise ERRORS.get(rc, CbxError)(msg)
