"""The config file front end: config.cpp:1-225 / config.h:29-69 restated.

One dotted ``key = value`` per line, ``#`` comments; defaults, then the
CASCADE_WORKERS environment variable, then the file, then ``key=value``
overrides, then validation.  Errors carry the reference's messages:
``CbxInvalidArgument`` (a ValueError, std::invalid_argument) for bad keys,
values and ranges, ``CbxRuntimeError`` (std::runtime_error) for an
unreadable file.  ``SimConfig.device`` / ``stencil`` are this package's own
fields and have no config key, as in the reference.
"""
from __future__ import annotations

import math
import os
import re
from typing import Iterable

from ._lib import CbxInvalidArgument, CbxRuntimeError
from .engine import SimConfig

_WS = " \t\r\n"
_LONG_MIN, _LONG_MAX = -(1 << 63), (1 << 63) - 1
# strtol / strtoull / strtod accept leading white space (isspace)
_LEAD = " \t\n\v\f\r"
_INT = re.compile(r"[+-]?[0-9]+")
_DEC = re.compile(r"[+-]?(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?")
_HEX = re.compile(r"[+-]?0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)(?:[pP][+-]?[0-9]+)?")
_SPECIAL = re.compile(r"[+-]?(?:inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?)", re.IGNORECASE)
_DBL_MIN = 2.2250738585072014e-308


def _trim(s: str) -> str:  # config.cpp:11-16
    return s.strip(_WS)


def _bad(key: str, why: str):  # config.cpp:18-20
    raise CbxInvalidArgument(f"{key}: {why}")


def _parse_long(key: str, v: str) -> int:  # config.cpp:22-30 (strtol, base 10)
    t = v.lstrip(_LEAD)
    if not _INT.fullmatch(t):
        _bad(key, f"expected an integer, got '{v}'")
    x = int(t)
    if not _LONG_MIN <= x <= _LONG_MAX:  # ERANGE
        _bad(key, f"expected an integer, got '{v}'")
    return x


def _parse_u64(key: str, v: str) -> int:  # config.cpp:32-40 (strtoull, no '-')
    t = v.lstrip(_LEAD)
    if "-" in v or not _INT.fullmatch(t):
        _bad(key, f"expected an unsigned integer, got '{v}'")
    x = int(t)
    if x > (1 << 64) - 1:
        _bad(key, f"expected an unsigned integer, got '{v}'")
    return x


def _strtod(t: str):
    """the value strtod parses from all of ``t`` and whether it set ERANGE;
    None when ``t`` is not one complete number"""
    if _SPECIAL.fullmatch(t):
        return float(t.split("(")[0]), False
    if _DEC.fullmatch(t):
        x = float(t)
        mant = re.sub(r"[eE].*", "", t)
        nonzero = any(c in "123456789" for c in mant)
    elif _HEX.fullmatch(t):
        sign = -1.0 if t[0] == "-" else 1.0
        body = t.lstrip("+-")
        if "p" not in body.lower():
            body += "p0"
        try:
            x = sign * float.fromhex(body)
        except OverflowError:
            return math.copysign(math.inf, -1.0 if t[0] == "-" else 1.0), True
        mant = re.split(r"[pP]", body)[0][2:]
        nonzero = any(c not in "0." for c in mant)
    else:
        return None
    erange = math.isinf(x) or (nonzero and abs(x) < _DBL_MIN)
    return x, erange


def _parse_double(key: str, v: str) -> float:  # config.cpp:42-50
    r = _strtod(v.lstrip(_LEAD))
    if r is None or r[1]:
        _bad(key, f"expected a number, got '{v}'")
    return r[0]


_LONG_AT = re.compile(r"[ \t\n\v\f\r]*([+-]?[0-9]+)")
_TOKEN_AT = re.compile(r"[ \t\n\v\f\r]*(\S+)")


def _parse_triple(key: str, v: str):  # config.cpp:52-64 (istringstream >> long)
    s = v.replace(",", " ")
    pos, out = 0, []
    for _ in range(3):
        m = _LONG_AT.match(s, pos)
        if not m or not _LONG_MIN <= int(m.group(1)) <= _LONG_MAX:
            _bad(key, f"expected three integers, got '{v}'")
        out.append(int(m.group(1)))
        pos = m.end()
    m = _TOKEN_AT.match(s, pos)
    if m:
        _bad(key, f"trailing text '{m.group(1)}'")
    return out


def apply_config_entry(cfg: SimConfig, key: str, value: str) -> None:
    """config.cpp:68-127: set one key; CbxInvalidArgument names the key"""
    if key == "box.x":
        cfg.box_x = _parse_long(key, value)
    elif key == "box.y":
        cfg.box_y = _parse_long(key, value)
    elif key == "box.z":
        cfg.box_z = _parse_long(key, value)
    elif key == "box.a0":
        cfg.a0 = _parse_double(key, value)
    elif key == "box.ghost_width":
        cfg.ghost_width = _parse_long(key, value)
    elif key == "temperature":
        cfg.temperature = _parse_double(key, value)
    elif key == "potential":
        cfg.potential_path = value
    elif key == "pka.site":
        cfg.pka.site = tuple(_parse_triple(key, value))
    elif key == "pka.energy":
        cfg.pka.energy_kev = _parse_double(key, value)
    elif key == "pka.direction":
        cfg.pka.direction = tuple(_parse_triple(key, value))
    elif key == "steps":
        cfg.steps = _parse_long(key, value)
    elif key == "max_time":
        cfg.max_time = _parse_double(key, value)
    elif key == "dt_max":
        cfg.dt_max = _parse_double(key, value)
    elif key == "max_disp":
        cfg.max_disp = _parse_double(key, value)
    elif key == "thermostat.mode":
        if value == "off":
            cfg.thermostat.enabled = False
        elif value == "rescale":
            cfg.thermostat.enabled = True
        else:
            _bad(key, f"expected 'off' or 'rescale', got '{value}'")
    elif key == "thermostat.interval":
        cfg.thermostat.interval = _parse_long(key, value)
    elif key == "thermostat.boundary_cells":
        cfg.thermostat.boundary_cells = _parse_long(key, value)
    elif key == "output.timeseries":
        cfg.output.timeseries = value
    elif key == "output.snapshot_prefix":
        cfg.output.snapshot_prefix = value
    elif key == "output.snapshot_interval":
        cfg.output.snapshot_interval = _parse_long(key, value)
    elif key == "output.defect_interval":
        cfg.output.defect_interval = _parse_long(key, value)
    elif key == "workers":
        cfg.workers = _int32(_parse_long(key, value))
    elif key == "seed":
        cfg.seed = _parse_u64(key, value)
    elif key == "equilibration_steps":
        cfg.equilibration_steps = _parse_long(key, value)
    elif key == "displacement_energy":
        cfg.displacement_energy = _parse_double(key, value)
    else:
        raise CbxInvalidArgument(f"unknown config key '{key}'")


def _int32(x: int) -> int:  # static_cast<int>(long)
    x &= 0xFFFFFFFF
    return x - (1 << 32) if x >= 1 << 31 else x


def parse_config_text(cfg: SimConfig, text: str, origin: str) -> None:
    """config.cpp:129-160: errors report origin:line"""
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    for lineno, line in enumerate(lines, 1):
        h = line.find("#")
        if h >= 0:
            line = line[:h]
        entry = _trim(line)
        if not entry:
            continue
        eq = entry.find("=")
        if eq < 0:
            raise CbxInvalidArgument(f"{origin}:{lineno}: expected 'key = value'")
        key, value = _trim(entry[:eq]), _trim(entry[eq + 1:])
        if not key:
            raise CbxInvalidArgument(f"{origin}:{lineno}: empty key")
        try:
            apply_config_entry(cfg, key, value)
        except CbxInvalidArgument as e:
            raise CbxInvalidArgument(f"{origin}:{lineno}: {e}") from None


def load_config(path: str, overrides: Iterable[str] = ()) -> SimConfig:
    """config.cpp:162-188: defaults, CASCADE_WORKERS, the file, overrides;
    validated before returning"""
    cfg = SimConfig()
    env = os.environ.get("CASCADE_WORKERS")
    if env is not None:
        cfg.workers = _int32(_parse_long("CASCADE_WORKERS", env))
    try:
        with open(path, "rb") as f:
            text = f.read().decode("utf-8", "surrogateescape")
    except OSError:
        raise CbxRuntimeError(f"cannot open config file {path}") from None
    parse_config_text(cfg, text, path)
    for ov in overrides:
        eq = ov.find("=")
        if eq < 0:
            raise CbxInvalidArgument(f"override '{ov}' is not of the form key=value")
        apply_config_entry(cfg, _trim(ov[:eq]), _trim(ov[eq + 1:]))
    validate_config(cfg)
    return cfg


def validate_config(cfg: SimConfig) -> None:
    """config.cpp:190-223: range/consistency checks naming the key"""
    if cfg.box_x < 1 or cfg.box_y < 1 or cfg.box_z < 1:
        _bad("box.x/box.y/box.z", "box must be at least 1 cell per axis")
    if cfg.a0 < 0.0:
        _bad("box.a0", "lattice constant cannot be negative")
    if cfg.ghost_width < 0:
        _bad("box.ghost_width", "cannot be negative")
    if cfg.temperature < 0.0:
        _bad("temperature", "cannot be negative")
    if not cfg.dt_max > 0.0:
        _bad("dt_max", "must be positive")
    if not cfg.max_disp > 0.0:
        _bad("max_disp", "must be positive")
    if cfg.a0 > 0.0 and cfg.max_disp >= cfg.a0 / 2.0:
        _bad("max_disp", "must stay below half the lattice constant")
    if cfg.pka.energy_kev < 0.0:
        _bad("pka.energy", "cannot be negative")
    if cfg.pka.energy_kev > 0.0 and tuple(cfg.pka.direction) == (0, 0, 0):
        _bad("pka.direction", "must not be the zero vector")
    sx, sy, sz = cfg.pka.site
    if not (sx < 0 and sy < 0 and sz < 0):
        if (sx < 0 or sy < 0 or sz < 0 or sx >= cfg.box_x or sy >= cfg.box_y
                or sz >= cfg.box_z):
            _bad("pka.site", "cell must lie inside the box")
    if cfg.steps < 0:
        _bad("steps", "cannot be negative")
    if cfg.max_time < 0.0:
        _bad("max_time", "cannot be negative")
    if cfg.thermostat.interval < 1:
        _bad("thermostat.interval", "must be >= 1")
    if cfg.thermostat.boundary_cells < 0:
        _bad("thermostat.boundary_cells", "cannot be negative")
    if cfg.output.snapshot_interval < 0:
        _bad("output.snapshot_interval", "cannot be negative")
    if cfg.output.defect_interval < 0:
        _bad("output.defect_interval", "cannot be negative")
    if cfg.workers < 1:
        _bad("workers", "must be >= 1")
    if cfg.equilibration_steps < 0:
        _bad("equilibration_steps", "cannot be negative")
    if not cfg.displacement_energy > 0.0:
        _bad("displacement_energy", "must be positive")


def nrt_displacements(pka_energy_ev: float, displacement_energy_ev: float) -> float:
    """analysis.cpp:58-65: the NRT displacement estimate"""
    if not displacement_energy_ev > 0.0:
        raise CbxInvalidArgument("displacement energy must be positive")
    if pka_energy_ev < displacement_energy_ev:
        return 0.0
    full = 0.8 * pka_energy_ev / (2.0 * displacement_energy_ev)
    return 1.0 if full < 1.0 else full


def dump_config(cfg: SimConfig) -> str:
    """every config field as ``key=value`` lines (%.17g doubles): the form the
    parity tests compare with the reference's parsed SimConfig"""
    p, t, o = cfg.pka, cfg.thermostat, cfg.output
    g = lambda x: "%.17g" % x  # noqa: E731
    rows = [("box.x", cfg.box_x), ("box.y", cfg.box_y), ("box.z", cfg.box_z),
            ("box.a0", g(cfg.a0)), ("box.ghost_width", cfg.ghost_width),
            ("temperature", g(cfg.temperature)), ("potential", cfg.potential_path),
            ("pka.site", "%d,%d,%d" % tuple(p.site)), ("pka.energy", g(p.energy_kev)),
            ("pka.direction", "%d,%d,%d" % tuple(p.direction)), ("steps", cfg.steps),
            ("max_time", g(cfg.max_time)), ("dt_max", g(cfg.dt_max)),
            ("max_disp", g(cfg.max_disp)), ("thermostat.enabled", int(t.enabled)),
            ("thermostat.interval", t.interval),
            ("thermostat.boundary_cells", t.boundary_cells),
            ("output.timeseries", o.timeseries), ("output.snapshot_prefix", o.snapshot_prefix),
            ("output.snapshot_interval", o.snapshot_interval),
            ("output.defect_interval", o.defect_interval), ("workers", cfg.workers),
            ("seed", cfg.seed), ("equilibration_steps", cfg.equilibration_steps),
            ("displacement_energy", g(cfg.displacement_energy))]
    return "".join(f"{k}={v}\n" for k, v in rows)
