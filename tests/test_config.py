"""The config / CLI front end: config.cpp and
tools/src/main.cpp restated in paper_2107_07866_b200.config / cli.

CPU: the restated config_test.cpp behaviours; the parsed SimConfig and every
error message against the real reference's load_config over many inputs
(oracle/_ref, when built); the synthetic table writer byte-identical to
synthetic::write_table; ``check`` and ``gen-potential`` end to end.
GPU: ``run`` and ``bench-mem`` through the device.
"""
import ctypes as C
import filecmp
import os
import subprocess
import sys

import pytest

from paper_2107_07866_b200 import SimConfig, _lib
from paper_2107_07866_b200.config import (apply_config_entry, dump_config, load_config,
                                          nrt_displacements, parse_config_text,
                                          validate_config)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ref_lib():
    from oracle import oracle
    if not os.path.exists(oracle.REF_LIB):
        pytest.skip("reference harness not built")
    lib = C.CDLL(oracle.REF_LIB)
    lib.ref_load_config.argtypes = [C.c_char_p, C.POINTER(C.c_char_p), C.c_int, C.c_char_p,
                                    C.c_long]
    lib.ref_nrt_displacements.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_double)]
    return lib


def ours(path, overrides):
    try:
        return 0, dump_config(load_config(path, overrides))
    except _lib.CbxInvalidArgument as e:
        return 1, str(e)
    except _lib.CbxRuntimeError as e:
        return 2, str(e)


def theirs(lib, path, overrides):
    ov = (C.c_char_p * max(1, len(overrides)))(*[o.encode() for o in overrides])
    buf = C.create_string_buffer(1 << 14)
    rc = lib.ref_load_config(path.encode(), ov, len(overrides), buf, len(buf))
    return rc, buf.value.decode()


# ---------------------------------------------------- config_test.cpp cases
def test_defaults_are_valid():
    c = SimConfig()
    assert (c.box_x, c.box_y, c.box_z, c.a0, c.ghost_width, c.temperature) == (10, 10, 10, 0.0,
                                                                                0, 0.0)
    assert c.pka.site == (-1, -1, -1) and c.pka.direction == (1, 3, 5)
    assert (c.steps, c.max_time, c.dt_max, c.max_disp) == (0, 0.0, 1e-3, 0.05)
    assert not c.thermostat.enabled and c.thermostat.interval == 10
    assert c.output.defect_interval == 10 and c.output.snapshot_interval == 0
    assert (c.workers, c.seed, c.equilibration_steps, c.displacement_energy) == (1, 12345, 0,
                                                                                 40.0)
    validate_config(c)


def test_every_key_and_malformed_values():
    c = SimConfig()
    for k, v in [("box.x", "20"), ("box.y", "16"), ("box.z", "12"), ("box.a0", "2.8553"),
                 ("box.ghost_width", "3"), ("temperature", "600"), ("potential", "Fe.eam"),
                 ("pka.site", "3,4,5"), ("pka.energy", "1.0"), ("pka.direction", "1 3 5"),
                 ("steps", "1000"), ("max_time", "5.0"), ("dt_max", "0.001"),
                 ("max_disp", "0.02"), ("thermostat.mode", "rescale"),
                 ("thermostat.interval", "25"), ("thermostat.boundary_cells", "2"),
                 ("output.timeseries", "out/defects.csv"), ("output.snapshot_prefix", "out/snap"),
                 ("output.snapshot_interval", "100"), ("output.defect_interval", "5"),
                 ("workers", "8"), ("seed", "987654321"), ("equilibration_steps", "50"),
                 ("displacement_energy", "35")]:
        apply_config_entry(c, k, v)
    assert (c.box_x, c.box_y, c.box_z, c.a0, c.ghost_width) == (20, 16, 12, 2.8553, 3)
    assert c.pka.site == (3, 4, 5) and c.pka.energy_kev == 1.0
    assert c.thermostat.enabled and c.thermostat.interval == 25
    assert c.output.snapshot_prefix == "out/snap" and c.seed == 987654321
    apply_config_entry(c, "thermostat.mode", "off")
    assert not c.thermostat.enabled
    for k, v, msg in [("steps", "ten", "expected an integer, got 'ten'"),
                      ("steps", "12x", "expected an integer"),
                      ("temperature", "warm", "expected a number, got 'warm'"),
                      ("seed", "-4", "expected an unsigned integer"),
                      ("pka.site", "1 2", "expected three integers, got '1 2'"),
                      ("pka.direction", "1 2 3 4", "trailing text '4'"),
                      ("thermostat.mode", "langevin",
                       "expected 'off' or 'rescale', got 'langevin'"),
                      ("cutoff", "5.6", "unknown config key 'cutoff'")]:
        with pytest.raises(_lib.CbxInvalidArgument, match=msg):
            apply_config_entry(c, k, v)


def test_text_comments_and_bad_lines():
    c = SimConfig()
    parse_config_text(c, "# setup\n\nbox.x = 8   # eight\n  temperature=300\npka.site = 1, 2, 3\n",
                      "test.cfg")
    assert c.box_x == 8 and c.temperature == 300.0 and c.pka.site == (1, 2, 3)
    for text, msg in [("box.x = 8\nsteps 100\n", "t.cfg:2: expected 'key = value'"),
                      ("= 5\n", "t.cfg:1: empty key"),
                      ("\n\nsteps = soon\n", "t.cfg:3: steps: expected an integer")]:
        with pytest.raises(_lib.CbxInvalidArgument, match=msg):
            parse_config_text(c, text, "t.cfg")


def test_layering_env_file_overrides(tmp_path, monkeypatch):
    p = tmp_path / "layered.cfg"
    p.write_text("box.x = 6\nbox.y = 6\nbox.z = 6\ntemperature = 150\n")
    monkeypatch.delenv("CASCADE_WORKERS", raising=False)
    assert load_config(str(p)).workers == 1
    monkeypatch.setenv("CASCADE_WORKERS", "9")
    assert load_config(str(p)).workers == 9
    p.write_text("box.x = 6\nworkers = 4\n")
    assert load_config(str(p)).workers == 4
    c = load_config(str(p), ["workers=2", "temperature = 700"])
    assert c.workers == 2 and c.temperature == 700.0
    with pytest.raises(_lib.CbxInvalidArgument, match="override 'workers' is not of the form"):
        load_config(str(p), ["workers"])
    monkeypatch.setenv("CASCADE_WORKERS", "lots")
    with pytest.raises(_lib.CbxInvalidArgument, match="CASCADE_WORKERS: expected an integer"):
        load_config(str(p))
    monkeypatch.delenv("CASCADE_WORKERS")
    with pytest.raises(_lib.CbxRuntimeError, match="cannot open config file"):
        load_config(str(tmp_path / "missing.cfg"))


# --------------------------------------------- against the real reference
CASES = [
    ("", []),
    ("box.x = 6\nbox.y = 7\nbox.z = 8\n", ["temperature=700", "seed = 18446744073709551615"]),
    ("box.x = 0\n", []),
    ("box.a0 = 2.8553\nmax_disp = 1.5\n", []),
    ("box.a0 = -1\n", []), ("box.ghost_width = -1\n", []), ("temperature = -10\n", []),
    ("dt_max = 0\n", []), ("dt_max = nan\n", []), ("max_disp = -0.1\n", []),
    ("pka.energy = -1\n", []), ("pka.energy = 1\npka.direction = 0,0,0\n", []),
    ("pka.site = 1,2\n", []), ("pka.site = 1 2 3 4\n", []), ("pka.site = 1,2,3x\n", []),
    ("pka.site = 1.5 2 3\n", []), ("pka.site = +1, -0, 9\n", []), ("pka.site = 0,0,10\n", []),
    ("pka.site = -1,-1,-1\n", []), ("pka.site = -1,2,3\n", []),
    ("pka.site = 99999999999999999999 1 1\n", []),
    ("steps = -3\n", []), ("steps = 1e3\n", []), ("steps = 0x10\n", []), ("steps = +12\n", []),
    ("steps = 9223372036854775807\n", []), ("steps = 9223372036854775808\n", []),
    ("seed = -4\n", []), ("seed = 18446744073709551616\n", []), ("seed = +7\n", []),
    ("temperature = 1e400\n", []), ("temperature = 1e-400\n", []),
    ("temperature = 1e-310\n", []), ("temperature = inf\n", []), ("temperature = 0x1p4\n", []),
    ("temperature = .5\n", []), ("temperature = 5.\n", []), ("temperature = 1e\n", []),
    ("temperature = 3e2\n", []), ("temperature = Infinity\n", []),
    ("max_time = -1\n", []), ("thermostat.mode = rescale\nthermostat.interval = 0\n", []),
    ("thermostat.mode = Rescale\n", []), ("thermostat.boundary_cells = -2\n", []),
    ("output.snapshot_interval = -1\n", []), ("output.defect_interval = -1\n", []),
    ("workers = 0\n", []), ("workers = 4294967297\n", []), ("equilibration_steps = -1\n", []),
    ("displacement_energy = 0\n", []), ("displacement_energy = 35\n", []),
    ("potential = /a b/c.eam  # trailing\n", []), ("output.timeseries=x.csv\r\n", []),
    ("no equals here\n", []), ("   = 4\n", []), ("cutoff = 5.6\n", []),
    ("box.x = 8 # c\n# only comment\n\n\tsteps\t=\t 12 \n", ["box.y=3", "box.z = 2"]),
    ("box.x = 4\n", ["box.y"]), ("box.x = 4\n", ["nope = 1"]), ("box.x = 4\n", ["box.z=0"]),
    ("box.x = 4\nsteps = 5\nsteps = soon\n", []),
]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_config_matches_reference(tmp_path, monkeypatch, i):
    lib = ref_lib()
    text, ov = CASES[i]
    p = tmp_path / "c.cfg"
    p.write_bytes(text.encode())
    monkeypatch.delenv("CASCADE_WORKERS", raising=False)
    assert ours(str(p), ov) == theirs(lib, str(p), ov)


def test_config_env_and_missing_file_match_reference(tmp_path, monkeypatch):
    lib = ref_lib()
    p = tmp_path / "c.cfg"
    p.write_text("box.x = 5\n")
    for env in ("3", "lots", " 7", "-2"):
        monkeypatch.setenv("CASCADE_WORKERS", env)
        assert ours(str(p), []) == theirs(lib, str(p), [])
    monkeypatch.delenv("CASCADE_WORKERS")
    missing = str(tmp_path / "none.cfg")
    assert ours(missing, []) == theirs(lib, missing, [])


def test_nrt_matches_reference():
    lib = ref_lib()
    for e, ed in [(0.0, 40.0), (39.9, 40.0), (40.0, 40.0), (100.0, 40.0), (1e4, 40.0),
                  (5e4, 35.0), (10.0, 0.0), (10.0, -1.0)]:
        out = C.c_double()
        rc = lib.ref_nrt_displacements(e, ed, C.byref(out))
        if rc:
            with pytest.raises(_lib.CbxInvalidArgument, match="displacement energy"):
                nrt_displacements(e, ed)
        else:
            assert nrt_displacements(e, ed) == out.value


# ------------------------------------------------------------ the CLI (CPU)
def cli(*args, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_2107_07866_b200", *args],
                          capture_output=True, text=True, cwd=cwd or ROOT, timeout=600)


@pytest.mark.parametrize("nrho,nr", [(5000, 5000), (7, 4), (4, 9)])
def test_synthetic_table_bytes_match_reference(tmp_path, nrho, nr):
    from oracle import oracle
    ours_p = str(tmp_path / "o.eam")
    _lib.check(_lib.load().cbx_write_synthetic_table(ours_p.encode(), nrho, nr))
    kind = "ref" if os.path.exists(oracle.REF_LIB) else "oracle"
    ref_p = str(tmp_path / "r.eam")
    oracle.write_synthetic_table(ref_p, nrho, nr, kind=kind)
    assert filecmp.cmp(ours_p, ref_p, shallow=False)


def test_synthetic_table_errors():
    lib = _lib.load()
    assert lib.cbx_write_synthetic_table(b"/tmp/x.eam", 3, 10) == 1
    assert "at least 4 knots" in lib.cbx_last_error(None).decode()
    assert lib.cbx_write_synthetic_table(b"/nonexistent/dir/x.eam", 10, 10) == 2
    assert "cannot open" in lib.cbx_last_error(None).decode()


def test_cli_gen_potential_and_check(tmp_path):
    out = str(tmp_path / "Fe.eam")
    r = cli("gen-potential", "--output", out, "--nrho", "500", "--nr", "400")
    assert r.returncode == 0, r.stderr
    assert r.stdout == f"wrote {out} (Nrho=500, Nr=400, cutoff 5.6 A); parse check OK\n"
    cfg = tmp_path / "c.cfg"
    cfg.write_text(f"potential = {out}\nbox.x = 20\nbox.y = 20\nbox.z = 20\nworkers = 4\n")
    r = cli("check", "--config", str(cfg))
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == "config OK: box 20x20x20 cells, 16000 atoms"
    assert lines[1] == "potential: Z=26, 55.84 amu, cutoff 5.6 A, a0 2.8553 A"
    assert lines[2] == "ghost width: 3 cells; index cutoff 6.457 A"
    assert lines[3] == "offsets per site: even 112 (half 46), odd 112 (half 66)"
    assert lines[4].startswith("partition: device cuda:0, 65 units")
    r = cli("check", "--config", str(cfg), "--set", "box.x=0")
    assert r.returncode == 1
    assert r.stderr == "error: box.x/box.y/box.z: box must be at least 1 cell per axis\n"
    r = cli("check", "--config", str(tmp_path / "missing.cfg"))
    assert r.returncode == 1 and "cannot open config file" in r.stderr


# ------------------------------------------------------------ the CLI (GPU)
@pytest.mark.gpu
def test_cli_run_matches_oracle_run(tmp_path, tables):
    import numpy as np
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import oracle
    o = tmp_path / "o"
    d = tmp_path / "d"
    os.makedirs(o)
    os.makedirs(d)
    spec = dict(steps=40, equilibration_steps=10, thermostat=True, thermostat_interval=5,
                boundary_cells=1, snapshot_interval=20, defect_interval=10)
    s = oracle.Sim(tables["baseline"], box=(6, 6, 6), temperature=600.0, seed=7,
                   pka_energy_kev=0.5, pka_site=(3, 3, 3), boundary_cells=1)
    s.run(oracle.run_spec(timeseries=str(o / "ts.csv"), snapshot_prefix=str(o / "snap"),
                          **spec), str(o / "log.txt"))
    cfg = tmp_path / "run.cfg"
    cfg.write_text(f"""# the oracle's run, through the front end
potential = {tables['baseline']}
box.x = 6
box.y = 6
box.z = 6
temperature = 600
seed = 7
pka.site = 3, 3, 3
pka.energy = 0.5
steps = 40
equilibration_steps = 10
thermostat.mode = rescale
thermostat.interval = 5
thermostat.boundary_cells = 1
output.snapshot_interval = 20
output.defect_interval = 10
""")
    r = cli("run", "--config", str(cfg), "--set", f"output.timeseries={d / 'ts.csv'}",
            "--set", f"output.snapshot_prefix={d / 'snap'}")
    assert r.returncode == 0, r.stderr
    assert filecmp.cmp(d / "ts.csv", o / "ts.csv", shallow=False)
    assert sorted(os.listdir(d)) == sorted(set(os.listdir(o)) - {"log.txt"})
    lines = r.stdout.splitlines()
    assert lines[0].startswith("box 6x6x6 cells, 432 atoms, device cuda:0")
    log = [ln for ln in lines if ln.startswith("step ")]
    ref_log = open(o / "log.txt").read().splitlines()
    assert [ln.split()[:2] for ln in log] == [ln.split()[:2] for ln in ref_log]
    t, dd = s.series()
    peak = int(dd[:, 2].max())
    assert any(ln.startswith("done: 50 steps") for ln in lines)
    assert f"frenkel pairs: peak {peak}" in r.stdout
    assert "nrt estimate: 5 displacements (Ed=40 eV)" in r.stdout
    assert f"final snapshot: {d / 'snap'}_final.xyz" in r.stdout
    assert np.array_equal(np.loadtxt(d / "ts.csv", delimiter=",", skiprows=1),
                          np.loadtxt(o / "ts.csv", delimiter=",", skiprows=1))


@pytest.mark.gpu
def test_cli_bench_mem(tmp_path, tables):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = tmp_path / "m.cfg"
    cfg.write_text(f"potential = {tables['baseline']}\nbox.x = 20\nbox.y = 20\nbox.z = 20\n")
    r = cli("bench-mem", "--config", str(cfg))
    assert r.returncode == 0, r.stderr
    kv = dict(ln.split(": ", 1) for ln in r.stdout.splitlines())
    assert kv["atoms"] == "16000"
    assert kv["slots"].startswith("35152 records")
    assert kv["offset lists"] == f"{4 * (112 + 112 + 46 + 66)} bytes"
    per_atom = float(kv["bytes/atom"])
    assert 100 < per_atom < 1000
