"""The run loop and its outputs: Simulation::run,
thermostat_rescale, the defect time series and the extended-XYZ snapshots
(sim.cpp:188-360, analysis.cpp:66-116).

CPU: the oracle's restatement writes byte-identical files to the real
reference's Simulation::run.  GPU: the device run loop against the oracle.
"""
import filecmp
import os

import numpy as np
import pytest

from helpers import assert_store_parity

SPEC = dict(steps=60, equilibration_steps=10, thermostat=True, thermostat_interval=5,
            boundary_cells=1, snapshot_interval=30, defect_interval=10)


def oracle_run(tables, kind, d, **over):
    from oracle import oracle
    os.makedirs(d, exist_ok=True)
    spec = dict(SPEC, **over)
    s = oracle.Sim(tables["baseline"], box=(6, 6, 6), temperature=600.0, seed=7,
                   pka_energy_kev=0.5, pka_site=(3, 3, 3), kind=kind,
                   boundary_cells=spec["boundary_cells"])
    s.run(oracle.run_spec(timeseries=os.path.join(d, "ts.csv"),
                          snapshot_prefix=os.path.join(d, "snap"), **spec),
          os.path.join(d, "log.txt"))
    return s


def test_oracle_run_matches_reference_bytes(tables, have_ref, tmp_path):
    """log, defect CSV and every snapshot byte-identical to the reference's run"""
    if not have_ref:
        pytest.skip("reference harness not built")
    a = oracle_run(tables, "oracle", str(tmp_path / "o"))
    b = oracle_run(tables, "ref", str(tmp_path / "r"))
    files = sorted(os.listdir(tmp_path / "o"))
    assert files == sorted(os.listdir(tmp_path / "r"))
    assert {"ts.csv", "log.txt", "snap_000000.xyz", "snap_000030.xyz", "snap_000060.xyz",
            "snap_final.xyz"} <= set(files)
    for f in files:
        assert filecmp.cmp(tmp_path / "o" / f, tmp_path / "r" / f, shallow=False), f
    assert a.state()["step"] == b.state()["step"] == 70
    ta, da = a.series()
    tb, db = b.series()
    assert np.array_equal(ta, tb) and np.array_equal(da, db)


def test_oracle_thermostat_matches_reference(tables, have_ref):
    """thermostat_rescale, whole box and a 2-cell boundary band"""
    if not have_ref:
        pytest.skip("reference harness not built")
    from oracle import oracle
    for band in (0, 2):
        a = oracle.Sim(tables["baseline"], box=(7, 6, 6), temperature=300.0, seed=3,
                       boundary_cells=band)
        b = oracle.Sim(tables["baseline"], box=(7, 6, 6), temperature=300.0, seed=3,
                       boundary_cells=band, kind="ref")
        a.step(1e-3, 3)
        b.step(1e-3, 3)
        a.thermostat_rescale()
        b.thermostat_rescale()
        assert a.state() == b.state()
        assert np.array_equal(a.store().vel, b.store().vel)


def test_oracle_run_time_cap_and_no_budget(tables, tmp_path):
    """max_time stops at the first step with t >= max_time; no caps = no steps"""
    from oracle import oracle
    s = oracle.Sim(tables["baseline"], box=(5, 5, 5), temperature=600.0, seed=1)
    s.run(oracle.run_spec(max_time=0.0049, defect_interval=0))
    st = s.state()
    assert st["t"] >= 0.0049 and st["t"] - st["dt"] < 0.0049
    t, d = s.series()
    assert len(t) == 2 and t[0] == 0.0  # start + end samples only
    s2 = oracle.Sim(tables["baseline"], box=(5, 5, 5), temperature=600.0, seed=1)
    s2.run(oracle.run_spec())
    assert s2.state()["step"] == 0 and len(s2.series()[0]) == 1


# --------------------------------------------------------------- on the GPU
@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2107_07866_b200 import _lib
    _lib.load()
    return True


def device_sim(tables, **spec):
    from paper_2107_07866_b200 import (OutputSpec, PkaSpec, SimConfig, Simulation,
                                       ThermostatSpec)
    sp = dict(SPEC, **spec)
    cfg = SimConfig(box_x=6, box_y=6, box_z=6, temperature=600.0, seed=7,
                    potential_path=tables["baseline"], steps=sp["steps"],
                    equilibration_steps=sp["equilibration_steps"],
                    max_time=sp.get("max_time", 0.0),
                    pka=PkaSpec(site=(3, 3, 3), energy_kev=0.5),
                    thermostat=ThermostatSpec(enabled=sp["thermostat"],
                                              interval=sp["thermostat_interval"],
                                              boundary_cells=sp["boundary_cells"]),
                    output=OutputSpec(snapshot_interval=sp["snapshot_interval"],
                                      defect_interval=sp["defect_interval"]))
    return Simulation(cfg), cfg


def read_xyz(path):
    lines = open(path).read().splitlines()
    rows = [ln.split() for ln in lines[2:]]
    tags = np.array([int(r[4]) for r in rows])
    pos = np.array([[float(x) for x in r[1:4]] for r in rows])
    return lines[0], lines[1], [r[0] for r in rows], tags, pos


@pytest.mark.gpu
@pytest.mark.parametrize("band", [0, 2])
def test_device_thermostat_matches_oracle(cuda, tables, band):
    from oracle import oracle
    from paper_2107_07866_b200 import DeviceStore, EamPotential
    ref = oracle.Sim(tables["baseline"], box=(7, 6, 6), temperature=300.0, seed=3,
                     boundary_cells=band)
    ref.step(1e-3, 3)
    dims, a0, g = ref.box
    dev = DeviceStore((*dims, a0, g), EamPotential.load(tables["baseline"]))
    dev.upload(ref.store())
    dev.set_state(ref.state())
    ref.thermostat_rescale()
    dev.thermostat_rescale(300.0, band)
    sr, sd = ref.state(), dev.state()
    assert abs(sd["kinetic"] - sr["kinetic"]) <= 1e-12 * sr["kinetic"]
    assert abs(sd["max_speed"] - sr["max_speed"]) <= 1e-12 * sr["max_speed"]
    assert_store_parity(ref.store(), dev.download(), rel=1e-10)


@pytest.mark.gpu
def test_device_snapshot_and_series_writers_bytes(cuda, tables, tmp_path):
    """for the same store the device writers produce the oracle's bytes"""
    from oracle import oracle
    from paper_2107_07866_b200 import DeviceStore, EamPotential, _lib
    import ctypes as C
    ref = oracle.Sim(tables["baseline"], box=(6, 6, 6), temperature=600.0, seed=11,
                     pka_energy_kev=1.0, pka_site=(3, 3, 3))
    ref.step(1e-3, 5)
    ref.inject_pka()
    ref.step(1e-4, 40)  # clash records in the store
    assert (ref.store().clash_ghost == 0).sum() > 0
    dims, a0, g = ref.box
    dev = DeviceStore((*dims, a0, g), EamPotential.load(tables["baseline"]))
    dev.upload(ref.store())
    t = ref.state()["t"]
    ref.write_snapshot(str(tmp_path / "o.xyz"))
    dev.write_snapshot(str(tmp_path / "d.xyz"), t)
    assert filecmp.cmp(tmp_path / "o.xyz", tmp_path / "d.xyz", shallow=False)
    ts = np.array([0.0, 0.5, 1.25e-3, 2.0])
    dd = np.array([0, 0, 0, 1, 2, 2, 3, 3, 3, 10, 12, 12], dtype=np.int64)
    _lib.check(_lib.load().cbx_write_timeseries(
        str(tmp_path / "d.csv").encode(), 4, ts.ctypes.data_as(C.POINTER(C.c_double)),
        dd.ctypes.data_as(C.POINTER(C.c_long))))
    oracle.lib().orc_write_timeseries(str(tmp_path / "o.csv").encode(), 4,
                                      ts.ctypes.data_as(C.POINTER(C.c_double)),
                                      dd.ctypes.data_as(C.POINTER(C.c_long)))
    assert filecmp.cmp(tmp_path / "o.csv", tmp_path / "d.csv", shallow=False)
    assert open(tmp_path / "d.csv").read().splitlines()[1] == "0.0,0,0,0"


@pytest.mark.gpu
def test_device_run_matches_oracle(cuda, tables, tmp_path):
    """equilibration with a boundary-band thermostat, PKA, 60 adaptive steps:
    the defect series is identical, the log lines and snapshots agree"""
    ref = oracle_run(tables, "oracle", str(tmp_path / "o"))
    sim, cfg = device_sim(tables)
    d = tmp_path / "d"
    os.makedirs(d)
    cfg.output.timeseries = str(d / "ts.csv")
    cfg.output.snapshot_prefix = str(d / "snap")
    sim.run(str(d / "log.txt"))
    assert sorted(os.listdir(d)) == sorted(os.listdir(tmp_path / "o"))
    assert filecmp.cmp(d / "ts.csv", tmp_path / "o" / "ts.csv", shallow=False)
    assert sim.state["step"] == ref.state()["step"] == 70
    t1, d1 = sim.series
    t0, d0 = ref.series()
    assert np.array_equal(d1, d0) and np.allclose(t1, t0, rtol=1e-12, atol=0)
    # log lines: same fields; energies / temperatures to their printed digits
    la = open(d / "log.txt").read().splitlines()
    lb = open(tmp_path / "o" / "log.txt").read().splitlines()
    assert len(la) == len(lb) == 6
    for x, y in zip(la, lb):
        fx, fy = x.split(), y.split()
        assert [f.split("=")[0] for f in fx] == [f.split("=")[0] for f in fy]
        assert fx[0:2] == fy[0:2] and fx[-1] == fy[-1]  # step number, FP count
        ex, ey = float(fx[4].split("=")[1]), float(fy[4].split("=")[1])
        assert abs(ex - ey) <= 2e-6 + 1e-9 * abs(ey)
    for f in ("snap_000000.xyz", "snap_000030.xyz", "snap_000060.xyz", "snap_final.xyz"):
        n0, h0, s0, tg0, p0 = read_xyz(tmp_path / "o" / f)
        n1, h1, s1, tg1, p1 = read_xyz(d / f)
        assert n0 == n1 and s0 == s1 and np.array_equal(tg0, tg1), f
        assert h0.split(" Time=")[0] == h1.split(" Time=")[0]
        assert np.abs(p0 - p1).max() <= 1e-7, f


@pytest.mark.gpu
def test_device_run_time_cap(cuda, tables):
    """max_time: the loop stops at the first step reaching it (per-step check)"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(6, 6, 6), temperature=600.0, seed=7)
    ref.run(oracle.run_spec(max_time=0.0049, defect_interval=2))
    sim, cfg = device_sim(tables, steps=0, equilibration_steps=0, thermostat=False,
                          snapshot_interval=0, defect_interval=2, max_time=0.0049)
    cfg.pka.energy_kev = 0.0
    sim.run()
    assert sim.state["step"] == ref.state()["step"]
    assert np.array_equal(sim.series[1], ref.series()[1])


@pytest.mark.gpu
def test_async_snapshot_overlaps_steps(cuda, tables, tmp_path):
    """cbx_write_snapshot_async (the run loop's snapshots, analysis.cpp:90-116):
    the store is packed on the step stream, copied on a side stream and
    written by a host thread while later steps run; the file holds the state
    at the call, byte-identical to the synchronous writer's and to the
    oracle's; two in flight, a third waits for the oldest"""
    from oracle import oracle
    from paper_2107_07866_b200 import DeviceStore, EamPotential
    ref = oracle.Sim(tables["baseline"], box=(7, 6, 5), temperature=600.0, seed=11,
                     pka_energy_kev=0.3, pka_site=(3, 3, 2))
    ref.step(1e-3, 3)
    ref.inject_pka()
    ref.step(1e-4, 30)  # off-lattice records in the clash list
    dims, a0, g = ref.box
    pot = EamPotential.load(tables["baseline"])
    a = DeviceStore((*dims, a0, g), pot)
    b = DeviceStore((*dims, a0, g), pot)
    for d in (a, b):
        d.upload(ref.store())
        d.set_state(ref.state())
    t = ref.state()["t"]
    ref.write_snapshot(str(tmp_path / "o.xyz"))
    a.write_snapshot(str(tmp_path / "a.xyz"), t)
    b.write_snapshot_async(str(tmp_path / "b1.xyz"), t)
    b.step(1e-4, 5)
    b.write_snapshot_async(str(tmp_path / "b2.xyz"))
    b.step(1e-4, 5)
    b.write_snapshot_async(str(tmp_path / "b3.xyz"))  # waits for b1's writer
    b.snapshot_wait()
    assert filecmp.cmp(tmp_path / "a.xyz", tmp_path / "b1.xyz", shallow=False)
    assert filecmp.cmp(tmp_path / "o.xyz", tmp_path / "b1.xyz", shallow=False)
    ref.step(1e-4, 5)
    ref.write_snapshot(str(tmp_path / "o2.xyz"))
    n0, h0, s0, tg0, p0 = read_xyz(tmp_path / "o2.xyz")
    n1, h1, s1, tg1, p1 = read_xyz(tmp_path / "b2.xyz")
    assert n0 == n1 and np.array_equal(tg0, tg1) and np.abs(p0 - p1).max() <= 1e-9
    assert os.path.getsize(tmp_path / "b3.xyz") > 0
