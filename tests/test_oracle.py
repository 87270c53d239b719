"""CPU: pin the oracle (plain-C restatement, oracle/cascade_oracle.c) before
trusting it -- against the reference's own known-answer tests and golden
values, against committed golden vectors generated from the
real reference (tests/golden/), and bit-for-bit against the real reference
core compiled from /root/reference (oracle/_ref, where it was built)."""
import json
import math
import os

import numpy as np
import pytest

from helpers import real_mask

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def O():
    from oracle import oracle
    return oracle


# ---------------------------------------------------------- known answers
def test_pka_speed_kat():
    """sim_test.cpp:41-55"""
    assert O().pka_speed(1000.0, 55.845) == pytest.approx(587.8323710323659, rel=1e-14)
    assert O().pka_speed(0.0, 55.845) == 0.0


def test_adaptive_dt_kat():
    """sim_test.cpp:57-67"""
    ad = O().adaptive_dt
    assert ad(0.0) == 1e-3
    assert ad(10.0) == 1e-3
    assert ad(587.8323710323659) == pytest.approx(8.505826229370246e-05, rel=1e-14)
    assert ad(1e9) == 1e-7
    assert ad(0.0, dt_max=2e-3) == 2e-3


def test_offset_shells(tables):
    """neighbors_test.cpp:24-53: BCC shells 58 within 5.6 A, 112 at the
    engine's index cutoff; half lists = positive offsets; centrosymmetry"""
    s = O().Sim(tables["synthetic"], box=(8, 8, 8), init_lattice=False)
    off = s.offsets()
    assert len(off["even_full"]) == 112 and len(off["odd_full"]) == 112
    assert len(off["even_half"]) + len(off["odd_half"]) == 112
    assert np.array_equal(off["even_half"], off["even_full"][off["even_full"] > 0])
    assert np.array_equal(np.sort(-off["even_full"]), off["odd_full"])
    assert off["z_reach"] == 2


def test_perfect_lattice_synthetic(tables):
    """forces_test.cpp:127-147: rho = 1 +- 1e-8, |f| <= 1e-9, -4.3 eV/atom"""
    s = O().Sim(tables["synthetic"], box=(5, 5, 5), temperature=0.0)
    st = s.store()
    m = real_mask(st)
    assert m.sum() == 250
    assert np.abs(st.rho[m] - 1.0).max() <= 1e-8
    assert np.abs(st.force[m]).max() <= 1e-9
    e = s.state()
    assert (e["embedding"] + e["pair"]) / 250 == pytest.approx(-4.3, rel=1e-4)


def test_baseline_kat(tables):
    """BASELINE table at rho_max = 40, perfect lattice"""
    s = O().Sim(tables["baseline40"], box=(5, 5, 5), temperature=0.0)
    st = s.store()
    m = real_mask(st)
    assert np.abs(st.rho[m] - 11.80956811317917).max() <= 2.2e-13
    assert np.abs(st.df[m] + 0.145496650894856).max() <= 1e-14
    e = s.state()
    assert e["embedding"] / 250 == pytest.approx(-3.4365052179757, abs=1e-12)
    assert e["pair"] / 250 == pytest.approx(-3.6755476296970, abs=1e-11)
    assert np.abs(st.force[m]).max() <= 1e-13


def test_guard_counters(tables):
    """forces_test.cpp:487-531"""
    s = O().Sim(tables["synthetic"], box=(4, 4, 4), init_lattice=False)
    _, a, g = s.box
    c = np.array([4 * a, 4 * a, 4 * a])
    for i, o in enumerate([(0.010, 0.011, 0.009), (-0.012, 0.008, -0.010),
                           (0.009, -0.011, 0.010), (-0.008, -0.009, -0.011)]):
        s.insert(c + o, i)
    s.fill_ghosts()
    s.eval_forces()
    assert s.guards() == (0, 4)
    s2 = O().Sim(tables["synthetic"], box=(4, 4, 4), init_lattice=False)
    s2.insert(c, 1)
    s2.insert(c + [5e-4, 0, 0], 2)
    s2.fill_ghosts()
    s2.compute_density()
    s2.compute_embedding()
    s2.compute_pair()
    assert s2.guards()[0] == 3


def test_overlap_message(tables):
    """forces_test.cpp:533-557"""
    s = O().Sim(tables["synthetic"], box=(4, 4, 4), init_lattice=False)
    _, a, g = s.box
    c = np.array([4 * a, 4 * a, 4 * a])
    s.insert(c, 11)
    s.insert(c + [5e-7, 0, 0], 22)
    s.fill_ghosts()
    with pytest.raises(RuntimeError) as e:
        s.compute_density()
    assert "overlap" in str(e.value) and "11" in str(e.value) and "22" in str(e.value)


def test_cold_lattice_fixed_point(tables):
    """sim_test.cpp:161-183"""
    s = O().Sim(tables["synthetic"], box=(5, 5, 5), temperature=0.0)
    s.step(-1, 5)
    st = s.state()
    assert st["step"] == 5 and st["kinetic"] <= 1e-20 and st["max_speed"] <= 1e-10
    assert s.count_defects() == (0, 0, 0)


def test_nve_conservation_synthetic(tables):
    """sim_test.cpp:185-199 (shortened: 60 steps at 300 K on 6^3)"""
    s = O().Sim(tables["synthetic"], box=(6, 6, 6), temperature=300.0, seed=2027)
    e = lambda st: st["kinetic"] + st["pair"] + st["embedding"]
    e0 = e(s.state())
    s.step(1e-3, 60)
    assert abs(e(s.state()) - e0) <= 1e-4 * abs(e0)
    st = s.store()
    m = real_mask(st)
    p = st.vel[m].sum(axis=0) + st.clash_vel[st.clash_ghost == 0].sum(axis=0)
    assert np.abs(p).max() <= 1e-8


# ------------------------------------------------ committed golden vectors
def _golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} missing (run tests/golden/make_golden.py)")
    return np.load(path)


def test_golden_cascade_vectors(tables):
    """tests/golden/cascade_8.npz: a 1 keV cascade on an 8^3 box generated
    by the REAL reference (make_golden.py); the oracle must reproduce every
    bit of the final store and state"""
    g = _golden("cascade_8.npz")
    meta = json.loads(str(g["meta"]))
    from paper_2107_07866_b200.potential import write_baseline_table
    s = O().Sim(tables["baseline"], **meta["sim"])
    s.step(meta["dt0"], meta["n0"])
    s.inject_pka()
    s.step(meta["dt1"], meta["n1"])
    st = s.store()
    m = real_mask(st)
    assert np.array_equal(np.nonzero(m)[0], g["slot_ids"])
    assert np.array_equal(st.tag[m], g["slot_tag"])
    assert np.array_equal(st.pos[m], g["slot_pos"])
    assert np.array_equal(st.force[m], g["slot_force"])
    assert np.array_equal(st.rho[m], g["slot_rho"])
    assert np.array_equal(st.clash_key, g["clash_key"])
    assert np.array_equal(st.clash_tag, g["clash_tag"])
    assert np.array_equal(st.clash_pos, g["clash_pos"])
    e = s.state()
    assert [e[k] for k in ("kinetic", "pair", "embedding")] == list(g["energies"])
    assert list(s.count_defects()) == list(g["defects"])


def test_golden_table_checksum(tables):
    """the BASELINE table writer is deterministic: its spline tables hash to
    the committed value"""
    g = _golden("cascade_8.npz")
    s = O().Sim(tables["baseline"], box=(4, 4, 4), init_lattice=False)
    h = 0.0
    for w in range(3):
        _, _, seg = s.spline(w)
        h += float(np.abs(seg).sum())
    assert h == float(g["table_abs_sum"])


# ----------------------------------------- bit-for-bit vs the real reference
def _same(a, b):
    A, B = a.store(), b.store()
    for f in A.__dataclass_fields__:
        if not np.array_equal(getattr(A, f), getattr(B, f)):
            return f
    return None if a.state() == b.state() else "state"


@pytest.mark.parametrize("box,temp,pka", [((8, 8, 8), 600.0, 1.0), ((3, 2, 4), 300.0, 0.0),
                                          ((1, 1, 1), 300.0, 0.0)])
def test_oracle_equals_reference(tables, have_ref, box, temp, pka):
    if not have_ref:
        pytest.skip("reference harness not built (oracle/_ref)")
    kw = dict(box=box, temperature=temp, seed=12345, pka_energy_kev=pka,
              pka_site=tuple(b // 2 for b in box))
    a = O().Sim(tables["baseline"], kind="oracle", **kw)
    b = O().Sim(tables["baseline"], kind="ref", **kw)
    assert _same(a, b) is None
    a.step(1e-3, 10)
    b.step(1e-3, 10)
    assert _same(a, b) is None
    if pka:
        a.inject_pka()
        b.inject_pka()
        for _ in range(6):
            a.step(1e-4, 20)
            b.step(1e-4, 20)
            assert _same(a, b) is None
            assert a.count_defects() == b.count_defects()


def test_oracle_equals_reference_clash_scenario(tables, have_ref):
    if not have_ref:
        pytest.skip("reference harness not built (oracle/_ref)")
    sims = [O().Sim(tables["synthetic"], box=(4, 4, 4), temperature=0.0, kind=k)
            for k in ("oracle", "ref")]
    for s in sims:
        dims, a, g = s.box
        tx, ty = dims[0] + 2 * g, dims[1] + 2 * g
        cid = lambda x, y, z: (z * ty + y) * 2 * tx + x
        site = lambda x, y, z: (np.array([0.5 * x * a, y * a, z * a]) if x % 2 == 0 else
                                np.array([0.5 * (x - 1) * a + 0.5 * a, y * a + 0.5 * a,
                                          z * a + 0.5 * a]))
        s.set_atom(cid(10, 5, 5), pos=site(11, 5, 5) + [0.15, 0.02, -0.04])
        s.set_atom(cid(7, 3, 3), pos=site(6, 3, 3) + [-0.12, 0.08, 0.1])
        s.set_atom(cid(12, 4, 6), pos=site(13, 5, 6) + [0.15, 0.0, 0.05])
        s.set_atom(cid(12, 6, 6), pos=site(13, 5, 6) + [-0.1, 0.12, -0.06])
        s.rehash()
        s.eval_forces()
    assert _same(*sims) is None
