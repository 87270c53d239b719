"""GPU parity: the sm_100a path through the C ABI against the CPU oracle
(oracle/cascade_oracle.c, itself pinned bit-for-bit to the reference in
tests/test_oracle.py) on identical seeded inputs.

Tolerances (BASELINE.json north star): slot/clash structure, hash ids and
neighbour sets bit-exact; rho, dF, per-atom forces within 1e-10 relative
(forces: relative to max(|f|, 1 eV/A)); energies within 1e-10 relative.
Mirrors the reference's forces_test.cpp / sim_test.cpp / store_test.cpp.
"""
import math

import numpy as np
import pytest

from helpers import assert_store_parity, by_tag, real_mask, structure

pytestmark = pytest.mark.gpu

REL = 1e-10


@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2107_07866_b200 import _lib
    _lib.load()
    return True


def device_for(sim, path, stencil="newton3"):
    from paper_2107_07866_b200 import DeviceStore, EamPotential
    dims, a0, g = sim.box
    dev = DeviceStore((*dims, a0, g), EamPotential.load(path), stencil=stencil)
    dev.upload(sim.store())
    return dev


def close(a, b, rel=REL):
    return abs(a - b) <= rel * max(abs(a), abs(b), 1e-300)


# --------------------------------------------------------------- storage
def test_init_bcc_bit_identical(cuda, tables):
    """init_bcc (sim.cpp:100-130): positions, velocities, tags bit-equal"""
    from oracle import oracle
    from paper_2107_07866_b200 import DeviceStore, EamPotential
    ref = oracle.Sim(tables["baseline"], box=(7, 6, 5), temperature=600.0, seed=4242)
    dims, a0, g = ref.box
    dev = DeviceStore((*dims, a0, g), EamPotential.load(tables["baseline"]))
    n = dev.init_bcc(600.0, 4242)
    assert n == 2 * 7 * 6 * 5
    a, b = ref.store(), dev.download()
    m = real_mask(a)
    assert np.array_equal(m, real_mask(b))
    assert np.array_equal(a.pos[m], b.pos[m])
    assert np.array_equal(a.vel[m], b.vel[m])
    assert np.array_equal(a.tag[m], b.tag[m])
    # ghost shell regenerated on the device = fill_ghosts (store.cpp:120-195)
    gm = a.valid.astype(bool) & a.ghost.astype(bool)
    assert np.array_equal(gm, b.valid.astype(bool) & b.ghost.astype(bool))
    assert np.array_equal(a.pos[gm], b.pos[gm])
    assert np.array_equal(a.tag[gm], b.tag[gm])


# ----------------------------------------------------------- force engine
@pytest.mark.parametrize("stencil", ["newton3", "full", "reference"])
@pytest.mark.parametrize("temp", [0.0, 600.0])
def test_eval_forces_lattice(cuda, tables, stencil, temp):
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(8, 8, 8), temperature=temp, seed=12345)
    if temp:
        ref.step(1e-3, 5)  # thermal disorder
    dev = device_for(ref, tables["baseline"], stencil)
    e_ref = ref.eval_forces()
    e_dev = dev.eval_forces()
    assert close(e_ref[0], e_dev[0]) and close(e_ref[1], e_dev[1]), (e_ref, e_dev)
    assert_store_parity(ref.store(), dev.download(), what=f"{stencil} T={temp}")


def test_perfect_lattice_kat(cuda, tables):
    """SURVEY §8(c) KAT for the BASELINE table at rho_max = 40"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline40"], box=(5, 5, 5), temperature=0.0)
    dev = device_for(ref, tables["baseline40"])
    emb, pair = dev.eval_forces()
    s = dev.download()
    m = real_mask(s)
    n = m.sum()
    assert n == 250
    assert np.abs(s.rho[m] - 11.80956811317917).max() < 1e-11
    assert np.abs(s.df[m] + 0.145496650894856).max() < 1e-12
    assert abs(emb / n + 3.4365052179757) < 1e-11
    assert abs(pair / n + 3.6755476296970) < 1e-11
    assert np.abs(s.force[m]).max() < 1e-12


def test_synthetic_potential_perfect_lattice(cuda, tables):
    """forces_test.cpp:127-147 on the reference's own synthetic table"""
    from oracle import oracle
    ref = oracle.Sim(tables["synthetic"], box=(5, 5, 5), temperature=0.0)
    dev = device_for(ref, tables["synthetic"])
    emb, pair = dev.eval_forces()
    s = dev.download()
    m = real_mask(s)
    assert np.abs(s.force[m]).max() <= 1e-9
    assert np.abs(s.rho[m] - 1.0).max() <= 1e-8
    assert (emb + pair) / m.sum() == pytest.approx(-4.3, rel=1e-4)


def _clash_scenario(path, a0=None):
    """forces_test.cpp:262-306: interior, boundary and stacked clash buckets"""
    from oracle import oracle
    ref = oracle.Sim(path, box=(4, 4, 4), a0=a0 or 0.0, temperature=0.0, init_lattice=True)
    dims, a, g = ref.box
    tx, ty = dims[0] + 2 * g, dims[1] + 2 * g

    def cid(x, y, z):
        return (z * ty + y) * 2 * tx + x

    def site(x, y, z):
        if x % 2 == 0:
            return np.array([0.5 * x * a, y * a, z * a])
        return np.array([0.5 * (x - 1) * a + 0.5 * a, y * a + 0.5 * a, z * a + 0.5 * a])

    ref.set_atom(cid(10, 5, 5), pos=site(11, 5, 5) + [0.15, 0.02, -0.04])
    ref.set_atom(cid(7, 3, 3), pos=site(6, 3, 3) + [-0.12, 0.08, 0.1])
    ref.set_atom(cid(12, 4, 6), pos=site(13, 5, 6) + [0.15, 0.0, 0.05])
    ref.set_atom(cid(12, 6, 6), pos=site(13, 5, 6) + [-0.1, 0.12, -0.06])
    ref.rehash()
    return ref


@pytest.mark.parametrize("stencil", ["newton3", "full", "reference"])
@pytest.mark.parametrize("table", ["baseline", "synthetic"])
def test_clash_buckets_interior_boundary_stacked(cuda, tables, table, stencil):
    ref = _clash_scenario(tables[table])
    s0 = ref.store()
    assert (s0.clash_ghost == 0).sum() >= 4
    dev = device_for(ref, tables[table], stencil)
    # the device's own ghost images of the clash buckets equal fill_ghosts'
    assert structure(s0)[1] == structure(dev.download())[1]
    e_ref = ref.eval_forces()
    e_dev = dev.eval_forces()
    assert close(e_ref[0], e_dev[0]) and close(e_ref[1], e_dev[1]), (e_ref, e_dev)
    assert_store_parity(ref.store(), dev.download(), what=table)


@pytest.mark.parametrize("stencil", ["newton3", "full"])
@pytest.mark.parametrize("box", [(1, 1, 1), (2, 3, 1), (3, 3, 3), (4, 2, 5)])
def test_tiny_boxes_many_images(cuda, tables, box, stencil):
    """boxes thinner than the ghost shell: several images per atom, self
    images (acceptance.cpp:100-130 sweeps 1..6^3)"""
    from oracle import oracle
    ref = oracle.Sim(tables["synthetic"], box=box, temperature=300.0, seed=7)
    ref.step(1e-3, 2)
    dev = device_for(ref, tables["synthetic"], stencil)
    e_ref, e_dev = ref.eval_forces(), dev.eval_forces()
    assert close(e_ref[0], e_dev[0], 1e-9) and close(e_ref[1], e_dev[1], 1e-9), (e_ref, e_dev)
    assert_store_parity(ref.store(), dev.download(), what=str(box))


def test_serial_contracts(cuda, tables):
    """compute_density / compute_embedding_derivative / compute_pair_forces"""
    from oracle import oracle
    ref = _clash_scenario(tables["baseline"])
    dev = device_for(ref, tables["baseline"])
    ref.compute_density()
    dev.compute_density()
    a, b = by_tag(ref.store()), by_tag(dev.download())
    for t in a:
        assert close(a[t][3], b[t][3]), t
    assert close(ref.compute_embedding(), dev.compute_embedding_derivative())
    assert close(ref.compute_pair(), dev.compute_pair_forces())
    assert_store_parity(ref.store(), dev.download())


def test_beyond_cutoff_silent(cuda, tables):
    """forces_test.cpp:99-125"""
    from oracle import oracle
    ref = oracle.Sim(tables["synthetic"], box=(4, 4, 4), init_lattice=False)
    _, a, g = ref.box
    p = np.array([3 * a, 4 * a, 4 * a])
    ref.insert(p, 1)
    ref.insert(p + [5.7, 0, 0], 2)
    ref.fill_ghosts()
    dev = device_for(ref, tables["synthetic"])
    emb, pair = dev.eval_forces()
    assert pair == 0.0
    s = dev.download()
    m = real_mask(s)
    assert np.all(s.rho[m] == 0.0) and np.all(s.force[m] == 0.0)


def test_dimer_antisymmetric(cuda, tables):
    """forces_test.cpp:54-97: closed form, bit-exact antisymmetry"""
    from oracle import oracle
    ref = oracle.Sim(tables["synthetic"], box=(4, 4, 4), init_lattice=False)
    _, a, g = ref.box
    p = np.array([4 * a, 4 * a, 4 * a])
    ref.insert(p, 1)
    ref.insert(p + [2.2, 0, 0], 2)
    ref.fill_ghosts()
    dev = device_for(ref, tables["synthetic"])
    dev.eval_forces()
    t = by_tag(dev.download())
    f1, f2 = t[1][2], t[2][2]
    assert f1[0] == -f2[0] and f1[1] == 0.0 and f1[2] == 0.0 and f2[1] == 0.0
    want_rho = ref.potential_eval(0, 2.2)[0]
    assert abs(t[1][3] - want_rho) <= 1e-12 * want_rho


def test_guard_counters(cuda, tables):
    """forces_test.cpp:487-531: 4 rho clamps; 3 short-range guard hits"""
    from oracle import oracle
    from paper_2107_07866_b200 import DeviceStore, EamPotential
    ref = oracle.Sim(tables["synthetic"], box=(4, 4, 4), init_lattice=False)
    dims, a, g = ref.box
    c = np.array([4 * a, 4 * a, 4 * a])
    for i, o in enumerate([(0.010, 0.011, 0.009), (-0.012, 0.008, -0.010),
                           (0.009, -0.011, 0.010), (-0.008, -0.009, -0.011)]):
        ref.insert(c + o, i)
    ref.fill_ghosts()
    dev = device_for(ref, tables["synthetic"])
    dev.eval_forces()
    assert dev.guards() == (0, 4)
    ref2 = oracle.Sim(tables["synthetic"], box=(4, 4, 4), init_lattice=False)
    ref2.insert(c, 1)
    ref2.insert(c + [5e-4, 0, 0], 2)
    ref2.fill_ghosts()
    dev2 = device_for(ref2, tables["synthetic"])
    dev2.eval_forces()
    assert dev2.guards()[0] == 3


def test_overlap_names_both_tags(cuda, tables):
    """forces_test.cpp:533-557"""
    from oracle import oracle
    from paper_2107_07866_b200._lib import CbxRuntimeError
    ref = oracle.Sim(tables["synthetic"], box=(4, 4, 4), init_lattice=False)
    _, a, g = ref.box
    c = np.array([4 * a, 4 * a, 4 * a])
    ref.insert(c, 11)
    ref.insert(c + [5e-7, 0, 0], 22)
    ref.fill_ghosts()
    dev = device_for(ref, tables["synthetic"])
    with pytest.raises(CbxRuntimeError) as e:
        dev.compute_density()
    msg = str(e.value)
    assert "overlap" in msg and "11" in msg and "22" in msg


# ------------------------------------------------------------ step loop
@pytest.mark.parametrize("stencil", ["newton3", "full", "reference"])
def test_trajectory_config1_shape(cuda, tables, stencil):
    """BASELINE config 1 shape (600 K, dt 1 fs) on a 10^3 box: 100 steps,
    state checked every 25 steps; energies and drift against the oracle"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(10, 10, 10), temperature=600.0, seed=12345)
    dev = device_for(ref, tables["baseline"], stencil)
    dev.set_state(ref.state())
    e0 = ref.state()
    for chunk in range(4):
        ref.step(1e-3, 25)
        st = dev.step(1e-3, 25)
        sr = ref.state()
        assert st["step"] == sr["step"]
        for k in ("kinetic", "pair", "embedding"):
            assert abs(st[k] - sr[k]) <= 1e-9 * abs(sr[k]), (k, st[k], sr[k])
        assert_store_parity(ref.store(), dev.download(), pos_tol=1e-9, rel=1e-8,
                            what=f"chunk {chunk}")
    etot = lambda s: s["kinetic"] + s["pair"] + s["embedding"]
    drift_ref = etot(ref.state()) - etot(e0)
    drift_dev = etot(dev.state()) - etot(e0)
    assert abs(drift_dev - drift_ref) <= 0.01 * abs(drift_ref) + 1e-9 * abs(etot(e0))


@pytest.mark.parametrize("stencil", ["newton3", "full"])
def test_cascade_clash_and_defects(cuda, tables, stencil):
    """PKA cascade on a 10^3 box: off-lattice atoms go through the device
    clash list; hash ids, bucket membership/order and Wigner-Seitz counts
    match the oracle at every checkpoint"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(10, 10, 10), temperature=600.0, seed=12345,
                     pka_energy_kev=1.0, pka_site=(5, 5, 5))
    ref.step(1e-3, 10)
    dev = device_for(ref, tables["baseline"], stencil)
    dev.set_state(ref.state())
    ref.inject_pka()
    st = ref.state()
    s = ref.store()
    _, a, g = ref.box
    tx = 10 + 2 * g
    site = ((g + 5) * tx + (g + 5)) * 2 * tx + 2 * (g + 5)
    dev.inject_pka(site, s.vel[site])
    assert abs(dev.state()["kinetic"] - st["kinetic"]) <= 1e-12 * st["kinetic"]
    saw_clash = False
    for chunk in range(8):
        ref.step(1e-4, 25)
        sd = dev.step(1e-4, 25)
        # StepState of a multi-step call: the sums of the last step (clash
        # records included) after the merged / deferred kicks are flushed
        sr = ref.state()
        assert sd["step"] == sr["step"]
        for k in ("kinetic", "pair", "embedding", "max_speed"):
            assert close(sd[k], sr[k], 1e-9), (chunk, k, sd[k], sr[k])
        rs, ds = ref.store(), dev.download()
        saw_clash |= (rs.clash_ghost == 0).sum() > 0
        assert ref.count_defects() == dev.count_defects(), chunk
        assert_store_parity(rs, ds, pos_tol=1e-8, rel=1e-7, what=f"cascade chunk {chunk}")
    assert saw_clash


@pytest.mark.parametrize("rho_k,compressed", [(2.0, 1), (12.0, 0)])
def test_density_record_guard_local(cuda, tables, tmp_path, rho_k, compressed):
    """The compressed density records (fp32 A, B) are used only where the
    local guard of setup_fast holds: for every segment of the staged window
    the fp32 rounding moves rho(s) by <= 1e-12 of the smallest |rho| the
    segment takes.  BASELINE (rho = exp(-2(r - 2.48))): 1.5e-13, compressed;
    a steep rho = exp(-12(r - 2.48)): 5.4e-12, so the fp64 records are kept.
    Both meet the 1e-10 parity with the oracle."""
    from oracle import oracle
    from paper_2107_07866_b200.potential import write_baseline_table
    path = (tables["baseline"] if rho_k == 2.0 else
            write_baseline_table(str(tmp_path / "steep.eam"), rho_k=rho_k))
    ref = oracle.Sim(path, box=(8, 8, 8), temperature=600.0, seed=5)
    ref.step(1e-3, 3)
    dev = device_for(ref, path)
    assert dev.describe()["fp32_density"] == compressed
    e_ref, e_dev = ref.eval_forces(), dev.eval_forces()
    assert close(e_ref[0], e_dev[0]) and close(e_ref[1], e_dev[1]), (e_ref, e_dev)
    assert_store_parity(ref.store(), dev.download(), what=f"rho_k={rho_k}")


def test_unit_schedule_by_box_size(cuda, tables):
    """Round-robin unit batches (14 units per batch, one batch per CTA and
    round) need several rounds to balance; a box with fewer than two rounds of
    units -- config 2's 50^3 has 1027 units for 148 CTAs -- keeps one contiguous
    unit range per CTA (describe()["unit_rr"] == 0)"""
    from paper_2107_07866_b200 import DeviceStore, EamPotential
    pot = EamPotential.load(tables["baseline"])
    small = DeviceStore((50, 50, 50, 2.855, 3), pot)
    d = small.describe()
    assert d["unit_rr"] == 0, d
    big = DeviceStore((128, 128, 64, 2.855, 3), pot)
    d = big.describe()
    units = (128 * 128 // 32) * (64 // 4)
    assert units >= 2 * 14 * d["sm_count"] and d["unit_rr"] == 14, d


@pytest.mark.parametrize("stencil", ["newton3", "full"])
def test_force_window_gap(cuda, tables, stencil):
    """The force table's shared-memory window skips a stretch of r between two
    neighbour shells (capi.cu force_window_setup; BASELINE lattice: inside
    2.855..4.04 A) and everything below the first shell's margin; pairs there
    fetch their records by texture.  Atoms displaced by up to +-0.55 A per
    component put pairs inside the gap, at both its edges and below the
    window: rho, dF, forces and energies against the oracle"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(8, 7, 6), temperature=0.0, seed=5)
    n = 2 * 8 * 7 * 6
    rng = np.random.default_rng(77)
    ref.displace_interior(rng.uniform(-0.55, 0.55, size=(n, 3)))
    ref.rehash()
    dev = device_for(ref, tables["baseline"], stencil)
    d = dev.describe()
    lo, gap_lo, gap_n, cap = d["force_window"]
    assert gap_lo > lo and gap_n > 0 and cap < 3300, d
    # pairs inside the gap / below the window exist in this configuration
    pot_h = 5.6 / 5000
    s = ref.store()
    m = real_mask(s)
    x = s.pos[m]
    _, a0, _g = ref.box
    L = np.array([8, 7, 6]) * a0
    dd = x[:, None, :] - x[None, :, :]
    dd -= L * np.round(dd / L)
    r = np.sqrt((dd ** 2).sum(-1))[np.triu_indices(len(x), 1)]
    seg = np.floor((r - pot_h) / pot_h).astype(int)
    assert ((seg >= gap_lo) & (seg < gap_lo + gap_n)).sum() > 100
    assert ((seg < lo) & (seg >= 0)).sum() > 10
    e_ref, e_dev = ref.eval_forces(), dev.eval_forces()
    assert close(e_ref[0], e_dev[0]) and close(e_ref[1], e_dev[1]), (e_ref, e_dev)
    assert_store_parity(ref.store(), dev.download(), what=f"window gap {stencil}")


@pytest.mark.parametrize("stencil", ["newton3", "full"])
def test_rows_of_whole_strips(cuda, tables, stencil):
    """Boxes whose rows hold whole 32-cell strips (bx % 32 == 0, as configs 4
    and 5) take the force pass's row accumulation of partner shares and the
    column unit order: a thermal 32 x 5 x 7 box with x and y images, then a
    PKA cascade (off-lattice records, ghost partners), against the oracle"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(32, 5, 7), temperature=600.0, seed=21,
                     pka_energy_kev=0.5, pka_site=(16, 2, 3))
    ref.step(1e-3, 4)
    dev = device_for(ref, tables["baseline"], stencil)
    dev.set_state(ref.state())
    e_ref, e_dev = ref.eval_forces(), dev.eval_forces()
    assert close(e_ref[0], e_dev[0]) and close(e_ref[1], e_dev[1]), (e_ref, e_dev)
    assert_store_parity(ref.store(), dev.download(), what=f"aligned eval {stencil}")
    ref.step(1e-3, 10)
    dev.step(1e-3, 10)
    assert_store_parity(ref.store(), dev.download(), pos_tol=1e-10, rel=1e-9,
                        what=f"aligned thermal {stencil}")
    ref.inject_pka()
    s = ref.store()
    _, a, g = ref.box
    tx, ty = 32 + 2 * g, 5 + 2 * g
    site = ((g + 3) * ty + (g + 2)) * 2 * tx + 2 * (g + 16)
    dev.inject_pka(site, s.vel[site])
    for chunk in range(3):
        ref.step(1e-4, 20)
        dev.step(1e-4, 20)
        assert ref.count_defects() == dev.count_defects(), chunk
        assert_store_parity(ref.store(), dev.download(), pos_tol=1e-8, rel=1e-7,
                            what=f"aligned cascade {stencil} {chunk}")


@pytest.mark.parametrize("stencil", ["newton3", "full"])
def test_skin_pruning_regional_bounds(cuda, tables, stencil):
    """Density-pass skin pruning by regional displacement bounds (bx % 32 ==
    0): a skin shell farther than cutoff + 2U (U the largest displacement of
    any atom from its own site in the neighbouring 32-cell chunks) is skipped.
    The pair sets, rho, dF and forces stay the oracle's: one step from
    identical inputs within 1e-10, then a PKA cascade whose chunks (atoms off
    their sites, slots refilled by update_hash pass 2) lose their bound --
    and the thermal regions still prune most of the skin"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(128, 4, 6), temperature=600.0, seed=33,
                     pka_energy_kev=1.0, pka_site=(40, 2, 3))
    ref.step(1e-3, 6)
    dev = device_for(ref, tables["baseline"], stencil)
    dev.set_state(ref.state())
    # rows of whole 128-cell virtual blocks: the TMA-staged kick/drift sweep too
    desc = dev.describe()
    assert desc["skin_prune"] == 1 and desc["kick_drift_bulk"] == 1, desc
    # after an upload no bound is valid: the first density pass prunes nothing
    dev.skin_stats(True)
    e_ref, e_dev = ref.eval_forces(), dev.eval_forces()
    seen, listed = dev.skin_stats(False)
    assert listed > 0 and seen == listed, (seen, listed)
    assert close(e_ref[0], e_dev[0]) and close(e_ref[1], e_dev[1]), (e_ref, e_dev)
    # one step from identical inputs: the step's own kick/drift publishes the
    # bounds its density pass uses
    dev.skin_stats(True)
    ref.step(1e-3, 1)
    dev.step(1e-3, 1)
    seen, listed = dev.skin_stats(False)
    assert seen < 0.5 * listed, (seen, listed)
    assert_store_parity(ref.store(), dev.download(), pos_tol=1e-12,
                        what=f"pruned step {stencil}")
    ref.step(1e-3, 8)
    dev.step(1e-3, 8)
    assert_store_parity(ref.store(), dev.download(), pos_tol=1e-10, rel=1e-9,
                        what=f"pruned thermal {stencil}")
    ref.inject_pka()
    s = ref.store()
    _, a, g = ref.box
    tx, ty = 128 + 2 * g, 4 + 2 * g
    site = ((g + 3) * ty + (g + 2)) * 2 * tx + 2 * (g + 40)
    dev.inject_pka(site, s.vel[site])
    saw_clash = False
    for chunk in range(4):
        dev.skin_stats(True)
        ref.step(1e-4, 25)
        dev.step(1e-4, 25)
        seen, listed = dev.skin_stats(False)
        assert seen < listed, (chunk, seen, listed)
        rs = ref.store()
        saw_clash |= (rs.clash_ghost == 0).sum() > 0
        assert ref.count_defects() == dev.count_defects(), chunk
        assert_store_parity(rs, dev.download(), pos_tol=1e-8, rel=1e-7,
                            what=f"pruned cascade {stencil} {chunk}")
    assert saw_clash


@pytest.mark.parametrize("shift", [0.0, 0.2, 0.45])
def test_skin_pruning_displaced_atom(cuda, tables, shift):
    """A perfect lattice (every displacement bound ~0, so the skin shells are
    pruned) with one atom moved by `shift` A toward its shell-6 neighbour at
    2 a0 = 5.71 A: at 0.2 A the pair (5.51 A) and, at 0.45 A, a shell-7 pair
    enter the cutoff (5.6 A) and must be found -- the moved atom's own bound
    and its chunk's bound lift the skin threshold for every warp that can
    pair with it; the rest of the box keeps pruning"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(64, 4, 8), temperature=0.0, seed=3)
    dims, a0, g = ref.box
    tx, ty = 64 + 2 * g, 4 + 2 * g
    site = ((g + 3) * ty + (g + 1)) * 2 * tx + 2 * (g + 30)  # corner atom of cell (30, 1, 3)
    s = ref.store()
    ref.set_atom(site, pos=s.pos[site] + np.array([shift, 0.0, 0.0]))
    ref.rehash()
    dev = device_for(ref, tables["baseline"])
    dev.skin_stats(True)
    ref.step(1e-3, 1)
    dev.step(1e-3, 1)
    seen, listed = dev.skin_stats(False)
    assert seen < 0.5 * listed, (seen, listed)
    assert_store_parity(ref.store(), dev.download(), pos_tol=1e-12,
                        what=f"displaced atom {shift}")
    # the shifted atom's partners: pairs beyond the lattice shells were counted
    if shift > 0.0:
        a, b = by_tag(ref.store()), by_tag(dev.download())
        t = int(ref.store().tag[site])
        assert np.abs(a[t][2] - b[t][2]).max() <= 1e-10 * max(1.0, np.abs(a[t][2]).max())


def test_overlap_halts_multi_step_call(cuda, tables):
    """An overlap found in step 2 of a 5-step call (fixed dt: merged kicks and
    deferred StepState sums) ends the call at step 2 like the reference's
    throw from refresh_forces (sim.cpp:225-231, forces.cpp:414-447): same
    message, StepState of the completed step 1 with step = 2, and the store
    as the failing step left it -- positions and velocities of step 2's
    drift, rho of its density pass -- not several drifts further.

    Setup: a 10 keV-class interstitial shot at a lattice atom of a cold 6^3
    box along +x; its offset (0.18497741167859 A) was found by a secant
    search on the oracle so that the pair passes 2.9e-8 A apart exactly at
    step 2 (overlap threshold 1e-6 A, forces.cpp:15).  Deviation by design:
    the device clears the force accumulators in the step's first kernel, so
    the failing step's forces read 0 where the reference keeps step 1's."""
    from oracle import oracle
    from paper_2107_07866_b200._lib import CbxRuntimeError
    ref = oracle.Sim(tables["baseline"], box=(6, 6, 6), temperature=0.0, seed=1)
    _, a, g = ref.box
    site = np.array([(g + 3) * a] * 3)
    ref.insert(site + [0.18497741167859, 0.0, 0.0], 900001, vel=(-1000.0, 0.0, 0.0))
    ref.fill_ghosts()
    ref.refresh_forces()
    dev = device_for(ref, tables["baseline"])
    dev.set_state(ref.state())
    with pytest.raises(RuntimeError) as er:
        ref.step(1e-4, 5)
    with pytest.raises(CbxRuntimeError) as ed:
        dev.step(1e-4, 5)
    assert str(er.value).startswith("step 2: atoms 900001 and ")
    assert str(ed.value) == str(er.value)
    sr, sd = ref.state(), dev.state()
    assert sd["step"] == sr["step"] == 2
    assert sd["t"] == sr["t"]
    assert close(sd["kinetic"], sr["kinetic"], 1e-12)
    rs, ds = ref.store(), dev.download()
    assert structure(rs) == structure(ds)
    a_, b_ = by_tag(rs), by_tag(ds)
    for t, (pa, va, fa, ra, da) in a_.items():
        pb, vb, fb, rb, db = b_[t]
        assert np.abs(pa - pb).max() <= 1e-12, t
        assert np.abs(va - vb).max() <= 1e-9 * max(1.0, np.abs(va).max()), t
        assert abs(ra - rb) <= REL * max(abs(ra), 1e-300), t


def test_adaptive_dt_matches(cuda, tables):
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(6, 6, 6), temperature=600.0, seed=3)
    dev = device_for(ref, tables["baseline"])
    dev.set_state(ref.state())
    ref.step(-1, 5)
    st = dev.step(-1, 5)
    assert st["dt"] == ref.state()["dt"]
    assert abs(st["t"] - ref.state()["t"]) <= 1e-15


def test_deferred_finalize_state(cuda, tables):
    """With a fixed dt the StepState sums of a step run inside the next
    step's first kernel (or before the host reads the status): one call of
    n steps and n calls of one step give identical StepStates, equal to the
    oracle's, and a measure right after a multi-step call sees the final
    state"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(7, 6, 5), temperature=600.0, seed=17)
    a = device_for(ref, tables["baseline"])
    b = device_for(ref, tables["baseline"])
    a.set_state(ref.state())
    b.set_state(ref.state())
    sa = a.step(1e-3, 6)
    for _ in range(6):
        sb = b.step(1e-3, 1)
    ref.step(1e-3, 6)
    r = ref.state()
    # (partner contributions are atomic adds: sums agree to rounding, not bitwise)
    assert sa["step"] == sb["step"] == r["step"] and sa["t"] == sb["t"] == r["t"]
    for k in ("kinetic", "pair", "embedding", "max_speed"):
        assert close(sa[k], sb[k], 1e-12) and close(sa[k], r[k]), k
    assert a.state() == sa


def test_simulation_facade(cuda, tables):
    """Simulation (sim.h) over the device equals the oracle's constructor"""
    from oracle import oracle
    from paper_2107_07866_b200 import SimConfig, Simulation
    cfg = SimConfig(box_x=6, box_y=6, box_z=6, temperature=600.0, seed=99,
                    potential_path=tables["baseline"])
    sim = Simulation(cfg)
    ref = oracle.Sim(tables["baseline"], box=(6, 6, 6), temperature=600.0, seed=99)
    a, b = ref.state(), sim.state
    for k in ("kinetic", "pair", "embedding", "max_speed"):
        assert close(a[k], b[k], 1e-12), k
    assert sim.atom_count() == 432
    assert np.abs(sim.total_momentum()).max() < 1e-8


def test_near_cutoff_pairs_exact(cuda, tables):
    """pairs placed within 1e-12 A of the cutoff on both sides: the fp32
    filter must hand them to the exact test (in-cutoff set bit-identical)"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(5, 5, 5), init_lattice=False)
    _, a, g = ref.box
    base = np.array([4.0 * a, 4.0 * a, 4.0 * a])
    rc = 5.6
    tag = 0
    for k, dr in enumerate([-1e-12, -1e-14, 0.0, 1e-14, 1e-12, 1e-9]):
        p0 = base + np.array([0.0, 0.37 * a * (k % 3), 0.41 * a * (k // 3)])
        ref.insert(p0, tag)
        ref.insert(p0 + np.array([rc + dr, 0.0, 0.0]), tag + 1)
        tag += 2
    ref.fill_ghosts()
    for stencil in ("newton3", "full", "reference"):
        r2 = oracle.Sim(tables["baseline"], box=(5, 5, 5), init_lattice=False)
        s = ref.store()
        dev = device_for(ref, tables["baseline"], stencil)
        e_ref = ref.eval_forces()
        e_dev = dev.eval_forces()
        assert close(e_ref[1], e_dev[1], 1e-12), (stencil, e_ref, e_dev)
        a_, b_ = by_tag(ref.store()), by_tag(dev.download())
        for t in a_:
            assert (a_[t][3] == 0.0) == (b_[t][3] == 0.0), (stencil, t)
            assert close(a_[t][3], b_[t][3]), (stencil, t)


def test_bench_steps_timed_graph(cuda, tables):
    """the benchmark loop (timed graph with event nodes, L2 flush) advances
    the same trajectory as plain steps"""
    import ctypes as C
    from oracle import oracle
    from paper_2107_07866_b200 import _lib
    ref = oracle.Sim(tables["baseline"], box=(8, 8, 8), temperature=600.0, seed=5)
    dev = device_for(ref, tables["baseline"])
    dev.set_state(ref.state())
    out = (C.c_double * 8)()
    _lib.check(dev.lib.cbx_bench_steps(dev.h, 1e-3, 6, 64.0, out), dev.h)
    assert out[6] == 6 and out[5] > 0 and out[7] > 0 and out[5] > out[7]
    _lib.check(dev.lib.cbx_bench_phases(dev.h, 1), dev.h)
    _lib.check(dev.lib.cbx_bench_steps(dev.h, 1e-3, 4, 64.0, out), dev.h)
    ref.step(1e-3, 10)
    assert out[6] == 4 and out[5] > 0 and out[2] > 0 and out[0] > 0
    assert dev.state()["step"] == ref.state()["step"]
    assert_store_parity(ref.store(), dev.download(), pos_tol=1e-9, rel=1e-8)


def test_cxx_host_on_device(cuda, tables, tmp_path):
    """the C++ mirror drives a device run (Simulation ctor + 10 steps)"""
    import os
    import subprocess
    from paper_2107_07866_b200 import _lib
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "cxx_host")
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(root, "include"),
                    os.path.join(root, "examples", "cxx_host.cpp"), "-L", libdir,
                    "-l:libcascade_b200.so", f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    out = subprocess.run([exe, tables["baseline"], "gpu"], capture_output=True, text=True,
                         check=True).stdout
    assert "atoms 1024" in out and "-> step 10" in out


def test_two_contexts_interleaved(cuda, tables):
    """two engines with different boxes on one GPU, used alternately: each
    re-binds its own stencil tables (the __constant__ copy is per device)"""
    from oracle import oracle
    r1 = oracle.Sim(tables["baseline"], box=(6, 7, 8), temperature=600.0, seed=1)
    r2 = oracle.Sim(tables["baseline"], box=(9, 6, 5), temperature=600.0, seed=2)
    d1 = device_for(r1, tables["baseline"])
    d2 = device_for(r2, tables["baseline"])
    for ref, dev in ((r1, d1), (r2, d2), (r1, d1), (r2, d2)):
        dev.set_state(ref.state())
    for _ in range(2):
        for ref, dev in ((r1, d1), (r2, d2)):
            ref.step(1e-3, 5)
            dev.step(1e-3, 5)
            assert_store_parity(ref.store(), dev.download(), pos_tol=1e-10, rel=1e-9)
