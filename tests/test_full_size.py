"""Parity and size-independent properties at the BASELINE configurations'
full sizes: config 2 (250k atoms) and config 3 (2M atoms)
against the oracle on identical inputs; config 4 (16M atoms, one GPU)
through its perfect-lattice known answers and exact pair counts; a config-3
cascade through momentum conservation and Newton-3 antisymmetry.
"""
import numpy as np
import pytest

from helpers import assert_store_parity, real_mask

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2107_07866_b200 import _lib
    _lib.load()
    return True


def oracle_state(path, w):
    """the workload's initial state in the oracle (bench.py's reference arm)"""
    from oracle import oracle
    from paper_2107_07866_b200.workloads import displacements
    s = oracle.Sim(path, box=w.cells, temperature=w.temperature, seed=w.seed)
    if w.displacement > 0:
        s.displace_interior(displacements(w, w.atoms))
        s.rehash()
        s.refresh_forces()
    return s


def device_for(sim, path):
    from paper_2107_07866_b200 import DeviceStore, EamPotential
    dims, a0, g = sim.box
    dev = DeviceStore((*dims, a0, g), EamPotential.load(path))
    dev.upload(sim.store())
    dev.set_state(sim.state())
    return dev


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_full_size_forces_and_step(cuda, tables, cfg):
    """forces, densities, dF and energies of the full configuration equal the
    oracle's (1e-10), and so does one velocity-Verlet step"""
    from paper_2107_07866_b200.workloads import CONFIGS
    w = CONFIGS[cfg]
    ref = oracle_state(tables["baseline"], w)
    dev = device_for(ref, tables["baseline"])
    e_ref = ref.eval_forces()
    e_dev = dev.eval_forces()
    # totals: the oracle adds ~29 N pair terms into one running sum, whose
    # rounding alone reaches ~4e-10 relative at 2M atoms on the perfect
    # lattice (identical terms round the same way); the device sums a tree
    # of partials.  Bound: 1e-10 plus the serial-sum bound n u (u = 2^-53).
    n_terms = 30 * w.atoms
    tol = 1e-10 + n_terms * 2.0 ** -53
    for a, b in zip(e_ref, e_dev):
        assert abs(a - b) <= tol * abs(a), (a, b)
    # per-atom quantities: the north-star 1e-10
    assert_store_parity(ref.store(), dev.download(), what=f"{cfg} eval")
    ref.step(w.dt, 1)
    dev.step(w.dt, 1)
    sr, sd = ref.state(), dev.state()
    for k in ("kinetic", "pair", "embedding"):
        assert abs(sd[k] - sr[k]) <= tol * abs(sr[k]), k
    assert_store_parity(ref.store(), dev.download(), pos_tol=1e-12, rel=1e-10,
                        what=f"{cfg} step")


def test_config4_perfect_lattice_known_answers(cuda, tables):
    """16M atoms at T = 0 (BASELINE table, rho_max = 40): every atom has the
    SURVEY §8(c) known answers, zero force, and exactly 56 candidates / 29
    in-cutoff pairs per atom"""
    from paper_2107_07866_b200 import DeviceStore, EamPotential, SimConfig, make_box
    pot = EamPotential.load(tables["baseline40"])
    box, _ = make_box(SimConfig(box_x=200, box_y=200, box_z=200), pot)
    dev = DeviceStore(box, pot)
    n = dev.init_bcc(0.0, 12345)
    assert n == 16_000_000
    cand, pairs = dev.count_pairs()
    assert cand == 56 * n and pairs == 29 * n
    emb, pair = dev.eval_forces()
    assert abs(emb / n + 3.4365052179757) < 1e-10
    assert abs(pair / n + 3.6755476296970) < 1e-10
    s = dev.download()
    m = real_mask(s)
    assert m.sum() == n
    assert np.abs(s.rho[m] - 11.80956811317917).max() < 1e-11
    assert np.abs(s.df[m] + 0.145496650894856).max() < 1e-12
    assert np.abs(s.force[m]).max() < 1e-11


def test_config3_cascade_conservation(cuda, tables):
    """10 keV PKA in the 2M-atom box, 100 adaptive steps: Newton-3 pair forces
    cancel (total force ~ 0) and the total momentum is conserved"""
    from paper_2107_07866_b200 import PkaSpec, SimConfig, Simulation
    cfg = SimConfig(box_x=100, box_y=100, box_z=100, temperature=600.0, seed=12345,
                    potential_path=tables["baseline"],
                    pka=PkaSpec(site=(50, 50, 50), energy_kev=10.0))
    sim = Simulation(cfg)
    sim.inject_pka()
    p0 = sim.total_momentum()
    st = sim.step(None, 100)
    assert st["step"] == 100 and st["dt"] < 1e-3  # the adaptive dt followed the PKA
    s = sim.store()
    m = real_mask(s)
    ftot = s.force[m].sum(axis=0) + s.clash_force[s.clash_ghost == 0].sum(axis=0)
    fmax = np.abs(s.force[m]).max()
    assert np.abs(ftot).max() <= 1e-9 * fmax * m.sum() ** 0.5
    p1 = sim.total_momentum()
    pka_p = np.abs(p0).max()
    assert np.abs(p1 - p0).max() <= 1e-9 * max(pka_p, 1.0)
    vac, inter, fp = sim.count_defects()
    assert fp >= 0 and vac >= 0 and inter >= 0
