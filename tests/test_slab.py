"""z-slab decomposition.

GPU: n virtual slab ranks on one device, exchanging through device buffers
(LocalExchange), against the single-box oracle -- forces, densities,
energies, trajectories and a cascade whose PKA crosses slab boundaries.
CPU: the torch.distributed exchange (gloo, world_size 2 and 3) routes every
buffer to the right neighbour and reduces the energies like the local one.
"""
import os
import socket

import numpy as np
import pytest

from helpers import assert_store_parity
from paper_2107_07866_b200 import _lib
from paper_2107_07866_b200 import slab as S


# ------------------------------------------------------------- host logic
def test_slab_bounds_cover_box():
    for bz in (5, 10, 17, 64):
        for n in (1, 2, 3, 4):
            b = [S.slab_bounds(bz, r, n) for r in range(n)]
            assert b[0][0] == 0 and b[-1][1] == bz
            assert all(b[i][1] == b[i + 1][0] for i in range(n - 1))


def test_reduce_states():
    a = np.array([1.0, 2.0, 3.0, 4.0, 1, 0, 7, 0.5])
    b = np.array([10.0, 20.0, 30.0, 2.0, 2, 3, 7, 0.5])
    r = S.reduce_states([a, b])
    assert list(r[:3]) == [11.0, 22.0, 33.0]
    assert r[3] == 4.0 and r[4] == 3 and r[5] == 3 and r[6] == 7 and r[7] == 0.5


class MockRank:
    """stands in for a SlabRank: packets encode (sender, kind, direction)"""

    def __init__(self, rank, nranks):
        import torch
        self.torch = torch
        self.rank, self.nranks = rank, nranks
        self.got = {}
        self.comm_device = "cpu"

    def pack(self, kind, direction):
        n = 16 + 8 * kind + (3 if direction > 0 else 0)  # distinct ragged sizes
        t = self.torch.full((64,), 0, dtype=self.torch.uint8)
        t[0], t[1], t[2] = self.rank, kind, 1 if direction > 0 else 0
        t[3:n] = 200
        return t, n

    def unpack(self, kind, source, tensor, nbytes):
        a = tensor[:nbytes].numpy().copy()
        self.got[(kind, source)] = (int(a[0]), int(a[1]), int(a[2]), nbytes)

    def local_state(self):
        return np.array([1.0 + self.rank, 2.0, 3.0, 0.5 * self.rank, 1, 0, 4, 0.25])


def _expect(rank, n):
    lo, hi = S.neighbours(rank, n)
    out = {}
    for kind in range(5):
        out[(kind, -1)] = (lo, kind, 1, 16 + 8 * kind + 3)   # the rank below's "up" packet
        out[(kind, +1)] = (hi, kind, 0, 16 + 8 * kind)       # the rank above's "down" packet
    return out


def _gloo_worker(rank, n, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=n)
    try:
        r = MockRank(rank, n)
        ex = S.DistExchange(r)
        for kind in range(5):
            ex.exchange(kind)
        red = ex.allreduce([r.local_state()])
        q.put((rank, r.got, list(red)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n", [2, 3])
def test_dist_exchange_gloo(n):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, n, port, q)) for r in range(n)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(n):
        rank, got, red = q.get(timeout=120)
        res[rank] = (got, red)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    local = S.reduce_states([MockRank(r, n).local_state() for r in range(n)])
    for r in range(n):
        got, red = res[r]
        assert got == _expect(r, n), r
        assert np.allclose(red[:6], local[:6])


def test_local_exchange_routing():
    n = 3
    ranks = [MockRank(r, n) for r in range(n)]
    ex = S.LocalExchange(ranks)
    for kind in range(5):
        ex.exchange(kind)
    for r in range(n):
        assert ranks[r].got == _expect(r, n)


# ------------------------------------------------------------- on the GPU
@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2107_07866_b200 import _lib
    _lib.load()
    return True


def _interior(s):
    """drop ghost clash replicas so slab and single-box stores compare"""
    import dataclasses
    keep = s.clash_ghost == 0
    d = {f.name: getattr(s, f.name) for f in dataclasses.fields(s)}
    for k in list(d):
        if k.startswith("clash_"):
            d[k] = d[k][keep]
    return type(s)(**d)


def slab_domain(ref, path, n):
    from paper_2107_07866_b200 import EamPotential
    dims, a0, g = ref.box
    pot = EamPotential.load(path)
    ranks = [S.SlabRank((*dims, a0, g), pot, r, n) for r in range(n)]
    st = ref.state()
    for r in ranks:
        r.upload_global(ref.store())
        r.set_state(st)
    dom = S.SlabDomain(ranks, S.LocalExchange(ranks))
    dom._pot = pot
    return dom


def gather(dom, ref):
    """the slabs' interiors assembled into one global store"""
    s = _interior(ref.store())
    Sg = len(s.tag)
    g = dict(pos=np.zeros((Sg, 3)), vel=np.zeros((Sg, 3)), force=np.zeros((Sg, 3)),
             rho=np.zeros(Sg), df=np.zeros(Sg), tag=np.zeros(Sg, np.uint64),
             valid=np.zeros(Sg, np.uint8), ghost=np.zeros(Sg, np.uint8))
    cap = 4096
    g.update(clash_key=np.zeros(cap, np.int64), clash_idx=np.zeros(cap, np.int32),
             clash_pos=np.zeros((cap, 3)), clash_vel=np.zeros((cap, 3)),
             clash_force=np.zeros((cap, 3)), clash_rho=np.zeros(cap), clash_df=np.zeros(cap),
             clash_tag=np.zeros(cap, np.uint64), clash_ghost=np.zeros(cap, np.uint8))
    n = 0
    for r in dom.ranks:
        n = r.download_global(g, n)
    for k in list(g):
        if k.startswith("clash_"):
            g[k] = g[k][:n]
    return type(s)(**g)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 3, 4])
def test_slab_eval_matches_single_box(cuda, tables, n):
    """forces / rho / dF / energies of the decomposed evaluation equal the
    single-box reference (oracle) on a thermalised lattice"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(8, 7, 13), temperature=600.0, seed=77)
    dom = slab_domain(ref, tables["baseline"], n)
    dom.prime()
    sr, sd = ref.state(), dom.state()
    for k in ("kinetic", "pair", "embedding"):
        assert abs(sd[k] - sr[k]) <= 1e-10 * abs(sr[k]), (k, sd[k], sr[k])
    assert_store_parity(_interior(ref.store()), gather(dom, ref), what=f"slab eval n={n}")


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 3])
def test_slab_trajectory(cuda, tables, n):
    """60 steps at 600 K: trajectories of the decomposed run follow the
    single-box oracle (atoms migrate between slabs through the z faces)"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(8, 8, 9), temperature=600.0, seed=12345)
    dom = slab_domain(ref, tables["baseline"], n)
    dom.prime()
    for chunk in range(3):
        ref.step(1e-3, 20)
        dom.step(1e-3, 20)
        sr, sd = ref.state(), dom.state()
        assert sd["step"] == sr["step"]
        for k in ("kinetic", "pair", "embedding"):
            assert abs(sd[k] - sr[k]) <= 1e-9 * abs(sr[k]), (chunk, k, sd[k], sr[k])
        assert_store_parity(_interior(ref.store()), gather(dom, ref), pos_tol=1e-9, rel=1e-8,
                            what=f"slab n={n} chunk {chunk}")


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 3])
def test_slab_cascade(cuda, tables, n):
    """a PKA cascade whose recoils cross slab faces: off-lattice atoms move
    between ranks as clash records; Wigner-Seitz counts, bucket structure and
    forces match the single-box oracle; adaptive dt is agreed globally"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(10, 10, 10), temperature=600.0, seed=12345,
                     pka_energy_kev=1.0, pka_site=(5, 5, 3))
    ref.step(1e-3, 5)
    ref.inject_pka()
    dom = slab_domain(ref, tables["baseline"], n)
    dom.prime()
    assert abs(dom.state()["kinetic"] - ref.state()["kinetic"]) <= 1e-12 * ref.state()["kinetic"]
    saw_clash = False
    for chunk in range(6):
        ref.step(-1, 20)
        dom.step(-1, 20)
        rs = ref.store()
        saw_clash |= (rs.clash_ghost == 0).sum() > 0
        assert dom.state()["t"] == pytest.approx(ref.state()["t"], rel=1e-12, abs=0)
        assert ref.count_defects() == dom.count_defects(), chunk
        assert_store_parity(_interior(rs), gather(dom, ref), pos_tol=1e-8, rel=1e-7,
                            what=f"slab cascade n={n} chunk {chunk}")
    assert saw_clash


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 3])
def test_slab_init_bcc_matches_single_box(cuda, tables, n):
    """init_bcc on slab ranks keeps each slab's planes of the global lattice:
    the same RNG stream and momentum removal as the single box"""
    from oracle import oracle
    from paper_2107_07866_b200 import EamPotential
    ref = oracle.Sim(tables["baseline"], box=(7, 6, 9), temperature=600.0, seed=4242)
    dims, a0, g = ref.box
    pot = EamPotential.load(tables["baseline"])
    ranks = [S.SlabRank((*dims, a0, g), pot, r, n) for r in range(n)]
    tot = sum(r.init_bcc(600.0, 4242) for r in ranks)
    assert tot == 2 * 7 * 6 * 9
    dom = S.SlabDomain(ranks, S.LocalExchange(ranks))
    a, b = _interior(ref.store()), gather(dom, ref)
    m = a.valid.astype(bool) & ~a.ghost.astype(bool)
    mb = b.valid.astype(bool) & ~b.ghost.astype(bool)
    assert np.array_equal(m, mb)
    assert np.array_equal(a.pos[m], b.pos[m])
    assert np.array_equal(a.vel[m], b.vel[m])
    assert np.array_equal(a.tag[m], b.tag[m])


def native_rank(ref, path, transport):
    """one slab rank that owns the whole box, exchanging with itself inside
    its step graph (the n == 1 case of the multi-GPU path): NCCL self
    send/recv, or the peer-memory kernels mapped onto the rank itself"""
    from paper_2107_07866_b200 import EamPotential
    dims, a0, g = ref.box
    r = S.SlabRank((*dims, a0, g), EamPotential.load(path), 0, 1)
    r.connect("p2p" if transport.startswith("p2p") else transport)
    if transport.startswith("p2p"):
        # the reverse halos as staged exchanges (default) or fused into the
        # passes (peer atomics into the neighbours' accumulators)
        assert not r.fused
        if transport == "p2p-fused":
            _lib.check(r.lib.cbx_slab_p2p_set_fused(r.h, 1), r.h)
            assert r.lib.cbx_slab_p2p_fused(r.h)
    r.upload_global(ref.store())
    r.set_state(ref.state())
    return r


@pytest.mark.gpu
def test_slab_local_exchange_single_rank(cuda, tables):
    """the phase-driven path with one rank: halos are its own periodic images"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(8, 8, 8), temperature=600.0, seed=5)
    dom = slab_domain(ref, tables["baseline"], 1)
    dom.prime()
    ref.step(1e-3, 10)
    dom.step(1e-3, 10)
    assert_store_parity(_interior(ref.store()), gather(dom, ref), pos_tol=1e-10, rel=1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["p2p", "p2p-fused", "nccl"])
def test_slab_graph_eval_and_trajectory(cuda, tables, transport):
    """exchanges captured in the step graph (NCCL self send/recv, or the
    flag-synchronised peer-memory kernels): forces, energies and a 60-step
    trajectory equal the single-box oracle"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(8, 7, 9), temperature=600.0, seed=12345)
    r = native_rank(ref, tables["baseline"], transport)
    e_emb, e_pair = r.eval_forces()
    r.measure()
    sr = ref.state()
    assert abs(e_pair - sr["pair"]) <= 1e-10 * abs(sr["pair"])
    assert abs(e_emb - sr["embedding"]) <= 1e-10 * abs(sr["embedding"])
    assert abs(r.state()["kinetic"] - sr["kinetic"]) <= 1e-12 * sr["kinetic"]
    dom = S.SlabDomain([r], None)
    assert_store_parity(_interior(ref.store()), gather(dom, ref), what="nccl eval")
    launches0 = r.kernel_launches()
    for chunk in range(3):
        ref.step(1e-3, 20)
        st = r.step(1e-3, 20)
        sr = ref.state()
        assert st["step"] == sr["step"]
        for k in ("kinetic", "pair", "embedding"):
            assert abs(st[k] - sr[k]) <= 1e-9 * abs(sr[k]), (chunk, k, st[k], sr[k])
        assert_store_parity(_interior(ref.store()), gather(dom, ref), pos_tol=1e-9, rel=1e-8,
                            what=f"nccl chunk {chunk}")
    assert r.kernel_launches() > launches0


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["p2p", "p2p-fused", "nccl"])
def test_slab_graph_cascade(cuda, tables, transport):
    """cascade with adaptive dt through the NCCL step graph: clash records,
    defect counts and the global-max-speed time step match the oracle"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(10, 10, 10), temperature=600.0, seed=12345,
                     pka_energy_kev=1.0, pka_site=(5, 5, 3))
    ref.step(1e-3, 5)
    ref.inject_pka()
    r = native_rank(ref, tables["baseline"], transport)
    r.eval_forces()
    r.measure()
    dom = S.SlabDomain([r], None)
    saw_clash = False
    for chunk in range(6):
        ref.step(-1, 20)
        r.step(-1, 20)
        rs = ref.store()
        saw_clash |= (rs.clash_ghost == 0).sum() > 0
        assert r.state()["t"] == pytest.approx(ref.state()["t"], rel=1e-12, abs=0)
        assert ref.count_defects() == r.count_defects(), chunk
        assert_store_parity(_interior(rs), gather(dom, ref), pos_tol=1e-8, rel=1e-7,
                            what=f"nccl cascade chunk {chunk}")
    assert saw_clash


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 3])
def test_slab_whole_rows_bulk_and_pruning(cuda, tables, n):
    """slab ranks whose rows hold whole 128-cell virtual blocks (as config 5
    per GPU): the TMA-staged kick/drift sweep and the density pass's skin
    pruning run on every rank (z halos from the neighbours keep their chunks
    unbounded); a PKA cascade crossing the slab faces at fixed dt matches the
    single-box oracle"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(128, 4, 12), temperature=600.0, seed=99,
                     pka_energy_kev=0.5, pka_site=(64, 2, 6 if n == 2 else 4))
    ref.step(1e-3, 5)
    ref.inject_pka()
    dom = slab_domain(ref, tables["baseline"], n)
    for r in dom.ranks:
        d = r.describe()
        assert d["kick_drift_bulk"] == 1 and d["skin_prune"] == 1, d
    dom.prime()
    saw_clash = False
    for chunk in range(4):
        ref.step(1e-4, 15)
        dom.step(1e-4, 15)
        rs = ref.store()
        saw_clash |= (rs.clash_ghost == 0).sum() > 0
        assert ref.count_defects() == dom.count_defects(), chunk
        assert_store_parity(_interior(rs), gather(dom, ref), pos_tol=1e-8, rel=1e-7,
                            what=f"slab rows n={n} chunk {chunk}")
    assert saw_clash


@pytest.mark.gpu
def test_slab_graph_whole_rows_p2p(cuda, tables):
    """the in-graph peer-memory step (merged kick on a slab rank) with the
    TMA-staged kick/drift and skin pruning: 40 steps against the oracle"""
    from oracle import oracle
    ref = oracle.Sim(tables["baseline"], box=(128, 4, 8), temperature=600.0, seed=7)
    r = native_rank(ref, tables["baseline"], "p2p")
    assert r.describe()["kick_drift_bulk"] == 1
    r.eval_forces()
    r.measure()
    dom = S.SlabDomain([r], None)
    for chunk in range(2):
        ref.step(1e-3, 20)
        st = r.step(1e-3, 20)
        sr = ref.state()
        for k in ("kinetic", "pair", "embedding"):
            assert abs(st[k] - sr[k]) <= 1e-9 * abs(sr[k]), (chunk, k, st[k], sr[k])
        assert_store_parity(_interior(ref.store()), gather(dom, ref), pos_tol=1e-9, rel=1e-8,
                            what=f"p2p rows chunk {chunk}")


# ------------------------------------------ two processes, peer memory
def _p2p_lockstep_worker(rank, n, port, table, q):
    """one slab rank per process, both on GPU 0: CUDA IPC mappings of the
    neighbour's receive region, the peer-memory pack/flag/unpack kernels in
    lockstep (P2PLockstep), the StepState reduction over gloo"""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=n)
    try:
        from oracle import oracle
        from paper_2107_07866_b200 import EamPotential
        ref = oracle.Sim(table, box=(8, 7, 10), temperature=600.0, seed=777,
                         pka_energy_kev=0.5, pka_site=(4, 3, 5))
        ref.step(1e-3, 3)
        ref.inject_pka()  # at the slab face: recoils migrate between the processes
        dims, a0, g = ref.box
        r = S.SlabRank((*dims, a0, g), EamPotential.load(table), rank, n, device=0)
        r.connect("p2p")
        assert r.transport == "p2p" and not r.fused  # one device: staged reverse halos
        r.upload_global(ref.store())
        r.set_state(ref.state())
        dom = S.SlabDomain([r], S.P2PLockstep(r))
        dom.prime()
        out = []
        for chunk in range(3):
            dom.step(1e-4, 10)
            s = _interior(ref.store())
            Sg = len(s.tag)
            gd = dict(pos=np.zeros((Sg, 3)), vel=np.zeros((Sg, 3)), force=np.zeros((Sg, 3)),
                      rho=np.zeros(Sg), df=np.zeros(Sg), tag=np.zeros(Sg, np.uint64),
                      valid=np.zeros(Sg, np.uint8), ghost=np.zeros(Sg, np.uint8))
            cap = 4096
            gd.update(clash_key=np.zeros(cap, np.int64), clash_idx=np.zeros(cap, np.int32),
                      clash_pos=np.zeros((cap, 3)), clash_vel=np.zeros((cap, 3)),
                      clash_force=np.zeros((cap, 3)), clash_rho=np.zeros(cap),
                      clash_df=np.zeros(cap), clash_tag=np.zeros(cap, np.uint64),
                      clash_ghost=np.zeros(cap, np.uint8))
            nc = r.download_global(gd, 0)
            for k in list(gd):
                if k.startswith("clash_"):
                    gd[k] = gd[k][:nc]
            parts = [None] * n
            dist.all_gather_object(parts, gd)
            st = dom.state()
            out.append((chunk, st, r.count_defects() if rank == 0 else None))
            if rank == 0:
                ref.step(1e-4, 10)
                merged = {k: (np.concatenate([p[k] for p in parts]) if k.startswith("clash_")
                              else sum(p[k] for p in parts)) for k in parts[0]}
                got = type(s)(**merged)
                sr = ref.state()
                for k in ("kinetic", "pair", "embedding"):
                    assert abs(st[k] - sr[k]) <= 1e-9 * abs(sr[k]), (chunk, k, st[k], sr[k])
                assert_store_parity(_interior(ref.store()), got, pos_tol=1e-8, rel=1e-7,
                                    what=f"two-process p2p chunk {chunk}")
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001 -- reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_slab_p2p_two_processes_lockstep(cuda, tables):
    """the peer-memory transport between two PROCESSES (CUDA IPC handles
    exchanged over torch.distributed, packets and flags stored into the other
    process's memory, clash records and migrants crossing), two z slabs of an
    8 x 7 x 10 box with a 0.5 keV PKA at the slab face, 30 steps against the
    single-box oracle.  Both ranks share GPU 0, so the exchange runs in
    lockstep (send, barrier, receive): no kernel waits on the other process's
    kernels (ranks spinning on each other on one GPU raise Xid 109)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_lockstep_worker, args=(r, 2, port, tables["baseline"], q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        rank, msg = q.get(timeout=600)
        res[rank] = msg
    for p in procs:
        p.join(timeout=120)
    assert res == {0: "ok", 1: "ok"}, res
    assert all(p.exitcode == 0 for p in procs)
