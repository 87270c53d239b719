"""Multi-GPU z-slab domain decomposition of the EAM step.

The reference has one process and periodic ghost replication (store.cpp:
120-195); the paper decomposes space over MPI ranks.  Here rank r of n owns
the global interior z planes [r*bz/n, (r+1)*bz/n) (cbx_create_slab), keeps
g = ghost_width halo planes on each side and stays in the global frame for
positions, hashes and keys, so the decomposed run visits exactly the pairs of
the single-box reference.  One MD step (sim.cpp:248-273) is driven phase by
phase with five neighbour exchanges:

    phase 0  kick, drift, wrap, hash        -> MIGRANTS  (update_hash across slabs)
    phase 1  rehash, x/y ghosts             -> POS       (fill_ghosts in z)
    phase 2  clash images, density          -> RHO       (fold_rho, reverse)
    phase 3  embedding                      -> DF        (refresh_ghosts)
    phase 4  force                          -> FRC       (fold_force, reverse)
    phase 5  second kick, local sums        -> all-reduce of energies / KE / v_max

Exchanges are point-to-point with the z-neighbours (ring of n): NCCL over
NVLink/NVSwitch through torch.distributed in a multi-process run
(`DistExchange`), or device-to-device within one process for virtual ranks
on one GPU (`LocalExchange`, used to validate the decomposition against the
single-box run when only one GPU is available).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import check
from .engine import DeviceStore

MIGRANTS, POS, RHO, DF, FRC = 0, 1, 2, 3, 4
KIND_NAMES = {MIGRANTS: "migrants", POS: "pos", RHO: "rho", DF: "df", FRC: "frc"}


def slab_bounds(bz: int, rank: int, nranks: int):
    """[z0, z1) interior z planes of `rank` (the split cbx_create_slab uses)"""
    return rank * bz // nranks, (rank + 1) * bz // nranks


def neighbours(rank: int, nranks: int):
    """(rank below, rank above) on the periodic ring"""
    return (rank - 1) % nranks, (rank + 1) % nranks


class SlabRank(DeviceStore):
    """One z slab resident on one GPU (a cbx_ctx made by cbx_create_slab).

    Two ways to drive it: phase by phase with host-side exchanges
    (`SlabDomain` + `LocalExchange` / `DistExchange`), or -- the production
    path -- `init_comm` once, after which `step`, `eval_forces`, `measure` and
    the bench run the decomposed step as one CUDA graph per rank with the
    NCCL exchanges inside it."""

    def __init__(self, gbox, potential, rank: int, nranks: int, device: int = 0,
                 stencil: str = "newton3"):
        lib = _lib.load()
        self.lib = lib
        self.potential = potential
        self.rank, self.nranks, self.device = rank, nranks, device
        self.gbox = gbox if isinstance(gbox, _lib.Box) else _lib.Box(*gbox)
        self.box = self.gbox
        h = C.c_void_p()
        check(lib.cbx_create_slab(C.byref(self.gbox), potential.handle, None, rank, nranks,
                                  device, C.byref(h)))
        self.h = h
        self.n_slots = lib.cbx_slot_count(h)
        info = (C.c_long * 8)()
        check(lib.cbx_slab_info(h, info), h)
        self.info = tuple(info)
        self._buf = None
        if stencil != "newton3":
            self.set_stencil(stencil)

    @property
    def comm_device(self):
        import torch
        return torch.device("cuda", self.device)

    @property
    def buf(self):
        """two device send buffers per exchange kind (toward below / above)"""
        if self._buf is None:
            import torch
            self._buf = {}
            for k in KIND_NAMES:
                nb = self.lib.cbx_slab_buffer_bytes(self.h, k)
                self._buf[k] = (torch.empty(nb, dtype=torch.uint8, device=self.comm_device),
                                torch.empty(nb, dtype=torch.uint8, device=self.comm_device))
        return self._buf

    @staticmethod
    def nccl_unique_id() -> bytes:
        # torch first: its libnccl.so.2 (newer) must be the one the process maps;
        # the library dlopens by soname and then shares it
        import torch  # noqa: F401
        b = C.create_string_buffer(128)
        check(_lib.load().cbx_nccl_unique_id(b, 128))
        return b.raw

    def init_comm(self, uid: bytes):
        """collective: every rank of the decomposition passes rank 0's id"""
        import torch  # noqa: F401  (see nccl_unique_id)
        b = C.create_string_buffer(uid, 128)
        self._check(self.lib.cbx_slab_comm_init(self.h, b, 128))

    P2P_HANDLE_BYTES = 256  # CBX_P2P_HANDLE_BYTES

    def p2p_handle(self) -> bytes:
        """this rank's peer-memory handle: CUDA IPC handles of its receive
        region and of its rho / force accumulators, plus its slab geometry"""
        n = self.P2P_HANDLE_BYTES
        b = C.create_string_buffer(n)
        self._check(self.lib.cbx_slab_p2p_handle(self.h, b, n))
        return b.raw

    def init_p2p(self, handles):
        """handles: every rank's p2p_handle, in rank order"""
        blob = b"".join(handles)
        b = C.create_string_buffer(blob, len(blob))
        self._check(self.lib.cbx_slab_p2p_init(self.h, b, len(blob)))

    def connect(self, transport: str = "p2p", group=None):
        """set up the in-graph exchange with the other ranks of a
        torch.distributed job (one rank per process and GPU); with one rank
        the slab exchanges with itself"""
        world = 1
        if self.nranks > 1:
            import torch.distributed as dist
            world = dist.get_world_size(group)
            if world != self.nranks:
                raise ValueError("slab nranks does not match the process group")
        if transport == "p2p":
            h = [self.p2p_handle()]
            if world > 1:
                import torch.distributed as dist
                allh = [None] * world
                dist.all_gather_object(allh, h[0], group=group)
                h = allh
            ok, err = True, ""
            try:
                self.init_p2p(h)
            except _lib.CbxError as e:  # e.g. no peer access between these GPUs
                ok, err = False, str(e)
            if world > 1:  # every rank must agree, or the exchanges would hang
                import torch.distributed as dist
                flags = [None] * world
                dist.all_gather_object(flags, ok, group=group)
                ok = all(flags)
            if not ok:
                import sys
                print(f"slab: peer-memory transport unavailable ({err or 'another rank'}); "
                      "using NCCL", file=sys.stderr)
                if not err:  # this rank mapped its peers: undo
                    self._check(self.lib.cbx_slab_p2p_close(self.h))
                self.transport = "nccl"
                return self.connect("nccl", group)
            # the reverse halos fused into the passes only if every rank can
            fused = bool(self.lib.cbx_slab_p2p_fused(self.h))
            if world > 1:
                import torch.distributed as dist
                flags = [None] * world
                dist.all_gather_object(flags, fused, group=group)
                if not all(flags) and fused:
                    self._check(self.lib.cbx_slab_p2p_set_fused(self.h, 0))
                fused = all(flags)
            self.fused = fused
            self.transport = "p2p"
        elif transport == "nccl":
            uid = [SlabRank.nccl_unique_id() if self.rank == 0 else None]
            if world > 1:
                import torch.distributed as dist
                dist.broadcast_object_list(uid, src=0, group=group)
            self.init_comm(uid[0])
            self.fused = False
            self.transport = "nccl"
        else:
            raise ValueError(f"unknown transport {transport!r}")

    def p2p_send(self, kind: int):
        self._check(self.lib.cbx_slab_p2p_send(self.h, kind))

    def p2p_recv(self, kind: int):
        self._check(self.lib.cbx_slab_p2p_recv(self.h, kind))

    def bench_steps(self, dt: float, n: int, flush_mb: float = 0.0):
        out = (C.c_double * 8)()
        self._check(self.lib.cbx_bench_steps(self.h, dt, n, flush_mb, out))
        return list(out)

    def _check(self, rc):
        check(rc, self.h)

    def phase(self, p: int, dt: float = 0.0):
        self._check(self.lib.cbx_slab_phase(self.h, p, dt))

    def pack(self, kind: int, direction: int):
        t = self.buf[kind][0 if direction < 0 else 1]
        n = C.c_long()
        self._check(self.lib.cbx_slab_pack(self.h, kind, direction, C.c_void_p(t.data_ptr()),
                                           t.numel(), C.byref(n)))
        return t, n.value

    def unpack(self, kind: int, source: int, tensor, nbytes: int):
        self._check(self.lib.cbx_slab_unpack(self.h, kind, source,
                                             C.c_void_p(tensor.data_ptr()), nbytes))

    def local_state(self) -> np.ndarray:
        out = (C.c_double * 8)()
        self._check(self.lib.cbx_slab_local_state(self.h, out))
        return np.array(out[:])

    def commit(self, vals):
        v = (C.c_double * 4)(*[float(x) for x in vals[:4]])
        self._check(self.lib.cbx_slab_commit(self.h, v))

    def upload_global(self, s):
        from .engine import _ptr
        arrs = _store_arrays(s)
        st = _lib.Store(len(arrs["tag"]), *[_ptr(arrs[k]) for k in (
            "pos", "vel", "force", "rho", "df", "tag", "valid", "ghost")],
            len(arrs["clash_key"]), *[_ptr(arrs[k]) for k in (
                "clash_key", "clash_idx", "clash_pos", "clash_vel", "clash_force", "clash_rho",
                "clash_df", "clash_tag", "clash_ghost")])
        self._check(self.lib.cbx_upload_store_global(self.h, C.byref(st)))

    def download_global(self, g: dict, n_clash: int) -> int:
        from .engine import _ptr
        st = _lib.Store(len(g["tag"]), *[_ptr(g[k]) for k in (
            "pos", "vel", "force", "rho", "df", "tag", "valid", "ghost")],
            len(g["clash_key"]), *[_ptr(g[k]) for k in (
                "clash_key", "clash_idx", "clash_pos", "clash_vel", "clash_force", "clash_rho",
                "clash_df", "clash_tag", "clash_ghost")])
        n = C.c_long(n_clash)
        self._check(self.lib.cbx_download_store_global(self.h, C.byref(st), C.byref(n)))
        return n.value


def _store_arrays(s) -> dict:
    f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    n = len(s.clash_key)
    S = len(s.tag)
    return dict(pos=f64(s.pos), vel=f64(s.vel), force=f64(s.force), rho=f64(s.rho),
                df=f64(s.df), tag=np.ascontiguousarray(s.tag, dtype=np.uint64),
                valid=np.ascontiguousarray(s.valid, dtype=np.uint8),
                ghost=np.ascontiguousarray(getattr(s, "ghost", np.zeros(S)), dtype=np.uint8),
                clash_key=np.ascontiguousarray(s.clash_key, dtype=np.int64),
                clash_idx=np.zeros(n, np.int32), clash_pos=f64(s.clash_pos).reshape(n, 3),
                clash_vel=f64(s.clash_vel).reshape(n, 3),
                clash_force=f64(s.clash_force).reshape(n, 3), clash_rho=f64(s.clash_rho),
                clash_df=f64(s.clash_df),
                clash_tag=np.ascontiguousarray(s.clash_tag, dtype=np.uint64),
                clash_ghost=np.ascontiguousarray(s.clash_ghost, dtype=np.uint8))


# ------------------------------------------------------------- exchanges
def reduce_states(states: List[np.ndarray]) -> np.ndarray:
    """sum kinetic / pair / embedding / guard counters, max of max_speed"""
    a = np.array(states)
    out = a.sum(axis=0)
    out[3] = a[:, 3].max()
    out[6:8] = a[0, 6:8]
    return out


class LocalExchange:
    """All ranks live in this process (virtual ranks, e.g. on one GPU):
    the receiver unpacks straight from the sender's device buffer."""

    def __init__(self, ranks: List):
        self.ranks = ranks
        self.bytes_moved = 0

    def exchange(self, kind: int):
        n = len(self.ranks)
        packed = [(r.pack(kind, -1), r.pack(kind, +1)) for r in self.ranks]
        for i, r in enumerate(self.ranks):
            lo, hi = neighbours(i, n)
            (tb, nb) = packed[lo][1]  # the rank below sent its "up" buffer
            (ta, na) = packed[hi][0]  # the rank above sent its "down" buffer
            r.unpack(kind, -1, tb, nb)
            r.unpack(kind, +1, ta, na)
            self.bytes_moved += nb + na

    def allreduce(self, states: List[np.ndarray]) -> np.ndarray:
        return reduce_states(states)


class DistExchange:
    """One rank per process over torch.distributed (NCCL on GPUs, gloo on
    CPU): two rounds of paired send/recv with the ring neighbours, sizes
    first, then payloads."""

    def __init__(self, rank_obj, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.r = rank_obj
        self.rank = dist.get_rank(group)
        self.n = dist.get_world_size(group)
        self.group = group
        self.bytes_moved = 0

    def _sendrecv(self, send_t, dst, recv_t, src):
        dist = self.dist
        ops = [dist.P2POp(dist.isend, send_t, dst, self.group),
               dist.P2POp(dist.irecv, recv_t, src, self.group)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()

    def exchange(self, kind: int):
        import torch
        lo, hi = neighbours(self.rank, self.n)
        out = {}
        for direction, dst, src in ((-1, lo, hi), (+1, hi, lo)):
            t, nb = self.r.pack(kind, direction)
            dev = t.device
            size_out = torch.tensor([nb], dtype=torch.int64, device=dev)
            size_in = torch.zeros(1, dtype=torch.int64, device=dev)
            self._sendrecv(size_out, dst, size_in, src)
            m = int(size_in.item())
            recv = torch.empty(max(m, 1), dtype=torch.uint8, device=dev)
            self._sendrecv(t[:max(nb, 1)], dst, recv, src)
            out[-direction] = (recv, m)  # what I got came from the other side
            self.bytes_moved += nb
        self.r.unpack(kind, -1, *out[-1])
        self.r.unpack(kind, +1, *out[+1])

    def allreduce(self, states: List[np.ndarray]) -> np.ndarray:
        import torch
        s = states[0]
        dev = getattr(self.r, "comm_device", "cpu")
        t = torch.tensor(np.concatenate([s[[0, 1, 2, 4, 5]], [s[3]]]), dtype=torch.float64,
                         device=dev)
        sums = t[:5].clone()
        mx = t[5:].clone()
        self.dist.all_reduce(sums, op=self.dist.ReduceOp.SUM, group=self.group)
        self.dist.all_reduce(mx, op=self.dist.ReduceOp.MAX, group=self.group)
        out = s.copy()
        out[[0, 1, 2, 4, 5]] = sums.cpu().numpy()
        out[3] = float(mx.cpu().item())
        return out


class P2PLockstep:
    """The peer-memory transport driven from the host, one rank per process:
    each exchange is a send (the rank's kernel stores its packets into the
    neighbours' mapped buffers and raises their flags, and completes), a
    barrier of all ranks, and a receive (the flags are up: unpack).  No
    kernel waits on another rank's kernel, so ranks may share one GPU.  The
    StepState reduction goes through torch.distributed (gloo or NCCL)."""

    def __init__(self, rank_obj, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.r = rank_obj
        self.group = group
        self.rank = dist.get_rank(group)
        self.n = dist.get_world_size(group)

    def exchange(self, kind: int):
        self.r.p2p_send(kind)
        self.dist.barrier(group=self.group)
        self.r.p2p_recv(kind)
        self.dist.barrier(group=self.group)  # receive buffers free for the next send

    def allreduce(self, states: List[np.ndarray]) -> np.ndarray:
        import torch
        s = states[0]
        sums = torch.tensor(s[[0, 1, 2, 4, 5]], dtype=torch.float64)
        mx = torch.tensor([s[3]], dtype=torch.float64)
        self.dist.all_reduce(sums, op=self.dist.ReduceOp.SUM, group=self.group)
        self.dist.all_reduce(mx, op=self.dist.ReduceOp.MAX, group=self.group)
        out = s.copy()
        out[[0, 1, 2, 4, 5]] = sums.numpy()
        out[3] = float(mx.item())
        return out


class SlabDomain:
    """Drives one or more slab ranks through the phases of a step."""

    def __init__(self, ranks: List, exchange):
        self.ranks = ranks
        self.ex = exchange

    def _all(self, p, dt=0.0):
        for r in self.ranks:
            r.phase(p, dt)

    def _reduce_commit(self):
        g = self.ex.allreduce([r.local_state() for r in self.ranks])
        for r in self.ranks:
            r.commit(g)
        return g

    def prime(self):
        """fill the z halos and evaluate forces (the Simulation constructor's
        refresh_forces + measure, sim.cpp:145-147)"""
        self.ex.exchange(POS)
        self._all(2)
        self.ex.exchange(RHO)
        self._all(3)
        self.ex.exchange(DF)
        self._all(4)
        self.ex.exchange(FRC)
        self._all(6)
        self._all(7)
        return self._reduce_commit()

    def step(self, dt: float = -1.0, n: int = 1):
        g = None
        for _ in range(n):
            self._all(0, dt)
            self.ex.exchange(MIGRANTS)
            self._all(1)
            self.ex.exchange(POS)
            self._all(2)
            self.ex.exchange(RHO)
            self._all(3)
            self.ex.exchange(DF)
            self._all(4)
            self.ex.exchange(FRC)
            self._all(5)
            g = self._reduce_commit()
        return g

    def state(self) -> dict:
        """the committed (already reduced) step state; every rank holds it"""
        s = self.ranks[0].local_state()
        return {"kinetic": s[0], "pair": s[1], "embedding": s[2], "max_speed": s[3],
                "r_underflow": int(s[4]), "rho_clamp": int(s[5]), "step": int(s[6]),
                "t": s[7]}

    def count_defects(self):
        tot = np.zeros(3, dtype=np.int64)
        for r in self.ranks:
            tot += np.array(r.count_defects())
        return int(tot[0]), int(tot[1]), int(max(tot[0], tot[1]))
