"""CPU (gloo, world_size 2 and 3) tests of the slab decomposition's host logic:
the driver (paper_1412_3784_b200/slab.py), its torch.distributed transport and
the exchange protocol, with a numpy stand-in engine whose arithmetic is the
oracle's.  Checks: migration conserves particles and lands each one on the
rank owning its cell layer; one-layer halos suffice for exact forces; the
all-gathered layer partials reproduce the single-domain energy and virial."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
from paper_1412_3784_b200 import workloads as W


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class NumpyRank:
    """Test engine with the SlabRank phase interface; arithmetic by the oracle."""

    def __init__(self, rank, P, w, q_own, p_own, gid_own):
        self.rank, self.P, self.w = rank, P, w
        self.q, self.p, self.gid = q_own.copy(), p_own.copy(), gid_own.copy()
        self.n = len(q_own)
        cap = 1 << 16
        z = lambda k: torch.zeros((cap, k), dtype=torch.float64)  # noqa: E731
        self.recv = [z(8), z(8)]
        self.hrecv = [z(4), z(4)]

    def layers(self):
        _, _, dims = oracle.cell_keys(oracle.DO, self.q[:1], self.w.L, self.w.rc)
        l3 = int(dims[2])
        return self.rank * l3 // self.P, (self.rank + 1) * l3 // self.P, l3

    def _layer(self, q):
        cell, _, dims = oracle.cell_keys(oracle.DO, q, self.w.L, self.w.rc)
        return cell // (int(dims[0]) * int(dims[1]))

    def migrate(self):
        klo, khi, l3 = self.layers()
        self.q = oracle.wrap(self.q, self.w.L)
        lay = self._layer(self.q)
        to_lo = lay == (klo - 1) % l3
        to_hi = lay == khi % l3
        stay = (lay >= klo) & (lay < khi)
        assert np.all(stay | to_lo | to_hi)

        def rec(m):
            r = np.zeros((int(m.sum()), 8))
            r[:, :3], r[:, 3], r[:, 4:7] = self.q[m], self.gid[m], self.p[m]
            return torch.from_numpy(r)

        s_lo, s_hi = rec(to_lo), rec(to_hi)
        self.q, self.p, self.gid = self.q[stay], self.p[stay], self.gid[stay]
        self.n = len(self.q)
        return (s_lo, len(s_lo), s_hi, len(s_hi))

    def absorb(self, from_lo, n_lo, from_hi, n_hi):
        for rec, k in ((from_lo, n_lo), (from_hi, n_hi)):
            r = rec[:k].numpy()
            self.q = np.concatenate([self.q, r[:, :3]])
            self.gid = np.concatenate([self.gid, r[:, 3].astype(np.int64)])
            self.p = np.concatenate([self.p, r[:, 4:7]])
        self.n = len(self.q)

    def halo(self):
        klo, khi, _ = self.layers()
        lay = self._layer(self.q)

        def rec(m):
            r = np.zeros((int(m.sum()), 4))
            r[:, :3], r[:, 3] = self.q[m], self.gid[m]
            return torch.from_numpy(r)

        h_lo, h_hi = rec(lay == klo), rec(lay == khi - 1)
        return (h_lo, len(h_lo), h_hi, len(h_hi))

    def forces(self, h_lo, n_lo, h_hi, n_hi, want_parts=True):
        klo, khi, _ = self.layers()
        allq = np.concatenate([self.q, h_lo[:n_lo, :3].numpy(), h_hi[:n_hi, :3].numpy()])
        r = oracle.evaluate(oracle.DO, allq, self.w.L, self.w.rc, ushift=self.w.ushift,
                            idx=np.arange(self.n), want=("F", "U", "W", "digest"))
        self.F = r.F
        self.halo_gids = np.concatenate([h_lo[:n_lo, 3].numpy(), h_hi[:n_hi, 3].numpy()]).astype(np.int64)
        lay = self._layer(self.q) - klo
        from paper_1412_3784_b200.slab import NPART

        parts = np.zeros((khi - klo, NPART))
        np.add.at(parts[:, 0], lay, r.U_i)
        for k in range(6):
            np.add.at(parts[:, 1 + k], lay, r.W_i[:, k])
        np.add.at(parts[:, 7], lay, r.cnt.astype(np.float64))
        return parts

    # the split evaluation (SlabSystem overlaps the halo payload with forces_begin)
    def forces_begin(self, n_lo, n_hi):
        self.pending_counts = (n_lo, n_hi)

    def forces_end(self, h_lo, n_lo, h_hi, n_hi, want_parts=True):
        assert (n_lo, n_hi) == self.pending_counts, "counts of begin and end agree"
        return self.forces(h_lo, n_lo, h_hi, n_hi, want_parts)

    def reduce(self, allp):
        tot = allp.sum(axis=0)
        return tot[0], tot[1:7], {"interactions": tot[7]}


def worker(rank, P, port, out):
    from paper_1412_3784_b200.slab import DistTransport, SlabSystem

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.distributed.init_process_group("gloo", rank=rank, world_size=P)
    try:
        w = W.make(2, scale=2)
        q = oracle.wrap(W.positions(w, k=2), w.L)
        p = W.momenta(w, k=2)
        n = len(q)
        cell, _, dims = oracle.cell_keys(oracle.DO, q, w.L, w.rc)
        layer = cell // (int(dims[0]) * int(dims[1]))
        l3 = int(dims[2])
        klo, khi = rank * l3 // P, (rank + 1) * l3 // P
        own = np.nonzero((layer >= klo) & (layer < khi))[0]
        eng = NumpyRank(rank, P, w, q[own], p[own], own.astype(np.int64))
        sysm = SlabSystem([eng], DistTransport(rank, P, "cpu"))
        # (1) forces through halo exchange == single-domain oracle forces
        U, Wv, st = sysm.forces(True)
        ref = oracle.evaluate(oracle.DO, q, w.L, w.rc, ushift=w.ushift)
        ferr = np.abs(eng.F - ref.F[eng.gid]).max()
        # (2) migration after a random displacement of up to 0.3 sigma
        rng = np.random.default_rng(100 + rank)
        eng.q = eng.q + rng.uniform(-0.3, 0.3, size=eng.q.shape)
        sends = [eng.migrate()]
        recvs = sysm.tr.exchange(sends, [eng.recv])
        eng.absorb(*recvs[0])
        gids = [None] * P
        torch.distributed.all_gather_object(gids, eng.gid.tolist())
        lay_ok = bool(np.all((eng._layer(oracle.wrap(eng.q, w.L)) >= klo) & (eng._layer(oracle.wrap(eng.q, w.L)) < khi)))
        out.put((rank, ferr, U, ref.U, np.abs(Wv - ref.W).max(), np.abs(ref.W).max(), st["interactions"],
                 ref.interactions, sorted(sum(gids, [])) == list(range(n)), lay_ok))
    finally:
        torch.distributed.destroy_process_group()


@pytest.mark.parametrize("P", [2, 3])
def test_slab_protocol_gloo(P):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, P, port, out)) for r in range(P)]
    for pr in procs:
        pr.start()
    res = [out.get(timeout=600) for _ in range(P)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for (rank, ferr, U, Uref, werr, wmax, inter, iref, conserved, lay_ok) in res:
        assert ferr < 1e-11, (rank, ferr)
        assert U == pytest.approx(Uref, rel=1e-12)
        assert werr <= 1e-12 * wmax
        assert inter == iref
        assert conserved and lay_ok


def _allgather_worker(rank, P, port, out):
    from paper_1412_3784_b200.slab import DistTransport

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.distributed.init_process_group("gloo", rank=rank, world_size=P)
    try:
        n = 3 + 2 * rank  # variable lengths
        q = torch.full((n, 3), float(rank))
        gid = torch.arange(n, dtype=torch.int32) + 100 * rank
        owner = torch.full((n,), (rank + 1) % P, dtype=torch.int64)
        tq, tg, to = DistTransport(rank, P, "cpu").allgather_tensors([(q, gid, owner)])
        out.put((rank, tq.tolist(), tg.tolist(), to.tolist()))
    finally:
        torch.distributed.destroy_process_group()


@pytest.mark.parametrize("P", [2, 3])
def test_repartition_allgather_gloo(P):
    """The all-gather behind SlabSystem.repartition (counts, padded payload, rank order) over gloo."""
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_allgather_worker, args=(r, P, port, out)) for r in range(P)]
    for pr in procs:
        pr.start()
    res = sorted(out.get(timeout=300) for _ in range(P))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    exp_g = sum([[k + 100 * r for k in range(3 + 2 * r)] for r in range(P)], [])
    exp_q = sum([[[float(r)] * 3] * (3 + 2 * r) for r in range(P)], [])
    for rank, tq, tg, to in res:
        assert tg == exp_g and tq == exp_q
        assert to == sum([[(r + 1) % P] * (3 + 2 * r) for r in range(P)], [])
