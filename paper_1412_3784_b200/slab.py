"""Slab decomposition of the cell-list path over several GPUs.

One rank per GPU.  The box is cut into slabs of whole cell layers along the
third lattice direction (lambda_3: DS layer floor(lambda_3 c_3), DO layer
floor(z/w_3) with z = r_33 lambda_3 -- the same axis for both variants, so the
DO rearrangement never crosses a slab).  Rank r owns layers
[floor(r l3/P), floor((r+1) l3/P)).  One SLLOD step:

  kick + drift (own particles)                      nc_slab_kick_drift
  wrap, split leavers by layer, pack                nc_slab_migrate
  exchange migration records with r-1, r+1          transport
  append arrivals                                   nc_slab_unpack
  pack the two boundary layers as halo records      nc_slab_halo
  exchange halo records with r-1, r+1               transport
  cells over own + halo, K3 over own layers only    nc_slab_forces
  second kick                                       nc_slab_kick
  layer partials all-gathered, fixed-order sum      nc_slab_reduce

Every arithmetic step runs in libnemdcell.so; this module only moves buffers
(torch.distributed P2P: NCCL over NVLink between GPUs, gloo on CPU) and keeps
the bookkeeping.  Halo = one cell layer (thickness >= r_c), positions + gid
only; full i-side accumulation means no reverse force communication.
Results are bitwise identical to a single-device evaluation (same cell
contents in (cell, gid) order, same per-layer reductions, same final sum).
"""
from __future__ import annotations

import numpy as np

from . import nemdcell as nc

NPART = 13


class SlabRank:
    """State of one rank: own particles (device tensors), its context, buffers."""

    def __init__(self, rank: int, nranks: int, *, variant="do", prec="f32", rc=2.5, eps=1.0, sigma=1.0,
                 u_shift=None, mass=1.0, capacity=1 << 16, max_cells=0, device=0, stream=None, ctx_capacity=None,
                 count_buffers=True):
        import torch

        self.torch = torch
        self.rank, self.nranks = rank, nranks
        self.cl = nc.CellList(variant, prec, rc=rc, eps=eps, sigma=sigma, u_shift=u_shift, mass=mass,
                              capacity=ctx_capacity or capacity, max_cells=max_cells, device=device, stream=stream)
        self.ctx = self.cl.ctx
        self.dev = f"cuda:{device}"
        self.dtype = self.cl.dtype
        self.cap = capacity
        t = lambda *s: torch.zeros(*s, dtype=self.dtype, device=self.dev)  # noqa: E731
        self.q, self.p, self.F = t(capacity, 3), t(capacity, 3), t(capacity, 3)
        self.q2, self.p2 = t(capacity, 3), t(capacity, 3)
        self.gid = torch.zeros(capacity, dtype=torch.int32, device=self.dev)
        self.gid2 = torch.zeros_like(self.gid)
        self.bcap = max(4096, capacity // 4)
        if count_buffers:  # the host-count step's record buffers (SlabRankDev has its own messages)
            self.send = [t(self.bcap, 8), t(self.bcap, 8)]           # migration records to r-1, r+1
            self.recv = [t(self.bcap, 8), t(self.bcap, 8)]           # from r-1, r+1
            self.hsend = [t(self.bcap, 4), t(self.bcap, 4)]          # halo records to r-1, r+1
            self.hrecv = [t(self.bcap, 4), t(self.bcap, 4)]
        self.n = 0
        self.pending_dt = 0.0  # a deferred closing half kick (see kick)
        self.last_l3 = None    # cell layers of the box the particles were last distributed on

    def set_flow(self, A, policy, t0, **kw):
        self.cl.set_flow(A, policy, t0, **kw)

    def layers(self):
        return nc.nc_slab_layers(self.ctx, self.rank, self.nranks)

    def load(self, q_own, p_own, gid_own):
        self.pending_dt = 0.0
        n = len(q_own)
        assert n <= self.cap
        self.q[:n].copy_(self.torch.as_tensor(q_own))
        self.p[:n].copy_(self.torch.as_tensor(p_own))
        self.gid[:n].copy_(self.torch.as_tensor(np.asarray(gid_own, dtype=np.int32)))
        self.n = n
        self.last_l3 = self.layers()[2]

    # ---------------------------------------------------------------- phases
    def kick_drift(self, dt):
        # the previous step's closing half kick, if deferred, runs in the same pass
        nc.nc_slab_kick_kick_drift(self.ctx, self.q, self.p, self.F, self.n, self.pending_dt, dt)
        self.pending_dt = 0.0

    def l3_changed(self):
        return self.layers()[2] != self.last_l3

    def owned(self):
        """(q, p, gid, owner rank) of the own particles, q wrapped, owners for the CURRENT l3
        (nc_slab_layer_of): the input of a repartition."""
        torch = self.torch
        n = self.n
        layer = torch.empty(max(n, 1), dtype=torch.int32, device=self.dev)
        nc.nc_slab_layer_of(self.ctx, self.q, n, layer)
        _, _, l3 = self.layers()
        bounds = torch.tensor([r * l3 // self.nranks for r in range(1, self.nranks)], dtype=torch.int32,
                              device=self.dev)
        owner = torch.bucketize(layer[:n], bounds, right=True)  # r with floor(r l3/P) <= layer < floor((r+1) l3/P)
        return self.q[:n].clone(), self.p[:n].clone(), self.gid[:n].clone(), owner

    def take(self, q, p, gid):
        """Replace the own particles (after a repartition)."""
        n = len(q)
        assert n <= self.cap, "slab capacity exceeded"
        self.q[:n].copy_(q)
        self.p[:n].copy_(p)
        self.gid[:n].copy_(gid)
        self.n = n
        self.last_l3 = self.layers()[2]

    def migrate(self):
        klo, khi, _ = self.layers()
        ns, nlo, nhi = nc.nc_slab_migrate(self.ctx, self.q, self.p, self.gid, self.n, klo, khi, self.q2, self.p2,
                                          self.gid2, self.send[0], self.send[1], self.bcap)
        self.q, self.q2 = self.q2, self.q
        self.p, self.p2 = self.p2, self.p
        self.gid, self.gid2 = self.gid2, self.gid
        self.n = ns
        return (self.send[0], nlo, self.send[1], nhi)

    def absorb(self, from_lo, n_lo, from_hi, n_hi):
        for rec, k in ((from_lo, n_lo), (from_hi, n_hi)):
            if k:
                assert self.n + k <= self.cap, "slab capacity exceeded"
                nc.nc_slab_unpack(self.ctx, rec, k, self.q[self.n:], self.p[self.n:], self.gid[self.n:])
                self.n += k

    def halo(self):
        if self.nranks == 1:  # a single slab wraps onto itself: no halo
            return (self.hsend[0], 0, self.hsend[1], 0)
        klo, khi, _ = self.layers()
        nlo, nhi = nc.nc_slab_halo(self.ctx, self.q, self.gid, self.n, klo, khi, self.hsend[0], self.hsend[1],
                                   self.bcap)
        return (self.hsend[0], nlo, self.hsend[1], nhi)

    def forces(self, h_lo, n_lo, h_hi, n_hi, want_parts=True):
        klo, khi, _ = self.layers()
        return nc.nc_slab_forces(self.ctx, self.q, self.gid, self.n, h_lo, n_lo, h_hi, n_hi, klo, khi, self.F,
                                 want_parts)

    def forces_begin(self, n_lo, n_hi):
        """Own particles into cells and K3 on the interior layers (the halo counts are known)."""
        klo, khi, _ = self.layers()
        nc.nc_slab_forces_begin(self.ctx, self.q, self.gid, self.n, n_lo, n_hi, klo, khi)

    def forces_end(self, h_lo, n_lo, h_hi, n_hi, want_parts=True):
        """Halo particles in, K3 on the boundary layers, reduction, forces (bitwise = forces())."""
        klo, khi, _ = self.layers()
        return nc.nc_slab_forces_end(self.ctx, h_lo, h_hi, self.F, klo, khi, want_parts)

    def kick(self, dt):
        # closing half kick: deferred into the next kick_drift (p and F in this rank's order stay
        # untouched until then); flush() applies it when the momenta are read
        self.pending_dt = dt

    def flush(self):
        if self.pending_dt > 0:
            nc.nc_slab_kick(self.ctx, self.p, self.F, self.n, self.pending_dt)
            self.pending_dt = 0.0

    def reduce(self, all_parts):
        return nc.nc_slab_reduce(self.ctx, all_parts)

    def close(self):
        self.cl.close()


class SlabRankDev(SlabRank):
    """A rank of the HOST-SYNCHRONIZATION-FREE slab step (csrc/slab_dc.cuh): the own count lives on the
    device, every kernel runs over the capacity, messages are fixed-capacity buffers whose first record
    carries the count, and the own particles of the force evaluation sit at fixed sorted slots so the
    interior layers' pair kernel runs before any halo count is known.  Nothing in step() reads the
    device; `n` (and status()) synchronize when asked.  Bitwise the same trajectory as SlabRank."""

    def __init__(self, rank: int, nranks: int, *, capacity=1 << 16, hcap=None, mcap=None, **kw):
        hcap = int(hcap or max(4096, capacity // 4))
        mcap = int(mcap or max(4096, capacity // 16))
        # the context indexes own + two halo layers' worth of slots
        super().__init__(rank, nranks, capacity=capacity, ctx_capacity=capacity + 2 * hcap, count_buffers=False, **kw)
        torch = self.torch
        t = lambda *s: torch.zeros(*s, dtype=self.dtype, device=self.dev)  # noqa: E731
        self.hcap, self.mcap = hcap, mcap
        self.msend = [t(1 + mcap, 8), t(1 + mcap, 8)]    # migration messages (header record + records)
        self.mrecv = [t(1 + mcap, 8), t(1 + mcap, 8)]
        self.hsend = [t(1 + hcap, 4), t(1 + hcap, 4)]    # halo messages
        self.hrecv = [t(1 + hcap, 4), t(1 + hcap, 4)]

    @property
    def n(self):
        return nc.nc_sd_status(self.ctx)[0] if getattr(self, "_dev_ready", False) else self._n0

    @n.setter
    def n(self, v):
        self._n0 = v

    def status(self):
        return nc.nc_sd_status(self.ctx)

    def load(self, q_own, p_own, gid_own):
        super().load(q_own, p_own, gid_own)
        nc.nc_sd_load(self.ctx, len(q_own))
        self._dev_ready = True

    def take(self, q, p, gid):
        super().take(q, p, gid)
        nc.nc_sd_load(self.ctx, len(q))

    def kick_drift(self, dt):
        nc.nc_sd_kick_drift(self.ctx, self.q, self.p, self.F, self.cap, self.pending_dt, dt)
        self.pending_dt = 0.0

    def migrate(self):
        klo, khi, _ = self.layers()
        nc.nc_sd_migrate(self.ctx, self.q, self.p, self.gid, self.cap, klo, khi, self.q2, self.p2, self.gid2,
                         self.msend[0], self.msend[1], self.mcap)
        self.q, self.q2 = self.q2, self.q
        self.p, self.p2 = self.p2, self.p
        self.gid, self.gid2 = self.gid2, self.gid
        return self.msend

    def absorb_msgs(self):
        nc.nc_sd_absorb(self.ctx, self.mrecv[0], self.mrecv[1], self.mcap, self.q, self.p, self.gid, self.cap)

    def halo(self):
        if self.nranks == 1:  # a single slab wraps onto itself: no halo (the receive headers stay 0)
            return None
        klo, khi, _ = self.layers()
        nc.nc_sd_halo(self.ctx, self.q, self.gid, self.cap, klo, khi, self.hsend[0], self.hsend[1], self.hcap)
        return self.hsend

    def forces_begin_dev(self):
        klo, khi, _ = self.layers()
        nc.nc_sd_forces_begin(self.ctx, self.q, self.gid, self.cap, self.hcap, klo, khi)

    def forces_end_dev(self, want_parts=True):
        """Forces of the own particles, which adopt their sorted (cell, gid) order at the same time (q, p,
        gid and F permuted together): the next step's kernels read spatially ordered arrays."""
        klo, khi, _ = self.layers()
        parts = nc.nc_sd_forces_end_sorted(self.ctx, self.hrecv[0], self.hrecv[1], self.p, self.q2, self.p2,
                                           self.gid2, self.F, want_parts, khi - klo)
        self.q, self.q2 = self.q2, self.q
        self.p, self.p2 = self.p2, self.p
        self.gid, self.gid2 = self.gid2, self.gid
        return parts

    def flush(self):
        if self.pending_dt > 0:
            nc.nc_sd_kick(self.ctx, self.p, self.F, self.cap, self.pending_dt)
            self.pending_dt = 0.0


# -------------------------------------------------------------------- transports

class LoopbackTransport:
    """All ranks in one process (tests on one GPU): rank r's send_lo is rank r-1's
    from_hi, its send_hi is rank r+1's from_lo (periodic in the rank index)."""

    # fixed-capacity messages of the host-synchronization-free step (whole buffers, counts inside)
    def exchange_msgs(self, sends, recv_bufs):
        P = len(sends)
        for r in range(P):
            recv_bufs[r][0].copy_(sends[(r - 1) % P][1])  # from r-1: its upper message
            recv_bufs[r][1].copy_(sends[(r + 1) % P][0])  # from r+1: its lower message

    def start_msgs(self, sends, recv_bufs):
        self.exchange_msgs(sends, recv_bufs)

    def finish_msgs(self):
        pass

    # split exchange (counts first, then the payload) for the overlapped force evaluation
    def counts(self, sends):
        P = len(sends)
        return [(sends[(r - 1) % P][3], sends[(r + 1) % P][1]) for r in range(P)]

    def start(self, sends, recv_bufs, counts):
        return self.exchange(sends, recv_bufs)

    def finish(self, pending):
        return pending

    def exchange(self, sends, recv_bufs):
        P = len(sends)
        out = []
        for r in range(P):
            lo_src = sends[(r - 1) % P]   # rank r-1 sends its upper boundary up
            hi_src = sends[(r + 1) % P]   # rank r+1 sends its lower boundary down
            b_lo, b_hi = recv_bufs[r]
            n_lo, n_hi = lo_src[3], hi_src[1]
            b_lo[:n_lo].copy_(lo_src[2][:n_lo])
            b_hi[:n_hi].copy_(hi_src[0][:n_hi])
            out.append((b_lo, n_lo, b_hi, n_hi))
        return out

    def gather(self, parts):
        return np.concatenate(parts, axis=0)

    def allgather_tensors(self, per_rank):
        """per_rank[r] = tuple of tensors of rank r -> tuple of concatenations over the ranks."""
        import torch

        return tuple(torch.cat([t[k] for t in per_rank]) for k in range(len(per_rank[0])))


def _dist_allgather_tensors(dist, torch, device, tensors):
    """All-gather of variable-length tensors (counts first, padded payload) through torch.distributed:
    the rare repartition after an l3 change, not the per-step data plane."""
    n = torch.tensor([len(tensors[0])], dtype=torch.int64, device=device)
    P = dist.get_world_size()
    ns = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(P)]
    dist.all_gather(ns, n)
    counts = [int(x.item()) for x in ns]
    mx = max(max(counts), 1)
    out = []
    for t in tensors:
        src = t.to(device)
        buf = torch.zeros((mx,) + tuple(src.shape[1:]), dtype=src.dtype, device=device)
        buf[:len(src)] = src
        bufs = [torch.zeros_like(buf) for _ in range(P)]
        dist.all_gather(bufs, buf)
        out.append(torch.cat([b[:c] for b, c in zip(bufs, counts)]).to(t.device))
    return tuple(out)


class DistTransport:
    """One rank of a torch.distributed group (NCCL between GPUs, gloo on CPU).
    Messages to one peer are matched in issue order: each rank sends to r-1
    first, then to r+1, and receives from r+1 first, then from r-1."""

    def __init__(self, rank, nranks, device, stream=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.rank, self.P = rank, nranks
        self.device = device
        # the stream the library's kernels run on (cfg.stream): the exchange is waited for ON it, so
        # nc_slab_forces_end never reads a halo buffer before it has arrived, whatever the caller's
        # current stream
        self.stream = stream

    def _p2p(self, tensors_out, tensors_in):
        dist = self.dist
        lo, hi = (self.rank - 1) % self.P, (self.rank + 1) % self.P
        ops = [dist.P2POp(dist.isend, tensors_out[0], lo), dist.P2POp(dist.isend, tensors_out[1], hi),
               dist.P2POp(dist.irecv, tensors_in[1], hi), dist.P2POp(dist.irecv, tensors_in[0], lo)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()

    def exchange_msgs(self, sends, recv_bufs):
        (s_lo, s_hi), = sends
        r_lo, r_hi = recv_bufs[0]
        self._p2p([s_lo, s_hi], [r_lo, r_hi])

    def start_msgs(self, sends, recv_bufs):
        self.exchange_msgs(sends, recv_bufs)

    def finish_msgs(self):
        pass

    def counts(self, sends):
        torch = self.torch
        (s_lo, n_lo, s_hi, n_hi), = sends
        cnt_out = [torch.tensor([n_lo], dtype=torch.int64, device=self.device),
                   torch.tensor([n_hi], dtype=torch.int64, device=self.device)]
        cnt_in = [torch.zeros(1, dtype=torch.int64, device=self.device) for _ in range(2)]
        self._p2p(cnt_out, cnt_in)
        return [(int(cnt_in[0].item()), int(cnt_in[1].item()))]

    def start(self, sends, recv_bufs, counts):
        """Issue the payload exchange and return without waiting (NCCL runs on its own stream)."""
        dist = self.dist
        (s_lo, n_lo, s_hi, n_hi), = sends
        b_lo, b_hi = recv_bufs[0]
        (m_lo, m_hi), = counts
        assert m_lo <= len(b_lo) and m_hi <= len(b_hi), "receive buffer too small"
        lo, hi = (self.rank - 1) % self.P, (self.rank + 1) % self.P
        ops = [dist.P2POp(dist.isend, s_lo[:max(n_lo, 1)], lo), dist.P2POp(dist.isend, s_hi[:max(n_hi, 1)], hi),
               dist.P2POp(dist.irecv, b_hi[:max(m_hi, 1)], hi), dist.P2POp(dist.irecv, b_lo[:max(m_lo, 1)], lo)]
        return dist.batch_isend_irecv(ops), [(b_lo, m_lo, b_hi, m_hi)]

    def finish(self, pending):
        works, out = pending
        if self.stream is not None and str(self.device).startswith("cuda"):
            with self.torch.cuda.stream(self.torch.cuda.ExternalStream(self.stream)):
                for w in works:
                    w.wait()  # the library's stream waits for the exchange
        else:
            for w in works:
                w.wait()
        return out

    def exchange(self, sends, recv_bufs):
        torch = self.torch
        (s_lo, n_lo, s_hi, n_hi), = sends
        b_lo, b_hi = recv_bufs[0]
        cnt_out = [torch.tensor([n_lo], dtype=torch.int64, device=self.device),
                   torch.tensor([n_hi], dtype=torch.int64, device=self.device)]
        cnt_in = [torch.zeros(1, dtype=torch.int64, device=self.device) for _ in range(2)]
        self._p2p(cnt_out, cnt_in)
        m_lo, m_hi = int(cnt_in[0].item()), int(cnt_in[1].item())
        assert m_lo <= len(b_lo) and m_hi <= len(b_hi), "receive buffer too small"
        self._p2p([s_lo[:max(n_lo, 1)], s_hi[:max(n_hi, 1)]], [b_lo[:max(m_lo, 1)], b_hi[:max(m_hi, 1)]])
        return [(b_lo, m_lo, b_hi, m_hi)]

    def allgather_tensors(self, per_rank):
        return _dist_allgather_tensors(self.dist, self.torch, self.device, per_rank[0])

    def gather(self, parts):
        torch, dist = self.torch, self.dist
        part, = parts
        n = torch.tensor([part.shape[0]], dtype=torch.int64, device=self.device)
        ns = [torch.zeros(1, dtype=torch.int64, device=self.device) for _ in range(self.P)]
        dist.all_gather(ns, n)
        mx = max(int(x.item()) for x in ns)
        buf = torch.zeros((mx, NPART), dtype=torch.float64, device=self.device)
        buf[:part.shape[0]] = torch.as_tensor(part, device=self.device)
        bufs = [torch.zeros_like(buf) for _ in range(self.P)]
        dist.all_gather(bufs, buf)
        return np.concatenate([b[:int(k.item())].cpu().numpy() for b, k in zip(bufs, ns)], axis=0)


class HostStagedTransport(DistTransport):
    """gloo between processes (e.g. ranks that share one GPU in a test): every device buffer crosses
    through host memory, so no rank's kernels ever wait on another rank's on the device."""

    def __init__(self, rank, nranks):
        super().__init__(rank, nranks, "cpu")

    def _p2p(self, tensors_out, tensors_in):
        outs = [t.cpu() for t in tensors_out]
        ins = [self.torch.empty(t.shape, dtype=t.dtype) for t in tensors_in]
        super()._p2p(outs, ins)
        for t, c in zip(tensors_in, ins):
            t.copy_(c)

    def start(self, sends, recv_bufs, counts):
        (s_lo, n_lo, s_hi, n_hi), = sends
        b_lo, b_hi = recv_bufs[0]
        (m_lo, m_hi), = counts
        assert m_lo <= len(b_lo) and m_hi <= len(b_hi), "receive buffer too small"
        self._p2p([s_lo[:max(n_lo, 1)], s_hi[:max(n_hi, 1)]], [b_lo[:max(m_lo, 1)], b_hi[:max(m_hi, 1)]])
        return [(b_lo, m_lo, b_hi, m_hi)]

    def finish(self, pending):
        return pending


class IpcTransport(DistTransport):
    """The peer-memory data plane (csrc/ipc_slab.cuh) for the host-synchronization-free step (SlabRankDev,
    P >= 2): every rank exports double-buffered receive buffers for the halo and migration messages and
    maps its neighbours', and the packing kernels (nc_sd_halo, nc_sd_migrate) write their messages
    straight into the neighbours' receive buffers -- pack and transfer in one pass over peer memory
    (NVLink between GPUs), no send buffer, copy or collective.  An exchange is then ordering only:
    interprocess events recorded after the packing ("sent") and after the reads of the previous messages
    ("consumed"), a host barrier (a stream wait binds to the record issued before it), and stream waits
    on the neighbours' events -- no kernel ever spins on another rank.  The energy partials and the rare
    repartition go through torch.distributed like DistTransport."""

    KINDS = ("h", "m")  # halo (4 words per record), migration (8 words per record)

    def __init__(self, slab_rank, rank: int, nranks: int):
        import torch
        import torch.distributed as dist

        assert nranks >= 2, "the peer-memory data plane needs neighbour ranks (P >= 2)"
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        super().__init__(rank, nranks, dev)
        sr = self.sr = slab_rank
        isz = sr.torch.empty(0, dtype=sr.dtype).element_size()
        nbytes = {"h": (1 + sr.hcap) * 4 * isz, "m": (1 + sr.mcap) * 8 * isz}
        self.words = {"h": 4, "m": 8}
        own, blob = {}, b""
        for k in self.KINDS:                      # receive buffers: [kind][side: from r-1, from r+1][parity]
            for side in (0, 1):
                for par in (0, 1):
                    own[(k, side, par)], h = nc.nc_ipc_alloc(sr.ctx, nbytes[k])
                    blob += h
        self.ev = {}
        for k in self.KINDS:
            for e in ("S", "C"):
                self.ev[(k, e)], h = nc.nc_ipc_event(sr.ctx)
                blob += h
        # handles and the per-exchange barrier on the host (gloo): an NCCL barrier would synchronize the
        # device, which the host-synchronization-free step never does
        self.cpu_group = dist.new_group(backend="gloo") if dist.get_backend() == "nccl" else None
        t = torch.frombuffer(bytearray(blob), dtype=torch.uint8)
        allb = [torch.zeros_like(t) for _ in range(nranks)]
        dist.all_gather(allb, t, group=self.cpu_group)
        allb = [bytes(x.numpy().tobytes()) for x in allb]

        def mem_handle(r, k, side, par):
            i = (self.KINDS.index(k) * 2 + side) * 2 + par
            return allb[r][64 * i:64 * (i + 1)]

        def ev_handle(r, k, e):
            i = 8 + self.KINDS.index(k) * 2 + ("S", "C").index(e)
            return allb[r][64 * i:64 * (i + 1)]

        lo, hi = (rank - 1) % nranks, (rank + 1) % nranks
        # our low message lands in r-1's "from r+1" buffer, our high message in r+1's "from r-1" buffer
        self.send = {k: [[nc.nc_ipc_open(sr.ctx, mem_handle(lo, k, 1, par)),
                          nc.nc_ipc_open(sr.ctx, mem_handle(hi, k, 0, par))] for par in (0, 1)] for k in self.KINDS}
        self.recv = {k: [[own[(k, 0, par)], own[(k, 1, par)]] for par in (0, 1)] for k in self.KINDS}
        peers = [lo] if lo == hi else [lo, hi]
        self.pev = {(k, e): [nc.nc_ipc_event_open(sr.ctx, ev_handle(r, k, e)) for r in peers]
                    for k in self.KINDS for e in ("S", "C")}
        self.par = {k: 0 for k in self.KINDS}
        self._point("h", send_par=0, recv_par=0)
        self._point("m", send_par=0, recv_par=0)

    def _point(self, k, send_par, recv_par):
        """The rank's message pointers: the next packing writes parity send_par of the neighbours'
        buffers, the next reads take parity recv_par of its own."""
        if k == "h":
            self.sr.hsend, self.sr.hrecv = self.send[k][send_par], self.recv[k][recv_par]
        else:
            self.sr.msend, self.sr.mrecv = self.send[k][send_par], self.recv[k][recv_par]

    def _records(self, k):
        ctx = self.sr.ctx
        nc.nc_ipc_record(ctx, self.ev[(k, "C")])  # the reads of the previous messages are queued before
        nc.nc_ipc_record(ctx, self.ev[(k, "S")])  # our messages are in the neighbours' buffers
        self.dist.barrier(group=self.cpu_group)   # every record is issued before any neighbour's wait

    def _waits(self, k):
        ctx = self.sr.ctx
        for i in self.pev[(k, "S")]:   # the neighbours' messages to us have landed
            nc.nc_ipc_wait(ctx, i)
        for i in self.pev[(k, "C")]:   # they are done with the parity our next packing writes
            nc.nc_ipc_wait(ctx, i)
        p = self.par[k]
        self._point(k, send_par=1 - p, recv_par=p)
        self.par[k] = 1 - p

    def exchange_msgs(self, sends, recv_bufs):   # migration: packed by nc_sd_migrate into the neighbours
        self._records("m")
        self._waits("m")

    def start_msgs(self, sends, recv_bufs):      # halo: the interior layers' K3 runs between start and finish
        self._records("h")
        self._pending = "h"

    def finish_msgs(self):
        self._waits(self._pending)


class NcclTransport:
    """The data plane inside libnemdcell.so (nc_slab_exchange*, nc_slab_allgather over NCCL, on the
    library's communication stream): one rank per process, the host only broadcasts rank 0's NCCL
    unique id (torch.distributed, any backend).  A single rank (P = 1) runs the same calls as a self
    ring, which is how it is exercised on one GPU."""

    def __init__(self, slab_rank, group_rank: int, nranks: int):
        self.sr = slab_rank
        self.rank, self.P = group_rank, nranks
        if nranks > 1:
            import torch
            import torch.distributed as dist

            dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
            t = torch.zeros(128, dtype=torch.uint8, device=dev)
            if group_rank == 0:
                t.copy_(torch.frombuffer(bytearray(nc.nc_nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(t, 0)
            uid = bytes(t.cpu().numpy().tobytes())
        else:
            uid = nc.nc_nccl_unique_id()
        nc.nc_slab_comm_init(slab_rank.ctx, group_rank, nranks, uid)

    @staticmethod
    def _words(buf):
        return int(buf.shape[1]) // 4

    def start_msgs(self, sends, recv_bufs):
        (s_lo, s_hi), = sends
        r_lo, r_hi = recv_bufs[0]
        nc.nc_sd_exchange_start(self.sr.ctx, s_lo, s_hi, r_lo, r_hi, int(s_lo.shape[0]) - 1, self._words(s_lo))

    def finish_msgs(self):
        nc.nc_slab_exchange_wait(self.sr.ctx)

    def exchange_msgs(self, sends, recv_bufs):
        self.start_msgs(sends, recv_bufs)
        self.finish_msgs()

    def counts(self, sends):
        """Counts AND the payload launch (the library exchanges the counts, then leaves the payload in
        flight on its communication stream); start() hands the result over, finish() waits."""
        (s_lo, n_lo, s_hi, n_hi), = sends
        b_lo, b_hi = self.sr.hrecv
        m_lo, m_hi = nc.nc_slab_exchange_start(self.sr.ctx, s_lo, n_lo, s_hi, n_hi, b_lo, b_hi, len(b_lo),
                                               self._words(s_lo))
        self._inflight = [(b_lo, m_lo, b_hi, m_hi)]
        return [(m_lo, m_hi)]

    def start(self, sends, recv_bufs, counts):
        return self._inflight

    def finish(self, pending):
        nc.nc_slab_exchange_wait(self.sr.ctx)
        return pending

    def exchange(self, sends, recv_bufs):
        (s_lo, n_lo, s_hi, n_hi), = sends
        b_lo, b_hi = recv_bufs[0]
        m_lo, m_hi = nc.nc_slab_exchange(self.sr.ctx, s_lo, n_lo, s_hi, n_hi, b_lo, b_hi, len(b_lo), self._words(s_lo))
        return [(b_lo, m_lo, b_hi, m_hi)]

    def allgather_tensors(self, per_rank):
        import torch
        import torch.distributed as dist

        if self.P == 1:
            return per_rank[0]
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        return _dist_allgather_tensors(dist, torch, dev, per_rank[0])

    def gather(self, parts):
        part, = parts
        klo, khi, l3 = self.sr.layers()
        rows = -(-l3 // self.P)
        allp = nc.nc_slab_allgather(self.sr.ctx, part, rows, self.P)
        out = [allp[k * rows:k * rows + ((k + 1) * l3 // self.P - k * l3 // self.P)] for k in range(self.P)]
        return np.concatenate(out, axis=0)


# -------------------------------------------------------------------- driver

def own_particles(cl, q_all, rank, nranks):
    """Initial split (not on the timed path): the cell layer of every particle from the library
    (nc_slab_layer_of, the same canonical wrap and layer as its cell keys), in chunks that fit the
    context's capacity -- a small context with the full box suffices; returns the own indices."""
    import torch

    n = len(q_all)
    chunk = max(1, min(int(cl.cfg.capacity), n))
    dev = f"cuda:{cl.device}"
    layer = np.empty(n, dtype=np.int64)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        qc = torch.as_tensor(q_all[lo:hi]).to(dev, dtype=cl.dtype).contiguous().clone()  # wrapped in place
        lc = torch.empty(hi - lo, dtype=torch.int32, device=dev)
        nc.nc_slab_layer_of(cl.ctx, qc, hi - lo, lc)
        layer[lo:hi] = lc.cpu().numpy()
    _, _, l3 = nc.nc_slab_layers(cl.ctx, 0, 1)
    klo, khi = rank * l3 // nranks, (rank + 1) * l3 // nranks
    return np.nonzero((layer >= klo) & (layer < khi))[0]


class SlabSystem:
    """Runs the slab step for the local ranks through a transport (loopback: all
    ranks here; distributed: the one rank of this process)."""

    def __init__(self, ranks, transport):
        self.ranks = ranks
        self.tr = transport
        self.repartitions = 0

    def forces(self, want_uw=True):
        if self._dev():
            return self.forces_dev(want_uw)
        hs = [r.halo() for r in self.ranks]
        if hasattr(self.tr, "start") and all(hasattr(r, "forces_begin") for r in self.ranks):
            # overlapped: counts, then the payload in flight while the interior layers are evaluated
            cnt = self.tr.counts(hs)
            pend = self.tr.start(hs, [r.hrecv for r in self.ranks], cnt)
            for r, (m_lo, m_hi) in zip(self.ranks, cnt):
                r.forces_begin(m_lo, m_hi)
            hr = self.tr.finish(pend)
            parts = [r.forces_end(*h, want_parts=want_uw) for r, h in zip(self.ranks, hr)]
        else:
            hr = self.tr.exchange(hs, [r.hrecv for r in self.ranks])
            parts = [r.forces(*h, want_parts=want_uw) for r, h in zip(self.ranks, hr)]
        if not want_uw:
            return None
        allp = self.tr.gather(parts)
        return self.ranks[0].reduce(allp)

    def flush(self):
        """Apply deferred closing kicks (before the momenta are read)."""
        for r in self.ranks:
            if hasattr(r, "flush"):
                r.flush()

    def repartition(self):
        """After the cell-layer count l3 changed (GKR boxes, DS under general flows): every
        particle goes to the rank owning its layer in the new grid (all-gather, then each rank keeps its
        own).  Rare; results stay bitwise those of one device (cells are rebuilt in (cell, gid) order)."""
        owned = [r.owned() for r in self.ranks]
        q, p, gid, owner = self.tr.allgather_tensors(owned)
        for r in self.ranks:
            m = owner == r.rank
            r.take(q[m], p[m], gid[m])
        self.repartitions += 1

    def _dev(self):
        return all(isinstance(r, SlabRankDev) for r in self.ranks)

    def forces_dev(self, want_uw=True):
        """The force evaluation of the host-synchronization-free step: halo messages in flight while the
        interior layers are evaluated; nothing is read back unless the energies are wanted."""
        hs = [r.halo() for r in self.ranks]
        if all(h is not None for h in hs):
            self.tr.start_msgs(hs, [r.hrecv for r in self.ranks])
        for r in self.ranks:
            r.forces_begin_dev()
        if all(h is not None for h in hs):
            self.tr.finish_msgs()
        parts = [r.forces_end_dev(want_parts=want_uw) for r in self.ranks]
        if not want_uw:
            return None
        allp = self.tr.gather(parts)
        return self.ranks[0].reduce(allp)

    def step(self, dt, want_uw=True):
        if self._dev():
            for r in self.ranks:
                r.kick_drift(dt)
            if any(r.l3_changed() for r in self.ranks):
                self.repartition()
            else:
                sends = [r.migrate() for r in self.ranks]
                self.tr.exchange_msgs(sends, [r.mrecv for r in self.ranks])
                for r in self.ranks:
                    r.absorb_msgs()
            out = self.forces_dev(want_uw)
            for r in self.ranks:
                r.kick(dt)
            return out
        for r in self.ranks:
            r.kick_drift(dt)
        if any(getattr(r, "l3_changed", lambda: False)() for r in self.ranks):
            self.repartition()
        else:
            sends = [r.migrate() for r in self.ranks]
            recvs = self.tr.exchange(sends, [r.recv for r in self.ranks])
            for r, rv in zip(self.ranks, recvs):
                r.absorb(*rv)
        out = self.forces(want_uw)
        for r in self.ranks:
            r.kick(dt)
        return out
