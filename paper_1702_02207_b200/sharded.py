"""Multi-GPU long-chain integration: 1-D domain decomposition + halo exchange.

BASELINE configs[2]: one wall-anchored chain of s cells split into
contiguous shards, one per rank (rank 0 owns the wall, the last rank the free
end).  A step's dependency radius is 2 cells of x and v, so every T steps each
rank refreshes a ghost zone of g = 2T cells on each side from its neighbours
and then advances its own cells T steps with the temporally blocked kernel
(``osc_rk4_chain_advance``).  Every owned cell goes through exactly the
operations it goes through on one GPU, so the result is byte-identical for
any number of ranks -- the GPU form of the reference engine's
"bitwise-identical for every worker count" contract (parallel.py:11-14,
test_parallel.py:259-271).

Two transports:

* ``"nccl"`` (default): per period the interior tiles (which read no ghost
  cell) are launched first, the ghost exchange runs on a side stream (NCCL
  send/recv of 2 x g doubles per neighbour; gloo stages through the host),
  and the two edge tiles are launched after it.
* ``"peer"``: the fused compute + exchange.  Each rank maps its neighbours'
  state buffers (CUDA IPC; NVLink peer memory between GPUs) and the tile
  kernel itself stores its boundary cells into the neighbours' next-input
  ghost zones (``osc_peer_t``), so there is no exchange step at all.  Order is
  kept on the device only: after its period-p launch a rank's stream stores
  p + 1 into its period counter (``osc_stream_write_u64``, fenced after the
  kernel's peer stores), and before period p its stream waits until each
  neighbour's counter reaches p (``osc_stream_wait_u64``) -- the neighbour's
  period p-1 both produced our ghosts and finished reading the buffer we are
  about to write into (ping-pong buffers, parity from the global period
  count).  The waits happen in the GPU front-end: no host barrier per period,
  and no kernel ever waits on another GPU.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import torch
import torch.distributed as dist


def partition(s: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous slice [lo, hi) of s cells for rank."""
    return s * rank // world, s * (rank + 1) // world


@dataclass
class ShardLayout:
    s: int          # global chain length
    lo: int         # first owned global cell
    hi: int         # one past the last owned global cell
    blo: int        # first buffered global cell (incl. left ghosts)
    bhi: int        # one past the last buffered global cell
    g: int          # ghost width = 2 * halo_steps

    @property
    def n(self) -> int:
        return self.bhi - self.blo

    @property
    def own(self) -> tuple[int, int]:
        return self.lo - self.blo, self.hi - self.blo

    @property
    def left_ghost(self) -> int:
        return self.lo - self.blo

    @property
    def right_ghost(self) -> int:
        return self.bhi - self.hi


def layout(s: int, rank: int, world: int, halo_steps: int) -> ShardLayout:
    lo, hi = partition(s, rank, world)
    g = 2 * halo_steps
    if world > 1 and (hi - lo) < g:
        raise ValueError(f"shard of {hi - lo} cells is narrower than the {g}-cell ghost zone")
    return ShardLayout(s, lo, hi, max(0, lo - g), min(s, hi + g), g)


def _cuda_advance(m, C, xin, vin, xout, vout, own_lo, own_hi, dt, nsteps, step0, first_bad,
                  stream=None, left=None, right=None):
    from . import batched

    batched.chain_advance(m, C, xin, vin, xout, vout, own_lo, own_hi, dt, nsteps, step0,
                          first_bad, stream=stream, left=left, right=right)


class ShardedChain:
    """One rank's shard of a chain; ``run`` integrates nsteps with halo exchange.

    ``m, C, x0, v0`` are the GLOBAL arrays (numpy or tensors); each rank
    copies its buffered slice.  ``advance`` defaults to the CUDA kernel; tests
    inject the oracle to check the exchange logic on CPU ranks.
    """

    # interior/edge split: an edge region is at least one tile of owned cells
    EDGE_CELLS = 4096  # >= any tile (K x threads) so interior tiles never slide into ghosts

    def __init__(self, m, C, x0, v0, dt, *, halo_steps=32, group=None, device=None,
                 advance=None, rank=None, world=None, transport="nccl"):
        if transport not in ("nccl", "peer"):
            raise ValueError(f"transport must be 'nccl' or 'peer', got {transport!r}")
        self.transport = transport
        self.group = group
        distributed = rank is None  # rank/world given explicitly: an in-process shard
        if rank is None:
            rank = dist.get_rank(group) if dist.is_initialized() else 0
            world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank, self.world = rank, world
        self.dt = float(dt)
        self.T = int(halo_steps)
        s = len(m)
        self.L = layout(s, self.rank, self.world, self.T)
        self.device = device or (torch.device("cuda", torch.cuda.current_device())
                                 if torch.cuda.is_available() else torch.device("cpu"))
        self.advance = advance or _cuda_advance
        sl = slice(self.L.blo, self.L.bhi)

        def t(a):
            a = a if isinstance(a, torch.Tensor) else torch.as_tensor(a)
            # always a private copy: the caller's arrays are never aliased
            return a[sl].to(device=self.device, dtype=torch.float64, copy=True).contiguous()

        self.m, self.C = t(m), t(C)
        self.x, self.v = t(x0), t(v0)
        self.x2, self.v2 = self.x.clone(), self.v.clone()
        self.first_bad = torch.zeros(1, dtype=torch.int64, device=self.device)
        g = self.L.g
        self.send_l = torch.empty(2, g, dtype=torch.float64, device=self.device)
        self.send_r = torch.empty_like(self.send_l)
        self.recv_l = torch.empty_like(self.send_l)
        self.recv_r = torch.empty_like(self.send_l)
        self.cuda = self.device.type == "cuda"
        self.comm_stream = torch.cuda.Stream(self.device) if self.cuda else None
        self.peer_bufs = {}  # neighbour rank -> ((x, v) of its buffer 0, (x, v) of buffer 1, blo)
        if transport == "peer" and self.world > 1 and dist.is_initialized() and distributed:
            self._setup_peer()

    # -- fused exchange over peer memory --------------------------------------
    def peer_descriptors(self, p):
        """(left, right) osc_peer_t tuples for GLOBAL period p (counted over all
        runs since setup, so the ping-pong parity stays right across runs with
        an odd number of periods): the neighbours' buffer (p+1) % 2 -- the one
        they read next period -- and our cell offsets."""
        g = self.L.g
        out = []
        for nb in (self.rank - 1, self.rank + 1):
            if nb not in self.peer_bufs:
                out.append(None)
                continue
            bufs, nblo = self.peer_bufs[nb]
            x, v = bufs[(p + 1) % 2]
            ptr = lambda t: t if isinstance(t, int) else t.data_ptr()  # noqa: E731
            out.append((ptr(x), ptr(v), self.L.blo - nblo, g))
        return tuple(out)

    def _setup_peer(self):
        """Own state and period counter in exportable allocations; map the
        neighbours' (CUDA IPC: NVLink peer memory between GPUs)."""
        from . import peer

        self.host_group = dist.new_group(backend="gloo")
        self.peer_counters = {}
        n = self.L.n
        self._own = [peer.DeviceVector(n, self.device) for _ in range(4)]
        for dst, src in zip(self._own, (self.x, self.v, self.x2, self.v2)):
            dst.tensor.copy_(src)
        self.x, self.v, self.x2, self.v2 = (b.tensor for b in self._own)
        # period counter: our stream stores p + 1 after our period p; the
        # neighbours' streams wait on it (no host barrier per period)
        self._counter = peer.DeviceVector(1, self.device)
        self._counter.tensor.zero_()
        self._period = 0
        torch.cuda.synchronize(self.device)
        mine = {"blo": self.L.blo, "bufs": [b.handle() for b in self._own],
                "counter": self._counter.handle()}
        infos = [None] * self.world
        dist.all_gather_object(infos, mine, group=self.host_group)
        self._imported = []
        for nb in (self.rank - 1, self.rank + 1):
            if 0 <= nb < self.world:
                ptrs = [peer.import_buffer(h) for h in infos[nb]["bufs"]]
                self._imported += ptrs
                self.peer_bufs[nb] = (((ptrs[0], ptrs[1]), (ptrs[2], ptrs[3])), infos[nb]["blo"])
                self.peer_counters[nb] = peer.import_buffer(infos[nb]["counter"])
                self._imported.append(self.peer_counters[nb])
        # Can this system wait on the mapped counters from a stream?  Try a
        # wait that is already satisfied; every rank adopts host ordering if
        # any rank cannot (all ranks must order periods the same way).
        ok = True
        try:
            probe = torch.cuda.current_stream(self.device)
            for ptr in self.peer_counters.values():
                peer.stream_wait_u64(probe, ptr, 0)
                peer.stream_write_u64(probe, self._counter.ptr, 0)
            torch.cuda.synchronize(self.device)
        except RuntimeError:
            ok = False
        if os.environ.get("OSC_PEER_HOST_ORDER") == "1":  # exercise the fallback
            ok = False
        oks = [None] * self.world
        dist.all_gather_object(oks, ok, group=self.host_group)
        self._host_order = not all(oks)

    def close(self):
        """Release peer resources in a safe order: finish local work, unmap the
        neighbours' buffers and counters, wait until every rank has done so,
        then free the allocations this rank exported."""
        if not getattr(self, "_own", None):
            return
        from . import peer

        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.host_group)  # no rank still writes into anyone
        for ptr in self._imported:
            peer.close_buffer(ptr)
        self._imported, self.peer_counters = [], {}
        self.peer_bufs.clear()
        dist.barrier(group=self.host_group)  # every mapping of our memory is gone
        # keep the results readable: move them to ordinary tensors first
        self.x, self.v, self.x2, self.v2 = (t.clone() for t in (self.x, self.v, self.x2,
                                                                 self.v2))
        torch.cuda.synchronize(self.device)
        for b in self._own:
            b.free()
        self._counter.free()
        self._own = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _run_peer(self, nsteps):
        """Fused exchange, ordered on the device: before period q (a running
        count over runs) our stream waits until each neighbour's counter shows
        its period q-1 done -- it produced our ghosts and finished reading the
        buffer we now store into (ping-pong) -- and after our launch it stores
        q + 1 into our counter.  The waits happen in the GPU front-end; no
        kernel ever spins on another GPU and no host barrier is needed."""
        from . import peer

        main = torch.cuda.current_stream(self.device)
        a, b = self.L.own
        k = 0
        while k < nsteps:
            n = min(self.T, nsteps - k)
            q = self._period
            self._order_before(main, q)
            left, right = self.peer_descriptors(q)
            self.advance(self.m, self.C, self.x, self.v, self.x2, self.v2, a, b, self.dt, n, k,
                         self.first_bad, left=left, right=right)
            self._order_after(main, q)
            self.x, self.x2 = self.x2, self.x
            self.v, self.v2 = self.v2, self.v
            self._period += 1
            k += n
        # neighbours' final writes land only in ghost zones; our owned cells are
        # complete on our stream.  Make sure no peer kernel still targets us.
        self._order_before(main, self._period)

    # Period ordering: stream counters when every rank's system takes stream
    # memory operations on the mapped counters (decided together at setup),
    # else host ordering -- finish our period, then a host barrier: slower,
    # equally correct.
    def _order_before(self, main, q):
        from . import peer

        if not self._host_order:
            for ptr in self.peer_counters.values():
                peer.stream_wait_u64(main, ptr, q)

    def _order_after(self, main, q):
        from . import peer

        if self._host_order:
            torch.cuda.synchronize(self.device)  # our period (and its peer stores) done
            dist.barrier(group=self.host_group)
        else:
            peer.stream_write_u64(main, self._counter.ptr, q + 1)

    # -- ghost exchange ------------------------------------------------------
    def boundary(self, x, v):
        """Owned boundary cells to ship: (left [2][g], right [2][g])."""
        a, b = self.L.own
        g = self.L.g
        self.send_l[0].copy_(x[a:a + g])
        self.send_l[1].copy_(v[a:a + g])
        self.send_r[0].copy_(x[b - g:b])
        self.send_r[1].copy_(v[b - g:b])
        return self.send_l, self.send_r

    def fill_ghosts(self, x, v, from_left=None, from_right=None):
        a, b = self.L.own
        g = self.L.g
        if from_left is not None:
            x[a - g:a].copy_(from_left[0])
            v[a - g:a].copy_(from_left[1])
        if from_right is not None:
            x[b:b + g].copy_(from_right[0])
            v[b:b + g].copy_(from_right[1])

    def _exchange(self, x, v):
        """Refresh both ghost zones of (x, v) from the neighbours' owned cells."""
        self.boundary(x, v)
        left = self.rank - 1 if self.rank > 0 else None
        right = self.rank + 1 if self.rank < self.world - 1 else None
        # NCCL moves device buffers directly; other backends (gloo) stage
        # through host memory.
        stage = self.cuda and dist.get_backend(self.group) != "nccl"
        bufs = (self.send_l, self.recv_l, self.send_r, self.recv_r)
        if stage:
            bufs = tuple(b.cpu() for b in bufs)
        send_l, recv_l, send_r, recv_r = bufs
        ops = []
        if left is not None:
            ops.append(dist.P2POp(dist.isend, send_l, left, self.group))
            ops.append(dist.P2POp(dist.irecv, recv_l, left, self.group))
        if right is not None:
            ops.append(dist.P2POp(dist.isend, send_r, right, self.group))
            ops.append(dist.P2POp(dist.irecv, recv_r, right, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if stage:
            self.recv_l.copy_(recv_l)
            self.recv_r.copy_(recv_r)
        self.fill_ghosts(x, v, self.recv_l if left is not None else None,
                         self.recv_r if right is not None else None)

    def _advance(self, xin, vin, xout, vout, lo, hi, n, step0, stream=None):
        if hi > lo:
            kw = {"stream": stream} if self.cuda else {}
            self.advance(self.m, self.C, xin, vin, xout, vout, lo, hi, self.dt, n, step0,
                         self.first_bad, **kw)

    # -- one period of T steps, in three phases ------------------------------
    def _split(self):
        a, b = self.L.own
        return self.nranks > 1 and (b - a) > 2 * self.EDGE_CELLS + 2 * self.L.g

    def phase_interior(self, n, k):
        """Launch the tiles that read no ghost cell (all of them if unsplit)."""
        a, b = self.L.own
        E = self.EDGE_CELLS
        if self.nranks == 1:
            self._advance(self.x, self.v, self.x2, self.v2, a, b, n, k)
        elif self._split():
            self._advance(self.x, self.v, self.x2, self.v2, a + E, b - E, n, k)

    def phase_edges(self, n, k):
        """After the ghost exchange: the tiles next to the ghost zones."""
        a, b = self.L.own
        E = self.EDGE_CELLS
        if self.nranks == 1:
            pass
        elif self._split():
            self._advance(self.x, self.v, self.x2, self.v2, a, a + E, n, k)
            self._advance(self.x, self.v, self.x2, self.v2, b - E, b, n, k)
        else:
            self._advance(self.x, self.v, self.x2, self.v2, a, b, n, k)
        self.x, self.x2 = self.x2, self.x
        self.v, self.v2 = self.v2, self.v

    @property
    def nranks(self):
        return self.world

    def run(self, nsteps: int):
        """Advance the shard nsteps steps; returns the 1-based first bad step
        of the WHOLE chain (min over ranks) or 0."""
        if self.transport == "peer" and self.world > 1 and self.peer_bufs:
            self._run_peer(nsteps)
            return self._reduce_first_bad()
        k = 0
        while k < nsteps:
            n = min(self.T, nsteps - k)
            if self.world > 1 and self.cuda:
                # The exchange needs only the previous period's output, not the
                # interior tiles: it waits on an event recorded BEFORE they are
                # enqueued, so it overlaps them (interior tiles read owned cells
                # only; the exchange reads boundary cells and writes ghosts).
                main = torch.cuda.current_stream(self.device)
                ready = torch.cuda.Event()
                ready.record(main)
                self.phase_interior(n, k)
                self.comm_stream.wait_event(ready)
                with torch.cuda.stream(self.comm_stream):
                    self._exchange(self.x, self.v)
                main.wait_stream(self.comm_stream)
            else:
                self.phase_interior(n, k)
                if self.world > 1:
                    self._exchange(self.x, self.v)
            self.phase_edges(n, k)
            k += n
        return self._reduce_first_bad()

    def _reduce_first_bad(self) -> int:
        fb = self.first_bad.clone()
        if self.world > 1:
            big = torch.iinfo(torch.int64).max
            fb = torch.where(fb > 0, fb, torch.full_like(fb, big))
            dist.all_reduce(fb, op=dist.ReduceOp.MIN, group=self.group)
            fb = torch.where(fb == big, torch.zeros_like(fb), fb)
        return int(fb.item())

    def owned(self):
        """(x, v) of the owned cells (views)."""
        a, b = self.L.own
        return self.x[a:b], self.v[a:b]

    def gather(self):
        """Full chain state on every rank (validation only)."""
        x, v = self.owned()
        if self.world == 1:
            return x.clone(), v.clone()
        parts_x = [None] * self.world
        parts_v = [None] * self.world
        dist.all_gather_object(parts_x, x.cpu(), group=self.group)
        dist.all_gather_object(parts_v, v.cpu(), group=self.group)
        return torch.cat(parts_x), torch.cat(parts_v)


class LocalShardGroup:
    """All shards of a chain in ONE process, advanced in lockstep.

    Same per-shard kernels, layouts and interior/edge phases as the
    multi-process path, with the ghost exchange done by device copies.  Used to
    test the decomposition on a single GPU (no kernel ever waits on another, so
    this is safe to run with several shards on one device).
    """

    def __init__(self, m, C, x0, v0, dt, shards: int, *, halo_steps=32, device=None,
                 advance=None, transport="nccl"):
        self.transport = transport
        self.parts = [ShardedChain(m, C, x0, v0, dt, halo_steps=halo_steps, device=device,
                                   advance=advance, rank=r, world=shards)
                      for r in range(shards)]
        self._period = 0
        if transport == "peer":  # neighbours' buffers are plain local tensors here
            for r, p in enumerate(self.parts):
                for nb in (r - 1, r + 1):
                    if 0 <= nb < shards:
                        q = self.parts[nb]
                        p.peer_bufs[nb] = (((q.x, q.v), (q.x2, q.v2)), q.L.blo)

    def _run_peer(self, nsteps):
        """Fused exchange, all shards on one stream: stream order is the only
        synchronisation needed."""
        T = self.parts[0].T
        k = 0
        while k < nsteps:
            n = min(T, nsteps - k)
            p = self._period  # global: the ping-pong parity carries over runs
            for sh in self.parts:
                a, b = sh.L.own
                left, right = sh.peer_descriptors(p)
                sh.advance(sh.m, sh.C, sh.x, sh.v, sh.x2, sh.v2, a, b, sh.dt, n, k,
                           sh.first_bad, left=left, right=right)
            for sh in self.parts:
                sh.x, sh.x2 = sh.x2, sh.x
                sh.v, sh.v2 = sh.v2, sh.v
            k += n
            self._period += 1

    def run(self, nsteps: int) -> int:
        if self.transport == "peer":
            self._run_peer(nsteps)
            bad = [int(p.first_bad.item()) for p in self.parts if int(p.first_bad.item()) > 0]
            return min(bad) if bad else 0
        T = self.parts[0].T
        k = 0
        while k < nsteps:
            n = min(T, nsteps - k)
            for p in self.parts:
                p.phase_interior(n, k)
            sends = [tuple(t.clone() for t in p.boundary(p.x, p.v)) for p in self.parts]
            for r, p in enumerate(self.parts):
                left = sends[r - 1][1] if r > 0 else None
                right = sends[r + 1][0] if r + 1 < len(self.parts) else None
                p.fill_ghosts(p.x, p.v, left, right)
            for p in self.parts:
                p.phase_edges(n, k)
            k += n
        bad = [int(p.first_bad.item()) for p in self.parts]
        bad = [b for b in bad if b > 0]
        return min(bad) if bad else 0

    def gather(self):
        xs, vs = zip(*(p.owned() for p in self.parts))
        return torch.cat(xs), torch.cat(vs)
