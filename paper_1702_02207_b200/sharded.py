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
  ghost zones (``osc_peer_t``), so there is no exchange step at all.  Order
  is kept on the device, per edge tile (``osc_edge_sync_t``): only the tiles
  next to a ghost zone depend on a neighbour, so each period's launch runs
  its interior tiles first, and an edge tile's CTA waits -- bounded, in the
  kernel -- until the neighbour's edge counter shows that the neighbour's
  previous period stored our ghosts and finished reading the buffer we store
  into (ping-pong buffers, parity from the global period count); the last
  edge tile of a side then posts our counter.  One launch per period, no
  stream-level wait, no host barrier.  A neighbour that stops making
  progress turns into a timeout record (``OSC_PEER_TIMEOUT_MS``, default
  30 s): the launch drains and ``run`` raises :class:`PeerTimeoutError`
  naming the rank, the period, the side and the counter value seen --
  instead of hanging (the reference guards its barrier the same way,
  parallel.py:205-255).
"""

from __future__ import annotations

import json
import os
import time
from dataclasses import dataclass

import torch
import torch.distributed as dist


class PeerTimeoutError(RuntimeError):
    """A neighbour's edge counter did not reach the awaited period in time
    (the fused exchange's bounded wait, osc_edge_sync_t)."""

    def __init__(self, rank, period, side, seen, trace):
        self.rank, self.period, self.side, self.seen = rank, period, side, seen
        self.trace = trace
        nb = rank - 1 if side == 0 else rank + 1
        super().__init__(
            f"rank {rank}: period {period} waited for rank {nb}'s "
            f"{'right' if side == 0 else 'left'} edge counter to reach {period}, saw {seen} "
            f"(last phases: {trace[-6:]})")


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
                  stream=None, left=None, right=None, sync=None, tiles=None, div2=None):
    from . import batched

    # the shard's parameters were validated once at construction
    batched.chain_advance(m, C, xin, vin, xout, vout, own_lo, own_hi, dt, nsteps, step0,
                          first_bad, stream=stream, left=left, right=right, trusted=True,
                          sync=sync, tiles=tiles, div2=div2)


class ShardedChain:
    """One rank's shard of a chain; ``run`` integrates nsteps with halo exchange.

    ``m, C, x0, v0`` are the GLOBAL arrays (numpy or tensors); each rank
    copies its buffered slice.  ``advance`` defaults to the CUDA kernel; tests
    inject the oracle to check the exchange logic on CPU ranks.
    """

    def __init__(self, m, C, x0, v0, dt, *, halo_steps=32, group=None, device=None,
                 advance=None, rank=None, world=None, transport="nccl", timeout_ms=None):
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
        self._t0 = time.monotonic()
        self.trace = []
        if timeout_ms is None:
            timeout_ms = float(os.environ.get("OSC_PEER_TIMEOUT_MS", "30000"))
        self.timeout_ns = int(timeout_ms * 1e6)
        self.div2 = None  # the shard's two-operation division table (CUDA advance only)
        if self.cuda and self.advance is _cuda_advance:
            self._validate(distributed)
            from . import batched

            self.div2 = batched.div2_table(self.m)
        if transport == "peer" and self.world > 1 and dist.is_initialized() and distributed:
            self._setup_peer()

    def _validate(self, distributed):
        """The parameter rule (oscillator.py:66-80) once, over the whole chain:
        each rank checks its buffer on the device (osc_validate_parameters),
        the ranks agree on the first offender (min over ranks of the global
        index; masses before springs), and every rank raises the same
        NonPositiveParameterError -- no rank is left waiting in a collective.
        Per-period launches then skip the check (OSC_TRUSTED)."""
        from . import _native, batched
        from .oscillator import NonPositiveParameterError

        big = 1 << 62
        found = [big, big]  # masses, springs (global cell index)
        try:
            batched.validate_parameters(self.m, self.C)
        except NonPositiveParameterError:
            which, idx = _native.last_invalid_parameter()
            found[which] = self.L.blo + idx
        if distributed and self.world > 1:
            t = torch.tensor(found, dtype=torch.int64)
            group = getattr(self, "host_group", None) or self.group
            if dist.get_backend(group) == "nccl":
                t = t.to(self.device)
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
            found = [int(u) for u in t.cpu()]
        for which, label in ((0, "masses"), (1, "springs")):
            if found[which] < big:
                raise NonPositiveParameterError(
                    f"{label}[{found[which]}]: must be positive and finite")

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
        """Own state and edge counters in exportable allocations; map the
        neighbours' (CUDA IPC: NVLink peer memory between GPUs)."""
        from . import peer

        self._phase("peer-setup")
        self.host_group = dist.new_group(backend="gloo")
        n = self.L.n
        self._own = [peer.DeviceVector(n, self.device) for _ in range(4)]
        for dst, src in zip(self._own, (self.x, self.v, self.x2, self.v2)):
            dst.tensor.copy_(src)
        self.x, self.v, self.x2, self.v2 = (b.tensor for b in self._own)
        # edge counters (osc_edge_sync_t.counters): [0]/[1] our left/right
        # edge done through period q, [2]/[3] tallies, [4..7] timeout record
        self._counters = peer.DeviceVector(8, self.device)
        self._counters.tensor.zero_()
        self._period = 0
        torch.cuda.synchronize(self.device)
        mine = {"blo": self.L.blo, "bufs": [b.handle() for b in self._own],
                "counters": self._counters.handle()}
        infos = [None] * self.world
        dist.all_gather_object(infos, mine, group=self.host_group)
        self._imported = []
        self._ready = [None, None]  # the neighbours' counters facing us
        for side, nb in enumerate((self.rank - 1, self.rank + 1)):
            if 0 <= nb < self.world:
                ptrs = [peer.import_buffer(h) for h in infos[nb]["bufs"]]
                ctr = peer.import_buffer(infos[nb]["counters"])
                self._imported += ptrs + [ctr]
                self.peer_bufs[nb] = (((ptrs[0], ptrs[1]), (ptrs[2], ptrs[3])), infos[nb]["blo"])
                # the left neighbour's RIGHT edge counter ([1]) and vice versa
                self._ready[side] = ctr + 8 * (1 - side)
        self._host_order = os.environ.get("OSC_PEER_HOST_ORDER") == "1"
        self._shard_desc = None
        self.host_s_per_period = None
        self._phase("peer-ready")

    def _phase(self, name, period=None):
        """Per-phase host timestamps (kept for the error report; dumped to
        $OSC_PEER_TRACE/rank<r>.json at close when set)."""
        self.trace.append((round(time.monotonic() - self._t0, 6), name, period))

    def close(self):
        """Release peer resources in a safe order: finish local work, unmap the
        neighbours' buffers and counters, wait until every rank has done so,
        then free the allocations this rank exported."""
        if not getattr(self, "_own", None):
            return
        torch.cuda.synchronize(self.device)
        self._phase("close")
        dist.barrier(group=self.host_group)  # no rank still writes into anyone
        self._release_peer()

    def _release_peer(self):
        from . import peer

        for ptr in self._imported:
            peer.close_buffer(ptr)
        self._imported = []
        self.peer_bufs.clear()
        dist.barrier(group=self.host_group)  # every mapping of our memory is gone
        # keep the results readable: move them to ordinary tensors first
        self.x, self.v, self.x2, self.v2 = (t.clone() for t in (self.x, self.v, self.x2,
                                                                 self.v2))
        torch.cuda.synchronize(self.device)
        for b in self._own:
            b.free()
        self._counters.free()
        self._own = []
        path = os.environ.get("OSC_PEER_TRACE")
        if path:
            os.makedirs(path, exist_ok=True)
            with open(os.path.join(path, f"rank{self.rank}.json"), "w") as f:
                json.dump(self.trace, f)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _run_peer(self, nsteps):
        """Fused exchange, one launch per period, ordered on the device: each
        launch's edge tiles wait (bounded) for the neighbours' edge counters
        to reach the global period q (a running count over runs, so the
        ping-pong parity carries across runs) and post ours when done.  With
        OSC_PEER_HOST_ORDER=1 the periods are ordered on the host instead
        (finish, host barrier): slower, same bytes."""
        a, b = self.L.own
        k = 0
        self._phase("run", self._period)
        if not self._host_order and self.advance is _cuda_advance:
            # the whole period loop in native code (osc_rk4_shard_run)
            t = time.perf_counter()
            periods = self._native_run(nsteps)
            self.host_s_per_period = (time.perf_counter() - t) / max(periods, 1)
            k = nsteps
        while k < nsteps:
            n = min(self.T, nsteps - k)
            q = self._period
            left, right = self.peer_descriptors(q)
            sync = None
            if not self._host_order:
                sync = (self._ready[0], self._ready[1], self._counters.ptr, q, self.timeout_ns)
            kw = {"div2": self.div2} if self.div2 is not None else {}
            self.advance(self.m, self.C, self.x, self.v, self.x2, self.v2, a, b, self.dt, n, k,
                         self.first_bad, left=left, right=right, sync=sync, **kw)
            if self._host_order:
                torch.cuda.synchronize(self.device)  # our period (and its peer stores) done
                dist.barrier(group=self.host_group)
            self.x, self.x2 = self.x2, self.x
            self.v, self.v2 = self.v2, self.v
            self._period += 1
            k += n
        self._phase("enqueued", self._period)
        self._check_sync()

    def _native_run(self, nsteps) -> int:
        """Enqueue every period of this run with one C call; returns the
        number of periods.  Buffer b of ours is (x, v) when the global
        period is even, (x2, v2) when odd -- the parity the Python loop
        keeps by swapping."""
        import ctypes

        from . import _native

        lib = _native.lib()
        own = self._own  # buffer 0 = _own[0:2], buffer 1 = _own[2:4]
        sh = self._shard_desc
        if sh is None:
            sh = self._shard_desc = _native.Shard()
            sh.m, sh.C = self.m.data_ptr(), self.C.data_ptr()
            for bidx in range(2):
                sh.x[bidx], sh.v[bidx] = own[2 * bidx].ptr, own[2 * bidx + 1].ptr
            for side, nb in enumerate((self.rank - 1, self.rank + 1)):
                if nb in self.peer_bufs:
                    bufs, nblo = self.peer_bufs[nb]
                    for bidx in range(2):
                        sh.nx[side][bidx], sh.nv[side][bidx] = bufs[bidx]
                    sh.offset[side] = self.L.blo - nblo
            sh.n = self.L.n
            sh.own_lo, sh.own_hi = self.L.own
            sh.ghost = self.L.g
            sh.first_bad = self.first_bad.data_ptr()
            sh.sync.ready[0] = self._ready[0]
            sh.sync.ready[1] = self._ready[1]
            sh.sync.counters = self._counters.ptr
            sh.sync.timeout_ns = self.timeout_ns
            sh.div2 = self.div2.data_ptr() if self.div2 is not None else None
        sh.sync.period = self._period
        # the state must be in buffer period % 2 (the Python loop's swaps keep
        # self.x on the current buffer; the native loop relies on parity)
        cur = own[2 * (self._period % 2)].ptr
        assert self.x.data_ptr() == cur, "shard state is not in buffer period % 2"
        rc = lib.osc_rk4_shard_run(ctypes.byref(sh), self.dt, int(nsteps), self.T, 0, 0,
                                   ctypes.c_void_p(torch.cuda.current_stream(self.device)
                                                   .cuda_stream))
        if rc != _native.OSC_OK:
            raise RuntimeError(f"osc_rk4_shard_run: {_native.last_error()}")
        periods = int(sh.sync.period) - self._period
        if periods % 2:
            self.x, self.x2 = self.x2, self.x
            self.v, self.v2 = self.v2, self.v
        self._period = int(sh.sync.period)
        return periods

    def _check_sync(self):
        """Finish our launches and read the timeout record: a wait that
        expired raises PeerTimeoutError here, before any collective (a stuck
        neighbour could not join one)."""
        from . import peer

        rec = peer.edge_sync_status(self._counters.ptr, torch.cuda.current_stream(self.device))
        self._phase("synced", self._period)
        if rec is not None:
            period, side, seen = rec
            raise PeerTimeoutError(self.rank, period, side, seen, list(self.trace))

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

    def _advance(self, n, step0, tiles=None, stream=None):
        """One launch over the owned range; ``tiles`` = "interior" / "edges"
        selects a subset of the same tile geometry (OSC_TILES_*), so the two
        subset launches of a period equal one whole launch byte for byte."""
        a, b = self.L.own
        kw = {"stream": stream} if self.cuda else {}
        if tiles is not None:
            kw["tiles"] = tiles
        if self.div2 is not None:
            kw["div2"] = self.div2
        self.advance(self.m, self.C, self.x, self.v, self.x2, self.v2, a, b, self.dt, n, step0,
                     self.first_bad, **kw)

    # -- one period of T steps -------------------------------------------------
    def phase_interior(self, n, k):
        """Launch the tiles that read no ghost cell (all of them on one rank)."""
        self._advance(n, k, tiles=None if self.world == 1 else "interior")

    def phase_edges(self, n, k, stream=None):
        """After the ghost exchange: ONE launch covering the tiles next to both
        ghost zones (the same tile geometry as the interior launch)."""
        if self.world > 1:
            self._advance(n, k, tiles="edges", stream=stream)

    def _swap(self):
        self.x, self.x2 = self.x2, self.x
        self.v, self.v2 = self.v2, self.v

    @property
    def nranks(self):
        return self.world

    def run(self, nsteps: int):
        """Advance the shard nsteps steps; returns the 1-based first bad step
        of the WHOLE chain (min over ranks) or 0.

        NCCL transport, per period: the interior launch goes on the main
        stream; the ghost exchange (NCCL P2P of 2 x g doubles per neighbour)
        and then one launch covering both edges go on a side stream that
        waited for the previous period only, so exchange and edge tiles run
        concurrently with the interior and its tail; the main stream waits
        for the edges before the next period."""
        if self.transport == "peer" and self.world > 1 and self.peer_bufs:
            self._run_peer(nsteps)
            return self._reduce_first_bad()
        if self._native_nccl():
            self._run_nccl_native(nsteps)
            return self._reduce_first_bad()
        k = 0
        t_host = time.perf_counter()
        periods = 0
        while k < nsteps:
            n = min(self.T, nsteps - k)
            if self.world > 1 and self.cuda:
                main = torch.cuda.current_stream(self.device)
                ready = torch.cuda.Event()
                ready.record(main)  # the previous period's output is complete
                self.phase_interior(n, k)
                self.comm_stream.wait_event(ready)
                with torch.cuda.stream(self.comm_stream):
                    self._exchange(self.x, self.v)
                    self.phase_edges(n, k, stream=self.comm_stream)
                main.wait_stream(self.comm_stream)
            else:
                self.phase_interior(n, k)
                if self.world > 1:
                    self._exchange(self.x, self.v)
                    self.phase_edges(n, k)
            self._swap()
            k += n
            periods += 1
        self.host_s_per_period = (time.perf_counter() - t_host) / max(periods, 1)
        return self._reduce_first_bad()

    def _native_nccl(self) -> bool:
        """The NCCL transport's period loop runs in native code
        (osc_rk4_shard_run_nccl) when the group is an NCCL group and the
        shard advances with the CUDA kernel; OSC_NCCL_PY=1 keeps the Python
        loop below (same schedule, same bytes)."""
        return (self.world > 1 and self.cuda and self.transport == "nccl"
                and self.advance is _cuda_advance and dist.is_initialized()
                and dist.get_backend(self.group) == "nccl"
                and os.environ.get("OSC_NCCL_PY") != "1")

    def _run_nccl_native(self, nsteps):
        """One C call enqueues every period: interior tiles on the current
        stream, the NCCL ghost refresh and the edge tiles on a side stream."""
        import ctypes

        from . import _native

        group = self.group or dist.distributed_c10d._get_default_group()
        comm = group._get_backend(self.device)._comm_ptr()
        sh = _native.Shard()
        sh.m, sh.C = self.m.data_ptr(), self.C.data_ptr()
        sh.x[0], sh.x[1] = self.x.data_ptr(), self.x2.data_ptr()
        sh.v[0], sh.v[1] = self.v.data_ptr(), self.v2.data_ptr()
        sh.n = self.L.n
        sh.own_lo, sh.own_hi = self.L.own
        sh.ghost = self.L.g
        sh.first_bad = self.first_bad.data_ptr()
        sh.div2 = self.div2.data_ptr() if self.div2 is not None else None
        sh.sync.period = 0  # buffer 0 = (x, v), the current state
        t = time.perf_counter()
        rc = _native.lib().osc_rk4_shard_run_nccl(
            ctypes.byref(sh), ctypes.c_void_p(comm), self.rank, self.world, self.dt,
            int(nsteps), self.T, 0, 0,
            ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))
        if rc != _native.OSC_OK:
            raise RuntimeError(f"osc_rk4_shard_run_nccl: {_native.last_error()}")
        periods = int(sh.sync.period)
        self.host_s_per_period = (time.perf_counter() - t) / max(periods, 1)
        if periods % 2:
            self._swap()

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
                kw = {"div2": sh.div2} if sh.div2 is not None else {}
                sh.advance(sh.m, sh.C, sh.x, sh.v, sh.x2, sh.v2, a, b, sh.dt, n, k,
                           sh.first_bad, left=left, right=right, **kw)
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
                p._swap()
            k += n
        bad = [int(p.first_bad.item()) for p in self.parts]
        bad = [b for b in bad if b > 0]
        return min(bad) if bad else 0

    def gather(self):
        xs, vs = zip(*(p.owned() for p in self.parts))
        return torch.cat(xs), torch.cat(vs)
