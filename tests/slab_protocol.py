"""TEST INFRASTRUCTURE: a host-driven slab protocol over the LOW-LEVEL slab
calls of include/rd.h (rd_create_slab, rd_row_ptr, rd_step_begin/finish,
RD_BLOCK_PUSH, rd_checkpoint/restore, rd_read_flags), kept to test those
building blocks. The product's multi-GPU path is rd_create_dist, which runs
the same decomposition inside librd (paper_1901_06535_b200.dist.DistSim).

Row-slab domain decomposition across GPUs.

Rank r of G owns global rows [r*H/G, (r+1)*H/G) and all W columns, with
`halo` ghost rows above and below (halo >= temporal-blocking depth k). After
every rd_step(k) (k <= halo) the slab edges are exchanged with rank +-1:
the owned top `halo` rows of u and v go to rank-1's bottom ghosts, the owned
bottom rows to rank+1's top ghosts. Global top/bottom edges use the no-flux
clamp inside the kernel, so the decomposition is bitwise invisible: the
G-slab result equals the single-grid result (tests/test_dist_*).

torch.distributed is the plumbing (process group; NCCL on B200, gloo in the
CPU tests); the data path is device-to-device send/recv of contiguous row
blocks straight out of the engine's planes. Inputs are generated in global
coordinates (rdinputs), so they do not depend on G.
"""
from __future__ import annotations

import numpy as np

from paper_1901_06535_b200 import (RD_ENONFINITE, RDError, rd_checkpoint, rd_create_slab, rd_destroy,
                                   rd_get_stats, rd_probe_latch)
from paper_1901_06535_b200 import (rd_probe_result, rd_read_fields, rd_read_flags, rd_restore, rd_row_ptr,
                                   rd_set_stream, rd_step)
from paper_1901_06535_b200 import (RD_BLOCK_PUSH, rd_flag_ptr, rd_ipc_export, rd_ipc_map, rd_plane_origins,
                                   rd_push_ghosts, rd_set_peer)
from paper_1901_06535_b200 import (rd_step_begin, rd_step_finish, rd_step_unchecked, rd_stimulate,
                                   rd_stream_signal, rd_stream_wait)
from paper_1901_06535_b200 import rd_write_fields
from paper_1901_06535_b200.dist import exchange_plan, ghost_extent, slab_rows  # noqa: F401


def exchange_post(tensors_by_peer, group=None):
    """Post one halo exchange: tensors_by_peer = [(peer, [send...], [recv...])],
    all sends/recvs as one batch (an NCCL group). With NCCL, device rows go
    GPU to GPU over NVLink on NCCL's stream, ordered after the work already
    queued on the current stream; with a CPU backend (gloo: tests) device rows
    are staged through host tensors. Returns the pending exchange."""
    import torch
    import torch.distributed as dist
    staged = dist.get_backend(group) != "nccl" and any(
        t.is_cuda for _, ss, rs in tensors_by_peer for t in list(ss) + list(rs))
    landing = []
    ops = []
    for peer, sends, recvs in tensors_by_peer:
        for s in sends:
            ops.append(dist.P2POp(dist.isend, s.cpu() if staged else s, peer, group))
        for r in recvs:
            buf = torch.empty(r.shape, dtype=r.dtype) if staged else r
            if staged:
                landing.append((buf, r))
            ops.append(dist.P2POp(dist.irecv, buf, peer, group))
    works = dist.batch_isend_irecv(ops) if ops else []
    return works, landing


def exchange_wait(pending):
    """Complete a posted exchange: the current stream waits for it (NCCL), or
    the staged rows land on the device (gloo)."""
    works, landing = pending
    for w in works:
        w.wait()
    for buf, r in landing:
        r.copy_(buf)


def exchange(tensors_by_peer, group=None):
    """One halo exchange, posted and completed."""
    exchange_wait(exchange_post(tensors_by_peer, group))


class _DevRows:
    """A contiguous device byte range as a __cuda_array_interface__ object."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


def _dev_rows(h, b: int, plane: int, r0: int, r1: int, cache=None):
    """Rows [r0, r1) of plane (0 = u, 1 = v) of instance b in the handle's
    current buffer, as a uint8 CUDA tensor view (cached by device address:
    the buffers alternate, so a slab reuses two sets of views)."""
    import torch
    ptr, pitch = rd_row_ptr(h, b, plane, r0)
    key = (ptr, pitch * (r1 - r0))
    if cache is not None and key in cache:
        return cache[key]
    t = torch.as_tensor(_DevRows(ptr, pitch * (r1 - r0)), device="cuda")
    if cache is not None:
        cache[key] = t
    return t


class SlabSim:
    """One rank's slab of a (batch of) grid(s), stepped with halo exchanges.

    transport: "dist" (torch.distributed process group) or a LoopbackGroup
    shared by several SlabSims on one device (virtual ranks for testing).
    """

    def __init__(self, W: int, H: int, rank: int, world: int, phi_fn, *, dtype=np.float32, halo: int = 4,
                 tb_depth: int = 0, batch: int = 1, transport="dist", group=None, params=None, flags: int = 0,
                 p2p: bool = False):
        self.W, self.H, self.rank, self.world, self.halo = W, H, rank, world, halo
        self.row0, self.rows = slab_rows(H, world, rank)
        if self.rows < halo and world > 1:
            raise ValueError("slab thinner than the halo")
        lo, hi = ghost_extent(H, self.row0, self.rows, halo)
        # phi_fn(b, row0, rows) -> host rows, or None: phi = 0 (paint on the device)
        phi = (None if phi_fn is None else
               np.stack([np.ascontiguousarray(phi_fn(b, lo, hi - lo), dtype=dtype) for b in range(batch)]))
        self.dtype = np.dtype(dtype)
        self.batch = batch
        self.h = rd_create_slab(W, self.rows, phi, self.row0, H, halo, batch=batch, dtype=dtype,
                                tb_depth=tb_depth or halo, flags=flags, params=params)
        self.transport = transport
        self.group = group
        self.plan = exchange_plan(world, rank, self.rows, halo)
        self.p2p = bool(p2p) and world > 1
        self.epoch = 0  # pushes done (peer-memory exchange): the neighbours count the same
        if not isinstance(transport, str):
            transport.register(self)
        else:
            import torch
            # NCCL work is ordered against torch's current stream: issue the
            # engine's kernels on that stream too.
            self.set_stream(torch.cuda.current_stream())
            if self.p2p:
                self._wire_peers()

    # ---- peer-memory exchange across GPUs (opt-in) ----
    # Each rank exports its plane allocation (CUDA IPC), maps its neighbours',
    # and registers their plane origins (rd_set_peer): a block's edge launch
    # then stores the send rows straight into the neighbours' ghost rows.
    # Ranks are ordered by stream-ordered counters in the same allocations:
    # after a push a rank adds one to each neighbour's word (rd_stream_signal);
    # before using ghost rows it waits for its own words (rd_stream_wait).
    # Not exercised on a one-GPU box (ranks must not wait on one another on a
    # shared GPU); LoopbackGroup(p2p=True) tests the same data path in one
    # process.
    def _wire_peers(self):
        import torch.distributed as dist
        handle, base = rd_ipc_export(self.h)
        (u0, u1), (v0, v1), stride = rd_plane_origins(self.h)
        mine = dict(handle=handle, base=base, u=(u0, u1), v=(v0, v1), stride=stride, rows=self.rows,
                    flags=(rd_flag_ptr(self.h, 0), rd_flag_ptr(self.h, 1)))
        every = [None] * self.world
        dist.all_gather_object(every, mine, group=self.group)
        self.peer_flags = {}
        for side, peer in ((0, self.rank - 1), (1, self.rank + 1)):
            if not 0 <= peer < self.world:
                continue
            d = every[peer]
            mapped = rd_ipc_map(self.h, d["handle"])
            rel = lambda p: mapped + (p - d["base"])  # noqa: E731
            rd_set_peer(self.h, side, (rel(d["u"][0]), rel(d["u"][1])), (rel(d["v"][0]), rel(d["v"][1])),
                        d["rows"], d["stride"])
            # my pushes arrive at the neighbour above as "from below" (its
            # word 1), at the neighbour below as "from above" (its word 0)
            self.peer_flags[side] = rel(d["flags"][1 - side])
        self.my_flags = {side: rd_flag_ptr(self.h, side) for side in self.peer_flags}

    def _signal(self):
        self.epoch += 1
        for f in self.peer_flags.values():
            rd_stream_signal(self.h, f, self.epoch)

    def _wait(self):
        for f in self.my_flags.values():
            rd_stream_wait(self.h, f, self.epoch)

    def close(self):
        self.__dict__.pop("_views", None)  # views of the planes freed below
        if self.h:
            rd_destroy(self.h)
            self.h = None

    def set_stream(self, stream):
        from paper_1901_06535_b200 import stream_handle
        rd_set_stream(self.h, stream_handle(stream))

    def write(self, b: int, u_fn, v_fn=None):
        """Write owned rows from global-row generators u_fn(b, row0, rows)."""
        u = np.ascontiguousarray(u_fn(b, self.row0, self.rows), dtype=self.dtype)
        v = None if v_fn is None else np.ascontiguousarray(v_fn(b, self.row0, self.rows), dtype=self.dtype)
        rd_write_fields(self.h, b, u, v)

    def fill_noise(self, b: int = -1, planes: int = 3, seed: int = 1, amplitude: float = 0.1):
        """Global-coordinate noise on the device, ghost rows included."""
        from paper_1901_06535_b200 import rd_fill_noise
        rd_fill_noise(self.h, b, planes, seed, amplitude)

    def stimulate(self, shape: dict, value: float = 1.0, at_step: int = 0, b: int = -1):
        rd_stimulate(self.h, b, shape, value, at_step)  # global coordinates; the slab clips

    def probe_latch(self, b, rect, threshold=0.1, stride=50):
        return rd_probe_latch(self.h, b, rect, threshold, stride)

    def probe_result(self, pid):
        return rd_probe_result(self.h, pid)

    def device_tensors(self, b: int):
        """[(peer, [send u, send v], [recv u, recv v])] for the current buffers."""
        out = []
        cache = self.__dict__.setdefault("_views", {})
        for peer, (s0, s1), (r0, r1) in self.plan:
            sends = [_dev_rows(self.h, b, p, s0, s1, cache) for p in (0, 1)]
            recvs = [_dev_rows(self.h, b, p, r0, r1, cache) for p in (0, 1)]
            out.append((peer, sends, recvs))
        return out

    def exchange(self):
        self.exchange_wait(self.exchange_post())

    def exchange_post(self):
        if self.world == 1 or not isinstance(self.transport, str):
            return None
        return [exchange_post(self.device_tensors(b), self.group) for b in range(self.batch)]

    def exchange_wait(self, pending):
        if self.world == 1:
            return
        if isinstance(self.transport, str):
            for p in pending:
                exchange_wait(p)
        else:
            self.transport.exchange(self)

    def any_rank(self, flag: bool) -> bool:
        """Logical OR of a flag over all ranks (MAX all-reduce)."""
        if self.world == 1:
            return bool(flag)
        import torch
        import torch.distributed as dist
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([1 if flag else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return bool(t.item())

    def step(self, n: int):
        """Advance n steps as one super-step: checkpoint; blocks of <= halo
        steps, each preceded by a halo exchange, with no host synchronisation;
        one flag read OR-reduced over ranks. If any rank produced a non-finite
        cell or tripped the fast-division guard, every rank restores and
        replays step by step (exchange + exact rd_step(1)), all stopping at the
        first failing step, which raises RD_ENONFINITE on every rank."""
        if n <= 0:
            return
        rd_checkpoint(self.h)
        if self.p2p and isinstance(self.transport, str):
            self._step_p2p(n)
        else:
            self._step_exchange(n)
        nonfinite, inexact = rd_read_flags(self.h)
        if not self.any_rank(nonfinite or inexact):
            return
        self._replay(n)

    def _step_p2p(self, n: int):
        """Blocks with the peer-memory push: the edge launches store the send
        rows into the neighbours' next input buffer. A block that is not a
        push block (a stimulus in it, a partial block) first re-pushes the
        send rows in full row storage -- the kernel pushes carry the interior
        columns only, whose mirrored ghost columns rd_step_finish refreshes --
        and steps plainly."""
        rd_push_ghosts(self.h)
        self._signal()
        done = 0
        while done < n:
            k = min(self.halo, n - done)
            started = rd_step_begin(self.h, k, RD_BLOCK_PUSH)
            self._wait()  # the neighbours' previous push has landed
            if started:
                rd_step_finish(self.h)
                self._signal()
            else:
                # full-row re-push (mirrored columns) for this block, step,
                # then -- once every neighbour has stepped too (a partial
                # block rewrites its kept ghost rows) -- push the new buffer's
                # send rows for the next block
                rd_push_ghosts(self.h)
                self._signal()
                self._wait()
                rd_step_unchecked(self.h, k)
                self._signal()
                self._wait()
                rd_push_ghosts(self.h)
                self._signal()
            done += k

    def _step_exchange(self, n: int):
        done = 0
        while done < n:
            # the exchange of this block's input rows is in
            # flight while the interior rows (which read no ghost row) run;
            # the edge bands follow once the ghosts have landed
            k = min(self.halo, n - done)
            pending = self.exchange_post()
            started = rd_step_begin(self.h, k) if self.world > 1 else False
            self.exchange_wait(pending)
            if started:
                rd_step_finish(self.h)
            else:
                rd_step_unchecked(self.h, k)
            done += k

    def _replay(self, n: int):
        rd_restore(self.h)
        for _ in range(n):
            self.exchange()
            err = None
            try:
                rd_step(self.h, 1)
            except RDError as e:
                if e.code != RD_ENONFINITE:
                    raise
                err = e
            if self.any_rank(err is not None):
                raise err or RDError(RD_ENONFINITE, "non-finite value produced on another rank")

    def read_owned(self, b: int = 0):
        u = np.empty((self.rows, self.W), dtype=self.dtype)
        v = np.empty((self.rows, self.W), dtype=self.dtype)
        rd_read_fields(self.h, b, u, v)
        return u, v

    def stats(self):
        return rd_get_stats(self.h)


class LoopbackGroup:
    """Virtual ranks on ONE device: an exchange is a set of device-to-device
    copies between the registered slabs (no kernel ever waits on another), run
    once every slab has finished its block. Used to test the decomposition
    bitwise on a single GPU."""

    def __init__(self, world: int, p2p: bool = False):
        self.world = world
        self.p2p = p2p
        self.slabs = {}
        self.arrived = set()

    def register(self, slab: SlabSim):
        self.slabs[slab.rank] = slab
        if self.p2p and len(self.slabs) == self.world:
            # peer-memory exchange emulated in one process: every virtual rank
            # on one stream (serial order replaces the cross-rank flags), each
            # registered with its neighbours' plane origins
            import torch
            for sl in self.slabs.values():
                sl.set_stream(torch.cuda.current_stream())
            for r, sl in self.slabs.items():
                for side, peer in ((0, r - 1), (1, r + 1)):
                    if 0 <= peer < self.world:
                        u, v, stride = rd_plane_origins(self.slabs[peer].h)
                        rd_set_peer(sl.h, side, u, v, self.slabs[peer].rows, stride)

    def exchange(self, slab: SlabSim):
        self.arrived.add(slab.rank)
        if len(self.arrived) < self.world:
            return
        self.arrived.clear()
        import torch
        torch.cuda.synchronize()  # every slab's queued work (its own stream) has produced the rows
        for b in range(self.slabs[0].batch):
            views = {r: dict((peer, (s, rv)) for peer, s, rv in sl.device_tensors(b)) for r, sl in self.slabs.items()}
            for r, peers in views.items():
                for peer, (sends, _) in peers.items():
                    _, recvs = views[peer][r]
                    for s, rv in zip(sends, recvs):
                        rv.copy_(s)
        import torch
        torch.cuda.synchronize()  # the engine's streams are non-blocking

    def step_all(self, n: int):
        """The SlabSim.step super-step protocol over all virtual ranks."""
        if n <= 0:
            return
        slabs = [self.slabs[r] for r in range(self.world)]
        halo = slabs[0].halo
        for sl in slabs:
            rd_checkpoint(sl.h)
        if self.p2p:
            self._step_all_p2p(slabs, n, halo)
        else:
            self._step_all_exchange(slabs, n, halo)
        if not any(any(rd_read_flags(sl.h)) for sl in slabs):
            return
        self._replay_all(slabs, n)

    def _step_all_p2p(self, slabs, n, halo):
        """SlabSim._step_p2p over the virtual ranks, in serial order on one
        stream: pushes land in the neighbours' next input buffers."""
        for sl in slabs:
            rd_push_ghosts(sl.h)
        done = 0
        while done < n:
            k = min(halo, n - done)
            started = [rd_step_begin(sl.h, k, RD_BLOCK_PUSH) for sl in slabs]
            assert all(started) or not any(started), "ranks disagree on a push block"
            if started[0]:
                for sl in slabs:
                    rd_step_finish(sl.h)
            else:
                for sl in slabs:
                    rd_push_ghosts(sl.h)  # full rows: mirrored columns too
                for sl in slabs:
                    rd_step_unchecked(sl.h, k)
                for sl in slabs:
                    rd_push_ghosts(sl.h)  # the new buffer's ghosts, for the next block
            done += k

    def _step_all_exchange(self, slabs, n, halo):
        done = 0
        while done < n:
            # interior rows first, then the exchange (the interior launches
            # finish before the copies land: a ghost read there would see stale
            # rows and break the bitwise tests), then the edge bands
            k = min(halo, n - done)
            started = [rd_step_begin(sl.h, k) for sl in slabs]
            for sl in slabs:
                sl.exchange()
            for sl, st in zip(slabs, started):
                if st:
                    rd_step_finish(sl.h)
                else:
                    rd_step_unchecked(sl.h, k)
            done += k

    def _replay_all(self, slabs, n):
        for sl in slabs:
            rd_restore(sl.h)
        for _ in range(n):
            for sl in slabs:
                sl.exchange()
            errs = []
            for sl in slabs:
                try:
                    rd_step(sl.h, 1)
                except RDError as e:
                    if e.code != RD_ENONFINITE:
                        raise
                    errs.append(e)
            if errs:
                raise errs[0]
