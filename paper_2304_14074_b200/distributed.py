"""Multi-GPU Parareal: time slices sharded contiguously over ranks.

Rank r of P owns slices [r*N/P, (r+1)*N/P).  Per iteration:

1. fine sweep over the rank's changed slices -- no communication;
2. coarse sweep as a chain: rank r receives U_{s0}^{k+1} (plus its
   "changed in this sweep" flag) from rank r-1, runs its coarse steps +
   corrections on the device, and sends U_{s1}^{k+1} to rank r+1
   (torch.distributed send/recv over NCCL / NVLink; one field per hop);
3. the increment max_{n,i} |dU| is an all-reduce(max) of one double.

The chain adds no arithmetic, so iterates are bit-identical for any P.
The local engine only needs the small interface used below, so the chain
logic is testable on CPU with gloo and a host engine (tests/test_distributed.py).
"""

from __future__ import annotations

import numpy as np


def shard(N: int, world: int, rank: int) -> tuple[int, int]:
    if N % world:
        raise ValueError(f"{N} slices do not shard evenly over {world} ranks")
    L = N // world
    return rank * L, (rank + 1) * L


class TorchComm:
    """Point-to-point hand-off and increment reduction over torch.distributed
    (NCCL over NVLink on the GPU box, gloo in the CPU tests)."""

    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world
        self._red_group = None
        if world > 1:
            # the increment all-reduce runs on its own communicator, so a deferred
            # reduction of iteration k never queues in front of the boundary
            # send/recv of iteration k+1 on the chain's communicator
            import torch.distributed as dist
            self._red_group = dist.new_group(list(range(world)))

    def send(self, t, dst: int) -> None:
        import torch.distributed as dist
        dist.send(t, dst=dst)

    def recv(self, t, src: int) -> None:
        import torch.distributed as dist
        dist.recv(t, src=src)

    def all_reduce_max(self, t, async_op: bool = False):
        if self.world == 1:
            return None
        import torch.distributed as dist
        return dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self._red_group, async_op=async_op)


class LoopbackComm:
    """Simulated ranks in one process: every shard engine lives on the
    same device, sends are device-to-device copies into a mailbox and the increment
    reduction is done by the driver (SimulatedRanks).  The chain runs shard after shard,
    so no kernel ever waits on another."""

    def __init__(self, world: int):
        self.world = world
        self.box = {}

    def view(self, rank: int):
        return _LoopbackEnd(self, rank)


class _LoopbackEnd:
    def __init__(self, hub: LoopbackComm, rank: int):
        self.hub, self.rank, self.world = hub, rank, hub.world

    def send(self, t, dst: int) -> None:
        self.hub.box.setdefault((self.rank, dst), []).append(t.clone())

    def recv(self, t, src: int) -> None:
        t.copy_(self.hub.box[(src, self.rank)].pop(0))

    def all_reduce_max(self, t, async_op: bool = False):
        return None                      # SimulatedRanks reduces across shards itself


class Mailbox:
    """One rank's receive side of the device-initiated hop (include/chp.h chp_hop): two
    slots of [B] boundary fields + [B] changed bytes, the flag the sender releases and the
    ack word this rank's *own* sends wait on, in one chp_mem_alloc allocation (so it can
    be exported with cudaIpc).  Layout (bytes): slot s field i at s*B*fs*8 + i*fs*8;
    changed at 2*B*fs*8 + s*B; flag at 2*B*fs*8 + 64 + ... (256-byte aligned words)."""

    def __init__(self, ctx, B: int, fs: int):
        import ctypes
        self.ctx, self.B, self.fs = ctx, B, fs
        self.off_changed = 2 * B * fs * 8
        self.off_flag = (self.off_changed + 2 * B + 255) // 256 * 256
        self.off_ack = self.off_flag + 256
        self.bytes = self.off_ack + 256
        p = ctypes.c_void_p()
        ctx.check(ctx.L.chp_mem_alloc(ctx.h, self.bytes, ctypes.byref(p)), "chp_mem_alloc")
        self.base = p.value

    def handle(self) -> bytes:
        import ctypes
        buf = ctypes.create_string_buffer(64)
        self.ctx.check(self.ctx.L.chp_ipc_export(self.ctx.h, ctypes.c_void_p(self.base), buf),
                       "chp_ipc_export")
        return buf.raw

    def free(self):
        import ctypes
        if self.base:
            self.ctx.L.chp_mem_free(self.ctx.h, ctypes.c_void_p(self.base))
            self.base = 0


class HopComm:
    """Device-initiated coarse-chain hand-off instead of dist.send/recv:
    rank r's coarse sweep stores U_{s1} straight into rank r+1's mailbox and releases a
    flag (fused into the cooperative 2D kernel's last correction; a put kernel otherwise);
    rank r+1's stream waits on the flag with a stream memory operation (no kernel spins),
    takes the mailbox and acknowledges into rank r's ack word, which gates the reuse of
    the mailbox slot two sends later.  ``peers``: {rank: base address of that rank's
    mailbox as seen from this process} -- cudaIpc mappings between processes
    (``HopComm.over_ipc``), or the plain addresses of shards living in one process
    (``HopComm.loopback``, the simulated ranks of tests/test_gpu_sharded.py).  The
    increment all-reduce stays on torch.distributed (``red``)."""

    fused = True

    def __init__(self, rank: int, world: int, box: Mailbox, peers: dict, red=None):
        self.rank, self.world, self.box, self.peers, self.red = rank, world, box, peers, red
        self.seq_out = 0
        self.seq_in = 0

    # -- construction ----------------------------------------------------------
    @classmethod
    def loopback(cls, ctx, world: int, B: int, fs: int):
        boxes = [Mailbox(ctx, B, fs) for _ in range(world)]
        peers = {r: boxes[r].base for r in range(world)}
        return [cls(r, world, boxes[r], peers) for r in range(world)]

    @classmethod
    def over_ipc(cls, ctx, rank: int, world: int, B: int, fs: int):
        """Exchange the mailboxes' cudaIpc handles over torch.distributed and map the
        neighbours' (one process per GPU on one node)."""
        import ctypes

        import torch.distributed as dist
        box = Mailbox(ctx, B, fs)
        handles = [None] * world
        dist.all_gather_object(handles, box.handle())
        peers = {rank: box.base}
        for r in (rank - 1, rank + 1):
            if 0 <= r < world:
                p = ctypes.c_void_p()
                ctx.check(ctx.L.chp_ipc_open(ctx.h, handles[r], ctypes.byref(p)), "chp_ipc_open")
                peers[r] = p.value
        return cls(rank, world, box, peers, red=TorchComm(rank, world))

    # -- the hop -----------------------------------------------------------------
    def hop(self, stream_ptr):
        """Descriptor of the next send (to rank+1), after gating on the slot's ack."""
        import ctypes

        from . import _native as N
        self.seq_out += 1
        seq, b = self.seq_out, self.box
        if seq > 2:        # slot seq % 2 last carried message seq - 2: wait until it was taken
            b.ctx.check(b.ctx.L.chp_hop_wait(b.ctx.h, ctypes.c_void_p(b.base + b.off_ack), seq - 2,
                                             stream_ptr), "chp_hop_wait")
        dst = self.peers[self.rank + 1]
        slot = seq % 2
        return N.ChpHop(dst + slot * b.B * b.fs * 8, b.fs, dst + b.off_changed + slot * b.B,
                        dst + b.off_flag, seq, 0)

    def take(self, eng, grid_native, stream_ptr) -> None:
        """Wait for the next message from rank-1 and move it into local slot 0."""
        import ctypes

        from . import _native as N
        self.seq_in += 1
        seq, b = self.seq_in, self.box
        L = b.ctx.L
        b.ctx.check(L.chp_hop_wait(b.ctx.h, ctypes.c_void_p(b.base + b.off_flag), seq, stream_ptr),
                    "chp_hop_wait")
        slot = seq % 2
        ack = self.peers[self.rank - 1] + b.off_ack
        b.ctx.check(L.chp_hop_take(
            b.ctx.h, grid_native, b.B, ctypes.c_void_p(b.base + slot * b.B * b.fs * 8), b.fs,
            ctypes.c_void_p(b.base + b.off_changed + slot * b.B), N.ptr(eng.U),
            eng.U.shape[1] * eng.U.shape[2], N.ptr(eng.changed), eng.changed.shape[1],
            ctypes.c_void_p(ack), seq, stream_ptr), "chp_hop_take")

    def all_reduce_max(self, t, async_op: bool = False):
        return None if self.red is None else self.red.all_reduce_max(t, async_op=async_op)


class ShardedParareal:
    """Parareal on one rank's contiguous slice shard, for ``batch`` independent ICs
    (all ICs of those slices live on the rank)."""

    def __init__(self, grid, fine, coarse, num_slices: int, fine_steps: int, *, rank: int = 0,
                 world: int = 1, engine_factory=None, inc_tol: float = 1e-10, device=None,
                 batch: int = 1, comm=None):
        import torch
        self.rank, self.world = rank, world
        self.N, self.J, self.B = num_slices, fine_steps, int(batch)
        self.s0, self.s1 = shard(num_slices, world, rank)
        self.local_slices = self.s1 - self.s0
        if engine_factory is None:
            from .engine import PararealEngine
            engine_factory = PararealEngine
        self.eng = engine_factory(grid, fine, coarse, self.local_slices, fine_steps,
                                  batch=self.B, device=device)
        self.grid = grid
        self.inc_tol = inc_tol
        self.k = 0
        self.converged = [None] * self.B
        self.incs: list = []              # per-iteration [B] increments
        self._torch = torch
        self._pending = []              # deferred increment reductions (iterate(defer=True))
        if comm is None:
            # CHP_HOP=ipc: boundaries by the device-initiated hop over cudaIpc mailboxes
            # (one process per GPU on one node) instead of dist.send/recv
            import os
            if world > 1 and os.environ.get("CHP_HOP", "") == "ipc":
                comm = HopComm.over_ipc(self.eng.ctx, rank, world, self.B, self.eng.fs)
            else:
                comm = TorchComm(rank, world)
        self.comm = comm

    # -- batch-1 views of the reference-shaped results -------------------------
    @property
    def converged_at(self):
        return self.converged[0] if self.B == 1 else self.converged

    @property
    def increments(self) -> list:
        return [float(x[0]) for x in self.incs] if self.B == 1 else list(self.incs)

    # -- communication helpers ------------------------------------------------
    def _recv_boundary(self):
        """U_{s0} (all ICs) and its changed flags from rank-1 into local slot 0; the
        local freeze bit (bit 1 of slot 0) is kept."""
        if self.rank == 0:
            return
        if getattr(self.comm, "fused", False):
            from . import _native as N
            self.comm.take(self.eng, self.eng._native_grid(), N.stream_ptr(None, self.eng.device))
            return
        torch = self._torch
        dev = self.eng.U.device
        buf = torch.empty((self.B, self.eng.U.shape[2]), dtype=torch.float64, device=dev)
        self.comm.recv(buf, src=self.rank - 1)
        self.eng.U[:, 0].copy_(buf)
        flag = torch.zeros(self.B, dtype=torch.uint8, device=dev)
        self.comm.recv(flag, src=self.rank - 1)
        self.eng.changed[:, 0] = (self.eng.changed[:, 0] & 2) | (flag & 1)

    def _hop(self):
        """The fused hand-off descriptor of this sweep (None: last rank, or send/recv comm)."""
        if self.rank == self.world - 1 or not getattr(self.comm, "fused", False):
            return None
        from . import _native as N
        return self.comm.hop(N.stream_ptr(None, self.eng.device))

    def _send_boundary(self):
        if self.rank == self.world - 1 or getattr(self.comm, "fused", False):
            return
        L = self.local_slices
        self.comm.send(self.eng.U[:, L].contiguous(), dst=self.rank + 1)
        self.comm.send((self.eng.changed[:, L] & 1).contiguous(), dst=self.rank + 1)

    # -- phases ---------------------------------------------------------------
    def load(self, u0s) -> None:
        if self.rank == 0:
            self.eng.load(u0s if isinstance(u0s, (list, tuple)) else [u0s])

    def coarse_init(self) -> None:
        self._recv_boundary()
        hop = self._hop()
        if hop is None:
            self.eng.coarse_range(0, 0, self.local_slices)
        else:
            self.eng.coarse_range(0, 0, self.local_slices, hop=hop)
        self._send_boundary()
        self.eng.changed.fill_(1)        # every F(U_n^0) is needed at k = 0
        self.k = 0

    def fine_phase(self, force_all: bool = False, fine_chunks=None) -> None:
        """F(U_n^k) for the local slices whose U_n changed in the last sweep (writes F
        only: U is untouched, so this can run ahead of the increment test)."""
        eng = self.eng
        flags = eng.changed.cpu().numpy()
        if force_all:
            flags[:, : self.local_slices] |= 1
        if fine_chunks is None:
            eng.fine_sweep(flags)
        else:
            for lo, hi, ev in fine_chunks:
                if ev is not None:
                    self._torch.cuda.current_stream().wait_event(ev)
                part = np.zeros_like(flags)
                part[:, lo:hi] = flags[:, lo:hi]
                part[:, 0] |= flags[:, 0] & 2
                eng.fine_sweep(part)

    def coarse_phase(self, force_all: bool = False, coarse_after=None, coarse_chunks=None,
                     on_coarse_chunk=None):
        """The local part of the coarse chain (receive, sweep + correction, send);
        returns the local per-IC increments (device tensor)."""
        eng = self.eng
        if coarse_after is not None:
            self._torch.cuda.current_stream().wait_event(coarse_after)
        eng.inc.zero_()
        self._recv_boundary()
        if self.rank == 0:
            eng.changed[:, 0] = (eng.changed[:, 0] & 2) | (1 if force_all else 0)
        elif force_all:
            eng.changed[:, 0] |= 1
        hop = self._hop()
        if coarse_chunks is None:
            coarse_chunks = [(0, self.local_slices)]
        for c, (n0, n1) in enumerate(coarse_chunks):
            if hop is not None and c == len(coarse_chunks) - 1:
                eng.coarse_range(1, n0, n1, hop=hop)       # the last range hands U_{s1} on
            else:
                eng.coarse_range(1, n0, n1)
            if on_coarse_chunk is not None:
                on_coarse_chunk(n0, n1)
        self._send_boundary()
        eng.check_status()
        return eng.inc.clone()

    def iterate(self, force_all: bool = False, coarse_after=None, defer: bool = False,
                fine_chunks=None, coarse_chunks=None, on_coarse_chunk=None):
        """One Parareal iteration.  ``coarse_after``: an optional CUDA event the
        coarse sweep waits for (an input copy overlapped with the fine sweep).
        ``defer``: do not wait for the all-ranks increment (returns None; call
        ``flush()``): rank r then starts iteration k+1 as soon as its own part of
        the coarse chain of iteration k is done, while ranks r+1.. are still in
        the chain (pipelined Parareal across ranks; same arithmetic).
        ``fine_chunks``: [(lo, hi, event)] -- the fine sweep runs slice range
        [lo, hi) after ``event`` (its inputs' copy) completes; ``coarse_chunks``:
        [(n0, n1)] -- the coarse sweep runs in these consecutive ranges, calling
        ``on_coarse_chunk(n0, n1)`` after each (e.g. to start copying the
        finished iterates out).  Same arithmetic as one sweep."""
        self.fine_phase(force_all, fine_chunks)
        inc = self.coarse_phase(force_all, coarse_after, coarse_chunks, on_coarse_chunk)
        if defer:
            work = self.comm.all_reduce_max(inc, async_op=True)
            self.k += 1
            self._pending.append((self.k, work, inc))
            return None
        self.comm.all_reduce_max(inc)
        self.k += 1
        return self._record(self.k, inc)

    def _record(self, k, inc):
        """Fold the all-ranks increments of iteration k: per-IC convergence, and ICs
        that converged are frozen on this rank (changed slot 0, bit 1)."""
        v = inc.cpu().numpy().astype(np.float64).reshape(-1).copy()
        for i in range(self.B):
            if self.converged[i] is not None:
                v[i] = 0.0
        self.incs.append(v)
        for i in range(self.B):
            if self.converged[i] is None and v[i] < self.inc_tol:
                self.converged[i] = k
                self.eng.changed[i, 0] |= 2
        return float(v[0]) if self.B == 1 else v

    def flush(self) -> None:
        """Complete the deferred increment reductions (in iteration order)."""
        for k, work, inc in self._pending:
            if work is not None:
                work.wait()
            self._record(k, inc)
        self._pending = []

    def done(self) -> bool:
        return all(c is not None for c in self.converged)

    def run(self, max_iter: int | None = None, pipelined: bool = True):
        """Coarse init, then iterate to the increment stop on every IC.  ``pipelined``:
        the fine sweep of iteration k+1 (it writes F only) is issued before waiting for
        the all-ranks increment of iteration k, so rank r overlaps its next fine sweep
        with the rest of the coarse chain and the reduction; if iteration k turns out to
        be the last, that fine sweep is discarded and the iterates are those of k.
        Same arithmetic and stopping iteration as the synchronous loop."""
        if max_iter is None:
            max_iter = self.N + 2
        self.coarse_init()
        if not pipelined:
            while not self.done() and self.k < max_iter:
                self.iterate()
            return self.converged_at
        self.fine_phase()
        while not self.done() and self.k < max_iter:
            inc = self.coarse_phase()
            work = self.comm.all_reduce_max(inc, async_op=True)
            self.k += 1
            if self.k < max_iter:
                self.fine_phase()                 # speculative: U is not touched
            if work is not None:
                work.wait()
            self._record(self.k, inc)
        return self.converged_at

    def local_iterates(self, i: int = 0) -> np.ndarray:
        """Host copy of U_{s0+1} .. U_{s1} (and U_0 on rank 0) of IC i."""
        U = self.eng.iterates_host(i)
        return U if self.rank == 0 else U[1:]


    # -- measurement helpers (bench.py) ----------------------------------------
    def time_fine_sweep(self) -> float:
        """Device time (ms) of one fine sweep over every local slice."""
        torch = self._torch
        flags = np.ones((1, self.local_slices + 1), dtype=np.uint8)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        self.eng.fine_sweep(flags)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    def e2e_step_rate(self, steps: int, warmup: int = 1, chunks: int = 2,
                      coarse_chunked: bool = True) -> dict:
        """Same metric with host-resident iterates: per step the local iterates
        and coarse values are copied H2D from pinned memory, one forced
        iteration runs, and the new iterates and coarse values are copied back D2H
        (the whole PararealState round-trips through the host).  The engine state is
        restored afterwards.  The coarse
        values are only read by the coarse sweep, so their copy runs on a side
        stream under the fine sweep.  The iterates move in ``chunks`` slice
        ranges: chunk c+1 is copied in while the fine sweep of chunk c runs, and
        the coarse sweep runs chunk by chunk with each finished range copied out
        under the next range's sweep -- only the first chunk's input and the
        last chunk's output copies stay exposed."""
        torch = self._torch
        eng = self.eng
        hU = torch.empty(eng.U.shape, dtype=torch.float64, pin_memory=True)
        hG = torch.empty(eng.G.shape, dtype=torch.float64, pin_memory=True)
        hOut = torch.empty(eng.U.shape, dtype=torch.float64, pin_memory=True)
        hGout = torch.empty(eng.G.shape, dtype=torch.float64, pin_memory=True)
        hU.copy_(eng.U)
        hG.copy_(eng.G)
        saved = (eng.changed.clone(), self.k, list(self.incs), list(self.converged))
        side = torch.cuda.Stream(device=eng.U.device)
        h2d = torch.cuda.Stream(device=eng.U.device)
        d2h = torch.cuda.Stream(device=eng.U.device)
        main = torch.cuda.current_stream()
        L = self.local_slices
        nch = max(1, min(chunks, L))
        bounds = [L * c // nch for c in range(nch + 1)]

        def step():
            # U^k in slice chunks on a copy stream; the fine sweep of chunk c
            # starts when its rows have landed (chunk c+1 copies meanwhile)
            h2d.wait_stream(main)
            h2d.wait_stream(d2h)                      # last step's read-out of U is done
            fine = []
            with torch.cuda.stream(h2d):
                for c in range(nch):
                    lo, hi = bounds[c], bounds[c + 1]
                    r1 = hi + 1 if c == nch - 1 else hi   # last chunk: U[L] as well
                    eng.U[:, lo:r1].copy_(hU[:, lo:r1], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(h2d)
                    fine.append((lo, hi, ev))
            side.wait_stream(main)                    # G is free: the last sweep is done
            with torch.cuda.stream(side):
                eng.G.copy_(hG, non_blocking=True)
                g_ready = torch.cuda.Event()
                g_ready.record(side)
            # (the last fine chunk waits for the last copy event, so the whole of
            # U is resident before the coarse sweep)

            def out_chunk(n0, n1):
                # U^{k+1}_{n0+1..n1} and G(U^{k+1}_{n0..n1-1}) are final: copy them out
                # under the next chunk's coarse sweep (U_0 with the first chunk)
                ev = torch.cuda.Event()
                ev.record(main)
                d2h.wait_event(ev)
                r0 = 0 if n0 == 0 else n0 + 1
                with torch.cuda.stream(d2h):
                    hOut[:, r0:n1 + 1].copy_(eng.U[:, r0:n1 + 1], non_blocking=True)
                    hGout[:, n0:n1].copy_(eng.G[:, n0:n1], non_blocking=True)

            # the result U^{k+1} goes to its own buffer: every step starts from the
            # same consistent host state (U^k, G(U^k))
            if coarse_chunked:
                self.iterate(force_all=True, coarse_after=g_ready, defer=True, fine_chunks=fine,
                             coarse_chunks=[(bounds[c], bounds[c + 1]) for c in range(nch)],
                             on_coarse_chunk=out_chunk)
            else:
                self.iterate(force_all=True, coarse_after=g_ready, defer=True, fine_chunks=fine)
                out_chunk(0, L)

        for _ in range(warmup):
            step()
        self.flush()
        torch.cuda.synchronize()
        assert torch.equal(hOut.to(eng.U.device), eng.U), "e2e read-out differs from U"
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            step()
        self.flush()
        main.wait_stream(d2h)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / steps
        # restore the engine state the measurement started from (U^k, G(U^k), k)
        eng.U.copy_(hU)
        eng.G.copy_(hG)
        eng.changed.copy_(saved[0])
        self.k, self.incs, self.converged = saved[1], saved[2], saved[3]
        torch.cuda.synchronize()
        if self.world > 1:
            t = torch.tensor([ms], device=eng.U.device, dtype=torch.float64)
            import torch.distributed as dist
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        pts = self.N * self.J * self.grid.interior_count
        nbytes = eng.U.numel() * 8
        return {"value": pts / (ms * 1e-3), "unit": "grid-point-steps/s",
                "h2d_bytes_per_step": 2 * nbytes, "d2h_bytes_per_step": 2 * nbytes,
                "ms_per_step": ms,
                "path": "pinned host iterates -> engine (chp_propagate/chp_coarse_sweep) -> host",
                "copies": f"{nch} slice chunks, overlapped with the fine and coarse sweeps"}


class SimulatedRanks:
    """``world`` shards of one run in ONE process on one device: the
    shard engines are the real device engines, the boundary hand-off is a
    device-to-device copy (LoopbackComm), the coarse chain runs shard after shard and
    the increment is the max over shards -- the sharding logic of ShardedParareal
    exercised on one GPU, with no kernels waiting on one another."""

    def __init__(self, grid, fine, coarse, num_slices: int, fine_steps: int, world: int, *,
                 batch: int = 1, inc_tol: float = 1e-10, engine_factory=None, device=None,
                 hop: bool = False):
        """``hop``: hand the boundaries over with the device-initiated hop (HopComm over
        plain device addresses: fused stores + flag from the coarse sweep, stream wait and
        take on the receiving shard) instead of mailbox copies."""
        if hop:
            import torch

            from . import _native as N
            dev = torch.device(device) if device is not None else torch.device(
                "cuda", torch.cuda.current_device())
            ctx = N.Context.get(dev.index if dev.index is not None else torch.cuda.current_device())
            comms = HopComm.loopback(ctx, world, batch, grid.device_size)
            self._boxes = [c.box for c in comms]
        else:
            hub = LoopbackComm(world)
            comms = [hub.view(r) for r in range(world)]
        self.shards = [ShardedParareal(grid, fine, coarse, num_slices, fine_steps, rank=r,
                                       world=world, engine_factory=engine_factory,
                                       inc_tol=inc_tol, device=device, batch=batch,
                                       comm=comms[r])
                       for r in range(world)]
        self.world, self.B = world, batch
        self.N = num_slices

    def load(self, u0s) -> None:
        self.shards[0].load(u0s)

    def coarse_init(self) -> None:
        for sh in self.shards:
            sh.coarse_init()

    def iterate(self, force_all: bool = False):
        for sh in self.shards:
            sh.fine_phase(force_all)
        incs = [sh.coarse_phase(force_all) for sh in self.shards]
        inc = incs[0]
        for t in incs[1:]:
            inc = self.shards[0]._torch.maximum(inc, t.to(inc.device))
        out = None
        for sh in self.shards:
            sh.k += 1
            out = sh._record(sh.k, inc)
        return out

    def run(self, max_iter: int | None = None):
        if max_iter is None:
            max_iter = self.N + 2
        self.coarse_init()
        sh0 = self.shards[0]
        while not sh0.done() and sh0.k < max_iter:
            self.iterate()
        return sh0.converged_at

    @property
    def increments(self):
        return self.shards[0].increments

    def iterates(self, i: int = 0) -> np.ndarray:
        return np.concatenate([sh.local_iterates(i) for sh in self.shards])
