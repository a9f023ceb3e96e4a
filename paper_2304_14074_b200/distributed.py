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


class ShardedParareal:
    def __init__(self, grid, fine, coarse, num_slices: int, fine_steps: int, *, rank: int = 0,
                 world: int = 1, engine_factory=None, inc_tol: float = 1e-10, device=None):
        import torch
        self.rank, self.world = rank, world
        self.N, self.J = num_slices, fine_steps
        self.s0, self.s1 = shard(num_slices, world, rank)
        self.local_slices = self.s1 - self.s0
        if engine_factory is None:
            from .engine import PararealEngine
            engine_factory = PararealEngine
        self.eng = engine_factory(grid, fine, coarse, self.local_slices, fine_steps, batch=1,
                                  device=device)
        self.grid = grid
        self.inc_tol = inc_tol
        self.k = 0
        self.converged_at = None
        self.increments = []
        self._torch = torch
        self._pending = []              # deferred increment reductions (iterate(defer=True))
        self._red_group = None
        if world > 1:
            # the increment all-reduce runs on its own communicator, so a deferred
            # reduction of iteration k never queues in front of the boundary
            # send/recv of iteration k+1 on the chain's communicator
            import torch.distributed as dist
            self._red_group = dist.new_group(list(range(world)))

    # -- communication helpers ------------------------------------------------
    def _dist(self):
        import torch.distributed as dist
        return dist

    def _recv_boundary(self):
        """U_{s0} and its changed flag from rank-1 into local slot 0."""
        if self.rank == 0:
            return
        dist = self._dist()
        dist.recv(self.eng.U[0, 0], src=self.rank - 1)
        flag = self._torch.zeros(1, dtype=self._torch.uint8, device=self.eng.U.device)
        dist.recv(flag, src=self.rank - 1)
        self.eng.changed[0, 0] = flag[0]

    def _send_boundary(self):
        if self.rank == self.world - 1:
            return
        dist = self._dist()
        L = self.local_slices
        dist.send(self.eng.U[0, L].contiguous(), dst=self.rank + 1)
        flag = self.eng.changed[0, L:L + 1].clone()
        dist.send(flag, dst=self.rank + 1)

    # -- phases ---------------------------------------------------------------
    def load(self, u0) -> None:
        if self.rank == 0:
            self.eng.load([u0])

    def coarse_init(self) -> None:
        self._recv_boundary()
        self.eng.coarse_range(0, 0, self.local_slices)
        self._send_boundary()
        self.eng.changed.fill_(1)        # every F(U_n^0) is needed at k = 0
        self.k = 0

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
        if coarse_after is not None:
            self._torch.cuda.current_stream().wait_event(coarse_after)
        eng.inc.zero_()
        self._recv_boundary()
        if self.rank == 0:
            eng.changed[0, 0] = 1 if force_all else 0
        elif force_all:
            eng.changed[0, 0] = 1
        if coarse_chunks is None:
            eng.coarse_range(1, 0, self.local_slices)
        else:
            for n0, n1 in coarse_chunks:
                eng.coarse_range(1, n0, n1)
                if on_coarse_chunk is not None:
                    on_coarse_chunk(n0, n1)
        self._send_boundary()
        eng.check_status()
        inc = eng.inc.clone()
        if defer:
            work = None
            if self.world > 1:
                work = self._dist().all_reduce(inc, op=self._dist().ReduceOp.MAX,
                                               group=self._red_group, async_op=True)
            self.k += 1
            self._pending.append((self.k, work, inc))
            return None
        if self.world > 1:
            self._dist().all_reduce(inc, op=self._dist().ReduceOp.MAX, group=self._red_group)
        self.k += 1
        return self._record(self.k, inc)

    def _record(self, k, inc) -> float:
        val = float(inc[0])
        self.increments.append(val)
        if self.converged_at is None and val < self.inc_tol:
            self.converged_at = k
        return val

    def flush(self) -> None:
        """Complete the deferred increment reductions (in iteration order)."""
        for k, work, inc in self._pending:
            if work is not None:
                work.wait()
            self._record(k, inc)
        self._pending = []

    def run(self, max_iter: int | None = None):
        if max_iter is None:
            max_iter = self.N + 2
        self.coarse_init()
        while self.converged_at is None and self.k < max_iter:
            self.iterate()
        return self.converged_at

    def local_iterates(self) -> np.ndarray:
        """Host copy of U_{s0+1} .. U_{s1} (and U_0 on rank 0)."""
        U = self.eng.iterates_host(0)
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
        iteration runs, and the new iterates are copied back D2H.  The coarse
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
        hU.copy_(eng.U)
        hG.copy_(eng.G)
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
                # U^{k+1}_{n0+1..n1} are final: copy them out under the next chunk's
                # coarse sweep (U_0 with the first chunk)
                ev = torch.cuda.Event()
                ev.record(main)
                d2h.wait_event(ev)
                r0 = 0 if n0 == 0 else n0 + 1
                with torch.cuda.stream(d2h):
                    hOut[:, r0:n1 + 1].copy_(eng.U[:, r0:n1 + 1], non_blocking=True)

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
        if self.world > 1:
            t = torch.tensor([ms], device=eng.U.device, dtype=torch.float64)
            self._dist().all_reduce(t, op=self._dist().ReduceOp.MAX)
            ms = float(t.item())
        pts = self.N * self.J * self.grid.interior_count
        nbytes = eng.U.numel() * 8
        return {"value": pts / (ms * 1e-3), "unit": "grid-point-steps/s",
                "h2d_bytes_per_step": 2 * nbytes, "d2h_bytes_per_step": nbytes,
                "ms_per_step": ms,
                "path": "pinned host iterates -> engine (chp_propagate/chp_coarse_sweep) -> host",
                "copies": f"{nch} slice chunks, overlapped with the fine and coarse sweeps"}
