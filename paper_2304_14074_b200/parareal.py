"""The Parareal engine API on the B200.

Drop-in for ``chparareal.parareal`` (reference parareal.py, ``__all__`` at
parareal.py:26-39): same names, signatures, defaults, return types and
exceptions.  The bodies run on the device through ``engine.PararealEngine``:
the fine sweep over all slices is one batched launch, the coarse sweep and
correction ``U_{n+1} = (G(U_n^{k+1}) + F(U_n^k)) - G(U_n^k)`` (parareal.py:249,
same evaluation order) is one device-side sequential sweep.

Additions:
* ``iterate_increment(state)`` -- max_{n,i} |U_n^k - U_n^{k-1}|;
* ``run(..., stop="increment", increment_tol=1e-10)`` -- the BASELINE
  convergence test on the iterate increment;
* ``run_batch(u0s, ...)`` -- independent initial conditions in one engine,
  per-IC stopping (converged ICs are frozen, not re-iterated).

``workers`` is accepted and ignored: slices are batched into one launch
instead of threads (results are worker-count independent, as the reference
guarantees, parareal.py:11-14).
"""

from __future__ import annotations

import enum
import math
import time
from dataclasses import dataclass, field

import numpy as np

from .engine import PararealEngine
from .grid import (Field, energy, field_stats, from_device_layout, l2_norm, mass, stats_energy,
                   stats_l2, stats_mass)
from .schemes import NewtonStats, PropagatorSpec, Scheme

__all__ = [
    "AlgorithmVariant",
    "TimePartition",
    "PararealState",
    "IterationRecord",
    "RunTrace",
    "propagator_pair",
    "serial_fine_reference",
    "coarse_init",
    "initial_state",
    "parareal_iteration",
    "error_against_reference",
    "run",
    "iterate_increment",
    "run_batch",
]


class AlgorithmVariant(enum.Enum):
    """Fine/coarse pairing of the five variants (parareal.py:42-70)."""

    PA1 = "pa1"
    PA2 = "pa2"
    PA3 = "pa3"
    NPA1 = "npa1"
    NPA2 = "npa2"

    @property
    def fine_scheme(self) -> Scheme:
        return _PAIRINGS[self][0]

    @property
    def coarse_scheme(self) -> Scheme:
        return _PAIRINGS[self][1]

    @property
    def is_nonlinear(self) -> bool:
        return self in (AlgorithmVariant.NPA1, AlgorithmVariant.NPA2)


_PAIRINGS = {
    AlgorithmVariant.PA1: (Scheme.LINEAR_A, Scheme.LINEAR_A),
    AlgorithmVariant.PA2: (Scheme.LINEAR_B, Scheme.LINEAR_B),
    AlgorithmVariant.PA3: (Scheme.LINEAR_B, Scheme.LINEAR_A),
    AlgorithmVariant.NPA1: (Scheme.NONLINEAR_EYRE, Scheme.LINEAR_A),
    AlgorithmVariant.NPA2: (Scheme.NONLINEAR_EYRE, Scheme.NONLINEAR_EYRE),
}


@dataclass(frozen=True)
class TimePartition:
    """N coarse slices of T, each split into J fine steps (parareal.py:73-93)."""

    total_time: float
    num_slices: int
    fine_steps: int

    def __post_init__(self) -> None:
        if self.total_time <= 0:
            raise ValueError("total_time must be positive")
        if self.num_slices < 1 or self.fine_steps < 1:
            raise ValueError("num_slices and fine_steps must be at least 1")

    @property
    def coarse_dt(self) -> float:
        return self.total_time / self.num_slices

    @property
    def fine_dt(self) -> float:
        return self.coarse_dt / self.fine_steps


def propagator_pair(variant: AlgorithmVariant, partition: TimePartition, eps: float, *,
                    newton_tol: float = 1e-10, newton_max_iter: int = 50, nn=None
                    ) -> tuple[PropagatorSpec, PropagatorSpec]:
    """Fine and coarse specs (parareal.py:96-126)."""
    fine_scheme = Scheme.NN_LINEAR_A if nn is not None else variant.fine_scheme
    fine = PropagatorSpec(fine_scheme, partition.fine_dt, eps, newton_tol, newton_max_iter, nn)
    coarse = PropagatorSpec(variant.coarse_scheme, partition.coarse_dt, eps, newton_tol,
                            newton_max_iter)
    return fine, coarse


@dataclass
class PararealState:
    """Interface values at the coarse nodes (parareal.py:129-142).  ``_engine``
    (private) lets consecutive ``parareal_iteration`` calls continue on the
    device without re-deriving F."""

    iterates: list
    coarse_values: list
    fine_reference: list
    k: int
    previous: list | None = field(default=None)
    _engine: object = field(default=None, repr=False, compare=False)


def _engine_for(u0: Field, variant, partition, eps, newton_tol, newton_max_iter, nn,
                batch=1) -> PararealEngine:
    fine, coarse = propagator_pair(variant, partition, eps, newton_tol=newton_tol,
                                   newton_max_iter=newton_max_iter, nn=nn)
    return PararealEngine(u0.grid, fine, coarse, partition.num_slices, partition.fine_steps,
                          batch=batch)


def _fields(eng: PararealEngine, tensor, count: int, offset: int = 0) -> list:
    shape = eng._dev_shape()
    return [Field._trusted(eng.grid, tensor[0, offset + n].view(shape)) for n in range(count)]


def serial_fine_reference(u0: Field, variant: AlgorithmVariant, partition: TimePartition,
                          eps: float, *, newton_tol: float = 1e-10, newton_max_iter: int = 50,
                          nn=None, stats: NewtonStats | None = None) -> list:
    """Sequential fine propagation stored at every coarse node (parareal.py:145-164)."""
    eng = _engine_for(u0, variant, partition, eps, newton_tol, newton_max_iter, nn)
    eng.load([u0])
    R, si = eng.serial_fine()
    if stats is not None and eng.fine.scheme is Scheme.NONLINEAR_EYRE:
        stats.absorb(si)
    return _fields(eng, R, partition.num_slices + 1)


def coarse_init(u0: Field, variant: AlgorithmVariant, partition: TimePartition, eps: float, *,
                newton_tol: float = 1e-10, newton_max_iter: int = 50,
                stats: NewtonStats | None = None) -> list:
    """U_n^0 = G^n(u0) (parareal.py:167-185)."""
    eng = _engine_for(u0, variant, partition, eps, newton_tol, newton_max_iter, None)
    eng.load([u0])
    eng.coarse_init()
    if stats is not None:
        _merge(stats, eng.newton)
    return _fields(eng, eng.U, partition.num_slices + 1)


def _merge(dst: NewtonStats, src: NewtonStats) -> None:
    dst.steps += src.steps
    dst.total_iterations += src.total_iterations
    dst.max_iterations = max(dst.max_iterations, src.max_iterations)
    dst.max_residual = max(dst.max_residual, src.max_residual)


def initial_state(u0: Field, variant: AlgorithmVariant, partition: TimePartition, eps: float,
                  *, newton_tol: float = 1e-10, newton_max_iter: int = 50, nn=None,
                  stats: NewtonStats | None = None) -> PararealState:
    """Serial reference + coarse init (parareal.py:188-213)."""
    reference = serial_fine_reference(u0, variant, partition, eps, newton_tol=newton_tol,
                                      newton_max_iter=newton_max_iter, nn=nn, stats=stats)
    eng = _engine_for(u0, variant, partition, eps, newton_tol, newton_max_iter, nn)
    eng.load([u0])
    eng.coarse_init()
    if stats is not None:
        _merge(stats, eng.newton)
        eng.newton = NewtonStats()
    st = PararealState(iterates=_fields(eng, eng.U.clone(), partition.num_slices + 1),
                       coarse_values=_fields(eng, eng.G.clone(), partition.num_slices),
                       fine_reference=reference, k=0, _engine=eng)
    return st


def parareal_iteration(state: PararealState, variant: AlgorithmVariant,
                       partition: TimePartition, eps: float, *, workers: int = 1,
                       newton_tol: float = 1e-10, newton_max_iter: int = 50, nn=None,
                       stats: NewtonStats | None = None) -> PararealState:
    """One prediction-correction sweep over all slices (parareal.py:216-259)."""
    del workers
    Nsl = partition.num_slices
    eng = state._engine
    fine, coarse = propagator_pair(variant, partition, eps, newton_tol=newton_tol,
                                   newton_max_iter=newton_max_iter, nn=nn)
    # the cached engine is reused only for exactly the specs this call would build
    # (the reference rebuilds propagator_pair on every call, parareal.py:229-232)
    fresh = (eng is not None and eng.k == state.k and eng.N == Nsl
             and eng.J == partition.fine_steps and eng.fine == fine and eng.coarse == coarse)
    if not fresh:
        u0 = state.iterates[0]
        eng = _engine_for(u0, variant, partition, eps, newton_tol, newton_max_iter, nn)
        for n, f in enumerate(state.iterates):
            eng.U[0, n].copy_(f.device_values(eng.device).reshape(-1))
        for n, f in enumerate(state.coarse_values):
            eng.G[0, n].copy_(f.device_values(eng.device).reshape(-1))
        eng.changed.fill_(1)
        eng.k = state.k
    eng.iterate()
    if stats is not None:
        _merge(stats, eng.newton)
        eng.newton = NewtonStats()
    return PararealState(iterates=_fields(eng, eng.U.clone(), Nsl + 1),
                         coarse_values=_fields(eng, eng.G.clone(), Nsl),
                         fine_reference=state.fine_reference, k=state.k + 1,
                         previous=state.iterates, _engine=eng)


def _dev_flat(f: Field):
    return from_device_layout(f.grid, f.device_values())


def error_against_reference(state: PararealState) -> float:
    """Discrete L-infinity(0,T; L2) error at the coarse nodes (parareal.py:262-267)."""
    g = state.iterates[0].grid
    return max(math.sqrt(g.h ** g.dim * float(((_dev_flat(u) - _dev_flat(r)) ** 2).sum()))
               for u, r in zip(state.iterates, state.fine_reference))


def iterate_increment(state: PararealState) -> float:
    """max_{n,i} |U_n^k[i] - U_n^{k-1}[i]|."""
    if state.previous is None:
        raise ValueError("state has no previous iterate (k == 0)")
    return max(float((_dev_flat(a) - _dev_flat(b)).abs().max())
               for a, b in zip(state.iterates, state.previous))


@dataclass
class IterationRecord:
    """One row of the experiment trace (parareal.py:270-280)."""

    k: int
    error: float
    energy_end: float
    mass_end: float
    wall_seconds: float
    iterate_norms: tuple
    bound: float | None = None
    increment: float | None = None


@dataclass
class RunTrace:
    """Per-iteration records plus run-level diagnostics (parareal.py:283-296)."""

    records: list
    converged_at: int | None
    tolerance: float
    reference_seconds: float
    reference_norm: float
    newton: NewtonStats
    increments: tuple = ()
    fine_point_steps: int = 0
    engine: object = field(default=None, repr=False)   # device state of the final iterate

    @property
    def errors(self) -> tuple:
        return tuple(r.error for r in self.records)


def _record(eng: PararealEngine, R, eps: float, wall: float, inc=None) -> IterationRecord:
    """make_record (parareal.py:342-351) on the device: the error against the serial
    reference, the iterate norms and the tail's energy / mass come from one fixed-order
    reduction launch over the N+1 iterates (and one over the N+1 differences)."""
    g = eng.grid
    st = field_stats(g, eng.U[0])
    norms = [stats_l2(g, st[n]) for n in range(eng.N + 1)]
    err = float("nan")
    if R is not None:
        sd = field_stats(g, eng.U[0] - R[0])
        err = max(stats_l2(g, sd[n]) for n in range(eng.N + 1))
    return IterationRecord(k=eng.k, error=err, energy_end=stats_energy(g, st[eng.N], eps),
                           mass_end=stats_mass(g, st[eng.N]), wall_seconds=wall,
                           iterate_norms=tuple(norms), increment=inc)


def run(u0: Field, variant: AlgorithmVariant, partition: TimePartition, eps: float, *,
        tol: float = 1e-6, max_iter: int | None = None, workers: int = 1,
        newton_tol: float = 1e-10, newton_max_iter: int = 50, nn=None,
        stop: str = "error", increment_tol: float = 1e-10) -> RunTrace:
    """Iterate until the error against the fine reference is <= tol
    (parareal.py:299-374), or -- ``stop="increment"`` -- until the iterate
    increment drops below ``increment_tol``."""
    del workers
    if tol <= 0:
        raise ValueError("tol must be positive")
    if stop not in ("error", "increment"):
        raise ValueError("stop must be 'error' or 'increment'")
    if max_iter is None:
        max_iter = partition.num_slices + 2
    eng = _engine_for(u0, variant, partition, eps, newton_tol, newton_max_iter, nn)
    eng.inc_tol = increment_tol if stop == "increment" else 0.0
    eng.load([u0])
    t0 = time.perf_counter()
    R, si = eng.serial_fine()
    eng._sync()
    reference_seconds = time.perf_counter() - t0
    stats = NewtonStats()
    if eng.fine.scheme is Scheme.NONLINEAR_EYRE:
        stats.absorb(si)
    ref_fields = _fields(eng, R, partition.num_slices + 1)
    reference_norm = max(l2_norm(f) for f in ref_fields)
    t0 = time.perf_counter()
    eng.coarse_init()
    records = [_record(eng, R, eps, time.perf_counter() - t0)]
    converged_at = 0 if (stop == "error" and records[0].error <= tol) else None
    while converged_at is None and eng.k < max_iter:
        t0 = time.perf_counter()
        inc = float(eng.iterate()[0])
        eng._sync()
        records.append(_record(eng, R, eps, time.perf_counter() - t0, inc))
        if stop == "error" and records[-1].error <= tol:
            converged_at = eng.k
        elif stop == "increment" and inc < increment_tol:
            converged_at = eng.k
    _merge(stats, eng.newton)
    return RunTrace(records=records, converged_at=converged_at, tolerance=tol,
                    reference_seconds=reference_seconds, reference_norm=reference_norm,
                    newton=stats, increments=tuple(float(x[0]) for x in eng.increments),
                    fine_point_steps=eng.stats.fine_point_steps, engine=eng)


@dataclass
class BatchResult:
    converged_at: list
    increments: np.ndarray        # [k, B]
    engine: PararealEngine
    seconds: float


def run_batch(u0s: list, variant: AlgorithmVariant, partition: TimePartition, eps: float, *,
              increment_tol: float = 1e-10, max_iter: int | None = None,
              newton_tol: float = 1e-10, newton_max_iter: int = 50) -> BatchResult:
    """Independent ICs in one device engine with the increment stop per IC."""
    if not u0s:
        raise ValueError("need at least one initial condition")
    eng = _engine_for(u0s[0], variant, partition, eps, newton_tol, newton_max_iter, None,
                      batch=len(u0s))
    eng.inc_tol = increment_tol
    eng.load(list(u0s))
    t0 = time.perf_counter()
    conv = eng.run(max_iter=max_iter)
    eng._sync()
    return BatchResult(conv, np.array(eng.increments), eng, time.perf_counter() - t0)
