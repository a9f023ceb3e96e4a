"""One-step propagators on the B200.

Drop-in for ``chparareal.schemes`` (reference schemes.py, ``__all__`` at
schemes.py:37-49).  Every step runs in libchp.so (sm_100a); this module only
validates specs, launches, and turns per-system device status words into the
reference's exceptions:

* ``NewtonDivergenceError(iterations, residual, tol)``  (schemes.py:122-131)
* ``ValueError("field contains non-finite values")``    (grid.py:84-85)
* ``LinearSolveError``                                   (schemes.py:118-119)

``propagate_batch`` is the batched form the Parareal engine uses: one launch
advances any number of systems (slices x initial conditions).
"""

from __future__ import annotations

import enum
import threading
from dataclasses import dataclass
from typing import TYPE_CHECKING

import numpy as np

from . import _native as N
from .grid import Field, SpatialGrid, energy, native_grid

if TYPE_CHECKING:  # pragma: no cover
    pass

__all__ = [
    "Scheme",
    "PropagatorSpec",
    "StepReport",
    "NewtonStats",
    "LinearSolveError",
    "NewtonDivergenceError",
    "step_linear_a",
    "step_linear_b",
    "step_nonlinear",
    "propagate",
    "clear_factorization_cache",
]


class Scheme(enum.Enum):
    """Which one-step method advances the field over one dt (schemes.py:52-58)."""

    LINEAR_A = "linear-a"
    LINEAR_B = "linear-b"
    NONLINEAR_EYRE = "nonlinear-eyre"
    NN_LINEAR_A = "nn-linear-a"


_NATIVE_SCHEME = {Scheme.LINEAR_A: N.CHP_LINEAR_A, Scheme.LINEAR_B: N.CHP_LINEAR_B,
                  Scheme.NONLINEAR_EYRE: N.CHP_NONLINEAR_EYRE}

# 2D variable-coefficient solves (LINEAR_A, Newton) run matrix-free CG on the
# SPD form K^-1 + B; relative residual target (SURVEY.md 8(c), 3rd hard part).
CG_TOL = 1e-14
CG_MAX_ITER = 200


@dataclass(frozen=True)
class PropagatorSpec:
    """Immutable description of a one-step propagator (schemes.py:61-86)."""

    scheme: Scheme
    dt: float
    eps: float
    newton_tol: float = 1e-10
    newton_max_iter: int = 50
    nn: object = None

    def __post_init__(self) -> None:
        if self.dt <= 0:
            raise ValueError(f"dt must be positive, got {self.dt}")
        if self.eps <= 0:
            raise ValueError(f"eps must be positive, got {self.eps}")
        if self.newton_tol <= 0:
            raise ValueError("newton_tol must be positive")
        if self.newton_max_iter < 1:
            raise ValueError("newton_max_iter must be at least 1")
        if (self.scheme is Scheme.NN_LINEAR_A) != (self.nn is not None):
            raise ValueError("nn parameters go with, and only with, the NN scheme")

    def native(self):
        if self.scheme is Scheme.NN_LINEAR_A:
            raise ValueError("NN_LINEAR_A launches through chp_nn_propagate (ddm.py)")
        return N.ChpSpec(_NATIVE_SCHEME[self.scheme], int(self.newton_max_iter), float(self.dt),
                         float(self.eps), self.eps ** 2 * self.dt, float(self.newton_tol),
                         CG_TOL, CG_MAX_ITER, 0)


@dataclass(frozen=True)
class StepReport:
    """Diagnostics of a single implicit step (schemes.py:89-97)."""

    newton_iterations: int
    residual_norm: float
    energy_before: float
    energy_after: float
    residual_history: tuple = ()


class NewtonStats:
    """Thread-safe aggregate of Newton behaviour (schemes.py:100-115)."""

    def __init__(self) -> None:
        self._lock = threading.Lock()
        self.steps = 0
        self.total_iterations = 0
        self.max_iterations = 0
        self.max_residual = 0.0

    def record(self, report: StepReport) -> None:
        with self._lock:
            self.steps += 1
            self.total_iterations += report.newton_iterations
            self.max_iterations = max(self.max_iterations, report.newton_iterations)
            self.max_residual = max(self.max_residual, report.residual_norm)

    def absorb(self, info: np.ndarray) -> None:
        """Fold device per-system aggregates (chp_sys_info) in."""
        if info.size == 0:
            return
        with self._lock:
            self.steps += int(info["newton_steps"].sum())
            self.total_iterations += int(info["newton_total"].sum())
            self.max_iterations = max(self.max_iterations, int(info["newton_max"].max()))
            self.max_residual = max(self.max_residual, float(info["newton_maxres"].max()))


class LinearSolveError(RuntimeError):
    """Implicit step system could not be solved (schemes.py:118-119)."""


class NewtonDivergenceError(RuntimeError):
    """Newton iteration did not reach the residual tolerance (schemes.py:122-131)."""

    def __init__(self, iterations: int, residual: float, tol: float):
        super().__init__(f"Newton did not converge in {iterations} iterations: "
                         f"residual {residual:.3e} > tol {tol:.3e}")
        self.iterations = iterations
        self.residual = residual


def clear_factorization_cache() -> None:
    """The device factor/table caches live in the per-device context and are
    keyed exactly like schemes._FACTOR_CACHE; they are immutable once built, so
    clearing is a no-op kept for API compatibility."""


# ---------------------------------------------------------------------------
# batched device launch
# ---------------------------------------------------------------------------

def new_sysinfo(n: int, device=None):
    import torch
    return torch.zeros((max(n, 1), 7), dtype=torch.int64, device=device)


def read_sysinfo(info) -> np.ndarray:
    return info.cpu().numpy().reshape(-1).view(N.SYSINFO_DTYPE)


def raise_on_status(info: np.ndarray, spec: PropagatorSpec, labels=None) -> None:
    """Raise the reference's exception for the first failed system."""
    bad = np.nonzero(info["status"] != N.SYS_OK)[0]
    if bad.size == 0:
        return
    s = int(bad[0])
    code = int(info["status"][s])
    where = f" (slice {labels[s]})" if labels is not None else ""
    if code == N.SYS_NEWTON:
        exc = NewtonDivergenceError(int(info["fail_iter"][s]), float(info["fail_resid"][s]),
                                    spec.newton_tol)
        exc.args = (exc.args[0] + where,)
        raise exc
    if code == N.SYS_NONFINITE:
        raise ValueError("field contains non-finite values" + where)
    if code == N.SYS_SINGULAR:
        raise LinearSolveError("direct solve failed (singular pivot)" + where)
    if code == N.SYS_CG:
        raise LinearSolveError("CG did not reach the relative residual target" + where)
    if code == N.SYS_NN:
        from .ddm import _raise_nn
        _raise_nn(info[s], spec.nn, where)
    raise RuntimeError(f"unknown device status {code}{where}")


def propagate_batch(grid: SpatialGrid, spec: PropagatorSpec, steps: int, src, out,
                    sys_index=None, info=None, stream=None, ctx=None, hist=None):
    """Advance ``steps`` steps on a batch of device fields (async).

    ``src``/``out``: CUDA float64 tensors whose leading dimension enumerates
    fields of ``grid.device_size`` doubles (contiguous).  ``sys_index``: int32
    CUDA tensor selecting which fields to advance (default all).  ``info``:
    ``new_sysinfo(len(src))`` tensor accumulating per-field outcomes.  ``hist``:
    optional float64 CUDA tensor of nsys x hist_len receiving the Newton residual
    history of the last step (chp_propagate_hist).
    """
    if steps < 1:
        raise ValueError(f"steps must be at least 1, got {steps}")
    if spec.scheme is Scheme.NN_LINEAR_A:        # schemes.py:326-329 -> ddm
        from .ddm import nn_propagate_batch
        return nn_propagate_batch(grid, spec.nn, spec.dt, spec.eps, steps, src, out,
                                  sys_index=sys_index, info=info, stream=stream, ctx=ctx)
    ctx = ctx or N.Context.get(src.device.index)
    fs = grid.device_size
    nfields = src.numel() // fs
    nsys = nfields if sys_index is None else int(sys_index.numel())
    if info is None:
        info = new_sysinfo(nfields, src.device)
    if hist is None:
        st = ctx.L.chp_propagate(ctx.h, native_grid(grid), spec.native(), int(steps), nsys,
                                 N.ptr(src), fs, N.ptr(out), fs, N.ptr(sys_index), N.ptr(info),
                                 N.stream_ptr(stream, src.device))
    else:
        st = ctx.L.chp_propagate_hist(ctx.h, native_grid(grid), spec.native(), int(steps), nsys,
                                      N.ptr(src), fs, N.ptr(out), fs, N.ptr(sys_index),
                                      N.ptr(info), N.ptr(hist), int(hist.numel() // max(nsys, 1)),
                                      N.stream_ptr(stream, src.device))
    _check_ctx(ctx, st, "chp_propagate")
    return info


def _check_ctx(ctx, st, what):
    if st == 1:
        msg = ctx.L.chp_last_error(ctx.h).decode()
        if "positive definite" in msg:
            raise np.linalg.LinAlgError(msg)
    ctx.check(st, what)


# ---------------------------------------------------------------------------
# reference-shaped single-field entry points
# ---------------------------------------------------------------------------

def _run_one(u: Field, spec: PropagatorSpec, steps: int, hist=None):
    import torch
    src = u.device_values()
    out = torch.empty_like(src)
    info = propagate_batch(u.grid, spec, steps, src, out, hist=hist)
    si = read_sysinfo(info)[:1]
    raise_on_status(si, spec)
    return Field._trusted(u.grid, out), si


def _require(spec: PropagatorSpec, scheme: Scheme) -> None:
    if spec.scheme is not scheme:
        raise ValueError(f"spec.scheme is {spec.scheme}, expected {scheme}")


def step_linear_a(u: Field, spec: PropagatorSpec) -> Field:
    """One stabilized-splitting step (schemes.py:235-246)."""
    _require(spec, Scheme.LINEAR_A)
    return _run_one(u, spec, 1)[0]


def step_linear_b(u: Field, spec: PropagatorSpec) -> Field:
    """One constant-coefficient step (schemes.py:249-267)."""
    _require(spec, Scheme.LINEAR_B)
    return _run_one(u, spec, 1)[0]


def step_nonlinear(u: Field, spec: PropagatorSpec) -> tuple[Field, StepReport]:
    """One fully implicit Eyre step solved by Newton (schemes.py:270-305); the
    device records the residual norm of every Newton iteration
    (``chp_propagate_hist``) for ``StepReport.residual_history``."""
    import torch
    _require(spec, Scheme.NONLINEAR_EYRE)
    src = u.device_values()
    hlen = int(spec.newton_max_iter) + 1
    hist = torch.full((hlen,), float("nan"), dtype=torch.float64, device=src.device)
    out, si = _run_one(u, spec, 1, hist=hist)
    it = int(si["newton_total"][0])
    res = float(si["newton_maxres"][0])
    history = tuple(float(x) for x in hist[: it + 1].cpu().numpy())
    return out, StepReport(it, res, energy(u, spec.eps), energy(out, spec.eps), history)


def propagate(u: Field, spec: PropagatorSpec, steps: int,
              stats: NewtonStats | None = None) -> Field:
    """Compose ``steps`` single steps (schemes.py:321-333) -- one launch."""
    if steps < 1:
        raise ValueError(f"steps must be at least 1, got {steps}")
    if spec.scheme is Scheme.NN_LINEAR_A:        # schemes.py:326-329
        from .ddm import nn_propagate
        return nn_propagate(u, spec, steps)
    out, si = _run_one(u, spec, steps)
    if stats is not None and spec.scheme is Scheme.NONLINEAR_EYRE:
        stats.absorb(si)
    return out
