"""Neumann-Neumann fine propagator (Scheme.NN_LINEAR_A) on the B200.

Mirror of the reference's ``chparareal.ddm`` (ddm.py): the same public names,
argument meanings and exceptions.  The step itself -- per-subdomain Dirichlet
and Neumann solves of the mixed (u, v) system, the relaxed interface
iteration on the traces and the assembly -- runs in one CUDA kernel per launch
(``csrc/chp_ddm.cu`` through ``chp_nn_propagate``), batched over systems; one
warp segment per system, one lane per subdomain.  There is no host fallback.

1D only, as the reference (ddm.py:77-80); at most 32 subdomains (one warp).
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from functools import lru_cache

import numpy as np

from . import _native as N
from .grid import Field, SpatialGrid, native_grid

__all__ = [
    "NNParams",
    "Decomposition",
    "InterfaceTraces",
    "NNConvergenceError",
    "nn_time_step",
    "nn_propagate",
    "nn_propagator",
]


@dataclass(frozen=True)
class NNParams:
    """Relaxation, tolerance and budget of the interface iteration (ddm.py:51-66)."""

    n_subdomains: int = 8
    theta: float = 0.25
    tol: float = 1e-10
    max_iter: int = 100
    warm_start: bool = False

    def __post_init__(self) -> None:
        if self.n_subdomains < 2:
            raise ValueError("need at least 2 subdomains")
        if not 0.0 < self.theta < 1.0:
            raise ValueError(f"theta must lie in (0, 1), got {self.theta}")
        if self.tol <= 0 or self.max_iter < 1:
            raise ValueError("tol must be positive and max_iter at least 1")


@dataclass(frozen=True)
class Decomposition:
    """Equal split of the 1D interior into subdomains sharing grid points
    (ddm.py:69-108)."""

    grid: SpatialGrid
    n_subdomains: int

    def __post_init__(self) -> None:
        if self.grid.dim != 1:
            raise ValueError("domain decomposition is implemented in 1D only")
        if self.n_subdomains < 2:
            raise ValueError("need at least 2 subdomains")
        cells = self.grid.nodes_per_axis - 1
        if cells % self.n_subdomains != 0:
            raise ValueError(f"{cells} mesh cells do not split evenly into "
                             f"{self.n_subdomains} subdomains")
        if cells // self.n_subdomains < 2:
            raise ValueError("subdomains must span at least 2 mesh cells")

    @property
    def nodes_per_subdomain(self) -> int:
        return (self.grid.nodes_per_axis - 1) // self.n_subdomains

    @property
    def interface_nodes(self) -> np.ndarray:
        """Global node indices of the N0-1 shared interface points."""
        return np.arange(1, self.n_subdomains) * self.nodes_per_subdomain

    def span(self, i: int) -> tuple[int, int]:
        """Global node range [a, b] of subdomain i, end points included."""
        step = self.nodes_per_subdomain
        return i * step, (i + 1) * step


@dataclass
class InterfaceTraces:
    """Current u-traces (g) and v-traces (h) at the interfaces (ddm.py:111-118)."""

    g: np.ndarray
    h: np.ndarray
    iterations: int = 0

    @classmethod
    def zeros(cls, decomp: Decomposition) -> "InterfaceTraces":
        n = decomp.n_subdomains - 1
        return cls(g=np.zeros(n), h=np.zeros(n))


class NNConvergenceError(RuntimeError):
    """The interface iteration ran out of budget (ddm.py:121-133)."""

    def __init__(self, iterations: int, g_increment: float, h_increment: float, tol: float):
        super().__init__(
            f"Neumann-Neumann iteration did not converge in {iterations} sweeps: "
            f"last increments {g_increment:.3e} (u-trace), {h_increment:.3e} "
            f"(v-trace) > tol {tol:.3e}")
        self.iterations = iterations
        self.g_increment = g_increment
        self.h_increment = h_increment


def _native_params(grid: SpatialGrid, params: NNParams) -> N.ChpNNParams:
    return N.ChpNNParams(int(params.n_subdomains), int(params.max_iter),
                         int(bool(params.warm_start)), 0, float(params.theta),
                         float(params.tol), float(grid.h ** 2))


def nn_propagate_batch(grid: SpatialGrid, params: NNParams, dt: float, eps: float, steps: int,
                       src, out, sys_index=None, info=None, traces_in=None, traces_out=None,
                       stream=None, ctx=None):
    """``steps`` NN steps on a batch of device fields (async), the batched
    counterpart of nn_propagate (ddm.py:360-372).  ``src``/``out``/``sys_index``/
    ``info`` as schemes.propagate_batch; ``traces_in``/``traces_out``: optional
    float64 CUDA tensors of shape (fields, 2, n_subdomains-1) (g then h)."""
    from .schemes import new_sysinfo
    if steps < 1:
        raise ValueError(f"steps must be at least 1, got {steps}")
    _decomposition_for(grid, params.n_subdomains)   # reference validation and messages
    ctx = ctx or N.Context.get(src.device.index)
    fs = grid.device_size
    nfields = src.numel() // fs
    nsys = nfields if sys_index is None else int(sys_index.numel())
    if info is None:
        info = new_sysinfo(nfields, src.device)
    st = ctx.L.chp_nn_propagate(ctx.h, native_grid(grid), _native_params(grid, params),
                                float(dt), float(eps ** 2), int(steps), nsys, N.ptr(src), fs,
                                N.ptr(out), fs, N.ptr(sys_index), N.ptr(traces_in),
                                N.ptr(traces_out), N.ptr(info), N.stream_ptr(stream, src.device))
    ctx.check(st, "chp_nn_propagate")
    return info


def _raise_nn(info_row, params: NNParams, where: str = "") -> None:
    code = int(info_row["status"])
    if code == N.SYS_NN:
        exc = NNConvergenceError(int(info_row["fail_iter"]), float(info_row["fail_resid"]),
                                 float(info_row["newton_maxres"]), params.tol)
        exc.args = (exc.args[0] + where,)
        raise exc
    if code == N.SYS_NONFINITE:
        raise ValueError("field contains non-finite values" + where)
    if code != N.SYS_OK:
        raise RuntimeError(f"unexpected device status {code}{where}")


def _nn_solve(u_n: Field, decomp: Decomposition, params: NNParams, dt: float, eps: float,
              traces: InterfaceTraces | None = None) -> tuple[Field, InterfaceTraces]:
    """One NN step from the given traces (ddm.py:268-340); returns the new
    field and the converged traces with their sweep count."""
    import torch
    from .schemes import read_sysinfo
    grid = decomp.grid
    if u_n.grid != grid:
        raise ValueError("field grid does not match the decomposition")
    src = u_n.device_values()
    out = torch.empty_like(src)
    S = decomp.n_subdomains
    tin = None
    if traces is not None:
        tin = torch.as_tensor(np.stack([traces.g, traces.h]).astype(np.float64),
                              device=src.device).reshape(1, 2, S - 1)
    tout = torch.empty((1, 2, S - 1), dtype=torch.float64, device=src.device)
    p = replace(params, n_subdomains=S)
    info = nn_propagate_batch(grid, p, dt, eps, 1, src, out, traces_in=tin, traces_out=tout)
    si = read_sysinfo(info)[0]
    _raise_nn(si, p)
    t = tout.cpu().numpy()[0]
    return Field._trusted(grid, out), InterfaceTraces(g=t[0].copy(), h=t[1].copy(),
                                                      iterations=int(si["newton_total"]))


@lru_cache(maxsize=None)
def _decomposition_for(grid: SpatialGrid, n_subdomains: int) -> Decomposition:
    return Decomposition(grid, n_subdomains)


def nn_time_step(u_n: Field, decomp: Decomposition, params: NNParams, dt: float,
                 eps: float) -> Field:
    """Advance one fine step with the Neumann-Neumann interface iteration
    (ddm.py:343-357); traces start from zero."""
    out, _ = _nn_solve(u_n, decomp, params, dt, eps)
    return out


def nn_propagate(u: Field, spec, steps: int) -> Field:
    """Compose fine NN steps in one launch; warm starting reuses the previous
    step's traces (ddm.py:360-372)."""
    import torch
    from .schemes import read_sysinfo
    params: NNParams = spec.nn
    _decomposition_for(u.grid, params.n_subdomains)
    src = u.device_values()
    out = torch.empty_like(src)
    info = nn_propagate_batch(u.grid, params, spec.dt, spec.eps, steps, src, out)
    _raise_nn(read_sysinfo(info)[0], params)
    return Field._trusted(u.grid, out)


def nn_propagator(decomp: Decomposition, params: NNParams, dt: float, eps: float):
    """Wrap the NN step as a propagator spec usable by the parareal engine
    (ddm.py:375-381)."""
    from .schemes import PropagatorSpec, Scheme
    if params.n_subdomains != decomp.n_subdomains:
        params = replace(params, n_subdomains=decomp.n_subdomains)
    return PropagatorSpec(scheme=Scheme.NN_LINEAR_A, dt=dt, eps=eps, nn=params)
