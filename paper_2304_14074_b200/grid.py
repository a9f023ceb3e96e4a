"""Uniform Dirichlet grids on (0,1)^d and device-aware fields.

Drop-in for ``chparareal.grid`` (reference grid.py, ``__all__`` at
grid.py:19-30).  ``Field`` keeps the reference's public fields (``grid``,
``values``) and validation (grid.py:77-86) but may hold a CUDA tensor: then
``values`` materialises a host copy lazily and the finite check runs on the
device.  Operators are never assembled on the hot path; the CUDA kernels
apply the stencils matrix-free with the same coefficients (see
``native_grid``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

__all__ = [
    "SpatialGrid",
    "Field",
    "DiscreteOperator",
    "build_laplacian",
    "laplacian_eigenvalues",
    "operator_eigenvalues",
    "l2_norm",
    "norm_of_values",
    "energy",
    "mass",
]


@dataclass(frozen=True)
class SpatialGrid:
    """Uniform mesh of (0,1)^dim; ``nodes_per_axis`` counts boundary points
    (reference grid.py:33-67)."""

    dim: int
    nodes_per_axis: int

    def __post_init__(self) -> None:
        if self.dim not in (1, 2):
            raise ValueError(f"dim must be 1 or 2, got {self.dim}")
        if self.nodes_per_axis < 4:
            raise ValueError(f"nodes_per_axis must be at least 4, got {self.nodes_per_axis}")

    @property
    def h(self) -> float:
        return 1.0 / (self.nodes_per_axis - 1)

    @property
    def interior_per_axis(self) -> int:
        return self.nodes_per_axis - 2

    @property
    def interior_count(self) -> int:
        return self.interior_per_axis ** self.dim

    @property
    def pitch(self) -> int:
        """Device row pitch: a 2D row is [0, v_1 .. v_m] (m+1 = N doubles: the
        leading zero is the Dirichlet boundary, so storage index = math index and
        rows are 16-byte aligned); 1D fields are unpadded."""
        m = self.interior_per_axis
        return m if self.dim == 1 else m + 1

    @property
    def device_size(self) -> int:
        """Doubles one device field occupies."""
        m = self.interior_per_axis
        return m if self.dim == 1 else m * self.pitch

    def interior_coordinates(self) -> np.ndarray:
        x = np.arange(1, self.nodes_per_axis - 1) * self.h
        if self.dim == 1:
            return x
        gx, gy = np.meshgrid(x, x, indexing="ij")
        return np.column_stack([gx.ravel(), gy.ravel()])


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class Field:
    """Solution values at the interior nodes of a grid (grid.py:70-86).

    ``values`` may be array-like (coerced to contiguous float64 numpy exactly as
    the reference does) or a CUDA ``torch.Tensor`` in either the flat
    (interior_count,) layout or the padded device layout ``(m, pitch)``.
    """

    __slots__ = ("grid", "_host", "_dev")

    def __init__(self, grid: SpatialGrid, values):
        object.__setattr__(self, "grid", grid)
        if _is_torch(values):
            import torch
            t = values.detach()
            if t.dtype != torch.float64:
                t = t.to(torch.float64)
            n = grid.interior_count
            m = grid.interior_per_axis
            if tuple(t.shape) == (n,):
                dev = to_device_layout(grid, t)
            elif grid.dim == 2 and tuple(t.shape) == (m, grid.pitch):
                dev = t.contiguous()
            else:
                raise ValueError(f"expected {n} interior values, got shape {tuple(t.shape)}")
            if not bool(torch.isfinite(from_device_layout(grid, dev)).all()):
                raise ValueError("field contains non-finite values")
            object.__setattr__(self, "_dev", dev)
            object.__setattr__(self, "_host", None)
        else:
            v = np.asarray(values, dtype=float)
            if v.shape != (grid.interior_count,):
                raise ValueError(f"expected {grid.interior_count} interior values, "
                                 f"got shape {v.shape}")
            if not np.all(np.isfinite(v)):
                raise ValueError("field contains non-finite values")
            object.__setattr__(self, "_host", v)
            object.__setattr__(self, "_dev", None)

    def __setattr__(self, name, value):
        raise AttributeError("Field is immutable")

    @classmethod
    def _trusted(cls, grid: SpatialGrid, dev) -> "Field":
        """Wrap a device tensor already validated on the device."""
        f = cls.__new__(cls)
        object.__setattr__(f, "grid", grid)
        object.__setattr__(f, "_dev", dev)
        object.__setattr__(f, "_host", None)
        return f

    @property
    def values(self) -> np.ndarray:
        if self._host is None:
            object.__setattr__(self, "_host",
                               from_device_layout(self.grid, self._dev).cpu().numpy())
        return self._host

    def device_values(self, device=None):
        """Padded device layout tensor (m,) / (m, pitch) on ``device``."""
        import torch
        if self._dev is None or (device is not None and self._dev.device != torch.device(device)):
            dev = to_device_layout(self.grid, torch.as_tensor(self.values), device=device)
            object.__setattr__(self, "_dev", dev)
        return self._dev

    def __repr__(self):
        where = "device" if self._dev is not None else "host"
        return f"Field(grid={self.grid!r}, {where})"


def to_device_layout(grid: SpatialGrid, flat, device=None, out=None):
    """(interior_count,) -> padded device layout on ``device`` (default cuda)."""
    import torch
    m = grid.interior_per_axis
    if device is None:
        device = flat.device if flat.is_cuda else torch.device("cuda", torch.cuda.current_device())
    if grid.dim == 1:
        t = flat.to(device=device, dtype=torch.float64, non_blocking=True)
        if out is not None:
            out.copy_(t)
            return out
        return t.contiguous()
    dst = out if out is not None else torch.zeros((m, grid.pitch), dtype=torch.float64,
                                                  device=device)
    dst[:, 0] = 0.0                                   # leading Dirichlet pad column
    dst[:, 1:].copy_(flat.view(m, m), non_blocking=True)
    return dst


def from_device_layout(grid: SpatialGrid, dev):
    """Padded device layout -> (interior_count,) view/copy on the same device."""
    if grid.dim == 1:
        return dev.reshape(-1)
    m = grid.interior_per_axis
    return dev.reshape(m, grid.pitch)[:, 1:].reshape(-1)


class DiscreteOperator:
    """Assembled Dirichlet Laplacian and its square (grid.py:89-118).

    Provided for API compatibility (user code that inspects the matrices); the
    propagators never assemble it.  Built with scipy.sparse exactly as the
    reference does."""

    def __init__(self, grid: SpatialGrid):
        import scipy.sparse as sp
        self.grid = grid
        m = grid.interior_per_axis
        h2 = grid.h ** 2
        one_d = sp.diags_array([np.ones(m - 1), -2.0 * np.ones(m), np.ones(m - 1)],
                               offsets=[-1, 0, 1]) / h2
        lap = one_d if grid.dim == 1 else (sp.kron(sp.eye_array(m), one_d)
                                          + sp.kron(one_d, sp.eye_array(m)))
        self.matrix = sp.csr_array(lap)
        self.squared = sp.csr_array(self.matrix @ self.matrix)
        if grid.dim == 1:
            self.lap_main = self.matrix.diagonal(0)
            self.lap_off = self.matrix.diagonal(1)
            self.sq_main = self.squared.diagonal(0)
            self.sq_off1 = self.squared.diagonal(1)
            self.sq_off2 = self.squared.diagonal(2)


@lru_cache(maxsize=None)
def build_laplacian(grid: SpatialGrid) -> DiscreteOperator:
    return DiscreteOperator(grid)


def laplacian_eigenvalues(grid: SpatialGrid) -> np.ndarray:
    """Analytic per-axis eigenvalues (grid.py:127-136)."""
    if grid.dim != 1:
        raise ValueError("laplacian_eigenvalues is the per-axis (1D) spectrum")
    p = np.arange(1, grid.nodes_per_axis - 1)
    return (2.0 / grid.h ** 2) * (np.cos(p * np.pi / (grid.nodes_per_axis - 1)) - 1.0)


def operator_eigenvalues(grid: SpatialGrid) -> np.ndarray:
    axis = laplacian_eigenvalues(SpatialGrid(1, grid.nodes_per_axis))
    if grid.dim == 1:
        return axis
    return (axis[:, None] + axis[None, :]).ravel()


def norm_of_values(grid: SpatialGrid, values) -> float:
    """sqrt(h^dim * sum v^2) (grid.py:147-149); device tensors reduce on device."""
    if _is_torch(values):
        return math.sqrt(grid.h ** grid.dim * float((values * values).sum()))
    return math.sqrt(grid.h ** grid.dim * float(np.dot(values, values)))


def field_stats(grid: SpatialGrid, dev, stream=None) -> np.ndarray:
    """Per-field sums behind l2_norm / energy / mass (grid.py:147-181), one fixed-order
    device reduction per field (C ABI chp_field_stats).  ``dev``: CUDA float64 tensor of
    fields in device layout (leading dims enumerate fields).  Returns [n, 4] host array:
    sum v^2, sum (v^2-1)^2, sum of squared axis differences (Dirichlet zeros at both
    ends), sum v."""
    import torch
    from . import _native as N
    fs = grid.device_size
    n = dev.numel() // fs
    out = torch.empty((n, 4), dtype=torch.float64, device=dev.device)
    ctx = N.Context.get(dev.device.index)
    ctx.check(ctx.L.chp_field_stats(ctx.h, native_grid(grid), n, N.ptr(dev), fs, N.ptr(out),
                                    N.stream_ptr(stream, dev.device)), "chp_field_stats")
    return out.cpu().numpy()


def _on_device(f: Field) -> bool:
    return f._dev is not None and f._host is None


def stats_l2(grid: SpatialGrid, st) -> float:
    return math.sqrt(grid.h ** grid.dim * float(st[0]))


def stats_energy(grid: SpatialGrid, st, eps: float) -> float:
    return grid.h ** grid.dim * (0.25 * float(st[1]) + 0.5 * eps ** 2 * float(st[2]) / grid.h ** 2)


def stats_mass(grid: SpatialGrid, st) -> float:
    return grid.h ** grid.dim * float(st[3])


def l2_norm(f: Field) -> float:
    """Cell-weighted L2 norm (grid.py:152-154); device fields reduce on the device."""
    if _on_device(f):
        return stats_l2(f.grid, field_stats(f.grid, f._dev)[0])
    return norm_of_values(f.grid, f.values)


def energy(f: Field, eps: float) -> float:
    """Discrete Ginzburg-Landau energy (grid.py:157-176); device fields reduce on the
    device (same quadrature, fixed-order sums)."""
    g = f.grid
    if _on_device(f):
        return stats_energy(g, field_stats(g, f._dev)[0], eps)
    v = f.values
    bulk = 0.25 * float(np.sum((v * v - 1.0) ** 2))
    if g.dim == 1:
        d = np.diff(v, prepend=0.0, append=0.0)
        grad2 = float(np.sum(d * d))
    else:
        arr = v.reshape(g.interior_per_axis, g.interior_per_axis)
        dx = np.diff(arr, axis=0, prepend=0.0, append=0.0)
        dy = np.diff(arr, axis=1, prepend=0.0, append=0.0)
        grad2 = float(np.sum(dx * dx) + np.sum(dy * dy))
    return g.h ** g.dim * (bulk + 0.5 * eps ** 2 * grad2 / g.h ** 2)


def mass(f: Field) -> float:
    """h^dim * sum(u) (grid.py:179-181); device fields reduce on the device."""
    if _on_device(f):
        return stats_mass(f.grid, field_stats(f.grid, f._dev)[0])
    return f.grid.h ** f.grid.dim * float(np.sum(f.values))


# ---------------------------------------------------------------------------
# C-ABI grid descriptor
# ---------------------------------------------------------------------------

def stencil_coefficients(grid: SpatialGrid) -> dict:
    """Coefficients of L and L@L with the roundings of the reference's sparse
    assembly: L data = {1, -2}/h2 (grid.py:102-105); the L@L entries are the
    sums scipy's csr_matmat forms row by row (grid.py:112), in its order."""
    h2 = grid.h ** 2
    c1 = 1.0 / h2
    q = c1 * c1
    four_q = (-2.0 * c1) * (-2.0 * c1)
    return dict(c1=c1,
                s_main=(q + four_q) + q,
                s_edge=four_q + q,
                s_off1=((-2.0 * c1) * c1) + (c1 * (-2.0 * c1)),
                s_off2=q)


def native_grid(grid: SpatialGrid):
    from ._native import ChpGrid
    k = stencil_coefficients(grid)
    return ChpGrid(grid.dim, grid.nodes_per_axis, grid.interior_per_axis, grid.pitch,
                   grid.h, grid.h ** grid.dim, k["c1"], k["s_main"], k["s_edge"],
                   k["s_off1"], k["s_off2"])
