"""CPU oracle for the Parareal / Cahn-Hilliard hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline leg (``cpu_baseline`` / ``--impl reference``) may use it, and there
only as the checker or as the timed CPU baseline -- never as the GPU path.

It restates, array-by-array, the arithmetic of the reference package
``chparareal`` (``/root/reference/pkg/src/chparareal``) on numpy / scipy.  The
reference is pure Python on numpy+scipy, so the restatement calls the *same*
third-party routines in the *same* order:

* Dirichlet Laplacian and its square as scipy CSR arrays, assembled the way
  ``grid.py:98-118`` assembles them (the CSR column order of ``L @ L`` sets the
  summation order of every bilaplacian mat-vec, so it must be identical);
* ``LINEAR_A`` / Newton solves through LAPACK ``dgbsv`` (1D, ``schemes.py:145-154,
  178-183``) or SuperLU (2D, ``schemes.py:157-160, 184-188``);
* ``LINEAR_B`` through a cached banded Cholesky (1D ``dpbtrf``/``dpbtrs``) or a
  cached SuperLU factor (2D) (``schemes.py:191-227``).

Two knobs make the oracle usable as a like-for-like checker for the GPU:

``cube``
    ``"numpy"`` computes ``v**3`` with numpy exactly as the reference does
    (``schemes.py:260, 287``).  numpy's float64 power is host dependent (SVML
    on AVX-512 hosts, libm elsewhere), so it is only 1-ulp reproducible.
    ``"exact"`` computes the cube with a fixed sequence of IEEE operations on
    exact two-products (Dekker), which is bit-reproducible on any host and is
    what the CUDA kernels compute.
``spectral``
    ``False`` (default) uses the reference's LAPACK/SuperLU solvers.  ``True``
    replaces the constant-coefficient ``LINEAR_B`` solve by the orthonormal
    DST-I (``scipy.fft.dstn(type=1, norm="ortho")``) -- the exact
    diagonalisation used on the GPU in 2D ("CPU-DST
    oracle").
``pcg``
    ``True`` solves the 2D variable-coefficient systems (``LINEAR_A``, the
    Newton update) by DST-preconditioned CG to 1e-14 instead of SuperLU -- the
    "PCG ``_solve_shifted``" of the CPU-DST oracle, fast enough for truncated
    runs at the config-4 grid (SuperLU needs ~18 s per 511^2 solve).

With ``cube="numpy", spectral=False`` the oracle is pinned bit-for-bit against
golden vectors produced by the unmodified reference (tests/golden/).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np
import scipy.fft as sfft
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

LINEAR_A, LINEAR_B, EYRE = "linear-a", "linear-b", "nonlinear-eyre"

# fine / coarse scheme per variant -- reference parareal.py:64-70
VARIANTS = {
    "pa1": (LINEAR_A, LINEAR_A),
    "pa2": (LINEAR_B, LINEAR_B),
    "pa3": (LINEAR_B, LINEAR_A),
    "npa1": (EYRE, LINEAR_A),
    "npa2": (EYRE, EYRE),
}


class NewtonFailure(RuntimeError):
    """Mirrors reference schemes.py:122-131 (NewtonDivergenceError)."""

    def __init__(self, iterations, residual, tol):
        super().__init__(f"Newton did not converge in {iterations} iterations: "
                         f"residual {residual:.3e} > tol {tol:.3e}")
        self.iterations = iterations
        self.residual = residual


# ----------------------------------------------------------------------------
# Mesh and operators (reference grid.py:33-124)
# ----------------------------------------------------------------------------

@dataclass(frozen=True)
class Mesh:
    dim: int
    nx: int  # nodes per axis, boundary included (grid.py:37-38)

    @property
    def h(self) -> float:           # grid.py:49-51
        return 1.0 / (self.nx - 1)

    @property
    def m(self) -> int:             # grid.py:53-55
        return self.nx - 2

    @property
    def size(self) -> int:          # grid.py:57-59
        return self.m ** self.dim

    def coords(self) -> np.ndarray:  # grid.py:61-67 (x-major, "ij" indexing)
        x = np.arange(1, self.nx - 1) * self.h
        if self.dim == 1:
            return x
        gx, gy = np.meshgrid(x, x, indexing="ij")
        return np.column_stack([gx.ravel(), gy.ravel()])


@dataclass
class Operators:
    mesh: Mesh
    L: sp.csr_array
    L2: sp.csr_array
    diag: dict = field(default_factory=dict)


@lru_cache(maxsize=None)
def operators(mesh: Mesh) -> Operators:
    """Assemble L and L@L exactly as grid.py:98-118 does (same scipy calls, so
    the CSR structure -- and therefore every mat-vec's summation order -- is
    identical)."""
    m, hh = mesh.m, mesh.h ** 2
    t = sp.diags_array([np.ones(m - 1), -2.0 * np.ones(m), np.ones(m - 1)],
                       offsets=[-1, 0, 1]) / hh
    if mesh.dim == 2:
        e = sp.eye_array(m)
        t = sp.kron(e, t) + sp.kron(t, e)
    L = sp.csr_array(t)
    L2 = sp.csr_array(L @ L)
    ops = Operators(mesh, L, L2)
    if mesh.dim == 1:
        ops.diag = dict(lap_main=L.diagonal(0), lap_off=L.diagonal(1),
                        sq_main=L2.diagonal(0), sq_off1=L2.diagonal(1),
                        sq_off2=L2.diagonal(2))
    return ops


def axis_eigenvalues(nx: int) -> np.ndarray:
    """grid.py:127-136: (2/h^2)(cos(p*pi/(nx-1)) - 1), p = 1..nx-2."""
    h = 1.0 / (nx - 1)
    p = np.arange(1, nx - 1)
    return (2.0 / h ** 2) * (np.cos(p * np.pi / (nx - 1)) - 1.0)


def l2(mesh: Mesh, v: np.ndarray) -> float:
    """grid.py:147-149: sqrt(h^d * dot(v, v))."""
    return math.sqrt(mesh.h ** mesh.dim * float(np.dot(v, v)))


def ginzburg_landau_energy(mesh: Mesh, v: np.ndarray, eps: float) -> float:
    """grid.py:157-176."""
    bulk = 0.25 * float(np.sum((v * v - 1.0) ** 2))
    if mesh.dim == 1:
        d = np.diff(v, prepend=0.0, append=0.0)
        g2 = float(np.sum(d * d))
    else:
        a = v.reshape(mesh.m, mesh.m)
        dx = np.diff(a, axis=0, prepend=0.0, append=0.0)
        dy = np.diff(a, axis=1, prepend=0.0, append=0.0)
        g2 = float(np.sum(dx * dx) + np.sum(dy * dy))
    return mesh.h ** mesh.dim * (bulk + 0.5 * eps ** 2 * g2 / mesh.h ** 2)


def total_mass(mesh: Mesh, v: np.ndarray) -> float:
    """grid.py:179-181."""
    return mesh.h ** mesh.dim * float(np.sum(v))


# ----------------------------------------------------------------------------
# The cube
# ----------------------------------------------------------------------------

_SPLIT = 134217729.0  # 2**27 + 1 (Veltkamp)


def _two_prod(a, b):
    """Exact a*b = p + e (Dekker; no FMA needed).  Same value as the GPU's
    fma-based two-product because both are exact."""
    p = a * b
    c = _SPLIT * a
    ah = c - (c - a)
    al = a - ah
    c = _SPLIT * b
    bh = c - (c - b)
    bl = b - bh
    e = ((ah * bh - p) + ah * bl + al * bh) + al * bl
    return p, e


def exact_cube(v: np.ndarray) -> np.ndarray:
    """v^3 as P + ((E) + e*v), with p+e = v*v and P+E = p*v exact.

    The operation sequence is fixed, so numpy, C and CUDA produce the same bits;
    the result is the correctly rounded cube except in rare double-rounding
    cases.  (chp_common.cuh: chp_cube implements the same sequence.)"""
    p, e = _two_prod(v, v)
    P, E = _two_prod(p, v)
    return P + (E + e * v)


def cube_of(v: np.ndarray, mode: str) -> np.ndarray:
    if mode == "numpy":
        return v ** 3        # schemes.py:260 / 287
    if mode == "exact":
        return exact_cube(v)
    raise ValueError(mode)


# ----------------------------------------------------------------------------
# Linear solves (schemes.py:145-227)
# ----------------------------------------------------------------------------

def band_rows(ops: Operators, a: float, b: float, c: np.ndarray) -> np.ndarray:
    """(2,2)-band storage of I - a*L*diag(c) + b*L^2, schemes.py:145-154."""
    d = ops.diag
    n = c.shape[0]
    ab = np.zeros((5, n))
    ab[2, :] = 1.0 - a * d["lap_main"] * c + b * d["sq_main"]
    ab[1, 1:] = -a * d["lap_off"] * c[1:] + b * d["sq_off1"]
    ab[3, :-1] = -a * d["lap_off"] * c[:-1] + b * d["sq_off1"]
    ab[0, 2:] = b * d["sq_off2"]
    ab[4, :-2] = b * d["sq_off2"]
    return ab


def pcg_solve_2d(mesh: Mesh, a: float, b: float, c: np.ndarray, rhs: np.ndarray,
                 tol: float = 1e-14, max_iter: int = 500) -> np.ndarray:
    """(I - a L diag(c) + b L^2) x = rhs in 2D by DST-preconditioned CG -- the
    "PCG _solve_shifted" of the CPU-DST oracle: the SPD form
    (K^-1 + bK + a diag(c)) x = K^-1 rhs (K = -L) in the orthonormal DST-I
    basis, preconditioner 1/kappa + b kappa + a mean(c), stop at |r| <= tol |b^|.
    Plain numpy/scipy.fft; the same algorithm as the GPU's, not its code."""
    m = mesh.m
    lam = axis_eigenvalues(mesh.nx)
    kap = -(lam[:, None] + lam[None, :])
    d = 1.0 / kap + b * kap
    cc = c.reshape(m, m)

    def S(x):
        return sfft.dstn(x, type=1, norm="ortho", workers=-1)

    bh = S(rhs.reshape(m, m)) / kap
    minv = 1.0 / (d + a * float(cc.mean()))
    x = np.zeros_like(bh)
    r = bh.copy()
    z = minv * r
    p = z.copy()
    rz = float(np.sum(r * z))
    rr0 = float(np.sum(r * r))
    if rr0 > 0.0:
        for _ in range(max_iter):
            q = d * p + a * S(cc * S(p))
            alpha = rz / float(np.sum(p * q))
            x += alpha * p
            r -= alpha * q
            if not float(np.sum(r * r)) > tol * tol * rr0:
                break
            z = minv * r
            rz_new = float(np.sum(r * z))
            p = z + (rz_new / rz) * p
            rz = rz_new
    return S(x).reshape(-1)


def variable_solve(ops: Operators, a: float, b: float, c: np.ndarray,
                   rhs: np.ndarray, pcg: bool = False) -> np.ndarray:
    """(I - a L diag(c) + b L^2) x = rhs -- schemes.py:175-188 (SuperLU in 2D),
    or, with ``pcg``, the CPU-DST/PCG oracle solve (2D only)."""
    if pcg and ops.mesh.dim == 2:
        return pcg_solve_2d(ops.mesh, a, b, c, rhs)
    if ops.mesh.dim == 1:
        return sla.solve_banded((2, 2), band_rows(ops, a, b, c), rhs,
                                check_finite=False)
    n = c.shape[0]
    A = sp.eye_array(n) - a * (ops.L @ sp.diags_array(c)) + b * ops.L2
    return spla.splu(sp.csc_array(A)).solve(rhs)


_CC_CACHE: dict = {}


def constant_solver(ops: Operators, dt: float, eps: float, spectral: bool):
    """Cached solver of (I - 2dt L + eps^2 dt L^2) x = r, schemes.py:191-227
    (key schemes.py:198), or its DST-I diagonalisation when ``spectral``."""
    mesh = ops.mesh
    key = (mesh.dim, mesh.nx, float(dt), float(eps), bool(spectral))
    hit = _CC_CACHE.get(key)
    if hit is not None:
        return hit
    a, b = 2.0 * dt, eps ** 2 * dt
    if spectral:
        lam = axis_eigenvalues(mesh.nx)
        if mesh.dim == 2:
            lam = lam[:, None] + lam[None, :]
        den = 1.0 - a * lam + b * lam * lam
        shape = (mesh.m,) * mesh.dim

        def solve(r):
            rr = r.reshape(shape)
            out = sfft.idstn(sfft.dstn(rr, type=1, norm="ortho") / den,
                             type=1, norm="ortho")
            return out.reshape(-1)
    elif mesh.dim == 1:
        d = ops.diag
        ab = np.zeros((3, mesh.m))
        ab[2, :] = 1.0 - a * d["lap_main"] + b * d["sq_main"]
        ab[1, 1:] = -a * d["lap_off"] + b * d["sq_off1"]
        ab[0, 2:] = b * d["sq_off2"]
        fac = sla.cholesky_banded(ab, check_finite=False)

        def solve(r):
            return sla.cho_solve_banded((fac, False), r, check_finite=False)
    else:
        n = mesh.size
        A = sp.eye_array(n) - a * (ops.L @ sp.diags_array(np.ones(n))) + b * ops.L2
        lu = spla.splu(sp.csc_array(A))

        def solve(r):
            return lu.solve(r)
    _CC_CACHE[key] = solve
    return solve


# ----------------------------------------------------------------------------
# One-step propagators (schemes.py:235-305)
# ----------------------------------------------------------------------------

@dataclass
class Knobs:
    cube: str = "numpy"
    spectral: bool = False
    pcg: bool = False          # 2D variable-coefficient solves by DST-preconditioned CG
    newton_tol: float = 1e-10
    newton_max_iter: int = 50
    nn: object = None          # NNSetup: the fine propagator is NN_LINEAR_A (parareal.py:111-125)


@dataclass
class NewtonCounter:
    """Aggregates as schemes.py:100-115 (steps, total, max, max residual)."""
    steps: int = 0
    total: int = 0
    max_iter: int = 0
    max_residual: float = 0.0
    per_step: list = field(default_factory=list)

    def add(self, it, res):
        self.steps += 1
        self.total += it
        self.max_iter = max(self.max_iter, it)
        self.max_residual = max(self.max_residual, res)
        self.per_step.append(it)


def step_a(mesh, v, dt, eps, knobs: Knobs):
    """schemes.py:235-246."""
    ops = operators(mesh)
    rhs = v - dt * (ops.L @ v)
    return variable_solve(ops, dt, eps ** 2 * dt, v * v, rhs, knobs.pcg)


def step_b(mesh, v, dt, eps, knobs: Knobs):
    """schemes.py:249-267."""
    ops = operators(mesh)
    rhs = v + dt * (ops.L @ (cube_of(v, knobs.cube) - 3.0 * v))
    return constant_solver(ops, dt, eps, knobs.spectral)(rhs)


def step_eyre(mesh, u, dt, eps, knobs: Knobs, counter: NewtonCounter | None = None):
    """schemes.py:270-305: undamped Newton, residual before every solve."""
    ops = operators(mesh)
    d = dt
    b = eps ** 2 * d
    yhat = u - d * (ops.L @ u)
    y = u
    for it in range(knobs.newton_max_iter + 1):
        cu = cube_of(y, knobs.cube)
        H = y + b * (ops.L2 @ y) - d * (ops.L @ cu) - yhat
        r = l2(mesh, H)
        if r <= knobs.newton_tol:
            if counter is not None:
                counter.add(it, r)
            return y
        if it == knobs.newton_max_iter or not np.isfinite(r):
            raise NewtonFailure(it, r, knobs.newton_tol)
        rhs = yhat - 2.0 * d * (ops.L @ cu)
        y = variable_solve(ops, 3.0 * d, b, y * y, rhs, knobs.pcg)
    raise AssertionError("unreachable")


def check_finite(v):
    """grid.py:84-85 -- every step result is wrapped in a validated Field."""
    if not np.all(np.isfinite(v)):
        raise ValueError("field contains non-finite values")
    return v


def advance(mesh, v, scheme, dt, eps, steps, knobs: Knobs, counter=None):
    """schemes.py:308-333: compose ``steps`` single steps."""
    if steps < 1:
        raise ValueError(f"steps must be at least 1, got {steps}")
    for _ in range(steps):
        if scheme == LINEAR_A:
            v = step_a(mesh, v, dt, eps, knobs)
        elif scheme == LINEAR_B:
            v = step_b(mesh, v, dt, eps, knobs)
        elif scheme == EYRE:
            v = step_eyre(mesh, v, dt, eps, knobs, counter)
        else:
            raise ValueError(scheme)
        v = check_finite(v)
    return v


# ----------------------------------------------------------------------------
# Neumann-Neumann fine step (ddm.py) -- Scheme.NN_LINEAR_A, 1D only
# ----------------------------------------------------------------------------

@dataclass(frozen=True)
class NNSetup:
    """ddm.py:51-66 (NNParams)."""
    n_subdomains: int = 8
    theta: float = 0.25
    tol: float = 1e-10
    max_iter: int = 100
    warm_start: bool = False


class NNFailure(RuntimeError):
    """ddm.py:121-133 (NNConvergenceError): sweeps, g/h increments."""

    def __init__(self, sweeps, g_inc, h_inc):
        super().__init__(f"NN did not converge in {sweeps} sweeps: {g_inc:.3e}, {h_inc:.3e}")
        self.sweeps, self.g_inc, self.h_inc = sweeps, g_inc, h_inc


def _mixed_block(k: int, hh: float, dt: float, eps2: float, c2: np.ndarray) -> np.ndarray:
    """The 2k x 2k mixed (u, v) matrix [[I, -dt*Lap], [eps2*Lap - diag(c2), I]]
    with the dense tridiagonal Lap = (1/h^2) tridiag(1, -2, 1) (ddm.py:136-142,
    167-173, 211-217)."""
    lap = np.zeros((k, k))
    r = np.arange(k)
    lap[r, r] = -2.0 / hh
    lap[r[:-1], r[:-1] + 1] = 1.0 / hh
    lap[r[1:], r[1:] - 1] = 1.0 / hh
    A = np.zeros((2 * k, 2 * k))
    A[:k, :k] = np.eye(k)
    A[:k, k:] = -dt * lap
    A[k:, :k] = eps2 * lap - np.diag(c2)
    A[k:, k:] = np.eye(k)
    return A


def nn_subdomain(nodes: int, i: int, n_sub: int, uf: np.ndarray, hh: float, dt: float,
                 eps2: float):
    """Dirichlet solution at zero traces + its trace responses, and the Neumann
    interface responses, of subdomain i (ddm.py:147-256).  ``uf``: the field
    with its two boundary zeros (nodes entries); dense LAPACK LU (getrf/getrs
    through scipy.linalg.lu_factor / lu_solve) exactly as the reference."""
    step = (nodes - 1) // n_sub
    a, b = i * step, (i + 1) * step
    c2f = uf * uf
    k = b - a - 1
    Ad = _mixed_block(k, hh, dt, eps2, c2f[a + 1:b])
    R = np.zeros((2 * k, 5))
    R[:k, 0] = uf[a + 1:b]
    R[k:, 0] = -uf[a + 1:b]
    R[k, 1] = -eps2 / hh
    R[0, 2] = dt / hh
    R[2 * k - 1, 3] = -eps2 / hh
    R[k - 1, 4] = dt / hh
    X = sla.lu_solve(sla.lu_factor(Ad, check_finite=False), R, check_finite=False)
    ends = [0, k - 1, k, 2 * k - 1]
    lo_if, hi_if = a > 0, b < nodes - 1
    an = a if lo_if else a + 1
    bn = b if hi_if else b - 1
    kn = bn - an + 1
    c2n = c2f[an:bn + 1]
    An = _mixed_block(kn, hh, dt, eps2, c2n)
    for side, p, q in ((lo_if, 0, 1), (hi_if, kn - 1, kn - 2)):
        if not side:
            continue
        # half-stencil interface rows (ddm.py:218-236)
        An[p, :] = 0.0
        An[p, p] = 0.5
        An[p, kn + p] = dt / hh
        An[p, kn + q] = -dt / hh
        An[kn + p, :] = 0.0
        An[kn + p, p] = -eps2 / hh - 0.5 * c2n[p]
        An[kn + p, q] = eps2 / hh
        An[kn + p, kn + p] = 0.5
    loads = np.zeros((2 * kn, 4))
    if lo_if:
        loads[0, 0] = 1.0
        loads[kn, 1] = 1.0
    if hi_if:
        loads[kn - 1, 2] = 1.0
        loads[2 * kn - 1, 3] = 1.0
    Y = sla.lu_solve(sla.lu_factor(An, check_finite=False), loads, check_finite=False)
    return dict(a=a, b=b, sol0=X[:, 0], resp=X[:, 1:], edge0=X[ends, 0],
                edge_resp=X[ends, 1:], neu=Y[[0, kn - 1, kn, 2 * kn - 1], :])


def nn_step(mesh: Mesh, v: np.ndarray, dt: float, eps: float, nn: NNSetup, g=None, h=None):
    """ddm.py:259-340 (_nn_solve): relaxed interface iteration on the traces,
    then assembly.  Returns (values, g, h, sweeps)."""
    if mesh.dim != 1:
        raise ValueError("domain decomposition is implemented in 1D only")
    nodes, hh, eps2, S = mesh.nx, mesh.h ** 2, eps ** 2, nn.n_subdomains
    step = (nodes - 1) // S
    iface = np.arange(1, S) * step
    uf = np.zeros(nodes)
    uf[1:-1] = v
    c2f = uf * uf
    subs = [nn_subdomain(nodes, i, S, uf, hh, dt, eps2) for i in range(S)]
    g = np.zeros(S - 1) if g is None else g.copy()
    h = np.zeros(S - 1) if h is None else h.copy()

    def traces(i):     # ddm.py:259-265
        return np.array([g[i - 1] if i > 0 else 0.0, h[i - 1] if i > 0 else 0.0,
                         g[i] if i < S - 1 else 0.0, h[i] if i < S - 1 else 0.0])

    gi = hi = np.inf
    for sweep in range(1, nn.max_iter + 1):
        E = np.array([sd["edge0"] + sd["edge_resp"] @ traces(i) for i, sd in enumerate(subs)])
        ju = g - dt * (E[:-1, 3] + E[1:, 2] - 2.0 * h) / hh - uf[iface]
        jv = eps2 * (E[:-1, 1] + E[1:, 0] - 2.0 * g) / hh - c2f[iface] * g + h + uf[iface]
        P = np.zeros((S, 4))
        for i, sd in enumerate(subs):
            ld = np.array([-ju[i - 1] if i > 0 else 0.0, -jv[i - 1] if i > 0 else 0.0,
                           ju[i] if i < S - 1 else 0.0, jv[i] if i < S - 1 else 0.0])
            P[i] = sd["neu"] @ ld
        dg = nn.theta * (P[:-1, 1] - P[1:, 0])
        dh = nn.theta * (P[:-1, 3] - P[1:, 2])
        g -= dg
        h -= dh
        gi = math.sqrt(mesh.h * float(np.dot(dg, dg)))
        hi = math.sqrt(mesh.h * float(np.dot(dh, dh)))
        if gi <= nn.tol and hi <= nn.tol:
            break
    else:
        raise NNFailure(nn.max_iter, gi, hi)
    out = np.empty(mesh.size)
    for i, sd in enumerate(subs):
        sol = sd["sol0"] + sd["resp"] @ traces(i)
        k = sd["b"] - sd["a"] - 1
        out[sd["a"]:sd["b"] - 1] = sol[:k]
    out[iface - 1] = g
    return out, g, h, sweep


def nn_advance(mesh: Mesh, v: np.ndarray, dt: float, eps: float, nn: NNSetup, steps: int,
               sweeps: list | None = None):
    """ddm.py:360-372 (nn_propagate): traces restart from zero each step unless
    warm_start carries them over."""
    g = h = None
    for _ in range(steps):
        v, g1, h1, sw = nn_step(mesh, v, dt, eps, nn, g, h)
        v = check_finite(v)
        if sweeps is not None:
            sweeps.append(sw)
        if nn.warm_start:
            g, h = g1, h1
    return v


# ----------------------------------------------------------------------------
# Parareal (parareal.py:145-374) with the increment stop of SURVEY.md 8(a) a20
# ----------------------------------------------------------------------------

@dataclass
class PararealResult:
    k: int | None                 # iteration where the increment test fired
    increments: list              # delta^k for k = 1..
    iterates: np.ndarray          # final U_n, shape (N+1, size)
    history: list                 # iterates after each iteration (optional)
    serial: np.ndarray | None     # serial fine reference at coarse nodes
    errors: list                  # L_inf(0,T;L2) error vs serial per k
    newton: NewtonCounter
    fine_props: int               # fine slice-propagations actually computed
    seconds: float


def fine_advance(mesh, v, fine, dt, eps, J, knobs: Knobs, counter=None):
    """F: the variant's fine scheme, or the NN step when ``knobs.nn`` is set
    (parareal.py:111-125 replaces the fine spec by Scheme.NN_LINEAR_A)."""
    if knobs.nn is not None:
        return nn_advance(mesh, v, dt, eps, knobs.nn, J)
    return advance(mesh, v, fine, dt, eps, J, knobs, counter)


def serial_fine(mesh, u0, variant, T, N, J, eps, knobs: Knobs, counter=None):
    """parareal.py:145-164."""
    fine = VARIANTS[variant][0]
    out = [u0]
    for _ in range(N):
        out.append(fine_advance(mesh, out[-1], fine, T / N / J, eps, J, knobs, counter))
    return np.array(out)


def coarse_start(mesh, u0, variant, T, N, eps, knobs: Knobs, counter=None):
    """parareal.py:167-185: U_n^0 = G^n(u0)."""
    coarse = VARIANTS[variant][1]
    out = [u0]
    for _ in range(N):
        out.append(advance(mesh, out[-1], coarse, T / N, eps, 1, knobs, counter))
    return np.array(out)


def parareal(mesh, u0, variant, T, N, J, eps, knobs: Knobs | None = None, *,
             inc_tol=1e-10, max_iter=None, keep_history=False, with_serial=False,
             skip_stable=True, on_iteration=None, workers=1):
    """Parareal to the increment test max_{n,i}|U^{k+1}-U^k| < inc_tol.

    The update is parareal.py:236-251 verbatim in arithmetic:
    ``U_{n+1} = (G(U_n^{k+1}) + F(U_n^k)) - G(U_n^k)`` with the cached
    coarse values (parareal.py:207-212, 338-340).  ``skip_stable`` reuses
    F(U_n) / G(U_n) whenever U_n is bit-identical to its previous value; since F
    and G are deterministic this changes no value.
    """
    knobs = knobs or Knobs()
    fine, coarse = VARIANTS[variant]
    dT = T / N
    dt = dT / J
    if max_iter is None:
        max_iter = N + 2
    counter = NewtonCounter()
    t0 = time.perf_counter()
    serial = serial_fine(mesh, u0, variant, T, N, J, eps, knobs) if with_serial else None
    U = coarse_start(mesh, u0, variant, T, N, eps, knobs, counter)
    G = U[1:].copy()
    Fv = np.zeros_like(G)
    changed = np.ones(N + 1, bool)   # U_n changed since F/G were computed
    incs, hist, errs = [], [], []
    fine_props = 0
    k_done = None
    k = 0
    while k < max_iter:
        todo = [n for n in range(N) if changed[n] or not skip_stable]
        if workers > 1:
            # the reference's thread pool over slices (parareal.py:239-243)
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(max_workers=workers) as pool:
                outs = list(pool.map(lambda n: fine_advance(mesh, U[n], fine, dt, eps, J, knobs,
                                                            counter), todo))
            for n, v in zip(todo, outs):
                Fv[n] = v
        else:
            for n in todo:
                Fv[n] = fine_advance(mesh, U[n], fine, dt, eps, J, knobs, counter)
        fine_props += len(todo)
        newU = U.copy()
        new_changed = np.zeros(N + 1, bool)
        for n in range(N):
            if skip_stable and not new_changed[n]:
                g = G[n]          # G(U_n^{k+1}) == G(U_n^k): same input bits
            else:
                g = advance(mesh, newU[n], coarse, dT, eps, 1, knobs, counter)
            val = check_finite((g + Fv[n]) - G[n])
            new_changed[n + 1] = not np.array_equal(val.view(np.int64),
                                                    U[n + 1].view(np.int64))
            newU[n + 1] = val
            G[n] = g
        inc = float(np.max(np.abs(newU - U)))
        U = newU
        changed = new_changed
        k += 1
        incs.append(inc)
        if keep_history:
            hist.append(U.copy())
        if serial is not None:
            errs.append(max(l2(mesh, U[n] - serial[n]) for n in range(N + 1)))
        if on_iteration is not None:
            on_iteration(k, inc, U)
        if inc < inc_tol:
            k_done = k
            break
    return PararealResult(k_done, incs, U, hist, serial, errs, counter, fine_props,
                          time.perf_counter() - t0)


# ----------------------------------------------------------------------------
# Seeded inputs of BASELINE.json configs
# ----------------------------------------------------------------------------

CONFIGS = {
    1: dict(dim=1, nx=257, eps=0.05, T=1.0, N=16, J=256, variant="pa3"),
    2: dict(dim=1, nx=1025, eps=0.03, T=2.0, N=64, J=512, variant="npa1", batch=64),
    3: dict(dim=2, nx=257, eps=0.02, T=0.5, N=64, J=128, variant="pa3"),
    4: dict(dim=2, nx=513, eps=0.015, T=0.5, N=128, J=128, variant="npa1"),
    5: dict(dim=2, nx=1025, eps=0.01, T=2.0, N=512, J=256, variant="pa3"),
}


def initial_condition(cfg: int, ic: int = 0) -> np.ndarray:
    c = CONFIGS[cfg]
    mesh = Mesh(c["dim"], c["nx"])
    n = mesh.size
    if cfg == 1:
        x = mesh.coords()
        return 0.1 * np.sin(2 * np.pi * x) + np.random.default_rng(ic).uniform(-0.01, 0.01, n)
    if cfg == 2:
        return np.random.default_rng(ic).uniform(-0.05, 0.05, n)
    if cfg == 3:
        v = np.random.default_rng(ic).uniform(-0.05, 0.05, n)
        return v - v.mean()
    if cfg == 4:
        return np.random.default_rng(ic).uniform(-0.05, 0.05, n)
    if cfg == 5:
        return 0.1 + np.random.default_rng(ic).uniform(-0.05, 0.05, n)
    raise ValueError(cfg)
