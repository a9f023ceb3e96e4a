"""BASELINE.json configs 1-5 and their seeded synthetic initial conditions
(SURVEY.md 8(d)): the workloads bench.py and the time-to-tolerance runs use.

BASELINE.json names no dataset; these generators are the whole input.  Draws follow
the reference's interior ordering (grid.py:61-67, x-major), so "zero at the boundary"
is automatic (interior-only storage).
"""

from __future__ import annotations

import numpy as np

# variant per config: PA3 (LINEAR_B fine / LINEAR_A coarse) for the linear configs,
# NPA1 (Newton-Eyre fine / LINEAR_A coarse) for the nonlinear ones
CONFIGS = {
    1: dict(dim=1, nx=257, eps=0.05, T=1.0, N=16, J=256, variant="pa3"),
    2: dict(dim=1, nx=1025, eps=0.03, T=2.0, N=64, J=512, variant="npa1", batch=64),
    3: dict(dim=2, nx=257, eps=0.02, T=0.5, N=64, J=128, variant="pa3"),
    4: dict(dim=2, nx=513, eps=0.015, T=0.5, N=128, J=128, variant="npa1"),
    5: dict(dim=2, nx=1025, eps=0.01, T=2.0, N=512, J=256, variant="pa3"),
}


def initial_condition(cfg: int, ic: int = 0) -> np.ndarray:
    """Seeded u0 of config ``cfg`` (initial condition ``ic`` of config 2's batch), as
    the reference's interior value vector."""
    c = CONFIGS[cfg]
    m = c["nx"] - 2
    n = m ** c["dim"]
    if cfg == 1:
        x = np.arange(1, c["nx"] - 1) * (1.0 / (c["nx"] - 1))
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
    raise ValueError(f"unknown config {cfg}")
