"""B200-native Parareal solver for the Cahn-Hilliard equation.

Drop-in for the hot path of the arXiv 2304.14074 reference package
``chparareal``: modules ``grid``, ``schemes`` and ``parareal`` mirror the
reference modules of the same names; the arithmetic runs in hand-written
sm_100a CUDA kernels in ``libchp.so`` (see ``include/chp.h``).
"""

__version__ = "0.1.0"

from . import grid, schemes, parareal, ddm  # noqa: F401,E402
