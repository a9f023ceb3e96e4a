"""C-ABI boundary checks that need no GPU: libchp.so loads and exports every
entry point include/chp.h declares; host-side descriptors match the reference."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "chp.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(chp_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2304_14074_b200 import _native
    lib = _native.load_library()
    names = declared_symbols()
    assert len(names) >= 9
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_native.EXPORTS)
    assert lib.chp_version().decode().startswith("chp-b200")
    assert lib.chp_status_str(1).decode() == "invalid argument"


def test_struct_layouts():
    from paper_2304_14074_b200 import _native as N
    assert ctypes.sizeof(N.ChpGrid) == 4 * 4 + 7 * 8
    assert ctypes.sizeof(N.ChpSpec) == 2 * 4 + 5 * 8 + 2 * 4
    assert ctypes.sizeof(N.ChpSysInfo) == N.SYSINFO_DTYPE.itemsize == 56


def test_null_context_rejected():
    from paper_2304_14074_b200 import _native as N
    lib = N.load_library()
    assert lib.chp_propagate(None, None, None, 1, 1, None, 0, None, 0, None, None, None) == 1
    assert lib.chp_ctx_create(0, None) == 1
    assert lib.chp_nn_propagate(None, None, None, 1e-4, 1e-3, 1, 1, None, 0, None, 0, None, None,
                                None, None, None) == 1
    assert lib.chp_propagate_hist(None, None, None, 1, 1, None, 0, None, 0, None, None, None, 0,
                                  None) == 1
    assert ctypes.sizeof(N.ChpNNParams) == 4 * 4 + 3 * 8


@pytest.mark.parametrize("nx", [4, 5, 10, 17, 257, 1025, 1000])
def test_stencil_coefficients_match_reference_assembly(nx):
    from oracle import chp_oracle as O
    from paper_2304_14074_b200.grid import SpatialGrid, stencil_coefficients
    k = stencil_coefficients(SpatialGrid(1, nx))
    d = O.operators(O.Mesh(1, nx)).diag
    assert np.all(d["lap_off"] == k["c1"]) and np.all(d["lap_main"] == -2.0 * k["c1"])
    assert d["sq_main"][0] == d["sq_main"][-1] == k["s_edge"]
    if nx > 5:
        assert np.all(d["sq_main"][1:-1] == k["s_main"])
    assert np.all(d["sq_off1"] == k["s_off1"]) and np.all(d["sq_off2"] == k["s_off2"])


def test_spec_and_partition_validation():
    from paper_2304_14074_b200.parareal import AlgorithmVariant, TimePartition, propagator_pair
    from paper_2304_14074_b200.schemes import PropagatorSpec, Scheme
    from paper_2304_14074_b200.grid import SpatialGrid
    with pytest.raises(ValueError):
        PropagatorSpec(Scheme.LINEAR_A, 0.0, 0.1)
    with pytest.raises(ValueError):
        PropagatorSpec(Scheme.LINEAR_A, 0.1, -1.0)
    with pytest.raises(ValueError):
        PropagatorSpec(Scheme.NONLINEAR_EYRE, 0.1, 0.1, newton_tol=0.0)
    with pytest.raises(ValueError):
        PropagatorSpec(Scheme.NONLINEAR_EYRE, 0.1, 0.1, newton_max_iter=0)
    with pytest.raises(ValueError):
        PropagatorSpec(Scheme.NN_LINEAR_A, 0.1, 0.1)
    with pytest.raises(ValueError):
        TimePartition(0.0, 4, 4)
    with pytest.raises(ValueError):
        TimePartition(1.0, 0, 4)
    with pytest.raises(ValueError):
        SpatialGrid(3, 10)
    with pytest.raises(ValueError):
        SpatialGrid(1, 3)
    f, c = propagator_pair(AlgorithmVariant.NPA1, TimePartition(2.0, 64, 512), 0.03)
    assert f.scheme is Scheme.NONLINEAR_EYRE and c.scheme is Scheme.LINEAR_A
    assert f.dt == 2.0 / 64 / 512 and c.dt == 2.0 / 64
    s = f.native()
    assert s.b == 0.03 ** 2 * (2.0 / 64 / 512)


def test_field_validation_host():
    from paper_2304_14074_b200.grid import Field, SpatialGrid
    g = SpatialGrid(1, 10)
    with pytest.raises(ValueError, match="non-finite"):
        Field(g, np.array([np.nan] + [0.0] * 7))
    with pytest.raises(ValueError):
        Field(g, np.zeros(7))
    f = Field(g, np.arange(8.0))
    assert f.values.dtype == np.float64
    with pytest.raises(AttributeError):
        f.values = 1
