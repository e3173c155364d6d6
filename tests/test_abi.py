"""The C ABI library loads, exports every symbol include/prismdg_b200.h declares,
and the device path refuses to run without a GPU (no CPU fallback)."""
import ctypes

import pytest

import paper_1607_03399_b200 as pdg
from conftest import HAS_GPU
from paper_1607_03399_b200 import capi


def test_header_symbols_exported():
    syms = capi.header_symbols()
    assert len(syms) >= 40
    handle = ctypes.CDLL(capi.LIB_PATH)
    missing = [s for s in syms if not hasattr(handle, s)]
    assert not missing, missing
    assert set(syms) == set(capi.SIGNATURES), set(syms) ^ set(capi.SIGNATURES)


def test_abi_version_and_errors():
    assert capi.lib().pdg_abi_version() == 1
    with pytest.raises(pdg.ConfigError):
        pdg.build_discretization(pdg.structured_wedge_box(1), 10)
    with pytest.raises(pdg.MeshError):
        pdg.structured_hybrid_box(0, 1, 1, 0)
    with pytest.raises(pdg.ConfigError):
        pdg.perturb_vertically(pdg.structured_wedge_box(2), 0.5, 7)


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    d = pdg.build_discretization(pdg.structured_wedge_box(1), 1)
    with pytest.raises(pdg.DeviceError):
        d.device()
    import numpy as np
    with pytest.raises(pdg.DeviceError):
        pdg.compute_rhs(d, np.zeros(d.total_dofs))
