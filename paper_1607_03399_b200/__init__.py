"""prismdg-b200: B200-native time stepping for reduced-storage nodal DG on
vertically mapped wedge / tetrahedral meshes (arXiv 1607.03399).

The product is the C ABI in include/prismdg_b200.h, implemented by the in-tree
shared library paper_1607_03399_b200/_lib/libprismdg_b200.so (host C++ setup +
sm_100a CUDA kernels).  This package is a thin ctypes mirror of the
reference's C++ API; importing it loads the library and fails loudly when it
has not been built.
"""
from . import capi
from .capi import ConfigError, DeviceError, MeshError, NumericalError, PdgError
from .solver import (Discretization, DeviceContext, HybridMesh, LayerSpec, RunOptions, RunResult,
                     SolutionState, assemble_global, spectrum, arnold_wedge_box, build_discretization, compute_energy, compute_rhs,
                     estimate_dt, fit_rate, l2_error, layered_mesh, load_mesh, make_family_mesh,
                     make_initial_state, perturb_vertically, run_simulation, spectra_mesh, stack_layers,
                     structured_hybrid_box, structured_surface, structured_wedge_box, unstructured_wedge_box,
                     write_vtk_snapshot, export_arrays, discretization_from_arrays)

capi.lib()  # load now: no silent fallback

__all__ = [n for n in dir() if not n.startswith("_")]
