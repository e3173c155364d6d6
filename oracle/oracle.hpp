#pragma once
// ============================================================================
// CPU ORACLE -- TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
// arm may load or call this code, and only as the checker or the timed CPU
// baseline.  The product path (paper_1607_03399_b200, include/prismdg_b200.h)
// never calls it; the product fails loudly without a GPU.
//
// What it is: a plain C++ restatement of the reference's hot path, operation
// for operation, consuming the same host Discretization the device path is
// built from:
//   compute_rhs            proj/src/solver.cpp:362-377
//   wedge_volume_elem      proj/src/solver.cpp:164-218 (10 triangle-matrix
//                          applications per wedge, as the reference does)
//   tet_volume_elem        proj/src/solver.cpp:220-254
//   surface_elem           proj/src/solver.cpp:258-335
//   scale_media            proj/src/solver.cpp:337-346
//   LSERK45 step           proj/src/solver.cpp:536-557 (serial update loop,
//                          "faithful"; optional OpenMP update)
//   compute_energy         proj/src/solver.cpp:402-435
//   run_simulation         proj/src/solver.cpp:591-666
// plus the reference test suite's independent oracles (proj/tests/oracles.cpp):
// dense quadrature-built wedge/tet operators, GLL by Newton, random elements,
// the vertically-mapped-wedge property suite.
//
// Parity pinning: the reference cannot be compiled here (Eigen3, doctest and
// CLI11 are absent, proj/CMakeLists.txt:12-15; no network), so there is no
// oracle/_ref build.  The restatement is pinned against (a) the reference's
// own known-answer and property tests ported in tests/cpp/test_host.cpp
// (Kronecker vs dense <= 1e-11, energy == 4.0 for p = 1, storage 38 / 838,
// 1152-DOF spectra mesh, 8 wedge-tet interface faces, GLL vs Newton 1e-13,
// Lemma-1 suite 1e-13, ...) and (b) the paper's published L2 errors and rates
// in tests/golden/paper_convergence.json.
// ============================================================================

#include "prismdg/discretization.hpp"

#include <array>
#include <random>

namespace oracle {

using prismdg::Discretization;
using prismdg::Mat;
using prismdg::Vec;

void compute_rhs(const Discretization& d, const double* u, double* rhs, int threads);
void wedge_volume_phase(const Discretization& d, const double* u, double* rhs);
void wedge_surface_phase(const Discretization& d, const double* u, double* rhs);
void tet_volume_phase(const Discretization& d, const double* u, double* rhs);
void tet_surface_phase(const Discretization& d, const double* u, double* rhs);
double compute_energy(const Discretization& d, const double* u, int threads);
/// nsteps LSERK45 steps; parallel_update=false reproduces the reference's serial update
void lserk_steps(const Discretization& d, double* u, std::size_t n, double dt, int nsteps, int threads,
                 bool parallel_update);

/// nsteps of TimeStepper::step with IntegratorKind::ab3 from an empty history
/// (solver.cpp:559-581): two LSERK45 bootstrap steps recording f, then AB3
void ab3_steps(const Discretization& d, double* u, std::size_t n, double dt, int nsteps, int threads);

/// nmacro multi-rate AB3 macro steps (pdg_step_mrab's algorithm): level[e] in
/// [0, nlev) is element e's rate level (step 2^level dt); the first two macro
/// steps are the LSERK45 bootstrap at dt
void mrab_steps(const Discretization& d, double* u, std::size_t n, const int* level, int nlev, double dt, int nmacro,
                int threads);

struct RunOut {
  int steps = 0;
  double dt = 0, final_time = 0, initial_energy = 0, final_energy = 0, max_energy_increase = 0;
  bool stable = true;
};
RunOut run_simulation(const Discretization& d, std::vector<double>& u, double& time, double final_time,
                      double cfl, double fixed_dt, double energy_interval, int threads);

// ---- tests/oracles.cpp restatements -------------------------------------
void gll_newton(int npts, Vec& x, Vec& w);
struct DenseWedgeOps {
  Mat mass, dx, dy, dz;
  std::array<Mat, 5> lift;
};
DenseWedgeOps dense_wedge_ops(const prismdg::WedgeVerts& verts, const prismdg::References& refs);
struct DenseTetOps {
  Mat mass, dx, dy, dz;
  std::array<Mat, 4> lift;
};
DenseTetOps dense_tet_ops(const prismdg::TetVerts& verts, const prismdg::References& refs);
void wedge_jacobian_matrix(const prismdg::WedgeVerts& v, double r, double s, double t, double A[3][3]);
prismdg::WedgeVerts random_vertical_wedge(std::mt19937_64& gen);
prismdg::TetVerts random_tet(std::mt19937_64& gen);
double vertical_wedge_property_violation(const prismdg::WedgeVerts& verts);

} // namespace oracle
