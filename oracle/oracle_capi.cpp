// CPU ORACLE (test infrastructure only; see oracle.hpp): C entry points used by
// tests/ (ctypes) and bench.py's CPU baseline.  Handles are the product's
// pdg_disc (a prismdg::Discretization*), built by include/prismdg_b200.h.
#include <chrono>
#include <cstdint>
#include <exception>
#include <string>

#include "oracle.hpp"

using prismdg::Discretization;

namespace {
thread_local std::string g_err;
const Discretization* D(const void* p) { return static_cast<const Discretization*>(p); }
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
} // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

/// compute_rhs (solver.cpp:362-377), reference layout, OpenMP over elements
int orc_rhs(const void* disc, const double* u, double* rhs, int threads) {
  return guard([&] { oracle::compute_rhs(*D(disc), u, rhs, threads); });
}

/// phase functions (solver.cpp:379-396): 0 wedge volume, 1 wedge surface,
/// 2 tet volume, 3 tet surface
int orc_phase(const void* disc, int which, const double* u, double* rhs) {
  return guard([&] {
    switch (which) {
      case 0: oracle::wedge_volume_phase(*D(disc), u, rhs); break;
      case 1: oracle::wedge_surface_phase(*D(disc), u, rhs); break;
      case 2: oracle::tet_volume_phase(*D(disc), u, rhs); break;
      default: oracle::tet_surface_phase(*D(disc), u, rhs); break;
    }
  });
}

/// nsteps LSERK45 steps in place; parallel_update=0 is the reference's serial update
int orc_lserk(const void* disc, double* u, double dt, int nsteps, int threads, int parallel_update) {
  return guard([&] {
    oracle::lserk_steps(*D(disc), u, D(disc)->total_dofs, dt, nsteps, threads, parallel_update != 0);
  });
}

int orc_ab3(const void* disc, double* u, double dt, int nsteps, int threads) {
  return guard([&] { oracle::ab3_steps(*D(disc), u, D(disc)->total_dofs, dt, nsteps, threads); });
}

int orc_energy(const void* disc, const double* u, int threads, double* out) {
  return guard([&] { *out = oracle::compute_energy(*D(disc), u, threads); });
}

/// run_simulation on the CPU; out = {steps, dt, final_time, E0, E_final, max dE, stable}
int orc_run(const void* disc, double* u, double* time, double final_time, double cfl, double fixed_dt,
            double energy_interval, int threads, double* out) {
  return guard([&] {
    std::vector<double> st(u, u + D(disc)->total_dofs);
    const auto r = oracle::run_simulation(*D(disc), st, *time, final_time, cfl, fixed_dt, energy_interval, threads);
    std::copy(st.begin(), st.end(), u);
    out[0] = r.steps;
    out[1] = r.dt;
    out[2] = r.final_time;
    out[3] = r.initial_energy;
    out[4] = r.final_energy;
    out[5] = r.max_energy_increase;
    out[6] = r.stable ? 1.0 : 0.0;
  });
}

int orc_gll_newton(int npts, double* x, double* w) {
  return guard([&] {
    prismdg::Vec xv, wv;
    oracle::gll_newton(npts, xv, wv);
    std::copy(xv.begin(), xv.end(), x);
    std::copy(wv.begin(), wv.end(), w);
  });
}

} // extern "C"
