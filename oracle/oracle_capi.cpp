// CPU ORACLE (test infrastructure only; see oracle.hpp): C entry points used by
// tests/ (ctypes) and bench.py's CPU baseline.  Handles are a
// prismdg::Discretization*: either the product's pdg_disc (tests check the
// device path against the oracle on the very same Discretization) or one the
// oracle builds itself with orc_disc_stack_layers (bench.py's CPU arm, which
// must not load the product library).
#include <chrono>
#include <cstdint>
#include <exception>
#include <string>

#include "oracle.hpp"
#include "prismdg/solver.hpp"

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

int orc_mrab(const void* disc, double* u, const int* level, int nlev, double dt, int nmacro, int threads) {
  return guard([&] { oracle::mrab_steps(*D(disc), u, D(disc)->total_dofs, level, nlev, dt, nmacro, threads); });
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

/// the oracle's own Discretization of a stack_layers mesh (mesh.hpp:59-68;
/// the reference's "layers" config kind, config.cpp:232-243 + 152-178): xy[nv][2],
/// tris[ntri][3], z_bottom/z_top[nlayers][nv], sublayers[nlayers],
/// media[nlayers][2] = {rho, kappa}; exact mass, upwind flux
int orc_disc_stack_layers(int nv, const double* xy, int ntri, const int* tris, int nlayers, const double* z_bottom,
                          const double* z_top, const int* sublayers, const double* media, int degree, int threads,
                          void** out) {
  return guard([&] {
    std::vector<std::array<double, 2>> pts(nv);
    for (int v = 0; v < nv; ++v) pts[v] = {xy[2 * v], xy[2 * v + 1]};
    std::vector<std::array<int, 3>> tr(ntri);
    for (int t = 0; t < ntri; ++t) tr[t] = {tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]};
    std::vector<prismdg::LayerSpec> layers(nlayers);
    for (int l = 0; l < nlayers; ++l) {
      layers[l].z_bottom.assign(z_bottom + (std::size_t)l * nv, z_bottom + (std::size_t)(l + 1) * nv);
      layers[l].z_top.assign(z_top + (std::size_t)l * nv, z_top + (std::size_t)(l + 1) * nv);
      layers[l].sublayers = sublayers[l];
      layers[l].media.rho = media[2 * l];
      layers[l].media.kappa = media[2 * l + 1];
    }
    auto* d = new Discretization(prismdg::build_discretization(prismdg::stack_layers(pts, tr, layers), degree, {},
                                                               prismdg::QuadratureMode::exact, threads));
    *out = d;
  });
}

/// {total_dofs, num_wedges, num_tets}
int orc_disc_counts(const void* disc, long long* out) {
  return guard([&] {
    out[0] = (long long)D(disc)->total_dofs;
    out[1] = D(disc)->mesh.num_wedges();
    out[2] = D(disc)->mesh.num_tets();
  });
}

/// make_initial_state(gaussian_pulse(width, {cx, cy, cz})) (solver.cpp:469-502)
int orc_disc_gaussian(const void* disc, double width, double cx, double cy, double cz, double* u) {
  return guard([&] {
    const auto s = prismdg::make_initial_state(*D(disc), prismdg::gaussian_pulse(width, {cx, cy, cz}));
    std::copy(s.u.begin(), s.u.end(), u);
  });
}

/// estimate_dt (solver.cpp:437-447)
int orc_disc_estimate_dt(const void* disc, double cfl, double* dt) {
  return guard([&] { *dt = prismdg::estimate_dt(*D(disc), cfl); });
}

void orc_disc_free(void* disc) { delete static_cast<Discretization*>(disc); }

int orc_gll_newton(int npts, double* x, double* w) {
  return guard([&] {
    prismdg::Vec xv, wv;
    oracle::gll_newton(npts, xv, wv);
    std::copy(xv.begin(), xv.end(), x);
    std::copy(wv.begin(), wv.end(), w);
  });
}

} // extern "C"
