// Host shim: the reference's solver API routed through the C ABI to the GPU.
// run_simulation / step / compute_rhs keep proj/src/solver.cpp:362-666
// semantics; the host-only helpers live in analysis_host.cpp.
#include "prismdg/solver.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <ostream>

#include "prismdg_b200.h"

namespace prismdg {

namespace {

void check(int status) {
  if (status == PDG_OK) return;
  const std::string msg = pdg_last_error();
  switch (status) {
    case PDG_ERR_CONFIG: throw ConfigError(msg);
    case PDG_ERR_NUMERICAL: throw NumericalError(msg);
    case PDG_ERR_MESH: throw MeshError(msg);
    case PDG_ERR_ANALYSIS: throw AnalysisError(msg);
    default: throw DeviceError(msg);
  }
}

} // namespace

DeviceHandle::~DeviceHandle() {
  if (ctx) pdg_destroy(ctx);
}

pdg_ctx* device_context(const Discretization& d) {
  auto& dev = const_cast<Discretization&>(d).device;
  if (!dev) {
    auto h = std::make_shared<DeviceHandle>();
    check(pdg_create(reinterpret_cast<const pdg_disc*>(&d), 0, 0, &h->ctx));
    dev = h;
  }
  return dev->ctx;
}

void compute_rhs(const Discretization& d, const double* u, double* rhs) {
  check(pdg_rhs(device_context(d), u, rhs, 0));
}

namespace {
void phase(const Discretization& d, const double* u, double* rhs, int which) {
  // the reference's phases write (volume) or accumulate into (surface) the
  // caller's rhs: load it into the device rhs buffer, run, read it back
  pdg_ctx* c = device_context(d);
  check(pdg_set_state(c, u, 0));
  check(pdg_set_rhs(c, rhs, 0));
  int st = PDG_OK;
  switch (which) {
    case 0: st = pdg_wedge_volume(c); break;
    case 1: st = pdg_wedge_surface(c); break;
    case 2: st = pdg_tet_volume(c); break;
    default: st = pdg_tet_surface(c); break;
  }
  check(st);
  check(pdg_get_rhs(c, rhs, 0));
}
} // namespace

void wedge_volume_phase(const Discretization& d, const double* u, double* rhs) { phase(d, u, rhs, 0); }
void wedge_surface_phase(const Discretization& d, const double* u, double* rhs) { phase(d, u, rhs, 1); }
void tet_volume_phase(const Discretization& d, const double* u, double* rhs) { phase(d, u, rhs, 2); }
void tet_surface_phase(const Discretization& d, const double* u, double* rhs) { phase(d, u, rhs, 3); }

double compute_energy(const Discretization& d, const double* u) {
  pdg_ctx* c = device_context(d);
  check(pdg_set_state(c, u, 0));
  double e = 0.0;
  check(pdg_energy(c, &e));
  return e;
}

void step(const Discretization& d, SolutionState& state, double dt, TimeStepper& stepper) {
  if (stepper.kind() == IntegratorKind::lserk4) {
    pdg_ctx* c = device_context(d);
    check(pdg_set_state(c, state.u.data(), 0));
    check(pdg_step_lserk(c, dt, 1, &state.time));
    check(pdg_get_state(c, state.u.data(), 0));
    return;
  }
  auto rhs = [&d](const std::vector<double>& u, std::vector<double>& out, double) {
    out.resize(u.size());
    compute_rhs(d, u.data(), out.data());
  };
  stepper.step(state.u, state.time, dt, rhs, &state);
}

RunResult run_simulation(const Discretization& d, SolutionState& state, const RunOptions& opts) {
  pdg_ctx* c = device_context(d);
  pdg_run_options o{};
  o.final_time = opts.final_time;
  o.cfl = opts.cfl;
  o.fixed_dt = opts.fixed_dt;
  o.energy_interval = opts.energy_interval;
  o.watchdog_every = opts.watchdog_every;
  o.blowup_factor = opts.blowup_factor;
  o.integrator = opts.integrator == IntegratorKind::lserk4 ? 0 : 1;
  // snapshots: the device driver streams the state to host; the trampoline
  // wraps it in a SolutionState for the reference-style callback
  struct Tramp {
    const RunOptions* opts;
    std::size_t n;
  } tramp{&opts, d.total_dofs};
  if (opts.snapshot_cb && opts.snapshot_interval > 0.0) {
    o.snapshot_interval = opts.snapshot_interval;
    o.snapshot_cb = [](const double* u, double time, int index, void* user) {
      const auto* t = static_cast<const Tramp*>(user);
      SolutionState s;
      s.u.assign(u, u + t->n);
      s.time = time;
      t->opts->snapshot_cb(s, index);
    };
    o.snapshot_user = &tramp;
  }
  pdg_run_result r{};
  const int max_log = 1 << 20;
  std::vector<double> log(2 * (std::size_t)max_log);
  check(pdg_run_simulation(c, state.u.data(), &state.time, &o, &r, log.data(), max_log));
  RunResult res;
  res.steps = r.steps;
  res.dt = r.dt;
  res.final_time = r.final_time;
  res.initial_energy = r.initial_energy;
  res.final_energy = r.final_energy;
  res.max_energy_increase = r.max_energy_increase;
  for (int q = 0; q < std::min(r.num_logged, max_log); ++q) res.energy_log.emplace_back(log[2 * q], log[2 * q + 1]);
  if (opts.energy_csv) {
    *opts.energy_csv << "time,energy\n";
    for (const auto& [t, e] : res.energy_log) {
      char buf[80];
      std::snprintf(buf, sizeof(buf), "%.17g,%.17g\n", t, e);
      *opts.energy_csv << buf;
    }
  }
  return res;
}

} // namespace prismdg
