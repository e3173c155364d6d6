#pragma once
// Host-side solver API of the B200 framework -- the drop-in for the reference's
// time-stepping path (proj/include/prismdg/solver.hpp:61-149).
//
// compute_rhs / the phase functions / compute_energy / step / run_simulation
// keep the reference's signatures and semantics but execute on the GPU through
// the C ABI in include/prismdg_b200.h (no CPU fallback: they throw
// DeviceError when no sm_100 device is present).  Setup-side helpers
// (estimate_dt, initial states, l2_error) stay on the host like the reference.

#include "prismdg/discretization.hpp"

#include <array>
#include <complex>
#include <cstdint>
#include <functional>
#include <iosfwd>
#include <string>
#include <vector>

struct pdg_ctx;

namespace prismdg {

enum class IntegratorKind { lserk4, ab3 };

/// the device context the shim keeps per Discretization
struct DeviceHandle {
  pdg_ctx* ctx = nullptr;
  ~DeviceHandle();
};
pdg_ctx* device_context(const Discretization& d);

void compute_rhs(const Discretization& d, const double* u, double* rhs);         // solver.hpp:67
void wedge_volume_phase(const Discretization& d, const double* u, double* rhs);  // solver.hpp:71
void wedge_surface_phase(const Discretization& d, const double* u, double* rhs);
void tet_volume_phase(const Discretization& d, const double* u, double* rhs);
void tet_surface_phase(const Discretization& d, const double* u, double* rhs);
double compute_energy(const Discretization& d, const double* u);                 // solver.hpp:78
double estimate_dt(const Discretization& d, double cfl);                         // solver.hpp:81

struct SolutionState {
  std::vector<double> u;
  double time = 0.0;
  std::vector<std::vector<double>> history;
  int history_filled = 0;
};

struct FieldFunctions {
  std::function<double(double, double, double, double)> p, ux, uy, uz;
};
FieldFunctions standing_wave(double c = 1.0, double rho = 1.0);          // solver.cpp:449-467
FieldFunctions gaussian_pulse(double width, std::array<double, 3> center = {0.0, 0.0, 0.0});
SolutionState make_initial_state(const Discretization& d, const FieldFunctions& f, double t0 = 0.0);

using RhsFn = std::function<void(const std::vector<double>&, std::vector<double>&, double)>;

/// Generic explicit integrator over host vectors (solver.hpp:106-121).
class TimeStepper {
 public:
  TimeStepper(IntegratorKind kind, std::size_t n);
  void step(std::vector<double>& u, double& t, double dt, const RhsFn& rhs, SolutionState* state = nullptr);
  double dt_scale() const { return kind_ == IntegratorKind::ab3 ? 0.25 : 1.0; }
  IntegratorKind kind() const { return kind_; }

 private:
  IntegratorKind kind_;
  std::vector<double> res_, rhs_;
  std::vector<std::vector<double>> fhist_;
  int filled_ = 0;
};

/// One step on the device (LSERK45); AB3 runs through the generic stepper.
void step(const Discretization& d, SolutionState& state, double dt, TimeStepper& stepper);

struct RunOptions {
  double final_time = 1.0;
  double cfl = 0.5;
  IntegratorKind integrator = IntegratorKind::lserk4;
  double fixed_dt = 0.0;
  double energy_interval = 0.0;
  std::ostream* energy_csv = nullptr;
  int watchdog_every = 50;
  double blowup_factor = 10.0;
  double snapshot_interval = 0.0; // 0: no snapshots (solver.hpp:133-134)
  std::function<void(const SolutionState&, int)> snapshot_cb;
};

struct RunResult {
  int steps = 0;
  double dt = 0.0;
  double final_time = 0.0;
  double initial_energy = 0.0;
  double final_energy = 0.0;
  double max_energy_increase = 0.0;
  std::vector<std::pair<double, double>> energy_log;
};

RunResult run_simulation(const Discretization& d, SolutionState& state, const RunOptions& opts);

/// Legacy-ASCII VTK unstructured grid of the nodal lattice sub-cells with point
/// data p, u_x, u_y, u_z from the reference-layout state u (the reference's
/// snapshot writer format; csrc/host/snapshot.cpp)
void write_vtk_snapshot(const Discretization& d, const double* u, const std::string& path);

// ---- analysis helpers that stay on the host (analysis.hpp:30-87) ----------
double l2_error(const Discretization& d, const double* u,
                const std::function<double(double, double, double, double)>& exact_p, double time);
enum class MeshFamily { structured = 0, unstructured = 1, arnold = 2 };
struct FamilyParams {
  std::uint64_t seed = 20160311;
  double xy_jitter = 0.15;
  double z_amplitude = 0.3;
  double arnold_delta = 0.25;
};
HybridMesh make_family_mesh(MeshFamily family, double h, const FamilyParams& params = {});
HybridMesh spectra_mesh(std::uint64_t seed = 42, double amplitude = 0.3);
double fit_rate(const std::vector<double>& h, const std::vector<double>& error);

} // namespace prismdg
