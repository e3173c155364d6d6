// The C++ drop-in shim (paper_1607_03399_b200/csrc/host/solver_api.cpp) driven
// the way the reference's own code drives its solver API
// (proj/include/prismdg/solver.hpp:61-149): build_discretization, compute_rhs,
// the phase functions, compute_energy, step() with a TimeStepper (LSERK45 and
// AB3), run_simulation.  Every call goes through the C ABI to the GPU.  The
// results are written as raw doubles to <out_dir>/*.bin and checked against the
// CPU oracle by tests/test_gpu_shim.py (this binary links only the product).
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "prismdg/solver.hpp"

using namespace prismdg;

namespace {

void dump(const std::string& path, const std::vector<double>& v) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error("cannot write " + path);
  std::fwrite(v.data(), sizeof(double), v.size(), f);
  std::fclose(f);
}

} // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: test_shim <out_dir>\n");
    return 2;
  }
  const std::string out = argv[1];
  try {
    // configs[2]'s parity mesh shape at a small size: wedge layers over a tet cap
    const Discretization d = build_discretization(structured_hybrid_box(2, 2, 1, 1, {1.0, 1.0}, {1.0, 4.0}), 3);
    const std::size_t n = d.total_dofs;
    // u ~ U[-1, 1] from mt19937_64 seed 1607
    std::mt19937_64 gen(1607);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    std::vector<double> u(n);
    for (auto& x : u) x = uni(gen);
    dump(out + "/u.bin", u);

    std::vector<double> rhs(n, 0.0);
    compute_rhs(d, u.data(), rhs.data());
    dump(out + "/rhs.bin", rhs);

    // phases: volume writes, surface accumulates, no media scaling
    std::vector<double> ph(n, 0.0);
    wedge_volume_phase(d, u.data(), ph.data());
    wedge_surface_phase(d, u.data(), ph.data());
    tet_volume_phase(d, u.data(), ph.data());
    tet_surface_phase(d, u.data(), ph.data());
    dump(out + "/phases.bin", ph);

    dump(out + "/energy.bin", {compute_energy(d, u.data())});

    // step(): 3 LSERK45 steps and 5 AB3 steps (2 bootstrap + 3 AB3)
    const double dt = estimate_dt(d, 0.5);
    SolutionState s1{u, 0.0};
    TimeStepper lserk(IntegratorKind::lserk4, n);
    for (int k = 0; k < 3; ++k) step(d, s1, dt, lserk);
    dump(out + "/lserk3.bin", s1.u);
    SolutionState s2{u, 0.0};
    TimeStepper ab3(IntegratorKind::ab3, n);
    for (int k = 0; k < 5; ++k) step(d, s2, dt * ab3.dt_scale(), ab3);
    dump(out + "/ab3_5.bin", s2.u);

    // run_simulation of the standing wave to t = 0.25 (reference dt / steps rules)
    SolutionState s3 = make_initial_state(d, standing_wave());
    RunOptions opts;
    opts.final_time = 0.25;
    opts.energy_interval = 0.05;
    const RunResult r = run_simulation(d, s3, opts);
    dump(out + "/run_state.bin", s3.u);
    dump(out + "/run_result.bin", {(double)r.steps, r.dt, r.final_time, r.initial_energy, r.final_energy,
                                   r.max_energy_increase, (double)r.energy_log.size(), s3.time});
    std::printf("test_shim ok: %zu dofs, %d steps\n", n, r.steps);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "test_shim failed: %s\n", e.what());
    return 1;
  }
  return 0;
}
