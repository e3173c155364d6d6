// Host-only half of the solver API: setup and analysis helpers that never
// touch the device (solver.cpp:437-502 estimate_dt and the initial states,
// the generic TimeStepper of solver.cpp:505-581, analysis.cpp:53-139).  Kept
// apart from solver_api.cpp (the device shim) so the CPU oracle can link the
// host setup without the C ABI / CUDA objects.
#include "prismdg/solver.hpp"

#include <algorithm>
#include <cmath>
#include <limits>

namespace prismdg {

namespace {

// LSERK45 (solver.cpp:511-523) for the generic host integrator
const double kA[5] = {0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                      -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0};
const double kB[5] = {1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                      1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                      2277821191437.0 / 14882151754819.0};
const double kC[5] = {0.0, 1432997174477.0 / 9575080441755.0, 2526269341429.0 / 6820363962896.0,
                      2006345519317.0 / 3224310063776.0, 2802321613138.0 / 2924317926251.0};

} // namespace

double estimate_dt(const Discretization& d, double cfl) {
  // solver.cpp:437-447: cfl * min_k (vol/area) / (c_k (N+1)^2)
  if (!(cfl > 0.0)) throw ConfigError("cfl must be positive");
  const double n1 = d.degree + 1;
  double dt = std::numeric_limits<double>::max();
  const int nw = d.mesh.num_wedges();
  for (int e = 0; e < d.num_elements(); ++e) {
    const double h = e < nw ? d.wgeo[e].volume / d.wgeo[e].surface_area
                            : d.tgeo[e - nw].volume / d.tgeo[e - nw].surface_area;
    const double c = d.mesh.media[e].wavespeed();
    dt = std::min(dt, h / (c * n1 * n1));
  }
  return cfl * dt;
}

FieldFunctions standing_wave(double c, double rho) {
  const double k = M_PI / 2.0;
  const double omega = std::sqrt(3.0) * k * c;
  const double amp = k / (rho * omega);
  FieldFunctions f;
  f.p = [k, omega](double x, double y, double z, double t) {
    return std::cos(k * x) * std::cos(k * y) * std::cos(k * z) * std::cos(omega * t);
  };
  f.ux = [k, omega, amp](double x, double y, double z, double t) {
    return amp * std::sin(k * x) * std::cos(k * y) * std::cos(k * z) * std::sin(omega * t);
  };
  f.uy = [k, omega, amp](double x, double y, double z, double t) {
    return amp * std::cos(k * x) * std::sin(k * y) * std::cos(k * z) * std::sin(omega * t);
  };
  f.uz = [k, omega, amp](double x, double y, double z, double t) {
    return amp * std::cos(k * x) * std::cos(k * y) * std::sin(k * z) * std::sin(omega * t);
  };
  return f;
}

FieldFunctions gaussian_pulse(double width, std::array<double, 3> c) {
  FieldFunctions f;
  const double iw2 = 1.0 / (width * width);
  f.p = [iw2, c](double x, double y, double z, double) {
    const double r2 = (x - c[0]) * (x - c[0]) + (y - c[1]) * (y - c[1]) + (z - c[2]) * (z - c[2]);
    return std::exp(-r2 * iw2);
  };
  auto zero = [](double, double, double, double) { return 0.0; };
  f.ux = f.uy = f.uz = zero;
  return f;
}

SolutionState make_initial_state(const Discretization& d, const FieldFunctions& f, double t0) {
  SolutionState s;
  s.u.assign(d.total_dofs, 0.0);
  s.time = t0;
#pragma omp parallel for schedule(dynamic, 256)
  for (int e = 0; e < d.num_elements(); ++e) {
    const int np = d.np(e);
    const std::size_t base = d.elem_offset[e];
    for (int n = 0; n < np; ++n) {
      const Vert3 x = d.node_xyz(e, n);
      s.u[base + n] = f.p(x[0], x[1], x[2], t0);
      s.u[base + np + n] = f.ux(x[0], x[1], x[2], t0);
      s.u[base + 2 * np + n] = f.uy(x[0], x[1], x[2], t0);
      s.u[base + 3 * np + n] = f.uz(x[0], x[1], x[2], t0);
    }
  }
  return s;
}

TimeStepper::TimeStepper(IntegratorKind kind, std::size_t n) : kind_(kind) {
  res_.assign(n, 0.0);
  rhs_.assign(n, 0.0);
  if (kind_ == IntegratorKind::ab3) fhist_.assign(3, std::vector<double>(n, 0.0));
}

void TimeStepper::step(std::vector<double>& u, double& t, double dt, const RhsFn& rhs, SolutionState* state) {
  // solver.cpp:536-581
  const std::size_t n = u.size();
  if (res_.size() != n) throw NumericalError("TimeStepper: state size mismatch");
  auto lserk = [&]() {
    std::fill(res_.begin(), res_.end(), 0.0);
    for (int s = 0; s < 5; ++s) {
      rhs(u, rhs_, t + kC[s] * dt);
      for (std::size_t i = 0; i < n; ++i) {
        res_[i] = kA[s] * res_[i] + dt * rhs_[i];
        u[i] += kB[s] * res_[i];
      }
    }
  };
  if (kind_ == IntegratorKind::lserk4) {
    lserk();
    t += dt;
    return;
  }
  if (state != nullptr && state->history.size() != 3) {
    state->history.assign(3, std::vector<double>(n, 0.0));
    state->history_filled = 0;
  }
  auto& h = state ? state->history : fhist_;
  int& hf = state ? state->history_filled : filled_;
  if (hf < 2) {
    rhs(u, h[2 - hf], t);
    lserk();
    t += dt;
    ++hf;
    return;
  }
  rhs(u, rhs_, t);
  for (std::size_t i = 0; i < n; ++i) u[i] += dt / 12.0 * (23.0 * rhs_[i] - 16.0 * h[1][i] + 5.0 * h[2][i]);
  std::swap(h[2], h[1]);
  std::swap(h[1], rhs_);
  t += dt;
}

double l2_error(const Discretization& d, const double* u,
                const std::function<double(double, double, double, double)>& exact_p, double time) {
  // analysis.cpp:53-91: (N+2)-Gauss in t x triangle cubature for wedges, tet cubature for tets
  const auto& refs = d.refs;
  const int nq = d.nq, nt = d.nt, nw = d.mesh.num_wedges();
  const auto& tri = refs.tri;
  const int qg = (int)refs.line.gq_nodes.size(), qc = (int)tri.cubature.weights.size();
  double acc = 0.0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : acc)
  for (int e = 0; e < d.num_elements(); ++e) {
    const std::size_t base = d.elem_offset[e];
    double part = 0.0;
    if (e < nw) {
      // Pc(qt, qs) = sum_{j,i} interp_gq(qt, j) P(j, i) interp_cub(qs, i), P(j,i) = u[i*nq + j]
      std::vector<double> tmp((std::size_t)qg * nt, 0.0);
      for (int a = 0; a < qg; ++a)
        for (int i = 0; i < nt; ++i) {
          double s = 0.0;
          for (int j = 0; j < nq; ++j) s += refs.line.interp_gq(a, j) * u[base + i * nq + j];
          tmp[(std::size_t)a * nt + i] = s;
        }
      const auto verts = d.mesh.wedge_verts(e);
      const auto& g = d.wgeo[e];
      for (int a = 0; a < qg; ++a)
        for (int b = 0; b < qc; ++b) {
          double pc = 0.0;
          for (int i = 0; i < nt; ++i) pc += tmp[(std::size_t)a * nt + i] * tri.interp_cub(b, i);
          const double r = tri.cubature.points(b, 0), s = tri.cubature.points(b, 1);
          const auto x = wedge_map(verts, r, s, refs.line.gq_nodes[a]);
          const double diff = pc - exact_p(x[0], x[1], x[2], time);
          part += refs.line.gq_weights[a] * tri.cubature.weights[b] * (g.j0 + g.jr * r + g.js * s) * diff * diff;
        }
    } else {
      const auto& tet = refs.tet;
      const auto verts = d.mesh.tet_verts(e - nw);
      const int np = tet.num_nodes;
      for (int q = 0; q < (int)tet.cubature.weights.size(); ++q) {
        double pc = 0.0;
        for (int n = 0; n < np; ++n) pc += tet.interp_cub(q, n) * u[base + n];
        const auto x = tet_map(verts, tet.cubature.points(q, 0), tet.cubature.points(q, 1), tet.cubature.points(q, 2));
        const double diff = pc - exact_p(x[0], x[1], x[2], time);
        part += tet.cubature.weights[q] * d.tgeo[e - nw].J * diff * diff;
      }
    }
    acc += part;
  }
  return std::sqrt(acc);
}

HybridMesh make_family_mesh(MeshFamily family, double h, const FamilyParams& params) {
  // analysis.cpp:110-124
  const int n = (int)std::lround(2.0 / h);
  if (n < 1 || std::abs(2.0 / n - h) > 1e-9 * h) throw ConfigError("mesh size must divide the box: h = 2/n");
  switch (family) {
    case MeshFamily::structured: return structured_wedge_box(n);
    case MeshFamily::unstructured:
      return unstructured_wedge_box(n, params.xy_jitter, params.z_amplitude, params.seed + 7919ull * (std::uint64_t)n);
    case MeshFamily::arnold: return arnold_wedge_box(n, params.arnold_delta);
  }
  throw ConfigError("bad mesh family");
}

HybridMesh spectra_mesh(std::uint64_t seed, double amplitude) {
  return perturb_vertically(structured_hybrid_box(2, 2, 2, 0), amplitude, seed);
}

double fit_rate(const std::vector<double>& h, const std::vector<double>& error) {
  const int n = (int)h.size(), m = std::min(3, n);
  if (m < 2) return 0.0;
  double sx = 0, sy = 0, sxx = 0, sxy = 0;
  for (int i = n - m; i < n; ++i) {
    const double x = std::log(h[i]), y = std::log(error[i]);
    sx += x;
    sy += y;
    sxx += x * x;
    sxy += x * y;
  }
  return (m * sxy - sx * sy) / (m * sxx - sx * sx);
}

} // namespace prismdg
