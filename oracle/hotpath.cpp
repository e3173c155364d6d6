// CPU ORACLE (test infrastructure only; see oracle.hpp): restatement of the
// reference's RHS, LSERK45 and energy, proj/src/solver.cpp:164-666.
#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "oracle.hpp"
#include "prismdg/solver.hpp"

namespace oracle {

using namespace prismdg;

namespace {

// Column-major (nq x nt) blocks as the reference's Eigen maps:
// X(j, i) lives at x[i*nq + j] (solver.cpp:173-180).
struct Block {
  int nq, nt;
  std::vector<double> v;
  Block(int q, int t) : nq(q), nt(t), v((std::size_t)q * t, 0.0) {}
  double& operator()(int j, int i) { return v[(std::size_t)i * nq + j]; }
  double operator()(int j, int i) const { return v[(std::size_t)i * nq + j]; }
};

// per-thread workspace, allocated once per compute_rhs call like the
// reference's thread_local workspace (solver.cpp:26-44)
struct Scratch {
  Block dr, ds, dt, w, tmp, rp;
  std::vector<double> fp, fu, lift_u, va, vb, vc, vd, tv;
  Scratch(int nq, int nt, int max_np, int max_nfp)
      : dr(nq, nt), ds(nq, nt), dt(nq, nt), w(nq, nt), tmp(nq, nt), rp(nq, nt), fp(max_nfp), fu(max_nfp),
        lift_u(max_np), va(max_np), vb(max_np), vc(max_np), vd(max_np), tv(nt) {}
};

// out(j,i) = sum_k X(j,k) M(i,k)   ("X * M^T")
void times_transpose(const double* X, int nq, int nt, const Mat& M, Block& out) {
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j < nq; ++j) {
      double s = 0.0;
      for (int k = 0; k < nt; ++k) s += X[(std::size_t)k * nq + j] * M(i, k);
      out(j, i) = s;
    }
}

// out(j,i) = sum_l D(j,l) X(l,i)
void left_times(const Mat& D, const double* X, int nq, int nt, Block& out) {
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j < nq; ++j) {
      double s = 0.0;
      for (int l = 0; l < nq; ++l) s += D(j, l) * X[(std::size_t)i * nq + l];
      out(j, i) = s;
    }
}

// L(i,k) of wedge w from the flat column-major storage
inline double Lik(const Discretization& d, int w, int i, int k) {
  return d.tri_lift[(std::size_t)w * d.nt * d.nt + (std::size_t)k * d.nt + i];
}

// out(j,i) = sum_k A(j,k) L(i,k)
void times_LT(const Discretization& d, int w, const Block& A, Block& out) {
  for (int i = 0; i < d.nt; ++i)
    for (int j = 0; j < d.nq; ++j) {
      double s = 0.0;
      for (int k = 0; k < d.nt; ++k) s += A(j, k) * Lik(d, w, i, k);
      out(j, i) = s;
    }
}

void wedge_volume_elem(const Discretization& d, int e, const double* u, double* rhs, Scratch& ws) {
  // solver.cpp:164-218
  const auto& refs = d.refs;
  const int nq = d.nq, nt = d.nt, np = d.np_wedge;
  const std::size_t base = d.elem_offset[e];
  const WedgeGeo& g = d.wgeo[e];
  const double* txJ = d.txJ.data() + (std::size_t)e * nq;
  const double* tyJ = d.tyJ.data() + (std::size_t)e * nq;
  const double* P = u + base;
  const double* UX = u + base + np;
  const double* UY = u + base + 2 * np;
  const double* UZ = u + base + 3 * np;
  double* RP = rhs + base;
  double* RUX = rhs + base + np;
  double* RUY = rhs + base + 2 * np;
  double* RUZ = rhs + base + 3 * np;
  Block& tmp = ws.tmp;

  // pressure gradient
  times_transpose(P, nq, nt, refs.tri.dr, ws.dr);
  times_transpose(P, nq, nt, refs.tri.ds, ws.ds);
  left_times(refs.line.diff, P, nq, nt, ws.dt);
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j < nq; ++j) ws.w(j, i) = txJ[j] * ws.dt(j, i);
  times_LT(d, e, ws.w, tmp);
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j < nq; ++j) RUX[i * nq + j] = -(tmp(j, i) + (g.rx * ws.dr(j, i) + g.sx * ws.ds(j, i)));
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j < nq; ++j) ws.w(j, i) = tyJ[j] * ws.dt(j, i);
  times_LT(d, e, ws.w, tmp);
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j < nq; ++j) RUY[i * nq + j] = -(tmp(j, i) + (g.ry * ws.dr(j, i) + g.sy * ws.ds(j, i)));
  times_LT(d, e, ws.dt, tmp);
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j < nq; ++j) RUZ[i * nq + j] = -g.tzJ * tmp(j, i);

  // velocity divergence with one folded lift application
  Block& rp = ws.rp;
  times_transpose(UX, nq, nt, refs.tri.dr, ws.dr);
  times_transpose(UX, nq, nt, refs.tri.ds, ws.ds);
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j < nq; ++j) rp(j, i) = g.rx * ws.dr(j, i) + g.sx * ws.ds(j, i);
  left_times(refs.line.diff, UX, nq, nt, ws.dt);
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j < nq; ++j) ws.w(j, i) = txJ[j] * ws.dt(j, i);
  times_transpose(UY, nq, nt, refs.tri.dr, ws.dr);
  times_transpose(UY, nq, nt, refs.tri.ds, ws.ds);
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j < nq; ++j) rp(j, i) += g.ry * ws.dr(j, i) + g.sy * ws.ds(j, i);
  left_times(refs.line.diff, UY, nq, nt, ws.dt);
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j < nq; ++j) ws.w(j, i) += tyJ[j] * ws.dt(j, i);
  left_times(refs.line.diff, UZ, nq, nt, ws.dt);
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j < nq; ++j) ws.w(j, i) += g.tzJ * ws.dt(j, i);
  times_LT(d, e, ws.w, tmp);
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j < nq; ++j) RP[i * nq + j] = -(rp(j, i) + tmp(j, i));
}

void tet_volume_elem(const Discretization& d, int e, const double* u, double* rhs, Scratch& ws) {
  // solver.cpp:220-254
  const auto& tet = d.refs.tet;
  const TetGeo& g = d.tgeo[e - d.mesh.num_wedges()];
  const int np = d.np_tet;
  const std::size_t base = d.elem_offset[e];
  const double* P = u + base;
  double* a = ws.va.data();
  double* b = ws.vb.data();
  double* c = ws.vc.data();
  auto mv = [&](const Mat& D, const double* x, double* y) {
    for (int n = 0; n < np; ++n) {
      double s = 0.0;
      for (int k = 0; k < np; ++k) s += D(n, k) * x[k];
      y[n] = s;
    }
  };
  mv(tet.dr, P, a);
  mv(tet.ds, P, b);
  mv(tet.dt, P, c);
  for (int n = 0; n < np; ++n) {
    rhs[base + np + n] = -(g.rx * a[n] + g.sx * b[n] + g.tx * c[n]);
    rhs[base + 2 * np + n] = -(g.ry * a[n] + g.sy * b[n] + g.ty * c[n]);
    rhs[base + 3 * np + n] = -(g.rz * a[n] + g.sz * b[n] + g.tz * c[n]);
  }
  double* rp = ws.vd.data();
  std::fill(rp, rp + np, 0.0);
  const double* comps[3] = {u + base + np, u + base + 2 * np, u + base + 3 * np};
  const double cr[3] = {g.rx, g.ry, g.rz}, cs[3] = {g.sx, g.sy, g.sz}, ct[3] = {g.tx, g.ty, g.tz};
  for (int q = 0; q < 3; ++q) {
    mv(tet.dr, comps[q], a);
    mv(tet.ds, comps[q], b);
    mv(tet.dt, comps[q], c);
    for (int n = 0; n < np; ++n) rp[n] += cr[q] * a[n] + cs[q] * b[n] + ct[q] * c[n];
  }
  for (int n = 0; n < np; ++n) rhs[base + n] = -rp[n];
}

void surface_elem(const Discretization& d, int e, const double* u, double* rhs, Scratch& ws) {
  // solver.cpp:258-335
  const auto& refs = d.refs;
  const bool wedge = d.mesh.kind(e) == ElemKind::wedge;
  const int np = d.np(e), nq = d.nq, nt = d.nt;
  const std::size_t base = d.elem_offset[e];
  const int nf = d.mesh.num_faces(e);
  for (int f = 0; f < nf; ++f) {
    const FaceConn& fc = d.conn.at(e, f);
    const FacePhys& ph = d.fphys[d.conn.face_offset[e] + f];
    const auto& my = d.my_nodes(e, f);
    const int nfp = (int)my.size();
    const double nx = ph.normal[0], ny = ph.normal[1], nz = ph.normal[2];
    if (fc.nbr >= 0) {
      const std::size_t nb = d.elem_offset[fc.nbr];
      const int npn = d.np(fc.nbr);
      for (int i = 0; i < nfp; ++i) {
        const int m = my[i];
        const int q = d.nbr_node(e, f, i);
        const double dp = u[nb + q] - u[base + m];
        const double dux = u[nb + npn + q] - u[base + np + m];
        const double duy = u[nb + 2 * npn + q] - u[base + 2 * np + m];
        const double duz = u[nb + 3 * npn + q] - u[base + 3 * np + m];
        const double dun = nx * dux + ny * duy + nz * duz;
        ws.fp[i] = 0.5 * (ph.tau_p * dp - dun);
        ws.fu[i] = 0.5 * (ph.tau_u * dun - dp);
      }
    } else {
      for (int i = 0; i < nfp; ++i) {
        const double dp = -2.0 * u[base + my[i]];
        ws.fp[i] = 0.5 * ph.tau_p * dp;
        ws.fu[i] = -0.5 * dp;
      }
    }
    std::fill(ws.lift_u.begin(), ws.lift_u.begin() + np, 0.0);
    if (wedge) {
      double* RP = rhs + base;
      double* LU = ws.lift_u.data();
      if (f < 2) {
        const bool bottom = f == 0;
        const bool exact = d.qmode == QuadratureMode::exact;
        const Vec& prof = exact ? (bottom ? refs.line.lift_bottom : refs.line.lift_top)
                                : (bottom ? refs.line.lumped_lift_bottom : refs.line.lumped_lift_top);
        const double jf = bottom ? d.wgeo[e].jf_bottom : d.wgeo[e].jf_top;
        double* tmp = ws.tv.data();
        for (int i = 0; i < nt; ++i) {
          double s = 0.0;
          for (int k = 0; k < nt; ++k) s += Lik(d, e, i, k) * ws.fp[k];
          tmp[i] = s;
        }
        for (int i = 0; i < nt; ++i)
          for (int j = 0; j < nq; ++j) RP[i * nq + j] += jf * prof[j] * tmp[i];
        for (int i = 0; i < nt; ++i) {
          double s = 0.0;
          for (int k = 0; k < nt; ++k) s += Lik(d, e, i, k) * ws.fu[k];
          tmp[i] = s;
        }
        for (int i = 0; i < nt; ++i)
          for (int j = 0; j < nq; ++j) LU[i * nq + j] += jf * prof[j] * tmp[i];
      } else {
        // F(j,a) = flux[a*nq + j];  RP(j,i) += sum_a F(j,a) QL(i,a)
        const double* Q = d.quad_lift.data() + ((std::size_t)e * 3 + (f - 2)) * nq * nt;
        for (int i = 0; i < nt; ++i)
          for (int j = 0; j < nq; ++j) {
            double sp = 0.0, su = 0.0;
            for (int a = 0; a < nq; ++a) {
              const double qa = Q[(std::size_t)a * nt + i];
              sp += ws.fp[a * nq + j] * qa;
              su += ws.fu[a * nq + j] * qa;
            }
            RP[i * nq + j] += sp;
            LU[i * nq + j] += su;
          }
      }
    } else {
      const auto& tet = refs.tet;
      const TetGeo& g = d.tgeo[e - d.mesh.num_wedges()];
      const int nfp_t = tet.num_face_nodes;
      for (int n = 0; n < np; ++n) {
        double sp = 0.0, su = 0.0;
        for (int m = 0; m < nfp_t; ++m) {
          sp += tet.lift(n, f * nfp_t + m) * ws.fp[m];
          su += tet.lift(n, f * nfp_t + m) * ws.fu[m];
        }
        rhs[base + n] += g.lift_scale[f] * sp;
        ws.lift_u[n] += g.lift_scale[f] * su;
      }
    }
    for (int n = 0; n < np; ++n) {
      rhs[base + np + n] += nx * ws.lift_u[n];
      rhs[base + 2 * np + n] += ny * ws.lift_u[n];
      rhs[base + 3 * np + n] += nz * ws.lift_u[n];
    }
  }
}

// ---- weight-adjusted (WADG) mode: an extension of the reference (SURVEY.md
// A.4).  Restated independently of the device factorisation: the exact system
// is M_k du/dt = S u + B with M_k = M^{tri,k} (x) M1D, so the WADG rhs is
//   Mtilde^{-1} M_k rhs_exact = (Mhat^{-1} M_{1/J} Mhat^{-1} M^{tri,k}) (x) I
// applied to the exact rhs, slice by slice, with M_{1/J} assembled here on the
// reference triangle cubature.  Tets are affine: WADG == exact there.
Mat inv_j_mass(const Discretization& d, int w) {
  const auto& tri = d.refs.tri;
  const WedgeGeo& g = d.wgeo[w];
  const int nt = d.nt, nc = (int)tri.cubature.weights.size();
  Mat m(nt, nt);
  for (int q = 0; q < nc; ++q) {
    const double J = g.j0 + g.jr * tri.cubature.points(q, 0) + g.js * tri.cubature.points(q, 1);
    for (int a = 0; a < nt; ++a)
      for (int b = 0; b < nt; ++b) m(a, b) += tri.cubature.weights[q] * tri.interp_cub(q, a) * tri.interp_cub(q, b) / J;
  }
  return m;
}

Mat wadg_transform_matrix(const Discretization& d, int w) {
  const Mat minv = inverse(d.refs.tri.mass);
  const WedgeGeo& g = d.wgeo[w];
  const Mat mk = wedge_tri_mass(g.j0, g.jr, g.js, d.refs);
  return matmul(matmul(minv, inv_j_mass(d, w)), matmul(minv, mk));
}

// block of one wedge (4 fields, node i*nq + j): x_j <- T x_j for every slice j
void wadg_apply(const Discretization& d, int w, double* block) {
  const int nq = d.nq, nt = d.nt, np = d.np_wedge;
  const Mat T = wadg_transform_matrix(d, w);
  std::vector<double> tmp(nt);
  for (int f = 0; f < 4; ++f)
    for (int j = 0; j < nq; ++j) {
      double* x = block + (std::size_t)f * np;
      for (int i = 0; i < nt; ++i) {
        double s = 0.0;
        for (int k = 0; k < nt; ++k) s += T(i, k) * x[k * nq + j];
        tmp[i] = s;
      }
      for (int i = 0; i < nt; ++i) x[i * nq + j] = tmp[i];
    }
}

inline bool is_wadg_wedge(const Discretization& d, int e) {
  return d.mass_mode == MassMode::wadg && d.mesh.kind(e) == ElemKind::wedge;
}

void scale_media(const Discretization& d, int e, double* rhs) {
  const int np = d.np(e);
  const std::size_t base = d.elem_offset[e];
  const double kappa = d.mesh.media[e].kappa, inv_rho = 1.0 / d.mesh.media[e].rho;
  for (int n = 0; n < np; ++n) rhs[base + n] *= kappa;
  for (int n = 0; n < 3 * np; ++n) rhs[base + np + n] *= inv_rho;
}

Scratch make_scratch(const Discretization& d) {
  const int max_np = std::max(d.np_wedge, d.np_tet);
  const int max_nfp = std::max(d.nq * d.nq, d.nt);
  return Scratch(d.nq, d.nt, max_np, max_nfp);
}

// LSERK45 (solver.cpp:511-523)
const double kA[5] = {0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                      -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0};
const double kB[5] = {1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                      1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                      2277821191437.0 / 14882151754819.0};

} // namespace

void compute_rhs(const Discretization& d, const double* u, double* rhs, int threads) {
  const int ne = d.num_elements();
#pragma omp parallel num_threads(std::max(1, threads))
  {
    Scratch ws = make_scratch(d);
#pragma omp for schedule(static)
    for (int e = 0; e < ne; ++e) {
      if (d.mesh.kind(e) == ElemKind::wedge)
        wedge_volume_elem(d, e, u, rhs, ws);
      else
        tet_volume_elem(d, e, u, rhs, ws);
      surface_elem(d, e, u, rhs, ws);
      if (is_wadg_wedge(d, e)) wadg_apply(d, e, rhs + d.elem_offset[e]);
      scale_media(d, e, rhs);
    }
  }
}

void wedge_volume_phase(const Discretization& d, const double* u, double* rhs) {
  Scratch ws = make_scratch(d);
  for (int e = 0; e < d.mesh.num_wedges(); ++e) {
    wedge_volume_elem(d, e, u, rhs, ws);
    if (is_wadg_wedge(d, e)) wadg_apply(d, e, rhs + d.elem_offset[e]);
  }
}
void wedge_surface_phase(const Discretization& d, const double* u, double* rhs) {
  Scratch ws = make_scratch(d);
  for (int e = 0; e < d.mesh.num_wedges(); ++e) {
    if (!is_wadg_wedge(d, e)) {
      surface_elem(d, e, u, rhs, ws);
      continue;
    }
    // WADG is linear: accumulate T * (surface part)
    double* blk = rhs + d.elem_offset[e];
    const std::vector<double> saved(blk, blk + 4 * d.np_wedge);
    std::fill(blk, blk + 4 * d.np_wedge, 0.0);
    surface_elem(d, e, u, rhs, ws);
    wadg_apply(d, e, blk);
    for (int n = 0; n < 4 * d.np_wedge; ++n) blk[n] += saved[n];
  }
}
void tet_volume_phase(const Discretization& d, const double* u, double* rhs) {
  Scratch ws = make_scratch(d);
  for (int e = d.mesh.num_wedges(); e < d.num_elements(); ++e) tet_volume_elem(d, e, u, rhs, ws);
}
void tet_surface_phase(const Discretization& d, const double* u, double* rhs) {
  Scratch ws = make_scratch(d);
  for (int e = d.mesh.num_wedges(); e < d.num_elements(); ++e) surface_elem(d, e, u, rhs, ws);
}

double compute_energy(const Discretization& d, const double* u, int threads) {
  // solver.cpp:402-435: per-element partials, fixed-order serial sum
  const int ne = d.num_elements();
  std::vector<double> partial(ne, 0.0);
#pragma omp parallel for schedule(static) num_threads(std::max(1, threads))
  for (int e = 0; e < ne; ++e) {
    const int np = d.np(e);
    const std::size_t base = d.elem_offset[e];
    const double ikap = 1.0 / d.mesh.media[e].kappa, rho = d.mesh.media[e].rho;
    double acc = 0.0;
    for (int field = 0; field < 4; ++field) {
      Vec v(u + base + field * np, u + base + (field + 1) * np), mu;
      if (is_wadg_wedge(d, e)) {
        // Mtilde = (Mhat M_{1/J}^{-1} Mhat) (x) M1D
        const Mat mt = matmul(matmul(d.refs.tri.mass, inverse(inv_j_mass(d, e))), d.refs.tri.mass);
        const int nq = d.nq, nt = d.nt;
        mu.assign(np, 0.0);
        for (int i = 0; i < nt; ++i)
          for (int j = 0; j < nq; ++j) {
            double s = 0.0;
            for (int k = 0; k < nt; ++k)
              for (int l = 0; l < nq; ++l) s += mt(i, k) * d.refs.line.mass(j, l) * v[k * nq + l];
            mu[i * nq + j] = s;
          }
      } else if (d.mesh.kind(e) == ElemKind::wedge) {
        const ElementGeometry g = d.geometry(e);
        apply_wedge_mass(g, d.refs, d.qmode, v, mu);
      } else {
        mu = matvec(d.refs.tet.mass, v);
        for (double& x : mu) x *= d.tgeo[e - d.mesh.num_wedges()].J;
      }
      double q = 0.0;
      for (int n = 0; n < np; ++n) q += v[n] * mu[n];
      acc += field == 0 ? ikap * q : rho * q;
    }
    partial[e] = 0.5 * acc;
  }
  double total = 0.0;
  for (double p : partial) total += p;
  return total;
}

void lserk_steps(const Discretization& d, double* u, std::size_t n, double dt, int nsteps, int threads,
                 bool parallel_update) {
  // TimeStepper::step, LSERK branch (solver.cpp:536-557)
  std::vector<double> res(n), rhs(n);
  for (int step = 0; step < nsteps; ++step) {
    std::fill(res.begin(), res.end(), 0.0);
    for (int s = 0; s < 5; ++s) {
      compute_rhs(d, u, rhs.data(), threads);
      const double a = kA[s], b = kB[s];
      if (parallel_update) {
#pragma omp parallel for schedule(static) num_threads(std::max(1, threads))
        for (long long i = 0; i < (long long)n; ++i) {
          res[i] = a * res[i] + dt * rhs[i];
          u[i] += b * res[i];
        }
      } else {
        for (std::size_t i = 0; i < n; ++i) {
          res[i] = a * res[i] + dt * rhs[i];
          u[i] += b * res[i];
        }
      }
    }
  }
}

void ab3_steps(const Discretization& d, double* u, std::size_t n, double dt, int nsteps, int threads) {
  // solver.cpp:559-581; h[2] = f_{n-2}, h[1] = f_{n-1}
  std::vector<std::vector<double>> h(3, std::vector<double>(n, 0.0));
  std::vector<double> f(n);
  int filled = 0;
  for (int step = 0; step < nsteps; ++step) {
    if (filled < 2) {
      compute_rhs(d, u, h[2 - filled].data(), threads);
      lserk_steps(d, u, n, dt, 1, threads, false);
      ++filled;
      continue;
    }
    compute_rhs(d, u, f.data(), threads);
    for (std::size_t i = 0; i < n; ++i) u[i] += dt / 12.0 * (23.0 * f[i] - 16.0 * h[1][i] + 5.0 * h[2][i]);
    std::swap(h[2], h[1]);
    std::swap(h[1], f);
  }
}

void mrab_steps(const Discretization& d, double* u, std::size_t n, const int* level, int nlev, double dt, int nmacro,
                int threads) {
  // Multi-rate AB3 restated element by element (the device's pdg_step_mrab;
  // PAPER.md:614).  Level g steps with h_g = 2^g dt, M = 2^(nlev-1) fine
  // substeps per macro step; the first two macro steps are LSERK45 at dt with
  // f_g recorded at t - h_g and t - 2 h_g (ab3_steps' bootstrap per level).
  const int M = 1 << (nlev - 1), ne = d.num_elements();
  std::vector<std::vector<double>> f(3, std::vector<double>(n, 0.0));
  std::vector<double> u0(n), r(n);
  std::vector<std::array<int, 3>> slot(nlev, std::array<int, 3>{0, 1, 2});
  auto for_level = [&](int g, auto&& fn) {
    for (int e = 0; e < ne; ++e)
      if (level[e] == g)
        for (std::size_t i = d.elem_offset[e]; i < d.elem_offset[e + 1]; ++i) fn(i);
  };
  for (int m = 0; m < nmacro; ++m) {
    if (m < 2) {
      for (int k = 0; k < M; ++k) {
        const int nb = m * M + k;
        bool need = false;
        for (int g = 0; g < nlev; ++g) need = need || nb == 2 * M - (1 << g) || nb == 2 * M - (2 << g);
        if (need) {
          compute_rhs(d, u, r.data(), threads);
          for (int g = 0; g < nlev; ++g) {
            if (nb == 2 * M - (1 << g)) for_level(g, [&](std::size_t i) { f[slot[g][1]][i] = r[i]; });
            if (nb == 2 * M - (2 << g)) for_level(g, [&](std::size_t i) { f[slot[g][2]][i] = r[i]; });
          }
        }
        lserk_steps(d, u, n, dt, 1, threads, false);
      }
      if (m == 1) std::copy(u, u + n, u0.begin());
      continue;
    }
    for (int k = 0; k < M; ++k) {
      bool any = false;
      for (int g = 0; g < nlev; ++g) any = any || k % (1 << g) == 0;
      if (any) compute_rhs(d, u, r.data(), threads);  // per element: identical to a per-level rhs
      for (int g = 0; g < nlev; ++g)
        if (k % (1 << g) == 0) for_level(g, [&](std::size_t i) { f[slot[g][0]][i] = r[i]; });
      for (int g = 0; g < nlev; ++g) {
        const int kk = k % (1 << g);
        const double h = std::ldexp(dt, g), th = (double)(kk + 1) / (1 << g);
        const double* f0 = f[slot[g][0]].data();
        const double* f1 = f[slot[g][1]].data();
        const double* f2 = f[slot[g][2]].data();
        if (kk + 1 == (1 << g)) {
          for_level(g, [&](std::size_t i) {
            const double v = u0[i] + (h / 12.0) * (23.0 * f0[i] - 16.0 * f1[i] + 5.0 * f2[i]);
            u[i] = v;
            u0[i] = v;
          });
          slot[g] = {slot[g][2], slot[g][0], slot[g][1]};
        } else {
          // integral over [0, th] of the backward-difference quadratic through f0, f1, f2
          const double c0 = th + 0.75 * th * th + th * th * th / 6.0, c1 = -th * th - th * th * th / 3.0,
                       c2 = 0.25 * th * th + th * th * th / 6.0;
          for_level(g, [&](std::size_t i) { u[i] = u0[i] + h * (c0 * f0[i] + c1 * f1[i] + c2 * f2[i]); });
        }
      }
    }
  }
}

RunOut run_simulation(const Discretization& d, std::vector<double>& u, double& time, double final_time, double cfl,
                      double fixed_dt, double energy_interval, int threads) {
  // solver.cpp:591-666 (LSERK, watchdog every 50 steps, blow-up factor 10)
  RunOut out;
  const double span = final_time - time;
  const double dt0 = fixed_dt > 0.0 ? fixed_dt : estimate_dt(d, cfl);
  const int steps = std::max(1, (int)std::ceil(span / dt0 - 1e-12));
  const double dt = span / steps;
  out.steps = steps;
  out.dt = dt;
  out.initial_energy = compute_energy(d, u.data(), threads);
  double last = out.initial_energy;
  double next_energy_t = time + energy_interval;
  auto log_energy = [&]() {
    const double en = compute_energy(d, u.data(), threads);
    out.max_energy_increase = std::max(out.max_energy_increase, en - last);
    last = en;
  };
  for (int n = 0; n < steps; ++n) {
    lserk_steps(d, u.data(), u.size(), dt, 1, threads, true);
    time += dt;
    if (energy_interval <= 0.0) {
      log_energy();
    } else if (time + 1e-12 >= next_energy_t) {
      log_energy();
      while (next_energy_t <= time + 1e-12) next_energy_t += energy_interval;
    }
    if ((n + 1) % 50 == 0 || n + 1 == steps) {
      for (double v : u)
        if (!std::isfinite(v)) {
          out.stable = false;
          return out;
        }
      if (compute_energy(d, u.data(), threads) > 10.0 * out.initial_energy + 1e-300) {
        out.stable = false;
        return out;
      }
    }
  }
  out.final_time = time;
  out.final_energy = compute_energy(d, u.data(), threads);
  return out;
}

} // namespace oracle
