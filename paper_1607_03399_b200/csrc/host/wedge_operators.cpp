// Reduced-storage wedge operators and their Kronecker-factored actions.
// Follows proj/src/operators.cpp:5-183.
#include "prismdg/operators.hpp"

#include <algorithm>
#include <cmath>

namespace prismdg {

Mat wedge_tri_mass(double j0, double jr, double js, const References& refs) {
  const Mat& M = refs.tri.mass;
  Mat out(M.rows, M.cols);
  for (std::size_t q = 0; q < out.a.size(); ++q)
    out.a[q] = j0 * M.a[q] + jr * refs.tri.moment_r.a[q] + js * refs.tri.moment_s.a[q];
  return out;
}

Mat wedge_edge_mass_embedded(int e, double jf0, double jf1, const References& refs) {
  // operators.cpp:35-47: Gauss (N+2) rule, J_f affine along the edge
  const auto& line = refs.line;
  const int nq = refs.degree + 1, nt = refs.tri.num_nodes;
  const int ng = (int)line.gq_nodes.size();
  Mat emass(nq, nq);
  for (int q = 0; q < ng; ++q) {
    const double xi = line.gq_nodes[q];
    const double wq = line.gq_weights[q] * (jf0 * (1.0 - xi) / 2.0 + jf1 * (1.0 + xi) / 2.0);
    for (int a = 0; a < nq; ++a)
      for (int b = 0; b < nq; ++b) emass(a, b) += line.interp_gq(q, a) * wq * line.interp_gq(q, b);
  }
  Mat emb(nt, nq);
  for (int a = 0; a < nq; ++a)
    for (int b = 0; b < nq; ++b) emb(refs.tri.edge_nodes[e][a], b) = emass(a, b);
  return emb;
}

bool wedge_lifts_flat(double j0, double jr, double js, const double jf_end[3][2],
                      const References& refs, double* out_L, double* out_Q) {
  const int nt = refs.tri.num_nodes, nq = refs.degree + 1;
  const Mat Mk = wedge_tri_mass(j0, jr, js, refs);
  // right-hand sides: [Mhat | E_0 | E_1 | E_2]
  Mat rhs(nt, nt + 3 * nq);
  for (int i = 0; i < nt; ++i)
    for (int k = 0; k < nt; ++k) rhs(i, k) = refs.tri.mass(i, k);
  for (int e = 0; e < 3; ++e) {
    const Mat E = wedge_edge_mass_embedded(e, jf_end[e][0], jf_end[e][1], refs);
    for (int i = 0; i < nt; ++i)
      for (int a = 0; a < nq; ++a) rhs(i, nt + e * nq + a) = E(i, a);
  }
  Mat X;
  if (!cholesky_solve(Mk, rhs, X)) return false;
  for (int k = 0; k < nt; ++k)
    for (int i = 0; i < nt; ++i) out_L[(std::size_t)k * nt + i] = X(i, k);
  if (out_Q)
    for (int e = 0; e < 3; ++e)
      for (int a = 0; a < nq; ++a)
        for (int i = 0; i < nt; ++i) out_Q[((std::size_t)e * nq + a) * nt + i] = X(i, nt + e * nq + a);
  return true;
}

WedgeOperators build_wedge_operators(const ElementGeometry& g, const References& refs) {
  // operators.cpp:10-51
  const int nt = refs.tri.num_nodes, nq = refs.degree + 1;
  WedgeOperators ops;
  ops.txJ = g.txJ;
  ops.tyJ = g.tyJ;
  ops.tzJ = g.tzJ;
  ops.rx = g.rx;
  ops.ry = g.ry;
  ops.sx = g.sx;
  ops.sy = g.sy;
  ops.jf_bottom = g.faces[0].jf;
  ops.jf_top = g.faces[1].jf;
  double ends[3][2];
  for (int e = 0; e < 3; ++e) {
    ends[e][0] = g.faces[2 + e].jf_edge[0];
    ends[e][1] = g.faces[2 + e].jf_edge[nq - 1];
  }
  std::vector<double> L((std::size_t)nt * nt), Q((std::size_t)3 * nq * nt);
  if (!wedge_lifts_flat(g.j0, g.j_r, g.j_s, ends, refs, L.data(), Q.data()))
    throw NumericalError("weighted triangle mass matrix is not SPD");
  ops.tri_lift = Mat(nt, nt);
  for (int k = 0; k < nt; ++k)
    for (int i = 0; i < nt; ++i) ops.tri_lift(i, k) = L[(std::size_t)k * nt + i];
  for (int e = 0; e < 3; ++e) {
    ops.quad_lift[e] = Mat(nt, nq);
    for (int a = 0; a < nq; ++a)
      for (int i = 0; i < nt; ++i) ops.quad_lift[e](i, a) = Q[((std::size_t)e * nq + a) * nt + i];
  }
  return ops;
}

TetOperators build_tet_operators(const ElementGeometry& g) {
  TetOperators ops;
  ops.rx = g.rx;
  ops.ry = g.ry;
  ops.rz = g.rz;
  ops.sx = g.sx;
  ops.sy = g.sy;
  ops.sz = g.sz;
  ops.tx = g.tx;
  ops.ty = g.ty;
  ops.tz = g.tz;
  for (int f = 0; f < 4; ++f) ops.lift_scale[f] = g.faces[f].jf / g.j0;
  return ops;
}

LumpedWedgeOperators build_lumped_wedge_operators(const ElementGeometry& g, const References& refs) {
  LumpedWedgeOperators lw;
  lw.tri_mass = wedge_tri_mass(g, refs);
  lw.t_weights = refs.line.weights;
  lw.base = build_wedge_operators(g, refs);
  return lw;
}

// ---------------------------------------------------------------------------
// Kronecker actions on a t-fast nodal vector: value of (tri node i, slice j)
// at u[i*nq + j]  (operators.cpp:88-163)
// ---------------------------------------------------------------------------

void apply_wedge_derivatives(const WedgeOperators& ops, const References& refs, const Vec& u,
                             Vec& dx, Vec& dy, Vec& dz) {
  const int nq = refs.degree + 1, nt = refs.tri.num_nodes;
  dx.assign(u.size(), 0.0);
  dy.assign(u.size(), 0.0);
  dz.assign(u.size(), 0.0);
  std::vector<double> dr((std::size_t)nq * nt), ds(dr.size()), dt(dr.size());
  for (int j = 0; j < nq; ++j)
    for (int i = 0; i < nt; ++i) {
      double a = 0, b = 0, c = 0;
      for (int k = 0; k < nt; ++k) {
        a += refs.tri.dr(i, k) * u[k * nq + j];
        b += refs.tri.ds(i, k) * u[k * nq + j];
      }
      for (int l = 0; l < nq; ++l) c += refs.line.diff(j, l) * u[i * nq + l];
      dr[i * nq + j] = a;
      ds[i * nq + j] = b;
      dt[i * nq + j] = c;
    }
  for (int j = 0; j < nq; ++j)
    for (int i = 0; i < nt; ++i) {
      double ldt = 0.0;
      for (int k = 0; k < nt; ++k) ldt += ops.tri_lift(i, k) * dt[k * nq + j];
      const int n = i * nq + j;
      dx[n] = ops.rx * dr[n] + ops.sx * ds[n] + ops.txJ[j] * ldt;
      dy[n] = ops.ry * dr[n] + ops.sy * ds[n] + ops.tyJ[j] * ldt;
      dz[n] = ops.tzJ * ldt;
    }
}

void apply_wedge_lift(const WedgeOperators& ops, const References& refs, QuadratureMode mode,
                      int face, const Vec& flux, Vec& out) {
  const int nq = refs.degree + 1, nt = refs.tri.num_nodes;
  if (face < 2) {
    const bool bottom = face == 0;
    const Vec& prof = mode == QuadratureMode::exact
                          ? (bottom ? refs.line.lift_bottom : refs.line.lift_top)
                          : (bottom ? refs.line.lumped_lift_bottom : refs.line.lumped_lift_top);
    const double jf = bottom ? ops.jf_bottom : ops.jf_top;
    const Vec tmp = matvec(ops.tri_lift, flux);
    for (int i = 0; i < nt; ++i)
      for (int j = 0; j < nq; ++j) out[i * nq + j] += jf * prof[j] * tmp[i];
  } else {
    const Mat& Q = ops.quad_lift[face - 2];
    for (int i = 0; i < nt; ++i)
      for (int j = 0; j < nq; ++j) {
        double s = 0.0;
        for (int a = 0; a < nq; ++a) s += flux[a * nq + j] * Q(i, a);
        out[i * nq + j] += s;
      }
  }
}

void apply_wedge_mass(const ElementGeometry& g, const References& refs, QuadratureMode mode,
                      const Vec& u, Vec& out) {
  const int nq = refs.degree + 1, nt = refs.tri.num_nodes;
  const Mat M = wedge_tri_mass(g, refs);
  std::vector<double> um((std::size_t)nq * nt, 0.0); // (U M)(l,i)
  for (int l = 0; l < nq; ++l)
    for (int i = 0; i < nt; ++i) {
      double s = 0.0;
      for (int k = 0; k < nt; ++k) s += u[k * nq + l] * M(k, i);
      um[i * nq + l] = s;
    }
  out.assign(u.size(), 0.0);
  for (int j = 0; j < nq; ++j)
    for (int i = 0; i < nt; ++i) {
      double s = 0.0;
      if (mode == QuadratureMode::exact) {
        for (int l = 0; l < nq; ++l) s += refs.line.mass(j, l) * um[i * nq + l];
      } else {
        s = refs.line.weights[j] * um[i * nq + j];
      }
      out[i * nq + j] = s;
    }
}

void apply_tet_derivatives(const TetOperators& ops, const References& refs, const Vec& u, Vec& dx,
                           Vec& dy, Vec& dz) {
  const Vec a = matvec(refs.tet.dr, u), b = matvec(refs.tet.ds, u), c = matvec(refs.tet.dt, u);
  dx.resize(u.size());
  dy.resize(u.size());
  dz.resize(u.size());
  for (std::size_t n = 0; n < u.size(); ++n) {
    dx[n] = ops.rx * a[n] + ops.sx * b[n] + ops.tx * c[n];
    dy[n] = ops.ry * a[n] + ops.sy * b[n] + ops.ty * c[n];
    dz[n] = ops.rz * a[n] + ops.sz * b[n] + ops.tz * c[n];
  }
}

void apply_tet_lift(const TetOperators& ops, const References& refs, int face, const Vec& flux,
                    Vec& out) {
  const int nfp = refs.tet.num_face_nodes;
  for (int n = 0; n < refs.tet.num_nodes; ++n) {
    double s = 0.0;
    for (int m = 0; m < nfp; ++m) s += refs.tet.lift(n, face * nfp + m) * flux[m];
    out[n] += ops.lift_scale[face] * s;
  }
}

void apply_tet_mass(const ElementGeometry& g, const References& refs, const Vec& u, Vec& out) {
  out = matvec(refs.tet.mass, u);
  for (double& v : out) v *= g.j0;
}

Mat wedge_inv_j_mass(double j0, double jr, double js, const References& refs) {
  const auto& tri = refs.tri;
  const int nt = tri.num_nodes, nc = (int)tri.cubature.weights.size();
  Mat out(nt, nt);
  for (int q = 0; q < nc; ++q) {
    const double J = j0 + jr * tri.cubature.points(q, 0) + js * tri.cubature.points(q, 1);
    const double wq = tri.cubature.weights[q] / J;
    for (int a = 0; a < nt; ++a)
      for (int b = 0; b < nt; ++b) out(a, b) += tri.interp_cub(q, a) * wq * tri.interp_cub(q, b);
  }
  return out;
}

WadgTables build_wadg_tables(const References& refs) {
  const auto& tri = refs.tri;
  WadgTables w;
  w.nt = tri.num_nodes;
  w.nq = refs.degree + 1;
  w.nc = (int)tri.cubature.weights.size();
  w.inv_mass = inverse(tri.mass);
  w.Kr = matmul(w.inv_mass, tri.moment_r);
  w.Ks = matmul(w.inv_mass, tri.moment_s);
  w.kd[0] = tri.dr;
  w.kd[1] = matmul(w.Kr, tri.dr);
  w.kd[2] = matmul(w.Ks, tri.dr);
  w.kd[3] = tri.ds;
  w.kd[4] = matmul(w.Kr, tri.ds);
  w.kd[5] = matmul(w.Ks, tri.ds);
  Mat vw = transpose(tri.interp_cub); // nt x nc
  for (int a = 0; a < w.nt; ++a)
    for (int q = 0; q < w.nc; ++q) vw(a, q) *= tri.cubature.weights[q];
  w.Pw = matmul(w.inv_mass, vw);
  w.Vq = tri.interp_cub;
  w.qr.resize(w.nc);
  w.qs.resize(w.nc);
  for (int q = 0; q < w.nc; ++q) {
    w.qr[q] = tri.cubature.points(q, 0);
    w.qs[q] = tri.cubature.points(q, 1);
  }
  for (int e = 0; e < 3; ++e) {
    w.R0[e] = matmul(w.inv_mass, wedge_edge_mass_embedded(e, 1.0, 0.0, refs));
    w.R1[e] = matmul(w.inv_mass, wedge_edge_mass_embedded(e, 0.0, 1.0, refs));
  }
  return w;
}

StorageReport storage_report(int degree, const std::vector<WedgeOperators>& wedges,
                             const std::vector<TetOperators>& tets) {
  StorageReport rep;
  rep.degree = degree;
  rep.num_wedges = wedges.size();
  rep.num_tets = tets.size();
  const std::size_t nt = (std::size_t)(degree + 1) * (degree + 2) / 2;
  rep.budget_per_wedge = nt * nt + 3u * nt * (degree + 1) + 8u * (degree + 1);
  for (const auto& w : wedges) {
    rep.wedge_floats_per_elem = std::max(rep.wedge_floats_per_elem, w.storage_floats());
    rep.total_floats += w.storage_floats();
  }
  for (const auto& t : tets) {
    rep.tet_floats_per_elem = std::max(rep.tet_floats_per_elem, t.storage_floats());
    rep.total_floats += t.storage_floats();
  }
  return rep;
}

} // namespace prismdg
