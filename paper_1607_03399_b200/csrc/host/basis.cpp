// Polynomial bases, quadrature rules and nodal reference elements (host setup).
//
// Follows the reference's construction so node positions, orderings and
// operators agree to rounding:
//   Jacobi / Gauss / GLL ............ proj/src/jacobi.cpp:7-110
//   warp & blend (shared alpha) ..... proj/src/reference.cpp:13-73,196-228,396-482
//   modal bases ..................... proj/src/reference.cpp:75-150
//   cubatures ....................... proj/src/reference.cpp:259-279,518-540
//   element assembly ................ proj/src/reference.cpp:164-188,304-388,558-636
#include "prismdg/basis.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <string>

namespace prismdg {

// ===========================================================================
// 1D: orthonormal Jacobi polynomials and Gauss rules
// ===========================================================================

namespace {

// integral of the Jacobi weight (1-x)^a (1+x)^b over [-1,1]
double jacobi_weight_mass(double a, double b) {
  return std::pow(2.0, a + b + 1.0) / (a + b + 1.0) * std::tgamma(a + 1.0) *
         std::tgamma(b + 1.0) / std::tgamma(a + b + 1.0);
}

} // namespace

double jacobi_p(int n, double a, double b, double x) {
  // orthonormal three-term recurrence (jacobi.cpp:7-33)
  const double m0 = jacobi_weight_mass(a, b);
  double p_prev = 1.0 / std::sqrt(m0);
  if (n == 0) return p_prev;
  const double m1 = (a + 1.0) * (b + 1.0) / (a + b + 3.0) * m0;
  double p_cur = (0.5 * (a + b + 2.0) * x + 0.5 * (a - b)) / std::sqrt(m1);
  double c_prev = 2.0 / (2.0 + a + b) * std::sqrt((a + 1.0) * (b + 1.0) / (a + b + 3.0));
  for (int k = 1; k < n; ++k) {
    const double h = 2.0 * k + a + b;
    const double c_next = 2.0 / (h + 2.0) *
                          std::sqrt((k + 1.0) * (k + 1.0 + a + b) * (k + 1.0 + a) *
                                    (k + 1.0 + b) / (h + 1.0) / (h + 3.0));
    const double shift = -(a * a - b * b) / (h * (h + 2.0));
    const double p_next = ((x - shift) * p_cur - c_prev * p_prev) / c_next;
    p_prev = p_cur;
    p_cur = p_next;
    c_prev = c_next;
  }
  return p_cur;
}

double grad_jacobi_p(int n, double a, double b, double x) {
  return n == 0 ? 0.0 : std::sqrt(n * (n + a + b + 1.0)) * jacobi_p(n - 1, a + 1.0, b + 1.0, x);
}

void jacobi_gauss(int npts, double a, double b, Vec& x, Vec& w) {
  // Golub-Welsch (jacobi.cpp:40-77)
  if (npts < 1) throw ConfigError("jacobi_gauss: need at least one point");
  const double mu0 = jacobi_weight_mass(a, b);
  if (npts == 1) {
    x.assign(1, (b - a) / (a + b + 2.0));
    w.assign(1, mu0);
    return;
  }
  Vec diag(npts), off(npts - 1);
  for (int k = 0; k < npts; ++k) {
    const double h = 2.0 * k + a + b;
    diag[k] = -(a * a - b * b) / ((h + 2.0) * h);
  }
  if (a + b < 10.0 * std::numeric_limits<double>::epsilon()) diag[0] = 0.0;
  for (int k = 1; k < npts; ++k) {
    const double h = 2.0 * (k - 1) + a + b;
    off[k - 1] = 2.0 / (h + 2.0) *
                 std::sqrt(k * (k + a + b) * (k + a) * (k + b) / ((h + 1.0) * (h + 3.0)));
  }
  Vec v0;
  sym_tridiag_eig(diag, off, x, v0);
  w.resize(npts);
  for (int k = 0; k < npts; ++k) w[k] = mu0 * v0[k] * v0[k];
}

void gauss_lobatto(int npts, Vec& x, Vec& w) {
  // interior nodes are the Gauss-Jacobi(1,1) points (jacobi.cpp:79-96)
  if (npts < 2) throw ConfigError("gauss_lobatto: need at least two points");
  const int N = npts - 1;
  x.assign(npts, 0.0);
  x.front() = -1.0;
  x.back() = 1.0;
  if (N >= 2) {
    Vec xi, wi;
    jacobi_gauss(N - 1, 1.0, 1.0, xi, wi);
    std::copy(xi.begin(), xi.end(), x.begin() + 1);
  }
  w.resize(npts);
  for (int j = 0; j <= N; ++j) {
    const double pn = jacobi_p(N, 0.0, 0.0, x[j]);
    w[j] = (2.0 * N + 1.0) / (N * (N + 1.0) * pn * pn);
  }
}

Mat legendre_vandermonde(int degree, const Vec& x) {
  Mat V((int)x.size(), degree + 1);
  for (int i = 0; i < V.rows; ++i)
    for (int j = 0; j <= degree; ++j) V(i, j) = jacobi_p(j, 0.0, 0.0, x[i]);
  return V;
}

Mat legendre_grad_vandermonde(int degree, const Vec& x) {
  Mat V((int)x.size(), degree + 1);
  for (int i = 0; i < V.rows; ++i)
    for (int j = 0; j <= degree; ++j) V(i, j) = grad_jacobi_p(j, 0.0, 0.0, x[i]);
  return V;
}

// ===========================================================================
// warp & blend node construction (one alpha table for triangle and tet)
// ===========================================================================

namespace {

// reference.cpp:16-20: shared optimised blend parameters, indexed by N-1
const double kBlendAlpha[15] = {0.0,    0.0,    0.0,    0.1002, 1.1332, 1.5608, 1.3413, 1.2577,
                                1.1603, 1.10153, 0.6080, 0.4523, 0.8856, 0.8717, 0.9655};

double blend_alpha(int N) { return N <= 15 ? kBlendAlpha[N - 1] : 1.0; }

void require_degree(int N) {
  if (N < 1 || N > kMaxDegree)
    throw ConfigError("polynomial degree must be in [1," + std::to_string(kMaxDegree) +
                      "], got " + std::to_string(N));
}

// 1D warp function evaluated at the points `r` (reference.cpp:29-44): the
// Lagrange interpolant through the equispaced points (descending) of the
// displacement to GLL, with both end roots divided out.
Vec warp_1d(int p, const Vec& gll_desc, const Vec& r) {
  Vec eq(p + 1);
  for (int i = 0; i <= p; ++i) eq[i] = -1.0 + 2.0 * (p - i) / double(p);
  Vec out(r.size(), 0.0);
  for (std::size_t n = 0; n < r.size(); ++n) {
    double acc = 0.0;
    for (int i = 0; i <= p; ++i) {
      double term = gll_desc[i] - eq[i];
      for (int j = 1; j < p; ++j)
        if (j != i) term = term * (r[n] - eq[j]) / (eq[i] - eq[j]);
      if (i != 0) term = -term / (eq[i] - eq[0]);
      if (i != p) term = term / (eq[i] - eq[p]);
      acc += term;
    }
    out[n] = acc;
  }
  return out;
}

// 2D warp-and-blend displacement in the equilateral frame (reference.cpp:48-73)
void shift_2d(int p, double alpha, const Vec& L1, const Vec& L2, const Vec& L3, Vec& dx,
              Vec& dy) {
  Vec gll, wgll;
  gauss_lobatto(p + 1, gll, wgll);
  Vec gll_desc(gll.size());
  for (std::size_t i = 0; i < gll.size(); ++i) gll_desc[i] = -gll[i];
  const std::size_t n = L1.size();
  Vec a1(n), a2(n), a3(n);
  for (std::size_t i = 0; i < n; ++i) {
    a1[i] = L3[i] - L2[i];
    a2[i] = L1[i] - L3[i];
    a3[i] = L2[i] - L1[i];
  }
  const Vec w1 = warp_1d(p, gll_desc, a1), w2 = warp_1d(p, gll_desc, a2),
            w3 = warp_1d(p, gll_desc, a3);
  const double c23 = std::cos(2.0 * M_PI / 3.0), s23 = std::sin(2.0 * M_PI / 3.0);
  const double c43 = std::cos(4.0 * M_PI / 3.0), s43 = std::sin(4.0 * M_PI / 3.0);
  dx.assign(n, 0.0);
  dy.assign(n, 0.0);
  for (std::size_t i = 0; i < n; ++i) {
    const double b1 = L2[i] * L3[i] * (4.0 * w1[i]) * (1.0 + (alpha * L1[i]) * (alpha * L1[i]));
    const double b2 = L1[i] * L3[i] * (4.0 * w2[i]) * (1.0 + (alpha * L2[i]) * (alpha * L2[i]));
    const double b3 = L1[i] * L2[i] * (4.0 * w3[i]) * (1.0 + (alpha * L3[i]) * (alpha * L3[i]));
    dx[i] = b1 + c23 * b2 + c43 * b3;
    dy[i] = s23 * b2 + s43 * b3;
  }
}

// ---- modal simplex bases --------------------------------------------------

void rs_to_ab(double r, double s, double& a, double& b) {
  a = (std::abs(s - 1.0) > 1e-12) ? 2.0 * (1.0 + r) / (1.0 - s) - 1.0 : -1.0;
  b = s;
}

double tri_mode(double a, double b, int i, int j) {
  return std::sqrt(2.0) * jacobi_p(i, 0.0, 0.0, a) * jacobi_p(j, 2.0 * i + 1.0, 0.0, b) *
         std::pow(1.0 - b, i);
}

void tri_mode_grad(double a, double b, int i, int j, double& dr, double& ds) {
  // reference.cpp:86-104
  const double fa = jacobi_p(i, 0.0, 0.0, a), dfa = grad_jacobi_p(i, 0.0, 0.0, a);
  const double gb = jacobi_p(j, 2.0 * i + 1.0, 0.0, b);
  const double dgb = grad_jacobi_p(j, 2.0 * i + 1.0, 0.0, b);
  const double hb = 0.5 * (1.0 - b);
  const double hb_im1 = (i > 0) ? std::pow(hb, i - 1) : 1.0;
  dr = dfa * gb * hb_im1;
  ds = dfa * gb * 0.5 * (1.0 + a) * hb_im1;
  double tmp = dgb * std::pow(hb, i);
  if (i > 0) tmp -= 0.5 * i * gb * hb_im1;
  ds += fa * tmp;
  const double scale = std::pow(2.0, i + 0.5);
  dr *= scale;
  ds *= scale;
}

void rst_to_abc(double r, double s, double t, double& a, double& b, double& c) {
  a = (std::abs(s + t) > 1e-12) ? 2.0 * (1.0 + r) / (-s - t) - 1.0 : -1.0;
  b = (std::abs(t - 1.0) > 1e-12) ? 2.0 * (1.0 + s) / (1.0 - t) - 1.0 : -1.0;
  c = t;
}

double tet_mode(double a, double b, double c, int i, int j, int k) {
  return 2.0 * std::sqrt(2.0) * jacobi_p(i, 0.0, 0.0, a) * jacobi_p(j, 2.0 * i + 1.0, 0.0, b) *
         std::pow(1.0 - b, i) * jacobi_p(k, 2.0 * (i + j) + 2.0, 0.0, c) *
         std::pow(1.0 - c, i + j);
}

void tet_mode_grad(double a, double b, double c, int i, int j, int k, double& dr, double& ds,
                   double& dt) {
  // reference.cpp:119-150
  const double fa = jacobi_p(i, 0.0, 0.0, a), dfa = grad_jacobi_p(i, 0.0, 0.0, a);
  const double gb = jacobi_p(j, 2.0 * i + 1.0, 0.0, b);
  const double dgb = grad_jacobi_p(j, 2.0 * i + 1.0, 0.0, b);
  const double hc = jacobi_p(k, 2.0 * (i + j) + 2.0, 0.0, c);
  const double dhc = grad_jacobi_p(k, 2.0 * (i + j) + 2.0, 0.0, c);
  const double hb = 0.5 * (1.0 - b), hcc = 0.5 * (1.0 - c);
  dr = dfa * gb * hc;
  if (i > 0) dr *= std::pow(hb, i - 1);
  if (i + j > 0) dr *= std::pow(hcc, i + j - 1);
  ds = 0.5 * (1.0 + a) * dr;
  double tmp = dgb * std::pow(hb, i);
  if (i > 0) tmp -= 0.5 * i * gb * std::pow(hb, i - 1);
  tmp *= hc;
  if (i + j > 0) tmp *= std::pow(hcc, i + j - 1);
  tmp *= fa;
  ds += tmp;
  dt = 0.5 * (1.0 + a) * dr + 0.5 * (1.0 + b) * tmp;
  double tmp2 = dhc * std::pow(hcc, i + j);
  if (i + j > 0) tmp2 -= 0.5 * (i + j) * hc * std::pow(hcc, i + j - 1);
  dt += fa * gb * tmp2 * std::pow(hb, i);
  const double scale = std::pow(2.0, 2 * i + j + 1.5);
  dr *= scale;
  ds *= scale;
  dt *= scale;
}

Mat tri_vandermonde(int N, const Vec& r, const Vec& s) {
  const int np = (N + 1) * (N + 2) / 2;
  Mat V((int)r.size(), np);
  for (int n = 0; n < V.rows; ++n) {
    double a, b;
    rs_to_ab(r[n], s[n], a, b);
    int col = 0;
    for (int i = 0; i <= N; ++i)
      for (int j = 0; j <= N - i; ++j) V(n, col++) = tri_mode(a, b, i, j);
  }
  return V;
}

void tri_grad_vandermonde(int N, const Vec& r, const Vec& s, Mat& Vr, Mat& Vs) {
  const int np = (N + 1) * (N + 2) / 2;
  Vr = Mat((int)r.size(), np);
  Vs = Mat((int)r.size(), np);
  for (int n = 0; n < Vr.rows; ++n) {
    double a, b;
    rs_to_ab(r[n], s[n], a, b);
    int col = 0;
    for (int i = 0; i <= N; ++i)
      for (int j = 0; j <= N - i; ++j, ++col) tri_mode_grad(a, b, i, j, Vr(n, col), Vs(n, col));
  }
}

Mat tet_vandermonde(int N, const Vec& r, const Vec& s, const Vec& t) {
  const int np = (N + 1) * (N + 2) * (N + 3) / 6;
  Mat V((int)r.size(), np);
  for (int n = 0; n < V.rows; ++n) {
    double a, b, c;
    rst_to_abc(r[n], s[n], t[n], a, b, c);
    int col = 0;
    for (int i = 0; i <= N; ++i)
      for (int j = 0; j <= N - i; ++j)
        for (int k = 0; k <= N - i - j; ++k) V(n, col++) = tet_mode(a, b, c, i, j, k);
  }
  return V;
}

void tet_grad_vandermonde(int N, const Vec& r, const Vec& s, const Vec& t, Mat& Vr, Mat& Vs,
                          Mat& Vt) {
  const int np = (N + 1) * (N + 2) * (N + 3) / 6;
  Vr = Mat((int)r.size(), np);
  Vs = Mat((int)r.size(), np);
  Vt = Mat((int)r.size(), np);
  for (int n = 0; n < Vr.rows; ++n) {
    double a, b, c;
    rst_to_abc(r[n], s[n], t[n], a, b, c);
    int col = 0;
    for (int i = 0; i <= N; ++i)
      for (int j = 0; j <= N - i; ++j)
        for (int k = 0; k <= N - i - j; ++k, ++col)
          tet_mode_grad(a, b, c, i, j, k, Vr(n, col), Vs(n, col), Vt(n, col));
  }
}

Vec column(const Mat& M, int c) {
  Vec v(M.rows);
  for (int i = 0; i < M.rows; ++i) v[i] = M(i, c);
  return v;
}

} // namespace

// ===========================================================================
// interval
// ===========================================================================

Interval1D build_interval(int N) {
  // reference.cpp:164-188
  require_degree(N);
  Interval1D iv;
  iv.degree = N;
  gauss_lobatto(N + 1, iv.nodes, iv.weights);
  iv.vandermonde = legendre_vandermonde(N, iv.nodes);
  const Mat Vinv = inverse(iv.vandermonde);
  iv.diff = matmul(legendre_grad_vandermonde(N, iv.nodes), Vinv);
  iv.mass = matmul_tn(Vinv, Vinv);
  iv.inv_mass = inverse(iv.mass);
  iv.lift_bottom = column(iv.inv_mass, 0);
  iv.lift_top = column(iv.inv_mass, N);
  iv.lumped_lift_bottom.assign(N + 1, 0.0);
  iv.lumped_lift_bottom[0] = 1.0 / iv.weights[0];
  iv.lumped_lift_top.assign(N + 1, 0.0);
  iv.lumped_lift_top[N] = 1.0 / iv.weights[N];
  jacobi_gauss(N + 2, 0.0, 0.0, iv.gq_nodes, iv.gq_weights);
  iv.interp_gq = matmul(legendre_vandermonde(N, iv.gq_nodes), Vinv);
  return iv;
}

Mat interval_basis_at(const Interval1D& line, const Vec& pts) {
  return matmul(legendre_vandermonde(line.degree, pts), inverse(line.vandermonde));
}

Mat interval_grads_at(const Interval1D& line, const Vec& pts) {
  return matmul(legendre_grad_vandermonde(line.degree, pts), inverse(line.vandermonde));
}

// ===========================================================================
// triangle
// ===========================================================================

namespace {

void triangle_nodes(int N, Vec& r, Vec& s, std::vector<std::array<int, 2>>& lattice) {
  // reference.cpp:196-228: lattice loop j outer, i inner
  const int np = (N + 1) * (N + 2) / 2;
  Vec L1(np), L2(np), L3(np);
  lattice.clear();
  int m = 0;
  for (int j = 0; j <= N; ++j)
    for (int i = 0; i <= N - j; ++i, ++m) {
      L1[m] = double(j) / N;
      L3[m] = double(i) / N;
      L2[m] = 1.0 - L1[m] - L3[m];
      lattice.push_back({i, j});
    }
  Vec dx, dy;
  shift_2d(N, blend_alpha(N), L1, L2, L3, dx, dy);
  r.resize(np);
  s.resize(np);
  const double sq3 = std::sqrt(3.0);
  for (int n = 0; n < np; ++n) {
    const double x = -L2[n] + L3[n] + dx[n];
    const double y = (-L2[n] - L3[n] + 2.0 * L1[n]) / sq3 + dy[n];
    const double l1 = (sq3 * y + 1.0) / 3.0;
    const double l2 = (-3.0 * x - sq3 * y + 2.0) / 6.0;
    const double l3 = (3.0 * x - sq3 * y + 2.0) / 6.0;
    r[n] = -l2 + l3 - l1;
    s[n] = -l2 - l3 + l1;
  }
}

TriangleCubature triangle_cubature(int N) {
  // collapsed Gauss x Gauss-Jacobi(1,0), (N+2)^2 points, b outer (reference.cpp:259-279)
  const int n = N + 2;
  Vec xa, wa, xb, wb;
  jacobi_gauss(n, 0.0, 0.0, xa, wa);
  jacobi_gauss(n, 1.0, 0.0, xb, wb);
  TriangleCubature cub;
  cub.points = Mat(n * n, 2);
  cub.weights.resize(n * n);
  for (int ib = 0; ib < n; ++ib)
    for (int ia = 0; ia < n; ++ia) {
      const int q = ib * n + ia;
      cub.points(q, 0) = 0.5 * (1.0 + xa[ia]) * (1.0 - xb[ib]) - 1.0;
      cub.points(q, 1) = xb[ib];
      cub.weights[q] = 0.5 * wa[ia] * wb[ib];
    }
  cub.exact_degree = 2 * n - 1;
  return cub;
}

} // namespace

Mat triangle_basis_at(const TriangleRef& tri, const Mat& pts) {
  Vec r(pts.rows), s(pts.rows);
  for (int i = 0; i < pts.rows; ++i) {
    r[i] = pts(i, 0);
    s[i] = pts(i, 1);
  }
  return matmul(tri_vandermonde(tri.degree, r, s), tri.inv_vandermonde);
}

void triangle_grads_at(const TriangleRef& tri, const Mat& pts, Mat& dr, Mat& ds) {
  Vec r(pts.rows), s(pts.rows);
  for (int i = 0; i < pts.rows; ++i) {
    r[i] = pts(i, 0);
    s[i] = pts(i, 1);
  }
  Mat Vr, Vs;
  tri_grad_vandermonde(tri.degree, r, s, Vr, Vs);
  dr = matmul(Vr, tri.inv_vandermonde);
  ds = matmul(Vs, tri.inv_vandermonde);
}

TriangleRef build_triangle(int N) {
  // reference.cpp:304-354
  require_degree(N);
  TriangleRef tri;
  tri.degree = N;
  tri.num_nodes = (N + 1) * (N + 2) / 2;
  triangle_nodes(N, tri.r, tri.s, tri.lattice);
  tri.vandermonde = tri_vandermonde(N, tri.r, tri.s);
  tri.cond_vandermonde = cond2(tri.vandermonde);
  tri.inv_vandermonde = inverse(tri.vandermonde);
  Mat Vr, Vs;
  tri_grad_vandermonde(N, tri.r, tri.s, Vr, Vs);
  tri.dr = matmul(Vr, tri.inv_vandermonde);
  tri.ds = matmul(Vs, tri.inv_vandermonde);
  tri.mass = matmul_tn(tri.inv_vandermonde, tri.inv_vandermonde);
  tri.cubature = triangle_cubature(N);
  tri.interp_cub = triangle_basis_at(tri, tri.cubature.points);

  // first moments int l_i l_j r and int l_i l_j s, symmetrised
  const int Q = (int)tri.cubature.weights.size();
  Mat wr = tri.interp_cub, ws = tri.interp_cub;
  for (int q = 0; q < Q; ++q) {
    const double fr = tri.cubature.weights[q] * tri.cubature.points(q, 0);
    const double fs = tri.cubature.weights[q] * tri.cubature.points(q, 1);
    for (int j = 0; j < wr.cols; ++j) {
      wr(q, j) *= fr;
      ws(q, j) *= fs;
    }
  }
  const Mat mr = matmul_tn(tri.interp_cub, wr), ms = matmul_tn(tri.interp_cub, ws);
  tri.moment_r = Mat(mr.rows, mr.cols);
  tri.moment_s = Mat(ms.rows, ms.cols);
  for (int i = 0; i < mr.rows; ++i)
    for (int j = 0; j < mr.cols; ++j) {
      tri.moment_r(i, j) = 0.5 * (mr(i, j) + mr(j, i));
      tri.moment_s(i, j) = 0.5 * (ms(i, j) + ms(j, i));
    }

  // edges e0: s=-1 by r; e1: r+s=0 by s; e2: r=-1 by -s (reference.cpp:337-353)
  const double tol = 1e-8;
  for (int n = 0; n < tri.num_nodes; ++n) {
    if (std::abs(tri.s[n] + 1.0) < tol) tri.edge_nodes[0].push_back(n);
    if (std::abs(tri.r[n] + tri.s[n]) < tol) tri.edge_nodes[1].push_back(n);
    if (std::abs(tri.r[n] + 1.0) < tol) tri.edge_nodes[2].push_back(n);
  }
  std::sort(tri.edge_nodes[0].begin(), tri.edge_nodes[0].end(),
            [&](int a, int b) { return tri.r[a] < tri.r[b]; });
  std::sort(tri.edge_nodes[1].begin(), tri.edge_nodes[1].end(),
            [&](int a, int b) { return tri.s[a] < tri.s[b]; });
  std::sort(tri.edge_nodes[2].begin(), tri.edge_nodes[2].end(),
            [&](int a, int b) { return -tri.s[a] < -tri.s[b]; });
  for (const auto& e : tri.edge_nodes)
    if ((int)e.size() != N + 1) throw NumericalError("triangle edge node detection failed");
  return tri;
}

// ===========================================================================
// wedge
// ===========================================================================

WedgeRef build_wedge_ref(const TriangleRef& tri, const Interval1D& line) {
  // reference.cpp:360-388
  if (tri.degree != line.degree)
    throw ConfigError("wedge reference requires matching triangle/interval degrees");
  WedgeRef w;
  w.degree = tri.degree;
  const int nq = line.degree + 1;
  w.num_tri_nodes = tri.num_nodes;
  w.num_nodes = tri.num_nodes * nq;
  w.r.resize(w.num_nodes);
  w.s.resize(w.num_nodes);
  w.t.resize(w.num_nodes);
  for (int i = 0; i < tri.num_nodes; ++i)
    for (int j = 0; j < nq; ++j) {
      const int id = w.node_id(i, j);
      w.r[id] = tri.r[i];
      w.s[id] = tri.s[i];
      w.t[id] = line.nodes[j];
    }
  for (int i = 0; i < tri.num_nodes; ++i) {
    w.face_nodes[0].push_back(w.node_id(i, 0));
    w.face_nodes[1].push_back(w.node_id(i, nq - 1));
  }
  for (int e = 0; e < 3; ++e)
    for (int a = 0; a < nq; ++a)
      for (int j = 0; j < nq; ++j) w.face_nodes[2 + e].push_back(w.node_id(tri.edge_nodes[e][a], j));
  return w;
}

double wedge_vertex_function(int m, double r, double s, double t) {
  // reference.cpp:642-646
  const double l[3] = {-(r + s) / 2.0, (1.0 + r) / 2.0, (1.0 + s) / 2.0};
  return (m < 3) ? l[m] * (1.0 - t) / 2.0 : l[m - 3] * (1.0 + t) / 2.0;
}

std::array<double, 3> wedge_vertex_function_grad(int m, double r, double s, double t) {
  // reference.cpp:648-656
  const double l[3] = {-(r + s) / 2.0, (1.0 + r) / 2.0, (1.0 + s) / 2.0};
  const double lr[3] = {-0.5, 0.5, 0.0}, ls[3] = {-0.5, 0.0, 0.5};
  const int i = m % 3;
  if (m < 3) {
    const double z = (1.0 - t) / 2.0;
    return {lr[i] * z, ls[i] * z, -0.5 * l[i]};
  }
  const double z = (1.0 + t) / 2.0;
  return {lr[i] * z, ls[i] * z, 0.5 * l[i]};
}

// ===========================================================================
// tetrahedron
// ===========================================================================

namespace {

struct V3d {
  double x, y, z;
};
V3d operator-(V3d a, V3d b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
V3d operator+(V3d a, V3d b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
V3d operator*(double s, V3d a) { return {s * a.x, s * a.y, s * a.z}; }
V3d unit(V3d a) {
  const double n = std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z);
  return {a.x / n, a.y / n, a.z / n};
}

void tet_nodes(int N, Vec& r, Vec& s, Vec& t, std::vector<std::array<int, 3>>& lattice) {
  // reference.cpp:396-482: equispaced barycentric lattice (k, j, i loops),
  // face warps from the triangle warp with the shared alpha, then back to rst.
  const int np = (N + 1) * (N + 2) * (N + 3) / 6;
  const double alpha = blend_alpha(N);
  const double tol = 1e-10;
  Vec L1(np), L2(np), L3(np), L4(np);
  lattice.clear();
  int m = 0;
  for (int k = 0; k <= N; ++k)
    for (int j = 0; j <= N - k; ++j)
      for (int i = 0; i <= N - k - j; ++i, ++m) {
        const double re = -1.0 + 2.0 * i / N, se = -1.0 + 2.0 * j / N, te = -1.0 + 2.0 * k / N;
        L1[m] = (1.0 + te) / 2.0;
        L2[m] = (1.0 + se) / 2.0;
        L3[m] = -(1.0 + re + se + te) / 2.0;
        L4[m] = (1.0 + re) / 2.0;
        lattice.push_back({i, j, k});
      }
  const double s3 = std::sqrt(3.0), s6 = std::sqrt(6.0);
  const V3d v1{-1.0, -1.0 / s3, -1.0 / s6}, v2{1.0, -1.0 / s3, -1.0 / s6},
      v3{0.0, 2.0 / s3, -1.0 / s6}, v4{0.0, 0.0, 3.0 / s6};
  const V3d t1[4] = {unit(v2 - v1), unit(v2 - v1), unit(v3 - v2), unit(v3 - v1)};
  const V3d t2[4] = {unit(v3 - 0.5 * (v1 + v2)), unit(v4 - 0.5 * (v1 + v2)),
                     unit(v4 - 0.5 * (v2 + v3)), unit(v4 - 0.5 * (v1 + v3))};
  std::vector<V3d> xyz(np), shift(np, V3d{0, 0, 0});
  for (int n = 0; n < np; ++n)
    xyz[n] = L3[n] * v1 + L4[n] * v2 + L2[n] * v3 + L1[n] * v4;
  for (int face = 0; face < 4; ++face) {
    const Vec *La, *Lb, *Lc, *Ld;
    switch (face) {
      case 0: La = &L1; Lb = &L2; Lc = &L3; Ld = &L4; break;
      case 1: La = &L2; Lb = &L1; Lc = &L3; Ld = &L4; break;
      case 2: La = &L3; Lb = &L1; Lc = &L4; Ld = &L2; break;
      default: La = &L4; Lb = &L1; Lc = &L3; Ld = &L2; break;
    }
    Vec w1, w2;
    shift_2d(N, alpha, *Lb, *Lc, *Ld, w1, w2);
    for (int n = 0; n < np; ++n) {
      const double la = (*La)[n], lb = (*Lb)[n], lc = (*Lc)[n], ld = (*Ld)[n];
      double blend = lb * lc * ld;
      const double denom = (lb + 0.5 * la) * (lc + 0.5 * la) * (ld + 0.5 * la);
      if (denom > tol) blend = (1.0 + (alpha * la) * (alpha * la)) * blend / denom;
      shift[n] = shift[n] + (blend * w1[n]) * t1[face] + (blend * w2[n]) * t2[face];
      const int interior = int(lb > tol) + int(lc > tol) + int(ld > tol);
      if (la < tol && interior < 3) shift[n] = w1[n] * t1[face] + w2[n] * t2[face];
    }
  }
  Mat A(4, 4);
  const V3d vs[4] = {v1, v2, v3, v4};
  for (int c = 0; c < 4; ++c) {
    A(0, c) = vs[c].x;
    A(1, c) = vs[c].y;
    A(2, c) = vs[c].z;
    A(3, c) = 1.0;
  }
  const Mat Ai = inverse(A);
  r.resize(np);
  s.resize(np);
  t.resize(np);
  for (int n = 0; n < np; ++n) {
    const V3d p = xyz[n] + shift[n];
    const double rhs[4] = {p.x, p.y, p.z, 1.0};
    double L[4] = {0, 0, 0, 0};
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) L[a] += Ai(a, b) * rhs[b];
    r[n] = 2.0 * L[1] - 1.0;
    s[n] = 2.0 * L[2] - 1.0;
    t[n] = 2.0 * L[3] - 1.0;
  }
}

TetCubature tet_cubature(int N) {
  // collapsed Gauss x GJ(1,0) x GJ(2,0), (N+2)^3 points (reference.cpp:518-540)
  const int n = N + 2;
  Vec xa, wa, xb, wb, xc, wc;
  jacobi_gauss(n, 0.0, 0.0, xa, wa);
  jacobi_gauss(n, 1.0, 0.0, xb, wb);
  jacobi_gauss(n, 2.0, 0.0, xc, wc);
  TetCubature cub;
  cub.points = Mat(n * n * n, 3);
  cub.weights.resize(n * n * n);
  int q = 0;
  for (int ic = 0; ic < n; ++ic)
    for (int ib = 0; ib < n; ++ib)
      for (int ia = 0; ia < n; ++ia, ++q) {
        const double a = xa[ia], b = xb[ib], c = xc[ic];
        cub.points(q, 0) = (1.0 + a) * (1.0 - b) * (1.0 - c) / 4.0 - 1.0;
        cub.points(q, 1) = (1.0 + b) * (1.0 - c) / 2.0 - 1.0;
        cub.points(q, 2) = c;
        cub.weights[q] = wa[ia] * wb[ib] * wc[ic] / 8.0;
      }
  cub.exact_degree = 2 * n - 1;
  return cub;
}

} // namespace

Mat tet_basis_at(const TetRef& tet, const Mat& pts) {
  Vec r(pts.rows), s(pts.rows), t(pts.rows);
  for (int i = 0; i < pts.rows; ++i) {
    r[i] = pts(i, 0);
    s[i] = pts(i, 1);
    t[i] = pts(i, 2);
  }
  return matmul(tet_vandermonde(tet.degree, r, s, t), tet.inv_vandermonde);
}

void tet_grads_at(const TetRef& tet, const Mat& pts, Mat& dr, Mat& ds, Mat& dt) {
  Vec r(pts.rows), s(pts.rows), t(pts.rows);
  for (int i = 0; i < pts.rows; ++i) {
    r[i] = pts(i, 0);
    s[i] = pts(i, 1);
    t[i] = pts(i, 2);
  }
  Mat Vr, Vs, Vt;
  tet_grad_vandermonde(tet.degree, r, s, t, Vr, Vs, Vt);
  dr = matmul(Vr, tet.inv_vandermonde);
  ds = matmul(Vs, tet.inv_vandermonde);
  dt = matmul(Vt, tet.inv_vandermonde);
}

TetRef build_tet_ref(int N) {
  // reference.cpp:558-626
  require_degree(N);
  TetRef tet;
  tet.degree = N;
  tet.num_nodes = (N + 1) * (N + 2) * (N + 3) / 6;
  tet.num_face_nodes = (N + 1) * (N + 2) / 2;
  tet_nodes(N, tet.r, tet.s, tet.t, tet.lattice);
  tet.vandermonde = tet_vandermonde(N, tet.r, tet.s, tet.t);
  tet.cond_vandermonde = cond2(tet.vandermonde);
  tet.inv_vandermonde = inverse(tet.vandermonde);
  Mat Vr, Vs, Vt;
  tet_grad_vandermonde(N, tet.r, tet.s, tet.t, Vr, Vs, Vt);
  tet.dr = matmul(Vr, tet.inv_vandermonde);
  tet.ds = matmul(Vs, tet.inv_vandermonde);
  tet.dt = matmul(Vt, tet.inv_vandermonde);
  tet.mass = matmul_tn(tet.inv_vandermonde, tet.inv_vandermonde);
  tet.cubature = tet_cubature(N);
  tet.interp_cub = tet_basis_at(tet, tet.cubature.points);

  tet.face_vertices = {{{0, 1, 2}, {0, 1, 3}, {1, 2, 3}, {0, 2, 3}}};
  const double corners[4][3] = {{-1, -1, -1}, {1, -1, -1}, {-1, 1, -1}, {-1, -1, 1}};
  const TriangleRef tri = build_triangle(N);
  for (int f = 0; f < 4; ++f) {
    const double* c0 = corners[tet.face_vertices[f][0]];
    const double* c1 = corners[tet.face_vertices[f][1]];
    const double* c2 = corners[tet.face_vertices[f][2]];
    tet.face_nodes[f].resize(tet.num_face_nodes);
    for (int m = 0; m < tet.num_face_nodes; ++m) {
      const double l0 = -(tri.r[m] + tri.s[m]) / 2.0, l1 = (1.0 + tri.r[m]) / 2.0,
                   l2 = (1.0 + tri.s[m]) / 2.0;
      double p[3];
      for (int d = 0; d < 3; ++d) p[d] = l0 * c0[d] + l1 * c1[d] + l2 * c2[d];
      int best = -1;
      double bestd = 1e30;
      for (int n = 0; n < tet.num_nodes; ++n) {
        const double dx = tet.r[n] - p[0], dy = tet.s[n] - p[1], dz = tet.t[n] - p[2];
        const double d2 = dx * dx + dy * dy + dz * dz;
        if (d2 < bestd) {
          bestd = d2;
          best = n;
        }
      }
      if (std::sqrt(bestd) > 1e-10)
        throw NumericalError("tet face nodes do not conform to triangle nodes");
      tet.face_nodes[f][m] = best;
    }
  }
  // reference lift: (V V^T) * embedded triangle mass per face
  const int nfp = tet.num_face_nodes;
  const Mat vvt = matmul(tet.vandermonde, transpose(tet.vandermonde));
  tet.lift = Mat(tet.num_nodes, 4 * nfp);
  for (int f = 0; f < 4; ++f) {
    Mat emb(tet.num_nodes, nfp);
    for (int m = 0; m < nfp; ++m)
      for (int n = 0; n < nfp; ++n) emb(tet.face_nodes[f][m], n) = tri.mass(m, n);
    const Mat blk = matmul(vvt, emb);
    for (int i = 0; i < tet.num_nodes; ++i)
      for (int n = 0; n < nfp; ++n) tet.lift(i, f * nfp + n) = blk(i, n);
  }
  return tet;
}

References build_references(int N) {
  References refs;
  refs.degree = N;
  refs.line = build_interval(N);
  refs.tri = build_triangle(N);
  refs.wedge = build_wedge_ref(refs.tri, refs.line);
  refs.tet = build_tet_ref(N);
  return refs;
}

} // namespace prismdg
