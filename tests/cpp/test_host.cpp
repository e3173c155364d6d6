// Port of the reference's unit and acceptance checks that pin the hot path
// (proj/tests/test_*.cpp, proj/tests/acceptance.cpp), run against this repo's
// host setup library and the CPU oracle (oracle/).  CPU only: no CUDA calls.
// Usage: test_host [substring-filter]; prints one line per case, exit 1 on failure.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "oracle.hpp"
#include "prismdg/discretization.hpp"
#include "prismdg/solver.hpp"

using namespace prismdg;

namespace {

int g_fail = 0, g_checks = 0;
std::string g_case;

#define CHECK(cond)                                                                        \
  do {                                                                                     \
    ++g_checks;                                                                            \
    if (!(cond)) {                                                                         \
      ++g_fail;                                                                            \
      std::printf("  FAIL %s:%d [%s] %s\n", __FILE__, __LINE__, g_case.c_str(), #cond);   \
    }                                                                                      \
  } while (0)
#define CHECK_CLOSE(a, b, tol) CHECK(std::abs((a) - (b)) <= (tol) * std::max(1.0, std::abs(b)))
#define CHECK_THROWS(stmt, T)    \
  do {                           \
    bool thrown_ = false;        \
    try {                        \
      stmt;                      \
    } catch (const T&) {         \
      thrown_ = true;            \
    }                            \
    CHECK(thrown_);              \
  } while (0)

struct Case {
  const char* name;
  std::function<void()> fn;
};
std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
#define TEST(name) \
  static void name(); \
  static Reg reg_##name(#name, name); \
  static void name()

double u01(std::mt19937_64& g) { return double(g() >> 11) * 0x1.0p-53; }
Vec random_vec(int n, std::mt19937_64& g) {
  Vec v(n);
  for (int i = 0; i < n; ++i) v[i] = 2.0 * u01(g) - 1.0;
  return v;
}
double norm(const Vec& v) {
  double s = 0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}
double rel_err(const Vec& got, const Vec& want) {
  double s = 0;
  for (std::size_t i = 0; i < got.size(); ++i) s += (got[i] - want[i]) * (got[i] - want[i]);
  return std::sqrt(s) / std::max(norm(want), 1e-14);
}
double max_abs(const Vec& v) {
  double m = 0;
  for (double x : v) m = std::max(m, std::abs(x));
  return m;
}
const WedgeVerts kRefWedge = {{{-1, -1, -1}, {1, -1, -1}, {-1, 1, -1}, {-1, -1, 1}, {1, -1, 1}, {-1, 1, 1}}};

Discretization small_box(int n, int degree, FluxMode mode = FluxMode::upwind,
                         QuadratureMode qm = QuadratureMode::exact) {
  FluxConfig flux;
  flux.mode = mode;
  return build_discretization(structured_wedge_box(n), degree, flux, qm, 1);
}

} // namespace

// ---------------------------------------------------------------- jacobi (test_jacobi.cpp)
TEST(gauss_rules_exact) {
  for (int n = 1; n <= 8; ++n) {
    Vec x, w;
    jacobi_gauss(n, 0.0, 0.0, x, w);
    for (int k = 0; k <= 2 * n - 1; ++k) {
      double q = 0.0;
      for (int i = 0; i < n; ++i) q += w[i] * std::pow(x[i], k);
      CHECK(std::abs(q - ((k % 2 == 0) ? 2.0 / (k + 1.0) : 0.0)) < 1e-13);
    }
  }
  Vec x, w;
  jacobi_gauss(4, 1.0, 0.0, x, w);
  double sw = 0, sx = 0;
  for (int i = 0; i < 4; ++i) {
    sw += w[i];
    sx += w[i] * x[i];
  }
  CHECK_CLOSE(sw, 2.0, 1e-12);
  CHECK_CLOSE(sx, -2.0 / 3.0, 1e-12);
}

TEST(jacobi_orthonormal) {
  Vec x, w;
  jacobi_gauss(12, 0.0, 0.0, x, w);
  for (int m = 0; m <= 5; ++m)
    for (int n = 0; n <= 5; ++n) {
      double q = 0.0;
      for (std::size_t i = 0; i < x.size(); ++i) q += w[i] * jacobi_p(m, 0, 0, x[i]) * jacobi_p(n, 0, 0, x[i]);
      CHECK(std::abs(q - (m == n ? 1.0 : 0.0)) < 1e-12);
    }
}

TEST(gll_closed_form_and_newton) {
  Vec x, w;
  gauss_lobatto(3, x, w);
  CHECK_CLOSE(x[1], 0.0, 1e-14);
  CHECK_CLOSE(w[0], 1.0 / 3.0, 1e-14);
  CHECK_CLOSE(w[1], 4.0 / 3.0, 1e-14);
  for (int npts = 2; npts <= 10; ++npts) {
    Vec xo, wo;
    gauss_lobatto(npts, x, w);
    oracle::gll_newton(npts, xo, wo);
    CHECK(x[0] == -1.0 && x[npts - 1] == 1.0);
    for (int i = 0; i < npts; ++i) {
      CHECK(std::abs(x[i] - xo[i]) < 1e-13);
      CHECK(std::abs(w[i] - wo[i]) < 1e-13 * std::abs(wo[i]) + 1e-15);
      CHECK(std::abs(x[i] + x[npts - 1 - i]) < 1e-13);
      if (i) CHECK(x[i] > x[i - 1]);
    }
  }
}

// ---------------------------------------------------------------- reference elements
TEST(degree_range_enforced) {
  CHECK_THROWS(build_interval(0), ConfigError);
  CHECK_THROWS(build_interval(10), ConfigError);
  CHECK_THROWS(build_triangle(0), ConfigError);
  CHECK_THROWS(build_tet_ref(12), ConfigError);
}

TEST(triangle_basics) {
  for (int N = 1; N <= 7; ++N) {
    const TriangleRef tri = build_triangle(N);
    const Mat eye = matmul(tri.vandermonde, tri.inv_vandermonde);
    CHECK(max_abs_diff(eye, Mat::identity(tri.num_nodes)) < 1e-10);
    CHECK(std::isfinite(tri.cond_vandermonde) && tri.cond_vandermonde < 1e6);
    // derivative exactness on monomials r^a s^b, a+b <= N (test_reference.cpp:74-89)
    for (int a = 0; a <= N; ++a)
      for (int b = 0; a + b <= N; ++b) {
        Vec f(tri.num_nodes), fr(tri.num_nodes), fs(tri.num_nodes);
        for (int n = 0; n < tri.num_nodes; ++n) {
          f[n] = std::pow(tri.r[n], a) * std::pow(tri.s[n], b);
          fr[n] = a ? a * std::pow(tri.r[n], a - 1) * std::pow(tri.s[n], b) : 0.0;
          fs[n] = b ? b * std::pow(tri.r[n], a) * std::pow(tri.s[n], b - 1) : 0.0;
        }
        const Vec gr = matvec(tri.dr, f), gs = matvec(tri.ds, f);
        double er = 0, es = 0;
        for (int n = 0; n < tri.num_nodes; ++n) {
          er = std::max(er, std::abs(gr[n] - fr[n]));
          es = std::max(es, std::abs(gs[n] - fs[n]));
        }
        CHECK(er < 1e-10 && es < 1e-10);
      }
    double sw = 0, mr = 0, ms = 0;
    for (std::size_t q = 0; q < tri.cubature.weights.size(); ++q) {
      sw += tri.cubature.weights[q];
      mr += tri.cubature.weights[q] * tri.cubature.points((int)q, 0);
      ms += tri.cubature.weights[q] * tri.cubature.points((int)q, 1);
    }
    CHECK_CLOSE(sw, 2.0, 1e-13);
    CHECK_CLOSE(mr, -2.0 / 3.0, 1e-13);
    CHECK_CLOSE(ms, -2.0 / 3.0, 1e-13);
    // edges carry the GLL distribution
    Vec gll, wg;
    gauss_lobatto(N + 1, gll, wg);
    const double tv[3][2] = {{-1, -1}, {1, -1}, {-1, 1}};
    for (int e = 0; e < 3; ++e)
      for (int a = 0; a <= N; ++a) {
        const double xi = gll[a];
        const double er = tv[e][0] * (1 - xi) / 2 + tv[(e + 1) % 3][0] * (1 + xi) / 2;
        const double es = tv[e][1] * (1 - xi) / 2 + tv[(e + 1) % 3][1] * (1 + xi) / 2;
        const int id = tri.edge_nodes[e][a];
        CHECK(std::abs(tri.r[id] - er) < 1e-12 && std::abs(tri.s[id] - es) < 1e-12);
      }
  }
}

TEST(tet_faces_conform_and_derivatives) {
  for (int N = 1; N <= 6; ++N) {
    const References refs = build_references(N);
    const auto& tet = refs.tet;
    CHECK(tet.num_nodes == (N + 1) * (N + 2) * (N + 3) / 6);
    for (int a = 0; a <= N; ++a)
      for (int b = 0; a + b <= N; ++b)
        for (int c = 0; a + b + c <= N; ++c) {
          Vec f(tet.num_nodes), fr(tet.num_nodes);
          for (int n = 0; n < tet.num_nodes; ++n) {
            f[n] = std::pow(tet.r[n], a) * std::pow(tet.s[n], b) * std::pow(tet.t[n], c);
            fr[n] = a ? a * std::pow(tet.r[n], a - 1) * std::pow(tet.s[n], b) * std::pow(tet.t[n], c) : 0.0;
          }
          const Vec g = matvec(tet.dr, f);
          double err = 0;
          for (int n = 0; n < tet.num_nodes; ++n) err = std::max(err, std::abs(g[n] - fr[n]));
          CHECK(err < 1e-9);
        }
  }
}

TEST(wedge_reference_structure) {
  const References refs = build_references(3);
  CHECK(refs.wedge.num_nodes == 40);
  for (int i = 0; i < refs.tri.num_nodes; ++i)
    for (int j = 0; j <= 3; ++j) {
      const int id = refs.wedge.node_id(i, j);
      CHECK(refs.wedge.r[id] == refs.tri.r[i] && refs.wedge.t[id] == refs.line.nodes[j]);
    }
  const References r1 = build_references(1);
  CHECK(r1.wedge.num_nodes == 6);
  for (double r : {-0.7, 0.1}) {
    double sum = 0;
    for (int m = 0; m < 6; ++m) sum += wedge_vertex_function(m, r, -0.2, 0.3);
    CHECK(std::abs(sum - 1.0) < 1e-14);
  }
}

// ---------------------------------------------------------------- geometry (test_geometry.cpp)
TEST(geometry_identity_and_stretch) {
  const References refs = build_references(3);
  const ElementGeometry g = wedge_geometry(kRefWedge, refs);
  CHECK_CLOSE(g.rx, 1.0, 1e-14);
  CHECK(std::abs(g.ry) < 1e-14 && std::abs(g.sx) < 1e-14);
  CHECK_CLOSE(g.tzJ, 1.0, 1e-14);
  CHECK_CLOSE(g.j0, 1.0, 1e-14);
  CHECK_CLOSE(g.volume, 4.0, 1e-14);
  CHECK(max_abs(g.txJ) < 1e-14 && max_abs(g.tyJ) < 1e-14);
  auto v = kRefWedge;
  for (int i = 3; i < 6; ++i) v[i][2] = 3.0;
  const ElementGeometry gs = wedge_geometry(v, refs);
  CHECK_CLOSE(gs.j0, 2.0, 1e-14);
  CHECK_CLOSE(gs.tzJ, 1.0, 1e-14);
  CHECK(g.faces[2].normal[1] < -0.999999 && g.faces[4].normal[0] < -0.999999);
  CHECK(std::abs(g.faces[3].normal[0] - std::sqrt(0.5)) < 1e-14);
  CHECK(g.faces[0].normal[2] < -0.999999 && g.faces[1].normal[2] > 0.999999);
  auto bad = kRefWedge;
  for (int i = 3; i < 6; ++i) bad[i][2] = -1.0;
  CHECK_THROWS(wedge_geometry(bad, refs), MeshError);
}

TEST(lemma1_property_suite) {
  // acceptance criterion 6 (acceptance.cpp:239-247): worst violation < 1e-13
  std::mt19937_64 gen(777);
  double worst = 0.0;
  for (int trial = 0; trial < 100; ++trial)
    worst = std::max(worst, oracle::vertical_wedge_property_violation(oracle::random_vertical_wedge(gen)));
  CHECK(worst < 1e-13);
}

TEST(closed_form_factors_match_jacobian) {
  std::mt19937_64 gen(11);
  const References refs = build_references(3);
  for (int trial = 0; trial < 10; ++trial) {
    const auto v = oracle::random_vertical_wedge(gen);
    const ElementGeometry g = wedge_geometry(v, refs);
    for (double r : {-0.5, 0.2})
      for (double s : {-0.6, -0.1}) {
        double A[3][3], Ai[3][3];
        oracle::wedge_jacobian_matrix(v, r, s, 0.3, A);
        inv3(A, Ai);
        const double J = det3(A);
        CHECK(std::abs(Ai[0][0] - g.rx) < 1e-12 * std::max(1.0, std::abs(g.rx)));
        CHECK(std::abs(Ai[1][1] - g.sy) < 1e-12 * std::max(1.0, std::abs(g.sy)));
        CHECK(std::abs(Ai[2][2] * J - g.tzJ) < 1e-12 * std::max(1.0, std::abs(g.tzJ)));
        CHECK(std::abs(J - g.jacobian_at(r, s)) < 1e-12 * std::max(1.0, std::abs(J)));
      }
  }
}

// ---------------------------------------------------------------- operators (test_operators.cpp)
TEST(affine_prism_lift_is_scaled_identity) {
  const References refs = build_references(3);
  auto v = kRefWedge;
  for (int i = 3; i < 6; ++i) v[i][2] = 3.0;
  const WedgeOperators ops = build_wedge_operators(wedge_geometry(v, refs), refs);
  CHECK(max_abs_diff(ops.tri_lift, scaled(Mat::identity(refs.tri.num_nodes), 0.5)) < 1e-12);
}

TEST(kronecker_vs_dense_oracle) {
  // test_operators.cpp:43-75 (seed 99, N=1..4) and acceptance criterion 5
  std::mt19937_64 gen(99);
  double worst = 0;
  for (int N = 1; N <= 4; ++N) {
    const References refs = build_references(N);
    for (int trial = 0; trial < 3; ++trial) {
      const auto verts = oracle::random_vertical_wedge(gen);
      const ElementGeometry g = wedge_geometry(verts, refs);
      const WedgeOperators ops = build_wedge_operators(g, refs);
      const oracle::DenseWedgeOps dense = oracle::dense_wedge_ops(verts, refs);
      const int np = refs.wedge.num_nodes;
      const Vec u = random_vec(np, gen);
      Vec mu;
      apply_wedge_mass(g, refs, QuadratureMode::exact, u, mu);
      worst = std::max(worst, rel_err(mu, matvec(dense.mass, u)));
      Vec dx, dy, dz;
      apply_wedge_derivatives(ops, refs, u, dx, dy, dz);
      worst = std::max({worst, rel_err(dx, matvec(dense.dx, u)), rel_err(dy, matvec(dense.dy, u)),
                        rel_err(dz, matvec(dense.dz, u))});
      for (int f = 0; f < 5; ++f) {
        const Vec flux = random_vec((int)refs.wedge.face_nodes[f].size(), gen);
        Vec out(np, 0.0);
        apply_wedge_lift(ops, refs, QuadratureMode::exact, f, flux, out);
        worst = std::max(worst, rel_err(out, matvec(dense.lift[f], flux)));
      }
    }
  }
  std::printf("  kronecker vs dense worst rel %.3e\n", worst);
  CHECK(worst < 1e-11);
}

TEST(derivatives_exact_on_wedge_space) {
  std::mt19937_64 gen(7);
  const References refs = build_references(3);
  const auto verts = oracle::random_vertical_wedge(gen);
  const WedgeOperators ops = build_wedge_operators(wedge_geometry(verts, refs), refs);
  const int np = refs.wedge.num_nodes;
  Vec X(np), Y(np), Z(np), ones(np, 1.0), f(np), fx(np);
  for (int n = 0; n < np; ++n) {
    const auto x = wedge_map(verts, refs.wedge.r[n], refs.wedge.s[n], refs.wedge.t[n]);
    X[n] = x[0];
    Y[n] = x[1];
    Z[n] = x[2];
    f[n] = x[0] * x[1] * x[2];
    fx[n] = x[1] * x[2];
  }
  Vec dx, dy, dz;
  apply_wedge_derivatives(ops, refs, ones, dx, dy, dz);
  CHECK(max_abs(dx) < 1e-13 && max_abs(dy) < 1e-13 && max_abs(dz) < 1e-13);
  apply_wedge_derivatives(ops, refs, Z, dx, dy, dz);
  for (int n = 0; n < np; ++n) dz[n] -= 1.0;
  CHECK(max_abs(dx) < 1e-12 && max_abs(dy) < 1e-12 && max_abs(dz) < 1e-12);
  apply_wedge_derivatives(ops, refs, f, dx, dy, dz);
  for (int n = 0; n < np; ++n) dx[n] -= fx[n];
  CHECK(max_abs(dx) < 1e-11);
}

TEST(tet_operators_vs_dense) {
  const References refs = build_references(3);
  std::mt19937_64 gen(3);
  const auto verts = oracle::random_tet(gen);
  const ElementGeometry g = tet_geometry(verts);
  const TetOperators ops = build_tet_operators(g);
  const oracle::DenseTetOps dense = oracle::dense_tet_ops(verts, refs);
  const int np = refs.tet.num_nodes;
  const Vec w = random_vec(np, gen);
  Vec dx, dy, dz;
  apply_tet_derivatives(ops, refs, w, dx, dy, dz);
  CHECK(rel_err(dx, matvec(dense.dx, w)) < 1e-12);
  CHECK(rel_err(dz, matvec(dense.dz, w)) < 1e-12);
  Vec mu;
  apply_tet_mass(g, refs, w, mu);
  CHECK(rel_err(mu, matvec(dense.mass, w)) < 1e-12);
  for (int f = 0; f < 4; ++f) {
    const Vec flux = random_vec(refs.tet.num_face_nodes, gen);
    Vec out(np, 0.0);
    apply_tet_lift(ops, refs, f, flux, out);
    CHECK(rel_err(out, matvec(dense.lift[f], flux)) < 1e-11);
  }
}

TEST(storage_budget) {
  // test_operators.cpp:239-270: 38 doubles at N=1, 838 at N=5, tets 13
  for (int N = 1; N <= kMaxDegree; ++N) {
    const References refs = build_references(N);
    std::mt19937_64 gen(N);
    const WedgeOperators ops =
        build_wedge_operators(wedge_geometry(oracle::random_vertical_wedge(gen), refs), refs);
    const std::size_t nt = refs.tri.num_nodes;
    CHECK(ops.storage_floats() <= nt * nt + 3 * nt * (N + 1) + 8 * (N + 1));
    if (N == 1) CHECK(ops.storage_floats() == 38);
    if (N == 5) CHECK(ops.storage_floats() == 838);
  }
  CHECK(build_tet_operators(tet_geometry({{{-1, -1, -1}, {1, -1, -1}, {-1, 1, -1}, {-1, -1, 1}}})).storage_floats() == 13);
}

// ---------------------------------------------------------------- mesh (test_mesh.cpp)
TEST(mesh_counts_and_connectivity) {
  const HybridMesh hybrid = structured_hybrid_box(1, 1, 1, 1);
  CHECK(hybrid.num_wedges() == 2 && hybrid.num_tets() == 6);
  CHECK_CLOSE(mesh_volume(hybrid), 8.0, 1e-13);
  const HybridMesh tets = structured_hybrid_box(2, 2, 0, 2);
  CHECK(tets.num_tets() == 48);
  const References refs1 = build_references(1);
  const Connectivity ct = build_connectivity(tets, refs1);
  CHECK(ct.num_boundary_faces == 48);
  CHECK(ct.num_interior_pairs == (48 * 4 - 48) / 2);
  // hybrid: every wedge's bottom face pairs with a tet (8 pairs)
  const HybridMesh h2 = structured_hybrid_box(2, 2, 1, 1);
  const References refs3 = build_references(3);
  const Connectivity c2 = build_connectivity(h2, refs3);
  int pairs = 0;
  for (int w = 0; w < h2.num_wedges(); ++w) {
    const FaceConn& fc = c2.at(w, 0);
    CHECK(fc.nbr >= 0 && h2.kind(fc.nbr) == ElemKind::tet);
    ++pairs;
  }
  CHECK(pairs == 8);
  // single wedge: 5 boundary faces; two stacked wedges: identity permutation
  SurfaceTriangulation s;
  s.vertices = {{0, 0}, {1, 0}, {0, 1}};
  s.z_bottom.assign(3, 0.0);
  s.z_top.assign(3, 1.0);
  s.triangles = {{0, 1, 2}};
  const References refs2 = build_references(2);
  const Connectivity cs = build_connectivity(extrude_layer(s, 1), refs2);
  CHECK(cs.num_boundary_faces == 5 && cs.num_interior_pairs == 0);
  const Connectivity cst = build_connectivity(extrude_layer(s, 2), refs2);
  CHECK(cst.num_interior_pairs == 1);
  const FaceConn& fc = cst.at(0, 1);
  CHECK(fc.nbr == 1 && fc.nbr_face == 0);
  const auto& perm = cst.perm(0, 1);
  for (std::size_t i = 0; i < perm.size(); ++i) CHECK(perm[i] == (int)i);
}

TEST(perturbation_deterministic) {
  const HybridMesh base = structured_wedge_box(2);
  const HybridMesh a = perturb_vertically(base, 0.3, 7), b = perturb_vertically(base, 0.3, 7);
  bool same = a.vertices.size() == b.vertices.size();
  for (std::size_t v = 0; same && v < a.vertices.size(); ++v) same = a.vertices[v][2] == b.vertices[v][2];
  CHECK(same);
  const References refs = build_references(2);
  bool nonconst = false;
  for (int w = 0; w < a.num_wedges(); ++w) {
    CHECK(is_vertically_mapped(a.wedge_verts(w)));
    const ElementGeometry g = wedge_geometry(a.wedge_verts(w), refs);
    if (std::abs(g.j_r) + std::abs(g.j_s) > 1e-8) nonconst = true;
  }
  CHECK(nonconst);
  for (const auto& p : a.vertices)
    if (std::abs(std::abs(p[2]) - 1.0) < 0.4) CHECK(std::abs(std::abs(p[2]) - 1.0) < 1e-14);
  CHECK_THROWS(perturb_vertically(base, 0.5, 7), ConfigError);
  for (int n : {2, 4}) CHECK_CLOSE(mesh_volume(arnold_wedge_box(n, 0.25)), 8.0, 1e-12);
  for (int fam = 0; fam < 3; ++fam) {
    const HybridMesh m = make_family_mesh(static_cast<MeshFamily>(fam), 0.5);
    CHECK(m.num_wedges() == 128);
    CHECK_CLOSE(mesh_volume(m), 8.0, 1e-10);
  }
  CHECK_THROWS(make_family_mesh(MeshFamily::structured, 0.3), ConfigError);
}

TEST(hybrid_conformity_acceptance8) {
  // acceptance criterion 8: 8 wedge-tet faces, node distance <= 2e-10, jump <= 1e-12
  const Discretization d = build_discretization(structured_hybrid_box(2, 2, 1, 1), 3);
  int iface = 0;
  double worst = 0.0;
  for (int e = 0; e < d.num_elements(); ++e)
    for (int f = 0; f < d.mesh.num_faces(e); ++f) {
      const FaceConn& fc = d.conn.at(e, f);
      if (fc.nbr < 0 || d.mesh.kind(e) != ElemKind::wedge || d.mesh.kind(fc.nbr) != ElemKind::tet) continue;
      ++iface;
      const auto mine = face_node_coords(d.mesh, d.refs, e, f);
      const auto theirs = face_node_coords(d.mesh, d.refs, fc.nbr, fc.nbr_face);
      const auto& perm = d.conn.perm(e, f);
      for (std::size_t i = 0; i < mine.size(); ++i)
        worst = std::max(worst, std::hypot(mine[i][0] - theirs[perm[i]][0], mine[i][1] - theirs[perm[i]][1],
                                           mine[i][2] - theirs[perm[i]][2]));
    }
  CHECK(iface == 8);
  CHECK(worst <= 2e-10);
  const SolutionState s = make_initial_state(d, standing_wave(), 0.0);
  double jump = 0.0;
  for (int e = 0; e < d.num_elements(); ++e)
    for (int f = 0; f < d.mesh.num_faces(e); ++f) {
      if (d.conn.at(e, f).nbr < 0) continue;
      const int nbr = d.conn.at(e, f).nbr;
      const auto& my = d.my_nodes(e, f);
      for (std::size_t i = 0; i < my.size(); ++i)
        for (int fld = 0; fld < 4; ++fld)
          jump = std::max(jump, std::abs(s.u[d.elem_offset[e] + fld * d.np(e) + my[i]] -
                                         s.u[d.elem_offset[nbr] + fld * d.np(nbr) + d.nbr_node(e, f, (int)i)]));
    }
  CHECK(jump <= 1e-12);
}

// ---------------------------------------------------------------- mesh files (test_mesh.cpp:277-340)
static std::string tmp_file(const char* name) {
  const char* d = std::getenv("TMPDIR");
  return std::string(d && *d ? d : "/tmp") + "/" + name;
}
static void write_text(const std::string& path, const char* text) {
  std::FILE* f = std::fopen(path.c_str(), "w");
  std::fputs(text, f);
  std::fclose(f);
}

TEST(mesh_file_round_trip) {
  // perturbed hybrid mesh with media jumps and a boundary tag: every double survives the
  // 17-digit text form, and the reloaded mesh discretises to the same connectivity
  HybridMesh mesh = perturb_vertically(structured_hybrid_box(2, 2, 1, 1, {1.0, 1.0}, {1.5, 3.0}), 0.2, 7);
  mesh.boundary_tags[{0, 0}] = 3;
  const std::string path = tmp_file("pdg_roundtrip.mesh");
  save_mesh(mesh, path);
  const HybridMesh loaded = load_mesh(path);
  CHECK(loaded.vertices == mesh.vertices);
  CHECK(loaded.wedges == mesh.wedges);
  CHECK(loaded.tets == mesh.tets);
  CHECK(loaded.media.size() == mesh.media.size());
  for (std::size_t e = 0; e < mesh.media.size(); ++e)
    CHECK(loaded.media[e].rho == mesh.media[e].rho && loaded.media[e].kappa == mesh.media[e].kappa);
  CHECK(loaded.boundary_tags == mesh.boundary_tags);
  const Discretization a = build_discretization(mesh, 2), b = build_discretization(loaded, 2);
  bool same = a.total_dofs == b.total_dofs;
  for (int e = 0; same && e < a.num_elements(); ++e)
    for (int f = 0; f < a.mesh.num_faces(e); ++f)
      same = same && a.conn.at(e, f).nbr == b.conn.at(e, f).nbr && a.conn.at(e, f).nbr_face == b.conn.at(e, f).nbr_face &&
             a.conn.at(e, f).tag == b.conn.at(e, f).tag &&
             (a.conn.at(e, f).nbr < 0 || a.conn.perm(e, f) == b.conn.perm(e, f));
  CHECK(same);
  std::remove(path.c_str());
}

TEST(mesh_loader_rejects_invalid) {
  const std::string path = tmp_file("pdg_bad.mesh");
  // top vertex shifted in x: not vertically mapped, error names the wedge
  write_text(path, "$Vertices\n6\n0 0 0\n1 0 0\n0 1 0\n0.5 0 1\n1 0 1\n0 1 1\n$Wedges\n1\n1 2 3 4 5 6\n$Media\n1\n1 1\n");
  bool named = false;
  try {
    load_mesh(path);
  } catch (const MeshError& e) {
    named = std::string(e.what()).find("wedge 1") != std::string::npos;
  }
  CHECK(named);
  // negative bulk modulus
  write_text(path, "$Vertices\n6\n0 0 0\n1 0 0\n0 1 0\n0 0 1\n1 0 1\n0 1 1\n$Wedges\n1\n1 2 3 4 5 6\n$Media\n1\n1 -2\n");
  CHECK_THROWS(load_mesh(path), MeshError);
  // malformed record: error carries the line number
  write_text(path, "$Vertices\n3\nnot a number\n");
  bool lined = false;
  try {
    load_mesh(path);
  } catch (const MeshError& e) {
    lined = std::string(e.what()).find(":3") != std::string::npos;
  }
  CHECK(lined);
  write_text(path, "$Bogus\n0\n");
  CHECK_THROWS(load_mesh(path), MeshError);
  CHECK_THROWS(load_mesh(tmp_file("pdg_no_such_dir/x.mesh")), MeshError);
  std::remove(path.c_str());
}

TEST(surface_file_loads) {
  const std::string path = tmp_file("pdg_surface.txt");
  write_text(path, "$SurfaceVertices\n3\n0 0 0 1\n1 0 0 1\n0 1 0 1\n$SurfaceTriangles\n1\n1 2 3\n");
  const SurfaceTriangulation s = load_surface(path);
  CHECK(s.vertices.size() == 3);
  CHECK(s.triangles.size() == 1);
  const HybridMesh mesh = extrude_layer(s, 2);
  CHECK(mesh.num_wedges() == 2);
  CHECK_CLOSE(mesh_volume(mesh), 0.5, 1e-14);
  std::remove(path.c_str());
}

// ---------------------------------------------------------------- solver via the CPU oracle
TEST(oracle_zero_state_zero_rhs) {
  const Discretization d = small_box(1, 2);
  std::vector<double> u(d.total_dofs, 0.0), rhs(d.total_dofs, 1.0);
  oracle::compute_rhs(d, u.data(), rhs.data(), 1);
  bool all0 = true;
  for (double v : rhs) all0 = all0 && v == 0.0;
  CHECK(all0);
}

TEST(oracle_standing_wave_rhs_converges) {
  // test_solver.cpp:54-84: error ratio > 3 under h/2 at N=2
  std::vector<double> errs;
  const double k = M_PI / 2.0;
  for (int n : {1, 2, 4}) {
    const Discretization d = small_box(n, 2);
    const SolutionState s = make_initial_state(d, standing_wave(), 0.0);
    std::vector<double> rhs(d.total_dofs);
    oracle::compute_rhs(d, s.u.data(), rhs.data(), 1);
    double emax = 0.0;
    for (int e = 0; e < d.num_elements(); ++e)
      for (int q = 0; q < d.np(e); ++q) {
        const Vert3 x = d.node_xyz(e, q);
        const double px = -k * std::sin(k * x[0]) * std::cos(k * x[1]) * std::cos(k * x[2]);
        emax = std::max(emax, std::abs(rhs[d.elem_offset[e] + q]));
        emax = std::max(emax, std::abs(rhs[d.elem_offset[e] + d.np(e) + q] + px));
      }
    errs.push_back(emax);
  }
  CHECK(errs[1] < errs[0] && errs[2] < errs[1] && errs[1] / errs[2] > 3.0);
}

TEST(oracle_rhs_thread_invariant) {
  // test_solver.cpp:202-212: bitwise identical for 1 vs 4 threads
  const Discretization d = build_discretization(structured_hybrid_box(2, 2, 1, 1), 3);
  const SolutionState s = make_initial_state(d, standing_wave(), 0.0);
  std::vector<double> r1(d.total_dofs), r4(d.total_dofs);
  oracle::compute_rhs(d, s.u.data(), r1.data(), 1);
  oracle::compute_rhs(d, s.u.data(), r4.data(), 4);
  CHECK(r1 == r4);
}

TEST(oracle_energy_closed_form) {
  // test_solver.cpp:146-162: E(p=1) = 4.0 (rel 1e-12), 0 for zero state
  const Discretization d = small_box(2, 2);
  std::vector<double> u(d.total_dofs, 0.0);
  CHECK(oracle::compute_energy(d, u.data(), 1) == 0.0);
  for (int e = 0; e < d.num_elements(); ++e)
    for (int q = 0; q < d.np(e); ++q) u[d.elem_offset[e] + q] = 1.0;
  CHECK(std::abs(oracle::compute_energy(d, u.data(), 1) - 4.0) < 4e-12);
}

TEST(oracle_upwind_energy_decay) {
  Discretization d = small_box(2, 2);
  SolutionState s = make_initial_state(d, standing_wave(), 0.0);
  double t = 0.0;
  const auto r = oracle::run_simulation(d, s.u, t, 0.5, 0.5, 0.0, 0.0, 2);
  CHECK(r.stable);
  CHECK(r.max_energy_increase <= 1e-10 * r.initial_energy);
}

TEST(oracle_hybrid_run_error) {
  // test_analysis.cpp:147-158
  const Discretization d = build_discretization(structured_hybrid_box(2, 2, 1, 1), 2);
  SolutionState s = make_initial_state(d, standing_wave(), 0.0);
  double t = 0.0;
  const auto r = oracle::run_simulation(d, s.u, t, 0.2, 0.5, 0.0, 0.0, 2);
  CHECK(r.stable && r.max_energy_increase <= 1e-10 * r.initial_energy);
  CHECK(l2_error(d, s.u.data(), standing_wave().p, t) < 0.5);
}

TEST(l2_error_exact_and_unit) {
  const Discretization d = build_discretization(structured_wedge_box(2), 2);
  FieldFunctions poly;
  poly.p = [](double x, double y, double, double) { return 1.0 + x + 0.5 * x * y; };
  poly.ux = poly.uy = poly.uz = [](double, double, double, double) { return 0.0; };
  const SolutionState sp = make_initial_state(d, poly, 0.0);
  CHECK(l2_error(d, sp.u.data(), poly.p, 0.0) < 1e-12);
  std::vector<double> zero(d.total_dofs, 0.0);
  CHECK(std::abs(l2_error(d, zero.data(), standing_wave().p, 0.0) - 1.0) < 1e-12);
  const std::vector<double> h = {2.0, 1.0, 0.5, 0.25, 0.125};
  std::vector<double> err;
  for (double hh : h) err.push_back(0.7 * hh * hh * hh);
  CHECK(std::abs(fit_rate(h, err) - 3.0) < 1e-12);
  err[0] = 100.0;
  CHECK(std::abs(fit_rate(h, err) - 3.0) < 1e-12);
}

TEST(spectra_mesh_size) {
  const Discretization d = build_discretization(spectra_mesh(), 2);
  CHECK(d.mesh.num_wedges() == 16);
  CHECK(d.total_dofs == 1152);
}

TEST(dt_estimate_scaling_and_cfl_check) {
  // test_solver.cpp:86-98: dt doubles with the mesh, halves with c = 2; cfl < 0 throws
  const Discretization d1 = small_box(2, 2);
  HybridMesh scaled = structured_wedge_box(2);
  for (auto& v : scaled.vertices)
    for (auto& c : v) c *= 2.0;
  const Discretization d2 = build_discretization(std::move(scaled), 2, {}, QuadratureMode::exact, 1);
  CHECK_CLOSE(estimate_dt(d2, 0.5), 2.0 * estimate_dt(d1, 0.5), 1e-12);
  const Discretization d3 = build_discretization(structured_wedge_box(2, {1.0, 4.0}), 2, {}, QuadratureMode::exact, 1);
  CHECK_CLOSE(estimate_dt(d3, 0.5), 0.5 * estimate_dt(d1, 0.5), 1e-12);
  CHECK_THROWS(estimate_dt(d1, -1.0), ConfigError);
}

TEST(time_stepper_orders_scalar) {
  // test_solver.cpp:113-144: y' = lambda y, lambda = -0.4 + 1.3i, dt = 0.1, 0.05,
  // 0.025 to t = 1; order from dt halving: LSERK45 4 +- 8%, AB3 3 +- 8%
  const double lr = -0.4, li = 1.3;
  auto order_of = [&](IntegratorKind kind) {
    std::vector<double> errs;
    for (const double dt : {0.1, 0.05, 0.025}) {
      std::vector<double> y = {1.0, 0.0};
      double t = 0.0;
      TimeStepper st(kind, 2);
      const RhsFn rhs = [&](const std::vector<double>& u, std::vector<double>& out, double) {
        out.resize(2);
        out[0] = lr * u[0] - li * u[1];
        out[1] = li * u[0] + lr * u[1];
      };
      const int steps = (int)std::lround(1.0 / dt);
      for (int i = 0; i < steps; ++i) st.step(y, t, dt, rhs, nullptr);
      const double er = std::exp(lr) * std::cos(li), ei = std::exp(lr) * std::sin(li);
      errs.push_back(std::hypot(y[0] - er, y[1] - ei));
    }
    return std::log2(errs[0] / errs[2]) / 2.0;
  };
  const double o4 = order_of(IntegratorKind::lserk4), o3 = order_of(IntegratorKind::ab3);
  std::printf("    lserk4 order %.3f, ab3 order %.3f\n", o4, o3);
  CHECK(std::abs(o4 - 4.0) <= 0.32);
  CHECK(std::abs(o3 - 3.0) <= 0.24);
}

TEST(oracle_zero_rhs_fixes_state) {
  // test_solver.cpp:113-122: a zero state stays exactly zero through a step
  const Discretization d = small_box(1, 1);
  std::vector<double> u(d.total_dofs, 0.0);
  oracle::lserk_steps(d, u.data(), u.size(), 0.01, 1, 1, false);
  for (double v : u) CHECK(v == 0.0);
}

int main(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int ran = 0;
  for (const auto& c : registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    g_case = c.name;
    const int before = g_fail;
    c.fn();
    ++ran;
    std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", c.name);
    std::fflush(stdout);
  }
  std::printf("%d cases, %d checks, %d failures\n", ran, g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
