#pragma once
// Geometric factors of one element, computed once at setup and then either
// flattened into the device tables (context.cu) or used by host analysis.
//
// Vertically mapped wedges get the closed forms of the paper's Lemma 1: the
// (x, y) part of the map is affine on the triangle, so rx, ry, sx, sy are
// constants, J is linear in (r, s), and only z varies along t, which leaves
// t_x J, t_y J as per-slice vectors and t_z J as a constant.  Tets are affine.
// Field names follow proj/include/prismdg/geometry.hpp:11-55 so the
// reference's callers read the same members.

#include "prismdg/basis.hpp"

#include <array>
#include <vector>

namespace prismdg {

using Vert3 = std::array<double, 3>;
using WedgeVerts = std::array<Vert3, 6>; // bottom triangle, then top triangle
using TetVerts = std::array<Vert3, 4>;

/// one element face: outward unit normal and surface Jacobian
struct FaceGeometry {
  Vert3 normal{};
  double area = 0.0;
  double jf = 0.0; // triangles: area / 2 (reference-triangle area 2)
  Vec jf_edge;     // quads: J_f at the N+1 GLL nodes along t; jf = their mean
};

struct ElementGeometry {
  ElemKind kind = ElemKind::wedge;
  int nverts = 0;
  std::array<Vert3, 6> verts{};

  // --- constants of the affine (x, y) map (wedges and tets)
  double rx = 0, ry = 0, sx = 0, sy = 0;
  // --- J(r, s) = j0 + j_r r + j_s s on wedges; the constant J of a tet in j0
  double j0 = 0, j_r = 0, j_s = 0;
  Vec j_tri; // J at the triangle nodes
  // --- vertical factors of a wedge
  double tzJ = 0;
  Vec txJ, tyJ; // per GLL slice
  // --- remaining tet factors
  double rz = 0, sz = 0, tx = 0, ty = 0, tz = 0;

  std::vector<FaceGeometry> faces;
  double volume = 0, surface_area = 0, diameter = 0;

  auto jacobian_at(double r, double s) const -> double { return j0 + j_r * r + j_s * s; }
};

auto wedge_geometry(const WedgeVerts& v, const References& refs) -> ElementGeometry;
auto tet_geometry(const TetVerts& v) -> ElementGeometry;
/// reference coordinates -> physical point
auto wedge_map(const WedgeVerts& v, double r, double s, double t) -> Vert3;
auto tet_map(const TetVerts& v, double r, double s, double t) -> Vert3;
/// full 3x3 Jacobian determinant of the wedge map (validation of vertical mapping)
auto wedge_jacobian_det(const WedgeVerts& v, double r, double s, double t) -> double;

} // namespace prismdg
