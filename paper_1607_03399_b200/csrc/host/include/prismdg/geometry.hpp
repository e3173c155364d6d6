#pragma once
// Per-element geometric factors (host setup).
// Restates proj/include/prismdg/geometry.hpp:11-55: Lemma-1 closed forms for
// vertically mapped wedges and affine tetrahedra.

#include "prismdg/basis.hpp"

#include <array>
#include <vector>

namespace prismdg {

using Vert3 = std::array<double, 3>;
using WedgeVerts = std::array<Vert3, 6>;
using TetVerts = std::array<Vert3, 4>;

struct FaceGeometry {
  Vert3 normal{};  // unit outward normal (planar faces)
  double jf = 0.0; // tri / tet faces: area/2; quad faces: mean of jf_edge
  Vec jf_edge;     // quad faces: J_f at the N+1 GLL edge nodes
  double area = 0.0;
};

struct ElementGeometry {
  ElemKind kind = ElemKind::wedge;
  // wedge factors (geometry.cpp:64-118)
  double rx = 0, ry = 0, sx = 0, sy = 0, tzJ = 0;
  Vec txJ, tyJ;                    // at GLL t nodes
  double j0 = 0, j_r = 0, j_s = 0; // J(r,s) = j0 + j_r r + j_s s (tets: J in j0)
  Vec j_tri;
  // tet-only factors
  double rz = 0, sz = 0, tx = 0, ty = 0, tz = 0;
  std::vector<FaceGeometry> faces;
  double volume = 0, surface_area = 0, diameter = 0;
  int nverts = 0;
  std::array<Vert3, 6> verts{};
  double jacobian_at(double r, double s) const { return j0 + j_r * r + j_s * s; }
};

ElementGeometry wedge_geometry(const WedgeVerts& v, const References& refs);
ElementGeometry tet_geometry(const TetVerts& v);
Vert3 wedge_map(const WedgeVerts& v, double r, double s, double t);
Vert3 tet_map(const TetVerts& v, double r, double s, double t);
double wedge_jacobian_det(const WedgeVerts& v, double r, double s, double t);

} // namespace prismdg
