// build_discretization: geometry, reduced-storage operators, offsets and face
// penalties, flattened for large meshes.  Follows proj/src/solver.cpp:56-156.
#include "prismdg/discretization.hpp"

#include <algorithm>
#include <cmath>
#include <string>

namespace prismdg {

namespace {

double impedance(const Media& m) { return m.rho * m.wavespeed(); }

} // namespace

Vert3 Discretization::node_xyz(int e, int n) const {
  if (mesh.kind(e) == ElemKind::wedge)
    return wedge_map(mesh.wedge_verts(e), refs.wedge.r[n], refs.wedge.s[n], refs.wedge.t[n]);
  return tet_map(mesh.tet_verts(e - mesh.num_wedges()), refs.tet.r[n], refs.tet.s[n], refs.tet.t[n]);
}

ElementGeometry Discretization::geometry(int e) const {
  if (mesh.kind(e) == ElemKind::wedge) return wedge_geometry(mesh.wedge_verts(e), refs);
  return tet_geometry(mesh.tet_verts(e - mesh.num_wedges()));
}

WedgeOperators Discretization::wedge_operators(int w) const {
  WedgeOperators ops;
  const WedgeGeo& g = wgeo[w];
  ops.rx = g.rx;
  ops.ry = g.ry;
  ops.sx = g.sx;
  ops.sy = g.sy;
  ops.tzJ = g.tzJ;
  ops.jf_bottom = g.jf_bottom;
  ops.jf_top = g.jf_top;
  ops.txJ.assign(txJ.begin() + (std::size_t)w * nq, txJ.begin() + (std::size_t)(w + 1) * nq);
  ops.tyJ.assign(tyJ.begin() + (std::size_t)w * nq, tyJ.begin() + (std::size_t)(w + 1) * nq);
  ops.tri_lift = Mat(nt, nt);
  const double* L = tri_lift.data() + (std::size_t)w * nt * nt;
  for (int k = 0; k < nt; ++k)
    for (int i = 0; i < nt; ++i) ops.tri_lift(i, k) = L[k * nt + i];
  if (!quad_lift.empty()) {
    const double* Q = quad_lift.data() + (std::size_t)w * 3 * nq * nt;
    for (int e = 0; e < 3; ++e) {
      ops.quad_lift[e] = Mat(nt, nq);
      for (int a = 0; a < nq; ++a)
        for (int i = 0; i < nt; ++i) ops.quad_lift[e](i, a) = Q[(e * nq + a) * nt + i];
    }
  }
  return ops;
}

TetOperators Discretization::tet_operators(int t) const {
  const TetGeo& g = tgeo[t];
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
  for (int f = 0; f < 4; ++f) ops.lift_scale[f] = g.lift_scale[f];
  return ops;
}

Discretization build_discretization(HybridMesh mesh, int degree, FluxConfig flux,
                                    QuadratureMode qmode, int threads, MassMode mass_mode,
                                    bool with_quad_lift) {
  if (flux.mode == FluxMode::custom && (flux.tau_p < 0.0 || flux.tau_u < 0.0))
    throw ConfigError("flux penalties must be non-negative");
  if (mass_mode == MassMode::lumped) qmode = QuadratureMode::lumped;
  if (qmode == QuadratureMode::lumped && mass_mode == MassMode::exact) mass_mode = MassMode::lumped;
  Discretization d;
  d.mesh = std::move(mesh);
  d.refs = build_references(degree);
  d.conn = build_connectivity(d.mesh, d.refs);
  d.qmode = qmode;
  d.mass_mode = mass_mode;
  d.flux = flux;
  d.threads = std::max(1, threads);
  d.degree = degree;
  d.nq = degree + 1;
  d.nt = d.refs.tri.num_nodes;
  d.np_wedge = d.refs.wedge.num_nodes;
  d.np_tet = d.refs.tet.num_nodes;

  const int nw = d.mesh.num_wedges(), ntet = d.mesh.num_tets(), ne = d.mesh.num_elements();
  const int nq = d.nq, nt = d.nt;
  d.wgeo.resize(nw);
  d.txJ.resize((std::size_t)nw * nq);
  d.tyJ.resize((std::size_t)nw * nq);
  // WADG needs no per-wedge operator storage; the stored lifts are kept only
  // when asked for (the CPU oracle restates WADG through the exact lifts)
  const bool need_L = mass_mode != MassMode::wadg || with_quad_lift;
  if (need_L) d.tri_lift.resize((std::size_t)nw * nt * nt);
  if (with_quad_lift) d.quad_lift.resize((std::size_t)nw * 3 * nq * nt);
  d.tgeo.resize(ntet);

  int bad_wedge = -1;
  std::string geo_error;
#pragma omp parallel for schedule(dynamic, 64)
  for (int w = 0; w < nw; ++w) {
    try {
      const ElementGeometry g = wedge_geometry(d.mesh.wedge_verts(w), d.refs);
      WedgeGeo& o = d.wgeo[w];
      o.rx = g.rx;
      o.ry = g.ry;
      o.sx = g.sx;
      o.sy = g.sy;
      o.tzJ = g.tzJ;
      o.j0 = g.j0;
      o.jr = g.j_r;
      o.js = g.j_s;
      o.jf_bottom = g.faces[0].jf;
      o.jf_top = g.faces[1].jf;
      for (int e = 0; e < 3; ++e) {
        o.jf_quad[e][0] = g.faces[2 + e].jf_edge[0];
        o.jf_quad[e][1] = g.faces[2 + e].jf_edge[nq - 1];
      }
      o.volume = g.volume;
      o.surface_area = g.surface_area;
      for (int j = 0; j < nq; ++j) {
        d.txJ[(std::size_t)w * nq + j] = g.txJ[j];
        d.tyJ[(std::size_t)w * nq + j] = g.tyJ[j];
      }
      if (need_L) {
        if (!wedge_lifts_flat(g.j0, g.j_r, g.j_s, o.jf_quad, d.refs,
                              d.tri_lift.data() + (std::size_t)w * nt * nt,
                              with_quad_lift ? d.quad_lift.data() + (std::size_t)w * 3 * nq * nt : nullptr))
          throw NumericalError("weighted triangle mass matrix is not SPD");
      } else if (!(g.j0 - g.j_r - g.j_s > 0.0 && g.j0 + g.j_r - g.j_s > 0.0 && g.j0 - g.j_r + g.j_s > 0.0)) {
        // J is affine in (r, s): positive at the triangle vertices (-1,-1),
        // (1,-1), (-1,1) means positive everywhere, so M_{1/J} is SPD
        throw NumericalError("wedge Jacobian is not positive");
      }
    } catch (const std::exception& ex) {
#pragma omp critical
      if (bad_wedge < 0 || w < bad_wedge) {
        bad_wedge = w;
        geo_error = ex.what();
      }
    }
  }
  if (bad_wedge >= 0) {
    if (geo_error.find("SPD") != std::string::npos) throw NumericalError(geo_error);
    throw MeshError("wedge " + std::to_string(bad_wedge + 1) + ": " + geo_error);
  }
  for (int t = 0; t < ntet; ++t) {
    const ElementGeometry g = tet_geometry(d.mesh.tet_verts(t));
    TetGeo& o = d.tgeo[t];
    o.rx = g.rx;
    o.ry = g.ry;
    o.rz = g.rz;
    o.sx = g.sx;
    o.sy = g.sy;
    o.sz = g.sz;
    o.tx = g.tx;
    o.ty = g.ty;
    o.tz = g.tz;
    o.J = g.j0;
    for (int f = 0; f < 4; ++f) o.lift_scale[f] = g.faces[f].jf / g.j0;
    o.volume = g.volume;
    o.surface_area = g.surface_area;
  }

  d.elem_offset.resize(ne + 1);
  d.node_offset.resize(ne + 1);
  d.elem_offset[0] = d.node_offset[0] = 0;
  for (int e = 0; e < ne; ++e) {
    d.elem_offset[e + 1] = d.elem_offset[e] + 4u * d.np(e);
    d.node_offset[e + 1] = d.node_offset[e] + d.np(e);
  }
  d.total_dofs = d.elem_offset[ne];
  d.total_nodes = d.node_offset[ne];

  // face normals and penalties (solver.cpp:116-154)
  d.fphys.resize(d.conn.faces.size());
#pragma omp parallel for schedule(dynamic, 256)
  for (int e = 0; e < ne; ++e) {
    const bool wedge = d.mesh.kind(e) == ElemKind::wedge;
    Vert3 normals[5];
    if (wedge) {
      // normals straight from the wedge closed forms (geometry.cpp:124-150)
      const ElementGeometry g = wedge_geometry(d.mesh.wedge_verts(e), d.refs);
      for (int f = 0; f < 5; ++f) normals[f] = g.faces[f].normal;
    } else {
      const ElementGeometry g = tet_geometry(d.mesh.tet_verts(e - nw));
      for (int f = 0; f < 4; ++f) normals[f] = g.faces[f].normal;
    }
    for (int f = 0; f < d.mesh.num_faces(e); ++f) {
      const FaceConn& fc = d.conn.at(e, f);
      FacePhys& fp = d.fphys[d.conn.face_offset[e] + f];
      for (int c = 0; c < 3; ++c) fp.normal[c] = normals[f][c];
      const double z = fc.nbr >= 0 ? 0.5 * (impedance(d.mesh.media[e]) + impedance(d.mesh.media[fc.nbr]))
                                   : impedance(d.mesh.media[e]);
      switch (d.flux.mode) {
        case FluxMode::upwind:
          fp.tau_p = 1.0 / z;
          fp.tau_u = z;
          break;
        case FluxMode::central:
          fp.tau_p = 0.0;
          fp.tau_u = 0.0;
          break;
        case FluxMode::custom:
          fp.tau_p = d.flux.tau_p;
          fp.tau_u = d.flux.tau_u;
          break;
      }
    }
  }
  return d;
}

} // namespace prismdg
