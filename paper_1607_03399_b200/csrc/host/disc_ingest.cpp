// pdg_disc_from_arrays: a Discretization assembled from a caller's arrays --
// the reference's own Discretization (proj/include/prismdg/solver.hpp:29-59)
// flattened member by member (mesh, geom, wedge_ops, tet_ops, face_data), so
// the device path can run on operators built by the reference's Eigen setup
// (proj/src/solver.cpp:56-156, operators.cpp:10-66) instead of ours.
//
// Only the shared References (reference.hpp:13-112) are rebuilt from the
// degree; the caller's face-node lists are checked against them.  The
// connectivity (Connectivity::perms, mesh.hpp:94-107) is recovered from the
// caller's nbr_nodes: each face's neighbour nodes must be a permutation of one
// face-node list of the neighbour.
#include <algorithm>
#include <cmath>
#include <map>
#include <string>

#include "prismdg/discretization.hpp"
#include "prismdg_b200.h"

namespace prismdg {

Discretization discretization_from_arrays(const pdg_disc_arrays& a) {
  auto need = [](const void* p, const char* what) {
    if (!p) throw ConfigError(std::string("pdg_disc_arrays: missing ") + what);
  };
  if (a.degree < 1 || a.degree > 9) throw ConfigError("pdg_disc_arrays: degree out of range");
  if (a.qmode < 0 || a.qmode > 2) throw ConfigError("pdg_disc_arrays: unknown quadrature / mass mode");
  if (a.num_vertices < 0 || a.num_wedges < 0 || a.num_tets < 0 || a.num_wedges + a.num_tets <= 0)
    throw ConfigError("pdg_disc_arrays: bad element counts");
  const bool wadg = a.qmode == 2;
  need(a.vertices, "vertices");
  need(a.media, "media");
  need(a.face_nbr, "face_nbr");
  need(a.face_tau, "face_tau");
  need(a.face_normal, "face_normal");
  need(a.face_nbr_nodes, "face_nbr_nodes");
  if (a.num_wedges > 0) {
    need(a.wedges, "wedges");
    need(a.wedge_geom, "wedge_geom");
    need(a.txJ, "txJ");
    need(a.tyJ, "tyJ");
    need(a.wedge_scalars, "wedge_scalars");
    if (!wadg) {
      need(a.tri_lift, "tri_lift");
      need(a.quad_lift, "quad_lift");
    }
  }
  if (a.num_tets > 0) {
    need(a.tets, "tets");
    need(a.tet_geom, "tet_geom");
    need(a.tet_scalars, "tet_scalars");
  }

  Discretization d;
  // ---- mesh (mesh.hpp:35-49), validated like load_mesh ------------------------
  const long long nv = a.num_vertices, nw = a.num_wedges, ntet = a.num_tets, ne = nw + ntet;
  d.mesh.vertices.resize(nv);
  for (long long v = 0; v < nv; ++v)
    d.mesh.vertices[v] = {a.vertices[3 * v], a.vertices[3 * v + 1], a.vertices[3 * v + 2]};
  d.mesh.wedges.resize(nw);
  for (long long w = 0; w < nw; ++w)
    for (int q = 0; q < 6; ++q) d.mesh.wedges[w][q] = a.wedges[6 * w + q];
  d.mesh.tets.resize(ntet);
  for (long long t = 0; t < ntet; ++t)
    for (int q = 0; q < 4; ++q) d.mesh.tets[t][q] = a.tets[4 * t + q];
  d.mesh.media.resize(ne);
  for (long long e = 0; e < ne; ++e) {
    d.mesh.media[e] = Media{a.media[2 * e], a.media[2 * e + 1]};
    if (!(d.mesh.media[e].rho > 0.0 && d.mesh.media[e].kappa > 0.0))
      throw MeshError("element " + std::to_string(e + 1) + ": media must be positive");
  }
  validate_mesh(d.mesh);

  // ---- shared reference data, sizes -------------------------------------------
  const int N = a.degree;
  d.refs = build_references(N);
  d.degree = N;
  d.nq = N + 1;
  d.nt = d.refs.tri.num_nodes;
  d.np_wedge = d.refs.wedge.num_nodes;
  d.np_tet = d.refs.tet.num_nodes;
  d.qmode = a.qmode == 1 ? QuadratureMode::lumped : QuadratureMode::exact;
  d.mass_mode = a.qmode == 1 ? MassMode::lumped : (wadg ? MassMode::wadg : MassMode::exact);
  d.flux.mode = static_cast<FluxMode>(std::clamp(a.flux_mode, 0, 2));
  d.flux.tau_p = a.tau_p;
  d.flux.tau_u = a.tau_u;
  const int nq = d.nq, nt = d.nt;

  // ---- geometry and per-element operators --------------------------------------
  d.wgeo.resize(nw);
  d.txJ.assign(a.txJ ? a.txJ : nullptr, a.txJ ? a.txJ + nw * nq : nullptr);
  d.tyJ.assign(a.tyJ ? a.tyJ : nullptr, a.tyJ ? a.tyJ + nw * nq : nullptr);
  for (long long w = 0; w < nw; ++w) {
    const double* s = a.wedge_scalars + 7 * w;
    const double* g = a.wedge_geom + 11 * w;
    WedgeGeo& o = d.wgeo[w];
    o.tzJ = s[0];
    o.rx = s[1];
    o.ry = s[2];
    o.sx = s[3];
    o.sy = s[4];
    o.jf_bottom = s[5];
    o.jf_top = s[6];
    o.j0 = g[0];
    o.jr = g[1];
    o.js = g[2];
    o.volume = g[3];
    o.surface_area = g[4];
    for (int e = 0; e < 3; ++e) {
      o.jf_quad[e][0] = g[5 + 2 * e];
      o.jf_quad[e][1] = g[6 + 2 * e];
    }
    // J affine in (r, s): positive at the three triangle vertices = positive everywhere
    if (!(o.j0 - o.jr - o.js > 0.0 && o.j0 + o.jr - o.js > 0.0 && o.j0 - o.jr + o.js > 0.0))
      throw MeshError("wedge " + std::to_string(w + 1) + ": Jacobian is not positive");
  }
  if (a.tri_lift) d.tri_lift.assign(a.tri_lift, a.tri_lift + (std::size_t)nw * nt * nt);
  if (a.quad_lift) d.quad_lift.assign(a.quad_lift, a.quad_lift + (std::size_t)nw * 3 * nq * nt);
  d.tgeo.resize(ntet);
  for (long long t = 0; t < ntet; ++t) {
    const double* s = a.tet_scalars + 13 * t;
    const double* g = a.tet_geom + 3 * t;
    TetGeo& o = d.tgeo[t];
    o.rx = s[0];
    o.ry = s[1];
    o.rz = s[2];
    o.sx = s[3];
    o.sy = s[4];
    o.sz = s[5];
    o.tx = s[6];
    o.ty = s[7];
    o.tz = s[8];
    for (int f = 0; f < 4; ++f) o.lift_scale[f] = s[9 + f];
    o.J = g[0];
    o.volume = g[1];
    o.surface_area = g[2];
    if (!(o.J > 0.0)) throw MeshError("tet " + std::to_string(t + 1) + ": Jacobian is not positive");
  }
  d.elem_offset.resize(ne + 1);
  d.node_offset.resize(ne + 1);
  d.elem_offset[0] = d.node_offset[0] = 0;
  for (long long e = 0; e < ne; ++e) {
    d.elem_offset[e + 1] = d.elem_offset[e] + 4u * d.np((int)e);
    d.node_offset[e + 1] = d.node_offset[e] + d.np((int)e);
  }
  d.total_dofs = d.elem_offset[ne];
  d.total_nodes = d.node_offset[ne];

  // ---- faces: connectivity recovered from the neighbour node maps ---------------
  const int max_nfp = std::max(nq * nq, nt);
  d.conn.face_offset.resize(ne + 1);
  d.conn.face_offset[0] = 0;
  for (long long e = 0; e < ne; ++e) d.conn.face_offset[e + 1] = d.conn.face_offset[e] + d.mesh.num_faces((int)e);
  const std::size_t nfaces = (std::size_t)d.conn.face_offset[ne];
  d.conn.faces.assign(nfaces, FaceConn{});
  d.fphys.resize(nfaces);
  std::map<std::vector<int>, int> perm_id;
  for (long long e = 0; e < ne; ++e) {
    const bool wedge = d.mesh.kind((int)e) == ElemKind::wedge;
    for (int f = 0; f < d.mesh.num_faces((int)e); ++f) {
      const std::size_t q = (std::size_t)d.conn.face_offset[e] + f;
      const auto& my = wedge ? d.refs.wedge.face_nodes[f] : d.refs.tet.face_nodes[f];
      const int nfp = (int)my.size();
      if (a.face_my_nodes)
        for (int i = 0; i < nfp; ++i)
          if (a.face_my_nodes[q * max_nfp + i] != my[i])
            throw ConfigError("element " + std::to_string(e + 1) + " face " + std::to_string(f) +
                              ": face-node list differs from the reference construction");
      FacePhys& fp = d.fphys[q];
      for (int c = 0; c < 3; ++c) fp.normal[c] = a.face_normal[3 * q + c];
      fp.tau_p = a.face_tau[2 * q];
      fp.tau_u = a.face_tau[2 * q + 1];
      if (!(fp.tau_p >= 0.0 && fp.tau_u >= 0.0)) throw ConfigError("flux penalties must be non-negative");
      FaceConn& fc = d.conn.faces[q];
      const int nb = a.face_nbr[q];
      if (nb < 0) {
        ++d.conn.num_boundary_faces;
        continue;
      }
      if (nb >= ne || nb == e) throw MeshError("face neighbour out of range");
      const int* nbn = a.face_nbr_nodes + q * max_nfp;
      const bool nwedge = d.mesh.kind(nb) == ElemKind::wedge;
      int found = -1;
      std::vector<int> perm(nfp);
      for (int g = 0; g < d.mesh.num_faces(nb) && found < 0; ++g) {
        const auto& lst = nwedge ? d.refs.wedge.face_nodes[g] : d.refs.tet.face_nodes[g];
        if ((int)lst.size() != nfp) continue;
        bool ok = true;
        for (int i = 0; i < nfp && ok; ++i) {
          const auto it = std::find(lst.begin(), lst.end(), nbn[i]);
          ok = it != lst.end();
          if (ok) perm[i] = (int)(it - lst.begin());
        }
        if (ok) {
          std::vector<int> sorted(perm);
          std::sort(sorted.begin(), sorted.end());
          for (int i = 0; i < nfp && ok; ++i) ok = sorted[i] == i;
        }
        if (ok) found = g;
      }
      if (found < 0)
        throw MeshError("element " + std::to_string(e + 1) + " face " + std::to_string(f) +
                        ": nbr_nodes do not map onto a face of element " + std::to_string(nb + 1));
      fc.nbr = nb;
      fc.nbr_face = found;
      auto ins = perm_id.emplace(perm, (int)d.conn.perms.size());
      if (ins.second) d.conn.perms.push_back(perm);
      fc.perm_id = ins.first->second;
      if (e < nb) ++d.conn.num_interior_pairs;
    }
  }
  // the pairing must be symmetric (both sides name each other)
  for (long long e = 0; e < ne; ++e)
    for (int f = 0; f < d.mesh.num_faces((int)e); ++f) {
      const FaceConn& fc = d.conn.at((int)e, f);
      if (fc.nbr >= 0 && d.conn.at(fc.nbr, fc.nbr_face).nbr != e)
        throw MeshError("face pairing is not symmetric at element " + std::to_string(e + 1));
    }
  return d;
}

} // namespace prismdg
