#pragma once
// The fixed-over-a-run discretization (host setup).
//
// Mirrors prismdg::Discretization / build_discretization of the reference
// (proj/include/prismdg/solver.hpp:29-63, proj/src/solver.cpp:56-156): same state
// layout (element-major, [p|ux|uy|uz] per element, wedge node i*(N+1)+j), same
// elem_offset / total_dofs, same face maps and penalties.  Storage is flat so
// that 1e6-element meshes fit: per-element operators live in contiguous arrays
// (L^{tri,k} column-major per wedge), face tables are indexed through
// Connectivity::face_offset, and node coordinates are evaluated on demand.

#include "prismdg/geometry.hpp"
#include "prismdg/mesh.hpp"
#include "prismdg/operators.hpp"

#include <array>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <vector>

struct pdg_disc_arrays; // include/prismdg_b200.h

namespace prismdg {

enum class FluxMode { upwind = 0, central = 1, custom = 2 };

struct FluxConfig {
  FluxMode mode = FluxMode::upwind;
  double tau_p = 0.0, tau_u = 0.0; // custom only, >= 0
};

/// Mass treatment.  exact / lumped are the reference's QuadratureMode
/// (operators.hpp:17); wadg is the weight-adjusted extension of the north star.
enum class MassMode { exact = 0, lumped = 1, wadg = 2 };

struct WedgeGeo {
  double rx, ry, sx, sy, tzJ;
  double j0, jr, js;       // J = j0 + jr r + js s
  double jf_bottom, jf_top;
  double jf_quad[3][2];    // quad-face J_f at the two edge ends
  double volume, surface_area;
};

struct TetGeo {
  double rx, ry, rz, sx, sy, sz, tx, ty, tz;
  double J;
  double lift_scale[4];    // J_f / J
  double volume, surface_area;
};

struct FacePhys {
  double normal[3];
  double tau_p, tau_u;
};

struct DeviceHandle; // owned device context of the host shim (solver_api.cpp)

struct Discretization {
  HybridMesh mesh;
  References refs;
  Connectivity conn;
  QuadratureMode qmode = QuadratureMode::exact;
  MassMode mass_mode = MassMode::exact;
  FluxConfig flux;
  int threads = 1;

  int degree = 0, nq = 0, nt = 0, np_wedge = 0, np_tet = 0;

  std::vector<std::size_t> elem_offset; // ne+1
  std::size_t total_dofs = 0;
  std::vector<std::size_t> node_offset; // ne+1
  std::size_t total_nodes = 0;

  std::vector<WedgeGeo> wgeo;     // per wedge
  std::vector<double> txJ, tyJ;   // per wedge, nq each
  std::vector<double> tri_lift;   // per wedge nt*nt, [k*nt + i] = L(i,k)
  std::vector<double> quad_lift;  // per wedge 3*nq*nt, [(e*nq + a)*nt + i] = QL_e(i,a)
  std::vector<TetGeo> tgeo;       // per tet
  std::vector<FacePhys> fphys;    // per element face, indexed like conn.faces

  std::shared_ptr<DeviceHandle> device; // lazily created by the host shim

  int num_elements() const { return mesh.num_elements(); }
  int np(int e) const { return mesh.kind(e) == ElemKind::wedge ? np_wedge : np_tet; }
  const std::vector<int>& my_nodes(int e, int f) const {
    return mesh.kind(e) == ElemKind::wedge ? refs.wedge.face_nodes[f] : refs.tet.face_nodes[f];
  }
  /// neighbour local volume node aligned with my face node i (solver.cpp:129-134)
  int nbr_node(int e, int f, int i) const {
    const FaceConn& fc = conn.at(e, f);
    const auto& lst = mesh.kind(fc.nbr) == ElemKind::wedge ? refs.wedge.face_nodes[fc.nbr_face]
                                                           : refs.tet.face_nodes[fc.nbr_face];
    return lst[conn.perms[fc.perm_id][i]];
  }
  /// physical coordinates of local node n of element e (solver.cpp:95-114)
  Vert3 node_xyz(int e, int n) const;
  ElementGeometry geometry(int e) const;
  WedgeOperators wedge_operators(int w) const;
  TetOperators tet_operators(int t) const;
};

/// solver.cpp:56-156.  `with_quad_lift` = false skips the quad-lift storage
/// (the device path can rebuild it from L); the CPU oracle needs it.
Discretization build_discretization(HybridMesh mesh, int degree, FluxConfig flux = {},
                                    QuadratureMode qmode = QuadratureMode::exact, int threads = 1,
                                    MassMode mass_mode = MassMode::exact, bool with_quad_lift = true);

/// A Discretization from a caller's flattened arrays (pdg_disc_arrays,
/// include/prismdg_b200.h; csrc/host/disc_ingest.cpp)
Discretization discretization_from_arrays(const ::pdg_disc_arrays& a);

} // namespace prismdg
