#pragma once
// Hybrid wedge/tet meshes, generators and face connectivity (host setup).
// Restates proj/include/prismdg/mesh.hpp:14-123.  Element ids enumerate wedges
// first, then tets (mesh.hpp:25,36).  Generators reproduce the reference's
// vertex / element numbering and RNG draw order exactly, so meshes are
// bit-identical with the reference for the same parameters.
//
// Connectivity is stored flat (one FaceConn per element face plus a table of
// distinct node permutations) instead of one std::vector per face; the
// permutation content is bit-identical with the reference's greedy matcher
// (mesh.cpp:398-481).

#include "prismdg/basis.hpp"
#include "prismdg/geometry.hpp"

#include <array>
#include <cmath>
#include <cstdint>
#include <map>
#include <string>
#include <utility>
#include <vector>

namespace prismdg {

constexpr int kReflectiveTag = 1; // mesh.hpp:14

struct Media {
  double rho = 1.0;
  double kappa = 1.0;
  double wavespeed() const { return std::sqrt(kappa / rho); }
};

struct HybridMesh {
  std::vector<Vert3> vertices;
  std::vector<std::array<int, 6>> wedges;
  std::vector<std::array<int, 4>> tets;
  std::vector<Media> media; // per element
  std::map<std::pair<int, int>, int> boundary_tags;

  int num_wedges() const { return (int)wedges.size(); }
  int num_tets() const { return (int)tets.size(); }
  int num_elements() const { return num_wedges() + num_tets(); }
  ElemKind kind(int e) const { return e < num_wedges() ? ElemKind::wedge : ElemKind::tet; }
  int num_faces(int e) const { return kind(e) == ElemKind::wedge ? 5 : 4; }
  WedgeVerts wedge_verts(int w) const;
  TetVerts tet_verts(int t) const;
};

struct SurfaceTriangulation {
  std::vector<std::array<double, 2>> vertices;
  std::vector<double> z_bottom, z_top;
  std::vector<std::array<int, 3>> triangles;
};

struct LayerSpec {
  std::vector<double> z_bottom, z_top;
  int sublayers = 1;
  Media media;
};

bool is_vertically_mapped(const WedgeVerts& v);
HybridMesh extrude_layer(const SurfaceTriangulation& surface, int layers, Media media = {});
HybridMesh stack_layers(const std::vector<std::array<double, 2>>& xy,
                        const std::vector<std::array<int, 3>>& triangles,
                        const std::vector<LayerSpec>& layers);
HybridMesh structured_hybrid_box(int nx, int ny, int nz_wedge, int nz_tet, Media wedge_media = {},
                                 Media tet_media = {});
HybridMesh structured_wedge_box(int n, Media media = {});
HybridMesh unstructured_wedge_box(int n, double xy_jitter, double z_amplitude, std::uint64_t seed,
                                  Media media = {});
HybridMesh perturb_vertically(const HybridMesh& mesh, double amplitude, std::uint64_t seed);
HybridMesh arnold_wedge_box(int n, double delta, Media media = {});

/// Structured (n x n) surface grid of [-1,1]^2 split into 2n^2 triangles, the
/// pattern of config.cpp:232-243 ("layers" mesh kind).
void structured_surface(int n, std::vector<std::array<double, 2>>& xy,
                        std::vector<std::array<int, 3>>& tris);
/// Surface functions of config.cpp:152-178: "flat:z0" or "sine:z0:amp:kx:ky".
double eval_surface_function(const std::string& spec, double x, double y);

struct FaceConn {
  int nbr = -1;      // neighbour element, -1 on the boundary
  int nbr_face = -1;
  int tag = kReflectiveTag;
  int perm_id = -1;  // index into Connectivity::perms (-1 on the boundary)
};

struct Connectivity {
  std::vector<FaceConn> faces;        // element e, face f at face_offset[e] + f
  std::vector<std::int64_t> face_offset; // size ne+1
  std::vector<std::vector<int>> perms;   // distinct node permutations
  int num_interior_pairs = 0;
  int num_boundary_faces = 0;
  const FaceConn& at(int e, int f) const { return faces[face_offset[e] + f]; }
  /// my face node i <-> neighbour face node perm(e,f)[i] (reference FaceConn::perm)
  const std::vector<int>& perm(int e, int f) const { return perms[at(e, f).perm_id]; }
};

std::vector<int> face_vertex_ids(const HybridMesh& mesh, int e, int f);
std::vector<Vert3> face_node_coords(const HybridMesh& mesh, const References& refs, int e, int f);
Connectivity build_connectivity(const HybridMesh& mesh, const References& refs);
void validate_mesh(const HybridMesh& mesh);
double mesh_volume(const HybridMesh& mesh);

HybridMesh load_mesh(const std::string& path);
void save_mesh(const HybridMesh& mesh, const std::string& path);
SurfaceTriangulation load_surface(const std::string& path);

} // namespace prismdg
