#pragma once
// Hybrid wedge/tet meshes: container, generators, validation, file I/O and the
// face connectivity the device path is built from.
//
// Same public names as the reference's mesh API (proj/include/prismdg/mesh.hpp)
// so callers port unchanged; element ids enumerate wedges first, then tets.
// The generators reproduce the reference's vertex and element numbering and
// its RNG draw order, so meshes are bit-identical for equal parameters.
// Connectivity is stored flat (one FaceConn per element face and a table of
// the distinct node permutations) rather than one vector per face; the
// permutations equal the reference's greedy matcher's node for node.

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

/// boundary tag of every generated boundary face (reflecting wall)
constexpr int kReflectiveTag = 1;

/// acoustic medium of one element; c = sqrt(kappa / rho)
struct Media {
  double rho = 1.0, kappa = 1.0;
  auto wavespeed() const -> double { return std::sqrt(kappa / rho); }
};

struct HybridMesh {
  std::vector<Vert3> vertices;
  std::vector<std::array<int, 6>> wedges; // v0 v1 v2 bottom, v3 v4 v5 top
  std::vector<std::array<int, 4>> tets;
  std::vector<Media> media;                          // indexed by element id
  std::map<std::pair<int, int>, int> boundary_tags;  // (element, face) -> tag

  auto num_wedges() const -> int { return static_cast<int>(wedges.size()); }
  auto num_tets() const -> int { return static_cast<int>(tets.size()); }
  auto num_elements() const -> int { return num_wedges() + num_tets(); }
  auto kind(int e) const -> ElemKind { return e < num_wedges() ? ElemKind::wedge : ElemKind::tet; }
  auto num_faces(int e) const -> int { return kind(e) == ElemKind::wedge ? 5 : 4; }
  auto wedge_verts(int w) const -> WedgeVerts;
  auto tet_verts(int t) const -> TetVerts;
};

/// a triangulated surface with bottom/top heights per vertex (one layer)
struct SurfaceTriangulation {
  std::vector<std::array<double, 2>> vertices;
  std::vector<double> z_bottom, z_top;
  std::vector<std::array<int, 3>> triangles;
};

/// one material layer of a stacked mesh: heights per surface vertex
struct LayerSpec {
  std::vector<double> z_bottom, z_top;
  int sublayers = 1;
  Media media;
};

// ---- generators --------------------------------------------------------------
auto extrude_layer(const SurfaceTriangulation& surface, int layers, Media media = {}) -> HybridMesh;
auto stack_layers(const std::vector<std::array<double, 2>>& xy, const std::vector<std::array<int, 3>>& triangles,
                  const std::vector<LayerSpec>& layers) -> HybridMesh;
auto structured_hybrid_box(int nx, int ny, int nz_wedge, int nz_tet, Media wedge_media = {},
                           Media tet_media = {}) -> HybridMesh;
auto structured_wedge_box(int n, Media media = {}) -> HybridMesh;
auto unstructured_wedge_box(int n, double xy_jitter, double z_amplitude, std::uint64_t seed, Media media = {})
    -> HybridMesh;
auto arnold_wedge_box(int n, double delta, Media media = {}) -> HybridMesh;
auto perturb_vertically(const HybridMesh& mesh, double amplitude, std::uint64_t seed) -> HybridMesh;
/// n x n grid of [-1,1]^2 cut into 2 n^2 triangles (the "layers" mesh kind's surface)
void structured_surface(int n, std::vector<std::array<double, 2>>& xy, std::vector<std::array<int, 3>>& tris);
/// "flat:z0" or "sine:z0:amp:kx:ky" surface height functions
auto eval_surface_function(const std::string& spec, double x, double y) -> double;

// ---- checks, measures, I/O ------------------------------------------------------
auto is_vertically_mapped(const WedgeVerts& v) -> bool;
void validate_mesh(const HybridMesh& mesh);
auto mesh_volume(const HybridMesh& mesh) -> double;
auto load_mesh(const std::string& path) -> HybridMesh;
void save_mesh(const HybridMesh& mesh, const std::string& path);
auto load_surface(const std::string& path) -> SurfaceTriangulation;

// ---- face connectivity ------------------------------------------------------------
struct FaceConn {
  int nbr = -1, nbr_face = -1;  // neighbour element / its face (-1: boundary)
  int tag = kReflectiveTag;
  int perm_id = -1;             // row of Connectivity::perms (-1: boundary)
};

struct Connectivity {
  std::vector<FaceConn> faces;            // (e, f) at face_offset[e] + f
  std::vector<std::int64_t> face_offset;  // num_elements + 1 entries
  std::vector<std::vector<int>> perms;    // distinct face-node permutations
  int num_interior_pairs = 0, num_boundary_faces = 0;

  auto at(int e, int f) const -> const FaceConn& { return faces[face_offset[e] + f]; }
  /// my face node i matches neighbour face node perm(e, f)[i]
  auto perm(int e, int f) const -> const std::vector<int>& { return perms[at(e, f).perm_id]; }
};

auto face_vertex_ids(const HybridMesh& mesh, int e, int f) -> std::vector<int>;
auto face_node_coords(const HybridMesh& mesh, const References& refs, int e, int f) -> std::vector<Vert3>;
auto build_connectivity(const HybridMesh& mesh, const References& refs) -> Connectivity;

} // namespace prismdg
