// Face connectivity and face-node permutations (host setup).
//
// Semantics follow proj/src/mesh.cpp:361-481: faces are keyed by their sorted
// vertex ids; the element seen first in (element, face) order owns the pair;
// perm[i] is the neighbour face node nearest to my face node i, chosen
// greedily among unused nodes with tolerance 1e-10 x max(diam_a, diam_b).
//
// The reference's std::map + O(nfp^2) greedy search per face is too slow for
// 1e6-element meshes.  Here faces are paired by sorting packed keys, and the
// greedy permutation is computed once per *vertex-correspondence signature*
// (which of my face vertices coincides with which neighbour face vertex) and
// then re-verified node by node on every face that reuses it (O(nfp)).  When
// every node lies within the tolerance of its cached partner and node spacing
// exceeds twice the tolerance, the greedy nearest-unused search provably picks
// the same partner, so the result is bit-identical.  A face that fails the
// verification falls back to the full greedy search.
#include "prismdg/mesh.hpp"

#include <algorithm>
#include <cmath>
#include <map>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace prismdg {

std::vector<int> face_vertex_ids(const HybridMesh& mesh, int e, int f) {
  // mesh.cpp:361-381
  if (mesh.kind(e) == ElemKind::wedge) {
    const auto& w = mesh.wedges[e];
    switch (f) {
      case 0: return {w[0], w[1], w[2]};
      case 1: return {w[3], w[4], w[5]};
      case 2: return {w[0], w[1], w[4], w[3]};
      case 3: return {w[1], w[2], w[5], w[4]};
      case 4: return {w[2], w[0], w[3], w[5]};
    }
  } else {
    const auto& t = mesh.tets[e - mesh.num_wedges()];
    switch (f) {
      case 0: return {t[0], t[1], t[2]};
      case 1: return {t[0], t[1], t[3]};
      case 2: return {t[1], t[2], t[3]};
      case 3: return {t[0], t[2], t[3]};
    }
  }
  throw MeshError("face_vertex_ids: bad face index");
}

std::vector<Vert3> face_node_coords(const HybridMesh& mesh, const References& refs, int e, int f) {
  std::vector<Vert3> out;
  if (mesh.kind(e) == ElemKind::wedge) {
    const auto v = mesh.wedge_verts(e);
    for (int id : refs.wedge.face_nodes[f])
      out.push_back(wedge_map(v, refs.wedge.r[id], refs.wedge.s[id], refs.wedge.t[id]));
  } else {
    const auto tv = mesh.tet_verts(e - mesh.num_wedges());
    for (int id : refs.tet.face_nodes[f])
      out.push_back(tet_map(tv, refs.tet.r[id], refs.tet.s[id], refs.tet.t[id]));
  }
  return out;
}

namespace {

double element_diameter(const HybridMesh& mesh, int e) {
  const int* ids;
  int n;
  if (mesh.kind(e) == ElemKind::wedge) {
    ids = mesh.wedges[e].data();
    n = 6;
  } else {
    ids = mesh.tets[e - mesh.num_wedges()].data();
    n = 4;
  }
  double d = 0.0;
  const auto& vs = mesh.vertices;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      d = std::max(d, std::hypot(vs[ids[i]][0] - vs[ids[j]][0], vs[ids[i]][1] - vs[ids[j]][1],
                                 vs[ids[i]][2] - vs[ids[j]][2]));
  return d;
}

double dist(const Vert3& a, const Vert3& b) {
  return std::hypot(a[0] - b[0], a[1] - b[1], a[2] - b[2]);
}

// the reference's greedy nearest-unused matcher (mesh.cpp:452-475); returns
// false (and the offending distance) if some node has no partner within tol
bool greedy_match(const std::vector<Vert3>& ca, const std::vector<Vert3>& cb, double tol,
                  std::vector<int>& perm, double& worst) {
  const int nfp = (int)ca.size();
  perm.assign(nfp, -1);
  std::vector<char> used(nfp, 0);
  for (int i = 0; i < nfp; ++i) {
    int best = -1;
    double bestd = 1e300;
    for (int j = 0; j < nfp; ++j) {
      if (used[j]) continue;
      const double d = dist(ca[i], cb[j]);
      if (d < bestd) {
        bestd = d;
        best = j;
      }
    }
    if (best < 0 || bestd > tol) {
      worst = bestd;
      return false;
    }
    perm[i] = best;
    used[best] = 1;
  }
  return true;
}

std::string fmt17(double x) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", x);
  return buf;
}

struct FaceKey {
  std::array<int, 4> v; // sorted vertex ids, -1 padded
  int e, f;
};

} // namespace

Connectivity build_connectivity(const HybridMesh& mesh, const References& refs) {
  const int ne = mesh.num_elements();
  Connectivity conn;
  conn.face_offset.resize(ne + 1);
  conn.face_offset[0] = 0;
  for (int e = 0; e < ne; ++e) conn.face_offset[e + 1] = conn.face_offset[e] + mesh.num_faces(e);
  conn.faces.assign(conn.face_offset[ne], FaceConn{});

  std::vector<FaceKey> keys(conn.face_offset[ne]);
#pragma omp parallel for schedule(static)
  for (int e = 0; e < ne; ++e)
    for (int f = 0; f < mesh.num_faces(e); ++f) {
      auto ids = face_vertex_ids(mesh, e, f);
      std::sort(ids.begin(), ids.end());
      FaceKey& k = keys[conn.face_offset[e] + f];
      k.v = {-1, -1, -1, -1};
      for (std::size_t q = 0; q < ids.size(); ++q) k.v[q] = ids[q];
      k.e = e;
      k.f = f;
    }
  // keys are generated in (e,f) order, so a stable sort keeps the reference's
  // insertion order inside each group (list[0] = first seen = owner)
  std::stable_sort(keys.begin(), keys.end(), [](const FaceKey& a, const FaceKey& b) { return a.v < b.v; });

  struct Pair {
    int ea, fa, eb, fb;
  };
  std::vector<Pair> pairs;
  pairs.reserve(keys.size() / 2 + 1);
  for (std::size_t s = 0; s < keys.size();) {
    std::size_t t = s + 1;
    while (t < keys.size() && keys[t].v == keys[s].v) ++t;
    const std::size_t cnt = t - s;
    if (cnt == 1) {
      const int e = keys[s].e, f = keys[s].f;
      auto it = mesh.boundary_tags.find({e, f});
      conn.faces[conn.face_offset[e] + f].tag = (it != mesh.boundary_tags.end()) ? it->second : kReflectiveTag;
      conn.num_boundary_faces += 1;
    } else if (cnt != 2) {
      throw MeshError("mesh is not manifold: face shared by " + std::to_string(cnt) + " elements");
    } else {
      const auto& a = keys[s];
      const auto& b = keys[s + 1];
      if (a.v[3] >= 0 && (mesh.kind(a.e) != ElemKind::wedge || mesh.kind(b.e) != ElemKind::wedge))
        throw MeshError("quad faces may only pair wedge elements");
      pairs.push_back({a.e, a.f, b.e, b.f});
      conn.num_interior_pairs += 1;
    }
    s = t;
  }

  // signature: kinds, faces and the position in b's vertex list of each of a's
  // face vertices; the greedy permutation depends only on it (see header)
  auto signature = [&](const Pair& p) {
    const auto va = face_vertex_ids(mesh, p.ea, p.fa);
    const auto vb = face_vertex_ids(mesh, p.eb, p.fb);
    long long sig = (long long)mesh.kind(p.ea) * 2 + (long long)mesh.kind(p.eb);
    sig = sig * 8 + p.fa;
    sig = sig * 8 + p.fb;
    for (int x : va) {
      const int pos = (int)(std::find(vb.begin(), vb.end(), x) - vb.begin());
      sig = sig * 8 + pos;
    }
    return sig;
  };

  std::map<long long, int> sig_slot;          // signature -> cached perm id
  std::map<std::vector<int>, int> perm_index; // distinct permutations
  auto intern = [&](const std::vector<int>& p) {
    auto it = perm_index.find(p);
    if (it != perm_index.end()) return it->second;
    const int id = (int)conn.perms.size();
    conn.perms.push_back(p);
    perm_index.emplace(p, id);
    return id;
  };
  auto fail = [&](const Pair& p, double worst) {
    throw MeshError("face node matching failed between element " + std::to_string(p.ea + 1) +
                    " face " + std::to_string(p.fa + 1) + " and element " + std::to_string(p.eb + 1) +
                    " face " + std::to_string(p.fb + 1) + " (distance " + fmt17(worst) + ")");
  };

  std::vector<long long> sigs(pairs.size());
#pragma omp parallel for schedule(static)
  for (long long k = 0; k < (long long)pairs.size(); ++k) sigs[k] = signature(pairs[k]);
  // first occurrence of each signature: full greedy search (serial, few)
  for (std::size_t k = 0; k < pairs.size(); ++k) {
    if (sig_slot.count(sigs[k])) continue;
    const Pair& p = pairs[k];
    const auto ca = face_node_coords(mesh, refs, p.ea, p.fa);
    const auto cb = face_node_coords(mesh, refs, p.eb, p.fb);
    if (ca.size() != cb.size())
      throw MeshError("face node count mismatch between elements " + std::to_string(p.ea + 1) +
                      " and " + std::to_string(p.eb + 1));
    const double tol = 1e-10 * std::max(element_diameter(mesh, p.ea), element_diameter(mesh, p.eb));
    std::vector<int> perm;
    double worst = 0.0;
    if (!greedy_match(ca, cb, tol, perm, worst)) fail(p, worst);
    sig_slot[sigs[k]] = intern(perm);
  }

  // every pair: verify the cached permutation, fall back to greedy if needed
  std::vector<int> pid_ab(pairs.size());
  std::vector<std::vector<int>> fallback(pairs.size());
  std::vector<char> failed(pairs.size(), 0);
  std::vector<double> fail_dist(pairs.size(), 0.0);
#pragma omp parallel for schedule(dynamic, 256)
  for (long long k = 0; k < (long long)pairs.size(); ++k) {
    const Pair& p = pairs[k];
    const int cached = sig_slot.at(sigs[k]);
    const auto& perm = conn.perms[cached];
    const auto ca = face_node_coords(mesh, refs, p.ea, p.fa);
    const auto cb = face_node_coords(mesh, refs, p.eb, p.fb);
    const double tol = 1e-10 * std::max(element_diameter(mesh, p.ea), element_diameter(mesh, p.eb));
    bool ok = ca.size() == cb.size() && perm.size() == ca.size();
    for (std::size_t i = 0; ok && i < ca.size(); ++i) ok = dist(ca[i], cb[perm[i]]) <= tol;
    if (ok) {
      pid_ab[k] = cached;
    } else {
      pid_ab[k] = -1;
      double worst = 0.0;
      if (ca.size() != cb.size() || !greedy_match(ca, cb, tol, fallback[k], worst)) {
        failed[k] = 1;
        fail_dist[k] = worst;
      }
    }
  }
  for (std::size_t k = 0; k < pairs.size(); ++k) {
    if (failed[k]) fail(pairs[k], fail_dist[k]);
    if (pid_ab[k] < 0) pid_ab[k] = intern(fallback[k]);
  }
  // inverse permutations for the b side
  std::map<int, int> inverse_of;
  for (std::size_t k = 0; k < pairs.size(); ++k) {
    const int ida = pid_ab[k];
    auto it = inverse_of.find(ida);
    int idb;
    if (it == inverse_of.end()) {
      const auto& pa = conn.perms[ida];
      std::vector<int> pb(pa.size());
      for (std::size_t i = 0; i < pa.size(); ++i) pb[pa[i]] = (int)i;
      idb = intern(pb);
      inverse_of[ida] = idb;
    } else {
      idb = it->second;
    }
    const Pair& p = pairs[k];
    FaceConn& A = conn.faces[conn.face_offset[p.ea] + p.fa];
    FaceConn& B = conn.faces[conn.face_offset[p.eb] + p.fb];
    A = FaceConn{p.eb, p.fb, 0, ida};
    B = FaceConn{p.ea, p.fa, 0, idb};
  }
  return conn;
}

} // namespace prismdg
