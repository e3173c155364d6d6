// extern "C" implementation of include/prismdg_b200.h.
// Opaque handles: pdg_mesh* is a prismdg::HybridMesh*, pdg_disc* a
// prismdg::Discretization*, pdg_ctx* the device context (cuda/context.hpp).
#include "prismdg_b200.h"
#include "prismdg/solver.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>

#include "../cuda/context.hpp"
#include "prismdg/discretization.hpp"
#include "prismdg/solver.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace prismdg;

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return PDG_OK;
  } catch (const ConfigError& e) {
    g_last_error = e.what();
    return PDG_ERR_CONFIG;
  } catch (const NumericalError& e) {
    g_last_error = e.what();
    return PDG_ERR_NUMERICAL;
  } catch (const MeshError& e) {
    g_last_error = e.what();
    return PDG_ERR_MESH;
  } catch (const AnalysisError& e) {
    g_last_error = e.what();
    return PDG_ERR_ANALYSIS;
  } catch (const DeviceError& e) {
    g_last_error = e.what();
    return PDG_ERR_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PDG_ERR_CONFIG;
  }
}

HybridMesh* M(pdg_mesh* m) { return reinterpret_cast<HybridMesh*>(m); }
const HybridMesh* M(const pdg_mesh* m) { return reinterpret_cast<const HybridMesh*>(m); }
const Discretization* D(const pdg_disc* d) { return reinterpret_cast<const Discretization*>(d); }
pdg_mesh* wrap(HybridMesh&& m) { return reinterpret_cast<pdg_mesh*>(new HybridMesh(std::move(m))); }

Media media_of(const double* m) { return m ? Media{m[0], m[1]} : Media{}; }

void need(const void* p, const char* what) {
  if (!p) throw ConfigError(std::string("null ") + what);
}

} // namespace

extern "C" {

const char* pdg_last_error(void) { return g_last_error.c_str(); }
int pdg_abi_version(void) { return 1; }

// ------------------------------------------------------------------ meshes
int pdg_mesh_structured_hybrid_box(int nx, int ny, int nz_wedge, int nz_tet, const double wm[2],
                                   const double tm[2], pdg_mesh** out) {
  return guarded([&] { *out = wrap(structured_hybrid_box(nx, ny, nz_wedge, nz_tet, media_of(wm), media_of(tm))); });
}

int pdg_mesh_unstructured_wedge_box(int n, double xy_jitter, double z_amplitude, uint64_t seed,
                                    const double media[2], pdg_mesh** out) {
  return guarded([&] { *out = wrap(unstructured_wedge_box(n, xy_jitter, z_amplitude, seed, media_of(media))); });
}

int pdg_mesh_arnold_wedge_box(int n, double delta, const double media[2], pdg_mesh** out) {
  return guarded([&] { *out = wrap(arnold_wedge_box(n, delta, media_of(media))); });
}

int pdg_mesh_stack_layers(int nv, const double* xy, int ntri, const int* tris, int nlayers,
                          const double* z_bottom, const double* z_top, const int* sublayers,
                          const double* media, pdg_mesh** out) {
  return guarded([&] {
    std::vector<std::array<double, 2>> pts(nv);
    for (int v = 0; v < nv; ++v) pts[v] = {xy[2 * v], xy[2 * v + 1]};
    std::vector<std::array<int, 3>> tr(ntri);
    for (int t = 0; t < ntri; ++t) tr[t] = {tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]};
    std::vector<LayerSpec> layers(nlayers);
    for (int l = 0; l < nlayers; ++l) {
      layers[l].z_bottom.assign(z_bottom + (std::size_t)l * nv, z_bottom + (std::size_t)(l + 1) * nv);
      layers[l].z_top.assign(z_top + (std::size_t)l * nv, z_top + (std::size_t)(l + 1) * nv);
      layers[l].sublayers = sublayers[l];
      layers[l].media = media_of(media ? media + 2 * l : nullptr);
    }
    *out = wrap(stack_layers(pts, tr, layers));
  });
}

int pdg_mesh_perturb_vertically(const pdg_mesh* in, double amplitude, uint64_t seed, pdg_mesh** out) {
  return guarded([&] {
    need(in, "mesh");
    *out = wrap(perturb_vertically(*M(in), amplitude, seed));
  });
}

int pdg_mesh_family(int family, double h, uint64_t seed, double xy_jitter, double z_amplitude,
                    double arnold_delta, pdg_mesh** out) {
  return guarded([&] {
    if (family < 0 || family > 2) throw ConfigError("unknown mesh family");
    FamilyParams fp;
    fp.seed = seed;
    fp.xy_jitter = xy_jitter;
    fp.z_amplitude = z_amplitude;
    fp.arnold_delta = arnold_delta;
    *out = wrap(make_family_mesh(static_cast<MeshFamily>(family), h, fp));
  });
}

int pdg_mesh_spectra(uint64_t seed, double amplitude, pdg_mesh** out) {
  return guarded([&] { *out = wrap(spectra_mesh(seed, amplitude)); });
}

int pdg_mesh_from_arrays(int64_t nv, const double* vertices, int64_t nw, const int* wedges, int64_t nt,
                         const int* tets, const double* media, pdg_mesh** out) {
  return guarded([&] {
    HybridMesh m;
    m.vertices.resize(nv);
    for (int64_t v = 0; v < nv; ++v) m.vertices[v] = {vertices[3 * v], vertices[3 * v + 1], vertices[3 * v + 2]};
    m.wedges.resize(nw);
    for (int64_t w = 0; w < nw; ++w)
      for (int q = 0; q < 6; ++q) m.wedges[w][q] = wedges[6 * w + q];
    m.tets.resize(nt);
    for (int64_t t = 0; t < nt; ++t)
      for (int q = 0; q < 4; ++q) m.tets[t][q] = tets[4 * t + q];
    m.media.resize(nw + nt);
    for (int64_t e = 0; e < nw + nt; ++e) m.media[e] = media_of(media ? media + 2 * e : nullptr);
    validate_mesh(m);
    *out = wrap(std::move(m));
  });
}

int pdg_mesh_load(const char* path, pdg_mesh** out) {
  return guarded([&] { *out = wrap(load_mesh(path)); });
}

int pdg_mesh_save(const pdg_mesh* mesh, const char* path) {
  return guarded([&] {
    need(mesh, "mesh");
    save_mesh(*M(mesh), path);
  });
}

int pdg_mesh_counts(const pdg_mesh* mesh, int64_t counts[3]) {
  return guarded([&] {
    need(mesh, "mesh");
    counts[0] = (int64_t)M(mesh)->vertices.size();
    counts[1] = M(mesh)->num_wedges();
    counts[2] = M(mesh)->num_tets();
  });
}

int pdg_mesh_export(const pdg_mesh* mesh, double* vertices, int* wedges, int* tets, double* media) {
  return guarded([&] {
    need(mesh, "mesh");
    const HybridMesh& m = *M(mesh);
    if (vertices)
      for (std::size_t v = 0; v < m.vertices.size(); ++v)
        for (int d = 0; d < 3; ++d) vertices[3 * v + d] = m.vertices[v][d];
    if (wedges)
      for (std::size_t w = 0; w < m.wedges.size(); ++w)
        for (int q = 0; q < 6; ++q) wedges[6 * w + q] = m.wedges[w][q];
    if (tets)
      for (std::size_t t = 0; t < m.tets.size(); ++t)
        for (int q = 0; q < 4; ++q) tets[4 * t + q] = m.tets[t][q];
    if (media)
      for (std::size_t e = 0; e < m.media.size(); ++e) {
        media[2 * e] = m.media[e].rho;
        media[2 * e + 1] = m.media[e].kappa;
      }
  });
}

int pdg_mesh_volume(const pdg_mesh* mesh, double* volume) {
  return guarded([&] {
    need(mesh, "mesh");
    *volume = mesh_volume(*M(mesh));
  });
}

void pdg_mesh_free(pdg_mesh* mesh) { delete M(mesh); }

// ------------------------------------------------------------------ discretization
int pdg_disc_build(const pdg_mesh* mesh, int degree, int flux_mode, double tau_p, double tau_u,
                   int mass_mode, int threads, pdg_disc** out) {
  return pdg_disc_build_ex(mesh, degree, flux_mode, tau_p, tau_u, mass_mode, threads, 0, out);
}

int pdg_disc_build_ex(const pdg_mesh* mesh, int degree, int flux_mode, double tau_p, double tau_u,
                      int mass_mode, int threads, int flags, pdg_disc** out) {
  return guarded([&] {
    need(mesh, "mesh");
    if (flux_mode < 0 || flux_mode > 2) throw ConfigError("unknown flux mode");
    if (mass_mode < 0 || mass_mode > 2) throw ConfigError("unknown mass mode");
    if ((flags & PDG_DISC_NO_HOST_LIFTS) && mass_mode != PDG_MASS_WADG)
      throw ConfigError("PDG_DISC_NO_HOST_LIFTS requires the weight-adjusted mass mode");
    FluxConfig flux;
    flux.mode = static_cast<FluxMode>(flux_mode);
    flux.tau_p = tau_p;
    flux.tau_u = tau_u;
    const QuadratureMode qm = mass_mode == PDG_MASS_LUMPED ? QuadratureMode::lumped : QuadratureMode::exact;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#endif
    auto* d = new Discretization(build_discretization(*M(mesh), degree, flux, qm, std::max(1, threads),
                                                      static_cast<MassMode>(mass_mode),
                                                      !(flags & PDG_DISC_NO_HOST_LIFTS)));
    *out = reinterpret_cast<pdg_disc*>(d);
  });
}

int pdg_disc_get_info(const pdg_disc* dh, pdg_disc_info* info) {
  return guarded([&] {
    need(dh, "discretization");
    const Discretization& d = *D(dh);
    info->degree = d.degree;
    info->nq = d.nq;
    info->nt = d.nt;
    info->np_wedge = d.np_wedge;
    info->np_tet = d.np_tet;
    info->num_wedges = d.mesh.num_wedges();
    info->num_tets = d.mesh.num_tets();
    info->total_dofs = (int64_t)d.total_dofs;
    info->total_nodes = (int64_t)d.total_nodes;
    info->num_faces = (int64_t)d.conn.faces.size();
    info->num_perms = (int)d.conn.perms.size();
    info->num_interior_pairs = d.conn.num_interior_pairs;
    info->num_boundary_faces = d.conn.num_boundary_faces;
    info->flux_mode = (int)d.flux.mode;
    info->mass_mode = (int)d.mass_mode;
  });
}

int pdg_disc_elem_offset(const pdg_disc* dh, int64_t* out) {
  return guarded([&] {
    need(dh, "discretization");
    const auto& off = D(dh)->elem_offset;
    for (std::size_t q = 0; q < off.size(); ++q) out[q] = (int64_t)off[q];
  });
}

int pdg_disc_face_table(const pdg_disc* dh, int* nbr, int* nbr_face, int* perm_id) {
  return guarded([&] {
    need(dh, "discretization");
    const auto& faces = D(dh)->conn.faces;
    for (std::size_t q = 0; q < faces.size(); ++q) {
      if (nbr) nbr[q] = faces[q].nbr;
      if (nbr_face) nbr_face[q] = faces[q].nbr_face;
      if (perm_id) perm_id[q] = faces[q].perm_id;
    }
  });
}

int pdg_disc_perm(const pdg_disc* dh, int perm_id, int* out, int* len) {
  return guarded([&] {
    need(dh, "discretization");
    const auto& perms = D(dh)->conn.perms;
    if (perm_id < 0 || perm_id >= (int)perms.size()) throw ConfigError("perm id out of range");
    *len = (int)perms[perm_id].size();
    if (out) std::copy(perms[perm_id].begin(), perms[perm_id].end(), out);
  });
}

int pdg_disc_face_nodes(const pdg_disc* dh, int64_t e, int f, int* my_nodes, int* nbr_nodes, int* len) {
  return guarded([&] {
    need(dh, "discretization");
    const Discretization& d = *D(dh);
    if (e < 0 || e >= d.num_elements() || f < 0 || f >= d.mesh.num_faces((int)e))
      throw ConfigError("face index out of range");
    const auto& my = d.my_nodes((int)e, f);
    *len = (int)my.size();
    if (my_nodes) std::copy(my.begin(), my.end(), my_nodes);
    if (nbr_nodes) {
      const bool interior = d.conn.at((int)e, f).nbr >= 0;
      for (std::size_t i = 0; i < my.size(); ++i) nbr_nodes[i] = interior ? d.nbr_node((int)e, f, (int)i) : -1;
    }
  });
}

int pdg_disc_face_phys(const pdg_disc* dh, double* normals, double* tau_p, double* tau_u) {
  return guarded([&] {
    need(dh, "discretization");
    const auto& fp = D(dh)->fphys;
    for (std::size_t q = 0; q < fp.size(); ++q) {
      if (normals)
        for (int a = 0; a < 3; ++a) normals[3 * q + a] = fp[q].normal[a];
      if (tau_p) tau_p[q] = fp[q].tau_p;
      if (tau_u) tau_u[q] = fp[q].tau_u;
    }
  });
}

int pdg_disc_node_coords(const pdg_disc* dh, double* xyz) {
  return guarded([&] {
    need(dh, "discretization");
    const Discretization& d = *D(dh);
#pragma omp parallel for schedule(dynamic, 256)
    for (int e = 0; e < d.num_elements(); ++e)
      for (int n = 0; n < d.np(e); ++n) {
        const Vert3 x = d.node_xyz(e, n);
        for (int a = 0; a < 3; ++a) xyz[3 * (d.node_offset[e] + n) + a] = x[a];
      }
  });
}

int pdg_disc_initial_state(const pdg_disc* dh, int kind, const double* params, double t0, double* u) {
  return guarded([&] {
    need(dh, "discretization");
    FieldFunctions f;
    if (kind == 0)
      f = standing_wave(params ? params[0] : 1.0, params ? params[1] : 1.0);
    else if (kind == 1)
      f = gaussian_pulse(params ? params[0] : 0.25, params ? std::array<double, 3>{params[1], params[2], params[3]}
                                                          : std::array<double, 3>{0.0, 0.0, 0.0});
    else
      throw ConfigError("unknown initial state kind");
    const SolutionState s = make_initial_state(*D(dh), f, t0);
    std::copy(s.u.begin(), s.u.end(), u);
  });
}

int pdg_disc_estimate_dt(const pdg_disc* dh, double cfl, double* dt) {
  return guarded([&] {
    need(dh, "discretization");
    *dt = estimate_dt(*D(dh), cfl);
  });
}

int pdg_disc_l2_error(const pdg_disc* dh, const double* u, double time, double* err) {
  return guarded([&] {
    need(dh, "discretization");
    *err = l2_error(*D(dh), u, standing_wave().p, time);
  });
}

int pdg_disc_wedge_ops(const pdg_disc* dh, int64_t w, double* tri_lift, double* quad_lift, double* scalars) {
  return guarded([&] {
    need(dh, "discretization");
    const Discretization& d = *D(dh);
    if (w < 0 || w >= d.mesh.num_wedges()) throw ConfigError("wedge index out of range");
    const std::size_t nt2 = (std::size_t)d.nt * d.nt, nql = (std::size_t)3 * d.nq * d.nt;
    if (tri_lift && d.tri_lift.empty()) throw ConfigError("discretization was built without host lifts");
    if (tri_lift) std::copy(d.tri_lift.begin() + w * nt2, d.tri_lift.begin() + (w + 1) * nt2, tri_lift);
    if (quad_lift && !d.quad_lift.empty())
      std::copy(d.quad_lift.begin() + w * nql, d.quad_lift.begin() + (w + 1) * nql, quad_lift);
    if (scalars) {
      const WedgeGeo& g = d.wgeo[w];
      const double v[18] = {g.rx, g.ry, g.sx, g.sy, g.tzJ, g.j0, g.jr, g.js, g.jf_bottom, g.jf_top,
                            g.jf_quad[0][0], g.jf_quad[0][1], g.jf_quad[1][0], g.jf_quad[1][1],
                            g.jf_quad[2][0], g.jf_quad[2][1], g.volume, g.surface_area};
      std::copy(v, v + 18, scalars);
    }
  });
}

int pdg_write_vtk(const pdg_disc* dh, const double* u, const char* path) {
  return guarded([&] {
    need(dh, "discretization");
    need(u, "state");
    need(path, "path");
    write_vtk_snapshot(*D(dh), u, path);
  });
}

int pdg_disc_from_arrays(const pdg_disc_arrays* a, pdg_disc** out) {
  return guarded([&] {
    need(a, "arrays");
    need(out, "output");
    *out = reinterpret_cast<pdg_disc*>(new Discretization(discretization_from_arrays(*a)));
  });
}

int pdg_disc_export_arrays(const pdg_disc* dh, double* wedge_geom, double* tet_geom, double* txJ, double* tyJ,
                           double* wedge_scalars, double* tet_scalars, int* face_nbr, double* face_tau,
                           double* face_normal, int* face_nbr_nodes) {
  return guarded([&] {
    need(dh, "discretization");
    const Discretization& d = *D(dh);
    const int nw = d.mesh.num_wedges(), ntet = d.mesh.num_tets(), nq = d.nq;
    for (int w = 0; w < nw; ++w) {
      const WedgeGeo& g = d.wgeo[w];
      if (wedge_geom) {
        const double v[11] = {g.j0, g.jr, g.js, g.volume, g.surface_area, g.jf_quad[0][0], g.jf_quad[0][1],
                              g.jf_quad[1][0], g.jf_quad[1][1], g.jf_quad[2][0], g.jf_quad[2][1]};
        std::copy(v, v + 11, wedge_geom + 11 * (std::size_t)w);
      }
      if (wedge_scalars) {
        const double v[7] = {g.tzJ, g.rx, g.ry, g.sx, g.sy, g.jf_bottom, g.jf_top};
        std::copy(v, v + 7, wedge_scalars + 7 * (std::size_t)w);
      }
      for (int j = 0; j < nq; ++j) {
        if (txJ) txJ[(std::size_t)w * nq + j] = d.txJ[(std::size_t)w * nq + j];
        if (tyJ) tyJ[(std::size_t)w * nq + j] = d.tyJ[(std::size_t)w * nq + j];
      }
    }
    for (int t = 0; t < ntet; ++t) {
      const TetGeo& g = d.tgeo[t];
      if (tet_geom) {
        tet_geom[3 * (std::size_t)t] = g.J;
        tet_geom[3 * (std::size_t)t + 1] = g.volume;
        tet_geom[3 * (std::size_t)t + 2] = g.surface_area;
      }
      if (tet_scalars) {
        const double v[13] = {g.rx, g.ry, g.rz, g.sx, g.sy, g.sz, g.tx, g.ty, g.tz,
                              g.lift_scale[0], g.lift_scale[1], g.lift_scale[2], g.lift_scale[3]};
        std::copy(v, v + 13, tet_scalars + 13 * (std::size_t)t);
      }
    }
    const int max_nfp = std::max(d.nq * d.nq, d.nt);
    for (int e = 0; e < d.num_elements(); ++e)
      for (int f = 0; f < d.mesh.num_faces(e); ++f) {
        const std::size_t q = (std::size_t)d.conn.face_offset[e] + f;
        const FaceConn& fc = d.conn.faces[q];
        if (face_nbr) face_nbr[q] = fc.nbr;
        if (face_tau) {
          face_tau[2 * q] = d.fphys[q].tau_p;
          face_tau[2 * q + 1] = d.fphys[q].tau_u;
        }
        if (face_normal)
          for (int c = 0; c < 3; ++c) face_normal[3 * q + c] = d.fphys[q].normal[c];
        if (face_nbr_nodes) {
          int* row = face_nbr_nodes + q * max_nfp;
          std::fill(row, row + max_nfp, -1);
          if (fc.nbr >= 0)
            for (int i = 0; i < (int)d.my_nodes(e, f).size(); ++i) row[i] = d.nbr_node(e, f, i);
        }
      }
  });
}

int pdg_disc_mesh_export(const pdg_disc* dh, int64_t counts[3], double* vertices, int* wedges, int* tets,
                         double* media) {
  return guarded([&] {
    need(dh, "discretization");
    const HybridMesh& m = D(dh)->mesh;
    if (counts) {
      counts[0] = (int64_t)m.vertices.size();
      counts[1] = m.num_wedges();
      counts[2] = m.num_tets();
    }
    if (vertices)
      for (std::size_t v = 0; v < m.vertices.size(); ++v)
        for (int c = 0; c < 3; ++c) vertices[3 * v + c] = m.vertices[v][c];
    if (wedges)
      for (int w = 0; w < m.num_wedges(); ++w)
        for (int c = 0; c < 6; ++c) wedges[6 * (std::size_t)w + c] = m.wedges[w][c];
    if (tets)
      for (int t = 0; t < m.num_tets(); ++t)
        for (int c = 0; c < 4; ++c) tets[4 * (std::size_t)t + c] = m.tets[t][c];
    if (media)
      for (int e = 0; e < m.num_elements(); ++e) {
        media[2 * (std::size_t)e] = m.media[e].rho;
        media[2 * (std::size_t)e + 1] = m.media[e].kappa;
      }
  });
}

void pdg_disc_free(pdg_disc* d) { delete reinterpret_cast<Discretization*>(d); }

// ------------------------------------------------------------------ device
int pdg_create(const pdg_disc* dh, int device, int flags, pdg_ctx** out) {
  return guarded([&] {
    need(dh, "discretization");
    *out = pdg::create_context(*D(dh), device, flags);
  });
}

void pdg_destroy(pdg_ctx* ctx) { pdg::destroy_context(ctx); }

int pdg_create_partitioned(const pdg_disc* dh, int device, int flags, const unsigned char* owned, pdg_ctx** out) {
  return guarded([&] {
    need(dh, "discretization");
    need(owned, "owned mask");
    *out = pdg::create_context(*D(dh), device, flags, owned);
  });
}

int pdg_active_counts(pdg_ctx* ctx, int64_t counts[4]) {
  return guarded([&] {
    need(ctx, "context");
    counts[0] = ctx->Kw_act;
    counts[1] = ctx->Kt_act;
    counts[2] = ctx->Kw;
    counts[3] = ctx->Kt;
  });
}

int pdg_partition_counts(pdg_ctx* ctx, int64_t counts[6]) {
  return guarded([&] {
    need(ctx, "context");
    counts[0] = ctx->Kw_act;
    counts[1] = ctx->Kt_act;
    counts[2] = ctx->Kw;
    counts[3] = ctx->Kt;
    counts[4] = ctx->Kw_int;
    counts[5] = ctx->Kt_int;
  });
}

int pdg_step_stage_part(pdg_ctx* ctx, double dt, int stage, int part) {
  return guarded([&] {
    need(ctx, "context");
    pdg::stage_lserk(ctx, dt, stage, part);
  });
}

int pdg_trace_offsets(pdg_ctx* ctx, int64_t n, const int64_t* elems, const int* faces, int64_t* out,
                      int64_t* count) {
  return guarded([&] {
    need(ctx, "context");
    static_assert(sizeof(int64_t) == sizeof(long long), "int64_t is long long");
    *count = pdg::trace_offsets(ctx, n, reinterpret_cast<const long long*>(elems), faces,
                                reinterpret_cast<long long*>(out));
  });
}

int pdg_gather_values(pdg_ctx* ctx, const int64_t* idx, int64_t n, double* buf, void* stream) {
  return guarded([&] {
    need(ctx, "context");
    pdg::gather_values(ctx, reinterpret_cast<const long long*>(idx), n, buf, static_cast<cudaStream_t>(stream));
  });
}

int pdg_scatter_values(pdg_ctx* ctx, const int64_t* idx, int64_t n, const double* buf, void* stream) {
  return guarded([&] {
    need(ctx, "context");
    pdg::scatter_values(ctx, reinterpret_cast<const long long*>(idx), n, buf, static_cast<cudaStream_t>(stream));
  });
}

int pdg_step_stage(pdg_ctx* ctx, double dt, int stage) {
  return guarded([&] {
    need(ctx, "context");
    pdg::stage_lserk(ctx, dt, stage);
  });
}

int pdg_pack_states(pdg_ctx* ctx, const int64_t* dev_elems, int64_t n, double* buf) {
  return guarded([&] {
    need(ctx, "context");
    pdg::pack_states(ctx, reinterpret_cast<const long long*>(dev_elems), n, buf);
  });
}

int pdg_unpack_states(pdg_ctx* ctx, const int64_t* dev_elems, int64_t n, const double* buf) {
  return guarded([&] {
    need(ctx, "context");
    pdg::unpack_states(ctx, reinterpret_cast<const long long*>(dev_elems), n, buf);
  });
}

int pdg_set_state(pdg_ctx* ctx, const double* u, int on_device) {
  return guarded([&] {
    need(ctx, "context");
    pdg::set_state(ctx, u, on_device != 0);
  });
}

int pdg_get_state(pdg_ctx* ctx, double* u, int on_device) {
  return guarded([&] {
    need(ctx, "context");
    pdg::get_state(ctx, u, on_device != 0);
  });
}

int pdg_rhs(pdg_ctx* ctx, const double* u, double* rhs, int on_device) {
  return guarded([&] {
    need(ctx, "context");
    pdg::compute_rhs(ctx, u, rhs, on_device != 0);
  });
}

int pdg_wedge_volume(pdg_ctx* ctx) { return guarded([&] { need(ctx, "context"); pdg::run_phase(ctx, true, true); }); }
int pdg_wedge_surface(pdg_ctx* ctx) { return guarded([&] { need(ctx, "context"); pdg::run_phase(ctx, true, false); }); }
int pdg_tet_volume(pdg_ctx* ctx) { return guarded([&] { need(ctx, "context"); pdg::run_phase(ctx, false, true); }); }
int pdg_tet_surface(pdg_ctx* ctx) { return guarded([&] { need(ctx, "context"); pdg::run_phase(ctx, false, false); }); }

int pdg_get_rhs(pdg_ctx* ctx, double* rhs, int on_device) {
  return guarded([&] {
    need(ctx, "context");
    pdg::get_rhs(ctx, rhs, on_device != 0);
  });
}

int pdg_set_rhs(pdg_ctx* ctx, const double* rhs, int on_device) {
  return guarded([&] {
    need(ctx, "context");
    pdg::set_rhs(ctx, rhs, on_device != 0);
  });
}

int pdg_step_lserk(pdg_ctx* ctx, double dt, int nsteps, double* t_inout) {
  return guarded([&] {
    need(ctx, "context");
    if (nsteps < 0) throw ConfigError("nsteps must be >= 0");
    pdg::step_lserk(ctx, dt, nsteps);
    if (t_inout)
      for (int n = 0; n < nsteps; ++n) *t_inout += dt;
  });
}

int pdg_step_mrab(pdg_ctx* ctx, double dt, int nmacro, double* t_inout) {
  return guarded([&] {
    need(ctx, "context");
    if (!(dt > 0.0)) throw ConfigError("dt must be positive");
    if (nmacro < 0) throw ConfigError("nmacro must be >= 0");
    pdg::step_mrab(ctx, dt, nmacro);
    if (t_inout) *t_inout += nmacro * std::ldexp(dt, std::max(ctx->mr_nlev - 1, 0));
  });
}

int pdg_mrab_levels(pdg_ctx* ctx, int* level, int* nlevels) {
  return guarded([&] {
    need(ctx, "context");
    if (nlevels) *nlevels = ctx->mr_nlev;
    if (level) {
      const long long ne = ctx->Kw + ctx->Kt;
      for (long long e = 0; e < ne; ++e) level[e] = ctx->mr_nlev ? ctx->mr_level_ref[e] : -1;
    }
  });
}

int pdg_step_ab3(pdg_ctx* ctx, double dt, int nsteps, double* t_inout) {
  return guarded([&] {
    need(ctx, "context");
    if (nsteps < 0) throw ConfigError("nsteps must be >= 0");
    pdg::step_ab3(ctx, dt, nsteps);
    if (t_inout)
      for (int n = 0; n < nsteps; ++n) *t_inout += dt;
  });
}

int pdg_assemble_operator(pdg_ctx* ctx, double* A) {
  return guarded([&] {
    need(ctx, "context");
    need(A, "output matrix");
    const std::size_t n = ctx->disc->total_dofs;
    if (n > 20000)
      throw AnalysisError("dense operator assembly capped at 20000 DOFs, mesh has " + std::to_string(n));
    if (ctx->Kw_act != ctx->Kw || ctx->Kt_act != ctx->Kt)
      throw ConfigError("operator assembly needs an unpartitioned context");
    pdg::assemble_operator(ctx, A);
  });
}

int pdg_energy(pdg_ctx* ctx, double* energy) {
  return guarded([&] {
    need(ctx, "context");
    *energy = pdg::energy(ctx);
  });
}

int pdg_check_finite(pdg_ctx* ctx, int64_t* first_bad_elem) {
  return guarded([&] {
    need(ctx, "context");
    *first_bad_elem = pdg::check_finite(ctx);
  });
}

int pdg_synchronize(pdg_ctx* ctx) {
  return guarded([&] {
    need(ctx, "context");
    pdg::synchronize(ctx);
  });
}

void* pdg_stream(pdg_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int pdg_kernel_times(pdg_ctx* ctx, double* wedge_ms, int64_t* wedge_launches, double* tet_ms,
                     int64_t* tet_launches, int reset) {
  return guarded([&] {
    need(ctx, "context");
    long long wl = 0, tl = 0;
    pdg::kernel_times(ctx, wedge_ms, &wl, tet_ms, &tl, reset != 0);
    *wedge_launches = wl;
    *tet_launches = tl;
  });
}

int pdg_stage_bytes(pdg_ctx* ctx, double* wedge_bytes, double* tet_bytes) {
  return guarded([&] {
    need(ctx, "context");
    pdg::stage_bytes(ctx, wedge_bytes, tet_bytes);
  });
}

int pdg_launch_info(pdg_ctx* ctx, int64_t out[8]) {
  return guarded([&] {
    need(ctx, "context");
    need(out, "output");
    for (int k = 0; k < 2; ++k) {
      const auto& li = ctx->last_launch[k];
      out[4 * k] = li.launched;
      out[4 * k + 1] = li.teams;
      out[4 * k + 2] = li.tickets;
      out[4 * k + 3] = li.per_ticket;
    }
  });
}

int pdg_device_order(pdg_ctx* ctx, int64_t* dev_to_ref) {
  return guarded([&] {
    need(ctx, "context");
    for (std::size_t q = 0; q < ctx->dev_to_ref_host.size(); ++q) dev_to_ref[q] = ctx->dev_to_ref_host[q];
  });
}

// ------------------------------------------------------------------ run driver
int pdg_run_simulation(pdg_ctx* ctx, double* u_inout, double* time_inout, const pdg_run_options* opts,
                       pdg_run_result* result, double* energy_log, int max_log) {
  // run_simulation (proj/src/solver.cpp:591-666) with the state resident on the device
  return guarded([&] {
    need(ctx, "context");
    need(opts, "options");
    if (opts->integrator < 0 || opts->integrator > 2) throw ConfigError("unknown integrator");
    const bool ab3 = opts->integrator >= 1, mrab = opts->integrator == 2;
    if (mrab && ctx->mr_nlev == 0)
      throw ConfigError("the multi-rate integrator needs a context created with PDG_CTX_MRAB_LEVELS(L)");
    const int substeps = mrab ? 1 << (ctx->mr_nlev - 1) : 1; // fine steps per (macro) step
    if (!(opts->final_time > *time_inout)) throw ConfigError("final time must exceed the state time");
    if (opts->watchdog_every < 1) throw ConfigError("watchdog_every must be >= 1");
    const double span = opts->final_time - *time_inout;
    // TimeStepper::dt_scale (solver.hpp:114): AB3 runs at a quarter of the LSERK step
    const double dt0 = opts->fixed_dt > 0.0 ? opts->fixed_dt
                                            : estimate_dt(*ctx->disc, opts->cfl) * (ab3 ? 0.25 : 1.0) * substeps;
    const int steps = std::max(1, (int)std::ceil(span / dt0 - 1e-12));
    const double dt = span / steps;
    pdg::set_state(ctx, u_inout, false);
    double t = *time_inout;
    pdg_run_result res{};
    res.steps = steps;
    res.dt = dt;
    res.initial_energy = pdg::energy(ctx);
    double last = res.initial_energy;
    int nlog = 0;
    auto log_energy = [&](double tcur, double en) {
      res.max_energy_increase = std::max(res.max_energy_increase, en - last);
      last = en;
      if (energy_log && nlog < max_log) {
        energy_log[2 * nlog] = tcur;
        energy_log[2 * nlog + 1] = en;
      }
      ++nlog;
    };
    log_energy(t, res.initial_energy);
    double next_energy_t = t + opts->energy_interval;
    pdg::SnapshotStream snaps(ctx, opts->snapshot_cb, opts->snapshot_user);
    const bool snapshots = opts->snapshot_cb && opts->snapshot_interval > 0.0;
    double next_snapshot_t = t;
    if (snapshots) {
      snaps.take(t);
      next_snapshot_t += opts->snapshot_interval;
    }
    // the reference leaves SolutionState at the failure time when the
    // watchdog throws (solver.cpp:647-661): hand the device state back first
    struct StateOnThrow {
      pdg_ctx* c;
      double* u;
      double* time;
      const double* t;
      bool armed = true;
      ~StateOnThrow() {
        if (!armed) return;
        try {
          pdg::get_state(c, u, false);
          *time = *t;
        } catch (...) {
        }
      }
    } on_throw{ctx, u_inout, time_inout, &t};
    for (int n = 0; n < steps; ++n) {
      if (mrab)
        pdg::step_mrab(ctx, dt / substeps, 1);
      else if (ab3)
        pdg::step_ab3(ctx, dt, 1);
      else
        pdg::step_lserk(ctx, dt, 1);
      t += dt;
      if (opts->energy_interval <= 0.0) {
        log_energy(t, pdg::energy(ctx));
      } else if (t + 1e-12 >= next_energy_t) {
        log_energy(t, pdg::energy(ctx));
        while (next_energy_t <= t + 1e-12) next_energy_t += opts->energy_interval;
      }
      if (snapshots && t + 1e-12 >= next_snapshot_t) {
        snaps.take(t);
        while (next_snapshot_t <= t + 1e-12) next_snapshot_t += opts->snapshot_interval;
      }
      if ((n + 1) % opts->watchdog_every == 0 || n + 1 == steps) {
        const long long bad = pdg::check_finite(ctx);
        if (bad >= 0)
          throw NumericalError("non-finite state in element " + std::to_string(bad + 1) + " at time " +
                               std::to_string(t));
        const double en = pdg::energy(ctx);
        if (en > opts->blowup_factor * res.initial_energy + 1e-300)
          throw NumericalError("instability detected: energy grew from " + std::to_string(res.initial_energy) +
                               " to " + std::to_string(en) + " at time " + std::to_string(t));
      }
    }
    snaps.flush();
    res.final_time = t;
    res.final_energy = pdg::energy(ctx);
    res.num_logged = nlog;
    on_throw.armed = false;
    pdg::get_state(ctx, u_inout, false);
    *time_inout = t;
    *result = res;
  });
}

} // extern "C"
