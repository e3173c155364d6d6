/*
 * prismdg_b200.h -- C ABI of the B200-native wedge/tet DG time-stepping path.
 *
 * The reference (prismdg, arXiv 1607.03399) is a C++ library; its hot path is
 *   run_simulation -> step -> TimeStepper::step (LSERK45) -> compute_rhs
 * (proj/src/solver.cpp:591-666, 583-589, 536-557, 362-377).  This header is the
 * thin C layer the reference's own C++ host code would call instead of its
 * OpenMP compute_rhs / serial update: plain pointers and sizes, no C++ or torch
 * types, status codes instead of exceptions.  Every entry point names the
 * reference interface it replaces.
 *
 * Status codes follow the reference's exception taxonomy and CLI exit codes
 * (proj/include/prismdg/types.hpp:14-34, proj/tools/main.cpp:84-98).
 * Calls on one pdg_ctx are stream-ordered and not thread-safe.  There is no CPU
 * fallback: pdg_create fails with PDG_ERR_CUDA when no sm_100 device exists.
 */
#ifndef PRISMDG_B200_H
#define PRISMDG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDG_OK 0
#define PDG_ERR_CONFIG 2    /* ConfigError    (types.hpp:15-18)  */
#define PDG_ERR_NUMERICAL 3 /* NumericalError (types.hpp:26-30)  */
#define PDG_ERR_MESH 4      /* MeshError      (types.hpp:20-24)  */
#define PDG_ERR_CUDA 5      /* device / CUDA runtime failure       */
#define PDG_ERR_ANALYSIS 6  /* AnalysisError  (types.hpp:32-34)  */

#define PDG_FLUX_UPWIND 0 /* FluxMode::upwind  (solver.hpp:14) */
#define PDG_FLUX_CENTRAL 1
#define PDG_FLUX_CUSTOM 2

#define PDG_MASS_EXACT 0  /* QuadratureMode::exact  (operators.hpp:17) */
#define PDG_MASS_LUMPED 1 /* QuadratureMode::lumped                      */
#define PDG_MASS_WADG 2   /* weight-adjusted inverse Mhat^-1 M_{1/J} Mhat^-1 (north-star
                             extension; tets stay exact) */

typedef struct pdg_mesh pdg_mesh; /* prismdg::HybridMesh      (mesh.hpp:22-41)   */
typedef struct pdg_disc pdg_disc; /* prismdg::Discretization  (solver.hpp:29-59) */
typedef struct pdg_ctx pdg_ctx;   /* device-resident discretization + state      */

/* Thread-local message of the last failing call (exception what()). */
const char* pdg_last_error(void);
int pdg_abi_version(void);

/* ---------------------------------------------------------------- meshes
 * Generators of proj/include/prismdg/mesh.hpp:61-92; media are {rho, kappa}. */
int pdg_mesh_structured_hybrid_box(int nx, int ny, int nz_wedge, int nz_tet,
                                   const double wedge_media[2], const double tet_media[2],
                                   pdg_mesh** out);                       /* mesh.hpp:70 */
int pdg_mesh_unstructured_wedge_box(int n, double xy_jitter, double z_amplitude, uint64_t seed,
                                    const double media[2], pdg_mesh** out); /* mesh.hpp:78 */
int pdg_mesh_arnold_wedge_box(int n, double delta, const double media[2],
                              pdg_mesh** out);                            /* mesh.hpp:92 */
/* stack_layers (mesh.hpp:63-65): xy[nv][2], tris[ntri][3] (0-based),
 * z_bottom/z_top[nlayers][nv], sublayers[nlayers], media[nlayers][2]. */
int pdg_mesh_stack_layers(int nv, const double* xy, int ntri, const int* tris, int nlayers,
                          const double* z_bottom, const double* z_top, const int* sublayers,
                          const double* media, pdg_mesh** out);
int pdg_mesh_perturb_vertically(const pdg_mesh* in, double amplitude, uint64_t seed,
                                pdg_mesh** out);                          /* mesh.hpp:86 */
/* family meshes of analysis.hpp:41-49 (0 structured, 1 unstructured, 2 arnold) */
int pdg_mesh_family(int family, double h, uint64_t seed, double xy_jitter, double z_amplitude,
                    double arnold_delta, pdg_mesh** out);                 /* analysis.cpp:110-124 */
int pdg_mesh_spectra(uint64_t seed, double amplitude, pdg_mesh** out);   /* analysis.cpp:237-239 */
/* a mesh from raw arrays (0-based ids, media[e] = {rho, kappa}); validated like
 * load_mesh (mesh.cpp:487-516).  Used to build a rank's local mesh. */
int pdg_mesh_from_arrays(int64_t nv, const double* vertices, int64_t nw, const int* wedges, int64_t nt,
                         const int* tets, const double* media, pdg_mesh** out);
int pdg_mesh_load(const char* path, pdg_mesh** out);                     /* mesh.hpp:117 */
int pdg_mesh_save(const pdg_mesh* mesh, const char* path);               /* mesh.hpp:118 */
/* counts[0..2] = vertices, wedges, tets */
int pdg_mesh_counts(const pdg_mesh* mesh, int64_t counts[3]);
/* any pointer may be NULL; sizes from pdg_mesh_counts (media per element) */
int pdg_mesh_export(const pdg_mesh* mesh, double* vertices, int* wedges, int* tets,
                    double* media);
int pdg_mesh_volume(const pdg_mesh* mesh, double* volume);               /* mesh.hpp:123 */
void pdg_mesh_free(pdg_mesh* mesh);

/* ---------------------------------------------------------------- discretization */
typedef struct {
  int degree, nq, nt, np_wedge, np_tet;
  int64_t num_wedges, num_tets, total_dofs, total_nodes, num_faces;
  int num_perms, num_interior_pairs, num_boundary_faces;
  int flux_mode, mass_mode;
} pdg_disc_info;

/* build_discretization (solver.hpp:61-63). threads = OpenMP threads for setup. */
int pdg_disc_build(const pdg_mesh* mesh, int degree, int flux_mode, double tau_p, double tau_u,
                   int mass_mode, int threads, pdg_disc** out);
/* build_discretization with flags.  PDG_DISC_NO_HOST_LIFTS (WADG only): do
 * not build the per-wedge exact lifts on the host either -- the reduced
 * storage of the weight-adjusted mode end to end (the CPU oracle cannot run
 * on such a discretization). */
#define PDG_DISC_NO_HOST_LIFTS 1
int pdg_disc_build_ex(const pdg_mesh* mesh, int degree, int flux_mode, double tau_p, double tau_u,
                      int mass_mode, int threads, int flags, pdg_disc** out);
int pdg_disc_get_info(const pdg_disc* d, pdg_disc_info* info);

/* A Discretization assembled from arrays the CALLER built -- the reference's
 * own Discretization (solver.hpp:29-59) flattened member by member, so the
 * device path runs on the reference's Eigen-built operators instead of this
 * library's host setup (export_to_pdg).  Layouts:
 * wedges first, then tets (mesh.hpp:25,36); nt = (N+1)(N+2)/2, nq = N+1;
 * faces in (element, face) order, 5 per wedge then 4 per tet;
 * max_nfp = max(nq*nq, nt).  Matrices are column-major (Eigen's default).
 * The shared reference data (References, reference.hpp:13-112: nodes,
 * derivative matrices, face-node lists, lift profiles) is rebuilt from the
 * degree -- the same construction, pinned against the reference's own unit
 * tests -- and the caller's face-node lists are checked against it. */
typedef struct pdg_disc_arrays {
  int degree;
  int qmode;            /* QuadratureMode (operators.hpp:17): 0 exact, 1 lumped; 2 = weight-adjusted */
  int flux_mode;        /* FluxConfig (solver.hpp:17-20), recorded; the per-face tau below are used */
  double tau_p, tau_u;
  /* HybridMesh (mesh.hpp:22-41) */
  int64_t num_vertices, num_wedges, num_tets;
  const double* vertices; /* [nv][3] */
  const int* wedges;      /* [nw][6], 0-based */
  const int* tets;        /* [ntet][4], 0-based */
  const double* media;    /* [ne][2] = {rho, kappa} */
  /* geom (ElementGeometry, geometry.hpp:20-38): per wedge {j0, j_r, j_s, volume,
   * surface_area, faces[2..4].jf_edge[0], .jf_edge[N]} (11); per tet {J (= j0),
   * volume, surface_area} (3) */
  const double* wedge_geom;
  const double* tet_geom;
  /* wedge_ops (WedgeOperators, operators.hpp:22-33) */
  const double* tri_lift;      /* [nw][nt*nt], tri_lift(i,k) at [k*nt + i]; may be NULL when qmode == 2 */
  const double* quad_lift;     /* [nw][3][nq*nt], quad_lift[e](i,a) at [(e*nq + a)*nt + i]; NULL when qmode == 2 */
  const double* txJ;           /* [nw][nq] */
  const double* tyJ;           /* [nw][nq] */
  const double* wedge_scalars; /* [nw][7] = {tzJ, rx, ry, sx, sy, jf_bottom, jf_top} */
  /* tet_ops (TetOperators, operators.hpp:37-42): [ntet][13] = {rx, ry, rz, sx, sy, sz, tx, ty, tz, lift_scale[4]} */
  const double* tet_scalars;
  /* face_data (Discretization::FaceData, solver.hpp:52-58) */
  const int* face_nbr;          /* [nfaces]: neighbour element, -1 = boundary (reflective) */
  const double* face_tau;       /* [nfaces][2] = {tau_p, tau_u} */
  const double* face_normal;    /* [nfaces][3] */
  const int* face_my_nodes;     /* [nfaces][max_nfp] or NULL (= the reference face-node lists) */
  const int* face_nbr_nodes;    /* [nfaces][max_nfp]: neighbour local volume node of my face node i */
} pdg_disc_arrays;

/* Validates (sizes, face maps onto a neighbour face, positive J) and copies;
 * the arrays may be freed afterwards.  PDG_ERR_CONFIG / PDG_ERR_MESH on bad input. */
int pdg_disc_from_arrays(const pdg_disc_arrays* a, pdg_disc** out);
/* The inverse: fill caller buffers with the per-element arrays of
 * the pdg_disc_arrays struct, same layouts; any pointer may be NULL; mesh arrays via
 * pdg_disc_mesh_export, lifts via pdg_disc_wedge_ops. */
int pdg_disc_export_arrays(const pdg_disc* d, double* wedge_geom, double* tet_geom, double* txJ, double* tyJ,
                           double* wedge_scalars, double* tet_scalars, int* face_nbr, double* face_tau,
                           double* face_normal, int* face_nbr_nodes);
/* the mesh a discretization was built on (sizes from pdg_disc_get_info /
 * pdg_disc_mesh_counts); any pointer may be NULL */
int pdg_disc_mesh_export(const pdg_disc* d, int64_t counts[3], double* vertices, int* wedges, int* tets,
                         double* media);
/* Discretization::elem_offset (solver.hpp:44), num_elements+1 entries */
int pdg_disc_elem_offset(const pdg_disc* d, int64_t* out);
/* per element face in (element, face) order: neighbour element (-1 boundary),
 * neighbour face, permutation id (Connectivity, mesh.hpp:94-107) */
int pdg_disc_face_table(const pdg_disc* d, int* nbr, int* nbr_face, int* perm_id);
int pdg_disc_perm(const pdg_disc* d, int perm_id, int* out, int* len);
/* FaceData::my_nodes / nbr_nodes of (e, f) (solver.hpp:52-58); len = nfp */
int pdg_disc_face_nodes(const pdg_disc* d, int64_t e, int f, int* my_nodes, int* nbr_nodes,
                        int* len);
/* FaceData::normal, tau_p, tau_u of every face */
int pdg_disc_face_phys(const pdg_disc* d, double* normals, double* tau_p, double* tau_u);
/* physical node coordinates node_x/y/z (solver.hpp:47-48), total_nodes x 3 */
int pdg_disc_node_coords(const pdg_disc* d, double* xyz);
/* make_initial_state (solver.hpp:98-99): kind 0 standing_wave(c,rho) params={c,rho},
 * kind 1 gaussian_pulse params={width,cx,cy,cz}; u has total_dofs entries */
int pdg_disc_initial_state(const pdg_disc* d, int kind, const double* params, double t0,
                           double* u);
int pdg_disc_estimate_dt(const pdg_disc* d, double cfl, double* dt);      /* solver.hpp:81 */
/* l2_error against the standing-wave pressure (analysis.hpp:30-32) */
int pdg_disc_l2_error(const pdg_disc* d, const double* u, double time, double* err);
/* per-element operator export for tests: L^{tri,k} (nt*nt, [k*nt+i]=L(i,k)),
 * quad lifts (3*nq*nt), wedge scalars {rx,ry,sx,sy,tzJ,j0,jr,js,jf_bottom,jf_top,
 * jf_quad[6],volume,surface_area} (18) */
int pdg_disc_wedge_ops(const pdg_disc* d, int64_t w, double* tri_lift, double* quad_lift,
                       double* scalars);
/* write_vtk_snapshot (snapshot.hpp / snapshot.cpp:68-139): legacy ASCII VTK of
 * the reference-layout state u on the nodal lattice sub-cells */
int pdg_write_vtk(const pdg_disc* d, const double* u, const char* path);
void pdg_disc_free(pdg_disc* d);

/* ---------------------------------------------------------------- device path */
#define PDG_CTX_NATIVE_ORDER 1 /* keep reference element order on device (no Morton) */
#define PDG_CTX_TIMING 2       /* bracket every stage kernel with CUDA events      */
/* multi-rate AB3: group the elements into up to L+1 rate levels by their
 * local stable step (level g steps with 2^g dt), for pdg_step_mrab */
#define PDG_CTX_MRAB_LEVELS(L) (((L) & 15) << 8)

/* Upload a discretization to `device`. Replaces the first use of the host
 * Discretization by compute_rhs / TimeStepper (solver.cpp:362-377, 536-557). */
int pdg_create(const pdg_disc* d, int device, int flags, pdg_ctx** out);
void pdg_destroy(pdg_ctx* ctx);
/* state in the reference layout (element-major [p|ux|uy|uz], node i*(N+1)+j);
 * u may be pageable or pinned host memory, or device memory when on_device=1 */
int pdg_set_state(pdg_ctx* ctx, const double* u, int on_device);
int pdg_get_state(pdg_ctx* ctx, double* u, int on_device);
/* compute_rhs(const Discretization&, const double* u, double* rhs)
 * (solver.hpp:67): writes every entry of rhs, reference layout */
int pdg_rhs(pdg_ctx* ctx, const double* u, double* rhs, int on_device);
/* the four phase functions (solver.hpp:71-74) on the context state: volume
 * writes, surface accumulates, neither scales media; result via pdg_get_rhs */
int pdg_wedge_volume(pdg_ctx* ctx);
int pdg_wedge_surface(pdg_ctx* ctx);
int pdg_tet_volume(pdg_ctx* ctx);
int pdg_tet_surface(pdg_ctx* ctx);
int pdg_get_rhs(pdg_ctx* ctx, double* rhs, int on_device);
/* load the context's rhs buffer (reference layout) -- the caller's rhs that a
 * surface phase then accumulates into, as the reference's phases do */
int pdg_set_rhs(pdg_ctx* ctx, const double* rhs, int on_device);
/* nsteps LSERK45 steps of TimeStepper::step (solver.cpp:536-557) on the
 * resident state; *t_inout += nsteps*dt.  Asynchronous on the context stream. */
int pdg_step_lserk(pdg_ctx* ctx, double dt, int nsteps, double* t_inout);
/* nsteps AB3 steps (TimeStepper::step with IntegratorKind::ab3, solver.cpp:559-581):
 * the first two steps after pdg_set_state record f and take an LSERK45 step
 * (bootstrap), then u += dt/12 (23 f_n - 16 f_{n-1} + 5 f_{n-2}).  The f
 * history lives on the device and is reset by pdg_set_state. */
int pdg_step_ab3(pdg_ctx* ctx, double dt, int nsteps, double* t_inout);
/* nmacro steps of the multi-rate Adams-Bashforth 3 integrator (the paper's
 * time integrator, after Goedel et al. 2010; not in the
 * reference code) on a context created with
 * PDG_CTX_MRAB_LEVELS(L).  Level g advances with 2^g dt, a macro step is
 * 2^(levels-1) fine steps of dt (*t_inout += that).  The first two macro
 * steps after pdg_set_state are LSERK45 steps at dt that fill every level's
 * history (the reference's AB3 bootstrap, solver.cpp:563-570).  With one
 * level this is exactly pdg_step_ab3.  Stability: dt <= AB3's step
 * (estimate_dt * 0.25, solver.hpp:114). */
int pdg_step_mrab(pdg_ctx* ctx, double dt, int nmacro, double* t_inout);
/* rate level of every reference element (-1 when multi-rate is off); *nlevels */
int pdg_mrab_levels(pdg_ctx* ctx, int* level, int* nlevels);
/* compute_energy (solver.hpp:78): deterministic device reduction */
int pdg_energy(pdg_ctx* ctx, double* energy);
/* watchdog scan (solver.cpp:647-655): first element (reference id) with a
 * non-finite DOF, or -1 */
int pdg_check_finite(pdg_ctx* ctx, int64_t* first_bad_elem);
int pdg_synchronize(pdg_ctx* ctx);
/* the cudaStream_t all work of this context is issued on */
void* pdg_stream(pdg_ctx* ctx);
/* with PDG_CTX_TIMING: per-kernel-family accumulated device time and launch
 * counts since the last reset; names: "wedge_stage","tet_stage","other" */
int pdg_kernel_times(pdg_ctx* ctx, double* wedge_ms, int64_t* wedge_launches, double* tet_ms,
                     int64_t* tet_launches, int reset);
/* algorithmic bytes moved per launch of the wedge / tet stage kernels */
int pdg_stage_bytes(pdg_ctx* ctx, double* wedge_bytes, double* tet_bytes);
/* the most recent wedge (out[0..3]) and tet (out[4..7]) stage launch:
 * {launched (0: empty element range, nothing launched), work teams started,
 *  tickets (work units handed out by the global work counter), elements per
 *  ticket}.  tickets / teams > 1 means teams loop over several work units. */
int pdg_launch_info(pdg_ctx* ctx, int64_t out[8]);
/* number of device elements and the device element -> reference element map */
int pdg_device_order(pdg_ctx* ctx, int64_t* dev_to_ref);

/* assemble_global (analysis.cpp:12-40): the dense RHS
 * operator A(i, j) = d rhs_i / d u_j, reference layout, column-major:
 * A[j * n + i], n = total_dofs.  Capped at 20000 DOFs like the reference
 * (kDenseDofCap, analysis.hpp:13; PDG_ERR_ANALYSIS above).  Built from
 * distance-2 element-coloured batches of unit probes on the device (one rhs
 * evaluation serves every element of a colour), bitwise equal to probing
 * column by column. */
int pdg_assemble_operator(pdg_ctx* ctx, double* A);

/* ---------------------------------------------------------------- partitions
 * Multi-GPU domain decomposition (no reference counterpart: SPEC.md:218 lists
 * distributed runs as a non-goal; this is the north star's sharding).  A rank
 * builds the discretization of its owned elements plus one ghost layer and
 * passes owned[e] (one byte per element of that discretization).  Only owned
 * elements are computed; before every LSERK stage the caller refreshes the
 * ghosts' states from their owners (pack on the owner, transfer, unpack). */
int pdg_create_partitioned(const pdg_disc* d, int device, int flags, const unsigned char* owned,
                           pdg_ctx** out);
/* counts[0..3] = owned wedges, owned tets, all wedges, all tets (device order:
 * owned wedges, ghost wedges, owned tets, ghost tets) */
int pdg_active_counts(pdg_ctx* ctx, int64_t counts[4]);
/* one LSERK45 stage (0..4) of the resident state (TimeStepper::step, solver.cpp:543-550) */
int pdg_step_stage(pdg_ctx* ctx, double dt, int stage);
/* whole element states of the current state, device element ids and device
 * buffers: buf[k * 4 * max(Np_wedge, Np_tet) + ...] = state of dev_elems[k] */
int pdg_pack_states(pdg_ctx* ctx, const int64_t* dev_elems, int64_t n, double* buf);
int pdg_unpack_states(pdg_ctx* ctx, const int64_t* dev_elems, int64_t n, const double* buf);
/* Owned elements are ordered interior (no ghost neighbour) first, then
 * boundary.  counts[0..5] = owned wedges, owned tets, all wedges, all tets,
 * interior wedges, interior tets. */
int pdg_partition_counts(pdg_ctx* ctx, int64_t counts[6]);
/* one LSERK stage over part 0 = all owned elements, 1 = interior only (needs
 * no ghost data; does not complete the stage), 2 = boundary only (after the
 * ghost refresh; completes the stage).  1 then 2 == 0, so the exchange can
 * overlap the interior launch. */
int pdg_step_stage_part(pdg_ctx* ctx, double dt, int stage, int part);
/* face-trace exchange: state offsets (device layout) of 4 fields x face nodes
 * of each (reference element, face) pair, written to out (host, capacity
 * n * 4 * max face nodes); *count = entries written.  Both ranks enumerate the
 * same pairs in the same order, so the lists align. */
int pdg_trace_offsets(pdg_ctx* ctx, int64_t n, const int64_t* elems, const int* faces, int64_t* out,
                      int64_t* count);
/* buf[k] = state[idx[k]] / state[idx[k]] = buf[k] on the current state
 * (device pointers).  stream: a cudaStream_t to issue on (e.g. an exchange
 * stream overlapping the interior stage launch), or NULL for the context's. */
int pdg_gather_values(pdg_ctx* ctx, const int64_t* idx, int64_t n, double* buf, void* stream);
int pdg_scatter_values(pdg_ctx* ctx, const int64_t* idx, int64_t n, const double* buf, void* stream);

/* ---------------------------------------------------------------- run driver */
typedef struct {
  double final_time;      /* RunOptions (solver.hpp:126-137) */
  double cfl;
  double fixed_dt;        /* > 0 overrides the estimate */
  double energy_interval; /* 0: log every step */
  int watchdog_every;
  double blowup_factor;
  int integrator;         /* 0 lserk4, 1 ab3 (dt = estimate * 0.25, solver.hpp:114),
                             2 multi-rate AB3 (context with PDG_CTX_MRAB_LEVELS; the step
                             counted is the macro step, fine dt = estimate * 0.25) */
  /* snapshots (RunOptions::snapshot_interval / snapshot_cb, solver.cpp:625-644):
   * at the start and whenever the time passes the next multiple of the
   * interval the state (reference layout) is streamed device -> pinned host
   * on a copy stream while stepping continues; snapshot_cb(u, time, index,
   * user) runs on the calling thread once the copy has landed (at the latest
   * by the next snapshot or the end of the run).  interval <= 0 or a NULL
   * callback: no snapshots. */
  double snapshot_interval;
  void (*snapshot_cb)(const double* u, double time, int index, void* user);
  void* snapshot_user;
} pdg_run_options;

typedef struct {
  int steps;              /* RunResult (solver.hpp:139-146) */
  double dt, final_time, initial_energy, final_energy, max_energy_increase;
  int num_logged;
} pdg_run_result;

/* run_simulation (solver.hpp:148-149) on the device; u_inout/time_inout hold
 * the SolutionState (reference layout, host).  energy_log (may be NULL) gets
 * up to max_log (time, energy) pairs.  When the watchdog fails
 * (PDG_ERR_NUMERICAL) u_inout / time_inout hold the state at the failure time,
 * as the reference's SolutionState does.  Difference from the reference: the
 * AB3 history is not part of the host state, so every call starts a fresh
 * history (two LSERK45 bootstrap steps); the reference resumes the history
 * kept in SolutionState::history (solver.hpp:84-90) across runs. */
int pdg_run_simulation(pdg_ctx* ctx, double* u_inout, double* time_inout,
                       const pdg_run_options* opts, pdg_run_result* result, double* energy_log,
                       int max_log);

#ifdef __cplusplus
}
#endif

#endif /* PRISMDG_B200_H */
