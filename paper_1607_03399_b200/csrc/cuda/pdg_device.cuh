#pragma once
// Device-side data layout and kernel interfaces of the B200 wedge/tet DG path.
//
// HBM layout:
//  * device element order: wedges [0,Kw) then tets [Kw,Kw+Kt); within a kind the
//    order is a locality-preserving (Morton) permutation of the reference ids.
//  * state blocks: wedge d at d*4*NPW doubles, [field][slice j][tri node i]
//    (tri node fastest -> a slice or a triangular face trace is one contiguous
//    run); tet d at Kw*4*NPW + (d-Kw)*4*NPT, [field][node].
//  * per-wedge L^{tri,k} stored [k][i] (thread i reads row i of L coalesced),
//    quad lifts stored in DMMA-fragment-major order (lfrag_of / qfrag_of), a
//    geometry/media record of WG doubles and a connectivity record of kWC ints
//    (5 x {neighbour device id, node-map id}, padded to 48 bytes).
#include <cstdint>

namespace pdg {

constexpr int kMaxN = 9;
constexpr int kMaxDevices = 64; // per-device launch-configuration caches

__host__ __device__ constexpr int nq_of(int N) { return N + 1; }
__host__ __device__ constexpr int nt_of(int N) { return (N + 1) * (N + 2) / 2; }
__host__ __device__ constexpr int npw_of(int N) { return nq_of(N) * nt_of(N); }
__host__ __device__ constexpr int npt_of(int N) { return (N + 1) * (N + 2) * (N + 3) / 6; }
__host__ __device__ constexpr int fw_of(int N) { return 2 * nt_of(N) + 3 * nq_of(N) * nq_of(N); }
/// device slice stride of the wedge state ([field][slice j][tri node i]).
/// PDG_SLICE_PAD_N5 pads N = 5 slices 21 -> 22 doubles so the DMMA state
/// fragment loads are bank-conflict free; measured slower (+4.8% state bytes
/// outweigh the conflicts, profiles/round1_pad_state_ab.txt), so off: every
/// kernel and layout routine honours nts_of / npd_of, the GPU suite passes
/// either way.
#ifndef PDG_SLICE_PAD_N5
#define PDG_SLICE_PAD_N5 0
#endif
__host__ __device__ constexpr int nts_of(int N) { return (PDG_SLICE_PAD_N5 && N == 5) ? nt_of(N) + 1 : nt_of(N); }
/// device per-field block of a wedge: NQ slices of nts_of(N) (== npw_of(N) unless padded)
__host__ __device__ constexpr int npd_of(int N) { return nq_of(N) * nts_of(N); }
/// doubles per wedge geometry record
__host__ __device__ constexpr int wg_of(int N) { return 44 + 2 * nq_of(N); }
constexpr int kTG = 38; // doubles per tet record (36 used; 38 spreads the shared-memory banks of
                        // the per-tet record reads in the tet DMMA kernel epilogue)
constexpr int kWC = 12; // ints per wedge connectivity record (5 x {nbr, map} + pad, 48 B)
__host__ __device__ constexpr int even_up(int x) { return (x + 1) & ~1; }
__host__ __device__ constexpr int ceil_div(int a, int b) { return (a + b - 1) / b; }
// DMMA (m8n8k4) tiling of the per-wedge products: IT row tiles of 8 tri nodes,
// KS k-steps of 4 over tri nodes, KT k-steps of 4 over slices
__host__ __device__ constexpr int it_of(int N) { return ceil_div(nt_of(N), 8); }
__host__ __device__ constexpr int ks_of(int N) { return ceil_div(nt_of(N), 4); }
__host__ __device__ constexpr int kt_of(int N) { return ceil_div(nq_of(N), 4); }
/// per-wedge L^{tri,k} in fragment-major order: [t][s][lane] = L(8t+lane/4, 4s+lane%4)
__host__ __device__ constexpr int lfrag_of(int N) { return it_of(N) * ks_of(N) * 32; }
/// per-wedge quad lifts: [t][face][s][lane] = QL_face(8t+lane/4, 4s+lane%4)
__host__ __device__ constexpr int qfrag_of(int N) { return it_of(N) * 3 * kt_of(N) * 32; }
/// compact per-wedge operators (host layouts, padded to an even count for
/// 16-byte TMA granularity): L [k][i], quad lifts [f][a][i]
__host__ __device__ constexpr int lcomp_of(int N) { return even_up(nt_of(N) * nt_of(N)); }
__host__ __device__ constexpr int qcomp_of(int N) { return even_up(3 * nq_of(N) * nt_of(N)); }

// Weight-adjusted (WADG) shared tables, one flat array (built by the context
// from prismdg::WadgTables, operators.hpp): row-major
//   kd[6][nt][nt]  Dr, Kr Dr, Ks Dr, Ds, Kr Ds, Ks Ds
//   Pw[nt][nc]     Mhat^{-1} V_q^T diag(w_q)
//   Vq[nc][nt]     triangle basis at the cubature points
//   R[2][3][nt][nq] quad-face lifts before Ltilde: jf0 R[0][e] + jf1 R[1][e]
//   qr[nc], qs[nc], wq[nc]  cubature points and weights
//   Mhat[nt][nt], M1D[nq][nq]
__host__ __device__ constexpr int wadg_nc(int N) { return (N + 2) * (N + 2); }
__host__ __device__ constexpr int wadg_off_pw(int N) { return 6 * nt_of(N) * nt_of(N); }
__host__ __device__ constexpr int wadg_off_vq(int N) { return wadg_off_pw(N) + nt_of(N) * wadg_nc(N); }
__host__ __device__ constexpr int wadg_off_r(int N) { return wadg_off_vq(N) + nt_of(N) * wadg_nc(N); }
__host__ __device__ constexpr int wadg_off_q(int N) { return wadg_off_r(N) + 6 * nt_of(N) * nq_of(N); }
__host__ __device__ constexpr int wadg_off_mhat(int N) { return wadg_off_q(N) + 3 * wadg_nc(N); }
__host__ __device__ constexpr int wadg_off_m1d(int N) { return wadg_off_mhat(N) + nt_of(N) * nt_of(N); }
__host__ __device__ constexpr int wadg_size(int N) { return wadg_off_m1d(N) + nq_of(N) * nq_of(N); }

// wedge record offsets
enum WRec : int {
  W_RX = 0, W_RY, W_SX, W_SY, W_TZJ, W_JFB, W_JFT, W_KAPPA, W_IRHO,
  W_TXJ = 9 // then TYJ at 9+nq, normals at 9+2nq (15), taup (5), tauu (5), j0 jr js jfq[6], pad
};
__host__ __device__ constexpr int w_tyj(int N) { return 9 + nq_of(N); }
__host__ __device__ constexpr int w_nrm(int N) { return 9 + 2 * nq_of(N); }
__host__ __device__ constexpr int w_taup(int N) { return 24 + 2 * nq_of(N); }
__host__ __device__ constexpr int w_tauu(int N) { return 29 + 2 * nq_of(N); }
__host__ __device__ constexpr int w_jac(int N) { return 34 + 2 * nq_of(N); } // j0 jr js jfq[6]

// tet record offsets
enum TRec : int {
  T_RX = 0, T_RY, T_RZ, T_SX, T_SY, T_SZ, T_TX, T_TY, T_TZ, T_LS = 9, T_KAPPA = 13, T_IRHO = 14,
  T_NRM = 15, T_TAUP = 27, T_TAUU = 31, T_J = 35
};

// stage kernel mode flags
enum : int {
  M_VOLUME = 1,    // volume terms
  M_SURFACE = 2,   // surface terms
  M_MEDIA = 4,     // scale by kappa, 1/rho
  M_ACCUM = 8,     // rhs_out += (phase API) instead of =
  M_LSERK = 16,    // fused LSERK45 stage update instead of writing rhs
  M_FIRST = 32,    // a == 0: do not read res
  M_AB3 = 64,      // fused AB3 step (exact DMMA wedge kernel): rhs_out = f_n, u_out = u_in + dt (23 f_n - 16 h1 + 5 h2)
                   // with dt = the step / 12 (solver.cpp:575-577)
};

/// what a stage launcher did (host side, filled by every launcher): whether a
/// kernel was launched at all (empty element ranges launch nothing), how many
/// independent work teams it started and how many tickets (work units of
/// per_ticket elements) those teams share through the global work counter
struct LaunchInfo {
  int launched = 0;
  long long teams = 0, tickets = 0;
  int per_ticket = 0;
};

struct StageParams {
  long long Kw, Kt;               // all device elements (addressing)
  long long Kw_active, Kt_active; // end of the computed range: owned elements come first, ghosts after
  long long Kw_begin, Kt_begin;   // start of the computed range (interior / boundary split launches)
  long long tet_base; // dof offset of the first tet block
  const double* __restrict__ u_in;
  double* __restrict__ u_out;
  double* __restrict__ res;
  double* __restrict__ rhs_out;
  double a, b, dt;
  int mode;
  // wedges
  const double* __restrict__ wgeo;
  const int* __restrict__ wconn;
  const double* __restrict__ Lt;
  const double* __restrict__ QL;
  const double* __restrict__ wadg; // WADG shared tables (null unless the mass mode is wadg)
  const double* __restrict__ wadg_frag; // the same, fragment-major (global-memory table variant)
  // tets
  const double* __restrict__ tgeo;
  const int* __restrict__ tconn;
  // shared reference tables
  const double* __restrict__ DrT;  // [k][i]
  const double* __restrict__ DsT;
  const double* __restrict__ Dt;   // [j][l]
  const double* __restrict__ prof; // [2][nq] tri-face lift profiles
  const int* __restrict__ wface_dev; // [FW] device-layout node of each wedge face node
  const double* __restrict__ tDrT; // [k][n]
  const double* __restrict__ tDsT;
  const double* __restrict__ tDtT;
  const double* __restrict__ tLiftT; // [4*nt][n]
  const int* __restrict__ tface; // [4*nt] tet face nodes
  const double* __restrict__ tet_frag; // fragment-major tet operators in global memory (N >= 6)
  const int* __restrict__ nbr_nodes; // [combo][max_nfp]
  int max_nfp;
  int nbr_nodes_len; // ints in nbr_nodes
  // dynamic element scheduling: element = atomicAdd(ticket, 1) - ticket_base
  unsigned long long* ticket;
  unsigned long long ticket_base;
  unsigned long long* ticket_host_next; // host side: next base (advanced by the launcher)
  int ticket_batch;                     // consecutive elements per ticket (set by the launcher)
  LaunchInfo* info;                     // host side, may be null: filled by the launcher
  const double* __restrict__ h1;        // M_AB3: f_{n-1}, f_{n-2}
  const double* __restrict__ h2;
};

struct EnergyParams {
  long long Kw, Kt, tet_base;
  const double* __restrict__ u;
  const double* __restrict__ wgeo;
  const double* __restrict__ tgeo;
  const double* __restrict__ Mtri;  // [nt][nt]
  const double* __restrict__ Xr;
  const double* __restrict__ Xs;
  const double* __restrict__ M1D;   // [nq][nq]
  const double* __restrict__ w1d;   // GLL weights
  const double* __restrict__ Mtet;  // [npt][npt]
  int lumped;
  const double* __restrict__ wadg; // non-null: wedges use the weight-adjusted mass
  double* __restrict__ partials;
};

// launchers (instantiated per degree in the .cu files)
cudaError_t launch_wedge_stage(int N, const StageParams& p, cudaStream_t s); // FP64 tensor-core (DMMA) kernel
bool wedge_stage_ab3_supported(int N); // the DMMA wedge kernel has the fused AB3 epilogue (M_AB3) at this N
cudaError_t launch_tet_stage(int N, const StageParams& p, cudaStream_t s);
/// warp-specialised wedge kernel (producer warp: tickets, TMA, gathers, fluxes; N = 4..7)
bool wedge_ws_supported(int N);
cudaError_t launch_wedge_ws_stage(int N, const StageParams& p, cudaStream_t s);
bool tet_dmma_supported(int N);
int wedge_simt_max_degree();
/// thread-per-DOF-column low-order exact wedge kernel (wedge_lo.cu, N = 1..3)
bool wedge_lo_supported(int N);
cudaError_t launch_wedge_lo_stage(int N, const StageParams& p, cudaStream_t s);
/// thread-per-(wedge, slice) exact wedge kernel (wedge_sl.cu, N = 1)
bool wedge_sl_supported(int N);
cudaError_t launch_wedge_sl_stage(int N, const StageParams& p, cudaStream_t s);
cudaError_t launch_wedge_simt_stage(int N, const StageParams& p, cudaStream_t s); // low-order CUDA-core wedge kernel
int wedge_wadg_simt_max_degree();
cudaError_t launch_wedge_wadg_simt_stage(int N, const StageParams& p, cudaStream_t s); // low-order WADG
cudaError_t launch_tet_dmma_stage(int N, const StageParams& p, cudaStream_t s); // batched DMMA tet kernel (N <= 7)
size_t tet_frag_size(int N);
cudaError_t launch_tet_frag_fill(int N, const StageParams& p, double* out, cudaStream_t s);
cudaError_t launch_wedge_wadg_stage(int N, const StageParams& p, cudaStream_t s); // WADG (DMMA) kernel
size_t wadg_frag_size(int N);
cudaError_t launch_wadg_frag_fill(int N, const double* wadg, double* out, cudaStream_t s);
/// Mtilde-norm wedge energy partials, one per block of wadg_energy_elems_per_block() wedges
cudaError_t launch_wadg_energy(int N, const EnergyParams& p, int* nblocks_out, cudaStream_t s);
int wedge_elems_per_block(int N);
bool wedge_dmma_compact_ops(); // true: the DMMA wedge kernel reads compact L / quad lifts
int tet_elems_per_block(int N);
cudaError_t launch_energy(int N, const EnergyParams& p, int* nblocks_out, cudaStream_t s);
cudaError_t launch_reduce_sum(const double* in, int n, double* out, cudaStream_t s);
cudaError_t launch_gather_values(const long long* idx, long long n, const double* u, double* buf, cudaStream_t s);
cudaError_t launch_scatter_values(const long long* idx, long long n, const double* buf, double* u, cudaStream_t s);
cudaError_t launch_ab3_update(long long n, double* u, const double* f0, const double* f1, const double* f2,
                              double dt, cudaStream_t s);
/// multi-rate AB3 update of one rate level (DOF ranges [w0,w1) and [t0,t1));
/// commit = end of the level's step (the AB3 formula, u0 <- u), else the
/// predictor at theta in (0,1) of the step
cudaError_t launch_mrab_update(long long w0, long long w1, long long t0, long long t1, double* u, double* u0,
                               const double* f0, const double* f1, const double* f2, double h, double theta,
                               int commit, cudaStream_t s);
cudaError_t launch_to_device_layout(int N, long long Kw, long long Kt, const int* dev_to_ref,
                                    const long long* ref_offset, const double* src_ref,
                                    double* dst_dev, cudaStream_t s);
cudaError_t launch_to_reference_layout(int N, long long Kw, long long Kt, const int* dev_to_ref,
                                       const long long* ref_offset, const double* src_dev,
                                       double* dst_ref, cudaStream_t s);
/// gather / scatter whole element states (halo exchange): buf[k] = state of dev_elems[k]
cudaError_t launch_pack_states(int N, long long Kw, const long long* dev_elems, long long n, const double* u,
                               double* buf, cudaStream_t s);
cudaError_t launch_unpack_states(int N, long long Kw, const long long* dev_elems, long long n, const double* buf,
                                 double* u, cudaStream_t s);
/// non-finite scan of the owned elements (wedges [0, Kw_act), tets [Kw, Kw + Kt_act))
cudaError_t launch_check_finite(int N, long long Kw, long long Kw_act, long long Kt_act, const double* u,
                                const int* dev_to_ref, unsigned long long* first_bad,
                                cudaStream_t s);

} // namespace pdg
