// Fused wedge stage kernel for the weight-adjusted (WADG) mass, FP64 tensor
// cores (DMMA m8n8k4).  The north star's reduced-storage update: no per-wedge
// matrix is stored or streamed -- only the state, the residual and the
// per-wedge record (j0, jr, js, quad-face J_f ends, metric, normals, media).
//
// Per wedge and slice (operators.hpp WadgTables):
//   rhs = Ltilde [ K (rx Dr + sx Ds) U + vertical terms + face terms ]
//   Ltilde = Mhat^{-1} M_{1/J} = Pw diag(1/J_q) Vq     (J = j0 + jr r + js s)
//   K      = Mhat^{-1} M^{tri,k} = j0 I + jr Kr + js Ks
// which is Mtilde^{-1} (S u + B) with Mtilde = Mhat M_{1/J}^{-1} Mhat (x) M1D:
// energy-stable in the Mtilde norm, and equal to the exact stored-lift
// operator when J is constant.  The CPU oracle restates it as
// (Mhat^{-1} M_{1/J} Mhat^{-1} M^{tri,k}) (x) I applied to the exact rhs.
//
// Work decomposition as in wedge_dmma.cu: a team of IT = ceil(NT/8) warps per
// wedge, warp w owns the 8-row tile of triangle nodes [8w, 8w+8), elements
// handed out by a global ticket, TMA bulk loads double-buffered per team.
// Per element (all products as 8x8x4 DMMA tiles):
//   A  Ltilde rows of the tile: (Pw diag(1/J)) Vq             (K = cubature)
//   B  gx, gy, dv with K folded into the A fragments:
//      K (rx Dr + sx Ds) = sum_m c_m kd_m, six shared tables     (K = tri nodes)
//   C  vp = txJ Dt UX + tyJ Dt UY + tzJ Dt UZ, pdt = P Dt^T      (K = slices)
//   D  quad faces: (jf0 R0_e + jf1 R1_e) [Fp_e | Fu_e]           (K = edge nodes)
//   E  assemble the pre-lift buffer B (4 fields x NQ slices) in shared memory
//   F  rhs = Ltilde B (A fragments of Ltilde by quad shuffles)   (K = tri nodes)
//   G  media scaling, LSERK45 stage update, streaming stores.
// Reference arithmetic it extends: wedge_volume_elem / surface_elem /
// scale_media / lserk (proj/src/solver.cpp:164-218, 258-335, 337-346, 541-551).
#include <cuda_runtime.h>

#include <cstdlib>

#include "pdg_device.cuh"
#include "tma.cuh"

namespace pdg {

namespace {

__host__ __device__ constexpr int r2(int x) { return (x + 1) & ~1; }
__host__ __device__ constexpr int r4(int x) { return (x + 3) & ~3; }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int cf_stride(int x) {
  return (x % 16 == 4 || x % 16 == 12) ? x : cf_stride(x + 1);
}

constexpr int kComboCapW = 2048; // ints of neighbour node maps kept in shared memory
#ifndef PDG_WADG_PAD_STATE
#define PDG_WADG_PAD_STATE 1
#endif
// permuted k order of the K-folded gradient products at odd NT and no
// end-of-element barrier (parity flux / 1/J buffers): see PDG_KPERM and
// PDG_NO_END_BARRIER in wedge_dmma.cu
#ifndef PDG_WADG_KPERM
#define PDG_WADG_KPERM 1
#endif
#ifndef PDG_WADG_NO_END_BARRIER
#define PDG_WADG_NO_END_BARRIER 1
#endif
// K-folded gradient and vertical products (phases B, C) before the flux phase,
// between issuing the neighbour gathers and using them
#ifndef PDG_WADG_VOL_FIRST
#define PDG_WADG_VOL_FIRST 1
#endif
// the pre-lift buffer exchange through an mbarrier instead of bar.sync: a warp
// arrives when its rows of B are written, forms its Ltilde rows (phase A, which
// needs only 1/J at the cubature) and then waits for the other warps' rows.
// Measured (profiles/round2_mbar_ab.txt): N = 4 / 5 / 6 / 7 -2.1 / -3.5 / -4.0 / -6.3%
// (Ltilde's accumulators are no longer live across phases D and E: no N = 7 spills)
#ifndef PDG_WADG_MB
#define PDG_WADG_MB 1
#endif
// (the flux exchange through an mbarrier too, with the volume products between its
// arrival and wait at N = 5, 6, measured +0.9 / -0.5% and removed: round2_mbar_ab.txt)
#ifndef PDG_WADG_NOEND_MAX_N
#define PDG_WADG_NOEND_MAX_N 7
#endif
__host__ __device__ constexpr int wkmap(int s, int tig, int KS, bool perm) {
  return (perm && s < 4 * (KS / 4)) ? 16 * (s >> 2) + 4 * tig + (s & 3) : 4 * s + tig;
}
// threads per CTA: 384 (>= 168 registers) at N <= 6, 512 at N = 7 (global tables)
// -- measured, profiles/round1_wadg_tables.txt
#ifndef PDG_WADG_THREAD_CAP
#define PDG_WADG_THREAD_CAP(N) ((N) >= 7 ? 512 : 384)
#endif

template <int N, int NST_, bool TG = false>
struct WCfg {
  // NP = device per-field block (NQ slices of ST doubles), ST = device slice stride
  static constexpr int NQ = nq_of(N), NT = nt_of(N), NP = npd_of(N), ST = nts_of(N), FW = fw_of(N), WG = wg_of(N);
  static constexpr int IT = it_of(N), KS = ks_of(N), KT = kt_of(N);
  static constexpr int NC = wadg_nc(N), KQ = ceil_div(NC, 4);
  static constexpr int JT = ceil_div(NQ, 8);     // slice column tiles
  static constexpr int CT = ceil_div(4 * NQ, 8); // (field, slice) column tiles of the final product
  static constexpr int T = IT;                   // warps per team
  // shared tables (doubles)
  static constexpr int KDT = IT * KS * 32;       // one K-folded derivative table
  static constexpr int PQT = IT * KQ * 32;       // Pw (A layout) / Vq (B layout)
  static constexpr int RT = IT * 3 * KT * 32;    // R0 or R1, all three faces
  static constexpr int DTT = JT * KT * 32;
  static constexpr int BIGTAB = 6 * KDT + 2 * PQT + 2 * RT; // K-folded, Pw, Vq, R tables
  // TG: the big tables stay in global memory (fragment-major, L1-resident) and
  // shared memory only holds the small ones, leaving room for more teams
  static constexpr int TABLES = r2((TG ? 0 : BIGTAB) + DTT + 2 * NQ + 2 * NC + ceil_div(FW, 2) + kComboCapW / 2);
  // per-stage buffers: state, residual, record + connectivity
  static constexpr int USTR = r4(4 * NP) + 2;
  static constexpr int STAGE = r2(2 * USTR + WG + kWC / 2);
  // work buffers
  static constexpr int BST = cf_stride(NT);                  // pre-lift buffer column stride
  static constexpr int BS = r2((8 * CT - 1) * BST + 4 * KS + 8);
  static constexpr int FQ = 3 * JT * KT * 32;                // fragment-major quad fluxes
  static constexpr int FTRI = r2(2 * NT);                    // bottom/top tri fluxes
  static constexpr int IJ = r2(4 * KQ);                      // 1/J at the cubature points
  // padded state copy for bank-conflict-free fragment loads (see wedge_dmma.cu)
  // measured: N = 4 5.05 -> 4.60 ms, N = 5 8.59 -> 8.86 ms (profiles/round1_pad_state_ab.txt)
  static constexpr bool KP = PDG_WADG_KPERM && (NT & 1) && ST == NT;
  static constexpr bool PAD = PDG_WADG_PAD_STATE && cf_stride(NT) != NT && N == 4 && !KP;
  static constexpr int SP = PAD ? cf_stride(NT) : ST;
  static constexpr int UPS = PAD ? r2((4 * NQ + 8 * JT + 4 * KT) * SP + 4 * KS + 8) : 0;
  static constexpr int FBW = 2 * (FTRI + FQ) + IJ; // flux buffers + 1/J, one element
  static constexpr int FBUF = (PDG_WADG_NO_END_BARRIER && !PAD && NST_ == 2 && N <= PDG_WADG_NOEND_MAX_N) ? 2 : 1;
  static constexpr int WORK = BS + FBUF * FBW + UPS;
  static constexpr int SMEM_BUDGET = 225 * 1024;
  static constexpr int HDR = 6; // 3 mbarriers + 3 schedule slots
  static constexpr int NSTAGE = (NST_ == 2 && (TABLES + HDR + 2 * STAGE + WORK) * 8 <= SMEM_BUDGET) ? 2 : 1;
  static constexpr int PER_TEAM = HDR + NSTAGE * STAGE + WORK;
  static constexpr bool NOEND = FBUF == 2 && NSTAGE == 2;
  // measured (profiles/round1_volfirst_ab.txt): N = 4 -1.2%, N = 7 -2.4%, N = 5 +5.7%, N = 6 +4.3%
  static constexpr bool VF = PDG_WADG_VOL_FIRST && (N == 4 || N == 7);
  static constexpr int TPB_SMEM = (SMEM_BUDGET / 8 - TABLES) / PER_TEAM;
  static constexpr int TPB = cmax(1, cmin(cmin(15, PDG_WADG_THREAD_CAP(N) / (32 * T)), TPB_SMEM)); // teams per CTA
  static constexpr int THREADS = 32 * T * TPB;
  static constexpr size_t SMEM_BYTES = (size_t)8 * (TABLES + TPB * PER_TEAM);
  static constexpr int QF_LANE = ceil_div(FW, 32 * T); // face nodes per team thread
  static_assert(BST >= 4 * KS, "pre-lift columns must hold the padded K range");
  static_assert(SMEM_BYTES <= 227 * 1024, "WADG tables do not fit in shared memory");
};

/// elements per ticket: batching cuts same-address atomics (the global work
/// counter) at low N, where an element is only a few hundred cycles of work
inline int ticket_batch(int N) {
  static const int env = [] {
    const char* v = std::getenv("PDG_TICKET_BATCH");
    return v ? std::atoi(v) : 0;
  }();
  if (env > 0) return env;
  // measured sweeps, round 1 (profiles/round1_ticket_batch.txt, round1_ticket_batch2.txt)
  return N <= 3 ? 8 : 4;
}

/// big WADG tables in L1-cached global memory instead of shared memory
inline bool wadg_tables_global_default(int N) { return N >= 7; } // measured: profiles/round1_wadg_tables.txt

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void team_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

/// fragment-major big tables [kd_m][Pw][Vq][R_m,e] from the flat WadgTables layout
template <int N>
__device__ void fill_wadg_tables(double* dst, const double* W, int tid, int nthr) {
  using C = WCfg<N, 1>;
  constexpr int NT = C::NT, NQ = C::NQ, NC = C::NC, IT = C::IT, KS = C::KS, KT = C::KT, KQ = C::KQ;
  double* sKD = dst;
  double* sPw = sKD + 6 * C::KDT;
  double* sVq = sPw + C::PQT;
  double* sR = sVq + C::PQT;
  for (int q = tid; q < 6 * C::KDT; q += nthr) {
    const int lane = q & 31, rest = q >> 5;
    const int s = rest % KS, t = (rest / KS) % IT, m = rest / (KS * IT);
    const int i = 8 * t + (lane >> 2), k = wkmap(s, lane & 3, KS, C::KP);
    sKD[q] = (i < NT && k < NT) ? W[(m * NT + i) * NT + k] : 0.0;
  }
  for (int q = tid; q < C::PQT; q += nthr) {
    const int lane = q & 31, rest = q >> 5;
    const int s = rest % KQ, t = rest / KQ;
    const int r = 8 * t + (lane >> 2), k = 4 * s + (lane & 3);
    const bool in = r < NT && k < NC;
    sPw[q] = in ? W[wadg_off_pw(N) + r * NC + k] : 0.0;
    sVq[q] = in ? W[wadg_off_vq(N) + k * NT + r] : 0.0;
  }
  for (int q = tid; q < 2 * C::RT; q += nthr) {
    const int lane = q & 31, rest = q >> 5;
    const int s = rest % KT, e = (rest / KT) % 3, t = (rest / (3 * KT)) % IT, m = rest / (3 * KT * IT);
    const int i = 8 * t + (lane >> 2), a = 4 * s + (lane & 3);
    sR[q] = (i < NT && a < NQ) ? W[wadg_off_r(N) + ((m * 3 + e) * NT + i) * NQ + a] : 0.0;
  }
}

template <int N>
__global__ void wadg_frag_kernel(const double* __restrict__ W, double* __restrict__ out) {
  fill_wadg_tables<N>(out, W, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

template <int N, int NST>
__device__ __forceinline__ void load_element(const StageParams& p, double* stg, long long e, const double* res_src,
                                             uint64_t* bar) {
  using C = WCfg<N, NST>;
  constexpr int NP = C::NP;
  double* U = stg;
  double* R = U + C::USTR;
  double* G = R + C::USTR;
  const uint32_t bytes = 8u * (4 * NP + C::WG) + 4u * kWC + (res_src ? 32u * NP : 0u);
  const uint64_t keep = l2_policy_evict_last(), stream = l2_policy_evict_first();
  mbar_arrive_expect_tx(bar, bytes);
  tma_load_1d_hint(U, p.u_in + e * 4 * NP, 32 * NP, bar, keep);
  if (res_src) tma_load_1d_hint(R, res_src + e * 4 * NP, 32 * NP, bar, stream);
  tma_load_1d_hint(G, p.wgeo + e * C::WG, 8 * C::WG, bar, stream);
  tma_load_1d_hint(G + C::WG, p.wconn + e * kWC, 4 * kWC, bar, stream);
}

template <int N, bool COMBO_SMEM, bool FUSED, int NST, bool TG>
__global__ void __launch_bounds__(WCfg<N, NST, TG>::THREADS, 1) wedge_wadg_kernel(const StageParams p) {
  using C = WCfg<N, NST, TG>;
  constexpr int NQ = C::NQ, NT = C::NT, NP = C::NP, FW = C::FW, WG = C::WG, T = C::T;
  constexpr int IT = C::IT, KS = C::KS, KT = C::KT, KQ = C::KQ, NC = C::NC, JT = C::JT, CT = C::CT;
  constexpr int BST = C::BST;
  constexpr int QL_ = C::QF_LANE;
  extern __shared__ __align__(16) double smem[];

  // ---- tables (fragment-major, zero padded) -----------------------------------
  double* sSmall = smem + (TG ? 0 : C::BIGTAB);
  double* sDt = sSmall;               // [jt][s][lane]   = Dt(8jt+gid, 4s+tig)
  double* sProf = sDt + C::DTT;       // [2][NQ]
  double* sQr = sProf + 2 * NQ;       // [NC]
  double* sQs = sQr + NC;             // [NC]
  int* sWface = reinterpret_cast<int*>(sQs + NC);
  int* sCombo = sWface + 2 * ceil_div(FW, 2);
  for (int q = threadIdx.x; q < (int)(C::SMEM_BYTES / 8); q += C::THREADS) smem[q] = 0.0;
  __syncthreads();
  const double* W = p.wadg;
  if (!TG) fill_wadg_tables<N>(smem, W, threadIdx.x, C::THREADS);
  const double* tKD = TG ? p.wadg_frag : smem; // [m][t][s][lane] = kd_m(8t+gid, 4s+tig)
  const double* tPw = tKD + 6 * C::KDT;        // [t][s][lane]    = Pw(8t+gid, 4s+tig)
  const double* tVq = tPw + C::PQT;            // [ct][s][lane]   = Vq(4s+tig, 8ct+gid)
  const double* tR = tVq + C::PQT;             // [m][t][e][s][lane] = R_m,e(8t+gid, 4s+tig)
  auto tab = [](const double* t, int idx) -> double { return TG ? __ldg(t + idx) : t[idx]; };
  for (int q = threadIdx.x; q < C::DTT; q += C::THREADS) {
    const int lane = q & 31, js = q >> 5, jt = js / KT, s = js - jt * KT;
    const int j = 8 * jt + (lane >> 2), l = 4 * s + (lane & 3);
    if (j < NQ && l < NQ) sDt[q] = p.Dt[j * NQ + l];
  }
  for (int q = threadIdx.x; q < 2 * NQ; q += C::THREADS) sProf[q] = p.prof[q];
  for (int q = threadIdx.x; q < NC; q += C::THREADS) {
    sQr[q] = W[wadg_off_q(N) + q];
    sQs[q] = W[wadg_off_q(N) + NC + q];
  }
  for (int q = threadIdx.x; q < FW; q += C::THREADS) sWface[q] = p.wface_dev[q];
  if (COMBO_SMEM)
    for (int q = threadIdx.x; q < p.nbr_nodes_len; q += C::THREADS) sCombo[q] = p.nbr_nodes[q];

  const int team = threadIdx.x / (32 * T);
  const int tt = threadIdx.x - team * 32 * T;
  const int w = tt >> 5, lane = tt & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int bar_id = 1 + team;
  double* tbase = smem + C::TABLES + (size_t)team * C::PER_TEAM;
  uint64_t* bar = reinterpret_cast<uint64_t*>(tbase);
  double* stg0 = tbase + C::HDR; // 2 mbarriers + 3 schedule slots + exchange mbarriers
  double* Bb = stg0 + NST * C::STAGE; // pre-lift buffer, column n = field*NQ + j, row = tri node
  double* const Fbase = Bb + C::BS;   // C::FBUF sets of {Ftp, Ftu, Fqp, Fqu, 1/J} (element parity)
  double* Upad = Fbase + C::FBUF * C::FBW; // padded state copy (C::PAD)
  constexpr int SP = C::SP;
  constexpr bool MB = PDG_WADG_MB && C::NOEND;
  uint64_t* vbar = bar + 5; // MB: pre-lift buffer exchange
  if (tt == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    if (MB) mbar_init(vbar, 32 * T);
    fence_barrier_init();
  }
  __syncthreads();

  int task_f[QL_], task_loc[QL_], task_my[QL_], task_pos[QL_];
#pragma unroll
  for (int q = 0; q < QL_; ++q) {
    const int m = tt + 32 * T * q;
    task_f[q] = -1;
    if (m < FW) {
      const int f = m < NT ? 0 : (m < 2 * NT ? 1 : 2 + (m - 2 * NT) / (NQ * NQ));
      const int loc = m < 2 * NT ? m - f * NT : (m - 2 * NT) - (f - 2) * NQ * NQ;
      task_f[q] = f;
      task_loc[q] = loc;
      task_my[q] = sWface[m];
      if (f < 2) {
        task_pos[q] = m;
      } else {
        const int a = loc / NQ, j = loc - a * NQ;
        task_pos[q] = ((((f - 2) * JT + j / 8) * KT + a / 4) << 5) + ((j & 7) << 2) + (a & 3);
      }
    }
  }

  const int mode = p.mode;
  const bool vol = FUSED || (mode & M_VOLUME), surf = FUSED || (mode & M_SURFACE);
  const bool lserk = FUSED || (mode & M_LSERK), media = FUSED || (mode & M_MEDIA);
  const bool first = mode & M_FIRST, accum = !FUSED && (mode & M_ACCUM);
  const double* res_src = lserk ? (first ? nullptr : p.res) : (accum ? p.rhs_out : nullptr);
  volatile long long* slot = reinterpret_cast<volatile long long*>(bar + 2);
  // tickets hand out batches of B consecutive elements (thread 0 of the team
  // keeps the current batch); one failing grab per team ends its loop
  const int B = p.ticket_batch;
  long long bnext = 0, bend = 0;
  auto grab = [&]() -> long long {
    if (bnext >= bend) {
      bnext = p.Kw_begin + (long long)(atomicAdd(p.ticket, (unsigned long long)B) - p.ticket_base);
      bend = bnext + B < p.Kw_active ? bnext + B : (bnext < p.Kw_active ? p.Kw_active : bnext + 1);
    }
    return bnext++;
  };
  if (tt == 0) {
    const long long e0 = grab();
    slot[0] = e0;
    if (e0 < p.Kw_active) load_element<N, NST>(p, stg0, e0, res_src, bar);
  }
  team_sync(bar_id, 32 * T);
  long long e = slot[0];

  for (int n = 0; e < p.Kw_active; ++n) {
    const int s = NST == 2 ? (n & 1) : 0;
    long long en = 0;
    if (tt == 0) {
      en = grab();
      slot[1 + (n & 1)] = en; // parity slots: rewritten only after every thread read it
    }
    const double* U = stg0 + s * C::STAGE;
    const double* R = U + C::USTR;
    const double* G = R + C::USTR;
    const int* Cn = reinterpret_cast<const int*>(G + WG);
    double* Ftp = Fbase + (C::NOEND ? (n & 1) * C::FBW : 0); // [2][NT]
    double* Ftu = Ftp + C::FTRI;
    double* Fqp = Ftu + C::FTRI; // [f][jt][s][lane]
    double* Fqu = Fqp + C::FQ;
    double* sIJ = Fqu + C::FQ;   // [4 KQ], zero beyond NC
    if (NST == 2 && !C::NOEND && tt == 0 && en < p.Kw_active) {
      fence_proxy_async_smem();
      load_element<N, NST>(p, stg0 + (s ^ 1) * C::STAGE, en, res_src, bar + (s ^ 1));
    }
    mbar_wait(bar + s, NST == 2 ? ((n >> 1) & 1) : (n & 1));
    const double j0 = G[w_jac(N)], jr = G[w_jac(N) + 1], js = G[w_jac(N) + 2];

    if (C::PAD)
      for (int q = tt; q < 4 * NP; q += 32 * T) {
        const int row = q / C::ST, col = q - row * C::ST;
        if (col < NT) Upad[row * SP + col] = U[q];
      }
    const double* Us = C::PAD ? Upad : U; // state with row stride SP, published by the flux barrier

    // ---- B, C (volume products; before the fluxes with PDG_WADG_VOL_FIRST) -------
    double gx[JT][2], gy[JT][2], dvx[JT][2], dvy[JT][2];
    double vp[JT][2], pdt[JT][2];
    const double tzJ = G[W_TZJ];
    auto vol_products = [&]() {
      const int iw = 8 * w + gid;
    // ---- B: K-folded gradients gx, gy and divergence parts dvx, dvy ----------
#pragma unroll
    for (int jt = 0; jt < JT; ++jt)
#pragma unroll
      for (int c = 0; c < 2; ++c) gx[jt][c] = gy[jt][c] = dvx[jt][c] = dvy[jt][c] = 0.0;
    if (vol) {
      const double rx = G[W_RX], ry = G[W_RY], sxm = G[W_SX], sym = G[W_SY];
      const double cx[6] = {rx * j0, rx * jr, rx * js, sxm * j0, sxm * jr, sxm * js};
      const double cy[6] = {ry * j0, ry * jr, ry * js, sym * j0, sym * jr, sym * js};
#pragma unroll
      for (int s2 = 0; s2 < KS; ++s2) {
        const int k = wkmap(s2, tig, KS, C::KP);
        const int fo = ((w * KS + s2) << 5) + lane;
        double ax = 0.0, ay = 0.0;
#pragma unroll
        for (int m = 0; m < 6; ++m) {
          const double d = tab(tKD, m * C::KDT + fo);
          ax += cx[m] * d;
          ay += cy[m] * d;
        }
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) {
          const int jb = 8 * jt + gid;
          const double bp = Us[jb * SP + k];
          dmma(gx[jt], ax, bp);
          dmma(gy[jt], ay, bp);
          dmma(dvx[jt], ax, Us[(NQ + jb) * SP + k]);
          dmma(dvy[jt], ay, Us[(2 * NQ + jb) * SP + k]);
        }
      }
    }

    // ---- C: vertical terms vp = txJ Dt UX + tyJ Dt UY + tzJ Dt UZ, pdt = P Dt^T
#pragma unroll
    for (int jt = 0; jt < JT; ++jt) vp[jt][0] = vp[jt][1] = pdt[jt][0] = pdt[jt][1] = 0.0;
    if (vol) {
#pragma unroll
      for (int jt = 0; jt < JT; ++jt) {
        const int jb = 8 * jt + gid;
        const int jc = jb < NQ ? jb : NQ - 1;
        const double sx_ = G[W_TXJ + jc], sy_ = G[w_tyj(N) + jc];
#pragma unroll
        for (int s2 = 0; s2 < KT; ++s2) {
          const int l = 4 * s2 + tig;
          const double bd = sDt[((jt * KT + s2) << 5) + lane];
          dmma(vp[jt], Us[(NQ + l) * SP + iw], sx_ * bd);
          dmma(vp[jt], Us[(2 * NQ + l) * SP + iw], sy_ * bd);
          dmma(vp[jt], Us[(3 * NQ + l) * SP + iw], tzJ * bd);
          dmma(pdt[jt], Us[l * SP + iw], bd);
        }
      }
    }

    };
    // ---- numerical fluxes on all face nodes; 1/J at the cubature points -------
    if (surf) {
      double nb[QL_][4];
#pragma unroll
      for (int q = 0; q < QL_; ++q) {
        const int f = task_f[q];
        if (f >= 0) {
          const int nbr = Cn[2 * f];
          if (nbr >= 0) {
            const int mi = Cn[2 * f + 1] * p.max_nfp + task_loc[q];
            const int node = COMBO_SMEM ? sCombo[mi] : __ldg(p.nbr_nodes + mi);
            const double* src;
            int fs;
            if (nbr < p.Kw) {
              src = p.u_in + (long long)nbr * 4 * NP + node;
              fs = NP;
            } else {
              src = p.u_in + p.tet_base + (long long)(nbr - p.Kw) * 4 * npt_of(N) + node;
              fs = npt_of(N);
            }
            nb[q][0] = __ldg(src);
            nb[q][1] = __ldg(src + fs);
            nb[q][2] = __ldg(src + 2 * fs);
            nb[q][3] = __ldg(src + 3 * fs);
          }
        }
      }
      if (C::VF) vol_products(); // while the gathers are in flight
#pragma unroll
      for (int q = 0; q < QL_; ++q) {
        const int f = task_f[q];
        if (f >= 0) {
          const int my = task_my[q];
          const double pm = U[my];
          const double nx = G[w_nrm(N) + 3 * f], ny = G[w_nrm(N) + 3 * f + 1], nz = G[w_nrm(N) + 3 * f + 2];
          const double taup = G[w_taup(N) + f], tauu = G[w_tauu(N) + f];
          double fp, fu;
          if (Cn[2 * f] >= 0) {
            const double dp = nb[q][0] - pm;
            const double dun = nx * (nb[q][1] - U[NP + my]) + ny * (nb[q][2] - U[2 * NP + my]) +
                               nz * (nb[q][3] - U[3 * NP + my]);
            fp = 0.5 * (taup * dp - dun);
            fu = 0.5 * (tauu * dun - dp);
          } else {
            const double dp = -2.0 * pm; // reflective: p+ = -p-, u+ = u-
            fp = 0.5 * taup * dp;
            fu = -0.5 * dp;
          }
          if (f < 2) {
            Ftp[task_pos[q]] = fp;
            Ftu[task_pos[q]] = fu;
          } else {
            Fqp[task_pos[q]] = fp;
            Fqu[task_pos[q]] = fu;
          }
        }
      }
    }
    if (C::VF && !surf) vol_products();
    for (int q = tt; q < NC; q += 32 * T) sIJ[q] = 1.0 / (j0 + jr * sQr[q] + js * sQs[q]);
    team_sync(bar_id, 32 * T);
    // every warp of the team has left the previous element: its stage may be refilled
    if (C::NOEND && tt == 0 && en < p.Kw_active) {
      fence_proxy_async_smem();
      load_element<N, NST>(p, stg0 + (s ^ 1) * C::STAGE, en, res_src, bar + (s ^ 1));
    }

    const int t = w;
    const int i = 8 * t + gid;
    // ---- A: Ltilde rows of tile t (columns = tri nodes, IT column tiles) ------
    double lt[IT][2];
    auto ltilde = [&]() {
#pragma unroll
    for (int ct = 0; ct < IT; ++ct) lt[ct][0] = lt[ct][1] = 0.0;
#pragma unroll
    for (int s2 = 0; s2 < KQ; ++s2) {
      const double a = tab(tPw, ((t * KQ + s2) << 5) + lane) * sIJ[4 * s2 + tig];
#pragma unroll
      for (int ct = 0; ct < IT; ++ct) dmma(lt[ct], a, tab(tVq, ((ct * KQ + s2) << 5) + lane));
    }
    };
    if (!MB) ltilde();

    if (!C::VF) vol_products();

    // ---- D: quad faces (jf0 R0_e + jf1 R1_e) [Fp_e | Fu_e] -------------------
    double qp[JT][2], qu[3][JT][2];
#pragma unroll
    for (int jt = 0; jt < JT; ++jt)
#pragma unroll
      for (int c = 0; c < 2; ++c) qp[jt][c] = qu[0][jt][c] = qu[1][jt][c] = qu[2][jt][c] = 0.0;
    if (surf) {
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        const double jf0 = G[w_jac(N) + 3 + 2 * f], jf1 = G[w_jac(N) + 4 + 2 * f];
#pragma unroll
        for (int s2 = 0; s2 < KT; ++s2) {
          const int ro = (((t * 3 + f) * KT + s2) << 5) + lane;
          const double qa = jf0 * tab(tR, ro) + jf1 * tab(tR, C::RT + ro);
#pragma unroll
          for (int jt = 0; jt < JT; ++jt) {
            const int fo = (((f * JT + jt) * KT + s2) << 5) + lane;
            dmma(qp[jt], qa, Fqp[fo]);
            dmma(qu[f][jt], qa, Fqu[fo]);
          }
        }
      }
    }

    // ---- E: pre-lift buffer B(i, field*NQ + j) ---------------------------------
    {
      const double* nrm = G + w_nrm(N);
      double n_[5][3];
#pragma unroll
      for (int f = 0; f < 5; ++f)
#pragma unroll
        for (int a = 0; a < 3; ++a) n_[f][a] = nrm[3 * f + a];
      const double jfb = G[W_JFB], jft = G[W_JFT];
      double tpb = 0.0, tpt = 0.0, tub = 0.0, tut = 0.0;
      if (surf && i < NT) {
        tpb = jfb * Ftp[i];
        tpt = jft * Ftp[NT + i];
        tub = jfb * Ftu[i];
        tut = jft * Ftu[NT + i];
      }
#pragma unroll
      for (int jt = 0; jt < JT; ++jt)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int j = 8 * jt + 2 * tig + c;
          if (i < NT && j < NQ) {
            double bp = -(vp[jt][c] + dvx[jt][c] + dvy[jt][c]);
            double bx = 0.0, by = 0.0, bz = 0.0;
            if (vol) {
              bx = -(gx[jt][c] + G[W_TXJ + j] * pdt[jt][c]);
              by = -(gy[jt][c] + G[w_tyj(N) + j] * pdt[jt][c]);
              bz = -(tzJ * pdt[jt][c]);
            }
            if (surf) {
              const double pb = sProf[j], pt = sProf[NQ + j];
              bp += tpb * pb + tpt * pt + qp[jt][c];
              const double t0 = tub * pb, t1 = tut * pt;
              const double u2 = qu[0][jt][c], u3 = qu[1][jt][c], u4 = qu[2][jt][c];
              bx += n_[0][0] * t0 + n_[1][0] * t1 + n_[2][0] * u2 + n_[3][0] * u3 + n_[4][0] * u4;
              by += n_[0][1] * t0 + n_[1][1] * t1 + n_[2][1] * u2 + n_[3][1] * u3 + n_[4][1] * u4;
              bz += n_[0][2] * t0 + n_[1][2] * t1 + n_[2][2] * u2 + n_[3][2] * u3 + n_[4][2] * u4;
            }
            Bb[j * BST + i] = bp;
            Bb[(NQ + j) * BST + i] = bx;
            Bb[(2 * NQ + j) * BST + i] = by;
            Bb[(3 * NQ + j) * BST + i] = bz;
          }
        }
    }
    if (MB) {
      mbar_arrive(vbar);
      ltilde(); // needs only 1/J: covers the other warps' pre-lift rows
      mbar_wait(vbar, n & 1);
    } else {
      team_sync(bar_id, 32 * T);
    }

    // ---- F: rhs rows of tile t = Ltilde B ------------------------------------------
    double acc[CT][2];
#pragma unroll
    for (int ct = 0; ct < CT; ++ct) acc[ct][0] = acc[ct][1] = 0.0;
#pragma unroll
    for (int s2 = 0; s2 < KS; ++s2) {
      const int srcl = gid * 4 + 2 * (s2 & 1) + (tig >> 1);
      const double v0 = __shfl_sync(0xffffffffu, lt[s2 >> 1][0], srcl);
      const double v1 = __shfl_sync(0xffffffffu, lt[s2 >> 1][1], srcl);
      const double a = (tig & 1) ? v1 : v0;
#pragma unroll
      for (int ct = 0; ct < CT; ++ct) dmma(acc[ct], a, Bb[(8 * ct + gid) * BST + 4 * s2 + tig]);
    }

    // ---- G: media, LSERK45 stage update, stores ------------------------------------
    {
      const double kappa = G[W_KAPPA], irho = G[W_IRHO];
      const double pa = p.a, pb = p.b, pdt_ = p.dt;
      const long long gofs = e * 4 * NP;
#pragma unroll
      for (int ct = 0; ct < CT; ++ct)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int col = 8 * ct + 2 * tig + c;
          if (i < NT && col < 4 * NQ) {
            const int f = col / NQ, j = col - f * NQ;
            double r = acc[ct][c];
            if (media) r *= f == 0 ? kappa : irho;
            const int o = f * NP + j * C::ST + i;
            if (lserk) {
              const double rr = first ? pdt_ * r : pa * R[o] + pdt_ * r;
              __stcs(p.res + gofs + o, rr);
              __stcs(p.u_out + gofs + o, Us[(f * NQ + j) * SP + i] + pb * rr);
            } else {
              __stcs(p.rhs_out + gofs + o, accum ? R[o] + r : r);
            }
          }
        }
    }
    if (!C::NOEND) team_sync(bar_id, 32 * T); // stage s and the work buffers are free again
    if (NST == 1 && tt == 0 && en < p.Kw_active) load_element<N, NST>(p, stg0, en, res_src, bar);
    e = slot[1 + (n & 1)];
  }
}

template <int N, bool CS, bool FUSED, int NST, bool TG>
cudaError_t launch_wadg_NC(const StageParams& p, cudaStream_t s) {
  using C = WCfg<N, NST, TG>;
  // one-time setup per device (the smem attribute is per device)
  static int grid_cap[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  auto kern = wedge_wadg_kernel<N, CS, FUSED, C::NSTAGE, TG>;
  if (grid_cap[dev] == 0) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::SMEM_BYTES);
    grid_cap[dev] = sms * (per_sm > 0 ? per_sm : 1);
  }
  const long long nact = p.Kw_active - p.Kw_begin; // elements of this launch
  if (p.info) *p.info = LaunchInfo{};
  if (nact <= 0) return cudaSuccess;
  const long long need = (nact + C::TPB - 1) / C::TPB;
  const int grid = (int)(need < grid_cap[dev] ? need : grid_cap[dev]);
  StageParams q = p;
  q.ticket_base = *p.ticket_host_next;
  q.ticket_batch = ticket_batch(N);
  const unsigned long long B = (unsigned long long)q.ticket_batch;
  *p.ticket_host_next += B * (((unsigned long long)nact + B - 1) / B + (unsigned long long)grid * C::TPB);
  kern<<<grid, C::THREADS, C::SMEM_BYTES, s>>>(q);
  if (p.info) *p.info = LaunchInfo{1, (long long)grid * C::TPB, (nact + (long long)B - 1) / (long long)B, (int)B};
  return cudaGetLastError();
}

template <int N, bool TG>
cudaError_t launch_wadg_NT(const StageParams& p, cudaStream_t s, bool fused, bool cs, int stages) {
  if (stages == 1) {
    if (fused) return cs ? launch_wadg_NC<N, true, true, 1, TG>(p, s) : launch_wadg_NC<N, false, true, 1, TG>(p, s);
    return cs ? launch_wadg_NC<N, true, false, 1, TG>(p, s) : launch_wadg_NC<N, false, false, 1, TG>(p, s);
  }
  if (fused) return cs ? launch_wadg_NC<N, true, true, 2, TG>(p, s) : launch_wadg_NC<N, false, true, 2, TG>(p, s);
  return cs ? launch_wadg_NC<N, true, false, 2, TG>(p, s) : launch_wadg_NC<N, false, false, 2, TG>(p, s);
}

template <int N>
cudaError_t launch_wadg_N(const StageParams& p, cudaStream_t s) {
  constexpr int F = M_VOLUME | M_SURFACE | M_MEDIA | M_LSERK;
  const bool fused = (p.mode & F) == F && !(p.mode & M_ACCUM);
  const bool cs = p.nbr_nodes_len <= kComboCapW;
  static const int stages = [] {
    const char* v = std::getenv("PDG_WEDGE_STAGES");
    return (v && v[0] == '1') ? 1 : 2;
  }();
  static const int tables = [] { // 0 default, 1 shared, 2 global
    const char* v = std::getenv("PDG_WADG_TABLES");
    return v ? (v[0] == 's' ? 1 : 2) : 0;
  }();
  const bool tg = tables == 2 || (tables == 0 && wadg_tables_global_default(N));
  return tg ? launch_wadg_NT<N, true>(p, s, fused, cs, stages) : launch_wadg_NT<N, false>(p, s, fused, cs, stages);
}

// ---------------------------------------------------------------------------
// Mtilde-norm energy of the wedges: one warp per wedge,
//   E_k = 1/2 sum_fields c_f sum_{j,j'} M1D(j,j') z_j^T z_j',  z_j = Lc^{-1} Mhat x_j,
// with Lc the Cholesky factor of M_{1/J} (Mtilde = Mhat M_{1/J}^{-1} Mhat (x) M1D).
// A diagnostic (compute_energy, solver.cpp:402-435), not on the stage path.
// ---------------------------------------------------------------------------
constexpr int kEnergyWarps = 4;

template <int N>
__global__ void __launch_bounds__(32 * kEnergyWarps) wadg_energy_kernel(const EnergyParams p) {
  constexpr int NQ = nq_of(N), NT = nt_of(N), NP = npd_of(N), ST = nts_of(N), NC = wadg_nc(N), WG = wg_of(N);
  constexpr int PER_WARP = NT * NT + NT * 4 * NQ + NC + 4 * NP;
  extern __shared__ double smem[];
  __shared__ double part[kEnergyWarps];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* M = smem + wid * PER_WARP; // M_{1/J}, then its Cholesky factor (lower)
  double* Y = M + NT * NT;           // [col = field*NQ + j][NT]
  double* iJ = Y + NT * 4 * NQ;      // w_q / J_q
  double* X = iJ + NC;               // the element state, device layout
  const double* Wt = p.wadg;
  const double* Vq = Wt + wadg_off_vq(N);
  const double* qr = Wt + wadg_off_q(N);
  const double* qs = qr + NC;
  const double* wq = qs + NC;
  const double* Mh = Wt + wadg_off_mhat(N);
  const double* M1 = Wt + wadg_off_m1d(N);
  const long long e = (long long)blockIdx.x * kEnergyWarps + wid;
  double val = 0.0;
  if (e < p.Kw) {
    const double* G = p.wgeo + e * WG;
    const double j0 = G[w_jac(N)], jr = G[w_jac(N) + 1], js = G[w_jac(N) + 2];
    for (int q = lane; q < NC; q += 32) iJ[q] = wq[q] / (j0 + jr * qr[q] + js * qs[q]);
    for (int q = lane; q < 4 * NP; q += 32) X[q] = p.u[e * 4 * NP + q];
    __syncwarp();
    for (int ab = lane; ab < NT * NT; ab += 32) {
      const int a = ab / NT, b = ab - a * NT;
      double sacc = 0.0;
      if (b <= a)
        for (int q = 0; q < NC; ++q) sacc += Vq[q * NT + a] * iJ[q] * Vq[q * NT + b];
      M[ab] = sacc;
    }
    // Y(:, col) = Mhat x_col, x_col = slice j of field f (device layout [f][j][i])
    for (int idx = lane; idx < NT * 4 * NQ; idx += 32) {
      const int col = idx / NT, a = idx - col * NT;
      const double* x = X + col * ST; // device layout: f*NP + j*ST = col*ST
      double sacc = 0.0;
      for (int k = 0; k < NT; ++k) sacc += Mh[a * NT + k] * x[k];
      Y[idx] = sacc;
    }
    __syncwarp();
    // Cholesky (lower, right-looking) of M
    for (int k = 0; k < NT; ++k) {
      if (lane == 0) M[k * NT + k] = sqrt(M[k * NT + k]);
      __syncwarp();
      const double dk = M[k * NT + k];
      for (int a = k + 1 + lane; a < NT; a += 32) M[a * NT + k] /= dk;
      __syncwarp();
      for (int ab = lane; ab < NT * NT; ab += 32) {
        const int a = ab / NT, b = ab - a * NT;
        if (a > k && b > k && b <= a) M[ab] -= M[a * NT + k] * M[b * NT + k];
      }
      __syncwarp();
    }
    // forward solve Lc Z = Y, one column per lane
    for (int col = lane; col < 4 * NQ; col += 32) {
      double* y = Y + col * NT;
      for (int a = 0; a < NT; ++a) {
        double sacc = y[a];
        for (int k = 0; k < a; ++k) sacc -= M[a * NT + k] * y[k];
        y[a] = sacc / M[a * NT + a];
      }
    }
    __syncwarp();
    const double ikap = 1.0 / G[W_KAPPA], rho = 1.0 / G[W_IRHO];
    for (int idx = lane; idx < 4 * NQ * NQ; idx += 32) {
      const int f = idx / (NQ * NQ), jj = idx - f * NQ * NQ, j = jj / NQ, l = jj - j * NQ;
      const double* zj = Y + (f * NQ + j) * NT;
      const double* zl = Y + (f * NQ + l) * NT;
      double dot = 0.0;
      for (int a = 0; a < NT; ++a) dot += zj[a] * zl[a];
      val += (f == 0 ? ikap : rho) * M1[j * NQ + l] * dot;
    }
    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
    val *= 0.5;
  }
  if (lane == 0) part[wid] = val;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sacc = 0.0;
    for (int q = 0; q < kEnergyWarps; ++q) sacc += part[q];
    p.partials[blockIdx.x] = sacc;
  }
}

template <int N>
cudaError_t launch_wadg_energy_N(const EnergyParams& p, int* nb, cudaStream_t s) {
  constexpr int NQ = nq_of(N), NT = nt_of(N), NP = npd_of(N), NC = wadg_nc(N);
  const size_t smem = (size_t)8 * kEnergyWarps * (NT * NT + NT * 4 * NQ + NC + 4 * NP);
  const int blocks = (int)((p.Kw + kEnergyWarps - 1) / kEnergyWarps);
  *nb = blocks;
  if (blocks == 0) return cudaSuccess;
  cudaError_t err = cudaFuncSetAttribute(wadg_energy_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  wadg_energy_kernel<N><<<blocks, 32 * kEnergyWarps, smem, s>>>(p);
  return cudaGetLastError();
}

} // namespace

cudaError_t launch_wedge_wadg_stage(int N, const StageParams& p, cudaStream_t s) {
  switch (N) {
#define PDG_CASE(n) case n: return launch_wadg_N<n>(p, s);
    PDG_CASE(1) PDG_CASE(2) PDG_CASE(3) PDG_CASE(4) PDG_CASE(5) PDG_CASE(6) PDG_CASE(7)
#undef PDG_CASE
  }
  return cudaErrorInvalidValue;
}

size_t wadg_frag_size(int N) {
  switch (N) {
#define PDG_CASE(n) case n: return (size_t)WCfg<n, 1>::BIGTAB;
    PDG_CASE(1) PDG_CASE(2) PDG_CASE(3) PDG_CASE(4) PDG_CASE(5) PDG_CASE(6) PDG_CASE(7)
#undef PDG_CASE
  }
  return 0;
}

cudaError_t launch_wadg_frag_fill(int N, const double* wadg, double* out, cudaStream_t s) {
  switch (N) {
#define PDG_CASE(n) case n: wadg_frag_kernel<n><<<64, 256, 0, s>>>(wadg, out); return cudaGetLastError();
    PDG_CASE(1) PDG_CASE(2) PDG_CASE(3) PDG_CASE(4) PDG_CASE(5) PDG_CASE(6) PDG_CASE(7)
#undef PDG_CASE
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_wadg_energy(int N, const EnergyParams& p, int* nblocks_out, cudaStream_t s) {
  switch (N) {
#define PDG_CASE(n) case n: return launch_wadg_energy_N<n>(p, nblocks_out, s);
    PDG_CASE(1) PDG_CASE(2) PDG_CASE(3) PDG_CASE(4) PDG_CASE(5) PDG_CASE(6) PDG_CASE(7)
#undef PDG_CASE
  }
  return cudaErrorInvalidValue;
}

} // namespace pdg
