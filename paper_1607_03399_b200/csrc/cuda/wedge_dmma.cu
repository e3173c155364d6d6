// Fused wedge stage kernel on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64).
//
// Work decomposition: a team of T = ceil(NT/8) warps owns one wedge at a time;
// warp w of the team owns the 8-row tile of triangle nodes i in [8w, 8w+8).
// Teams are independent (own TMA pipeline, named barriers), several per CTA.
// Per element and stage the work is a handful of small dense products, all
// issued as 8x8x4 DMMA tiles (rows i, columns j = slices, K as noted):
//   G1  V^T   = -(UX^T (txJ Dt)^T + UY^T (tyJ Dt)^T + tzJ UZ^T Dt^T)   (K = slices)
//   G2  gx    = (rx Dr + sx Ds) P,  gy = (ry Dr + sy Ds) P,
//       dv    = (rx Dr + sx Ds) UX + (ry Dr + sy Ds) UY                (K = tri nodes)
//   G3  [LP | L Fu_bottom | L Fu_top] = L [P | Fu0 | Fu1],  LV = L V     (K = tri nodes)
//   G4  LY    = LP Dt^T   (Dt along slices; A fragments by quad shuffles)
//   G5  qp = sum_f QL_f Fp_f,  qu_f = QL_f Fu_f (normals applied in the epilogue)
// The metric is folded into the A fragments (rx Dr + sx Ds), the bottom/top
// triangular-face pressure lifts are folded into V before G3, and
// the epilogue adds the n-scaled velocity lifts, media scaling and the LSERK45
// stage update res = a res + dt rhs, u = u + b res in shared memory.
//
// Layout for conflict-free fragment loads: L^{tri,k}, the quad lifts, Dr, Ds
// and Dt are stored fragment-major (one 256-byte row per 8x4 fragment, lane
// contiguous), the quad-face fluxes are written fragment-major by the flux
// phase, and V uses a row stride of 4 mod 16 doubles.
//
// Data movement per element (bulk / async, 16-byte granular):
//   TMA loads  (cp.async.bulk -> mbarrier): state, residual, L fragments, quad
//              lift fragments, geometry/media record, connectivity record;
//   gathers    neighbour face traces (LDG, L2-resident thanks to Morton order);
//   stores     updated state and residual straight from the DMMA fragments.
// Each team double-buffers its stage so the next element's loads overlap.
// Reference arithmetic: wedge_volume_elem / surface_elem / scale_media / lserk
// (proj/src/solver.cpp:164-218, 258-335, 337-346, 541-551).
#include <cuda_runtime.h>

#include <cstdlib>

#include "pdg_device.cuh"
#include "tma.cuh"

namespace pdg {

namespace {

__host__ __device__ constexpr int r4(int x) { return (x + 3) & ~3; }
__host__ __device__ constexpr int r2(int x) { return (x + 1) & ~1; }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
/// smallest stride >= x that is 4 or 12 mod 16 (8-byte words): conflict-free
/// for the (row*stride + col) patterns of 8x4 fragment loads
__host__ __device__ constexpr int cf_stride(int x) {
  return (x % 16 == 4 || x % 16 == 12) ? x : cf_stride(x + 1);
}

constexpr int kComboCap = 4096; // ints of neighbour node maps kept in shared memory
#ifndef PDG_WEDGE_STAGES
#define PDG_WEDGE_STAGES 2
#endif
constexpr int kWedgeStages = PDG_WEDGE_STAGES; // per-team TMA pipeline depth (1 or 2)
// compact L / quad lifts (no fragment padding in HBM; A fragments gathered
// from the compact shared-memory copy) instead of fragment-major storage
#ifndef PDG_COMPACT_OPS
#define PDG_COMPACT_OPS 1
#endif
#ifndef PDG_PAD_STATE
#define PDG_PAD_STATE 1
#endif
#ifndef PDG_THREAD_CAP
#define PDG_THREAD_CAP 384
#endif
// no end-of-element team barrier: the flux buffers alternate with the element
// parity and the next element's TMA copy is issued after the flux barrier (when
// every warp of the team has left the previous element), so one barrier per
// element goes
#ifndef PDG_NO_END_BARRIER
#define PDG_NO_END_BARRIER 1
#endif
#ifndef PDG_NOEND_MAX_N
#define PDG_NOEND_MAX_N 5
#endif
// volume products first: the metric-folded gradient / divergence products (G2's
// volume half) and the vertical product of G1 need only the element's own state,
// so they run between issuing the neighbour-trace gathers and using them
#ifndef PDG_VOL_FIRST
#define PDG_VOL_FIRST 1
#endif
// at N = 5 volume-first was +0.4% with bar.sync exchanges (round 1) and is -0.6%
// with the mbarrier exchanges (profiles/round2_mbar_ab.txt)
#ifndef PDG_VF_N5
#define PDG_VF_N5 1
#endif
// k permutation of the triangle products (G2/G3) at odd NT: in every block of four
// k-steps lane (gid, tig) takes k = 16 b + 4 tig + s instead of 4 s + tig, so the
// B reads {slice * stride + k} (odd stride) and the compact-L A reads {k * NT + i}
// hit 16 distinct bank pairs per half-warp instead of 2-way conflicts; the tail
// steps (4 KS not a multiple of 16) keep the contiguous order
#ifndef PDG_KPERM
#define PDG_KPERM 1
#endif

// shared derivative fragments (Dr, Ds of the warp's row tile, Dt) held in
// registers for the whole kernel instead of re-read from shared memory for
// every element (the row tile of a warp never changes): fewer shared-memory
// wavefronts, more registers.  On for N <= PDG_REG_OPS_MAXN.
#ifndef PDG_REG_OPS_MAXN
#define PDG_REG_OPS_MAXN 0
#endif

// per-element serial work spread over the team (N <= 5, no-end-barrier schedule):
// the ticket grab moves to the last warp (the one with the fewest flux tasks)
// and each warp issues its share of the element's bulk copies after the flux
// barrier (one arrive.expect_tx per warp), instead of warp 0 doing both while
// the others wait at the next team barrier
#ifndef PDG_SPLIT_ISSUE
#define PDG_SPLIT_ISSUE 0
#endif

// when a ticket (a batch of consecutive elements) is grabbed, prefetch the
// whole batch's streamed arrays into L2 (cp.async.bulk.prefetch.L2): the
// elements after the next one get their HBM reads in flight early, without
// shared memory or registers, so more bytes are in flight per SM
#ifndef PDG_MEMONLY
#define PDG_MEMONLY 0
#endif
#ifndef PDG_L2_PREFETCH
#define PDG_L2_PREFETCH 0
#endif

// the two per-element team exchanges (fluxes -> products, V -> its lift) through
// mbarriers instead of bar.sync: a warp arrives when its part is written and waits
// only where it reads the others' part.  With the volume products issued first, the
// L [P | Fu0 | Fu1] product and L V run behind the V wait and share their L fragments
// (PDG_MB_LP_LATE: one L read per element), and the quad-face lifts between the V
// arrival and the V wait absorb the warps' skew.  The flux exchange goes through an
// mbarrier where the parity flux buffers allow it (no end-of-element barrier, N <= 5).
// Measured (profiles/round2_mbar_ab.txt): N = 5 -1.7% (exchanges) and -1.1% (shared L),
// N = 4 -1.4% (both), N = 6 -0.5% (V exchange + shared L), N = 7 +2.7% (off).  Rejected
// there and removed after measurement: volume products between the flux arrival and
// wait, late ticket-slot publication, flux-lift dot products / Fu1 in the V padding
// column at N = 6, 7, 16-byte normal loads.
#ifndef PDG_MBAR_SYNC_N4
#define PDG_MBAR_SYNC_N4 1
#endif
#ifndef PDG_MBAR_SYNC_N6
#define PDG_MBAR_SYNC_N6 1
#endif
#ifndef PDG_MBAR_SYNC_N7
#define PDG_MBAR_SYNC_N7 0
#endif
#ifndef PDG_MBAR_SYNC
#define PDG_MBAR_SYNC(N) \
  ((N) == 5 || ((N) == 4 && PDG_MBAR_SYNC_N4) || ((N) == 6 && PDG_MBAR_SYNC_N6) || ((N) == 7 && PDG_MBAR_SYNC_N7))
#endif
#ifndef PDG_MB_LP_LATE
#define PDG_MB_LP_LATE 1
#endif

// LSERK stage: the media factor folded into the stage's dt (pdt kappa, pdt / rho once
// per element) instead of scaling every rhs value (4 FP64 multiplies per output less).
// Measured (profiles/round2_mbar_ab.txt): N = 6 / 7 -0.6 / -0.7% (FP64-pipe throttled),
// N = 5 +0.4%, so from N = 6 on
#ifndef PDG_EPI_FOLD_MIN_N
#define PDG_EPI_FOLD_MIN_N 6
#endif

/// k index of lane column tig in k-step s (see PDG_KPERM)
__host__ __device__ constexpr int kmap(int s, int tig, int KS, bool perm) {
  return (perm && s < 4 * (KS / 4)) ? 16 * (s >> 2) + 4 * tig + (s & 3) : 4 * s + tig;
}

template <int N, int NST_, bool AB3_ = false>
struct DCfg {
  // NP = device per-field block (NQ slices of ST doubles), ST = device slice stride
  static constexpr int NQ = nq_of(N), NT = nt_of(N), NP = npd_of(N), ST = nts_of(N), FW = fw_of(N), WG = wg_of(N);
  static constexpr int IT = it_of(N), KS = ks_of(N), KT = kt_of(N);
  static constexpr int JT = ceil_div(NQ, 8), NPJ = 8 * JT;   // slice column tiles
  static constexpr int JTL = ceil_div(NQ + 2, 8);            // [P | Fu0 | Fu1] tiles
  static constexpr int T = IT;                               // warps per team
  // per-wedge operator block sizes in HBM / the stage buffer
  static constexpr int LF = PDG_COMPACT_OPS ? lcomp_of(N) : lfrag_of(N);
  static constexpr int QF = PDG_COMPACT_OPS ? qcomp_of(N) : qfrag_of(N);
  // per-stage buffers (doubles), 16-byte aligned
  static constexpr int USTR = r4(4 * NP) + 2;
  // AB3 mode: the residual slot holds f_{n-1}, a second slot after the records f_{n-2}
  static constexpr int STAGE = r2(2 * USTR + LF + QF + WG + kWC / 2 + (AB3_ ? USTR : 0));
  // work buffers
  static constexpr bool KP = PDG_KPERM && (NT & 1) && ST == NT; // permuted k (odd slice stride)
  static constexpr int VST = KP ? NT : cf_stride(NT);        // V row stride (odd with KP)
  static constexpr int VS = r2((NPJ - 1) * VST + 4 * KS + 8);
  static constexpr int FQ = 3 * JT * KT * 32;                // fragment-major quad fluxes
  static constexpr int FTRI = r2(4 * KS + NT + 8);           // bottom/top tri fluxes (+ padding)
  static constexpr int ZS = r2(4 * KS);                      // zero column for padded B reads
  // padded copy of the state for bank-conflict-free fragment loads when NT is
  // not 4 or 12 mod 16 (row = field*NQ + slice, stride SP)
  // measured: N = 4 3.93 vs 4.22 ms, N = 5 6.55 vs 6.31 ms (profiles/round1_pad_state_ab.txt)
  static constexpr bool PAD = PDG_PAD_STATE && cf_stride(NT) != NT && N == 4 && !KP;
  static constexpr int SP = PAD ? cf_stride(NT) : ST;
  static constexpr int UPS = PAD ? r2((4 * NQ + 8 * JT + 4 * KT) * SP + 4 * KS + 8) : 0;
  static constexpr int FB = 2 * (FTRI + FQ);                 // one set of flux buffers
  // measured (profiles/round1_noend_ab.txt): N = 4 -0.5%, N = 5 -1.5%, N = 6 even,
  // N = 7 +6% (shorter prefetch lead), so on at N <= 5 only
  static constexpr int FBUF = (PDG_NO_END_BARRIER && !PAD && NST_ == 2 && N <= PDG_NOEND_MAX_N) ? 2 : 1;
  static constexpr int WORK = VS + FBUF * FB + ZS + UPS;
  static constexpr int TABLES = r2(2 * IT * KS * 32 + JT * KT * 32 + 2 * NQ + ceil_div(FW, 2) + kComboCap / 2);
  static constexpr int SMEM_BUDGET = 225 * 1024;
  // double-buffered stages unless even a single team would not fit
  // team header: 2 stage mbarriers + 3 schedule slots (+ 2 exchange mbarriers)
  static constexpr int HDR = PDG_MBAR_SYNC(N) ? 8 : 6;
  static constexpr int NSTAGE = (NST_ == 2 && (TABLES + HDR + 2 * STAGE + WORK) * 8 <= SMEM_BUDGET) ? 2 : 1;
  static constexpr int PER_TEAM = HDR + NSTAGE * STAGE + WORK;
  static constexpr bool NOEND = FBUF == 2 && NSTAGE == 2;
  // mbarrier exchanges need the parity flux buffers (no end-of-element barrier)
  // (the V exchange is safe with or without the end-of-element barrier: V of the next
  // element is written only after its flux exchange, i.e. after every warp has left
  // this one; the flux exchange needs the parity flux buffers)
  static constexpr bool MB = PDG_MBAR_SYNC(N) && !PDG_SPLIT_ISSUE; // V exchange
  static constexpr bool MBF = MB && NOEND;                          // flux exchange
  // measured (profiles/round1_volfirst_ab.txt): N = 4 -2.8%, N = 6 -4.5%, N = 7 -6.5%,
  // N = 5 +0.4% before the mbarrier exchanges, -0.6% with them (PDG_VF_N5)
  static constexpr bool VF = PDG_VOL_FIRST && (N != 5 || PDG_VF_N5);
  static constexpr bool VP = VF;                            // volume products outside G1 / G2
  static constexpr bool LPL = PDG_MB_LP_LATE && MB && VP;   // L [P | Fu0 | Fu1] behind the V wait
  static constexpr int TPB_SMEM = (SMEM_BUDGET / 8 - TABLES) / PER_TEAM;
  // <= PDG_THREAD_CAP threads per CTA: 384 keeps >= 168 registers per thread
  // (profiles/round1_compact_ops_ab.txt: compact operators + 384 beat 512)
  static constexpr int TPB = cmax(1, cmin(cmin(15, PDG_THREAD_CAP / (32 * T)), TPB_SMEM)); // teams per CTA
  static constexpr int THREADS = 32 * T * TPB;
  static constexpr size_t SMEM_BYTES = (size_t)8 * (TABLES + TPB * PER_TEAM);
  static constexpr int QF_LANE = ceil_div(FW, 32 * T); // face nodes per team thread
  static constexpr int QB = cmin(QF_LANE, 4);          // gathered per batch
};

/// elements per ticket: batching cuts same-address atomics (the global work
/// counter) at low N, where an element is only a few hundred cycles of work
inline int ticket_batch(int N) {
  static const int env = [] {
    const char* v = std::getenv("PDG_TICKET_BATCH");
    return v ? std::atoi(v) : 0;
  }();
  if (env > 0) return env;
  // measured sweeps, round 1 (profiles/round1_ticket_batch.txt; after the schedule
  // changes N = 4 prefers 4: profiles/round1_ticket_batch2.txt)
  // N = 7: one element per ticket, -0.8% after the round-2 schedule changes (profiles/round2_mbar_ab.txt)
  return N <= 3 ? 8 : (N == 4 ? 4 : (N >= 7 ? 1 : 2));
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void team_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int N, int NST, bool AB3 = false>
__device__ __forceinline__ void load_element(const StageParams& p, double* stg, long long e, const double* res_src,
                                             uint64_t* bar) {
  using C = DCfg<N, NST, AB3>;
  constexpr int NP = C::NP;
  double* U = stg;
  double* R = U + C::USTR;
  double* L = R + C::USTR;
  double* Q = L + C::LF;
  double* G = Q + C::QF;
  const uint32_t bytes = 8u * (4 * NP + C::LF + C::QF + C::WG) + 4u * kWC + (res_src ? 32u * NP : 0u) +
                         (AB3 ? 32u * NP : 0u);
  // the state stays in L2 for the neighbours' trace gathers of this stage;
  // everything else is touched once
  const uint64_t keep = l2_policy_evict_last(), stream = l2_policy_evict_first();
  mbar_arrive_expect_tx(bar, bytes);
  tma_load_1d_hint(U, p.u_in + e * 4 * NP, 32 * NP, bar, keep);
  if (res_src) tma_load_1d_hint(R, res_src + e * 4 * NP, 32 * NP, bar, stream);
  tma_load_1d_hint(L, p.Lt + e * C::LF, 8 * C::LF, bar, stream);
  tma_load_1d_hint(Q, p.QL + e * C::QF, 8 * C::QF, bar, stream);
  tma_load_1d_hint(G, p.wgeo + e * C::WG, 8 * C::WG, bar, stream);
  tma_load_1d_hint(G + C::WG, p.wconn + e * kWC, 4 * kWC, bar, stream);
  if (AB3) tma_load_1d_hint(G + C::WG + kWC / 2, p.h2 + e * 4 * NP, 32 * NP, bar, stream);
}

/// warp `part` of T issues copies c = part, part + T, ... of the element's
/// state / residual / L / quad lifts / record / connectivity, with its own
/// arrive.expect_tx (the barrier counts T arrivals)
template <int N, int NST>
__device__ __forceinline__ void load_element_part(const StageParams& p, double* stg, long long e,
                                                  const double* res_src, uint64_t* bar, int part) {
  constexpr int T = DCfg<N, NST>::T;
  using C = DCfg<N, NST>;
  constexpr int NP = C::NP;
  double* U = stg;
  double* R = U + C::USTR;
  double* L = R + C::USTR;
  double* Q = L + C::LF;
  double* G = Q + C::QF;
  auto size_of = [&](int c) -> uint32_t {
    return c == 0 ? 32u * NP : c == 1 ? (res_src ? 32u * NP : 0u) : c == 2 ? 8u * C::LF
         : c == 3 ? 8u * C::QF : c == 4 ? 8u * C::WG : 4u * kWC;
  };
  uint32_t bytes = 0;
#pragma unroll
  for (int c = 0; c < 6; ++c)
    if (c % T == part) bytes += size_of(c);
  const uint64_t keep = l2_policy_evict_last(), stream = l2_policy_evict_first();
  mbar_arrive_expect_tx(bar, bytes);
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    if (c % T != part) continue;
    if (c == 0) tma_load_1d_hint(U, p.u_in + e * 4 * NP, size_of(0), bar, keep);
    if (c == 1 && res_src) tma_load_1d_hint(R, res_src + e * 4 * NP, size_of(1), bar, stream);
    if (c == 2) tma_load_1d_hint(L, p.Lt + e * C::LF, size_of(2), bar, stream);
    if (c == 3) tma_load_1d_hint(Q, p.QL + e * C::QF, size_of(3), bar, stream);
    if (c == 4) tma_load_1d_hint(G, p.wgeo + e * C::WG, size_of(4), bar, stream);
    if (c == 5) tma_load_1d_hint(G + C::WG, p.wconn + e * kWC, size_of(5), bar, stream);
  }
}

template <int N, bool COMBO_SMEM, bool FUSED, int NST, bool AB3 = false>
__global__ void __launch_bounds__(DCfg<N, NST, AB3>::THREADS, 1) wedge_dmma_kernel(const StageParams p) {
  using C = DCfg<N, NST, AB3>;
  constexpr int NQ = C::NQ, NT = C::NT, NP = C::NP, ST = C::ST, FW = C::FW, WG = C::WG, T = C::T;
  constexpr int KS = C::KS, JT = C::JT, JTL = C::JTL, KT = C::KT, VST = C::VST, TPB = C::TPB;
  constexpr int QL_ = C::QF_LANE;
  extern __shared__ __align__(16) double smem[];

  // ---- shared reference tables (fragment-major, zero padded) ----------------
  double* sDr = smem;                        // [t][s][lane] = Dr(8t+gid, kmap(s, tig))
  double* sDs = sDr + C::IT * KS * 32;
  double* sDt = sDs + C::IT * KS * 32;       // [jt][s][lane] = Dt(8jt+gid, 4s+tig)
  double* sProf = sDt + JT * KT * 32;        // [2][NQ]
  int* sWface = reinterpret_cast<int*>(sProf + 2 * NQ);
  int* sCombo = sWface + 2 * ceil_div(FW, 2);
  for (int q = threadIdx.x; q < (int)(C::SMEM_BYTES / 8); q += C::THREADS) smem[q] = 0.0;
  __syncthreads();
  for (int q = threadIdx.x; q < C::IT * KS * 32; q += C::THREADS) {
    const int lane = q & 31, ts = q >> 5, t = ts / KS, s = ts - t * KS;
    const int i = 8 * t + (lane >> 2), k = kmap(s, lane & 3, KS, C::KP);
    if (i < NT && k < NT) {
      sDr[q] = p.DrT[k * NT + i];
      sDs[q] = p.DsT[k * NT + i];
    }
  }
  for (int q = threadIdx.x; q < JT * KT * 32; q += C::THREADS) {
    const int lane = q & 31, js = q >> 5, jt = js / KT, s = js - jt * KT;
    const int j = 8 * jt + (lane >> 2), l = 4 * s + (lane & 3);
    if (j < NQ && l < NQ) sDt[q] = p.Dt[j * NQ + l];
  }
  for (int q = threadIdx.x; q < 2 * NQ; q += C::THREADS) sProf[q] = p.prof[q];
  for (int q = threadIdx.x; q < FW; q += C::THREADS) sWface[q] = p.wface_dev[q];
  if (COMBO_SMEM)
    for (int q = threadIdx.x; q < p.nbr_nodes_len; q += C::THREADS) sCombo[q] = p.nbr_nodes[q];

  const int team = threadIdx.x / (32 * T);
  const int tt = threadIdx.x - team * 32 * T; // thread within team
  const int w = tt >> 5, lane = tt & 31;      // warp within team = row tile
  const int gid = lane >> 2, tig = lane & 3;
  const int bar_id = 1 + team;
  double* tbase = smem + C::TABLES + (size_t)team * C::PER_TEAM;
  uint64_t* bar = reinterpret_cast<uint64_t*>(tbase);
  double* stg0 = tbase + C::HDR; // 2 mbarriers + 3 schedule slots (+ 2 exchange mbarriers) + pad
  uint64_t* fbar = bar + 5;      // C::MBF: flux exchange
  uint64_t* vbar = bar + 6;      // C::MB: V exchange
  double* V = stg0 + NST * C::STAGE;
  double* const Fbase = V + C::VS; // C::FBUF sets of flux buffers (element parity)
  const double* Zero = Fbase + C::FBUF * C::FB; // ZS zeros, never written
  double* Upad = Fbase + C::FBUF * C::FB + C::ZS; // padded state copy (C::PAD)
  constexpr int SP = C::SP;
  constexpr bool SPLIT = PDG_SPLIT_ISSUE && C::NOEND;
  const bool grabber = SPLIT ? tt == 32 * (T - 1) : tt == 0; // thread that owns the ticket state
  if (tt == 0) {
    mbar_init(bar, SPLIT ? T : 1);
    mbar_init(bar + 1, SPLIT ? T : 1);
    if (C::MB) {
      mbar_init(fbar, 32 * T);
      mbar_init(vbar, 32 * T);
    }
    fence_barrier_init();
  }
  __syncthreads();

  constexpr bool RO = N <= PDG_REG_OPS_MAXN;
  double rDr[RO ? KS : 1], rDs[RO ? KS : 1], rDt[RO ? JT : 1][RO ? KT : 1];
  if (RO) {
#pragma unroll
    for (int s2 = 0; s2 < (RO ? KS : 1); ++s2) {
      rDr[s2] = sDr[((w * KS + s2) << 5) + lane];
      rDs[s2] = sDs[((w * KS + s2) << 5) + lane];
    }
#pragma unroll
    for (int jt = 0; jt < (RO ? JT : 1); ++jt)
#pragma unroll
      for (int s2 = 0; s2 < (RO ? KT : 1); ++s2) rDt[jt][s2] = sDt[((jt * KT + s2) << 5) + lane];
  }
  auto dr_of = [&](int s2) { return RO ? rDr[RO ? s2 : 0] : sDr[((w * KS + s2) << 5) + lane]; };
  auto ds_of = [&](int s2) { return RO ? rDs[RO ? s2 : 0] : sDs[((w * KS + s2) << 5) + lane]; };
  auto dt_of = [&](int jt, int s2) { return RO ? rDt[RO ? jt : 0][RO ? s2 : 0] : sDt[((jt * KT + s2) << 5) + lane]; };

  // ---- per-thread face-node tasks, fixed for the whole kernel -----------------
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
  // PDG_MEMONLY (measurement only, never a product build): all arithmetic off,
  // the same bulk copies, gathers-free, barriers and streaming stores -- the
  // memory-side floor of this pipeline structure
  const bool vol = !PDG_MEMONLY && (FUSED || (mode & M_VOLUME)),
             surf = !PDG_MEMONLY && (FUSED || (mode & M_SURFACE));
  const bool lserk = FUSED || (mode & M_LSERK), media = FUSED || (mode & M_MEDIA);
  const bool first = mode & M_FIRST, accum = !FUSED && (mode & M_ACCUM);
  const double* res_src = AB3 ? p.h1 : (lserk ? (first ? nullptr : p.res) : (accum ? p.rhs_out : nullptr));
  // dynamic scheduling keeps all teams on a narrow, L2-resident window of the
  // (Morton-ordered) element list, so neighbour traces hit in L2
  volatile long long* slot = reinterpret_cast<volatile long long*>(bar + 2);
  // tickets hand out batches of B consecutive elements (thread 0 of the team
  // keeps the current batch); one failing grab per team ends its loop
  const int B = p.ticket_batch;
  long long bnext = 0, bend = 0;
  auto grab = [&]() -> long long {
    if (bnext >= bend) {
      bnext = p.Kw_begin + (long long)(atomicAdd(p.ticket, (unsigned long long)B) - p.ticket_base);
      bend = bnext + B < p.Kw_active ? bnext + B : (bnext < p.Kw_active ? p.Kw_active : bnext + 1);
      if (PDG_L2_PREFETCH && bnext < p.Kw_active) {
        // the batch [bnext, bend) is contiguous in every streamed array
        const long long nb = bend - bnext;
        prefetch_l2_bulk(p.u_in + bnext * 4 * NP, (uint32_t)(nb * 32 * NP));
        if (res_src) prefetch_l2_bulk(res_src + bnext * 4 * NP, (uint32_t)(nb * 32 * NP));
        prefetch_l2_bulk(p.Lt + bnext * C::LF, (uint32_t)(nb * 8 * C::LF));
        prefetch_l2_bulk(p.QL + bnext * C::QF, (uint32_t)(nb * 8 * C::QF));
        prefetch_l2_bulk(p.wgeo + bnext * C::WG, (uint32_t)(nb * 8 * C::WG));
      }
    }
    return bnext++;
  };
  if (grabber) {
    const long long e0 = grab();
    slot[0] = e0;
    if (!SPLIT && e0 < p.Kw_active) load_element<N, NST, AB3>(p, stg0, e0, res_src, bar);
  }
  team_sync(bar_id, 32 * T);
  long long e = slot[0];
  if (SPLIT && lane == 0 && e < p.Kw_active) load_element_part<N, NST>(p, stg0, e, res_src, bar, w);

  // neighbour traces of this thread's face-node tasks (prefetching the next
  // element's during this element's products was measured slower: it exposes
  // the next stage's TMA wait, profiles/round1_gather_prefetch_ab.txt)
  double nb[QL_][4];
  auto gather = [&](const int* Cg) {
#pragma unroll
    for (int q = 0; q < QL_; ++q) {
      const int f = task_f[q];
      if (f >= 0) {
        const int nbr = Cg[2 * f];
        if (nbr >= 0) {
          const int mi = Cg[2 * f + 1] * p.max_nfp + task_loc[q];
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
  };

  for (int n = 0; e < p.Kw_active; ++n) {
    const int s = NST == 2 ? (n & 1) : 0;
    long long en = 0;
    if (grabber) {
      en = grab();
      slot[1 + (n & 1)] = en; // parity slots: rewritten only after every thread read it
    }
    const double* U = stg0 + s * C::STAGE;
    const double* R = U + C::USTR;
    const double* Lf = R + C::USTR;
    const double* Qf = Lf + C::LF;
    const double* G = Qf + C::QF;
    const int* Cn = reinterpret_cast<const int*>(G + WG);
    double* Ftp = Fbase + (C::NOEND ? (n & 1) * C::FB : 0); // tri-face fluxes: p part [2][NT]
    double* Ftu = Ftp + C::FTRI;                              //                  u part
    double* Fqp = Ftu + C::FTRI; // quad-face fluxes, fragment-major [f][jt][s][lane]
    double* Fqu = Fqp + C::FQ;
    if (NST == 2 && !C::NOEND && tt == 0 && en < p.Kw_active) {
      fence_proxy_async_smem();
      load_element<N, NST, AB3>(p, stg0 + (s ^ 1) * C::STAGE, en, res_src, bar + (s ^ 1));
    }
    mbar_wait(bar + s, NST == 2 ? ((n >> 1) & 1) : (n & 1));

    // ---- padded state copy (published by the flux barrier) ----------------------
    if (C::PAD)
      for (int q = tt; q < 4 * NP; q += 32 * T) {
        const int row = q / ST, col = q - row * ST;
        if (col < NT) Upad[row * SP + col] = U[q];
      }
    const double* Us = C::PAD ? Upad : U; // state with row stride SP

    // ---- volume products (C::VF): only the state, while the gathers are in flight
    double gx[JT][2], gy[JT][2], dvx[JT][2], dvy[JT][2], dg1[JT][2];
#pragma unroll
    for (int jt = 0; jt < JT; ++jt)
#pragma unroll
      for (int c = 0; c < 2; ++c) gx[jt][c] = gy[jt][c] = dvx[jt][c] = dvy[jt][c] = dg1[jt][c] = 0.0;
    auto volume_products = [&]() {
      if (vol) {
        const int i = 8 * w + gid;
        const double tzJ = G[W_TZJ];
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) {
          const int jb = 8 * jt + gid;
          const int jc = jb < NQ ? jb : NQ - 1;
          const double sx_ = G[W_TXJ + jc], sy_ = G[w_tyj(N) + jc];
#pragma unroll
          for (int s2 = 0; s2 < KT; ++s2) {
            const int l = 4 * s2 + tig;
            const double bd = dt_of(jt, s2);
            dmma(dg1[jt], Us[(NQ + l) * SP + i], sx_ * bd);
            dmma(dg1[jt], Us[(2 * NQ + l) * SP + i], sy_ * bd);
            dmma(dg1[jt], Us[(3 * NQ + l) * SP + i], tzJ * bd);
          }
        }
        const double rx = G[W_RX], ry = G[W_RY], sxm = G[W_SX], sym = G[W_SY];
#pragma unroll
        for (int s2 = 0; s2 < KS; ++s2) {
          const int k = kmap(s2, tig, KS, C::KP);
          const double dr = dr_of(s2), ds = ds_of(s2);
          const double cx = rx * dr + sxm * ds, cy = ry * dr + sym * ds;
#pragma unroll
          for (int jt = 0; jt < JT; ++jt) {
            const int jb = 8 * jt + gid;
            const double bp = jb < NQ ? Us[jb * SP + k] : 0.0; // padding columns are discarded
            dmma(gx[jt], cx, bp);
            dmma(gy[jt], cy, bp);
            dmma(dvx[jt], cx, Us[(NQ + jb) * SP + k]);
            dmma(dvy[jt], cy, Us[(2 * NQ + jb) * SP + k]);
          }
        }
      }
    };
    if (C::VF) {
      if (surf) gather(Cn);
      volume_products();
    }

    // ---- numerical fluxes on all face nodes -------------------------------------
    if (surf) {
      if (!C::VF) gather(Cn);
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
    if (C::MBF) {
      mbar_arrive(fbar);
      mbar_wait(fbar, n & 1);
    } else {
      team_sync(bar_id, 32 * T);
    }
    // every warp of the team has left the previous element: its stage may be refilled
    if (C::NOEND && !SPLIT && tt == 0 && en < p.Kw_active) {
      fence_proxy_async_smem();
      load_element<N, NST, AB3>(p, stg0 + (s ^ 1) * C::STAGE, en, res_src, bar + (s ^ 1));
    }
    if (SPLIT && lane == 0) {
      const long long enx = slot[1 + (n & 1)]; // written before the flux barrier by the grabber
      if (enx < p.Kw_active) {
        fence_proxy_async_smem();
        load_element_part<N, NST>(p, stg0 + (s ^ 1) * C::STAGE, enx, res_src, bar + (s ^ 1), w);
      }
    }

    // ---- G1: V[j][i] for row tile w, with the bottom/top pressure lifts folded in
    {
      const int i = 8 * w + gid;
      const double tzJ = G[W_TZJ], jfb = G[W_JFB], jft = G[W_JFT];
      const double fb = surf ? jfb * Ftp[i] : 0.0, ftop = surf ? jft * Ftp[NT + i] : 0.0;
#pragma unroll
      for (int jt = 0; jt < JT; ++jt) {
        double d[2] = {dg1[jt][0], dg1[jt][1]};
        if (vol && !C::VP) {
          const int jb = 8 * jt + gid;
          const int jc = jb < NQ ? jb : NQ - 1;
          const double sx_ = G[W_TXJ + jc], sy_ = G[w_tyj(N) + jc];
#pragma unroll
          for (int s2 = 0; s2 < KT; ++s2) {
            const int l = 4 * s2 + tig;
            const double bd = dt_of(jt, s2);
            dmma(d, Us[(NQ + l) * SP + i], sx_ * bd);
            dmma(d, Us[(2 * NQ + l) * SP + i], sy_ * bd);
            dmma(d, Us[(3 * NQ + l) * SP + i], tzJ * bd);
          }
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int j = 8 * jt + 2 * tig + c;
          if (i < NT && j < NQ) V[j * VST + i] = -d[c] + fb * sProf[j] + ftop * sProf[NQ + j];
        }
      }
    }
    if (C::MB)
      mbar_arrive(vbar); // L V waits for it after the V-independent products
    else
      team_sync(bar_id, 32 * T);

    // ---- row tile w: G2, G3, G4, G5 and the epilogue ---------------------------
    {
      const int t = w;
      const int i = 8 * t + gid;
      const double rx = G[W_RX], ry = G[W_RY], sxm = G[W_SX], sym = G[W_SY];
      const double* src[JTL]; // B column sources of the [P | Fu0 | Fu1] operand
#pragma unroll
      for (int jt = 0; jt < JTL; ++jt) {
        const int nc = 8 * jt + gid;
        src[jt] = nc < NQ ? Us + nc * SP : (nc == NQ ? Ftu : (nc == NQ + 1 ? Ftu + NT : Zero));
      }
      double lv[JT][2], lp[JTL][2];
#pragma unroll
      for (int jt = 0; jt < JT; ++jt) lv[jt][0] = lv[jt][1] = 0.0;
#pragma unroll
      for (int jt = 0; jt < JTL; ++jt) lp[jt][0] = lp[jt][1] = 0.0;
#pragma unroll
      for (int s2 = 0; s2 < (C::LPL ? 0 : KS); ++s2) {
        const int k = kmap(s2, tig, KS, C::KP);
        const int fo = ((t * KS + s2) << 5) + lane;
#if PDG_COMPACT_OPS
        const double la = (i < NT && k < NT) ? Lf[k * NT + i] : 0.0;
#else
        const double la = Lf[fo];
#endif
        double cx = 0.0, cy = 0.0;
        if (vol && !C::VP) {
          const double dr = dr_of(s2), ds = ds_of(s2);
          cx = rx * dr + sxm * ds;
          cy = ry * dr + sym * ds;
        }
#pragma unroll
        for (int jt = 0; jt < JTL; ++jt) {
          const double bp = src[jt][k];
          if (!PDG_MEMONLY) dmma(lp[jt], la, bp);
          if (jt < JT) {
            const int jb = 8 * jt + gid;
            if (vol && !C::VP) {
              dmma(gx[jt], cx, bp);
              dmma(gy[jt], cy, bp);
              dmma(dvx[jt], cx, Us[(NQ + jb) * SP + k]);
              dmma(dvy[jt], cy, Us[(2 * NQ + jb) * SP + k]);
            }
            if (!PDG_MEMONLY && !C::MB) dmma(lv[jt], la, V[jb * VST + k]);
          }
        }
      }
      // G4: LY = LP Dt^T, A fragments of LP gathered within each lane quad
      double ly[JT][2], lf0 = 0.0, lf1 = 0.0;
      auto finish_lp = [&]() {
#pragma unroll
      for (int jt = 0; jt < JT; ++jt) ly[jt][0] = ly[jt][1] = 0.0;
      if (vol) {
#pragma unroll
        for (int s2 = 0; s2 < KT; ++s2) {
          const int srcl = gid * 4 + 2 * (s2 & 1) + (tig >> 1);
          const double v0 = __shfl_sync(0xffffffffu, lp[s2 >> 1][0], srcl);
          const double v1 = __shfl_sync(0xffffffffu, lp[s2 >> 1][1], srcl);
          const double a = (tig & 1) ? v1 : v0;
#pragma unroll
          for (int jt = 0; jt < JT; ++jt) dmma(ly[jt], a, dt_of(jt, s2));
        }
      }
      // L fu_bottom, L fu_top of this row (columns NQ, NQ+1 of the G3 product)
      constexpr int c0 = NQ % 8, c1 = (NQ + 1) % 8;
      lf0 = __shfl_sync(0xffffffffu, lp[NQ / 8][c0 & 1], gid * 4 + c0 / 2);
      lf1 = __shfl_sync(0xffffffffu, lp[(NQ + 1) / 8][c1 & 1], gid * 4 + c1 / 2);
      };
      if (!C::LPL) finish_lp();
      // G5: quad-face lifts; the velocity lift of each face is kept separately
      // and scaled by that face's normal in the epilogue
      double qp[JT][2], qu[3][JT][2];
#pragma unroll
      for (int jt = 0; jt < JT; ++jt)
#pragma unroll
        for (int c = 0; c < 2; ++c) qp[jt][c] = qu[0][jt][c] = qu[1][jt][c] = qu[2][jt][c] = 0.0;
      const double* nrm = G + w_nrm(N);
      if (surf) {
#pragma unroll
        for (int f = 0; f < 3; ++f)
#pragma unroll
          for (int s2 = 0; s2 < KT; ++s2) {
#if PDG_COMPACT_OPS
            const int qa_a = 4 * s2 + tig;
            const double qa = (i < NT && qa_a < NQ) ? Qf[(f * NQ + qa_a) * NT + i] : 0.0;
#else
            const double qa = Qf[(((t * 3 + f) * KT + s2) << 5) + lane];
#endif
#pragma unroll
            for (int jt = 0; jt < JT; ++jt) {
              const int fo = (((f * JT + jt) * KT + s2) << 5) + lane;
              dmma(qp[jt], qa, Fqp[fo]);
              dmma(qu[f][jt], qa, Fqu[fo]);
            }
          }
      }
      if (C::MB) mbar_wait(vbar, n & 1); // every warp's V rows (and the next element index) are in
      if (C::MB && !PDG_MEMONLY) {
        // L V
#pragma unroll
        for (int s2 = 0; s2 < KS; ++s2) {
          const int k = kmap(s2, tig, KS, C::KP);
#if PDG_COMPACT_OPS
          const double la = (i < NT && k < NT) ? Lf[k * NT + i] : 0.0;
#else
          const double la = Lf[((t * KS + s2) << 5) + lane];
#endif
#pragma unroll
          for (int jt = 0; jt < JT; ++jt) dmma(lv[jt], la, V[(8 * jt + gid) * VST + k]);
          if (C::LPL) {
#pragma unroll
            for (int jt = 0; jt < JTL; ++jt) dmma(lp[jt], la, src[jt][k]);
          }
        }
      }
      if (C::LPL) finish_lp();
      // epilogue: rows i, columns j = 8 jt + 2 tig + c; results straight to HBM
      const double tzJ = G[W_TZJ], jfb = G[W_JFB], jft = G[W_JFT];
      const double kappa = G[W_KAPPA], irho = G[W_IRHO];
      const double pa = p.a, pb = p.b, pdt = p.dt;
      double n_[5][3];
#pragma unroll
      for (int f = 0; f < 5; ++f)
#pragma unroll
        for (int a = 0; a < 3; ++a) n_[f][a] = nrm[3 * f + a];
      // per-lane base offset of position (i, j = 2 tig); (jt, c, field) add constants
      const int lane_off = 2 * tig * ST + i;
      const double* Ul = Us + 2 * tig * SP + i; // padded rows: (field*NQ + j)*SP + i
      const double* Rl = R + lane_off;
      const double* F2l = G + WG + kWC / 2 + lane_off; // AB3: f_{n-2} (stage slot after the records)
      const long long gofs = e * 4 * NP + lane_off;
      double* resl = p.res + gofs;
      double* uol = p.u_out + gofs;
      double* rhsl = p.rhs_out + gofs;
#pragma unroll
      for (int jt = 0; jt < JT; ++jt)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int j = 8 * jt + 2 * tig + c;
          if (i < NT && j < NQ) {
            double rp = lv[jt][c], rux = 0.0, ruy = 0.0, ruz = 0.0;
            if (vol) {
              rp -= dvx[jt][c] + dvy[jt][c];
              rux = -(G[W_TXJ + j] * ly[jt][c] + gx[jt][c]);
              ruy = -(G[w_tyj(N) + j] * ly[jt][c] + gy[jt][c]);
              ruz = -(tzJ * ly[jt][c]);
            }
            if (surf) {
              const double t0 = jfb * sProf[j] * lf0, t1 = jft * sProf[NQ + j] * lf1;
              const double u2 = qu[0][jt][c], u3 = qu[1][jt][c], u4 = qu[2][jt][c];
              rp += qp[jt][c];
              rux += n_[0][0] * t0 + n_[1][0] * t1 + n_[2][0] * u2 + n_[3][0] * u3 + n_[4][0] * u4;
              ruy += n_[0][1] * t0 + n_[1][1] * t1 + n_[2][1] * u2 + n_[3][1] * u3 + n_[4][1] * u4;
              ruz += n_[0][2] * t0 + n_[1][2] * t1 + n_[2][2] * u2 + n_[3][2] * u3 + n_[4][2] * u4;
            }
            constexpr bool FOLD = N >= PDG_EPI_FOLD_MIN_N && !AB3;
            const bool fold = FOLD && lserk;
            if (media && !fold) {
              rp *= kappa;
              rux *= irho;
              ruy *= irho;
              ruz *= irho;
            }
            const double rv[4] = {rp, rux, ruy, ruz};
            const double sk = media ? pdt * kappa : pdt, si = media ? pdt * irho : pdt; // fold: per-field dt
            constexpr int cst[2] = {0, ST};
            constexpr int csp[2] = {0, SP};
#pragma unroll
            for (int f = 0; f < 4; ++f) {
              const int o = f * NP + 8 * jt * ST + cst[c];
              const int ou = (f * NQ + 8 * jt) * SP + csp[c];
              if (AB3) {
                // f_n to the history slot; u_{n+1} = u_n + dt/12 (23 f_n - 16 f_{n-1} + 5 f_{n-2})
                // with pdt = dt/12 and the update kernel's operation order (bitwise equal)
                __stcs(rhsl + o, rv[f]);
                __stcs(uol + o, Ul[ou] + pdt * (23.0 * rv[f] - 16.0 * Rl[o] + 5.0 * F2l[o]));
              } else if (lserk) {
                const double sc = fold ? (f == 0 ? sk : si) : pdt;
                const double rr = first ? sc * rv[f] : pa * Rl[o] + sc * rv[f];
                __stcs(resl + o, rr); // streaming stores: evict first
                __stcs(uol + o, Ul[ou] + pb * rr);
              } else {
                __stcs(rhsl + o, accum ? Rl[o] + rv[f] : rv[f]);
              }
            }
          }
        }
    }
    if (!C::NOEND) team_sync(bar_id, 32 * T); // stage s and the work buffers are free again
    if (NST == 1 && tt == 0 && en < p.Kw_active) load_element<N, NST, AB3>(p, stg0, en, res_src, bar);
    e = slot[1 + (n & 1)];
  }
}

template <int N, bool CS, bool FUSED, int NST, bool AB3 = false>
cudaError_t launch_dmma_NC(const StageParams& p, cudaStream_t s) {
  using C = DCfg<N, NST, AB3>;
  // one-time setup per device (the smem attribute is per device)
  static int grid_cap[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  auto kern = wedge_dmma_kernel<N, CS, FUSED, C::NSTAGE, AB3>;
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

template <int N>
cudaError_t launch_dmma_N(const StageParams& p, cudaStream_t s) {
  constexpr int F = M_VOLUME | M_SURFACE | M_MEDIA | M_LSERK;
  const bool fused = (p.mode & F) == F && !(p.mode & M_ACCUM);
  const bool cs = p.nbr_nodes_len <= kComboCap;
  static const int stages = [] {
    const char* v = std::getenv("PDG_WEDGE_STAGES");
    return (v && v[0] == '1') ? 1 : kWedgeStages;
  }();
  if (p.mode & M_AB3) {
    if constexpr (N >= 4 && N <= 7)
      return cs ? launch_dmma_NC<N, true, false, 2, true>(p, s) : launch_dmma_NC<N, false, false, 2, true>(p, s);
    return cudaErrorInvalidValue;
  }
  if (stages == 1) {
    if (fused) return cs ? launch_dmma_NC<N, true, true, 1>(p, s) : launch_dmma_NC<N, false, true, 1>(p, s);
    return cs ? launch_dmma_NC<N, true, false, 1>(p, s) : launch_dmma_NC<N, false, false, 1>(p, s);
  }
  if (fused) return cs ? launch_dmma_NC<N, true, true, 2>(p, s) : launch_dmma_NC<N, false, true, 2>(p, s);
  return cs ? launch_dmma_NC<N, true, false, 2>(p, s) : launch_dmma_NC<N, false, false, 2>(p, s);
}

} // namespace

cudaError_t launch_wedge_stage(int N, const StageParams& p, cudaStream_t s) {
  switch (N) {
#define PDG_CASE(n) case n: return launch_dmma_N<n>(p, s);
    PDG_CASE(1) PDG_CASE(2) PDG_CASE(3) PDG_CASE(4) PDG_CASE(5) PDG_CASE(6) PDG_CASE(7)
    PDG_CASE(8) PDG_CASE(9)
#undef PDG_CASE
  }
  return cudaErrorInvalidValue;
}

bool wedge_dmma_compact_ops() { return PDG_COMPACT_OPS != 0; }

bool wedge_stage_ab3_supported(int N) { return N >= 4 && N <= 7; }

int wedge_elems_per_block(int N) {
  switch (N) {
#define PDG_CASE(n) case n: return DCfg<n, kWedgeStages>::TPB;
    PDG_CASE(1) PDG_CASE(2) PDG_CASE(3) PDG_CASE(4) PDG_CASE(5) PDG_CASE(6) PDG_CASE(7)
    PDG_CASE(8) PDG_CASE(9)
#undef PDG_CASE
  }
  return 0;
}

} // namespace pdg
