// Fused tetrahedron stage kernel on the FP64 tensor cores (DMMA m8n8k4):
// volume + surface + media + LSERK45 update for batches of 8 tets.
//
// Tets are affine, so every operator is shared and the stage is a batched
// GEMM with per-tet scalars in the epilogue.  A team of IT = ceil(Np/8) warps
// takes a batch of 8 consecutive tets (one ticket); warp w owns the 8-row
// tile of volume nodes [8w, 8w+8) and computes, as 8x8x4 DMMA tiles with the
// 8 tets as the N dimension:
//   grad   gr, gs, gt = Dr P, Ds P, Dt P
//   div    dv = Dr W_r + Ds W_s + Dt W_t,  W_a = a_x UX + a_y UY + a_z UZ  (a = r, s, t)
//          -- 6 operator applications instead of the reference's 12
//          (tet_volume_elem, proj/src/solver.cpp:220-254)
//   lifts  lp = sum_f LIFT_f (ls_f Fp_f),  lu_f = LIFT_f (ls_f Fu_f)
//          (surface_elem tet branch, solver.cpp:321-333; ls_f = J_f / J)
// and the epilogue forms rp = -dv + lp, u_c = -(r_c gr + s_c gs + t_c gt) +
// sum_f n_{f,c} lu_f, scales by kappa / (1/rho) (scale_media, :337-346) and
// applies the LSERK45 stage (:541-551).  Dr, Ds, Dt and LIFT_f live in shared
// memory in DMMA-fragment-major order; the batch's state, records and
// connectivity arrive by TMA bulk copies (double-buffered per team), the
// residual is loaded straight into registers at the start of the batch.
#include <cuda_runtime.h>

#include <cstdlib>

#include "pdg_device.cuh"
#include "tma.cuh"

namespace pdg {

namespace {

__host__ __device__ constexpr int r2(int x) { return (x + 1) & ~1; }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int cf_stride(int x) {
  return (x % 16 == 4 || x % 16 == 12) ? x : cf_stride(x + 1);
}

// build the W_a columns between issuing the neighbour gathers and using them
#ifndef PDG_TET_BV_FIRST
#define PDG_TET_BV_FIRST 1
#endif
constexpr int kTB = 8; // tets per batch (the N dimension of every product)
// CTA size cap and stage depth: 640 / double-buffered measured best at N = 4
// (single-buffered 480/640-thread variants spill: 1.92 / 2.13 vs 1.65 ms)
// threads per CTA (register budget): 400 at N = 3, 640 otherwise (measured:
// N=3 0.97 vs 1.11 ms, N=4 1.65 vs 1.75 ms for 400)
#ifndef PDG_TET_CAP
#define PDG_TET_CAP(N) ((N) == 3 ? 400 : ((N) >= 6 ? PDG_TET_CAP_HI : 640))
#endif
#ifndef PDG_TET_CAP_HI
#define PDG_TET_CAP_HI 512
#endif
#ifndef PDG_TET_STAGES
#define PDG_TET_STAGES 2
#endif
constexpr int kComboCapT = 2048; // ints of neighbour node maps kept in shared memory

/// N >= 6: the operators (>= 0.25 MB) stay in L2/L1-resident global memory
#ifndef PDG_TET_TG_MIN_N
#define PDG_TET_TG_MIN_N 5 // measured: N=5 3.79 -> 3.16 ms, N=4 1.65 -> 1.85 ms with global tables
#endif
__host__ __device__ constexpr bool tet_tables_global(int N) { return N >= PDG_TET_TG_MIN_N; }

// residual loads issued after the flux phase instead of at the start of the batch
// (frees 16 registers across the gathers), and the face-node task indices
// recomputed in the flux loop instead of kept live across the gathers (at N = 4
// they were spilled to local memory, the hottest stall of the kernel).  Measured
// together (profiles/round2_tet_ab.txt): N = 3 / 4 / 5 -3.4 / -3.8 / -2.3%
#ifndef PDG_TET_RES_LATE
#define PDG_TET_RES_LATE 1
#endif
#ifndef PDG_TET_LAUNDER
#define PDG_TET_LAUNDER 1
#endif
// (Measured and removed, profiles/round2_tet_ab.txt / round2_mbar_ab.txt: interleaving
// the divergence chain with the gradient DMMAs -- equal, a dependent DMMA takes 26
// cycles against a 16-cycle issue interval, scripts/micro/dmma_latency.cu; the gradient
// products straight from the staged state before the fluxes -- +3..10%, registers;
// publishing the next batch index late -- neutral.)

// the next batch index in two slots alternating with the batch parity: a slot is
// rewritten only after every thread has read it, so the barrier that protected
// the single slot goes (two team barriers per batch instead of three)
#ifndef PDG_TET_SLOT_PARITY
#define PDG_TET_SLOT_PARITY 1
#endif

// end-of-batch barrier through an mbarrier (needs the slot parity and two stages):
// a warp arrives when it has finished the batch and only waits for the others
// right before it writes the work buffers of the next batch (after issuing that
// batch's neighbour gathers); thread 0 refills the freed stage after that wait.
// Measured with the slot parity (profiles/round2_mbar_ab.txt): N = 3 / 4 / 5
// -3.5 / -2.8 / -4.7% (slot parity alone: +0.2 / -0.6 / -0.1%)
#ifndef PDG_TET_END_MBAR
#define PDG_TET_END_MBAR 1
#endif

#ifndef PDG_TET_PAD_STATE
#define PDG_TET_PAD_STATE 1
#endif
__host__ __device__ constexpr int tet_slot_stride(int x) {
  return (x % 8 == 2 && x % 2 == 0) ? x : tet_slot_stride(x + 1);
}

template <int N, int NST_>
struct TDCfg {
  static constexpr int NP = npt_of(N), NT = nt_of(N);
  static constexpr int IT = ceil_div(NP, 8);  // row tiles = warps per team
  static constexpr int KS = ceil_div(NP, 4);  // k-steps over volume nodes
  static constexpr int KF = ceil_div(NT, 4);  // k-steps over one face
  static constexpr int T = IT;
  static constexpr int DTAB = IT * KS * 32;   // one of Dr, Ds, Dt
  static constexpr int LTAB = 4 * IT * KF * 32; // LIFT_f, f = 0..3
  static constexpr int BIGTAB = 3 * DTAB + LTAB;
  static constexpr bool TG = tet_tables_global(N);
  static constexpr int TABLES = r2((TG ? 0 : BIGTAB) + ceil_div(4 * NT, 2) + kComboCapT / 2);
  static constexpr int VST = cf_stride(NP);   // B-buffer column stride (volume)
  static constexpr int FST = cf_stride(NT);   // flux-buffer column stride
  // per-stage buffers: state, records, connectivity of 8 tets (the residual
  // goes straight from HBM into registers in the epilogue pattern)
  // per-tet state slot stride: 2 US = 4 or 12 mod 16 doubles, so the tets
  // 2 tig + c read by one warp instruction fall on distinct bank pairs
  // measured (profiles/round1_pad_state_ab.txt): N = 2, 3 -5%, N = 4, 5 neutral
  static constexpr int US = (PDG_TET_PAD_STATE && N <= 3) ? tet_slot_stride(4 * NP) : 4 * NP;
  static constexpr int UB = kTB * US;
  static constexpr int STAGE = r2(UB + kTB * kTG + kTB * 8 / 2);
  static constexpr int TASKS = ceil_div(kTB * 4 * NT, 32 * IT); // face-node tasks per thread
  static constexpr int BV = 4 * kTB * VST;    // [P | W_r | W_s | W_t] x 8 tets
  static constexpr int BF = 4 * kTB * FST;    // [face][tet][face node]
  static constexpr int WORK = BV + 2 * BF;
  static constexpr int SMEM_BUDGET = 225 * 1024;
  static constexpr int HDR = PDG_TET_SLOT_PARITY ? 6 : 4; // 2 mbarriers + 2 (3) slots
  static constexpr int NSTAGE = (NST_ == 2 && (TABLES + HDR + 2 * STAGE + WORK) * 8 <= SMEM_BUDGET) ? 2 : 1;
  static constexpr int PER_TEAM = HDR + NSTAGE * STAGE + WORK;
  static constexpr int TPB_SMEM = (SMEM_BUDGET / 8 - TABLES) / PER_TEAM;
  static constexpr int TPB = cmax(1, cmin(cmin(8, cmax(1, PDG_TET_CAP(N) / (32 * T))), TPB_SMEM));
  static constexpr int THREADS = 32 * T * TPB;
  static constexpr size_t SMEM_BYTES = (size_t)8 * (TABLES + TPB * PER_TEAM);
  static_assert(VST >= 4 * KS && FST >= 4 * KF, "padded K ranges must fit the column strides");
  static_assert(SMEM_BYTES <= 227 * 1024, "tet tables do not fit in shared memory");
};

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void team_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int N, int NST>
__device__ __forceinline__ void load_batch(const StageParams& p, double* stg, long long t0, int nel, uint64_t* bar) {
  using C = TDCfg<N, NST>;
  constexpr int NP = C::NP;
  double* U = stg;
  double* G = U + C::UB;
  const uint32_t ub = 32u * NP * nel;
  const uint32_t bytes = ub + 8u * kTG * nel + 32u * nel;
  const uint64_t keep = l2_policy_evict_last(), stream = l2_policy_evict_first();
  mbar_arrive_expect_tx(bar, bytes);
  if (C::US == 4 * NP) {
    tma_load_1d_hint(U, p.u_in + p.tet_base + t0 * 4 * NP, ub, bar, keep);
  } else {
    for (int t = 0; t < nel; ++t) // one bulk copy per tet into its padded slot
      tma_load_1d_hint(U + t * C::US, p.u_in + p.tet_base + (t0 + t) * 4 * NP, 32u * NP, bar, keep);
  }
  tma_load_1d_hint(G, p.tgeo + t0 * kTG, 8u * kTG * nel, bar, stream);
  tma_load_1d_hint(G + kTB * kTG, p.tconn + t0 * 8, 32u * nel, bar, stream);
}

/// fragment-major operator tables [D_r | D_s | D_t][t][s][lane], LIFT_f [f][t][s][lane]
template <int N>
__device__ void fill_tet_tables(double* dst, const StageParams& p, int tid, int nthr) {
  using C = TDCfg<N, 1>;
  constexpr int NP = C::NP, NT = C::NT, IT = C::IT, KS = C::KS, KF = C::KF;
  double* sD = dst;
  double* sL = dst + 3 * C::DTAB;
  for (int q = tid; q < 3 * C::DTAB; q += nthr) {
    const int lane = q & 31, rest = q >> 5;
    const int s = rest % KS, t = (rest / KS) % IT, a = rest / (KS * IT);
    const int n = 8 * t + (lane >> 2), k = 4 * s + (lane & 3);
    const double* src = a == 0 ? p.tDrT : (a == 1 ? p.tDsT : p.tDtT);
    sD[q] = (n < NP && k < NP) ? src[k * NP + n] : 0.0;
  }
  for (int q = tid; q < C::LTAB; q += nthr) {
    const int lane = q & 31, rest = q >> 5;
    const int s = rest % KF, t = (rest / KF) % IT, f = rest / (KF * IT);
    const int n = 8 * t + (lane >> 2), m = 4 * s + (lane & 3);
    sL[q] = (n < NP && m < NT) ? p.tLiftT[(f * NT + m) * NP + n] : 0.0;
  }
}

template <int N>
__global__ void tet_frag_kernel(const StageParams p, double* out) {
  fill_tet_tables<N>(out, p, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

template <int N, int NST>
__global__ void __launch_bounds__(TDCfg<N, NST>::THREADS, 1) tet_dmma_kernel(const StageParams p) {
  using C = TDCfg<N, NST>;
  constexpr int NP = C::NP, NT = C::NT, IT = C::IT, KS = C::KS, KF = C::KF, T = C::T;
  constexpr int VST = C::VST, FST = C::FST;
  extern __shared__ __align__(16) double smem[];
  double* sSmall = smem + (C::TG ? 0 : C::BIGTAB);
  int* sFace = reinterpret_cast<int*>(sSmall); // [4 NT] face node -> volume node
  int* sCombo = sFace + 2 * ceil_div(4 * NT, 2); // neighbour node maps (when they fit)
  for (int q = threadIdx.x; q < (int)(C::SMEM_BYTES / 8); q += C::THREADS) smem[q] = 0.0;
  __syncthreads();
  if (!C::TG) fill_tet_tables<N>(smem, p, threadIdx.x, C::THREADS);
  const double* sD = C::TG ? p.tet_frag : smem;   // [a][t][s][lane] = D_a(8t+gid, 4s+tig), a = r, s, t
  const double* sL = sD + 3 * C::DTAB;             // [f][t][s][lane] = LIFT(8t+gid, f NT + 4s+tig)
  auto tab = [](const double* t, int idx) -> double { return C::TG ? __ldg(t + idx) : t[idx]; };
  for (int q = threadIdx.x; q < 4 * NT; q += C::THREADS) sFace[q] = p.tface[q];
  const bool combo_smem = p.nbr_nodes_len <= kComboCapT;
  if (combo_smem)
    for (int q = threadIdx.x; q < p.nbr_nodes_len; q += C::THREADS) sCombo[q] = p.nbr_nodes[q];
  const int* combo = combo_smem ? sCombo : p.nbr_nodes;

  const int team = threadIdx.x / (32 * T);
  const int tt = threadIdx.x - team * 32 * T;
  const int w = tt >> 5, lane = tt & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int bar_id = 1 + team;
  double* tbase = smem + C::TABLES + (size_t)team * C::PER_TEAM;
  uint64_t* bar = reinterpret_cast<uint64_t*>(tbase);
  double* stg0 = tbase + C::HDR;
  double* BVb = stg0 + NST * C::STAGE; // column (g * 8 + tet) at g*8+tet times VST
  double* FPb = BVb + C::BV;           // column (face * 8 + tet) times FST
  double* FUb = FPb + C::BF;
  constexpr bool TMB = PDG_TET_END_MBAR && PDG_TET_SLOT_PARITY && NST == 2;
  uint64_t* ebar = bar + 5; // TMB: end of batch
  if (tt == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    if (TMB) mbar_init(ebar, 32 * T);
    fence_barrier_init();
  }
  __syncthreads();

  const int mode = p.mode;
  const bool vol = mode & M_VOLUME, surf = mode & M_SURFACE;
  const bool lserk = mode & M_LSERK, media = mode & M_MEDIA;
  const bool first = mode & M_FIRST, accum = mode & M_ACCUM;
  const double* res_src = lserk ? (first ? nullptr : p.res) : (accum ? p.rhs_out : nullptr);
  const long long nbatch = (p.Kt_active - p.Kt_begin + kTB - 1) / kTB;
  volatile long long* slot = reinterpret_cast<volatile long long*>(bar + 2);
  auto grab = [&]() -> long long { return (long long)(atomicAdd(p.ticket, 1ULL) - p.ticket_base); };
  auto nel_of = [&](long long b) -> int {
    const long long r = p.Kt_active - p.Kt_begin - b * kTB;
    return (int)(r < kTB ? r : kTB);
  };
  if (tt == 0) {
    const long long b0 = grab();
    slot[0] = b0;
    if (b0 < nbatch) load_batch<N, NST>(p, stg0, p.Kt_begin + b0 * kTB, nel_of(b0), bar);
  }
  team_sync(bar_id, 32 * T);
  long long b = slot[0];
  const double* ubase = p.u_in + p.tet_base;

  for (int it = 0; b < nbatch; ++it) {
    const int s = NST == 2 ? (it & 1) : 0;
    long long bn = 0;
    if (tt == 0) {
      bn = grab();
      slot[PDG_TET_SLOT_PARITY ? 1 + (it & 1) : 1] = bn;
    }
    const double* U = stg0 + s * C::STAGE;
    const double* G = U + C::UB;
    const int* Cn = reinterpret_cast<const int*>(G + kTB * kTG);
    if (NST == 2 && !TMB && tt == 0 && bn < nbatch) {
      fence_proxy_async_smem();
      load_batch<N, NST>(p, stg0 + (s ^ 1) * C::STAGE, p.Kt_begin + bn * kTB, nel_of(bn), bar + (s ^ 1));
    }
    // TMB: every thread has finished the previous batch (its stage and the work
    // buffers are free) -- waited once, before the first work-buffer write
    bool waited = !TMB;
    auto end_wait = [&]() {
      if (waited) return;
      waited = true;
      if (it > 0) mbar_wait(ebar, (it - 1) & 1);
      if (tt == 0 && bn < nbatch) {
        fence_proxy_async_smem();
        load_batch<N, NST>(p, stg0 + (s ^ 1) * C::STAGE, p.Kt_begin + bn * kTB, nel_of(bn), bar + (s ^ 1));
      }
    };
    mbar_wait(bar + s, NST == 2 ? ((it >> 1) & 1) : (it & 1));
    const long long t0 = p.Kt_begin + b * kTB;
    const int nel = nel_of(b);
    const int n = 8 * w + gid;
    // residual (or accumulated rhs) of this thread's 2 tets x 4 fields, loaded
    // now so the HBM latency overlaps the flux and product phases
    double rres[2][4];
    auto load_res = [&]() {
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int fld = 0; fld < 4; ++fld) {
        const int t = 2 * tig + c;
        rres[c][fld] = (res_src && n < NP && t < nel)
                           ? __ldcs(res_src + p.tet_base + (t0 + t) * 4 * NP + fld * NP + n) : 0.0;
      }
    };
    if (!PDG_TET_RES_LATE) load_res();

    // the W_a columns of the volume products (P, r/s/t-combinations of the velocity)
    // measured (profiles/round1_tet_bv_ab.txt): N = 3 -0.9%, N = 5 -0.6%, N = 6 -1.7%, N = 4 +2.5% (spills)
    constexpr bool kBvFirst = PDG_TET_BV_FIRST && N != 4;
    auto build_bv = [&]() {
    if (vol) {
      for (int m = tt; m < nel * NP; m += 32 * T) {
        const int t = m / NP, n = m - t * NP;
        const double* Ut = U + t * C::US;
        const double* Gt = G + t * kTG;
        const double ux = Ut[NP + n], uy = Ut[2 * NP + n], uz = Ut[3 * NP + n];
        BVb[t * VST + n] = Ut[n];
        BVb[(kTB + t) * VST + n] = Gt[T_RX] * ux + Gt[T_RY] * uy + Gt[T_RZ] * uz;
        BVb[(2 * kTB + t) * VST + n] = Gt[T_SX] * ux + Gt[T_SY] * uy + Gt[T_SZ] * uz;
        BVb[(3 * kTB + t) * VST + n] = Gt[T_TX] * ux + Gt[T_TY] * uy + Gt[T_TZ] * uz;
      }
    }
    };
    // ---- fluxes of the batch (scaled by J_f / J) and the W_a columns ------------
    if (kBvFirst && !surf) {
      end_wait();
      build_bv();
    }
    if (surf) {
      // all gathers of this thread's face-node tasks first (independent loads in
      // flight together), then the flux arithmetic
      double nbv[C::TASKS][4];
#pragma unroll
      for (int q = 0; q < C::TASKS; ++q) {
        const int m = tt + 32 * T * q;
        if (m < nel * 4 * NT) {
          const int t = m / (4 * NT), fm = m - t * 4 * NT;
          const int f = fm / NT, loc = fm - f * NT;
          const int nbr = Cn[t * 8 + 2 * f];
          if (nbr >= 0) {
            const int qn = combo[Cn[t * 8 + 2 * f + 1] * p.max_nfp + loc];
            const double* nb;
            int fs;
            if (nbr < p.Kw) {
              nb = p.u_in + (long long)nbr * 4 * npd_of(N) + qn;
              fs = npd_of(N);
            } else {
              nb = ubase + (long long)(nbr - p.Kw) * 4 * NP + qn;
              fs = NP;
            }
            nbv[q][0] = __ldg(nb);
            nbv[q][1] = __ldg(nb + fs);
            nbv[q][2] = __ldg(nb + 2 * fs);
            nbv[q][3] = __ldg(nb + 3 * fs);
          }
        }
      }
      end_wait();
      if (kBvFirst) build_bv(); // shared-memory work while the gathers are in flight
#pragma unroll
      for (int q = 0; q < C::TASKS; ++q) {
        int m = tt + 32 * T * q;
        if (PDG_TET_LAUNDER) asm volatile("" : "+r"(m)); // recomputed, not kept live
        if (m < nel * 4 * NT) {
          const int t = m / (4 * NT), fm = m - t * 4 * NT;
          const int f = fm / NT, loc = fm - f * NT;
          const double* Ut = U + t * C::US;
          const double* Gt = G + t * kTG;
          const int my = sFace[fm];
          const double pm = Ut[my];
          const double nx = Gt[T_NRM + 3 * f], ny = Gt[T_NRM + 3 * f + 1], nz = Gt[T_NRM + 3 * f + 2];
          const double taup = Gt[T_TAUP + f], tauu = Gt[T_TAUU + f];
          double fp, fu;
          if (Cn[t * 8 + 2 * f] >= 0) {
            const double dp = nbv[q][0] - pm;
            const double dun = nx * (nbv[q][1] - Ut[NP + my]) + ny * (nbv[q][2] - Ut[2 * NP + my]) +
                               nz * (nbv[q][3] - Ut[3 * NP + my]);
            fp = 0.5 * (taup * dp - dun);
            fu = 0.5 * (tauu * dun - dp);
          } else {
            const double dp = -2.0 * pm; // reflective: p+ = -p-, u+ = u-
            fp = 0.5 * taup * dp;
            fu = -0.5 * dp;
          }
          const double ls = Gt[T_LS + f];
          FPb[(f * kTB + t) * FST + loc] = ls * fp;
          FUb[(f * kTB + t) * FST + loc] = ls * fu;
        }
      }
    }
    end_wait();
    if (!kBvFirst) build_bv();
    if (PDG_TET_RES_LATE) load_res();
    team_sync(bar_id, 32 * T);

    // ---- row tile w: volume and lift products -------------------------------------
    double gr[2] = {0.0, 0.0}, gs[2] = {0.0, 0.0}, gt[2] = {0.0, 0.0}, dv[2] = {0.0, 0.0};
    double lp[2] = {0.0, 0.0}, lu[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    if (vol) {
#pragma unroll
      for (int s2 = 0; s2 < KS; ++s2) {
        const int fo = ((w * KS + s2) << 5) + lane;
        const double ar = tab(sD, fo), as = tab(sD, C::DTAB + fo), at = tab(sD, 2 * C::DTAB + fo);
        const int bo = gid * VST + 4 * s2 + tig;
        const double bp = BVb[bo];
        dmma(gr, ar, bp);
        dmma(gs, as, bp);
        dmma(gt, at, bp);
        dmma(dv, ar, BVb[kTB * VST + bo]);
        dmma(dv, as, BVb[2 * kTB * VST + bo]);
        dmma(dv, at, BVb[3 * kTB * VST + bo]);
      }
    }
    if (surf) {
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int s2 = 0; s2 < KF; ++s2) {
          const double a = tab(sL, (((f * IT + w) * KF + s2) << 5) + lane);
          const int bo = (f * kTB + gid) * FST + 4 * s2 + tig;
          dmma(lp, a, FPb[bo]);
          dmma(lu[f], a, FUb[bo]);
        }
    }

    // ---- epilogue: node n = 8w + gid, tets 2 tig + c --------------------------------
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int t = 2 * tig + c;
      if (n < NP && t < nel) {
        const double* Gt = G + t * kTG;
        double rp = 0.0, rux = 0.0, ruy = 0.0, ruz = 0.0;
        if (vol) {
          rp = -dv[c];
          rux = -(Gt[T_RX] * gr[c] + Gt[T_SX] * gs[c] + Gt[T_TX] * gt[c]);
          ruy = -(Gt[T_RY] * gr[c] + Gt[T_SY] * gs[c] + Gt[T_TY] * gt[c]);
          ruz = -(Gt[T_RZ] * gr[c] + Gt[T_SZ] * gs[c] + Gt[T_TZ] * gt[c]);
        }
        if (surf) {
          rp += lp[c];
#pragma unroll
          for (int f = 0; f < 4; ++f) {
            rux += Gt[T_NRM + 3 * f] * lu[f][c];
            ruy += Gt[T_NRM + 3 * f + 1] * lu[f][c];
            ruz += Gt[T_NRM + 3 * f + 2] * lu[f][c];
          }
        }
        if (media) {
          const double kappa = Gt[T_KAPPA], irho = Gt[T_IRHO];
          rp *= kappa;
          rux *= irho;
          ruy *= irho;
          ruz *= irho;
        }
        const double rv[4] = {rp, rux, ruy, ruz};
        const double* Ut = U + t * C::US;
        const long long go = p.tet_base + (t0 + t) * 4 * NP + n;
#pragma unroll
        for (int fld = 0; fld < 4; ++fld) {
          const int o = fld * NP + n;
          if (lserk) {
            const double rr = first ? p.dt * rv[fld] : p.a * rres[c][fld] + p.dt * rv[fld];
            __stcs(p.res + go + fld * NP, rr);
            __stcs(p.u_out + go + fld * NP, Ut[o] + p.b * rr);
          } else {
            __stcs(p.rhs_out + go + fld * NP, accum ? rres[c][fld] + rv[fld] : rv[fld]);
          }
        }
      }
    }
    if (TMB)
      mbar_arrive(ebar);
    else
      team_sync(bar_id, 32 * T); // stage s and the work buffers are free again
    if (NST == 1 && tt == 0 && bn < nbatch) load_batch<N, NST>(p, stg0, p.Kt_begin + bn * kTB, nel_of(bn), bar);
    b = slot[PDG_TET_SLOT_PARITY ? 1 + (it & 1) : 1];
    if (!PDG_TET_SLOT_PARITY) team_sync(bar_id, 32 * T);
  }
}

template <int N>
cudaError_t launch_tet_dmma_N(const StageParams& p, cudaStream_t s) {
  using C = TDCfg<N, PDG_TET_STAGES>;
  constexpr int NST = C::NSTAGE;
  // one-time setup per device (the smem attribute is per device)
  static int grid_cap[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  auto kern = tet_dmma_kernel<N, NST>;
  if (grid_cap[dev] == 0) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::SMEM_BYTES);
    grid_cap[dev] = sms * (per_sm > 0 ? per_sm : 1);
  }
  if (p.info) *p.info = LaunchInfo{};
  if (p.Kt_active - p.Kt_begin <= 0) return cudaSuccess;
  const long long nbatch = (p.Kt_active - p.Kt_begin + kTB - 1) / kTB;
  const long long need = (nbatch + C::TPB - 1) / C::TPB;
  const int grid = (int)(need < grid_cap[dev] ? need : grid_cap[dev]);
  StageParams q = p;
  q.ticket_base = *p.ticket_host_next;
  *p.ticket_host_next += (unsigned long long)nbatch + (unsigned long long)grid * C::TPB;
  kern<<<grid, C::THREADS, C::SMEM_BYTES, s>>>(q);
  if (p.info) *p.info = LaunchInfo{1, (long long)grid * C::TPB, nbatch, kTB};
  return cudaGetLastError();
}

} // namespace

bool tet_dmma_supported(int N) { return N >= 1 && N <= 7; }

size_t tet_frag_size(int N) {
  switch (N) {
#define PDG_CASE(n) case n: return tet_tables_global(n) ? (size_t)TDCfg<n, 1>::BIGTAB : 0;
    PDG_CASE(1) PDG_CASE(2) PDG_CASE(3) PDG_CASE(4) PDG_CASE(5) PDG_CASE(6) PDG_CASE(7)
#undef PDG_CASE
  }
  return 0;
}

cudaError_t launch_tet_frag_fill(int N, const StageParams& p, double* out, cudaStream_t s) {
  switch (N) {
#define PDG_CASE(n) \
  case n:           \
    if (!tet_tables_global(n)) return cudaSuccess; \
    tet_frag_kernel<n><<<64, 256, 0, s>>>(p, out); \
    return cudaGetLastError();
    PDG_CASE(1) PDG_CASE(2) PDG_CASE(3) PDG_CASE(4) PDG_CASE(5) PDG_CASE(6) PDG_CASE(7)
#undef PDG_CASE
  }
  return cudaSuccess;
}

cudaError_t launch_tet_dmma_stage(int N, const StageParams& p, cudaStream_t s) {
  switch (N) {
#define PDG_CASE(n) case n: return launch_tet_dmma_N<n>(p, s);
    PDG_CASE(1) PDG_CASE(2) PDG_CASE(3) PDG_CASE(4) PDG_CASE(5) PDG_CASE(6) PDG_CASE(7)
#undef PDG_CASE
  }
  return cudaErrorInvalidValue;
}

} // namespace pdg
