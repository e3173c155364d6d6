// Warp-specialised fused wedge stage kernel (N >= 4, FP64 tensor cores).
//
// The same per-element algebra as wedge_dmma.cu (G1..G5 + epilogue, the lift
// folds of SURVEY.md A.3; reference wedge_volume_elem / surface_elem /
// scale_media / lserk, proj/src/solver.cpp:164-218, 258-335, 337-346, 541-551),
// with the work of a team split by role:
//   * T compute warps (one 8-row tile of triangle nodes each) run the DMMA
//     products and the epilogue, exactly as in wedge_dmma.cu;
//   * one producer warp grabs tickets, issues the element's bulk TMA copies,
//     gathers the neighbour face traces (L2) and computes the numerical fluxes
//     of the NEXT element into a parity flux buffer while the compute warps
//     work on the current one.
// ncu on wedge_dmma.cu (profiles/round2_wedge_n5_sass.txt) put 13% of all
// stall samples on the first use of the gathered traces and 14% on the team
// barriers that the flux phase's imbalance feeds; here the compute warps never
// touch global gathers and meet only one named barrier per element (V).
//
// Stages: an element's bytes arrive in two bulk-copy groups, A = state +
// record + connectivity (read by both roles; ring of 3) and B = residual +
// L^{tri,k} + quad lifts (compute warps only; ring of 2).  When the compute
// warps finish element n-1 the producer issues A(n+2) and B(n+1), so the
// fluxes of element n+1 (whose A copy landed an element earlier) are computed
// during element n: only the neighbour gathers' L2 latency is on the
// producer's path, hidden behind a whole element of compute.
// Synchronisation per team (mbarriers in shared memory):
//   fullA[n%3], fullB[n&1] : the copies of element n landed
//   ffull[n&1]             : fluxes of element n written (32 producer lanes)
//   done[n&1]              : compute warps finished element n (32 T lanes)
// Element ids travel with the A slot (elem[n%3], written before the copy is
// issued; the arrive's release / the wait's acquire order it).  A ticket past
// the end is published as elem >= Kw_active with a plain arrive: both roles
// leave their loops on it.
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
__host__ __device__ constexpr int cf_stride(int x) { return (x % 16 == 4 || x % 16 == 12) ? x : cf_stride(x + 1); }
__host__ __device__ constexpr int kmap(int s, int tig, int KS, bool perm) {
  return (perm && s < 4 * (KS / 4)) ? 16 * (s >> 2) + 4 * tig + (s & 3) : 4 * s + tig;
}

constexpr int kComboCap = 4096; // ints of neighbour node maps kept in shared memory
#ifndef PDG_WS_THREAD_CAP
#define PDG_WS_THREAD_CAP 512
#endif
#ifndef PDG_WS_GATHER_BATCH
#define PDG_WS_GATHER_BATCH 5
#endif
// the producer also forms V (the vertical products G1 + the folded bottom/top
// pressure lifts) for every row tile, so the compute warps need no barrier at all
#ifndef PDG_WS_PRODUCER_V
#define PDG_WS_PRODUCER_V 1
#endif

template <int N>
struct WCfg {
  static constexpr int NQ = nq_of(N), NT = nt_of(N), NP = npd_of(N), ST = nts_of(N), FW = fw_of(N), WG = wg_of(N);
  static constexpr int IT = it_of(N), KS = ks_of(N), KT = kt_of(N);
  static constexpr int JT = ceil_div(NQ, 8), NPJ = 8 * JT, JTL = ceil_div(NQ + 2, 8);
  static constexpr int T = IT;        // compute warps per team
  static constexpr int WPT = T + 1;   // + the producer warp
  static constexpr int LF = lcomp_of(N), QF = qcomp_of(N);
  static constexpr int USTR = r4(4 * NP) + 2;
  static constexpr int STA = r2(USTR + WG + kWC / 2); // A: state, record, connectivity
  static constexpr int STB = r2(USTR + LF + QF);      // B: residual, L, quad lifts
  static constexpr bool KP = (NT & 1) && ST == NT;
  static constexpr int VST = KP ? NT : cf_stride(NT);
  static constexpr int VS = r2((NPJ - 1) * VST + 4 * KS + 8);
  static constexpr int FQ = 3 * JT * KT * 32;
  static constexpr int FTRI = r2(4 * KS + NT + 8);
  static constexpr int ZS = r2(4 * KS);
  static constexpr int FB = 2 * (FTRI + FQ);
  static constexpr int HDR = 12; // 9 mbarriers + elem[3]
  static constexpr int PER_TEAM = HDR + 3 * STA + 2 * STB + 2 * VS + 2 * FB + ZS;
  static constexpr int TABLES = r2(2 * IT * KS * 32 + JT * KT * 32 + 2 * NQ + ceil_div(FW, 2) + kComboCap / 2);
  static constexpr int SMEM_BUDGET = 225 * 1024;
  static constexpr int TPB_SMEM = (SMEM_BUDGET / 8 - TABLES) / PER_TEAM;
  static constexpr int TPB = cmax(1, cmin(PDG_WS_THREAD_CAP / (32 * WPT), TPB_SMEM));
  static constexpr int THREADS = 32 * WPT * TPB;
  static constexpr size_t SMEM_BYTES = (size_t)8 * (TABLES + TPB * PER_TEAM);
  static constexpr int FT_LANE = ceil_div(FW, 32); // producer face-node tasks per lane
  static constexpr int GB = cmin(FT_LANE, PDG_WS_GATHER_BATCH);
};

inline int ws_ticket_batch(int N) {
  static const int env = [] {
    const char* v = std::getenv("PDG_TICKET_BATCH");
    return v ? std::atoi(v) : 0;
  }();
  if (env > 0) return env;
  return N == 4 ? 4 : 2;
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int N>
__device__ __forceinline__ void ws_load_a(const StageParams& p, double* sa, long long e, uint64_t* bar) {
  using C = WCfg<N>;
  constexpr int NP = C::NP;
  // the state stays in L2 for the neighbours' trace gathers; the rest is touched once
  const uint64_t keep = l2_policy_evict_last(), stream = l2_policy_evict_first();
  mbar_arrive_expect_tx(bar, 8u * (4 * NP + C::WG) + 4u * kWC);
  tma_load_1d_hint(sa, p.u_in + e * 4 * NP, 32 * NP, bar, keep);
  tma_load_1d_hint(sa + C::USTR, p.wgeo + e * C::WG, 8 * C::WG, bar, stream);
  tma_load_1d_hint(sa + C::USTR + C::WG, p.wconn + e * kWC, 4 * kWC, bar, stream);
}

template <int N>
__device__ __forceinline__ void ws_load_b(const StageParams& p, double* sb, long long e, const double* res_src,
                                          uint64_t* bar) {
  using C = WCfg<N>;
  constexpr int NP = C::NP;
  const uint64_t stream = l2_policy_evict_first();
  mbar_arrive_expect_tx(bar, 8u * (C::LF + C::QF) + (res_src ? 32u * NP : 0u));
  if (res_src) tma_load_1d_hint(sb, res_src + e * 4 * NP, 32 * NP, bar, stream);
  tma_load_1d_hint(sb + C::USTR, p.Lt + e * C::LF, 8 * C::LF, bar, stream);
  tma_load_1d_hint(sb + C::USTR + C::LF, p.QL + e * C::QF, 8 * C::QF, bar, stream);
}

template <int N, bool COMBO_SMEM, bool FUSED>
__global__ void __launch_bounds__(WCfg<N>::THREADS, 1) wedge_ws_kernel(const StageParams p) {
  using C = WCfg<N>;
  constexpr int NQ = C::NQ, NT = C::NT, NP = C::NP, ST = C::ST, FW = C::FW, WG = C::WG, T = C::T;
  constexpr int KS = C::KS, JT = C::JT, JTL = C::JTL, KT = C::KT, VST = C::VST;
  extern __shared__ __align__(16) double smem[];

  // ---- shared reference tables (fragment-major, zero padded) ----------------
  double* sDr = smem;                  // [t][s][lane] = Dr(8t+gid, kmap(s, tig))
  double* sDs = sDr + C::IT * KS * 32;
  double* sDt = sDs + C::IT * KS * 32; // [jt][s][lane] = Dt(8jt+gid, 4s+tig)
  double* sProf = sDt + JT * KT * 32;  // [2][NQ]
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

  const int team = threadIdx.x / (32 * C::WPT);
  const int tw = (threadIdx.x >> 5) - team * C::WPT; // warp within team: < T compute, == T producer
  const int lane = threadIdx.x & 31;
  double* tbase = smem + C::TABLES + (size_t)team * C::PER_TEAM;
  uint64_t* fullA = reinterpret_cast<uint64_t*>(tbase);
  uint64_t* fullB = fullA + 3;
  uint64_t* ffull = fullA + 5;
  uint64_t* done = fullA + 7;
  volatile long long* elem = reinterpret_cast<volatile long long*>(fullA + 9);
  double* sA0 = tbase + C::HDR;
  double* sB0 = sA0 + 3 * C::STA;
  double* V0 = sB0 + 2 * C::STB;
  double* F0 = V0 + 2 * C::VS;
  const double* Zero = F0 + 2 * C::FB; // ZS zeros, never written
  if (tw == T && lane == 0) {
    for (int s = 0; s < 3; ++s) mbar_init(fullA + s, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(fullB + s, 1);
      mbar_init(ffull + s, 32);
      mbar_init(done + s, 32 * T);
    }
    fence_barrier_init();
  }
  __syncthreads(); // the last CTA-wide barrier: the roles below never meet again

  const int mode = p.mode;
  const bool vol = FUSED || (mode & M_VOLUME), surf = FUSED || (mode & M_SURFACE);
  const bool lserk = FUSED || (mode & M_LSERK), media = FUSED || (mode & M_MEDIA);
  const bool first = mode & M_FIRST, accum = !FUSED && (mode & M_ACCUM);
  const double* res_src = lserk ? (first ? nullptr : p.res) : (accum ? p.rhs_out : nullptr);

  if (tw == T) {
    // ======================= producer warp ===================================
    const int B = p.ticket_batch;
    long long bnext = 0, bend = 0;
    auto grab = [&]() -> long long {
      if (bnext >= bend) {
        bnext = p.Kw_begin + (long long)(atomicAdd(p.ticket, (unsigned long long)B) - p.ticket_base);
        bend = bnext + B < p.Kw_active ? bnext + B : (bnext < p.Kw_active ? p.Kw_active : bnext + 1);
      }
      return bnext++;
    };
    auto issue_a = [&](int n) { // lane 0: grab element n, copy its A group
      const long long e = grab();
      const int a = n % 3;
      elem[a] = e;
      if (e < p.Kw_active) {
        fence_proxy_async_smem();
        ws_load_a<N>(p, sA0 + a * C::STA, e, fullA + a);
      } else {
        mbar_arrive(fullA + a);
      }
    };
    auto issue_b = [&](int n) { // lane 0: the B group of element n (already grabbed)
      const long long e = elem[n % 3];
      if (e < p.Kw_active) {
        fence_proxy_async_smem();
        ws_load_b<N>(p, sB0 + (n & 1) * C::STB, e, res_src, fullB + (n & 1));
      }
    };
    if (lane == 0) {
      issue_a(0);
      issue_a(1);
      issue_b(0);
    }
    for (int n = 0;; ++n) {
      const int s = n & 1, a = n % 3;
      mbar_wait(fullA + a, (n / 3) & 1);
      if (elem[a] >= p.Kw_active) break;
      if (surf) {
        const double* U = sA0 + a * C::STA;
        const double* G = U + C::USTR;
        const int* Cn = reinterpret_cast<const int*>(G + WG);
        double* Ftp = F0 + s * C::FB; // tri-face fluxes: p part [2][NT]
        double* Ftu = Ftp + C::FTRI;  //                  u part
        double* Fqp = Ftu + C::FTRI;  // quad-face fluxes, fragment-major [f][jt][s][lane]
        double* Fqu = Fqp + C::FQ;
#pragma unroll
        for (int q0 = 0; q0 < C::FT_LANE; q0 += C::GB) {
          // gathers of a batch of face-node tasks first (all in flight), then fluxes
          double nb[C::GB][4];
          int tf[C::GB], tl[C::GB];
#pragma unroll
          for (int b = 0; b < C::GB; ++b) {
            const int m = lane + 32 * (q0 + b);
            tf[b] = -1;
            if (q0 + b < C::FT_LANE && m < FW) {
              const int f = m < NT ? 0 : (m < 2 * NT ? 1 : 2 + (m - 2 * NT) / (NQ * NQ));
              const int loc = m < 2 * NT ? m - f * NT : (m - 2 * NT) - (f - 2) * NQ * NQ;
              tf[b] = f;
              tl[b] = loc;
              const int nbr = Cn[2 * f];
              if (nbr >= 0) {
                const int mi = Cn[2 * f + 1] * p.max_nfp + loc;
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
                nb[b][0] = __ldg(src);
                nb[b][1] = __ldg(src + fs);
                nb[b][2] = __ldg(src + 2 * fs);
                nb[b][3] = __ldg(src + 3 * fs);
              }
            }
          }
#pragma unroll
          for (int b = 0; b < C::GB; ++b) {
            const int f = tf[b];
            if (f < 0) continue;
            const int m = lane + 32 * (q0 + b), loc = tl[b];
            const int my = sWface[m];
            const double pm = U[my];
            const double nx = G[w_nrm(N) + 3 * f], ny = G[w_nrm(N) + 3 * f + 1], nz = G[w_nrm(N) + 3 * f + 2];
            const double taup = G[w_taup(N) + f], tauu = G[w_tauu(N) + f];
            double fp, fu;
            if (Cn[2 * f] >= 0) {
              const double dp = nb[b][0] - pm;
              const double dun = nx * (nb[b][1] - U[NP + my]) + ny * (nb[b][2] - U[2 * NP + my]) +
                                 nz * (nb[b][3] - U[3 * NP + my]);
              fp = 0.5 * (taup * dp - dun);
              fu = 0.5 * (tauu * dun - dp);
            } else {
              const double dp = -2.0 * pm; // reflective: p+ = -p-, u+ = u-
              fp = 0.5 * taup * dp;
              fu = -0.5 * dp;
            }
            if (f < 2) {
              Ftp[m] = fp;
              Ftu[m] = fu;
            } else {
              const int a = loc / NQ, j = loc - a * NQ;
              const int pos = ((((f - 2) * JT + j / 8) * KT + a / 4) << 5) + ((j & 7) << 2) + (a & 3);
              Fqp[pos] = fp;
              Fqu[pos] = fu;
            }
          }
        }
      }
      if (PDG_WS_PRODUCER_V) {
        // V[j][i] of every row tile (G1 of wedge_dmma.cu), parity buffer s
        __syncwarp(); // the tri-face fluxes of all lanes are in shared memory
        const double* U = sA0 + a * C::STA;
        const double* G = U + C::USTR;
        const double* Ftp = F0 + s * C::FB;
        double* V = V0 + s * C::VS;
        const int gid = lane >> 2, tig = lane & 3;
        const double tzJ = G[W_TZJ], jfb = G[W_JFB], jft = G[W_JFT];
#pragma unroll
        for (int t = 0; t < C::IT; ++t) {
          const int i = 8 * t + gid;
          const double fb = surf ? jfb * Ftp[i] : 0.0, ftop = surf ? jft * Ftp[NT + i] : 0.0;
#pragma unroll
          for (int jt = 0; jt < JT; ++jt) {
            double d[2] = {0.0, 0.0};
            if (vol) {
              const int jb = 8 * jt + gid;
              const int jc = jb < NQ ? jb : NQ - 1;
              const double sx_ = G[W_TXJ + jc], sy_ = G[w_tyj(N) + jc];
#pragma unroll
              for (int s2 = 0; s2 < KT; ++s2) {
                const int l = 4 * s2 + tig;
                const double bd = sDt[((jt * KT + s2) << 5) + lane];
                dmma(d, U[(NQ + l) * ST + i], sx_ * bd);
                dmma(d, U[(2 * NQ + l) * ST + i], sy_ * bd);
                dmma(d, U[(3 * NQ + l) * ST + i], tzJ * bd);
              }
            }
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const int j = 8 * jt + 2 * tig + c;
              if (i < NT && j < NQ) V[j * VST + i] = -d[c] + fb * sProf[j] + ftop * sProf[NQ + j];
            }
          }
        }
      }
      mbar_arrive(ffull + s);
      // element n-1 done: its A slot takes element n+2, its B slot element n+1
      if (n >= 1) mbar_wait(done + (s ^ 1), ((n - 1) >> 1) & 1);
      if (lane == 0) {
        issue_a(n + 2);
        issue_b(n + 1);
      }
      __syncwarp();
    }
    return;
  }

  // ========================= compute warps ====================================
  const int w = tw, gid = lane >> 2, tig = lane & 3;
  const int bar_id = 1 + team;
  for (int n = 0;; ++n) {
    const int s = n & 1, ph = (n >> 1) & 1, a = n % 3;
    mbar_wait(fullA + a, (n / 3) & 1);
    const long long e = elem[a];
    if (e >= p.Kw_active) break;
    const double* U = sA0 + a * C::STA;
    const double* G = U + C::USTR;
    const double* R = sB0 + s * C::STB;
    const double* Lf = R + C::USTR;
    const double* Qf = Lf + C::LF;
    const double* Ftp = F0 + s * C::FB;
    const double* Ftu = Ftp + C::FTRI;
    const double* Fqp = Ftu + C::FTRI;
    const double* Fqu = Fqp + C::FQ;
    double* V = V0 + s * C::VS;
    const double* Us = U; // state, slice stride ST
    constexpr int SP = ST;
    mbar_wait(fullB + s, ph);
    mbar_wait(ffull + s, ph);

    // ---- G1: V[j][i] for row tile w, with the bottom/top pressure lifts folded in
    // (formed by the producer when PDG_WS_PRODUCER_V)
    if (!PDG_WS_PRODUCER_V) {
      const int i = 8 * w + gid;
      const double tzJ = G[W_TZJ], jfb = G[W_JFB], jft = G[W_JFT];
      const double fb = surf ? jfb * Ftp[i] : 0.0, ftop = surf ? jft * Ftp[NT + i] : 0.0;
#pragma unroll
      for (int jt = 0; jt < JT; ++jt) {
        double d[2] = {0.0, 0.0};
        if (vol) {
          const int jb = 8 * jt + gid;
          const int jc = jb < NQ ? jb : NQ - 1;
          const double sx_ = G[W_TXJ + jc], sy_ = G[w_tyj(N) + jc];
#pragma unroll
          for (int s2 = 0; s2 < KT; ++s2) {
            const int l = 4 * s2 + tig;
            const double bd = sDt[((jt * KT + s2) << 5) + lane];
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
    if (!PDG_WS_PRODUCER_V) named_sync(bar_id, 32 * T);

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
      double gx[JT][2], gy[JT][2], dvx[JT][2], dvy[JT][2], lv[JT][2], lp[JTL][2];
#pragma unroll
      for (int jt = 0; jt < JT; ++jt)
#pragma unroll
        for (int c = 0; c < 2; ++c) gx[jt][c] = gy[jt][c] = dvx[jt][c] = dvy[jt][c] = lv[jt][c] = 0.0;
#pragma unroll
      for (int jt = 0; jt < JTL; ++jt) lp[jt][0] = lp[jt][1] = 0.0;
#pragma unroll
      for (int s2 = 0; s2 < KS; ++s2) {
        const int k = kmap(s2, tig, KS, C::KP);
        const int fo = ((t * KS + s2) << 5) + lane;
        const double la = (i < NT && k < NT) ? Lf[k * NT + i] : 0.0;
        double cx = 0.0, cy = 0.0;
        if (vol) {
          const double dr = sDr[fo], ds = sDs[fo];
          cx = rx * dr + sxm * ds;
          cy = ry * dr + sym * ds;
        }
#pragma unroll
        for (int jt = 0; jt < JTL; ++jt) {
          const double bp = src[jt][k];
          dmma(lp[jt], la, bp);
          if (jt < JT) {
            const int jb = 8 * jt + gid;
            if (vol) {
              dmma(gx[jt], cx, bp);
              dmma(gy[jt], cy, bp);
              dmma(dvx[jt], cx, Us[(NQ + jb) * SP + k]);
              dmma(dvy[jt], cy, Us[(2 * NQ + jb) * SP + k]);
            }
            dmma(lv[jt], la, V[jb * VST + k]);
          }
        }
      }
      // G4: LY = LP Dt^T, A fragments of LP gathered within each lane quad
      double ly[JT][2];
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
          for (int jt = 0; jt < JT; ++jt) dmma(ly[jt], a, sDt[((jt * KT + s2) << 5) + lane]);
        }
      }
      constexpr int c0 = NQ % 8, c1 = (NQ + 1) % 8;
      const double lf0 = __shfl_sync(0xffffffffu, lp[NQ / 8][c0 & 1], gid * 4 + c0 / 2);
      const double lf1 = __shfl_sync(0xffffffffu, lp[(NQ + 1) / 8][c1 & 1], gid * 4 + c1 / 2);
      // G5: quad-face lifts; each face's velocity lift scaled by its normal in the epilogue
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
            const int qa_a = 4 * s2 + tig;
            const double qa = (i < NT && qa_a < NQ) ? Qf[(f * NQ + qa_a) * NT + i] : 0.0;
#pragma unroll
            for (int jt = 0; jt < JT; ++jt) {
              const int fo = (((f * JT + jt) * KT + s2) << 5) + lane;
              dmma(qp[jt], qa, Fqp[fo]);
              dmma(qu[f][jt], qa, Fqu[fo]);
            }
          }
      }
      // epilogue: rows i, columns j = 8 jt + 2 tig + c; results straight to HBM
      const double tzJ = G[W_TZJ], jfb = G[W_JFB], jft = G[W_JFT];
      const double kappa = G[W_KAPPA], irho = G[W_IRHO];
      const double pa = p.a, pb = p.b, pdt = p.dt;
      double n_[5][3];
#pragma unroll
      for (int f = 0; f < 5; ++f)
#pragma unroll
        for (int a = 0; a < 3; ++a) n_[f][a] = nrm[3 * f + a];
      const int lane_off = 2 * tig * ST + i;
      const double* Ul = Us + 2 * tig * SP + i;
      const double* Rl = R + lane_off;
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
            if (media) {
              rp *= kappa;
              rux *= irho;
              ruy *= irho;
              ruz *= irho;
            }
            const double rv[4] = {rp, rux, ruy, ruz};
            constexpr int cst[2] = {0, ST};
#pragma unroll
            for (int f = 0; f < 4; ++f) {
              const int o = f * NP + 8 * jt * ST + cst[c];
              if (lserk) {
                const double rr = first ? pdt * rv[f] : pa * Rl[o] + pdt * rv[f];
                __stcs(resl + o, rr); // streaming stores: evict first
                __stcs(uol + o, Ul[o] + pb * rr);
              } else {
                __stcs(rhsl + o, accum ? Rl[o] + rv[f] : rv[f]);
              }
            }
          }
        }
    }
    // this element's A and B slots and its flux set may be reused
    mbar_arrive(done + s);
  }
}

template <int N, bool CS, bool FUSED>
cudaError_t launch_ws_NC(const StageParams& p, cudaStream_t s) {
  using C = WCfg<N>;
  static int grid_cap[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  auto kern = wedge_ws_kernel<N, CS, FUSED>;
  if (grid_cap[dev] == 0) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::SMEM_BYTES);
    grid_cap[dev] = sms * (per_sm > 0 ? per_sm : 1);
  }
  const long long nact = p.Kw_active - p.Kw_begin;
  if (p.info) *p.info = LaunchInfo{};
  if (nact <= 0) return cudaSuccess;
  const long long need = (nact + C::TPB - 1) / C::TPB;
  const int grid = (int)(need < grid_cap[dev] ? need : grid_cap[dev]);
  StageParams q = p;
  q.ticket_base = *p.ticket_host_next;
  q.ticket_batch = ws_ticket_batch(N);
  const unsigned long long B = (unsigned long long)q.ticket_batch;
  // every team's producer grabs two tickets past the end (it runs two elements
  // ahead), so the counter ends exactly here and the next launch starts clean
  *p.ticket_host_next += B * (((unsigned long long)nact + B - 1) / B + 2ull * (unsigned long long)grid * C::TPB);
  kern<<<grid, C::THREADS, C::SMEM_BYTES, s>>>(q);
  if (p.info) *p.info = LaunchInfo{1, (long long)grid * C::TPB, (nact + (long long)B - 1) / (long long)B, (int)B};
  return cudaGetLastError();
}

template <int N>
cudaError_t launch_ws_N(const StageParams& p, cudaStream_t s) {
  constexpr int F = M_VOLUME | M_SURFACE | M_MEDIA | M_LSERK;
  const bool fused = (p.mode & F) == F && !(p.mode & M_ACCUM);
  const bool cs = p.nbr_nodes_len <= kComboCap;
  if (fused) return cs ? launch_ws_NC<N, true, true>(p, s) : launch_ws_NC<N, false, true>(p, s);
  return cs ? launch_ws_NC<N, true, false>(p, s) : launch_ws_NC<N, false, false>(p, s);
}

} // namespace

bool wedge_ws_supported(int N) { return N >= 4 && N <= 7; }

cudaError_t launch_wedge_ws_stage(int N, const StageParams& p, cudaStream_t s) {
  switch (N) {
    case 4: return launch_ws_N<4>(p, s);
    case 5: return launch_ws_N<5>(p, s);
    case 6: return launch_ws_N<6>(p, s);
    case 7: return launch_ws_N<7>(p, s);
  }
  return cudaErrorInvalidValue;
}

int wedge_ws_elems_per_block(int N) {
  switch (N) {
    case 4: return WCfg<4>::TPB;
    case 5: return WCfg<5>::TPB;
    case 6: return WCfg<6>::TPB;
    case 7: return WCfg<7>::TPB;
  }
  return 0;
}

} // namespace pdg
