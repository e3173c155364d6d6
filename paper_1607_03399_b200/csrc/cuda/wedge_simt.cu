// Fused wedge stage kernel for low orders (N <= 3), FP64 CUDA cores.
//
// At N = 1..3 a wedge is 24..160 DOFs and its triangle matrices are 3x3..10x10:
// an 8x8x4 tensor-core tile is mostly padding (9% useful at N=1) and a team of
// warps per wedge leaves the SM waiting on one element's latency chain.  Here
// one thread owns one (wedge, triangle node i) pair and every slice j of it,
// so a 128-thread CTA works on E = 128 / NT wedges at once (42 at N=1) and the
// per-element products are short register-resident dot products:
//   V(j,i)  = -(txJ_j Dt UX + tyJ_j Dt UY + tzJ Dt UZ)(j,i) + tri-face p lifts
//   gx, gy  = (rx Dr + sx Ds) P, (ry Dr + sy Ds) P          (row i)
//   dv      = (rx Dr + sx Ds) UX + (ry Dr + sy Ds) UY
//   LP, L Fu_bottom, L Fu_top, LV  with the row L(i, :) held in registers
//   LY      = LP Dt^T; quad-face lifts QL_f(i, :) [Fp_f | Fu_f]
// then media scaling and the LSERK45 stage, written straight to HBM.
// Same algebra and operation order per output as the DMMA kernel
// (wedge_dmma.cu), i.e. the reference's wedge_volume_elem / surface_elem /
// scale_media / lserk (proj/src/solver.cpp:164-218, 258-335, 337-346, 541-551)
// with the lift folds of SURVEY.md A.3.
//
// Data movement: the state, record and connectivity of the next chunk of E
// wedges are copied global -> shared with cp.async (16-byte LDGSTS) into
// per-element slots whose strides are chosen to spread the shared-memory
// banks, double-buffered against the current chunk's work; L^{tri,k} and the
// quad lifts (compact [k][i] / [f][a][i] layouts: no padding bytes) and the
// residual are read per thread from HBM into registers; neighbour traces are
// L2 gathers (chunks are handed out by a global ticket, so CTAs work on a
// narrow window of the Morton-ordered element list).
#include <cuda_runtime.h>

#include <cstdlib>

#include "pdg_device.cuh"
#include "tma.cuh"

namespace pdg {

namespace {

__host__ __device__ constexpr int r2(int x) { return (x + 1) & ~1; }

/// wavefronts a warp needs to read doubles at addresses {e*S + i}, lane = H (e*NT + i) + h
/// (16 eight-byte bank pairs, distinct addresses on one pair serialise; the H
/// lanes of one (e, i) read the same address)
__host__ __device__ constexpr int conflict_degree(int S, int NT, int H) {
  int worst = 0;
  for (int b = 0; b < 16; ++b) {
    int cnt = 0;
    for (int pr = 0; pr < 32 / H; ++pr) {
      const int e = pr / NT, i = pr - e * NT;
      if (((e * S + i) & 15) == b) ++cnt;
    }
    worst = cnt > worst ? cnt : worst;
  }
  return worst;
}
/// smallest even stride >= x with the least bank conflicts for the {e*S + i} pattern
__host__ __device__ constexpr int slot_stride(int x, int NT, int H) {
  int best = r2(x), bd = conflict_degree(r2(x), NT, H);
  for (int s = r2(x) + 2; s < r2(x) + 16; s += 2) {
    const int d = conflict_degree(s, NT, H);
    if (d < bd) {
      bd = d;
      best = s;
    }
  }
  return best;
}

// the chunk-start barrier (needed anyway: cp.async completion is per thread) also
// proves every thread has left the previous chunk, so the next chunk's copy is
// issued right after it and the end-of-chunk barrier goes
#ifndef PDG_SIMT_NO_END_BARRIER
#define PDG_SIMT_NO_END_BARRIER 1
#endif
#ifndef PDG_SIMT_THREADS
#define PDG_SIMT_THREADS 128
#endif
// minimum resident CTAs per SM (register budget): 4 at N = 1 with the slice
// split (3 without), 1 above (spills), profiles/round1_simt_variants_ab.txt
#ifndef PDG_SIMT_LATE_OPS
#define PDG_SIMT_LATE_OPS 1
#endif
// rows i of the three quad-face lifts loaded with L and the residual (before
// the V / gradient phase) instead of at their point of use
#ifndef PDG_SIMT_QL_EARLY
#define PDG_SIMT_QL_EARLY 1
#endif
// threads per (wedge, triangle node) in exact mode: 2 halves the per-thread
// slice arrays (registers) and the chunk, so more CTAs are resident.  Measured
// faster at N = 1 only (-6%; +18% at N = 2, 3), profiles/round1_simt_variants_ab.txt
#ifndef PDG_SIMT_SPLIT_MAXN
#define PDG_SIMT_SPLIT_MAXN 1
#endif
#ifndef PDG_SIMT_SPLIT
#define PDG_SIMT_SPLIT(N) ((N) <= PDG_SIMT_SPLIT_MAXN ? 2 : 1)
#endif
#ifndef PDG_SIMT_MINB
#ifdef PDG_SIMT_MINB_ALL
#define PDG_SIMT_MINB(N) (PDG_SIMT_MINB_ALL)
#else
#ifndef PDG_SIMT_MINB_N1
#define PDG_SIMT_MINB_N1 (PDG_SIMT_SPLIT(1) > 1 ? 4 : 3)
#endif
#define PDG_SIMT_MINB(N) ((N) == 1 ? PDG_SIMT_MINB_N1 : (PDG_SIMT_SPLIT(N) > 1 ? 3 : 1))
#endif
#endif

// the WADG variant has no slice split: min 3 CTAs/SM at N = 1 (4 spills), 1 above
#ifndef PDG_WADG_SIMT_MINB
#define PDG_WADG_SIMT_MINB(N) ((N) == 1 ? 3 : 1)
#endif

// prefetch the streamed arrays of the chunk two tickets ahead into L2 when its
// ticket is grabbed (cp.async.bulk.prefetch.L2), so its cp.async copies and
// the per-thread operand loads hit L2 and more HBM bytes are in flight
#ifndef PDG_SIMT_L2_PREFETCH
#define PDG_SIMT_L2_PREFETCH 0
#endif

// exact mode: the flux exchange of the chunk through an mbarrier -- a thread arrives
// when its flux tasks are in shared memory, runs the flux-free part of its work
// (vertical derivative of V, the gradient / divergence / L P products) and only
// then waits for the other threads' fluxes.  Bitwise the same results; measured
// (profiles/round2_mbar_ab.txt) N = 1 / 2: -0.3 / -0.3..-1.5%; N = 3 -0.7% and +3.5%
// on two boxes, so on at N <= 2 only
#ifndef PDG_SIMT_MB
#define PDG_SIMT_MB 1
#endif
#ifndef PDG_SIMT_MB_MAXN
#define PDG_SIMT_MB_MAXN 2
#endif

template <int N, bool WADG = false>
struct SCfg {
  static_assert(nts_of(N) == nt_of(N), "the low-order kernel assumes an unpadded slice stride");
  static constexpr int NQ = nq_of(N), NT = nt_of(N), NP = npd_of(N), FW = fw_of(N), WG = wg_of(N);
  static constexpr int THREADS = PDG_SIMT_THREADS;
  // H threads per (wedge, node); thread h owns slices j = h, h + H, ... (exact mode)
  static constexpr int H = WADG ? 1 : PDG_SIMT_SPLIT(N);
  static constexpr int JH = (NQ + H - 1) / H; // slices per thread
  static constexpr int E = THREADS / (H * NT); // wedges per chunk
  static constexpr int ACT = E * NT * H;       // threads with a (wedge, node) pair
  static constexpr int SU = slot_stride(4 * NP, NT, H);
  static constexpr int SG = slot_stride(WG + kWC / 2, NT, H); // record + connectivity
  static constexpr int STAGE = E * (SU + SG);
  static constexpr int FT = 4 * NT;                   // tri fluxes: [p|u][bottom|top][NT]
  static constexpr int FQ = 6 * NQ * NQ;              // quad fluxes: [p|u][face][a][j]
  static constexpr int SF = slot_stride(FT + FQ, NT, H);
  // exact: V(j, i) at j*NT + i; WADG: the pre-lift buffer B(field, j, i) + 1/J at the cubature
  static constexpr int NC = wadg_nc(N);
  static constexpr int SV = WADG ? slot_stride(4 * NQ * NT + NC, NT, H) : slot_stride(NQ * NT, NT, H);
  // exact: Dr^T, Ds^T; WADG adds kd_m^T [m][k][i], Pw^T [q][i], Vq [q][k], R [m][f][a][i], qr, qs
  static constexpr int WTAB = WADG ? 6 * NT * NT + 2 * NC * NT + 6 * NQ * NT + 2 * NC : 0;
  static constexpr int TABLES = r2(r2(2 * NT * NT + NQ * NQ + 2 * NQ + WTAB) + ceil_div(FW, 2) + 2048 / 2);
  static constexpr size_t SMEM_BYTES = (size_t)8 * (TABLES + 2 * STAGE + E * (SF + SV) + 6); // + slots, mbarrier
  static constexpr int TASKS = ceil_div(E * FW, THREADS);
  // measured (profiles/round1_simt_noend_ab.txt): exact N = 1 -5.5%, N = 3 -1.8%,
  // N = 2 +1%; WADG N = 2 -4.1%, N = 3 -5.2%, N = 1 +2.5%
  static constexpr bool NOEND = PDG_SIMT_NO_END_BARRIER && (WADG ? N >= 2 : N != 2);
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory");
}

/// copy the state, record and connectivity of wedges [e0, e0+nel) into stage slots
template <int N, bool WADG>
__device__ __forceinline__ void load_chunk(const StageParams& p, double* stg, long long e0, int nel) {
  using C = SCfg<N, WADG>;
  constexpr int UV = 4 * C::NP / 2;     // 16-byte vectors per state block
  constexpr int GV = C::WG / 2;         // per record
  constexpr int CV = kWC / 4;           // per connectivity record (ints)
  double* sU = stg;
  double* sG = stg + C::E * C::SU;
  for (int q = threadIdx.x; q < nel * UV; q += C::THREADS) {
    const int e = q / UV, v = q - e * UV;
    cp_async16(sU + e * C::SU + 2 * v, p.u_in + (e0 + e) * 4 * C::NP + 2 * v);
  }
  for (int q = threadIdx.x; q < nel * (GV + CV); q += C::THREADS) {
    const int e = q / (GV + CV), v = q - e * (GV + CV);
    if (v < GV)
      cp_async16(sG + e * C::SG + 2 * v, p.wgeo + (e0 + e) * C::WG + 2 * v);
    else
      cp_async16(sG + e * C::SG + C::WG + 2 * (v - GV), p.wconn + (e0 + e) * kWC + 4 * (v - GV));
  }
}

template <int N, bool WADG>
__global__ void __launch_bounds__(SCfg<N, WADG>::THREADS, WADG ? PDG_WADG_SIMT_MINB(N) : PDG_SIMT_MINB(N))
    wedge_simt_kernel(const StageParams p) {
  using C = SCfg<N, WADG>;
  constexpr int NQ = C::NQ, NT = C::NT, NP = C::NP, FW = C::FW, WG = C::WG, E = C::E;
  constexpr int SU = C::SU, SG = C::SG, SF = C::SF, SV = C::SV;
  extern __shared__ __align__(16) double smem[];
  double* sDrT = smem;                 // [k][i]
  double* sDsT = sDrT + NT * NT;       // [k][i]
  double* sDt = sDsT + NT * NT;        // [j][l]
  double* sProf = sDt + NQ * NQ;       // [2][NQ]
  double* sKD = sProf + 2 * NQ;        // WADG: kd_m^T [m][k][i]
  double* sPwT = sKD + 6 * NT * NT;    // WADG: Pw^T [q][i]
  double* sVq = sPwT + C::NC * NT;     // WADG: Vq [q][k]
  double* sR = sVq + C::NC * NT;       // WADG: R_m,f [m][f][a][i]
  double* sQr = sR + 6 * NQ * NT;      // WADG: cubature points
  double* sQs = sQr + C::NC;
  int* sWface = reinterpret_cast<int*>(smem + r2(2 * NT * NT + NQ * NQ + 2 * NQ + C::WTAB));
  int* sCombo = sWface + 2 * ceil_div(FW, 2);
  double* stg = smem + C::TABLES;      // 2 stages
  double* sF = stg + 2 * C::STAGE;     // per wedge fluxes
  double* sV = sF + E * SF;            // per wedge V
  volatile long long* slot = reinterpret_cast<volatile long long*>(sV + E * SV);
  constexpr bool MBS = PDG_SIMT_MB && !WADG && N <= PDG_SIMT_MB_MAXN;
  uint64_t* fxbar = reinterpret_cast<uint64_t*>(sV + E * SV + 4); // MBS: flux exchange
  for (int q = threadIdx.x; q < NT * NT; q += C::THREADS) {
    sDrT[q] = p.DrT[q];
    sDsT[q] = p.DsT[q];
  }
  for (int q = threadIdx.x; q < NQ * NQ; q += C::THREADS) sDt[q] = p.Dt[q];
  for (int q = threadIdx.x; q < 2 * NQ; q += C::THREADS) sProf[q] = p.prof[q];
  for (int q = threadIdx.x; q < FW; q += C::THREADS) sWface[q] = p.wface_dev[q];
  if (WADG) {
    constexpr int NC = C::NC;
    const double* W = p.wadg;
    for (int q = threadIdx.x; q < 6 * NT * NT; q += C::THREADS) {
      const int m = q / (NT * NT), r = q - m * NT * NT, k = r / NT, ii = r - k * NT;
      sKD[q] = W[(m * NT + ii) * NT + k];
    }
    for (int q = threadIdx.x; q < NC * NT; q += C::THREADS) {
      const int qq = q / NT, ii = q - qq * NT;
      sPwT[q] = W[wadg_off_pw(N) + ii * NC + qq];
      sVq[q] = W[wadg_off_vq(N) + q];
    }
    for (int q = threadIdx.x; q < 6 * NQ * NT; q += C::THREADS) {
      const int mf = q / (NQ * NT), r = q - mf * NQ * NT, a = r / NT, ii = r - a * NT;
      sR[q] = W[wadg_off_r(N) + (mf * NT + ii) * NQ + a];
    }
    for (int q = threadIdx.x; q < NC; q += C::THREADS) {
      sQr[q] = W[wadg_off_q(N) + q];
      sQs[q] = W[wadg_off_q(N) + NC + q];
    }
  }
  const bool combo_smem = p.nbr_nodes_len <= 2048;
  if (combo_smem)
    for (int q = threadIdx.x; q < p.nbr_nodes_len; q += C::THREADS) sCombo[q] = p.nbr_nodes[q];
  const int* combo = combo_smem ? sCombo : p.nbr_nodes;

  const int mode = p.mode;
  const bool vol = mode & M_VOLUME, surf = mode & M_SURFACE;
  const bool lserk = mode & M_LSERK, media = mode & M_MEDIA;
  const bool first = mode & M_FIRST, accum = mode & M_ACCUM;
  const double* res_src = lserk ? (first ? nullptr : p.res) : (accum ? p.rhs_out : nullptr);
  const long long nchunk = (p.Kw_active - p.Kw_begin + E - 1) / E;
  auto nel_of = [&](long long c) -> int {
    const long long r = p.Kw_active - p.Kw_begin - c * E;
    return (int)(r < E ? r : E);
  };
  if (threadIdx.x == 0) {
    if (MBS) {
      mbar_init(fxbar, C::THREADS);
      fence_barrier_init();
    }
    slot[0] = (long long)(atomicAdd(p.ticket, 1ULL) - p.ticket_base);
    slot[1] = (long long)(atomicAdd(p.ticket, 1ULL) - p.ticket_base);
  }
  __syncthreads();
  long long c = slot[0], cn = slot[1];
  if (c < nchunk) load_chunk<N, WADG>(p, stg, p.Kw_begin + c * E, nel_of(c));
  cp_async_commit();

  constexpr int H = C::H, JH = C::JH;
  const int pr = threadIdx.x / H, h = threadIdx.x - pr * H;
  const int el = pr / NT, i = pr - el * NT; // this thread's (wedge, node); slices h + H jj
  for (int it = 0; c < nchunk; ++it) {
    double* cur = stg + (it & 1) * C::STAGE;
    // prefetch the next chunk into the other stage (it was released by the
    // trailing barrier of the previous iteration)
    if (!C::NOEND) {
      if (cn < nchunk) load_chunk<N, WADG>(p, stg + ((it + 1) & 1) * C::STAGE, p.Kw_begin + cn * E, nel_of(cn));
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    // next ticket; the slot alternates with the iteration parity so it is never
    // rewritten before every thread has read it
    if (threadIdx.x == 0) {
      const long long cf = (long long)(atomicAdd(p.ticket, 1ULL) - p.ticket_base);
      slot[2 + (it & 1)] = cf;
      if (PDG_SIMT_L2_PREFETCH && cf < nchunk) {
        const long long f0 = p.Kw_begin + cf * E;
        const long long nf = nel_of(cf);
        prefetch_l2_bulk(p.u_in + f0 * 4 * NP, (uint32_t)(nf * 32 * NP));
        if (res_src) prefetch_l2_bulk(res_src + f0 * 4 * NP, (uint32_t)(nf * 32 * NP));
        if (!WADG) {
          prefetch_l2_bulk(p.Lt + f0 * lcomp_of(N), (uint32_t)(nf * 8 * lcomp_of(N)));
          prefetch_l2_bulk(p.QL + f0 * qcomp_of(N), (uint32_t)(nf * 8 * qcomp_of(N)));
        }
        prefetch_l2_bulk(p.wgeo + f0 * WG, (uint32_t)(nf * 8 * WG));
      }
    }
    __syncthreads();
    // every thread has left the previous chunk: its stage takes the next one
    if (C::NOEND) {
      if (cn < nchunk) load_chunk<N, WADG>(p, stg + ((it + 1) & 1) * C::STAGE, p.Kw_begin + cn * E, nel_of(cn));
      cp_async_commit();
    }
    const long long e0 = p.Kw_begin + c * E;
    const int nel = nel_of(c);
    const double* sU = cur;
    const double* sG = cur + E * SU;
    const bool active = threadIdx.x < C::ACT && el < nel;
    const double* U = sU + el * SU;
    const double* G = sG + el * SG;
    const long long ge = e0 + el;

    // per-thread operands from HBM: row i of L, rows i of the quad lifts, residual
    double Lr[NT], rres[4][JH];
    double Qr[PDG_SIMT_QL_EARLY && !WADG ? 3 * NQ : 1];
    auto load_operands = [&]() {
      if (active) {
        if (!WADG) {
          const double* L = p.Lt + ge * lcomp_of(N) + i;
#pragma unroll
          for (int k = 0; k < NT; ++k) Lr[k] = __ldcs(L + k * NT);
          if (PDG_SIMT_QL_EARLY && surf) {
            const double* QL = p.QL + ge * qcomp_of(N) + i;
#pragma unroll
            for (int fa = 0; fa < 3 * NQ; ++fa) Qr[fa] = __ldcs(QL + fa * NT);
          }
        }
#pragma unroll
        for (int f = 0; f < 4; ++f)
#pragma unroll
          for (int jj = 0; jj < JH; ++jj) {
            const int j = h + H * jj;
            rres[f][jj] = res_src && j < NQ ? __ldcs(res_src + ge * 4 * NP + f * NP + j * NT + i) : 0.0;
          }
      }
    };
    // per-thread operands from HBM (row i of L, residual): issued before the
    // flux phase, or (PDG_SIMT_LATE_OPS) right after the flux arithmetic so the
    // gathered traces and these registers are not live at the same time
    if (!PDG_SIMT_LATE_OPS) load_operands();

    // ---- numerical fluxes of the chunk -------------------------------------------
    if (surf) {
      double nbv[C::TASKS][4];
#pragma unroll
      for (int q = 0; q < C::TASKS; ++q) {
        const int m = threadIdx.x + C::THREADS * q;
        if (m < nel * FW) {
          const int e = m / FW, fm = m - e * FW;
          const int f = fm < NT ? 0 : (fm < 2 * NT ? 1 : 2 + (fm - 2 * NT) / (NQ * NQ));
          const int loc = fm < 2 * NT ? fm - f * NT : (fm - 2 * NT) - (f - 2) * NQ * NQ;
          const int* Cn = reinterpret_cast<const int*>(sG + e * SG + WG);
          const int nbr = Cn[2 * f];
          if (nbr >= 0) {
            const int node = combo[Cn[2 * f + 1] * p.max_nfp + loc];
            const double* src;
            int fs;
            if (nbr < p.Kw) {
              src = p.u_in + (long long)nbr * 4 * NP + node;
              fs = NP;
            } else {
              src = p.u_in + p.tet_base + (long long)(nbr - p.Kw) * 4 * npt_of(N) + node;
              fs = npt_of(N);
            }
            nbv[q][0] = __ldg(src);
            nbv[q][1] = __ldg(src + fs);
            nbv[q][2] = __ldg(src + 2 * fs);
            nbv[q][3] = __ldg(src + 3 * fs);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < C::TASKS; ++q) {
        const int m = threadIdx.x + C::THREADS * q;
        if (m < nel * FW) {
          const int e = m / FW, fm = m - e * FW;
          const int f = fm < NT ? 0 : (fm < 2 * NT ? 1 : 2 + (fm - 2 * NT) / (NQ * NQ));
          const int loc = fm < 2 * NT ? fm - f * NT : (fm - 2 * NT) - (f - 2) * NQ * NQ;
          const double* Ue = sU + e * SU;
          const double* Ge = sG + e * SG;
          const int* Cn = reinterpret_cast<const int*>(Ge + WG);
          const int my = sWface[fm];
          const double pm = Ue[my];
          const double nx = Ge[w_nrm(N) + 3 * f], ny = Ge[w_nrm(N) + 3 * f + 1], nz = Ge[w_nrm(N) + 3 * f + 2];
          const double taup = Ge[w_taup(N) + f], tauu = Ge[w_tauu(N) + f];
          double fp, fu;
          if (Cn[2 * f] >= 0) {
            const double dp = nbv[q][0] - pm;
            const double dun = nx * (nbv[q][1] - Ue[NP + my]) + ny * (nbv[q][2] - Ue[2 * NP + my]) +
                               nz * (nbv[q][3] - Ue[3 * NP + my]);
            fp = 0.5 * (taup * dp - dun);
            fu = 0.5 * (tauu * dun - dp);
          } else {
            const double dp = -2.0 * pm; // reflective: p+ = -p-, u+ = u-
            fp = 0.5 * taup * dp;
            fu = -0.5 * dp;
          }
          double* Fe = sF + e * SF;
          if (f < 2) {
            Fe[f * NT + loc] = fp;            // Ftp[f][loc]
            Fe[2 * NT + f * NT + loc] = fu;   // Ftu[f][loc]
          } else {
            Fe[4 * NT + (f - 2) * NQ * NQ + loc] = fp;            // Fqp[f-2][a][j]
            Fe[4 * NT + 3 * NQ * NQ + (f - 2) * NQ * NQ + loc] = fu; // Fqu
          }
        }
      }
    }
    if (PDG_SIMT_LATE_OPS) load_operands();
    if (WADG)
      for (int q = threadIdx.x; q < nel * C::NC; q += C::THREADS) {
        const int e = q / C::NC, qq = q - e * C::NC;
        const double* Ge = sG + e * SG;
        sV[e * SV + 4 * NQ * NT + qq] = 1.0 / (Ge[w_jac(N)] + Ge[w_jac(N) + 1] * sQr[qq] + Ge[w_jac(N) + 2] * sQs[qq]);
      }
    if (MBS)
      mbar_arrive(fxbar);
    else
      __syncthreads();
    if constexpr (!WADG) {
    // ---- V column i, gradients, L products, quad lifts (own slices j = h + H jj) -------
    double rp[JH], rux[JH], ruy[JH], ruz[JH], lp[JH];
    double lf0 = 0.0, lf1 = 0.0, dV[JH];
#pragma unroll
    for (int jj = 0; jj < JH; ++jj) rp[jj] = rux[jj] = ruy[jj] = ruz[jj] = lp[jj] = 0.0;
    // V column i: the vertical derivative dV plus the bottom / top pressure lifts
    auto write_V = [&]() {
      const double* Fe = sF + el * SF;
      const double jfb = G[W_JFB], jft = G[W_JFT];
      const double fb = surf ? jfb * Fe[i] : 0.0, ftop = surf ? jft * Fe[NT + i] : 0.0;
      double* Ve = sV + el * SV;
#pragma unroll
      for (int jj = 0; jj < JH; ++jj) {
        const int j = h + H * jj;
        if (j < NQ) Ve[j * NT + i] = -dV[jj] + fb * sProf[j] + ftop * sProf[NQ + j];
      }
    };
    if (active) {
      const double* Fe = sF + el * SF;
      const double tzJ = G[W_TZJ], jfb = G[W_JFB], jft = G[W_JFT];
      {
#pragma unroll
        for (int jj = 0; jj < JH; ++jj) {
          const int j = h + H * jj;
          dV[jj] = 0.0;
          if (j < NQ && vol) {
            const double sx_ = G[W_TXJ + j], sy_ = G[w_tyj(N) + j];
#pragma unroll
            for (int l = 0; l < NQ; ++l) {
              const double dt = sDt[j * NQ + l];
              dV[jj] += U[NP + l * NT + i] * (sx_ * dt);
              dV[jj] += U[2 * NP + l * NT + i] * (sy_ * dt);
              dV[jj] += U[3 * NP + l * NT + i] * (tzJ * dt);
            }
          }
        }
        if (!MBS) write_V();
      }
      const double rx = G[W_RX], ry = G[W_RY], sxm = G[W_SX], sym = G[W_SY];
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        const double lk = Lr[k];
        double cx = 0.0, cy = 0.0;
        if (vol) {
          const double dr = sDrT[k * NT + i], ds = sDsT[k * NT + i];
          cx = rx * dr + sxm * ds;
          cy = ry * dr + sym * ds;
        }
#pragma unroll
        for (int jj = 0; jj < JH; ++jj) {
          const int j = h + H * jj;
          if (j < NQ) {
            const double pk = U[j * NT + k];
            lp[jj] += lk * pk;
            if (vol) {
              rux[jj] -= cx * pk;
              ruy[jj] -= cy * pk;
              rp[jj] -= cx * U[NP + j * NT + k] + cy * U[2 * NP + j * NT + k];
            }
          }
        }
        if (surf && !MBS) {
          lf0 += lk * Fe[2 * NT + k];
          lf1 += lk * Fe[3 * NT + k];
        }
      }
    }
    if (MBS) {
      mbar_wait(fxbar, it & 1); // every thread's fluxes of the chunk are in
      if (active) {
        write_V();
        if (surf) {
          const double* Fe = sF + el * SF;
#pragma unroll
          for (int k = 0; k < NT; ++k) {
            lf0 += Lr[k] * Fe[2 * NT + k];
            lf1 += Lr[k] * Fe[3 * NT + k];
          }
        }
      }
    }
    if (active) {
      const double* Fe = sF + el * SF;
      if (surf) {
        const double* QL = p.QL + ge * qcomp_of(N) + i;
        const double* nrm = G + w_nrm(N);
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          double qu[JH];
#pragma unroll
          for (int jj = 0; jj < JH; ++jj) qu[jj] = 0.0;
#pragma unroll
          for (int a = 0; a < NQ; ++a) {
            const double q = PDG_SIMT_QL_EARLY ? Qr[(f * NQ + a) % (PDG_SIMT_QL_EARLY ? 3 * NQ : 1)]
                                               : __ldcs(QL + (f * NQ + a) * NT);
#pragma unroll
            for (int jj = 0; jj < JH; ++jj) {
              const int j = h + H * jj;
              if (j < NQ) {
                rp[jj] += q * Fe[4 * NT + (f * NQ + a) * NQ + j];
                qu[jj] += q * Fe[4 * NT + 3 * NQ * NQ + (f * NQ + a) * NQ + j];
              }
            }
          }
          const double nx = nrm[3 * (f + 2)], ny = nrm[3 * (f + 2) + 1], nz = nrm[3 * (f + 2) + 2];
#pragma unroll
          for (int jj = 0; jj < JH; ++jj) {
            rux[jj] += nx * qu[jj];
            ruy[jj] += ny * qu[jj];
            ruz[jj] += nz * qu[jj];
          }
        }
      }
    }
    __syncthreads(); // V complete
    // the whole column LP(:, i) for LY: the other slices come from the partner lanes
    double lpa[NQ];
#pragma unroll
    for (int l = 0; l < NQ; ++l) {
      const int hh = l % H, jj = l / H;
      double v = lp[jj];
      if (H > 1) v = __shfl_sync(0xffffffffu, v, (threadIdx.x & 31) - h + hh);
      lpa[l] = v;
    }

    // ---- L V, L Y, tri-face velocity lifts, media, LSERK -----------------------------
    if (active) {
      const double* Ve = sV + el * SV;
      const double tzJ = G[W_TZJ], jfb = G[W_JFB], jft = G[W_JFT];
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        const double lk = Lr[k];
#pragma unroll
        for (int jj = 0; jj < JH; ++jj) {
          const int j = h + H * jj;
          if (j < NQ) rp[jj] += lk * Ve[j * NT + k];
        }
      }
      const double* nrm = G + w_nrm(N);
      const double kappa = G[W_KAPPA], irho = G[W_IRHO];
#pragma unroll
      for (int jj = 0; jj < JH; ++jj) {
        const int j = h + H * jj;
        if (j >= NQ) continue;
        if (vol) {
          double ly = 0.0;
#pragma unroll
          for (int l = 0; l < NQ; ++l) ly += lpa[l] * sDt[j * NQ + l];
          rux[jj] -= G[W_TXJ + j] * ly;
          ruy[jj] -= G[w_tyj(N) + j] * ly;
          ruz[jj] -= tzJ * ly;
        }
        if (surf) {
          const double t0 = jfb * sProf[j] * lf0, t1 = jft * sProf[NQ + j] * lf1;
          rux[jj] += nrm[0] * t0 + nrm[3] * t1;
          ruy[jj] += nrm[1] * t0 + nrm[4] * t1;
          ruz[jj] += nrm[2] * t0 + nrm[5] * t1;
        }
        if (media) {
          rp[jj] *= kappa;
          rux[jj] *= irho;
          ruy[jj] *= irho;
          ruz[jj] *= irho;
        }
        const double rv[4] = {rp[jj], rux[jj], ruy[jj], ruz[jj]};
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          const int o = f * NP + j * NT + i;
          const long long go = ge * 4 * NP + o;
          if (lserk) {
            const double rr = first ? p.dt * rv[f] : p.a * rres[f][jj] + p.dt * rv[f];
            __stcs(p.res + go, rr);
            __stcs(p.u_out + go, U[o] + p.b * rr);
          } else {
            __stcs(p.rhs_out + go, accum ? rres[f][jj] + rv[f] : rv[f]);
          }
        }
      }
    }
    } else {
    // ---- WADG: Ltilde row i, pre-lift buffer B(field, j, i), then rhs = Ltilde B -------
    constexpr int NC = C::NC;
    double bp[NQ], bx[NQ], by[NQ], bz[NQ];
#pragma unroll
    for (int j = 0; j < NQ; ++j) bp[j] = bx[j] = by[j] = bz[j] = 0.0;
    if (active) {
      const double* Fe = sF + el * SF;
      const double* IJ = sV + el * SV + 4 * NQ * NT;
      const double j0 = G[w_jac(N)], jr = G[w_jac(N) + 1], js = G[w_jac(N) + 2];
      // Ltilde(i, :) = sum_q Pw(i, q) / J_q Vq(q, :)
#pragma unroll
      for (int k = 0; k < NT; ++k) Lr[k] = 0.0;
      for (int q = 0; q < NC; ++q) {
        const double a = sPwT[q * NT + i] * IJ[q];
#pragma unroll
        for (int k = 0; k < NT; ++k) Lr[k] += a * sVq[q * NT + k];
      }
      const double tzJ = G[W_TZJ];
      if (vol) {
        // K-folded horizontal derivatives: K (rx Dr + sx Ds) = sum_m c_m kd_m
        const double rx = G[W_RX], ry = G[W_RY], sxm = G[W_SX], sym = G[W_SY];
        const double cxm[6] = {rx * j0, rx * jr, rx * js, sxm * j0, sxm * jr, sxm * js};
        const double cym[6] = {ry * j0, ry * jr, ry * js, sym * j0, sym * jr, sym * js};
#pragma unroll
        for (int k = 0; k < NT; ++k) {
          double cx = 0.0, cy = 0.0;
#pragma unroll
          for (int m = 0; m < 6; ++m) {
            const double d = sKD[(m * NT + k) * NT + i];
            cx += cxm[m] * d;
            cy += cym[m] * d;
          }
#pragma unroll
          for (int j = 0; j < NQ; ++j) {
            const double pk = U[j * NT + k];
            bx[j] -= cx * pk;
            by[j] -= cy * pk;
            bp[j] -= cx * U[NP + j * NT + k] + cy * U[2 * NP + j * NT + k];
          }
        }
        // vertical terms
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
          const double sx_ = G[W_TXJ + j], sy_ = G[w_tyj(N) + j];
          double d = 0.0, pdt = 0.0;
#pragma unroll
          for (int l = 0; l < NQ; ++l) {
            const double dt = sDt[j * NQ + l];
            d += U[NP + l * NT + i] * (sx_ * dt) + U[2 * NP + l * NT + i] * (sy_ * dt) + U[3 * NP + l * NT + i] * (tzJ * dt);
            pdt += dt * U[l * NT + i];
          }
          bp[j] -= d;
          bx[j] -= sx_ * pdt;
          by[j] -= sy_ * pdt;
          bz[j] -= tzJ * pdt;
        }
      }
      if (surf) {
        const double* nrm = G + w_nrm(N);
        const double jfb = G[W_JFB], jft = G[W_JFT];
        const double tpb = jfb * Fe[i], tpt = jft * Fe[NT + i], tub = jfb * Fe[2 * NT + i], tut = jft * Fe[3 * NT + i];
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
          const double pb = sProf[j], pt = sProf[NQ + j];
          bp[j] += tpb * pb + tpt * pt;
          const double t0 = tub * pb, t1 = tut * pt;
          bx[j] += nrm[0] * t0 + nrm[3] * t1;
          by[j] += nrm[1] * t0 + nrm[4] * t1;
          bz[j] += nrm[2] * t0 + nrm[5] * t1;
        }
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          const double jf0 = G[w_jac(N) + 3 + 2 * f], jf1 = G[w_jac(N) + 4 + 2 * f];
          double qu[NQ];
#pragma unroll
          for (int j = 0; j < NQ; ++j) qu[j] = 0.0;
#pragma unroll
          for (int a = 0; a < NQ; ++a) {
            const double q = jf0 * sR[(f * NQ + a) * NT + i] + jf1 * sR[((3 + f) * NQ + a) * NT + i];
#pragma unroll
            for (int j = 0; j < NQ; ++j) {
              bp[j] += q * Fe[4 * NT + (f * NQ + a) * NQ + j];
              qu[j] += q * Fe[4 * NT + 3 * NQ * NQ + (f * NQ + a) * NQ + j];
            }
          }
          const double nx = nrm[3 * (f + 2)], ny = nrm[3 * (f + 2) + 1], nz = nrm[3 * (f + 2) + 2];
#pragma unroll
          for (int j = 0; j < NQ; ++j) {
            bx[j] += nx * qu[j];
            by[j] += ny * qu[j];
            bz[j] += nz * qu[j];
          }
        }
      }
      double* Be = sV + el * SV;
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        Be[j * NT + i] = bp[j];
        Be[(NQ + j) * NT + i] = bx[j];
        Be[(2 * NQ + j) * NT + i] = by[j];
        Be[(3 * NQ + j) * NT + i] = bz[j];
      }
    }
    __syncthreads(); // B complete
    if (active) {
      const double* Be = sV + el * SV;
      const double kappa = G[W_KAPPA], irho = G[W_IRHO];
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
          double r = 0.0;
#pragma unroll
          for (int k = 0; k < NT; ++k) r += Lr[k] * Be[(f * NQ + j) * NT + k];
          if (media) r *= f == 0 ? kappa : irho;
          const int o = f * NP + j * NT + i;
          const long long go = ge * 4 * NP + o;
          if (lserk) {
            const double rr = first ? p.dt * r : p.a * rres[f][j] + p.dt * r;
            __stcs(p.res + go, rr);
            __stcs(p.u_out + go, U[o] + p.b * rr);
          } else {
            __stcs(p.rhs_out + go, accum ? rres[f][j] + r : r);
          }
        }
    }
    }
    if (!C::NOEND) __syncthreads(); // the stage and the work buffers are free again
    c = cn;
    cn = slot[2 + (it & 1)];
  }
  cp_async_wait<0>();
}

template <int N, bool WADG>
cudaError_t launch_simt_N(const StageParams& p, cudaStream_t s) {
  using C = SCfg<N, WADG>;
  // one-time setup per device (the smem attribute is per device)
  static int grid_cap[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  auto kern = wedge_simt_kernel<N, WADG>;
  if (grid_cap[dev] == 0) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::SMEM_BYTES);
    grid_cap[dev] = sms * (per_sm > 0 ? per_sm : 1);
  }
  if (p.info) *p.info = LaunchInfo{};
  if (p.Kw_active - p.Kw_begin <= 0) return cudaSuccess;
  const long long nchunk = (p.Kw_active - p.Kw_begin + C::E - 1) / C::E;
  const int grid = (int)(nchunk < grid_cap[dev] ? nchunk : grid_cap[dev]);
  StageParams q = p;
  q.ticket_base = *p.ticket_host_next;
  // every CTA grabs until it gets two tickets past the end (one in flight)
  *p.ticket_host_next += (unsigned long long)nchunk + 2ull * (unsigned long long)grid;
  kern<<<grid, C::THREADS, C::SMEM_BYTES, s>>>(q);
  if (p.info) *p.info = LaunchInfo{1, (long long)grid, nchunk, C::E};
  return cudaGetLastError();
}

} // namespace

int wedge_simt_max_degree() {
  static const int env = [] {
    const char* v = std::getenv("PDG_SIMT_MAX_N");
    return v ? std::atoi(v) : 0;
  }();
  return env > 0 ? (env < 4 ? env : 4) : 3;
}

cudaError_t launch_wedge_simt_stage(int N, const StageParams& p, cudaStream_t s) {
  switch (N) {
    case 1: return launch_simt_N<1, false>(p, s);
    case 2: return launch_simt_N<2, false>(p, s);
    case 3: return launch_simt_N<3, false>(p, s);
    case 4: return launch_simt_N<4, false>(p, s);
  }
  return cudaErrorInvalidValue;
}

int wedge_wadg_simt_max_degree() {
  static const int env = [] {
    const char* v = std::getenv("PDG_WADG_SIMT_MAX_N");
    return v ? std::atoi(v) : -1;
  }();
  return env >= 0 ? (env < 3 ? env : 3) : 3;
}

cudaError_t launch_wedge_wadg_simt_stage(int N, const StageParams& p, cudaStream_t s) {
  switch (N) {
    case 1: return launch_simt_N<1, true>(p, s);
    case 2: return launch_simt_N<2, true>(p, s);
    case 3: return launch_simt_N<3, true>(p, s);
  }
  return cudaErrorInvalidValue;
}

} // namespace pdg
