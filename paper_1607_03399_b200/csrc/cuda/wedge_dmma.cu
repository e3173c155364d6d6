// Fused wedge stage kernel on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64).
//
// Work decomposition: one warp owns one wedge at a time (warp-private pipeline,
// no CTA-wide barriers after setup).  Per element the per-stage work is a
// handful of small dense products with tri-node rows i (tiles of 8) and slice
// columns j, all issued as 8x8x4 DMMA tiles:
//   G1  V^T   = -(UX^T (txJ Dt)^T + UY^T (tyJ Dt)^T + tzJ UZ^T Dt^T)   (K = slices)
//   G2  gx    = (rx Dr + sx Ds) P,  gy = (ry Dr + sy Ds) P,
//       dv    = (rx Dr + sx Ds) UX + (ry Dr + sy Ds) UY                (K = tri nodes)
//   G3  [LP | L Fu_bottom | L Fu_top] = L [P | Fu0 | Fu1],  LV = L V     (K = tri nodes)
//   G4  LY    = LP Dt^T   (Dt along the slices; A fragments via quad shuffles)
//   G5  [qp | qx | qy | qz] = [QL_0 QL_1 QL_2] [Fp ; n_c Fu] over the 3 quad faces
// The metric is folded into the A fragments (rx Dr + sx Ds), the bottom/top
// triangular-face pressure lifts are folded into V before G3,
// and the epilogue adds the n-scaled velocity lifts, media scaling and the
// LSERK45 stage update res = a res + dt rhs, u = u + b res in shared memory.
//
// Data movement per element (all bulk / async, 16-byte granular):
//   TMA loads  (cp.async.bulk -> mbarrier): state, residual, L^{tri,k}, quad
//              lifts, geometry/media record, connectivity record;
//   gathers    neighbour face traces (LDG, L2-resident thanks to Morton order);
//   TMA stores (cp.async.bulk global <- shared): updated state and residual.
// Each warp double-buffers its stage so the next element's loads overlap the
// current element's tensor-core work.
// Reference arithmetic: wedge_volume_elem / surface_elem / scale_media / lserk
// (proj/src/solver.cpp:164-218, 258-335, 337-346, 541-551).
#include <cuda_runtime.h>

#include "pdg_device.cuh"
#include "tma.cuh"

namespace pdg {

namespace {

__host__ __device__ constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ constexpr int r4(int x) { return (x + 3) & ~3; }
__host__ __device__ constexpr int r2(int x) { return (x + 1) & ~1; }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }

constexpr int kComboCap = 4096; // ints of neighbour node maps kept in shared memory

template <int N>
struct DCfg {
  static constexpr int NQ = nq_of(N), NT = nt_of(N), NP = npw_of(N), FW = fw_of(N), WG = wg_of(N);
  static constexpr int IT = cdiv(NT, 8), MP = 8 * IT;     // tri-node row tiles
  static constexpr int KS = cdiv(NT, 4), KP = 4 * KS;     // k-steps over tri nodes
  static constexpr int JT = cdiv(NQ, 8), NPJ = 8 * JT;    // slice column tiles
  static constexpr int JTL = cdiv(NQ + 2, 8);             // [P | Fu0 | Fu1] tiles
  static constexpr int KT = cdiv(NQ, 4), KTP = 4 * KT;    // k-steps over slices
  static constexpr int KQ = cdiv(3 * NQ, 4);              // k-steps over quad-face nodes
  // per-stage buffers (doubles); each row 16-byte aligned
  static constexpr int USTR = r4(4 * NP) + 2;
  static constexpr int RSTR = USTR;
  static constexpr int LSTR = r4(lg_of(N)) + 2;
  static constexpr int QSTR = r4(qg_of(N)) + 2;
  static constexpr int STAGE = r2(USTR + RSTR + LSTR + QSTR + WG + kWC / 2);
  // work buffers, padded so that padded fragment reads stay in bounds
  static constexpr int VS = r2(cmax(NP, (NPJ - 1) * NT + KP) + 8);
  static constexpr int FPAD = r2(cmax(FW, 2 * NT + (4 * KQ - 1) * NQ + NPJ) + 8);
  static constexpr int NSTAGE = 2;
  static constexpr int PER_WARP = 2 + NSTAGE * STAGE + VS + 2 * FPAD;
  static constexpr int TABLES = r2(2 * KP * MP + KTP * NPJ + 2 * NQ + cdiv(FW, 2) + kComboCap / 2);
  static constexpr int SMEM_BUDGET = 225 * 1024;
  static constexpr int WPB_SMEM = (SMEM_BUDGET / 8 - TABLES) / PER_WARP;
  static constexpr int WPB = cmin(16, cmax(1, WPB_SMEM));
  static constexpr size_t SMEM_BYTES = (size_t)8 * (TABLES + WPB * PER_WARP);
  static constexpr int QF = cdiv(FW, 32);      // face nodes per lane
  static constexpr int QB = cmin(QF, 5);       // gathered per batch
};

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int N>
__device__ __forceinline__ void load_element(const StageParams& p, double* stg, long long e, const double* res_src,
                                             uint64_t* bar) {
  using C = DCfg<N>;
  constexpr int NP = C::NP;
  double* U = stg;
  double* R = U + C::USTR;
  double* L = R + C::RSTR;
  double* Q = L + C::LSTR;
  double* G = Q + C::QSTR;
  const uint32_t bytes = 8u * (4 * NP + lg_of(N) + qg_of(N) + C::WG) + 4u * kWC + (res_src ? 32u * NP : 0u);
  mbar_arrive_expect_tx(bar, bytes);
  tma_load_1d(U, p.u_in + e * 4 * NP, 32 * NP, bar);
  if (res_src) tma_load_1d(R, res_src + e * 4 * NP, 32 * NP, bar);
  tma_load_1d(L, p.Lt + e * lg_of(N), 8 * lg_of(N), bar);
  tma_load_1d(Q, p.QL + e * qg_of(N), 8 * qg_of(N), bar);
  tma_load_1d(G, p.wgeo + e * C::WG, 8 * C::WG, bar);
  tma_load_1d(G + C::WG, p.wconn + e * kWC, 4 * kWC, bar);
}

template <int N>
__global__ void __launch_bounds__(32 * DCfg<N>::WPB, 1) wedge_dmma_kernel(const StageParams p) {
  using C = DCfg<N>;
  constexpr int NQ = C::NQ, NT = C::NT, NP = C::NP, FW = C::FW, WG = C::WG;
  constexpr int IT = C::IT, MP = C::MP, KS = C::KS, KP = C::KP, JT = C::JT, NPJ = C::NPJ;
  constexpr int JTL = C::JTL, KT = C::KT, KTP = C::KTP, KQ = C::KQ, WPB = C::WPB;
  extern __shared__ __align__(16) double smem[];

  // ---- shared reference tables (zero padded to whole fragments) ------------
  double* sDr = smem;                    // [KP][MP]: Dr(i,k) at k*MP + i
  double* sDs = sDr + KP * MP;
  double* sDtB = sDs + KP * MP;          // [KTP][NPJ]: Dt(j,l) at l*NPJ + j
  double* sProf = sDtB + KTP * NPJ;      // [2][NQ]
  int* sWface = reinterpret_cast<int*>(sProf + 2 * NQ);
  int* sCombo = sWface + 2 * cdiv(FW, 2);
  const int nthreads = 32 * WPB;
  for (int q = threadIdx.x; q < C::SMEM_BYTES / 8; q += nthreads) smem[q] = 0.0;
  __syncthreads();
  for (int q = threadIdx.x; q < KP * MP; q += nthreads) {
    const int k = q / MP, i = q - k * MP;
    if (k < NT && i < NT) {
      sDr[q] = p.DrT[k * NT + i];
      sDs[q] = p.DsT[k * NT + i];
    }
  }
  for (int q = threadIdx.x; q < KTP * NPJ; q += nthreads) {
    const int l = q / NPJ, j = q - l * NPJ;
    if (l < NQ && j < NQ) sDtB[q] = p.Dt[j * NQ + l];
  }
  for (int q = threadIdx.x; q < 2 * NQ; q += nthreads) sProf[q] = p.prof[q];
  for (int q = threadIdx.x; q < FW; q += nthreads) sWface[q] = p.wface_dev[q];
  const bool combo_in_smem = p.nbr_nodes_len <= kComboCap;
  if (combo_in_smem)
    for (int q = threadIdx.x; q < p.nbr_nodes_len; q += nthreads) sCombo[q] = p.nbr_nodes[q];
  const int* combo = combo_in_smem ? sCombo : p.nbr_nodes;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  double* wbase = smem + C::TABLES + (size_t)warp * C::PER_WARP;
  uint64_t* bar = reinterpret_cast<uint64_t*>(wbase);
  double* stg0 = wbase + 2;
  double* V = stg0 + C::NSTAGE * C::STAGE;
  double* Fp = V + C::VS;
  double* Fu = Fp + C::FPAD;
  if (lane == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_barrier_init();
  }
  __syncthreads();

  const int mode = p.mode;
  const bool vol = mode & M_VOLUME, surf = mode & M_SURFACE, lserk = mode & M_LSERK;
  const bool first = mode & M_FIRST, accum = mode & M_ACCUM, media = mode & M_MEDIA;
  const double* res_src = lserk ? (first ? nullptr : p.res) : (accum ? p.rhs_out : nullptr);
  const long long total_warps = (long long)gridDim.x * WPB;
  long long e = (long long)blockIdx.x * WPB + warp;
  if (e < p.Kw && lane == 0) load_element<N>(p, stg0, e, res_src, bar);

  for (int n = 0; e < p.Kw; ++n) {
    const int s = n & 1;
    const long long en = e + total_warps;
    double* U = stg0 + s * C::STAGE;
    double* R = U + C::USTR;
    const double* Ls = R + C::RSTR;
    const double* Qs = Ls + C::LSTR;
    const double* G = Qs + C::QSTR;
    const int* Cn = reinterpret_cast<const int*>(G + WG);
    if (lane == 0 && en < p.Kw) {
      bulk_wait_read<0>(); // the previous element's stores no longer read stage s^1
      fence_proxy_async_smem();
      load_element<N>(p, stg0 + (s ^ 1) * C::STAGE, en, res_src, bar + (s ^ 1));
    }
    mbar_wait(bar + s, (n >> 1) & 1);

    // ---- numerical fluxes on all face nodes (gathers batched per lane) -------
    if (surf) {
#pragma unroll
      for (int q0 = 0; q0 < C::QF; q0 += C::QB) {
        double nb[C::QB][4];
#pragma unroll
        for (int qq = 0; qq < C::QB; ++qq) {
          const int m = lane + 32 * (q0 + qq);
          if (q0 + qq < C::QF && m < FW) {
            int f, loc;
            if (m < NT) {
              f = 0;
              loc = m;
            } else if (m < 2 * NT) {
              f = 1;
              loc = m - NT;
            } else {
              const int r = m - 2 * NT;
              f = 2 + r / (NQ * NQ);
              loc = r - (f - 2) * NQ * NQ;
            }
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
              nb[qq][0] = __ldg(src);
              nb[qq][1] = __ldg(src + fs);
              nb[qq][2] = __ldg(src + 2 * fs);
              nb[qq][3] = __ldg(src + 3 * fs);
            }
          }
        }
#pragma unroll
        for (int qq = 0; qq < C::QB; ++qq) {
          const int m = lane + 32 * (q0 + qq);
          if (q0 + qq < C::QF && m < FW) {
            const int f = m < NT ? 0 : (m < 2 * NT ? 1 : 2 + (m - 2 * NT) / (NQ * NQ));
            const int my = sWface[m];
            const double pm = U[my];
            const double nx = G[w_nrm(N) + 3 * f], ny = G[w_nrm(N) + 3 * f + 1], nz = G[w_nrm(N) + 3 * f + 2];
            const double taup = G[w_taup(N) + f], tauu = G[w_tauu(N) + f];
            double fp, fu;
            if (Cn[2 * f] >= 0) {
              const double dp = nb[qq][0] - pm;
              const double dux = nb[qq][1] - U[NP + my];
              const double duy = nb[qq][2] - U[2 * NP + my];
              const double duz = nb[qq][3] - U[3 * NP + my];
              const double dun = nx * dux + ny * duy + nz * duz;
              fp = 0.5 * (taup * dp - dun);
              fu = 0.5 * (tauu * dun - dp);
            } else {
              const double dp = -2.0 * pm; // reflective: p+ = -p-, u+ = u-
              fp = 0.5 * taup * dp;
              fu = -0.5 * dp;
            }
            Fp[m] = fp;
            Fu[m] = fu;
          }
        }
      }
    }

    // ---- G1: vertical part of the pressure pre-lift buffer V[j][i] ---------
    if (vol) {
      const double tzJ = G[W_TZJ];
#pragma unroll
      for (int t = 0; t < IT; ++t) {
        const int i = 8 * t + gid;
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) {
          const int jb = 8 * jt + gid;
          const int jc = jb < NQ ? jb : NQ - 1;
          const double sx_ = G[W_TXJ + jc], sy_ = G[w_tyj(N) + jc];
          double d[2] = {0.0, 0.0};
#pragma unroll
          for (int s2 = 0; s2 < KT; ++s2) {
            const int l = 4 * s2 + tig;
            const double bd = sDtB[l * NPJ + jb];
            dmma(d, U[NP + l * NT + i], sx_ * bd);
            dmma(d, U[2 * NP + l * NT + i], sy_ * bd);
            dmma(d, U[3 * NP + l * NT + i], tzJ * bd);
          }
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int j = 8 * jt + 2 * tig + c;
            if (i < NT && j < NQ) V[j * NT + i] = -d[c];
          }
        }
      }
    } else {
      for (int q = lane; q < NP; q += 32) V[q] = 0.0;
    }
    __syncwarp();
    // bottom / top pressure lifts share the L application of V
    if (surf) {
      const double jfb = G[W_JFB], jft = G[W_JFT];
      for (int q = lane; q < NP; q += 32) {
        const int j = q / NT, i = q - j * NT;
        V[q] += jfb * sProf[j] * Fp[i] + jft * sProf[NQ + j] * Fp[NT + i];
      }
    }
    __syncwarp();

    // ---- per row tile: G2, G3, G4, G5 and the epilogue ------------------------
    const double rx = G[W_RX], ry = G[W_RY], sxm = G[W_SX], sym = G[W_SY];
    const double tzJ = G[W_TZJ];
    const double jfb = G[W_JFB], jft = G[W_JFT];
    const double kappa = G[W_KAPPA], irho = G[W_IRHO];
    const double* nrm = G + w_nrm(N);
    // lane-constant column sources for the [P | Fu0 | Fu1] operand
    const double* lcol[JTL];
#pragma unroll
    for (int jt = 0; jt < JTL; ++jt) {
      const int nc = 8 * jt + gid;
      lcol[jt] = nc < NQ ? U + nc * NT : (nc == NQ ? Fu : (nc == NQ + 1 ? Fu + NT : nullptr));
    }
#pragma unroll 1
    for (int t = 0; t < IT; ++t) {
      const int i = 8 * t + gid;
      double gx[JT][2], gy[JT][2], dv[JT][2], lv[JT][2], lp[JTL][2];
#pragma unroll
      for (int jt = 0; jt < JT; ++jt) gx[jt][0] = gx[jt][1] = gy[jt][0] = gy[jt][1] = dv[jt][0] = dv[jt][1] =
          lv[jt][0] = lv[jt][1] = 0.0;
#pragma unroll
      for (int jt = 0; jt < JTL; ++jt) lp[jt][0] = lp[jt][1] = 0.0;
#pragma unroll
      for (int s2 = 0; s2 < KS; ++s2) {
        const int k = 4 * s2 + tig;
        const double la = k < NT ? Ls[k * NT + i] : 0.0;
        if (vol) {
          const double dr = sDr[k * MP + i], ds = sDs[k * MP + i];
          const double cx = rx * dr + sxm * ds, cy = ry * dr + sym * ds;
#pragma unroll
          for (int jt = 0; jt < JT; ++jt) {
            const int jb = 8 * jt + gid;
            const double bp = U[jb * NT + k], bx = U[NP + jb * NT + k], by = U[2 * NP + jb * NT + k];
            dmma(gx[jt], cx, bp);
            dmma(gy[jt], cy, bp);
            dmma(dv[jt], cx, bx);
            dmma(dv[jt], cy, by);
          }
        }
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) dmma(lv[jt], la, V[(8 * jt + gid) * NT + k]);
        if (vol || surf) {
#pragma unroll
          for (int jt = 0; jt < JTL; ++jt) {
            const double b = lcol[jt] ? lcol[jt][k] : 0.0;
            dmma(lp[jt], la, b);
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
          const int src = gid * 4 + 2 * (s2 & 1) + (tig >> 1);
          const double v0 = __shfl_sync(0xffffffffu, lp[s2 >> 1][0], src);
          const double v1 = __shfl_sync(0xffffffffu, lp[s2 >> 1][1], src);
          const double a = (tig & 1) ? v1 : v0;
#pragma unroll
          for (int jt = 0; jt < JT; ++jt) dmma(ly[jt], a, sDtB[(4 * s2 + tig) * NPJ + 8 * jt + gid]);
        }
      }
      // L fu_bottom / L fu_top of this row (columns NQ and NQ+1 of the G3 product)
      constexpr int c0 = NQ % 8, c1 = (NQ + 1) % 8;
      const double lf0 = __shfl_sync(0xffffffffu, lp[NQ / 8][c0 & 1], gid * 4 + c0 / 2);
      const double lf1 = __shfl_sync(0xffffffffu, lp[(NQ + 1) / 8][c1 & 1], gid * 4 + c1 / 2);
      // G5: quad-face lifts
      double qp[JT][2], qx[JT][2], qy[JT][2], qz[JT][2];
#pragma unroll
      for (int jt = 0; jt < JT; ++jt) qp[jt][0] = qp[jt][1] = qx[jt][0] = qx[jt][1] = qy[jt][0] = qy[jt][1] =
          qz[jt][0] = qz[jt][1] = 0.0;
      if (surf) {
#pragma unroll
        for (int s2 = 0; s2 < KQ; ++s2) {
          const int k = 4 * s2 + tig;
          const double qa = k < 3 * NQ ? Qs[k * NT + i] : 0.0;
          const int fq = k < 3 * NQ ? k / NQ : 2;
          const double nx = nrm[6 + 3 * fq], ny = nrm[7 + 3 * fq], nz = nrm[8 + 3 * fq];
#pragma unroll
          for (int jt = 0; jt < JT; ++jt) {
            const int off = 2 * NT + k * NQ + 8 * jt + gid;
            const double bp = Fp[off], bu = Fu[off];
            dmma(qp[jt], qa, bp);
            dmma(qx[jt], qa, nx * bu);
            dmma(qy[jt], qa, ny * bu);
            dmma(qz[jt], qa, nz * bu);
          }
        }
      }
      // epilogue: rows i, columns j = 8 jt + 2 tig + c
#pragma unroll
      for (int jt = 0; jt < JT; ++jt)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int j = 8 * jt + 2 * tig + c;
          if (i < NT && j < NQ) {
            double rp = lv[jt][c], rux = 0.0, ruy = 0.0, ruz = 0.0;
            if (vol) {
              rp -= dv[jt][c];
              rux = -(G[W_TXJ + j] * ly[jt][c] + gx[jt][c]);
              ruy = -(G[w_tyj(N) + j] * ly[jt][c] + gy[jt][c]);
              ruz = -(tzJ * ly[jt][c]);
            }
            if (surf) {
              const double t0 = jfb * sProf[j] * lf0, t1 = jft * sProf[NQ + j] * lf1;
              rp += qp[jt][c];
              rux += nrm[0] * t0 + nrm[3] * t1 + qx[jt][c];
              ruy += nrm[1] * t0 + nrm[4] * t1 + qy[jt][c];
              ruz += nrm[2] * t0 + nrm[5] * t1 + qz[jt][c];
            }
            if (media) {
              rp *= kappa;
              rux *= irho;
              ruy *= irho;
              ruz *= irho;
            }
            const int idx = j * NT + i;
            const double rv[4] = {rp, rux, ruy, ruz};
#pragma unroll
            for (int f = 0; f < 4; ++f) {
              double& rr = R[f * NP + idx];
              if (lserk)
                rr = first ? p.dt * rv[f] : p.a * rr + p.dt * rv[f];
              else
                rr = accum ? rr + rv[f] : rv[f];
            }
          }
        }
    }
    __syncwarp();
    if (lserk) {
      const double b = p.b;
      for (int q = lane; q < 4 * NP; q += 32) U[q] += b * R[q];
    }
    __syncwarp();
    if (lane == 0) {
      fence_proxy_async_smem();
      if (lserk) {
        tma_store_1d(p.u_out + e * 4 * NP, U, 32 * NP);
        tma_store_1d(p.res + e * 4 * NP, R, 32 * NP);
      } else {
        tma_store_1d(p.rhs_out + e * 4 * NP, R, 32 * NP);
      }
      bulk_commit();
    }
    e = en;
  }
  if (lane == 0) bulk_wait<0>();
}

template <int N>
cudaError_t launch_dmma_N(const StageParams& p, cudaStream_t s) {
  using C = DCfg<N>;
  static int grid_cap = 0;
  if (grid_cap == 0) {
    cudaError_t err = cudaFuncSetAttribute(wedge_dmma_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)C::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wedge_dmma_kernel<N>, 32 * C::WPB, C::SMEM_BYTES);
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  if (p.Kw == 0) return cudaSuccess;
  const long long need = (p.Kw + C::WPB - 1) / C::WPB;
  const int grid = (int)(need < grid_cap ? need : grid_cap);
  wedge_dmma_kernel<N><<<grid, 32 * C::WPB, C::SMEM_BYTES, s>>>(p);
  return cudaGetLastError();
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

int wedge_elems_per_block(int N) {
  switch (N) {
#define PDG_CASE(n) case n: return DCfg<n>::WPB;
    PDG_CASE(1) PDG_CASE(2) PDG_CASE(3) PDG_CASE(4) PDG_CASE(5) PDG_CASE(6) PDG_CASE(7)
    PDG_CASE(8) PDG_CASE(9)
#undef PDG_CASE
  }
  return 0;
}

} // namespace pdg
