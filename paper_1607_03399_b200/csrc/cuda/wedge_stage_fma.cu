// Fused wedge stage kernel: volume + surface + media + LSERK45 stage update.
//
// Persistent CTAs (one per SM) walk groups of E consecutive wedges.  Each
// group's inputs -- state (4 fields x NQ x NT), L^{tri,k}, the three quad
// lifts, the geometry/media record and the connectivity record -- are
// contiguous in HBM and are staged into shared memory with bulk TMA copies
// (cp.async.bulk, completion on an mbarrier), double-buffered: while a group
// computes, the next group's bytes are already in flight.  The LSERK residual
// is prefetched into registers at the start of the group and consumed in the
// epilogue; neighbour face traces are gathered once per group with all loads
// of a thread in flight together.
//
// Thread (el, jh, i) owns triangle node i of wedge el and the slices
// j in [jh*JS, (jh+1)*JS) (paper's slice-parallel mapping, PAPER.md:620-661,
// split over S threads at high N).  Per group:
//   1. V = -(txJ Dt ux + tyJ Dt uy + tzJ Dt uz) per column (pressure pre-lift),
//   2. upwind / central / custom fluxes on all 2NT + 3NQ^2 face nodes,
//   3. fold the two triangular-face pressure lifts into V (L commutes with the
//      slice profile),
//   4. one pass over k accumulating (rx Dr + sx Ds) P, (ry Dr + sy Ds) P, the
//      divergence, L P and L V (metric folded into the matrix row),
//   5. Dt applied to L P across slices, quad-face lifts, n-scaled velocity
//      lifts, media, then res = a res + dt rhs, u_out = u_in + b res.
// Reference: wedge_volume_elem / surface_elem / scale_media / lserk
// (proj/src/solver.cpp:164-218, 258-335, 337-346, 541-551).
#include <cuda_runtime.h>

#include "pdg_device.cuh"
#include "tma.cuh"

namespace pdg {

namespace {

__host__ __device__ constexpr int round4(int x) { return (x + 3) & ~3; }
__host__ __device__ constexpr int slice_split(int N) { return N <= 4 ? 1 : (N == 8 ? 3 : 2); }

template <int N>
struct WCfg {
  static constexpr int NQ = nq_of(N), NT = nt_of(N), NP = npw_of(N), FW = fw_of(N);
  static constexpr int WG = wg_of(N);
  static constexpr int S = slice_split(N);
  static constexpr int JS = (NQ + S - 1) / S; // slices per thread
  static constexpr int TPE = NT * S;           // threads per element
  // shared-memory strides (doubles): stage rows are 16-byte aligned with an odd
  // 16-byte stride (bank spread); work rows have an odd 8-byte stride
  static constexpr int USTR = round4(4 * NP) + 2;
  static constexpr int LSTR = round4(lg_of(N)) + 2;
  static constexpr int QSTR = round4(qg_of(N)) + 2;
  static constexpr int VSTR = NP | 1;
  static constexpr int FSTR = (2 * FW) | 1;
  static constexpr int STAGE_PER_ELEM = USTR + LSTR + QSTR + WG + kWC / 2;
  static constexpr int WORK_PER_ELEM = VSTR + FSTR;
  static constexpr int PER_ELEM = 2 * STAGE_PER_ELEM + WORK_PER_ELEM;
  static constexpr int SMEM_BUDGET = 220 * 1024;
  static constexpr int E_SMEM = (SMEM_BUDGET - 64) / (8 * PER_ELEM);
  static constexpr int E_THR = 512 / TPE;
  static constexpr int E = (E_SMEM < E_THR ? E_SMEM : E_THR) > 0 ? (E_SMEM < E_THR ? E_SMEM : E_THR) : 1;
  static constexpr int THREADS = E * TPE;
  static constexpr int STAGE_DOUBLES = E * STAGE_PER_ELEM;
  static constexpr size_t SMEM_BYTES = 64 + (size_t)8 * (2 * STAGE_DOUBLES + E * WORK_PER_ELEM);
  static constexpr int MAXM = (FW + TPE - 1) / TPE; // face nodes per thread
};

template <int N>
struct Stage {
  double* U;
  double* L;
  double* Q;
  double* G;
  int* C;
};

template <int N>
__device__ __forceinline__ Stage<N> stage_ptrs(double* base, int s) {
  using C = WCfg<N>;
  double* p = base + (size_t)s * C::STAGE_DOUBLES;
  Stage<N> st;
  st.U = p;
  st.L = st.U + C::E * C::USTR;
  st.Q = st.L + C::E * C::LSTR;
  st.G = st.Q + C::E * C::QSTR;
  st.C = reinterpret_cast<int*>(st.G + C::E * C::WG);
  return st;
}

// issued by warp 0 of the CTA: bulk copies of one group into stage `st`
template <int N>
__device__ __forceinline__ void issue_group(const StageParams& p, const Stage<N>& st, long long g, uint64_t* bar,
                                            int lane) {
  using C = WCfg<N>;
  constexpr int NP = C::NP;
  const long long e0 = g * C::E;
  const int nel = (int)((p.Kw - e0) < C::E ? (p.Kw - e0) : C::E);
  const uint32_t bytes = (uint32_t)nel * (uint32_t)(8 * (4 * NP + lg_of(N) + qg_of(N) + C::WG) + 4 * kWC);
  if (lane == 0) mbar_arrive_expect_tx(bar, bytes);
  __syncwarp();
  for (int el = lane; el < nel; el += 32) {
    tma_load_1d(st.U + el * C::USTR, p.u_in + (e0 + el) * 4 * NP, 8 * 4 * NP, bar);
    tma_load_1d(st.L + el * C::LSTR, p.Lt + (e0 + el) * lg_of(N), 8 * lg_of(N), bar);
    tma_load_1d(st.Q + el * C::QSTR, p.QL + (e0 + el) * qg_of(N), 8 * qg_of(N), bar);
  }
  if (lane == 0) {
    tma_load_1d(st.G, p.wgeo + e0 * C::WG, 8 * C::WG * nel, bar);
    tma_load_1d(st.C, p.wconn + e0 * kWC, 4 * kWC * nel, bar);
  }
}

template <int N>
__global__ void __launch_bounds__(WCfg<N>::THREADS, 1)
wedge_stage_kernel(const StageParams p) {
  using C = WCfg<N>;
  constexpr int NQ = C::NQ, NT = C::NT, NP = C::NP, FW = C::FW, WG = C::WG, E = C::E;
  constexpr int S = C::S, JS = C::JS, TPE = C::TPE, MAXM = C::MAXM;
  extern __shared__ __align__(16) double smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  double* stage_base = smem + 8; // 64-byte header
  double* sV = stage_base + 2 * C::STAGE_DOUBLES;
  double* sF = sV + E * C::VSTR;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int el = tid / TPE;
  const int r = tid - el * TPE;
  const int jh = r / NT;
  const int i = r - jh * NT;
  const int j0 = jh * JS;
  const int mode = p.mode;
  const bool vol = mode & M_VOLUME, surf = mode & M_SURFACE;
  const bool lserk = mode & M_LSERK, first = mode & M_FIRST;
  const long long ngroups = (p.Kw + E - 1) / E;

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 0 && (long long)blockIdx.x < ngroups)
    issue_group<N>(p, stage_ptrs<N>(stage_base, 0), blockIdx.x, &bars[0], lane);

  double* V = sV + el * C::VSTR;
  double* Fp = sF + el * C::FSTR;
  double* Fu = Fp + FW;

  for (int it = 0;; ++it) {
    const long long g = (long long)blockIdx.x + (long long)it * gridDim.x;
    if (g >= ngroups) break;
    const int s = it & 1;
    const long long gn = g + gridDim.x;
    if (warp == 0 && gn < ngroups) {
      fence_proxy_async_smem();
      issue_group<N>(p, stage_ptrs<N>(stage_base, s ^ 1), gn, &bars[s ^ 1], lane);
    }
    const long long e0 = g * E;
    const int nel = (int)((p.Kw - e0) < E ? (p.Kw - e0) : E);
    const bool active = el < nel;
    const long long e = e0 + el;
    const long long obase = e * 4 * NP;

    // residual prefetch: consumed in the epilogue, latency hidden by the group
    double rres[4][JS];
    if (active && lserk && !first) {
#pragma unroll
      for (int jj = 0; jj < JS; ++jj) {
        const int j = j0 + jj;
        if (j < NQ) {
#pragma unroll
          for (int f = 0; f < 4; ++f) rres[f][jj] = p.res[obase + f * NP + j * NT + i];
        }
      }
    }

    mbar_wait(&bars[s], (it >> 1) & 1);
    const Stage<N> st = stage_ptrs<N>(stage_base, s);
    const double* U = st.U + el * C::USTR;
    const double* Lm = st.L + el * C::LSTR;
    const double* Q = st.Q + el * C::QSTR;
    const double* G = st.G + el * WG;
    const int* CN = st.C + el * kWC;

    // ---- 1. vertical part of the pressure pre-lift buffer ------------------
    if (active) {
      if (vol) {
        double ux[NQ], uy[NQ], uz[NQ];
#pragma unroll
        for (int l = 0; l < NQ; ++l) {
          ux[l] = U[NP + l * NT + i];
          uy[l] = U[2 * NP + l * NT + i];
          uz[l] = U[3 * NP + l * NT + i];
        }
        const double tzJ = G[W_TZJ];
#pragma unroll
        for (int jj = 0; jj < JS; ++jj) {
          const int j = j0 + jj;
          if (j < NQ) {
            double dx = 0.0, dy = 0.0, dz = 0.0;
#pragma unroll
            for (int l = 0; l < NQ; ++l) {
              const double dd = __ldg(p.Dt + j * NQ + l);
              dx += dd * ux[l];
              dy += dd * uy[l];
              dz += dd * uz[l];
            }
            V[j * NT + i] = -(G[W_TXJ + j] * dx + G[w_tyj(N) + j] * dy + tzJ * dz);
          }
        }
      } else {
#pragma unroll
        for (int jj = 0; jj < JS; ++jj)
          if (j0 + jj < NQ) V[(j0 + jj) * NT + i] = 0.0;
      }
    }

    // ---- 2. numerical fluxes: gather all neighbour values first, then compute
    if (active && surf) {
      double nb[MAXM][4];
#pragma unroll
      for (int q = 0; q < MAXM; ++q) {
        const int m = r + q * TPE;
        if (m < FW) {
          int f, loc;
          if (m < NT) {
            f = 0;
            loc = m;
          } else if (m < 2 * NT) {
            f = 1;
            loc = m - NT;
          } else {
            const int qq = m - 2 * NT;
            f = 2 + qq / (NQ * NQ);
            loc = qq - (f - 2) * NQ * NQ;
          }
          const int nbr = CN[2 * f];
          if (nbr >= 0) {
            const int node = __ldg(p.nbr_nodes + (long long)CN[2 * f + 1] * p.max_nfp + loc);
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
#pragma unroll
      for (int q = 0; q < MAXM; ++q) {
        const int m = r + q * TPE;
        if (m < FW) {
          int f;
          if (m < NT)
            f = 0;
          else if (m < 2 * NT)
            f = 1;
          else
            f = 2 + (m - 2 * NT) / (NQ * NQ);
          const int my = __ldg(p.wface_dev + m);
          const double pm = U[my];
          const double nx = G[w_nrm(N) + 3 * f], ny = G[w_nrm(N) + 3 * f + 1], nz = G[w_nrm(N) + 3 * f + 2];
          const double taup = G[w_taup(N) + f], tauu = G[w_tauu(N) + f];
          double fp, fu;
          if (CN[2 * f] >= 0) {
            const double dp = nb[q][0] - pm;
            const double dux = nb[q][1] - U[NP + my];
            const double duy = nb[q][2] - U[2 * NP + my];
            const double duz = nb[q][3] - U[3 * NP + my];
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
    __syncthreads();

    // ---- 3. triangular-face pressure lifts share the L application of V ----
    if (active && surf) {
      const double a0 = G[W_JFB] * Fp[i], a1 = G[W_JFT] * Fp[NT + i];
#pragma unroll
      for (int jj = 0; jj < JS; ++jj) {
        const int j = j0 + jj;
        if (j < NQ) V[j * NT + i] += a0 * __ldg(p.prof + j) + a1 * __ldg(p.prof + NQ + j);
      }
    }
    __syncthreads();

    // ---- 4. one pass over k ----------------------------------------------------
    double gx[JS], gy[JS], dv[JS], lp[JS], lv[JS];
#pragma unroll
    for (int jj = 0; jj < JS; ++jj) gx[jj] = gy[jj] = dv[jj] = lp[jj] = lv[jj] = 0.0;
    double lf0 = 0.0, lf1 = 0.0;
    if (active) {
      const double rx = G[W_RX], ry = G[W_RY], sx = G[W_SX], sy = G[W_SY];
      if (vol) {
#pragma unroll 3
        for (int k = 0; k < NT; ++k) {
          const double l = Lm[k * NT + i];
          const double dr = __ldg(p.DrT + k * NT + i), ds = __ldg(p.DsT + k * NT + i);
          const double cx = rx * dr + sx * ds, cy = ry * dr + sy * ds;
#pragma unroll
          for (int jj = 0; jj < JS; ++jj) {
            const int j = (j0 + jj < NQ) ? j0 + jj : NQ - 1;
            const double pk = U[j * NT + k], xk = U[NP + j * NT + k], yk = U[2 * NP + j * NT + k];
            gx[jj] += cx * pk;
            gy[jj] += cy * pk;
            dv[jj] += cx * xk + cy * yk;
            lp[jj] += l * pk;
            lv[jj] += l * V[j * NT + k];
          }
          if (surf) {
            lf0 += l * Fu[k];
            lf1 += l * Fu[NT + k];
          }
        }
      } else {
        for (int k = 0; k < NT; ++k) {
          const double l = Lm[k * NT + i];
#pragma unroll
          for (int jj = 0; jj < JS; ++jj) {
            const int j = (j0 + jj < NQ) ? j0 + jj : NQ - 1;
            lv[jj] += l * V[j * NT + k];
          }
          lf0 += l * Fu[k];
          lf1 += l * Fu[NT + k];
        }
      }
    }

    // L P for all slices is needed by the Dt application of the epilogue
    double lpall[NQ];
    if constexpr (S == 1) {
#pragma unroll
      for (int l = 0; l < NQ; ++l) lpall[l] = lp[l];
    } else {
      __syncthreads(); // every thread is done reading V
      if (active) {
#pragma unroll
        for (int jj = 0; jj < JS; ++jj)
          if (j0 + jj < NQ) V[(j0 + jj) * NT + i] = lp[jj];
      }
      __syncthreads();
      if (active) {
#pragma unroll
        for (int l = 0; l < NQ; ++l) lpall[l] = V[l * NT + i];
      }
    }

    // ---- 5. epilogue per owned slice --------------------------------------------
    if (active) {
      const double tzJ = G[W_TZJ], kappa = G[W_KAPPA], irho = G[W_IRHO];
      const double* nrm = G + w_nrm(N);
      const double jfb = G[W_JFB], jft = G[W_JFT];
#pragma unroll
      for (int jj = 0; jj < JS; ++jj) {
        const int j = j0 + jj;
        if (j >= NQ) break;
        double rp = lv[jj], rux = 0.0, ruy = 0.0, ruz = 0.0;
        if (vol) {
          double ly = 0.0;
#pragma unroll
          for (int l = 0; l < NQ; ++l) ly += __ldg(p.Dt + j * NQ + l) * lpall[l];
          rp -= dv[jj];
          rux = -(G[W_TXJ + j] * ly + gx[jj]);
          ruy = -(G[w_tyj(N) + j] * ly + gy[jj]);
          ruz = -(tzJ * ly);
        }
        if (surf) {
          const double t0 = jfb * __ldg(p.prof + j) * lf0, t1 = jft * __ldg(p.prof + NQ + j) * lf1;
          rux += nrm[0] * t0 + nrm[3] * t1;
          ruy += nrm[1] * t0 + nrm[4] * t1;
          ruz += nrm[2] * t0 + nrm[5] * t1;
#pragma unroll
          for (int f = 0; f < 3; ++f) {
            const double* Qf = Q + f * NQ * NT;
            const double* fpq = Fp + 2 * NT + f * NQ * NQ + j;
            const double* fuq = Fu + 2 * NT + f * NQ * NQ + j;
            double qp = 0.0, qu = 0.0;
#pragma unroll
            for (int a = 0; a < NQ; ++a) {
              const double qa = Qf[a * NT + i];
              qp += qa * fpq[a * NQ];
              qu += qa * fuq[a * NQ];
            }
            rp += qp;
            rux += nrm[6 + 3 * f] * qu;
            ruy += nrm[7 + 3 * f] * qu;
            ruz += nrm[8 + 3 * f] * qu;
          }
        }
        if (mode & M_MEDIA) {
          rp *= kappa;
          rux *= irho;
          ruy *= irho;
          ruz *= irho;
        }
        const int n = j * NT + i;
        const long long o = obase + n;
        const double rv[4] = {rp, rux, ruy, ruz};
        if (lserk) {
#pragma unroll
          for (int fld = 0; fld < 4; ++fld) {
            const long long of = o + fld * NP;
            const double rr = first ? p.dt * rv[fld] : p.a * rres[fld][jj] + p.dt * rv[fld];
            p.res[of] = rr;
            p.u_out[of] = U[fld * NP + n] + p.b * rr;
          }
        } else if (mode & M_ACCUM) {
#pragma unroll
          for (int fld = 0; fld < 4; ++fld) p.rhs_out[o + fld * NP] += rv[fld];
        } else {
#pragma unroll
          for (int fld = 0; fld < 4; ++fld) p.rhs_out[o + fld * NP] = rv[fld];
        }
      }
    }
    __syncthreads(); // stage s and the work buffers are free again
  }
}

template <int N>
cudaError_t launch_wedge_N(const StageParams& p, cudaStream_t s) {
  using C = WCfg<N>;
  static int grid_cap = 0;
  if (grid_cap == 0) {
    cudaError_t err = cudaFuncSetAttribute(wedge_stage_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)C::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wedge_stage_kernel<N>, C::THREADS, C::SMEM_BYTES);
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  if (p.Kw == 0) return cudaSuccess;
  const long long groups = (p.Kw + C::E - 1) / C::E;
  const int grid = (int)(groups < grid_cap ? groups : grid_cap);
  wedge_stage_kernel<N><<<grid, C::THREADS, C::SMEM_BYTES, s>>>(p);
  return cudaGetLastError();
}

} // namespace

int wedge_elems_per_block_fma(int N) {
  switch (N) {
#define PDG_CASE(n) case n: return WCfg<n>::E;
    PDG_CASE(1) PDG_CASE(2) PDG_CASE(3) PDG_CASE(4) PDG_CASE(5) PDG_CASE(6) PDG_CASE(7)
    PDG_CASE(8) PDG_CASE(9)
#undef PDG_CASE
  }
  return 0;
}

cudaError_t launch_wedge_stage_fma(int N, const StageParams& p, cudaStream_t s) {
  switch (N) {
#define PDG_CASE(n) case n: return launch_wedge_N<n>(p, s);
    PDG_CASE(1) PDG_CASE(2) PDG_CASE(3) PDG_CASE(4) PDG_CASE(5) PDG_CASE(6) PDG_CASE(7)
    PDG_CASE(8) PDG_CASE(9)
#undef PDG_CASE
  }
  return cudaErrorInvalidValue;
}

} // namespace pdg
