// Low-order fused wedge stage kernel, one thread per DOF column (N = 1..3, exact mass).
//
// The CUDA-core kernel of wedge_simt.cu gives a thread a (wedge, triangle node)
// pair and all N+1 slices of it: ~250 registers at N = 2, 3, so 8 warps per SM
// wait on FP64 dependency chains (ncu: `wait` 34-38%, issue 30%; the FP64 pipe
// is 15-21% busy, profiles/round2_ncu_per_degree.md).  Here a thread owns one
// (wedge, node i, slice j) column and computes the four outputs at (i, j):
//   phase A  gx, gy = (r_x Dr + s_x Ds)(i,:) P(:,j), dv = ... UX, UY, lp = L(i,:) P(:,j),
//            the vertical part of V(j,i) (-(txJ Dt UX + tyJ Dt UY + tzJ Dt UZ)),
//            the face fluxes of the chunk (neighbour traces gathered from L2);
//   phase B  LY(i,j) = Dt(j,:) LP(i,:) (LP exchanged through shared memory across
//            the one barrier between the phases),
//            LV with the folded bottom/top pressure lifts, L Fu_bottom/top, the
//            quad-face lifts, normals, media and the LSERK45 stage update.
// The same algebra as wedge_simt.cu / wedge_dmma.cu (the lift folds of
// SURVEY.md A.3) and the reference's wedge_volume_elem / surface_elem /
// scale_media / lserk (proj/src/solver.cpp:164-218, 258-335, 337-346, 541-551).
//
// Data movement: the state, L^{tri,k}, quad lifts, record and connectivity of
// a chunk of E = THREADS / Np wedges arrive by 16-byte cp.async into one
// contiguous shared-memory slot per wedge (double-buffered against the current
// chunk); each thread's four residual values are read coalesced from HBM into
// registers at the chunk start; outputs are written coalesced by (i, j).
#include <cuda_runtime.h>

#include <cstdlib>

#include "pdg_device.cuh"

namespace pdg {

namespace {

__host__ __device__ constexpr int r2(int x) { return (x + 1) & ~1; }

#ifndef PDG_LO_THREADS
#define PDG_LO_THREADS 256
#endif
#ifndef PDG_LO_MINB
#define PDG_LO_MINB 2
#endif

template <int N>
struct LCfg {
  static_assert(nts_of(N) == nt_of(N), "the low-order kernel assumes an unpadded slice stride");
  static constexpr int NQ = nq_of(N), NT = nt_of(N), NP = npd_of(N), FW = fw_of(N), WG = wg_of(N);
  static constexpr int THREADS = PDG_LO_THREADS;
  static constexpr int E = THREADS / NP;         // wedges per chunk
  static constexpr int ACT = E * NP;             // threads with a column
  static constexpr int LF = lcomp_of(N), QF = qcomp_of(N);
  static constexpr int SU = r2(4 * NP);
  static constexpr int SW = SU + LF + QF + WG + kWC / 2; // per-wedge slot: U | L | QL | record | connectivity
  static constexpr int STAGE = E * SW;
  static constexpr int FT = 4 * NT;              // tri fluxes [p|u][bottom|top][NT]
  static constexpr int FQ = 6 * NQ * NQ;         // quad fluxes [p|u][face][a][j]
  static constexpr int SF = r2(FT + FQ);
  static constexpr int SV = r2(2 * NQ * NT);     // vertical part of V [j][i], then LP [i][l]
  static constexpr int TABLES = r2(r2(2 * NT * NT + NQ * NQ + 2 * NQ) + ceil_div(FW, 2) + 2048 / 2);
  static constexpr size_t SMEM_BYTES = (size_t)8 * (TABLES + 2 * STAGE + E * (SF + SV) + 4);
  static constexpr int TASKS = ceil_div(E * FW, THREADS);
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

/// copy state, L, quad lifts, record and connectivity of wedges [e0, e0 + nel) into the stage
template <int N>
__device__ __forceinline__ void lo_load_chunk(const StageParams& p, double* stg, long long e0, int nel) {
  using C = LCfg<N>;
  constexpr int UV = 2 * C::NP, LV = C::LF / 2, QV = C::QF / 2, GV = C::WG / 2, CV = kWC / 4;
  constexpr int PER = UV + LV + QV + GV + CV; // 16-byte vectors per wedge
  for (int q = threadIdx.x; q < nel * PER; q += C::THREADS) {
    const int e = q / PER;
    int v = q - e * PER;
    double* slot = stg + e * C::SW;
    const long long ge = e0 + e;
    if (v < UV) {
      cp_async16(slot + 2 * v, p.u_in + ge * 4 * C::NP + 2 * v);
      continue;
    }
    v -= UV;
    if (v < LV) {
      cp_async16(slot + C::SU + 2 * v, p.Lt + ge * C::LF + 2 * v);
      continue;
    }
    v -= LV;
    if (v < QV) {
      cp_async16(slot + C::SU + C::LF + 2 * v, p.QL + ge * C::QF + 2 * v);
      continue;
    }
    v -= QV;
    if (v < GV) {
      cp_async16(slot + C::SU + C::LF + C::QF + 2 * v, p.wgeo + ge * C::WG + 2 * v);
      continue;
    }
    v -= GV;
    cp_async16(slot + C::SU + C::LF + C::QF + C::WG + 2 * v, p.wconn + ge * kWC + 4 * v);
  }
}

template <int N>
__global__ void __launch_bounds__(LCfg<N>::THREADS, PDG_LO_MINB) wedge_lo_kernel(const StageParams p) {
  using C = LCfg<N>;
  constexpr int NQ = C::NQ, NT = C::NT, NP = C::NP, FW = C::FW, WG = C::WG, E = C::E;
  constexpr int SW = C::SW, SF = C::SF, SV = C::SV;
  extern __shared__ __align__(16) double smem[];
  double* sDrT = smem;            // [k][i]
  double* sDsT = sDrT + NT * NT;  // [k][i]
  double* sDt = sDsT + NT * NT;   // [j][l]
  double* sProf = sDt + NQ * NQ;  // [2][NQ]
  int* sWface = reinterpret_cast<int*>(smem + r2(2 * NT * NT + NQ * NQ + 2 * NQ));
  int* sCombo = sWface + 2 * ceil_div(FW, 2);
  double* stg = smem + C::TABLES; // 2 stages
  double* sF = stg + 2 * C::STAGE; // per wedge fluxes
  double* sV = sF + E * SF;        // per wedge vertical part of V
  volatile long long* slot = reinterpret_cast<volatile long long*>(sV + E * SV);
  for (int q = threadIdx.x; q < NT * NT; q += C::THREADS) {
    sDrT[q] = p.DrT[q];
    sDsT[q] = p.DsT[q];
  }
  for (int q = threadIdx.x; q < NQ * NQ; q += C::THREADS) sDt[q] = p.Dt[q];
  for (int q = threadIdx.x; q < 2 * NQ; q += C::THREADS) sProf[q] = p.prof[q];
  for (int q = threadIdx.x; q < FW; q += C::THREADS) sWface[q] = p.wface_dev[q];
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
    slot[0] = (long long)(atomicAdd(p.ticket, 1ULL) - p.ticket_base);
    slot[1] = (long long)(atomicAdd(p.ticket, 1ULL) - p.ticket_base);
  }
  __syncthreads();
  long long c = slot[0], cn = slot[1];
  if (c < nchunk) lo_load_chunk<N>(p, stg, p.Kw_begin + c * E, nel_of(c));
  cp_async_commit();

  // this thread's column: wedge el of the chunk, triangle node i, slice j (fastest)
  const int el = threadIdx.x / NP, r = threadIdx.x - el * NP;
  const int i = r / NQ, j = r - i * NQ;
  // Dt(j, :) and the bottom / top profiles at slice j, fixed for the kernel
  double dtj[NQ];
#pragma unroll
  for (int l = 0; l < NQ; ++l) dtj[l] = sDt[j * NQ + l];
  const double prof0 = sProf[j], prof1 = sProf[NQ + j];

  for (int it = 0; c < nchunk; ++it) {
    double* cur = stg + (it & 1) * C::STAGE;
    cp_async_wait_all();
    if (threadIdx.x == 0) slot[2 + (it & 1)] = (long long)(atomicAdd(p.ticket, 1ULL) - p.ticket_base);
    __syncthreads();
    // every thread has left the previous chunk: its stage takes the one after this
    if (cn < nchunk) lo_load_chunk<N>(p, stg + ((it + 1) & 1) * C::STAGE, p.Kw_begin + cn * E, nel_of(cn));
    cp_async_commit();
    const long long e0 = p.Kw_begin + c * E;
    const int nel = nel_of(c);
    const bool active = threadIdx.x < C::ACT && el < nel;
    const double* S = cur + el * SW;
    const double* U = S;
    const double* Lw = S + C::SU;          // L [k][i]
    const double* Qw = Lw + C::LF;         // quad lifts [f][a][i]
    const double* G = Qw + C::QF;
    const long long ge = e0 + el;

    // residual of this column (4 fields), coalesced by (i, j), in flight during phase A
    double rres[4];
#pragma unroll
    for (int f = 0; f < 4; ++f)
      rres[f] = (active && res_src) ? __ldcs(res_src + ge * 4 * NP + f * NP + j * NT + i) : 0.0;

    // ---- phase A: gathers issued, volume products of the column, vertical V part, fluxes
    double nbv[C::TASKS][4];
    if (surf) {
#pragma unroll
      for (int q = 0; q < C::TASKS; ++q) {
        const int m = threadIdx.x + C::THREADS * q;
        if (m < nel * FW) {
          const int e = m / FW, fm = m - e * FW;
          const int f = fm < NT ? 0 : (fm < 2 * NT ? 1 : 2 + (fm - 2 * NT) / (NQ * NQ));
          const int loc = fm < 2 * NT ? fm - f * NT : (fm - 2 * NT) - (f - 2) * NQ * NQ;
          const int* Cn = reinterpret_cast<const int*>(cur + e * SW + C::SU + C::LF + C::QF + WG);
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
    }
    double gx = 0.0, gy = 0.0, dv = 0.0, lp = 0.0;
    if (active) {
      const double rx = G[W_RX], ry = G[W_RY], sxm = G[W_SX], sym = G[W_SY];
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        const double pk = U[j * NT + k];
        lp += Lw[k * NT + i] * pk;
        if (vol) {
          const double dr = sDrT[k * NT + i], ds = sDsT[k * NT + i];
          const double cx = rx * dr + sxm * ds, cy = ry * dr + sym * ds;
          gx += cx * pk;
          gy += cy * pk;
          dv += cx * U[NP + j * NT + k] + cy * U[2 * NP + j * NT + k];
        }
      }
      if (vol) {
        const double tzJ = G[W_TZJ], sx_ = G[W_TXJ + j], sy_ = G[w_tyj(N) + j];
        double d = 0.0;
#pragma unroll
        for (int l = 0; l < NQ; ++l) {
          const double dt = dtj[l];
          d += U[NP + l * NT + i] * (sx_ * dt);
          d += U[2 * NP + l * NT + i] * (sy_ * dt);
          d += U[3 * NP + l * NT + i] * (tzJ * dt);
        }
        sV[el * SV + j * NT + i] = -d;
      }
      sV[el * SV + NQ * NT + i * NQ + j] = lp; // LP(i, j) for the node's other slices
    }
    if (surf) {
#pragma unroll
      for (int q = 0; q < C::TASKS; ++q) {
        const int m = threadIdx.x + C::THREADS * q;
        if (m < nel * FW) {
          const int e = m / FW, fm = m - e * FW;
          const int f = fm < NT ? 0 : (fm < 2 * NT ? 1 : 2 + (fm - 2 * NT) / (NQ * NQ));
          const int loc = fm < 2 * NT ? fm - f * NT : (fm - 2 * NT) - (f - 2) * NQ * NQ;
          const double* Ue = cur + e * SW;
          const double* Ge = Ue + C::SU + C::LF + C::QF;
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
            Fe[4 * NT + (f - 2) * NQ * NQ + loc] = fp;               // Fqp[f-2][a][j]
            Fe[4 * NT + 3 * NQ * NQ + (f - 2) * NQ * NQ + loc] = fu; // Fqu
          }
        }
      }
    }
    __syncthreads(); // fluxes and V parts of the chunk complete

    // ---- phase B: the rest of the column and the stage update -----------------------
    if (active) {
      const double* Fe = sF + el * SF;
      const double* Ve = sV + el * SV;
      const double tzJ = G[W_TZJ], jfb = G[W_JFB], jft = G[W_JFT];
      double lv = 0.0, lp0 = 0.0, lp1 = 0.0, lf0 = 0.0, lf1 = 0.0;
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        const double lk = Lw[k * NT + i];
        if (vol) lv += lk * Ve[j * NT + k];
        if (surf) {
          lp0 += lk * Fe[k];
          lp1 += lk * Fe[NT + k];
          lf0 += lk * Fe[2 * NT + k];
          lf1 += lk * Fe[3 * NT + k];
        }
      }
      double rp = lv + jfb * prof0 * lp0 + jft * prof1 * lp1, rux = 0.0, ruy = 0.0, ruz = 0.0;
      if (vol) {
        double ly = 0.0; // LY(i, j) = Dt(j, :) LP(i, :)
#pragma unroll
        for (int l = 0; l < NQ; ++l) ly += Ve[NQ * NT + i * NQ + l] * dtj[l];
        rp -= dv;
        rux = -(G[W_TXJ + j] * ly + gx);
        ruy = -(G[w_tyj(N) + j] * ly + gy);
        ruz = -(tzJ * ly);
      }
      if (surf) {
        const double* nrm = G + w_nrm(N);
        const double t0 = jfb * prof0 * lf0, t1 = jft * prof1 * lf1;
        rux += nrm[0] * t0 + nrm[3] * t1;
        ruy += nrm[1] * t0 + nrm[4] * t1;
        ruz += nrm[2] * t0 + nrm[5] * t1;
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          double qp = 0.0, qu = 0.0;
#pragma unroll
          for (int a = 0; a < NQ; ++a) {
            const double q = Qw[(f * NQ + a) * NT + i];
            qp += q * Fe[4 * NT + (f * NQ + a) * NQ + j];
            qu += q * Fe[4 * NT + 3 * NQ * NQ + (f * NQ + a) * NQ + j];
          }
          rp += qp;
          rux += nrm[3 * (f + 2)] * qu;
          ruy += nrm[3 * (f + 2) + 1] * qu;
          ruz += nrm[3 * (f + 2) + 2] * qu;
        }
      }
      if (media) {
        const double kappa = G[W_KAPPA], irho = G[W_IRHO];
        rp *= kappa;
        rux *= irho;
        ruy *= irho;
        ruz *= irho;
      }
      const double rv[4] = {rp, rux, ruy, ruz};
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        const int o = f * NP + j * NT + i;
        const long long go = ge * 4 * NP + o;
        if (lserk) {
          const double rr = first ? p.dt * rv[f] : p.a * rres[f] + p.dt * rv[f];
          __stcs(p.res + go, rr);
          __stcs(p.u_out + go, U[o] + p.b * rr);
        } else {
          __stcs(p.rhs_out + go, accum ? rres[f] + rv[f] : rv[f]);
        }
      }
    }
    c = cn;
    cn = slot[2 + (it & 1)];
  }
  cp_async_wait_all();
}

template <int N>
cudaError_t launch_lo_N(const StageParams& p, cudaStream_t s) {
  using C = LCfg<N>;
  static int grid_cap[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  auto kern = wedge_lo_kernel<N>;
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

bool wedge_lo_supported(int N) { return N >= 1 && N <= 3; }

cudaError_t launch_wedge_lo_stage(int N, const StageParams& p, cudaStream_t s) {
  switch (N) {
    case 1: return launch_lo_N<1>(p, s);
    case 2: return launch_lo_N<2>(p, s);
    case 3: return launch_lo_N<3>(p, s);
  }
  return cudaErrorInvalidValue;
}

} // namespace pdg
