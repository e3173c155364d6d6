// Fused wedge stage kernel for N = 1, one thread per (wedge, slice).
//
// The per-node kernel (wedge_simt.cu) gives six threads a wedge at N = 1 (one
// per triangle node and slice half) and spreads the chunk's face-node flux
// tasks over the whole CTA, so a thread executes ~1100 instructions per chunk
// for four outputs (ncu: 44% issue, ~53% of the instructions integer index and
// control work).  Here the NQ threads of a wedge are adjacent lanes; thread j
// owns slice j -- every triangle node i of it, all four fields -- and the face
// nodes that lie on slice j (its triangle face, when j is the bottom or top
// slice, and node row j of the three quad faces).  The only cross-thread data
// are the two triangle faces' fluxes and the slice values of L P, exchanged by
// warp shuffles inside the wedge's lane group: no shared-memory exchange and
// no barrier besides the chunk's copy barrier.  Per (i, j):
//   rp  = L V(:, j) + jfb prof_b(j) L Fp_b + jft prof_t(j) L Fp_t - dv + sum_f QL_f Fqp_f(:, j)
//   u_c = -(c_J(j) LY + g_c) + n_b,c jfb prof_b(j) L Fu_b + n_t,c jft prof_t(j) L Fu_t
//         + sum_f n_f,c QL_f Fqu_f(:, j)
// with V = -(txJ Dt UX + tyJ Dt UY + tzJ Dt UZ), LY = LP Dt^T, g = (r_c Dr + s_c Ds) P,
// dv = (r_x Dr + s_x Ds) UX + (r_y Dr + s_y Ds) UY: the algebra of wedge_lo.cu /
// wedge_simt.cu (SURVEY.md A.3 lift folds) and the reference's wedge_volume_elem /
// surface_elem / scale_media / lserk (proj/src/solver.cpp:164-218, 258-335, 337-346,
// 541-551).  Opt-in (PDG_WEDGE_SL=1) until measured.
//
// Data movement: state, L^{tri,k}, quad lifts, record and connectivity of a chunk
// of E = THREADS / NQ wedges arrive by 16-byte cp.async into one contiguous slot
// per wedge (double-buffered); the residual of the thread's slice goes from HBM
// into registers at the chunk start; neighbour traces are L2 gathers.
#include <cuda_runtime.h>

#include <cstdlib>

#include "pdg_device.cuh"

namespace pdg {

namespace {

__host__ __device__ constexpr int r2(int x) { return (x + 1) & ~1; }
/// smallest slot stride >= x that is 2 mod 16 (doubles): the 16 wedges of a warp read
/// their slots on 8 distinct bank pairs (2 mod 16 is the best an even stride can do)
__host__ __device__ constexpr int slot16(int x) { return x % 16 == 2 ? x : slot16(x + 1); }

#ifndef PDG_SL_THREADS
#define PDG_SL_THREADS 128
#endif
#ifndef PDG_SL_MINB
#define PDG_SL_MINB 2
#endif

template <int N>
struct SLCfg {
  static_assert(nts_of(N) == nt_of(N), "the low-order kernel assumes an unpadded slice stride");
  static constexpr int NQ = nq_of(N), NT = nt_of(N), NP = npd_of(N), FW = fw_of(N), WG = wg_of(N);
  static_assert(32 % nq_of(N) == 0, "a wedge's slice threads must share a warp");
  static constexpr int THREADS = PDG_SL_THREADS;
  static constexpr int E = THREADS / NQ; // wedges per chunk
  static constexpr int LF = lcomp_of(N), QF = qcomp_of(N);
  static constexpr int SU = r2(4 * NP);
  // exact mode reads the record up to the WADG fields (w_jac), so only that part is copied
  static constexpr int WGX = w_jac(N);
  static_assert(WGX % 2 == 0, "16-byte copies of the record");
  static constexpr int SW = slot16(SU + LF + QF + WGX + kWC / 2); // per-wedge slot: U | L | QL | record | connectivity
  static constexpr int STAGE = E * SW;
  static constexpr int TABLES = r2(r2(2 * NT * NT + NQ * NQ + 2 * NQ) + ceil_div(FW, 2) + 2048 / 2);
  static constexpr size_t SMEM_BYTES = (size_t)8 * (TABLES + 2 * STAGE + 4);
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

/// the wedge's NQ threads copy its state, L, quad lifts, record and connectivity into
/// its slot (thread j takes vectors j, j + NQ, ...: compile-time offsets, no division)
template <int N>
__device__ __forceinline__ void sl_load_wedge(const StageParams& p, double* slot, long long ge, int j) {
  using C = SLCfg<N>;
  constexpr int NQ = C::NQ;
  constexpr int UV = 2 * C::NP, LV = C::LF / 2, QV = C::QF / 2, GV = C::WGX / 2, CV = kWC / 4;
  const double* u = p.u_in + ge * 4 * C::NP;
  const double* l = p.Lt + ge * C::LF;
  const double* q = p.QL + ge * C::QF;
  const double* g = p.wgeo + ge * C::WG;
  const int* cn = p.wconn + ge * kWC;
#pragma unroll
  for (int v = 0; v < UV; v += NQ)
    if (v + j < UV) cp_async16(slot + 2 * (v + j), u + 2 * (v + j));
#pragma unroll
  for (int v = 0; v < LV; v += NQ)
    if (v + j < LV) cp_async16(slot + C::SU + 2 * (v + j), l + 2 * (v + j));
#pragma unroll
  for (int v = 0; v < QV; v += NQ)
    if (v + j < QV) cp_async16(slot + C::SU + C::LF + 2 * (v + j), q + 2 * (v + j));
#pragma unroll
  for (int v = 0; v < GV; v += NQ)
    if (v + j < GV) cp_async16(slot + C::SU + C::LF + C::QF + 2 * (v + j), g + 2 * (v + j));
#pragma unroll
  for (int v = 0; v < CV; v += NQ)
    if (v + j < CV) cp_async16(slot + C::SU + C::LF + C::QF + C::WGX + 2 * (v + j), cn + 4 * (v + j));
}

template <int N>
__global__ void __launch_bounds__(SLCfg<N>::THREADS, PDG_SL_MINB) wedge_sl_kernel(const StageParams p) {
  using C = SLCfg<N>;
  constexpr int NQ = C::NQ, NT = C::NT, NP = C::NP, FW = C::FW, WG = C::WG, E = C::E, SW = C::SW;
  extern __shared__ __align__(16) double smem[];
  double* sDrT = smem;            // [k][i]
  double* sDsT = sDrT + NT * NT;  // [k][i]
  double* sDt = sDsT + NT * NT;   // [j][l]
  double* sProf = sDt + NQ * NQ;  // [2][NQ]
  int* sWface = reinterpret_cast<int*>(smem + r2(2 * NT * NT + NQ * NQ + 2 * NQ));
  int* sCombo = sWface + 2 * ceil_div(FW, 2);
  double* stg = smem + C::TABLES; // 2 stages
  volatile long long* slot = reinterpret_cast<volatile long long*>(stg + 2 * C::STAGE);
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
  // this thread: wedge el of the chunk, slice j; lanes lb .. lb + NQ - 1 hold the wedge
  const int el = threadIdx.x / NQ, j = threadIdx.x - el * NQ;
  if (c < nchunk && el < nel_of(c)) sl_load_wedge<N>(p, stg + el * SW, p.Kw_begin + c * E + el, j);
  cp_async_commit();
  const int lane = threadIdx.x & 31, lb = lane - j;
  double dtj[NQ];
#pragma unroll
  for (int l = 0; l < NQ; ++l) dtj[l] = sDt[j * NQ + l];
  const double prof0 = sProf[j], prof1 = sProf[NQ + j];
  // this thread's face nodes: its triangle face (bottom for j = 0, top for j = NQ-1; at
  // N >= 1 both ends exist) and node row j of each quad face
  constexpr int NFT = NT, NFQ = 3 * NQ;
  const int ftri = j == 0 ? 0 : (j == NQ - 1 ? 1 : -1);

  for (int it = 0; c < nchunk; ++it) {
    const double* cur = stg + (it & 1) * C::STAGE;
    cp_async_wait_all();
    if (threadIdx.x == 0) slot[2 + (it & 1)] = (long long)(atomicAdd(p.ticket, 1ULL) - p.ticket_base);
    __syncthreads();
    // every thread has left the previous chunk: its stage takes the one after this
    if (cn < nchunk && el < nel_of(cn))
      sl_load_wedge<N>(p, stg + ((it + 1) & 1) * C::STAGE + el * SW, p.Kw_begin + cn * E + el, j);
    cp_async_commit();
    const long long e0 = p.Kw_begin + c * E;
    const int nel = nel_of(c);
    const bool active = el < nel;
    const double* U = cur + el * SW;
    const double* Lw = U + C::SU;  // L [k][i]
    const double* Qw = Lw + C::LF; // quad lifts [f][a][i]
    const double* G = Qw + C::QF;
    const int* Cn = reinterpret_cast<const int*>(G + C::WGX);
    const long long ge = e0 + el;

    // residual of the slice (4 fields x NT nodes), in flight during the fluxes
    double rres[4][NT];
#pragma unroll
    for (int f = 0; f < 4; ++f)
#pragma unroll
      for (int i = 0; i < NT; ++i)
        rres[f][i] = (active && res_src) ? __ldg(res_src + ge * 4 * NP + f * NP + j * NT + i) : 0.0;

    // ---- fluxes on the slice's face nodes ------------------------------------------
    // tri: [p|u][node], quad: [p|u][face][a]
    double ftp[NFT], ftu[NFT], fqp[NFQ], fqu[NFQ];
#pragma unroll
    for (int q = 0; q < NFT; ++q) ftp[q] = ftu[q] = 0.0;
#pragma unroll
    for (int q = 0; q < NFQ; ++q) fqp[q] = fqu[q] = 0.0;
    if (surf && active) {
      double nbv[NFT + NFQ][4];
      // gathers first (all loads of the thread in flight together)
#pragma unroll
      for (int q = 0; q < NFT + NFQ; ++q) {
        const bool tri = q < NFT;
        const int f = tri ? ftri : 2 + (q - NFT) / NQ;
        if (f < 0) continue;
        const int loc = tri ? q : ((q - NFT) % NQ) * NQ + j;
        const int nbr = Cn[2 * f];
        if (nbr >= 0) {
          const int ci = Cn[2 * f + 1] * p.max_nfp + loc;
          const int node = combo_smem ? sCombo[ci] : __ldg(p.nbr_nodes + ci);
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
#pragma unroll
      for (int q = 0; q < NFT + NFQ; ++q) {
        const bool tri = q < NFT;
        const int f = tri ? ftri : 2 + (q - NFT) / NQ;
        if (f < 0) continue;
        const int loc = tri ? q : ((q - NFT) % NQ) * NQ + j;
        const int fm = f < 2 ? f * NT + loc : 2 * NT + (f - 2) * NQ * NQ + loc;
        const int my = sWface[fm];
        const double pm = U[my];
        const double nx = G[w_nrm(N) + 3 * f], ny = G[w_nrm(N) + 3 * f + 1], nz = G[w_nrm(N) + 3 * f + 2];
        const double taup = G[w_taup(N) + f], tauu = G[w_tauu(N) + f];
        double fp, fu;
        if (Cn[2 * f] >= 0) {
          const double dp = nbv[q][0] - pm;
          const double dun = nx * (nbv[q][1] - U[NP + my]) + ny * (nbv[q][2] - U[2 * NP + my]) +
                             nz * (nbv[q][3] - U[3 * NP + my]);
          fp = 0.5 * (taup * dp - dun);
          fu = 0.5 * (tauu * dun - dp);
        } else {
          const double dp = -2.0 * pm; // reflective: p+ = -p-, u+ = u-
          fp = 0.5 * taup * dp;
          fu = -0.5 * dp;
        }
        if (tri) {
          ftp[q] = fp;
          ftu[q] = fu;
        } else {
          fqp[q - NFT] = fp;
          fqu[q - NFT] = fu;
        }
      }
    }
    // the bottom (lane lb) and top (lane lb + NQ - 1) triangle faces' fluxes
    double fpb[NT], fpt[NT], fub[NT], fut[NT];
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      fpb[q] = __shfl_sync(0xffffffffu, ftp[q], lb);
      fub[q] = __shfl_sync(0xffffffffu, ftu[q], lb);
      fpt[q] = __shfl_sync(0xffffffffu, ftp[q], lb + NQ - 1);
      fut[q] = __shfl_sync(0xffffffffu, ftu[q], lb + NQ - 1);
    }

    // ---- products of the slice ----------------------------------------------------
    double lp[NT], gx[NT], gy[NT], dv[NT];
#pragma unroll
    for (int i = 0; i < NT; ++i) lp[i] = gx[i] = gy[i] = dv[i] = 0.0;
    if (active) {
      const double rx = G[W_RX], ry = G[W_RY], sxm = G[W_SX], sym = G[W_SY];
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        const double pk = U[j * NT + k], xk = U[NP + j * NT + k], yk = U[2 * NP + j * NT + k];
#pragma unroll
        for (int i = 0; i < NT; ++i) {
          lp[i] += Lw[k * NT + i] * pk;
          if (vol) {
            const double dr = sDrT[k * NT + i], ds = sDsT[k * NT + i];
            const double cx = rx * dr + sxm * ds, cy = ry * dr + sym * ds;
            gx[i] += cx * pk;
            gy[i] += cy * pk;
            dv[i] += cx * xk + cy * yk;
          }
        }
      }
    }
    // LP of the other slices (for LY = LP Dt^T)
    double ly[NT];
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      ly[i] = 0.0;
#pragma unroll
      for (int l = 0; l < NQ; ++l) ly[i] += __shfl_sync(0xffffffffu, lp[i], lb + l) * dtj[l];
    }
    if (active) {
      const double tzJ = G[W_TZJ], jfb = G[W_JFB], jft = G[W_JFT];
      const double sx_ = G[W_TXJ + j], sy_ = G[w_tyj(N) + j];
      // V(:, j): vertical part
      double v[NT];
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        double d = 0.0;
#pragma unroll
        for (int l = 0; l < NQ; ++l) {
          const double dt = dtj[l];
          d += U[NP + l * NT + k] * (sx_ * dt);
          d += U[2 * NP + l * NT + k] * (sy_ * dt);
          d += U[3 * NP + l * NT + k] * (tzJ * dt);
        }
        v[k] = -d;
      }
      const double* nrm = G + w_nrm(N);
      const double kappa = G[W_KAPPA], irho = G[W_IRHO];
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        double lv = 0.0, lp0 = 0.0, lp1 = 0.0, lf0 = 0.0, lf1 = 0.0;
#pragma unroll
        for (int k = 0; k < NT; ++k) {
          const double lk = Lw[k * NT + i];
          if (vol) lv += lk * v[k];
          if (surf) {
            lp0 += lk * fpb[k];
            lp1 += lk * fpt[k];
            lf0 += lk * fub[k];
            lf1 += lk * fut[k];
          }
        }
        double rp = lv + jfb * prof0 * lp0 + jft * prof1 * lp1, rux = 0.0, ruy = 0.0, ruz = 0.0;
        if (vol) {
          rp -= dv[i];
          rux = -(sx_ * ly[i] + gx[i]);
          ruy = -(sy_ * ly[i] + gy[i]);
          ruz = -(tzJ * ly[i]);
        }
        if (surf) {
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
              qp += q * fqp[f * NQ + a];
              qu += q * fqu[f * NQ + a];
            }
            rp += qp;
            rux += nrm[3 * (f + 2)] * qu;
            ruy += nrm[3 * (f + 2) + 1] * qu;
            ruz += nrm[3 * (f + 2) + 2] * qu;
          }
        }
        if (media) {
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
            const double rr = first ? p.dt * rv[f] : p.a * rres[f][i] + p.dt * rv[f];
            __stcs(p.res + go, rr);
            __stcs(p.u_out + go, U[o] + p.b * rr);
          } else {
            __stcs(p.rhs_out + go, accum ? rres[f][i] + rv[f] : rv[f]);
          }
        }
      }
    }
    c = cn;
    cn = slot[2 + (it & 1)];
  }
  cp_async_wait_all();
}

template <int N>
cudaError_t launch_sl_N(const StageParams& p, cudaStream_t s) {
  using C = SLCfg<N>;
  static int grid_cap[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  auto kern = wedge_sl_kernel<N>;
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

bool wedge_sl_supported(int N) { return N == 1; }

cudaError_t launch_wedge_sl_stage(int N, const StageParams& p, cudaStream_t s) {
  if (N == 1) return launch_sl_N<1>(p, s);
  return cudaErrorInvalidValue;
}

} // namespace pdg
