// Fused wedge stage kernel: volume + surface + media + LSERK45 stage update.
//
// One CTA processes E consecutive wedges; thread (el, i) owns triangle node i
// of wedge el and all N+1 slices j of that node (the paper's slice-parallel
// mapping).  Per stage and wedge the kernel
//   1. stages the wedge state (4 fields x NQ x NT, contiguous) in shared memory,
//   2. forms the vertical-derivative part of the pressure pre-lift buffer
//      V = -(txJ Dt ux + tyJ Dt uy + tzJ Dt uz) per column (registers),
//   3. evaluates upwind / central fluxes on all 2 NT + 3 NQ^2 face nodes with
//      neighbour traces gathered from u_in (reflective p+ = -p- on the boundary),
//   4. folds the two triangular-face pressure lifts into V (the lift commutes
//      with the slice profile) and runs one pass over k that
//      accumulates Dr/Ds (with the metric folded into the row), L P and L V,
//   5. applies Dt to L P in registers (L and Dt commute across slices), adds
//      the quad-face lifts and the n-scaled velocity lifts, scales by media and
//      either writes rhs or performs res = a res + dt rhs, u_out = u_in + b res.
// Reference: wedge_volume_elem / surface_elem / scale_media / lserk
// (proj/src/solver.cpp:164-218, 258-335, 337-346, 541-551).
#include <cuda_runtime.h>

#include "pdg_device.cuh"

namespace pdg {

namespace {

template <int N>
struct WCfg {
  static constexpr int NQ = nq_of(N), NT = nt_of(N), NP = npw_of(N), FW = fw_of(N);
  static constexpr int WG = wg_of(N);
  static constexpr int E = (192 / NT) > 0 ? (192 / NT) : 1;
  static constexpr int THREADS = E * NT;
  // odd per-element strides (in doubles) spread elements over smem banks
  static constexpr int USTR = (4 * NP) | 1;
  static constexpr int VSTR = NP | 1;
  static constexpr int FSTR = (2 * FW) | 1;
  static constexpr int SMEM_DOUBLES = E * (USTR + VSTR + FSTR + WG);
  static constexpr size_t SMEM_BYTES = (size_t)SMEM_DOUBLES * 8 + (size_t)E * 10 * 4;
};

template <int N>
__global__ void __launch_bounds__(WCfg<N>::THREADS)
wedge_stage_kernel(const StageParams p) {
  using C = WCfg<N>;
  constexpr int NQ = C::NQ, NT = C::NT, NP = C::NP, FW = C::FW, WG = C::WG, E = C::E;
  extern __shared__ double smem[];
  double* sU = smem;
  double* sV = sU + E * C::USTR;
  double* sF = sV + E * C::VSTR;
  double* sG = sF + E * C::FSTR;
  int* sC = reinterpret_cast<int*>(sG + E * WG);

  const long long e0 = (long long)blockIdx.x * E;
  const int nel = (int)((p.Kw - e0) < E ? (p.Kw - e0) : E);
  const int mode = p.mode;

  // ---- 1. stage state, geometry and connectivity of the E wedges -----------
  {
    const double2* src = reinterpret_cast<const double2*>(p.u_in + e0 * 4 * NP);
    // 4*NP is even for every N, so each element block is 16-byte aligned
    constexpr int H = 2 * NP; // double2 per element
    for (int idx = threadIdx.x; idx < nel * H; idx += blockDim.x) {
      const int el = idx / H, off = idx - el * H;
      const double2 v = __ldg(src + idx);
      double* d = sU + el * C::USTR + 2 * off;
      d[0] = v.x;
      d[1] = v.y;
    }
    const double* gsrc = p.wgeo + e0 * WG;
    for (int idx = threadIdx.x; idx < nel * WG; idx += blockDim.x) sG[idx] = __ldg(gsrc + idx);
    const int* csrc = p.wconn + e0 * 10;
    for (int idx = threadIdx.x; idx < nel * 10; idx += blockDim.x) sC[idx] = __ldg(csrc + idx);
  }
  __syncthreads();

  const int el = threadIdx.x / NT;
  const int i = threadIdx.x - el * NT;
  const bool active = el < nel;
  const long long e = e0 + el;
  double* U = sU + el * C::USTR;
  double* V = sV + el * C::VSTR;
  double* Fp = sF + el * C::FSTR;
  double* Fu = Fp + FW;
  const double* G = sG + el * WG;
  const int* CN = sC + el * 10;

  // ---- 2. vertical part of the pressure pre-lift buffer --------------------
  if (active) {
    if (mode & M_VOLUME) {
      double ux[NQ], uy[NQ], uz[NQ];
#pragma unroll
      for (int l = 0; l < NQ; ++l) {
        ux[l] = U[NP + l * NT + i];
        uy[l] = U[2 * NP + l * NT + i];
        uz[l] = U[3 * NP + l * NT + i];
      }
      const double tzJ = G[W_TZJ];
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        double dx = 0.0, dy = 0.0, dz = 0.0;
#pragma unroll
        for (int l = 0; l < NQ; ++l) {
          const double d = __ldg(p.Dt + j * NQ + l);
          dx += d * ux[l];
          dy += d * uy[l];
          dz += d * uz[l];
        }
        V[j * NT + i] = -(G[W_TXJ + j] * dx + G[w_tyj(N) + j] * dy + tzJ * dz);
      }
    } else {
#pragma unroll
      for (int j = 0; j < NQ; ++j) V[j * NT + i] = 0.0;
    }
  }

  // ---- 3. numerical fluxes on every face node -------------------------------
  if (active && (mode & M_SURFACE)) {
    for (int m = i; m < FW; m += NT) {
      int f, loc;
      if (m < NT) {
        f = 0;
        loc = m;
      } else if (m < 2 * NT) {
        f = 1;
        loc = m - NT;
      } else {
        const int q = m - 2 * NT;
        f = 2 + q / (NQ * NQ);
        loc = q - (f - 2) * NQ * NQ;
      }
      const int my = __ldg(p.wface_dev + m);
      const double pm = U[my];
      const double nx = G[w_nrm(N) + 3 * f], ny = G[w_nrm(N) + 3 * f + 1],
                   nz = G[w_nrm(N) + 3 * f + 2];
      const double taup = G[w_taup(N) + f], tauu = G[w_tauu(N) + f];
      const int nbr = CN[2 * f];
      double fp, fu;
      if (nbr >= 0) {
        const int q = __ldg(p.nbr_nodes + (long long)CN[2 * f + 1] * p.max_nfp + loc);
        const double* nb;
        int fs;
        if (nbr < p.Kw) {
          nb = p.u_in + (long long)nbr * 4 * NP;
          fs = NP;
        } else {
          nb = p.u_in + p.tet_base + (long long)(nbr - p.Kw) * 4 * npt_of(N);
          fs = npt_of(N);
        }
        const double dp = __ldg(nb + q) - pm;
        const double dux = __ldg(nb + fs + q) - U[NP + my];
        const double duy = __ldg(nb + 2 * fs + q) - U[2 * NP + my];
        const double duz = __ldg(nb + 3 * fs + q) - U[3 * NP + my];
        const double dun = nx * dux + ny * duy + nz * duz;
        fp = 0.5 * (taup * dp - dun);
        fu = 0.5 * (tauu * dun - dp);
      } else {
        const double dp = -2.0 * pm; // p+ = -p-, u+ = u-
        fp = 0.5 * taup * dp;
        fu = -0.5 * dp;
      }
      Fp[m] = fp;
      Fu[m] = fu;
    }
  }
  __syncthreads();

  // ---- 4a. triangular-face pressure lifts share the L application of V ------
  if (active && (mode & M_SURFACE)) {
    const double a0 = G[W_JFB] * Fp[i], a1 = G[W_JFT] * Fp[NT + i];
#pragma unroll
    for (int j = 0; j < NQ; ++j) V[j * NT + i] += a0 * __ldg(p.prof + j) + a1 * __ldg(p.prof + NQ + j);
  }
  __syncthreads();
  if (!active) return;

  // ---- 4b. one pass over k: Dr/Ds (metric folded), L P, L V, L fu_tri -------
  const double rx = G[W_RX], ry = G[W_RY], sx = G[W_SX], sy = G[W_SY];
  const double* L = p.Lt + e * NT * NT;
  double gx[NQ], gy[NQ], dv[NQ], lp[NQ], lv[NQ];
#pragma unroll
  for (int j = 0; j < NQ; ++j) gx[j] = gy[j] = dv[j] = lp[j] = lv[j] = 0.0;
  double lf0 = 0.0, lf1 = 0.0;
  const bool vol = mode & M_VOLUME, surf = mode & M_SURFACE;
  if (vol) {
#pragma unroll 2
    for (int k = 0; k < NT; ++k) {
      const double l = __ldg(L + k * NT + i);
      const double dr = __ldg(p.DrT + k * NT + i), ds = __ldg(p.DsT + k * NT + i);
      const double cx = rx * dr + sx * ds, cy = ry * dr + sy * ds;
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        const double pk = U[j * NT + k], xk = U[NP + j * NT + k], yk = U[2 * NP + j * NT + k];
        gx[j] += cx * pk;
        gy[j] += cy * pk;
        dv[j] += cx * xk + cy * yk;
        lp[j] += l * pk;
        lv[j] += l * V[j * NT + k];
      }
      if (surf) {
        lf0 += l * Fu[k];
        lf1 += l * Fu[NT + k];
      }
    }
  } else {
    for (int k = 0; k < NT; ++k) {
      const double l = __ldg(L + k * NT + i);
#pragma unroll
      for (int j = 0; j < NQ; ++j) lv[j] += l * V[j * NT + k];
      lf0 += l * Fu[k];
      lf1 += l * Fu[NT + k];
    }
  }

  // ---- 5. epilogue per slice --------------------------------------------------
  const double tzJ = G[W_TZJ], kappa = G[W_KAPPA], irho = G[W_IRHO];
  const double* nrm = G + w_nrm(N);
  const double* Q = p.QL + e * 3 * NQ * NT;
  const double jfb = G[W_JFB], jft = G[W_JFT];
  const long long obase = e * 4 * NP;
#pragma unroll
  for (int j = 0; j < NQ; ++j) {
    double rp = lv[j], rux = 0.0, ruy = 0.0, ruz = 0.0;
    if (vol) {
      double ly = 0.0;
#pragma unroll
      for (int l = 0; l < NQ; ++l) ly += __ldg(p.Dt + j * NQ + l) * lp[l];
      rp -= dv[j];
      rux = -(G[W_TXJ + j] * ly + gx[j]);
      ruy = -(G[w_tyj(N) + j] * ly + gy[j]);
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
          const double qa = __ldg(Qf + a * NT + i);
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
    if (mode & M_LSERK) {
      const double r[4] = {rp, rux, ruy, ruz};
#pragma unroll
      for (int fld = 0; fld < 4; ++fld) {
        const long long of = o + fld * NP;
        const double rr = (mode & M_FIRST) ? p.dt * r[fld] : p.a * p.res[of] + p.dt * r[fld];
        p.res[of] = rr;
        p.u_out[of] = U[fld * NP + n] + p.b * rr;
      }
    } else if (mode & M_ACCUM) {
      p.rhs_out[o] += rp;
      p.rhs_out[o + NP] += rux;
      p.rhs_out[o + 2 * NP] += ruy;
      p.rhs_out[o + 3 * NP] += ruz;
    } else {
      p.rhs_out[o] = rp;
      p.rhs_out[o + NP] = rux;
      p.rhs_out[o + 2 * NP] = ruy;
      p.rhs_out[o + 3 * NP] = ruz;
    }
  }
}

template <int N>
cudaError_t launch_wedge_N(const StageParams& p, cudaStream_t s) {
  using C = WCfg<N>;
  static bool configured = false;
  if (!configured) {
    cudaError_t err = cudaFuncSetAttribute(wedge_stage_kernel<N>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)C::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    configured = true;
  }
  if (p.Kw == 0) return cudaSuccess;
  const long long blocks = (p.Kw + C::E - 1) / C::E;
  wedge_stage_kernel<N><<<(unsigned)blocks, C::THREADS, C::SMEM_BYTES, s>>>(p);
  return cudaGetLastError();
}

} // namespace

int wedge_elems_per_block(int N) {
  switch (N) {
#define PDG_CASE(n) case n: return WCfg<n>::E;
    PDG_CASE(1) PDG_CASE(2) PDG_CASE(3) PDG_CASE(4) PDG_CASE(5) PDG_CASE(6) PDG_CASE(7)
    PDG_CASE(8) PDG_CASE(9)
#undef PDG_CASE
  }
  return 0;
}

cudaError_t launch_wedge_stage(int N, const StageParams& p, cudaStream_t s) {
  switch (N) {
#define PDG_CASE(n) case n: return launch_wedge_N<n>(p, s);
    PDG_CASE(1) PDG_CASE(2) PDG_CASE(3) PDG_CASE(4) PDG_CASE(5) PDG_CASE(6) PDG_CASE(7)
    PDG_CASE(8) PDG_CASE(9)
#undef PDG_CASE
  }
  return cudaErrorInvalidValue;
}

} // namespace pdg
