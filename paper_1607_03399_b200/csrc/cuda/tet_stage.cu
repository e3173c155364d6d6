// Fused tetrahedron stage kernel (CUDA cores): volume + surface + media + LSERK45
// update.  Used for N = 6..9; N <= 5 dispatches to the DMMA kernel (tet_dmma.cu).
//
// One CTA handles E tets, one thread per volume node.  Tets are affine, so the
// physical derivative rows are c_x(n,k) = rx Dr(n,k) + sx Ds(n,k) + tx Dt(n,k)
// (likewise y, z), formed on the fly from the shared reference matrices, and
// the surface term is lift_scale_f * LIFT_f * flux_f on the four faces.
// Reference: tet_volume_elem / surface_elem (tet branch) / scale_media
// (proj/src/solver.cpp:220-254, 321-333, 337-346).
#include <cuda_runtime.h>

#include <cstdlib>

#include "pdg_device.cuh"

namespace pdg {

namespace {

template <int N>
struct TCfg {
  static constexpr int NP = npt_of(N), NT = nt_of(N), FT = 4 * nt_of(N);
  static constexpr int E = (128 / NP) > 0 ? (128 / NP) : 1;
  static constexpr int THREADS = E * NP;
  static constexpr int USTR = (4 * NP) | 1;
  static constexpr int FSTR = (2 * FT) | 1;
  static constexpr size_t SMEM_BYTES = (size_t)E * (USTR + FSTR + kTG) * 8 + (size_t)E * 8 * 4;
};

template <int N>
__global__ void __launch_bounds__(TCfg<N>::THREADS)
tet_stage_kernel(const StageParams p) {
  using C = TCfg<N>;
  constexpr int NP = C::NP, NT = C::NT, FT = C::FT, E = C::E;
  extern __shared__ double smem[];
  double* sU = smem;
  double* sF = sU + E * C::USTR;
  double* sG = sF + E * C::FSTR;
  int* sC = reinterpret_cast<int*>(sG + E * kTG);

  const long long t0 = p.Kt_begin + (long long)blockIdx.x * E;
  const int nel = (int)((p.Kt_active - t0) < E ? (p.Kt_active - t0) : E);
  const int mode = p.mode;
  const double* ubase = p.u_in + p.tet_base;
  {
    const double* src = ubase + t0 * 4 * NP;
    for (int idx = threadIdx.x; idx < nel * 4 * NP; idx += blockDim.x) {
      const int el = idx / (4 * NP), off = idx - el * 4 * NP;
      sU[el * C::USTR + off] = __ldg(src + idx);
    }
    const double* gsrc = p.tgeo + t0 * kTG;
    for (int idx = threadIdx.x; idx < nel * kTG; idx += blockDim.x) sG[idx] = __ldg(gsrc + idx);
    const int* csrc = p.tconn + t0 * 8;
    for (int idx = threadIdx.x; idx < nel * 8; idx += blockDim.x) sC[idx] = __ldg(csrc + idx);
  }
  __syncthreads();

  const int el = threadIdx.x / NP;
  const int n = threadIdx.x - el * NP;
  const bool active = el < nel;
  double* U = sU + el * C::USTR;
  double* Fp = sF + el * C::FSTR;
  double* Fu = Fp + FT;
  const double* G = sG + el * kTG;
  const int* CN = sC + el * 8;

  if (active && (mode & M_SURFACE)) {
    for (int m = n; m < FT; m += NP) {
      const int f = m / NT, loc = m - f * NT;
      const int my = __ldg(p.tface + m);
      const double pm = U[my];
      const double nx = G[T_NRM + 3 * f], ny = G[T_NRM + 3 * f + 1], nz = G[T_NRM + 3 * f + 2];
      const double taup = G[T_TAUP + f], tauu = G[T_TAUU + f];
      const int nbr = CN[2 * f];
      double fp, fu;
      if (nbr >= 0) {
        const int q = __ldg(p.nbr_nodes + (long long)CN[2 * f + 1] * p.max_nfp + loc);
        const double* nb;
        int fs;
        if (nbr < p.Kw) {
          nb = p.u_in + (long long)nbr * 4 * npd_of(N);
          fs = npd_of(N);
        } else {
          nb = ubase + (long long)(nbr - p.Kw) * 4 * NP;
          fs = NP;
        }
        const double dp = __ldg(nb + q) - pm;
        const double dux = __ldg(nb + fs + q) - U[NP + my];
        const double duy = __ldg(nb + 2 * fs + q) - U[2 * NP + my];
        const double duz = __ldg(nb + 3 * fs + q) - U[3 * NP + my];
        const double dun = nx * dux + ny * duy + nz * duz;
        fp = 0.5 * (taup * dp - dun);
        fu = 0.5 * (tauu * dun - dp);
      } else {
        const double dp = -2.0 * pm;
        fp = 0.5 * taup * dp;
        fu = -0.5 * dp;
      }
      Fp[m] = fp;
      Fu[m] = fu;
    }
  }
  __syncthreads();
  if (!active) return;

  double rp = 0.0, rux = 0.0, ruy = 0.0, ruz = 0.0;
  if (mode & M_VOLUME) {
    const double rx = G[T_RX], ry = G[T_RY], rz = G[T_RZ], sx = G[T_SX], sy = G[T_SY],
                 sz = G[T_SZ], tx = G[T_TX], ty = G[T_TY], tz = G[T_TZ];
    double gx = 0.0, gy = 0.0, gz = 0.0, dv = 0.0;
#pragma unroll 4
    for (int k = 0; k < NP; ++k) {
      const double dr = __ldg(p.tDrT + k * NP + n), ds = __ldg(p.tDsT + k * NP + n),
                   dt = __ldg(p.tDtT + k * NP + n);
      const double cx = rx * dr + sx * ds + tx * dt;
      const double cy = ry * dr + sy * ds + ty * dt;
      const double cz = rz * dr + sz * ds + tz * dt;
      const double pk = U[k];
      gx += cx * pk;
      gy += cy * pk;
      gz += cz * pk;
      dv += cx * U[NP + k] + cy * U[2 * NP + k] + cz * U[3 * NP + k];
    }
    rp = -dv;
    rux = -gx;
    ruy = -gy;
    ruz = -gz;
  }
  if (mode & M_SURFACE) {
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      double sp = 0.0, su = 0.0;
      for (int m = 0; m < NT; ++m) {
        const double l = __ldg(p.tLiftT + (f * NT + m) * NP + n);
        sp += l * Fp[f * NT + m];
        su += l * Fu[f * NT + m];
      }
      const double ls = G[T_LS + f];
      rp += ls * sp;
      const double lu = ls * su;
      rux += G[T_NRM + 3 * f] * lu;
      ruy += G[T_NRM + 3 * f + 1] * lu;
      ruz += G[T_NRM + 3 * f + 2] * lu;
    }
  }
  if (mode & M_MEDIA) {
    const double kappa = G[T_KAPPA], irho = G[T_IRHO];
    rp *= kappa;
    rux *= irho;
    ruy *= irho;
    ruz *= irho;
  }
  const long long o = p.tet_base + (t0 + el) * 4 * NP + n;
  const double r[4] = {rp, rux, ruy, ruz};
  if (mode & M_LSERK) {
#pragma unroll
    for (int fld = 0; fld < 4; ++fld) {
      const long long of = o + fld * NP;
      const double rr = (mode & M_FIRST) ? p.dt * r[fld] : p.a * p.res[of] + p.dt * r[fld];
      p.res[of] = rr;
      p.u_out[of] = U[fld * NP + n] + p.b * rr;
    }
  } else if (mode & M_ACCUM) {
#pragma unroll
    for (int fld = 0; fld < 4; ++fld) p.rhs_out[o + fld * NP] += r[fld];
  } else {
#pragma unroll
    for (int fld = 0; fld < 4; ++fld) p.rhs_out[o + fld * NP] = r[fld];
  }
}

template <int N>
cudaError_t launch_tet_N(const StageParams& p, cudaStream_t s) {
  using C = TCfg<N>;
  static bool configured[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  if (!configured[dev]) {
    cudaError_t err = cudaFuncSetAttribute(tet_stage_kernel<N>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)C::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    configured[dev] = true;
  }
  if (p.info) *p.info = LaunchInfo{};
  if (p.Kt_active - p.Kt_begin <= 0) return cudaSuccess;
  const long long blocks = (p.Kt_active - p.Kt_begin + C::E - 1) / C::E;
  tet_stage_kernel<N><<<(unsigned)blocks, C::THREADS, C::SMEM_BYTES, s>>>(p);
  if (p.info) *p.info = LaunchInfo{1, blocks, blocks, C::E}; // static blocks, one unit each
  return cudaGetLastError();
}

} // namespace

int tet_elems_per_block(int N) {
  switch (N) {
#define PDG_CASE(n) case n: return TCfg<n>::E;
    PDG_CASE(1) PDG_CASE(2) PDG_CASE(3) PDG_CASE(4) PDG_CASE(5) PDG_CASE(6) PDG_CASE(7)
    PDG_CASE(8) PDG_CASE(9)
#undef PDG_CASE
  }
  return 0;
}

cudaError_t launch_tet_stage(int N, const StageParams& p, cudaStream_t s) {
  // N <= 5: batched tensor-core kernel (tet_dmma.cu); the thread-per-node
  // CUDA-core kernel below covers N = 6..9 (operators too large for shared
  // memory) and PDG_TET_KERNEL=simt
  static const bool simt = [] {
    const char* v = std::getenv("PDG_TET_KERNEL");
    return v && v[0] == 's';
  }();
  if (!simt && tet_dmma_supported(N)) return launch_tet_dmma_stage(N, p, s);
  switch (N) {
#define PDG_CASE(n) case n: return launch_tet_N<n>(p, s);
    PDG_CASE(1) PDG_CASE(2) PDG_CASE(3) PDG_CASE(4) PDG_CASE(5) PDG_CASE(6) PDG_CASE(7)
    PDG_CASE(8) PDG_CASE(9)
#undef PDG_CASE
  }
  return cudaErrorInvalidValue;
}

} // namespace pdg
