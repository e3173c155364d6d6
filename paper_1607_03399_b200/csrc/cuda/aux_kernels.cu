// Layout conversion, energy and watchdog kernels.
//  * layout: reference state (element-major, wedge node i*(N+1)+j, solver.hpp:27-28)
//    <-> device state (Morton element order, wedge [field][j][i]).
//  * energy: 1/2 sum_k (p^T M_k p / kappa + rho u^T M_k u), M_k = M1D (x) M^{tri,k}
//    for wedges (lumped: diag(w) (x) M^{tri,k}), J Mhat for tets
//    (compute_energy, proj/src/solver.cpp:402-435); deterministic two-pass sum.
//  * check_finite: first reference element holding a non-finite DOF
//    (run_simulation watchdog, proj/src/solver.cpp:647-655).
#include <cuda_runtime.h>

#include "pdg_device.cuh"

namespace pdg {

namespace {

template <int N, bool TO_DEVICE>
__global__ void layout_kernel(long long Kw, long long Kt, const int* __restrict__ dev_to_ref,
                              const long long* __restrict__ ref_offset,
                              const double* __restrict__ src, double* __restrict__ dst) {
  // device wedge block: 4 fields x NQ slices x ST (>= NT, padding entries are zero)
  constexpr int NQ = nq_of(N), NT = nt_of(N), NPW = npw_of(N), NPD = npd_of(N), ST = nts_of(N), NPT = npt_of(N);
  const long long wdofs = Kw * 4 * NPD;
  const long long total = wdofs + Kt * 4 * NPT;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long d, ref_local;
    if (idx < wdofs) {
      d = idx / (4 * NPD);
      const int off = (int)(idx - d * 4 * NPD);
      const int fld = off / NPD, node = off - fld * NPD;
      const int j = node / ST, i = node - j * ST;
      if (i >= NT) { // slice padding
        if (TO_DEVICE) dst[idx] = 0.0;
        continue;
      }
      ref_local = (long long)fld * NPW + i * NQ + j;
    } else {
      const long long t = (idx - wdofs) / (4 * NPT);
      d = Kw + t;
      ref_local = (idx - wdofs) - t * 4 * NPT; // tets keep node order
    }
    const long long ref = ref_offset[dev_to_ref[d]] + ref_local;
    if (TO_DEVICE)
      dst[idx] = src[ref];
    else
      dst[ref] = src[idx];
  }
}

template <int N>
__global__ void wedge_energy_kernel(const EnergyParams p, int elems_per_block) {
  // thread (el, i); partial energy of each block written to partials[block]
  // NP = device per-field block, ST = device slice stride
  constexpr int NQ = nq_of(N), NT = nt_of(N), NP = npd_of(N), ST = nts_of(N), WG = wg_of(N);
  extern __shared__ double smem[];
  const int E = elems_per_block;
  double* sU = smem;                // [E][4*NP]
  double* red = sU + E * 4 * NP;    // [blockDim]
  const long long e0 = (long long)blockIdx.x * E;
  const int nel = (int)((p.Kw - e0) < E ? (p.Kw - e0) : E);
  for (int idx = threadIdx.x; idx < nel * 4 * NP; idx += blockDim.x) sU[idx] = p.u[e0 * 4 * NP + idx];
  __syncthreads();
  const int el = threadIdx.x / NT, i = threadIdx.x - el * NT;
  double acc = 0.0;
  if (el < nel) {
    const double* G = p.wgeo + (e0 + el) * WG;
    const double j0 = G[w_jac(N)], jr = G[w_jac(N) + 1], js = G[w_jac(N) + 2];
    const double ikap = 1.0 / G[W_KAPPA], rho = 1.0 / G[W_IRHO];
    const double* U = sU + el * 4 * NP;
    for (int fld = 0; fld < 4; ++fld) {
      const double* v = U + fld * NP;
      double vm[NQ];
#pragma unroll
      for (int l = 0; l < NQ; ++l) vm[l] = 0.0;
      for (int k = 0; k < NT; ++k) {
        const double m = j0 * p.Mtri[k * NT + i] + jr * p.Xr[k * NT + i] + js * p.Xs[k * NT + i];
#pragma unroll
        for (int l = 0; l < NQ; ++l) vm[l] += v[l * ST + k] * m;
      }
      double q = 0.0;
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        double mv;
        if (p.lumped) {
          mv = p.w1d[j] * vm[j];
        } else {
          mv = 0.0;
#pragma unroll
          for (int l = 0; l < NQ; ++l) mv += p.M1D[j * NQ + l] * vm[l];
        }
        q += v[j * ST + i] * mv;
      }
      acc += (fld == 0 ? ikap : rho) * q;
    }
    acc *= 0.5;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  // fixed-order tree reduction (deterministic)
  for (int s = 1; s < blockDim.x; s <<= 1) {
    if ((threadIdx.x % (2 * s)) == 0 && threadIdx.x + s < blockDim.x) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) p.partials[blockIdx.x] = red[0];
}

template <int N>
__global__ void tet_energy_kernel(const EnergyParams p, int block_offset) {
  constexpr int NP = npt_of(N);
  __shared__ double sv[4 * NP];
  __shared__ double red[NP];
  const long long t = blockIdx.x;
  const double* u = p.u + p.tet_base + t * 4 * NP;
  for (int idx = threadIdx.x; idx < 4 * NP; idx += blockDim.x) sv[idx] = u[idx];
  __syncthreads();
  const int n = threadIdx.x;
  const double* G = p.tgeo + t * kTG;
  const double J = G[T_J], ikap = 1.0 / G[T_KAPPA], rho = 1.0 / G[T_IRHO];
  double acc = 0.0;
  for (int fld = 0; fld < 4; ++fld) {
    double mv = 0.0;
    for (int k = 0; k < NP; ++k) mv += p.Mtet[n * NP + k] * sv[fld * NP + k];
    acc += (fld == 0 ? ikap : rho) * sv[fld * NP + n] * (J * mv);
  }
  red[n] = 0.5 * acc;
  __syncthreads();
  for (int s = 1; s < NP; s <<= 1) {
    if ((n % (2 * s)) == 0 && n + s < NP) red[n] += red[n + s];
    __syncthreads();
  }
  if (n == 0) p.partials[block_offset + t] = red[0];
}

// AB3 update (TimeStepper::step, proj/src/solver.cpp:575-577):
// u += dt/12 (23 f_n - 16 f_{n-1} + 5 f_{n-2}), elementwise over the whole state
__global__ void ab3_update_kernel(long long n, double* __restrict__ u, const double* __restrict__ f0,
                                  const double* __restrict__ f1, const double* __restrict__ f2, double c) {
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x)
    u[idx] += c * (23.0 * f0[idx] - 16.0 * f1[idx] + 5.0 * f2[idx]);
}

// multi-rate AB3 (MRAB) update of one rate level, over its wedge DOF range
// [w0, w1) and tet DOF range [t0, t1) (levels are contiguous in device order):
//   commit (end of the level's step): u = u0 = u0 + h/12 (23 f0 - 16 f1 + 5 f2),
//     the single-rate AB3 formula (solver.cpp:575-577) from the step start;
//   predict (mid-step, read by finer neighbours): u = u0 + h (c0 f0 + c1 f1 + c2 f2),
//     the AB3 interpolant of the level's rhs history integrated over [0, theta h]
__global__ void mrab_update_kernel(long long w0, long long w1, long long t0, long long t1, double* __restrict__ u,
                                   double* __restrict__ u0, const double* __restrict__ f0,
                                   const double* __restrict__ f1, const double* __restrict__ f2, double h,
                                   double c0, double c1, double c2, int commit) {
  const long long nw = w1 - w0, n = nw + (t1 - t0);
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const long long idx = q < nw ? w0 + q : t0 + (q - nw);
    if (commit) {
      const double v = u0[idx] + (h / 12.0) * (23.0 * f0[idx] - 16.0 * f1[idx] + 5.0 * f2[idx]);
      u[idx] = v;
      u0[idx] = v;
    } else {
      u[idx] = u0[idx] + h * (c0 * f0[idx] + c1 * f1[idx] + c2 * f2[idx]);
    }
  }
}

__global__ void reduce_sum_kernel(const double* __restrict__ in, int n, double* __restrict__ out) {
  // single block, fixed order: strided partial sums then a tree
  __shared__ double red[1024];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += in[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

template <int N>
__global__ void check_finite_kernel(long long Kw, long long Kw_act, long long Kt_act, const double* __restrict__ u,
                                    const int* __restrict__ dev_to_ref,
                                    unsigned long long* first_bad) {
  // owned elements only: wedges [0, Kw_act), tets [Kw, Kw + Kt_act) (ghosts follow
  // the owned elements of their kind and belong to another rank)
  constexpr int NPW = npd_of(N), NPT = npt_of(N); // device wedge block (padding entries are zero)
  const long long wact = Kw_act * 4 * NPW, wall = Kw * 4 * NPW;
  const long long total = wact + Kt_act * 4 * NPT;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long at = idx < wact ? idx : wall + (idx - wact);
    if (!isfinite(u[at])) {
      const long long d = idx < wact ? idx / (4 * NPW) : Kw + (idx - wact) / (4 * NPT);
      atomicMin(first_bad, (unsigned long long)dev_to_ref[d]);
    }
  }
}

template <int N, bool PACK>
__global__ void pack_kernel(long long Kw, const long long* __restrict__ elems, long long n,
                            const double* __restrict__ src, double* __restrict__ dst) {
  // one CTA per listed element; wedge and tet blocks have different sizes
  // buffer entries: 4 x Np per element (device node order, no slice padding);
  // device state: wedge blocks of 4 x NPD (slices of ST)
  constexpr int NT = nt_of(N), NPW = npw_of(N), NPD = npd_of(N), ST = nts_of(N), NPT = npt_of(N);
  for (long long q = blockIdx.x; q < n; q += gridDim.x) {
    const long long d = elems[q];
    const bool wedge = d < Kw;
    const int len = 4 * (wedge ? NPW : NPT);
    const long long off = wedge ? d * 4 * NPD : Kw * 4 * NPD + (d - Kw) * 4 * NPT;
    const long long boff = q * 4 * (NPW > NPT ? NPW : NPT);
    for (int k = threadIdx.x; k < len; k += blockDim.x) {
      long long o = k;
      if (wedge && ST != NT) {
        const int fld = k / NPW, node = k - fld * NPW, j = node / NT, i = node - j * NT;
        o = (long long)fld * NPD + j * ST + i;
      }
      if (PACK)
        dst[boff + k] = src[off + o];
      else
        dst[off + o] = src[boff + k];
    }
  }
}

int grid_for(long long total, int threads) {
  long long b = (total + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  return (int)b;
}

} // namespace

#define PDG_DISPATCH(N, CALL)      \
  switch (N) {                     \
    case 1: { constexpr int NN = 1; CALL; } break; \
    case 2: { constexpr int NN = 2; CALL; } break; \
    case 3: { constexpr int NN = 3; CALL; } break; \
    case 4: { constexpr int NN = 4; CALL; } break; \
    case 5: { constexpr int NN = 5; CALL; } break; \
    case 6: { constexpr int NN = 6; CALL; } break; \
    case 7: { constexpr int NN = 7; CALL; } break; \
    case 8: { constexpr int NN = 8; CALL; } break; \
    case 9: { constexpr int NN = 9; CALL; } break; \
    default: return cudaErrorInvalidValue; \
  }

cudaError_t launch_to_device_layout(int N, long long Kw, long long Kt, const int* dev_to_ref,
                                    const long long* ref_offset, const double* src, double* dst,
                                    cudaStream_t s) {
  const long long total = Kw * 4 * npd_of(N) + Kt * 4 * npt_of(N);
  if (total == 0) return cudaSuccess;
  PDG_DISPATCH(N, (layout_kernel<NN, true><<<grid_for(total, 256), 256, 0, s>>>(Kw, Kt, dev_to_ref, ref_offset, src, dst)));
  return cudaGetLastError();
}

cudaError_t launch_to_reference_layout(int N, long long Kw, long long Kt, const int* dev_to_ref,
                                       const long long* ref_offset, const double* src, double* dst,
                                       cudaStream_t s) {
  const long long total = Kw * 4 * npd_of(N) + Kt * 4 * npt_of(N);
  if (total == 0) return cudaSuccess;
  PDG_DISPATCH(N, (layout_kernel<NN, false><<<grid_for(total, 256), 256, 0, s>>>(Kw, Kt, dev_to_ref, ref_offset, src, dst)));
  return cudaGetLastError();
}

cudaError_t launch_energy(int N, const EnergyParams& p, int* nblocks_out, cudaStream_t s) {
  int wb = 0;
  const int NT = nt_of(N);
  const int E = (256 / NT) > 0 ? 256 / NT : 1;
  if (p.Kw > 0) {
    wb = (int)((p.Kw + E - 1) / E);
    const size_t smem = ((size_t)E * 4 * npd_of(N) + (size_t)E * NT) * 8;
    PDG_DISPATCH(N, ({
      cudaFuncSetAttribute(wedge_energy_kernel<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      wedge_energy_kernel<NN><<<wb, E * NT, smem, s>>>(p, E);
    }));
  }
  if (p.Kt > 0) {
    PDG_DISPATCH(N, (tet_energy_kernel<NN><<<(unsigned)p.Kt, npt_of(NN), 0, s>>>(p, wb)));
  }
  *nblocks_out = wb + (int)p.Kt;
  return cudaGetLastError();
}

// face-trace exchange of the multi-GPU path: buf[k] = u[idx[k]] / u[idx[k]] = buf[k]
__global__ void gather_values_kernel(const long long* __restrict__ idx, long long n, const double* __restrict__ u,
                                     double* __restrict__ buf) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    buf[k] = u[idx[k]];
}
__global__ void scatter_values_kernel(const long long* __restrict__ idx, long long n, const double* __restrict__ buf,
                                      double* __restrict__ u) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    u[idx[k]] = buf[k];
}

cudaError_t launch_gather_values(const long long* idx, long long n, const double* u, double* buf, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  gather_values_kernel<<<(unsigned)((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8), 256, 0, s>>>(idx, n, u, buf);
  return cudaGetLastError();
}
cudaError_t launch_scatter_values(const long long* idx, long long n, const double* buf, double* u, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  scatter_values_kernel<<<(unsigned)((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8), 256, 0, s>>>(idx, n, buf, u);
  return cudaGetLastError();
}

cudaError_t launch_ab3_update(long long n, double* u, const double* f0, const double* f1, const double* f2,
                              double dt, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  ab3_update_kernel<<<148 * 8, 256, 0, s>>>(n, u, f0, f1, f2, dt / 12.0);
  return cudaGetLastError();
}

cudaError_t launch_mrab_update(long long w0, long long w1, long long t0, long long t1, double* u, double* u0,
                               const double* f0, const double* f1, const double* f2, double h, double theta,
                               int commit, cudaStream_t s) {
  const long long n = (w1 - w0) + (t1 - t0);
  if (n <= 0) return cudaSuccess;
  // int_0^theta of the backward-difference quadratic through f0 (s=0), f1 (s=-1), f2 (s=-2)
  const double th = theta, th2 = th * th, th3 = th2 * th;
  const double c0 = th + 0.75 * th2 + th3 / 6.0, c1 = -th2 - th3 / 3.0, c2 = 0.25 * th2 + th3 / 6.0;
  const long long want = (n + 255) / 256;
  const int grid = (int)(want < 148 * 8 ? want : 148 * 8);
  mrab_update_kernel<<<grid, 256, 0, s>>>(w0, w1, t0, t1, u, u0, f0, f1, f2, h, c0, c1, c2, commit);
  return cudaGetLastError();
}

cudaError_t launch_reduce_sum(const double* in, int n, double* out, cudaStream_t s) {
  reduce_sum_kernel<<<1, 1024, 0, s>>>(in, n, out);
  return cudaGetLastError();
}

cudaError_t launch_pack_states(int N, long long Kw, const long long* dev_elems, long long n, const double* u,
                               double* buf, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int grid = (int)(n < 148 * 16 ? n : 148 * 16);
  PDG_DISPATCH(N, (pack_kernel<NN, true><<<grid, 128, 0, s>>>(Kw, dev_elems, n, u, buf)));
  return cudaGetLastError();
}

cudaError_t launch_unpack_states(int N, long long Kw, const long long* dev_elems, long long n, const double* buf,
                                 double* u, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int grid = (int)(n < 148 * 16 ? n : 148 * 16);
  PDG_DISPATCH(N, (pack_kernel<NN, false><<<grid, 128, 0, s>>>(Kw, dev_elems, n, buf, u)));
  return cudaGetLastError();
}

cudaError_t launch_check_finite(int N, long long Kw, long long Kw_act, long long Kt_act, const double* u,
                                const int* dev_to_ref, unsigned long long* first_bad,
                                cudaStream_t s) {
  const long long total = Kw_act * 4 * npd_of(N) + Kt_act * 4 * npt_of(N);
  if (total == 0) return cudaSuccess;
  PDG_DISPATCH(N, (check_finite_kernel<NN><<<grid_for(total, 256), 256, 0, s>>>(Kw, Kw_act, Kt_act, u, dev_to_ref,
                                                                                   first_bad)));
  return cudaGetLastError();
}

} // namespace pdg
