// Device context: upload of a host Discretization into the B200 layout and the
// stream-ordered operations behind the C ABI.
#include "context.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <numeric>
#include <string>
#include <tuple>

#ifdef _OPENMP
#include <omp.h>
#endif

using prismdg::DeviceError;

#ifndef PDG_WEDGE_WS_DEFAULT
#define PDG_WEDGE_WS_DEFAULT 0
#endif

namespace pdg {

namespace {

#define PDG_CK(x)                                                                              \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess)                                                                     \
      throw DeviceError(std::string(#x) + " failed: " + cudaGetErrorString(e_));             \
  } while (0)

template <class T>
T* dalloc(std::size_t n) {
  T* p = nullptr;
  PDG_CK(cudaMalloc(&p, std::max<std::size_t>(n, 1) * sizeof(T)));
  return p;
}

template <class T>
T* upload(const std::vector<T>& h) {
  T* d = dalloc<T>(h.size());
  if (!h.empty()) PDG_CK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

// copy per-element blocks of `per` values from src (reference order) to dst
// (device order), through a pinned staging buffer in chunks
template <class T>
void upload_permuted(T* dst, const T* src, std::size_t per, const std::vector<long long>& order,
                     std::size_t dst_stride = 0, long long src_base = 0) {
  // src rows of `per` values indexed by order[q] - src_base; dst rows of dst_stride (>= per, zero padded)
  const std::size_t ne = order.size();
  if (dst_stride == 0) dst_stride = per;
  if (ne == 0 || per == 0) return;
  const std::size_t chunk = std::max<std::size_t>(1, (std::size_t(64) << 20) / (dst_stride * sizeof(T)));
  T* pin = nullptr;
  PDG_CK(cudaMallocHost(&pin, std::min(chunk, ne) * dst_stride * sizeof(T)));
  for (std::size_t c0 = 0; c0 < ne; c0 += chunk) {
    const std::size_t cn = std::min(chunk, ne - c0);
#pragma omp parallel for schedule(static)
    for (long long q = 0; q < (long long)cn; ++q) {
      std::memcpy(pin + q * dst_stride, src + (std::size_t)(order[c0 + q] - src_base) * per, per * sizeof(T));
      if (dst_stride > per) std::memset(pin + q * dst_stride + per, 0, (dst_stride - per) * sizeof(T));
    }
    PDG_CK(cudaMemcpy(dst + c0 * dst_stride, pin, cn * dst_stride * sizeof(T), cudaMemcpyHostToDevice));
  }
  cudaFreeHost(pin);
}

std::uint64_t spread_bits(std::uint64_t x) {
  x &= 0x1fffffULL;
  x = (x | x << 32) & 0x1f00000000ffffULL;
  x = (x | x << 16) & 0x1f0000ff0000ffULL;
  x = (x | x << 8) & 0x100f00f00f00f00fULL;
  x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
  x = (x | x << 2) & 0x1249249249249249ULL;
  return x;
}

// Morton order of element centroids (wedges and tets separately)
std::vector<long long> locality_order(const prismdg::HybridMesh& mesh, bool wedges, bool native) {
  const long long n = wedges ? mesh.num_wedges() : mesh.num_tets();
  const long long off = wedges ? 0 : mesh.num_wedges();
  std::vector<long long> order(n);
  std::iota(order.begin(), order.end(), off);
  if (native || n < 2) return order;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (const auto& v : mesh.vertices)
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::min(lo[d], v[d]);
      hi[d] = std::max(hi[d], v[d]);
    }
  std::vector<std::uint64_t> key(n);
#pragma omp parallel for schedule(static)
  for (long long q = 0; q < n; ++q) {
    double c[3] = {0, 0, 0};
    const int* ids = wedges ? mesh.wedges[q].data() : mesh.tets[q].data();
    const int nv = wedges ? 6 : 4;
    for (int a = 0; a < nv; ++a)
      for (int d = 0; d < 3; ++d) c[d] += mesh.vertices[ids[a]][d] / nv;
    std::uint64_t k = 0;
    for (int d = 0; d < 3; ++d) {
      const double span = hi[d] > lo[d] ? hi[d] - lo[d] : 1.0;
      const double t = std::min(1.0, std::max(0.0, (c[d] - lo[d]) / span));
      k |= spread_bits((std::uint64_t)(t * 2097151.0)) << d;
    }
    key[q] = k;
  }
  std::stable_sort(order.begin(), order.end(),
                   [&](long long a, long long b) { return key[a - off] < key[b - off]; });
  return order;
}

void check_device(int device) {
  int count = 0;
  cudaError_t err = cudaGetDeviceCount(&count);
  if (err != cudaSuccess || count == 0)
    throw DeviceError("no CUDA device available (prismdg_b200 has no CPU fallback): " +
                      std::string(cudaGetErrorString(err)));
  if (device < 0 || device >= count) throw DeviceError("device index out of range");
  cudaDeviceProp prop;
  PDG_CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    throw DeviceError(std::string("prismdg_b200 kernels are built for sm_100a; device is ") +
                      prop.name + " (sm_" + std::to_string(prop.major) + std::to_string(prop.minor) + ")");
}

int dev_node_of(const prismdg::Discretization& d, bool wedge, int nref) {
  if (!wedge) return nref;
  const int i = nref / d.nq, j = nref - i * d.nq;
  return j * nts_of(d.degree) + i; // device slice stride (padded at N = 5)
}

// exact-mode wedge kernel for N >= 4: the warp-specialised one (wedge_ws.cu)
// unless PDG_WEDGE_WS=0 selects the single-role DMMA kernel (wedge_dmma.cu)
bool use_wedge_ws(int N) {
  static const int env = [] {
    const char* v = std::getenv("PDG_WEDGE_WS");
    return v ? std::atoi(v) : -1;
  }();
  return wedge_ws_supported(N) && env != 0 && (env > 0 || PDG_WEDGE_WS_DEFAULT);
}

// exact-mode wedge kernel for N <= 3: the thread-per-DOF-column kernel
// (wedge_lo.cu) when PDG_WEDGE_LO=1 (or PDG_WEDGE_LO_DEFAULT), else wedge_simt.cu
#ifndef PDG_WEDGE_LO_DEFAULT
#define PDG_WEDGE_LO_DEFAULT 0
#endif
bool use_wedge_lo(int N) {
  static const int env = [] {
    const char* v = std::getenv("PDG_WEDGE_LO");
    return v ? std::atoi(v) : -1;
  }();
  return wedge_lo_supported(N) && env != 0 && (env > 0 || PDG_WEDGE_LO_DEFAULT);
}

// exact-mode wedge kernel at N = 1: the thread-per-(wedge, slice) kernel (wedge_sl.cu)
// when PDG_WEDGE_SL=1 (or PDG_WEDGE_SL_DEFAULT)
#ifndef PDG_WEDGE_SL_DEFAULT
#define PDG_WEDGE_SL_DEFAULT 0
#endif
bool use_wedge_sl(int N) {
  static const int env = [] {
    const char* v = std::getenv("PDG_WEDGE_SL");
    return v ? std::atoi(v) : -1;
  }();
  return wedge_sl_supported(N) && env != 0 && (env > 0 || PDG_WEDGE_SL_DEFAULT);
}

void launch_checked(pdg_ctx* c, const StageParams& p0, bool wedge) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->flags & 2) {
    PDG_CK(cudaEventCreate(&a));
    PDG_CK(cudaEventCreate(&b));
    PDG_CK(cudaEventRecord(a, c->stream));
  }
  LaunchInfo info;
  StageParams p = p0;
  p.info = &info;
  cudaError_t err = !wedge ? launch_tet_stage(c->N, p, c->stream)
                    : c->wadg ? (c->N <= wedge_wadg_simt_max_degree() ? launch_wedge_wadg_simt_stage(c->N, p, c->stream)
                                                                     : launch_wedge_wadg_stage(c->N, p, c->stream))
                    : c->wedge_simt ? (use_wedge_sl(c->N)   ? launch_wedge_sl_stage(c->N, p, c->stream)
                                       : use_wedge_lo(c->N) ? launch_wedge_lo_stage(c->N, p, c->stream)
                                                            : launch_wedge_simt_stage(c->N, p, c->stream))
                    : use_wedge_ws(c->N) ? launch_wedge_ws_stage(c->N, p, c->stream)
                                         : launch_wedge_stage(c->N, p, c->stream);
  if (err != cudaSuccess) {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
    throw DeviceError(std::string("stage kernel launch failed: ") + cudaGetErrorString(err));
  }
  c->last_launch[wedge ? 0 : 1] = info;
  if (c->flags & 2) {
    if (info.launched) {
      PDG_CK(cudaEventRecord(b, c->stream));
      c->pending.push_back({a, b, wedge ? 0 : 1});
    } else { // an empty element range launches nothing: neither timed nor counted
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
  }
}

StageParams base_params(pdg_ctx* c) {
  StageParams p{};
  p.Kw = c->Kw;
  p.Kt = c->Kt;
  p.Kw_active = c->Kw_act;
  p.Kt_active = c->Kt_act;
  p.tet_base = c->tet_base;
  p.wgeo = c->wgeo;
  p.wconn = c->wconn;
  p.Lt = c->Lt;
  p.QL = c->QL;
  p.wadg = c->wadg;
  p.wadg_frag = c->wadg_frag;
  p.tgeo = c->tgeo;
  p.tconn = c->tconn;
  p.DrT = c->DrT;
  p.DsT = c->DsT;
  p.Dt = c->Dt;
  p.prof = c->prof;
  p.wface_dev = c->wface_dev;
  p.tDrT = c->tDrT;
  p.tDsT = c->tDsT;
  p.tDtT = c->tDtT;
  p.tLiftT = c->tLiftT;
  p.tface = c->tface;
  p.tet_frag = c->tet_frag;
  p.nbr_nodes = c->nbr_nodes;
  p.max_nfp = c->max_nfp;
  p.nbr_nodes_len = c->nbr_nodes_len;
  p.ticket = c->ticket;
  p.ticket_host_next = &c->ticket_next;
  return p;
}

// LSERK45 coefficients, Carpenter & Kennedy (proj/src/solver.cpp:511-523)
const double kRK4A[5] = {0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                         -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0};
const double kRK4B[5] = {1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                         1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                         2277821191437.0 / 14882151754819.0};

// L^{tri,k} and the quad lifts of every wedge, repacked into DMMA fragment
// order (zero padded) and uploaded in device element order
void upload_wedge_fragments(pdg_ctx* c, const prismdg::Discretization& d, const std::vector<long long>& order) {
  const int N = c->N, nt = c->nt, nq = c->nq;
  const int IT = it_of(N), KS = ks_of(N), KT = kt_of(N);
  const std::size_t LF = lfrag_of(N), QF = qfrag_of(N);
  const std::size_t ne = order.size();
  const std::size_t chunk = std::max<std::size_t>(1, (std::size_t(64) << 20) / ((LF + QF) * 8));
  double* pin = nullptr;
  PDG_CK(cudaMallocHost(&pin, std::min(chunk, ne) * (LF + QF) * 8));
  for (std::size_t c0 = 0; c0 < ne; c0 += chunk) {
    const std::size_t cn = std::min(chunk, ne - c0);
    double* pl = pin;
    double* pq = pin + cn * LF;
#pragma omp parallel for schedule(static)
    for (long long q = 0; q < (long long)cn; ++q) {
      const std::size_t r = (std::size_t)order[c0 + q];
      const double* L = d.tri_lift.data() + r * nt * nt;        // [k*nt + i] = L(i,k)
      const double* Q = d.quad_lift.data() + r * 3 * nq * nt;   // [(f*nq + a)*nt + i]
      double* lf = pl + q * LF;
      double* qf = pq + q * QF;
      for (int t = 0; t < IT; ++t)
        for (int lane = 0; lane < 32; ++lane) {
          const int i = 8 * t + lane / 4, tg = lane % 4;
          for (int s = 0; s < KS; ++s) {
            const int k = 4 * s + tg;
            lf[((std::size_t)t * KS + s) * 32 + lane] = (i < nt && k < nt) ? L[(std::size_t)k * nt + i] : 0.0;
          }
          for (int f = 0; f < 3; ++f)
            for (int s = 0; s < KT; ++s) {
              const int a = 4 * s + tg;
              qf[(((std::size_t)t * 3 + f) * KT + s) * 32 + lane] =
                  (i < nt && a < nq) ? Q[((std::size_t)f * nq + a) * nt + i] : 0.0;
            }
        }
    }
    PDG_CK(cudaMemcpy(c->Lt + c0 * LF, pl, cn * LF * 8, cudaMemcpyHostToDevice));
    PDG_CK(cudaMemcpy(c->QL + c0 * QF, pq, cn * QF * 8, cudaMemcpyHostToDevice));
  }
  cudaFreeHost(pin);
}

// WADG shared tables in the flat layout of pdg_device.cuh (wadg_off_*)
std::vector<double> flatten_wadg(const prismdg::Discretization& d) {
  const int N = d.degree, nt = d.nt, nq = d.nq, nc = wadg_nc(N);
  const prismdg::WadgTables w = prismdg::build_wadg_tables(d.refs);
  if (w.nc != nc) throw prismdg::ConfigError("unexpected triangle cubature size for WADG");
  std::vector<double> f((std::size_t)wadg_size(N), 0.0);
  for (int m = 0; m < 6; ++m)
    for (int i = 0; i < nt; ++i)
      for (int k = 0; k < nt; ++k) f[((std::size_t)m * nt + i) * nt + k] = w.kd[m](i, k);
  for (int i = 0; i < nt; ++i)
    for (int q = 0; q < nc; ++q) {
      f[wadg_off_pw(N) + (std::size_t)i * nc + q] = w.Pw(i, q);
      f[wadg_off_vq(N) + (std::size_t)q * nt + i] = w.Vq(q, i);
    }
  for (int e = 0; e < 3; ++e)
    for (int i = 0; i < nt; ++i)
      for (int a = 0; a < nq; ++a) {
        f[wadg_off_r(N) + ((std::size_t)(0 * 3 + e) * nt + i) * nq + a] = w.R0[e](i, a);
        f[wadg_off_r(N) + ((std::size_t)(1 * 3 + e) * nt + i) * nq + a] = w.R1[e](i, a);
      }
  for (int q = 0; q < nc; ++q) {
    f[wadg_off_q(N) + q] = w.qr[q];
    f[wadg_off_q(N) + nc + q] = w.qs[q];
    f[wadg_off_q(N) + 2 * nc + q] = d.refs.tri.cubature.weights[q];
  }
  for (int i = 0; i < nt; ++i)
    for (int k = 0; k < nt; ++k) f[wadg_off_mhat(N) + (std::size_t)i * nt + k] = d.refs.tri.mass(i, k);
  for (int j = 0; j < nq; ++j)
    for (int l = 0; l < nq; ++l) f[wadg_off_m1d(N) + (std::size_t)j * nq + l] = d.refs.line.mass(j, l);
  return f;
}

} // namespace

pdg_ctx* create_context(const prismdg::Discretization& d, int device, int flags, const unsigned char* owned) {
  check_device(device);
  PDG_CK(cudaSetDevice(device));
  if (d.degree < 1 || d.degree > kMaxN) throw prismdg::ConfigError("degree out of range for device path");
  auto* c = new pdg_ctx();
  try {
    c->disc = &d;
    c->device = device;
    c->flags = flags;
    PDG_CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->N = d.degree;
    c->nq = d.nq;
    c->nt = d.nt;
    c->npw = d.np_wedge;
    c->npt = d.np_tet;
    c->fw = fw_of(c->N);
    c->Kw = d.mesh.num_wedges();
    c->Kt = d.mesh.num_tets();
    c->total_dofs = (long long)d.total_dofs;
    c->tet_base = c->Kw * 4 * npd_of(c->N);
    c->dev_dofs = c->tet_base + c->Kt * 4 * c->npt;
    c->mass_mode = d.mass_mode;
    const int N = c->N, nq = c->nq, nt = c->nt, npw = c->npw, npt = c->npt;
    const bool native = flags & 1;

    // ---- element order ------------------------------------------------------
    auto word = locality_order(d.mesh, true, native);
    auto tord = locality_order(d.mesh, false, native);
    c->Kw_act = c->Kw;
    c->Kt_act = c->Kt;
    c->Kw_int = c->Kw;
    c->Kt_int = c->Kt;
    const int mr_extra = (flags >> 8) & 15;
    if (mr_extra > 0) {
      // multi-rate levels from the local stable step h_e / c_e (h = volume /
      // surface area, estimate_dt's per-element term, solver.cpp:437-447):
      // level g holds the elements whose step is >= 2^g times the smallest
      if (owned) throw prismdg::ConfigError("multi-rate stepping on a partitioned context is not supported");
      const int ne = d.num_elements(), nw = d.mesh.num_wedges();
      std::vector<double> rate(ne);
      double rmin = std::numeric_limits<double>::max();
      for (int e = 0; e < ne; ++e) {
        const double h = e < nw ? d.wgeo[e].volume / d.wgeo[e].surface_area
                                : d.tgeo[e - nw].volume / d.tgeo[e - nw].surface_area;
        rate[e] = h / d.mesh.media[e].wavespeed();
        rmin = std::min(rmin, rate[e]);
      }
      c->mr_level_ref.assign(ne, 0);
      int top = 0;
      for (int e = 0; e < ne; ++e) {
        int g = 0;
        while (g < mr_extra && rate[e] >= std::ldexp(rmin, g + 1) * (1.0 - 1e-12)) ++g;
        c->mr_level_ref[e] = g;
        top = std::max(top, g);
      }
      c->mr_nlev = top + 1;
      auto by_level = [&](std::vector<long long>& ord, std::vector<long long>& bounds, long long base) {
        std::stable_sort(ord.begin(), ord.end(),
                         [&](long long a, long long b) { return c->mr_level_ref[a] < c->mr_level_ref[b]; });
        bounds.assign(c->mr_nlev + 1, 0);
        for (long long r : ord) ++bounds[c->mr_level_ref[r] + 1];
        for (int g = 0; g < c->mr_nlev; ++g) bounds[g + 1] += bounds[g];
        (void)base;
      };
      by_level(word, c->mr_w, 0);
      by_level(tord, c->mr_t, nw);
    }
    if (owned) {
      // owned interior (no ghost neighbour) first, then owned boundary, then
      // ghosts; stable, so each group keeps the locality order.  The interior
      // stage launch can then run while the ghost traces are exchanged.
      auto interior = [&](long long r) {
        if (!owned[r]) return false;
        for (int f = 0; f < d.mesh.num_faces((int)r); ++f) {
          const int nb = d.conn.at((int)r, f).nbr;
          if (nb >= 0 && !owned[nb]) return false;
        }
        return true;
      };
      auto split = [&](std::vector<long long>& ord, long long& n_act, long long& n_int) {
        std::stable_partition(ord.begin(), ord.end(), [&](long long r) { return owned[r] != 0; });
        n_act = (long long)std::count_if(ord.begin(), ord.end(), [&](long long r) { return owned[r] != 0; });
        std::stable_partition(ord.begin(), ord.begin() + n_act, interior);
        n_int = (long long)std::count_if(ord.begin(), ord.begin() + n_act, interior);
      };
      split(word, c->Kw_act, c->Kw_int);
      split(tord, c->Kt_act, c->Kt_int);
    }
    c->dev_to_ref_host.resize(c->Kw + c->Kt);
    std::copy(word.begin(), word.end(), c->dev_to_ref_host.begin());
    std::copy(tord.begin(), tord.end(), c->dev_to_ref_host.begin() + c->Kw);
    const long long K = c->Kw + c->Kt;
    std::vector<int> ref_to_dev(K);
    for (long long q = 0; q < K; ++q) ref_to_dev[c->dev_to_ref_host[q]] = (int)q;
    {
      std::vector<int> d2r(K);
      for (long long q = 0; q < K; ++q) d2r[q] = (int)c->dev_to_ref_host[q];
      c->dev_to_ref = upload(d2r);
      std::vector<long long> offs(d.elem_offset.begin(), d.elem_offset.end());
      c->ref_offset = upload(offs);
    }

    // ---- neighbour node maps (one per distinct (kind, face, perm)) ----------
    std::map<std::tuple<int, int, int>, int> combo_id;
    std::vector<std::vector<int>> combos;
    c->max_nfp = std::max(nq * nq, nt);
    auto combo_of = [&](int nbr_ref, int nbr_face, int perm_id) {
      const bool nw = d.mesh.kind(nbr_ref) == prismdg::ElemKind::wedge;
      const auto key = std::make_tuple(nw ? 0 : 1, nbr_face, perm_id);
      auto it = combo_id.find(key);
      if (it != combo_id.end()) return it->second;
      const auto& lst = nw ? d.refs.wedge.face_nodes[nbr_face] : d.refs.tet.face_nodes[nbr_face];
      const auto& perm = d.conn.perms[perm_id];
      std::vector<int> row(c->max_nfp, 0);
      for (std::size_t m = 0; m < perm.size(); ++m) row[m] = dev_node_of(d, nw, lst[perm[m]]);
      const int id = (int)combos.size();
      combos.push_back(row);
      combo_id.emplace(key, id);
      return id;
    };

    // ---- wedge records --------------------------------------------------------
    const int WG = wg_of(N);
    {
      std::vector<double> geo((std::size_t)c->Kw * WG, 0.0);
      std::vector<int> conn((std::size_t)c->Kw * kWC, -1);
      for (long long q = 0; q < c->Kw; ++q) {
        const int r = (int)word[q];
        const auto& g = d.wgeo[r];
        double* G = geo.data() + q * WG;
        G[W_RX] = g.rx;
        G[W_RY] = g.ry;
        G[W_SX] = g.sx;
        G[W_SY] = g.sy;
        G[W_TZJ] = g.tzJ;
        G[W_JFB] = g.jf_bottom;
        G[W_JFT] = g.jf_top;
        G[W_KAPPA] = d.mesh.media[r].kappa;
        G[W_IRHO] = 1.0 / d.mesh.media[r].rho;
        for (int j = 0; j < nq; ++j) {
          G[W_TXJ + j] = d.txJ[(std::size_t)r * nq + j];
          G[w_tyj(N) + j] = d.tyJ[(std::size_t)r * nq + j];
        }
        for (int f = 0; f < 5; ++f) {
          const auto& fp = d.fphys[d.conn.face_offset[r] + f];
          for (int a = 0; a < 3; ++a) G[w_nrm(N) + 3 * f + a] = fp.normal[a];
          G[w_taup(N) + f] = fp.tau_p;
          G[w_tauu(N) + f] = fp.tau_u;
          const auto& fc = d.conn.at(r, f);
          conn[q * kWC + 2 * f] = fc.nbr >= 0 ? ref_to_dev[fc.nbr] : -1;
          conn[q * kWC + 2 * f + 1] = fc.nbr >= 0 ? combo_of(fc.nbr, fc.nbr_face, fc.perm_id) : 0;
        }
        G[w_jac(N)] = g.j0;
        G[w_jac(N) + 1] = g.jr;
        G[w_jac(N) + 2] = g.js;
        for (int e = 0; e < 3; ++e) {
          G[w_jac(N) + 3 + 2 * e] = g.jf_quad[e][0];
          G[w_jac(N) + 4 + 2 * e] = g.jf_quad[e][1];
        }
      }
      c->wgeo = upload(geo);
      c->wconn = upload(conn);
      if (d.mass_mode == prismdg::MassMode::wadg) {
        // reduced storage: shared tables only, nothing per wedge beyond the record
        if (N > 7) throw prismdg::ConfigError("the WADG device path supports degrees 1..7");
        c->wadg = upload(flatten_wadg(d));
        c->wadg_frag = dalloc<double>(wadg_frag_size(N));
        PDG_CK(launch_wadg_frag_fill(N, c->wadg, c->wadg_frag, c->stream));
      } else {
        std::vector<long long> word0(word);
        if (c->Kw > 0 && d.quad_lift.empty()) throw prismdg::ConfigError("device path needs the quad lifts");
        static const bool force_dmma = [] {
          const char* v = std::getenv("PDG_WEDGE_KERNEL");
          return v && v[0] == 'd';
        }();
        c->wedge_simt = !force_dmma && N <= wedge_simt_max_degree();
        if (c->wedge_simt || wedge_dmma_compact_ops()) {
          // compact host layouts, no fragment padding: L [k][i], quad lifts [f][a][i]
          // (per-wedge stride padded to an even count for 16-byte TMA copies)
          c->Lt = dalloc<double>((std::size_t)c->Kw * lcomp_of(N));
          c->QL = dalloc<double>((std::size_t)c->Kw * qcomp_of(N));
          upload_permuted(c->Lt, d.tri_lift.data(), (std::size_t)nt * nt, word0, lcomp_of(N));
          upload_permuted(c->QL, d.quad_lift.data(), (std::size_t)3 * nq * nt, word0, qcomp_of(N));
        } else {
          c->Lt = dalloc<double>((std::size_t)c->Kw * lfrag_of(N));
          c->QL = dalloc<double>((std::size_t)c->Kw * qfrag_of(N));
          upload_wedge_fragments(c, d, word0);
        }
      }
    }

    // ---- tet records ------------------------------------------------------------
    {
      std::vector<double> geo((std::size_t)c->Kt * kTG, 0.0);
      std::vector<int> conn((std::size_t)c->Kt * 8, -1);
      const int nw = d.mesh.num_wedges();
      for (long long q = 0; q < c->Kt; ++q) {
        const int r = (int)tord[q];
        const auto& g = d.tgeo[r - nw];
        double* G = geo.data() + q * kTG;
        const double v[9] = {g.rx, g.ry, g.rz, g.sx, g.sy, g.sz, g.tx, g.ty, g.tz};
        for (int a = 0; a < 9; ++a) G[a] = v[a];
        for (int f = 0; f < 4; ++f) G[T_LS + f] = g.lift_scale[f];
        G[T_KAPPA] = d.mesh.media[r].kappa;
        G[T_IRHO] = 1.0 / d.mesh.media[r].rho;
        G[T_J] = g.J;
        for (int f = 0; f < 4; ++f) {
          const auto& fp = d.fphys[d.conn.face_offset[r] + f];
          for (int a = 0; a < 3; ++a) G[T_NRM + 3 * f + a] = fp.normal[a];
          G[T_TAUP + f] = fp.tau_p;
          G[T_TAUU + f] = fp.tau_u;
          const auto& fc = d.conn.at(r, f);
          conn[q * 8 + 2 * f] = fc.nbr >= 0 ? ref_to_dev[fc.nbr] : -1;
          conn[q * 8 + 2 * f + 1] = fc.nbr >= 0 ? combo_of(fc.nbr, fc.nbr_face, fc.perm_id) : 0;
        }
      }
      c->tgeo = upload(geo);
      c->tconn = upload(conn);
    }
    {
      std::vector<int> flat;
      for (const auto& row : combos) flat.insert(flat.end(), row.begin(), row.end());
      if (flat.empty()) flat.assign(c->max_nfp, 0);
      c->nbr_nodes = upload(flat);
      c->nbr_nodes_len = (int)flat.size();
    }

    // ---- shared reference tables ---------------------------------------------
    {
      const auto& tri = d.refs.tri;
      const auto& line = d.refs.line;
      std::vector<double> DrT((std::size_t)nt * nt), DsT(DrT.size()), Mtri(DrT.size()), Xr(DrT.size()),
          Xs(DrT.size());
      for (int k = 0; k < nt; ++k)
        for (int i = 0; i < nt; ++i) {
          DrT[(std::size_t)k * nt + i] = tri.dr(i, k);
          DsT[(std::size_t)k * nt + i] = tri.ds(i, k);
          Mtri[(std::size_t)k * nt + i] = tri.mass(k, i);
          Xr[(std::size_t)k * nt + i] = tri.moment_r(k, i);
          Xs[(std::size_t)k * nt + i] = tri.moment_s(k, i);
        }
      std::vector<double> Dt((std::size_t)nq * nq), M1D(Dt.size()), prof(2 * nq), w1d(nq);
      const bool lumped = d.qmode == prismdg::QuadratureMode::lumped;
      for (int j = 0; j < nq; ++j) {
        for (int l = 0; l < nq; ++l) {
          Dt[j * nq + l] = line.diff(j, l);
          M1D[j * nq + l] = line.mass(j, l);
        }
        prof[j] = lumped ? line.lumped_lift_bottom[j] : line.lift_bottom[j];
        prof[nq + j] = lumped ? line.lumped_lift_top[j] : line.lift_top[j];
        w1d[j] = line.weights[j];
      }
      std::vector<int> wface(c->fw);
      int m = 0;
      for (int f = 0; f < 5; ++f)
        for (int id : d.refs.wedge.face_nodes[f]) wface[m++] = dev_node_of(d, true, id);
      const auto& tet = d.refs.tet;
      std::vector<double> tDrT((std::size_t)npt * npt), tDsT(tDrT.size()), tDtT(tDrT.size()),
          Mtet(tDrT.size()), tLiftT((std::size_t)4 * nt * npt);
      for (int k = 0; k < npt; ++k)
        for (int n = 0; n < npt; ++n) {
          tDrT[(std::size_t)k * npt + n] = tet.dr(n, k);
          tDsT[(std::size_t)k * npt + n] = tet.ds(n, k);
          tDtT[(std::size_t)k * npt + n] = tet.dt(n, k);
          Mtet[(std::size_t)n * npt + k] = tet.mass(n, k);
        }
      for (int col = 0; col < 4 * nt; ++col)
        for (int n = 0; n < npt; ++n) tLiftT[(std::size_t)col * npt + n] = tet.lift(n, col);
      std::vector<int> tface(4 * nt);
      for (int f = 0; f < 4; ++f)
        for (int q = 0; q < nt; ++q) tface[f * nt + q] = tet.face_nodes[f][q];
      c->DrT = upload(DrT);
      c->DsT = upload(DsT);
      c->Dt = upload(Dt);
      c->prof = upload(prof);
      c->wface_dev = upload(wface);
      c->tDrT = upload(tDrT);
      c->tDsT = upload(tDsT);
      c->tDtT = upload(tDtT);
      c->tLiftT = upload(tLiftT);
      c->tface = upload(tface);
      c->Mtri = upload(Mtri);
      c->Xr = upload(Xr);
      c->Xs = upload(Xs);
      c->M1D = upload(M1D);
      c->w1d = upload(w1d);
      c->Mtet = upload(Mtet);
    }
    if (c->Kt > 0 && tet_frag_size(N) > 0) {
      c->tet_frag = dalloc<double>(tet_frag_size(N));
      StageParams tp = base_params(c);
      PDG_CK(launch_tet_frag_fill(N, tp, c->tet_frag, c->stream));
    }

    // ---- state buffers --------------------------------------------------------
    // device-layout buffers (slice padding stays zero: no kernel writes it) and
    // the reference-layout staging buffer
    const std::size_t nd = (std::size_t)c->dev_dofs;
    c->u[0] = dalloc<double>(nd);
    c->u[1] = dalloc<double>(nd);
    c->res = dalloc<double>(nd);
    c->stage = dalloc<double>(std::max<std::size_t>((std::size_t)c->total_dofs, nd));
    PDG_CK(cudaMemsetAsync(c->u[0], 0, nd * 8, c->stream));
    PDG_CK(cudaMemsetAsync(c->u[1], 0, nd * 8, c->stream));
    PDG_CK(cudaMemsetAsync(c->res, 0, nd * 8, c->stream));
    c->scalar = dalloc<double>(1);
    c->badflag = dalloc<unsigned long long>(1);
    c->ticket = dalloc<unsigned long long>(1);
    PDG_CK(cudaMemset(c->ticket, 0, 8));

    // ---- algorithmic bytes per launch --------
    const double w8 = 8.0;
    const double wb_state_first = w8 * 3 * 4 * npw;  // u_in, res write, u_out
    const double wb_state_later = w8 * 4 * 4 * npw;  // + res read
    // exact: L^{tri,k} + quad lifts + record; WADG: the record only
    const double wb_ops = c->wadg ? w8 * wg_of(N) + 4.0 * kWC
                                  : w8 * ((double)nt * nt + 3.0 * nt * nq + (34 + 2 * nq)) + 4.0 * kWC;
    c->wedge_bytes_first = (double)c->Kw_act * (wb_state_first + wb_ops);
    c->wedge_bytes_later = (double)c->Kw_act * (wb_state_later + wb_ops);
    const double tb_ops = w8 * 35 + 32.0;
    c->tet_bytes_first = (double)c->Kt_act * (w8 * 3 * 4 * npt + tb_ops);
    c->tet_bytes_later = (double)c->Kt_act * (w8 * 4 * 4 * npt + tb_ops);
    PDG_CK(cudaStreamSynchronize(c->stream));
  } catch (...) {
    destroy_context(c);
    throw;
  }
  return c;
}

void destroy_context(pdg_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& pe : c->pending) {
    cudaEventDestroy(pe.a);
    cudaEventDestroy(pe.b);
  }
  void* ptrs[] = {c->u[0], c->u[1], c->res, c->rhs, c->stage, c->wgeo, c->wconn, c->Lt, c->QL, c->wadg, c->wadg_frag, c->tet_frag,
                  c->tgeo, c->tconn, c->DrT, c->DsT, c->Dt, c->prof, c->wface_dev, c->tDrT,
                  c->tDsT, c->tDtT, c->tLiftT, c->tface, c->nbr_nodes, c->Mtri, c->Xr, c->Xs,
                  c->M1D, c->w1d, c->Mtet, c->partials, c->scalar, c->badflag, c->ticket, c->dev_to_ref,
                  c->fh[0], c->fh[1], c->fh[2], c->mr_u0, c->mr_tmp,
                  c->ref_offset};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

void set_state(pdg_ctx* c, const double* u, bool on_device) {
  PDG_CK(cudaSetDevice(c->device));
  const std::size_t bytes = (std::size_t)c->total_dofs * 8;
  const double* src = u;
  if (!on_device) {
    PDG_CK(cudaMemcpyAsync(c->stage, u, bytes, cudaMemcpyHostToDevice, c->stream));
    src = c->stage;
  }
  PDG_CK(launch_to_device_layout(c->N, c->Kw, c->Kt, c->dev_to_ref, c->ref_offset, src, c->u[c->cur], c->stream));
  c->ab3_filled = 0; // a new state starts a new AB3 history
  c->mr_boot = 0;     // ... and a new multi-rate bootstrap
}

void get_state(pdg_ctx* c, double* u, bool on_device) {
  PDG_CK(cudaSetDevice(c->device));
  const std::size_t bytes = (std::size_t)c->total_dofs * 8;
  double* dst = on_device ? u : c->stage;
  PDG_CK(launch_to_reference_layout(c->N, c->Kw, c->Kt, c->dev_to_ref, c->ref_offset, c->u[c->cur], dst, c->stream));
  if (!on_device) PDG_CK(cudaMemcpyAsync(u, c->stage, bytes, cudaMemcpyDeviceToHost, c->stream));
  PDG_CK(cudaStreamSynchronize(c->stream));
}

// whole-domain entry points read every neighbour's current state; on a
// partitioned context the ghosts' states are only valid right after the
// caller's exchange, which only the per-stage entry (stage_lserk) is told about
static void require_unpartitioned(const pdg_ctx* c, const char* what) {
  if (c->Kw_act != c->Kw || c->Kt_act != c->Kt)
    throw prismdg::ConfigError(std::string(what) +
                               " on a partitioned context would read stale ghost states; step it stage by stage "
                               "(pdg_step_stage / pdg_step_stage_part) with a ghost exchange before each stage");
}

static void ensure_rhs(pdg_ctx* c) {
  if (!c->rhs) {
    c->rhs = dalloc<double>((std::size_t)c->dev_dofs);
    PDG_CK(cudaMemsetAsync(c->rhs, 0, (std::size_t)c->dev_dofs * 8, c->stream));
  }
}

void run_phase(pdg_ctx* c, bool wedge, bool volume) {
  PDG_CK(cudaSetDevice(c->device));
  require_unpartitioned(c, "a phase function");
  ensure_rhs(c);
  StageParams p = base_params(c);
  p.u_in = c->u[c->cur];
  p.rhs_out = c->rhs;
  p.mode = volume ? M_VOLUME : (M_SURFACE | M_ACCUM);
  launch_checked(c, p, wedge);
}

void compute_rhs(pdg_ctx* c, const double* u, double* rhs, bool on_device) {
  PDG_CK(cudaSetDevice(c->device));
  require_unpartitioned(c, "compute_rhs");
  ensure_rhs(c);
  const std::size_t bytes = (std::size_t)c->total_dofs * 8;
  const double* src = u;
  if (!on_device) {
    PDG_CK(cudaMemcpyAsync(c->stage, u, bytes, cudaMemcpyHostToDevice, c->stream));
    src = c->stage;
  }
  double* tmp = c->u[1 - c->cur]; // ping-pong target is free between steps
  PDG_CK(launch_to_device_layout(c->N, c->Kw, c->Kt, c->dev_to_ref, c->ref_offset, src, tmp, c->stream));
  StageParams p = base_params(c);
  p.u_in = tmp;
  p.rhs_out = c->rhs;
  p.mode = M_VOLUME | M_SURFACE | M_MEDIA;
  launch_checked(c, p, true);
  launch_checked(c, p, false);
  double* dst = on_device ? rhs : c->stage;
  PDG_CK(launch_to_reference_layout(c->N, c->Kw, c->Kt, c->dev_to_ref, c->ref_offset, c->rhs, dst, c->stream));
  if (!on_device) PDG_CK(cudaMemcpyAsync(rhs, c->stage, bytes, cudaMemcpyDeviceToHost, c->stream));
  PDG_CK(cudaStreamSynchronize(c->stream));
}

void set_rhs(pdg_ctx* c, const double* rhs, bool on_device) {
  PDG_CK(cudaSetDevice(c->device));
  ensure_rhs(c);
  const std::size_t bytes = (std::size_t)c->total_dofs * 8;
  const double* src = rhs;
  if (!on_device) {
    PDG_CK(cudaMemcpyAsync(c->stage, rhs, bytes, cudaMemcpyHostToDevice, c->stream));
    src = c->stage;
  }
  PDG_CK(launch_to_device_layout(c->N, c->Kw, c->Kt, c->dev_to_ref, c->ref_offset, src, c->rhs, c->stream));
  PDG_CK(cudaStreamSynchronize(c->stream));
}

void get_rhs(pdg_ctx* c, double* rhs, bool on_device) {
  PDG_CK(cudaSetDevice(c->device));
  ensure_rhs(c);
  const std::size_t bytes = (std::size_t)c->total_dofs * 8;
  double* dst = on_device ? rhs : c->stage;
  PDG_CK(launch_to_reference_layout(c->N, c->Kw, c->Kt, c->dev_to_ref, c->ref_offset, c->rhs, dst, c->stream));
  if (!on_device) PDG_CK(cudaMemcpyAsync(rhs, c->stage, bytes, cudaMemcpyDeviceToHost, c->stream));
  PDG_CK(cudaStreamSynchronize(c->stream));
}

void step_lserk(pdg_ctx* c, double dt, int nsteps) {
  PDG_CK(cudaSetDevice(c->device));
  require_unpartitioned(c, "a whole LSERK step");
  StageParams p = base_params(c);
  p.res = c->res;
  p.dt = dt;
  for (int n = 0; n < nsteps; ++n)
    for (int s = 0; s < 5; ++s) {
      p.u_in = c->u[c->cur];
      p.u_out = c->u[1 - c->cur];
      p.a = kRK4A[s];
      p.b = kRK4B[s];
      p.mode = M_VOLUME | M_SURFACE | M_MEDIA | M_LSERK | (s == 0 ? M_FIRST : 0);
      launch_checked(c, p, true);
      launch_checked(c, p, false);
      if (s == 0) ++c->stage_launches_first; else ++c->stage_launches_later;
      c->cur = 1 - c->cur;
    }
}

// rhs of the current state (device layout) into dst: every kernel family in
// rhs mode (volume + surface + media), as compute_rhs (solver.cpp:362-377)
static void rhs_into(pdg_ctx* c, double* dst) {
  StageParams p = base_params(c);
  p.u_in = c->u[c->cur];
  p.rhs_out = dst;
  p.mode = M_VOLUME | M_SURFACE | M_MEDIA;
  launch_checked(c, p, true);
  launch_checked(c, p, false);
}

// the AB3 step fused into the exact DMMA wedge stage kernel (wedge-only meshes,
// N = 4..7); PDG_AB3_FUSED=0 keeps the rhs launch + update kernel
static bool ab3_fused(const pdg_ctx* c) {
  static const int env = [] {
    const char* v = std::getenv("PDG_AB3_FUSED");
    return v ? std::atoi(v) : 1;
  }();
  return env != 0 && c->Kt == 0 && !c->wadg && !c->wedge_simt && wedge_stage_ab3_supported(c->N) &&
         !use_wedge_ws(c->N);
}

void step_ab3(pdg_ctx* c, double dt, int nsteps) {
  PDG_CK(cudaSetDevice(c->device));
  require_unpartitioned(c, "AB3");
  const std::size_t nd = (std::size_t)c->dev_dofs;
  for (auto& h : c->fh)
    if (!h) {
      h = dalloc<double>(nd);
      PDG_CK(cudaMemsetAsync(h, 0, nd * 8, c->stream)); // slice padding stays zero
    }
  for (int n = 0; n < nsteps; ++n) {
    if (c->ab3_filled < 2) {
      // record f at the step start into h[2 - filled], then one LSERK step
      rhs_into(c, c->fh[2 - c->ab3_filled]);
      step_lserk(c, dt, 1);
      ++c->ab3_filled;
      continue;
    }
    if (ab3_fused(c)) {
      // one launch: f_n into the free history slot and u_{n+1} into the other
      // state buffer (the update kernel's arithmetic, in the stage epilogue)
      StageParams p = base_params(c);
      p.u_in = c->u[c->cur];
      p.u_out = c->u[1 - c->cur];
      p.rhs_out = c->fh[0];
      p.h1 = c->fh[1];
      p.h2 = c->fh[2];
      p.dt = dt / 12.0;
      p.mode = M_VOLUME | M_SURFACE | M_MEDIA | M_AB3;
      launch_checked(c, p, true);
      c->cur = 1 - c->cur;
    } else {
      rhs_into(c, c->fh[0]);
      PDG_CK(launch_ab3_update((long long)nd, c->u[c->cur], c->fh[0], c->fh[1], c->fh[2], dt, c->stream));
    }
    // h[2] <- h[1], h[1] <- f_n, the old h[2] becomes the free slot
    double* f2 = c->fh[2];
    c->fh[2] = c->fh[1];
    c->fh[1] = c->fh[0];
    c->fh[0] = f2;
  }
}

void step_mrab(pdg_ctx* c, double dt, int nmacro) {
  // Multi-rate Adams-Bashforth 3 (the paper's integrator, after
  // Goedel et al. 2010): level g advances with h_g = 2^g dt; a macro step is
  // M = 2^L fine substeps.  At substep k every level starting a step (k mod
  // 2^g == 0) evaluates its rhs (reading the current / predicted states of its
  // neighbours); then each level either commits its AB3 step or writes the
  // AB3 predictor at theta = (k mod 2^g + 1) / 2^g for the finer levels that
  // read it next.  Bootstrap: the first two macro steps are LSERK45 at dt
  // (the reference's AB3 bootstrap, solver.cpp:563-570, per level), recording
  // f_g at t - h_g and t - 2 h_g.
  PDG_CK(cudaSetDevice(c->device));
  require_unpartitioned(c, "multi-rate AB3");
  if (c->mr_nlev == 0)
    throw prismdg::ConfigError("multi-rate stepping needs a context created with PDG_CTX_MRAB_LEVELS(L)");
  const std::size_t nd = (std::size_t)c->dev_dofs;
  for (auto& h : c->fh)
    if (!h) {
      h = dalloc<double>(nd);
      PDG_CK(cudaMemsetAsync(h, 0, nd * 8, c->stream));
    }
  if (!c->mr_u0) {
    c->mr_u0 = dalloc<double>(nd);
    c->mr_tmp = dalloc<double>(nd);
    PDG_CK(cudaMemsetAsync(c->mr_tmp, 0, nd * 8, c->stream));
  }
  const int nlev = c->mr_nlev, M = 1 << (nlev - 1);
  const long long wblk = 4LL * npd_of(c->N), tblk = 4LL * c->npt;
  auto wr = [&](int g, long long& a, long long& b) {
    a = c->mr_w[g] * wblk;
    b = c->mr_w[g + 1] * wblk;
  };
  auto tr = [&](int g, long long& a, long long& b) {
    a = c->tet_base + c->mr_t[g] * tblk;
    b = c->tet_base + c->mr_t[g + 1] * tblk;
  };
  auto copy_level = [&](int g, const double* src, double* dst) {
    long long a, b;
    wr(g, a, b);
    if (b > a) PDG_CK(cudaMemcpyAsync(dst + a, src + a, (b - a) * 8, cudaMemcpyDeviceToDevice, c->stream));
    tr(g, a, b);
    if (b > a) PDG_CK(cudaMemcpyAsync(dst + a, src + a, (b - a) * 8, cudaMemcpyDeviceToDevice, c->stream));
  };
  for (int m = 0; m < nmacro; ++m) {
    if (c->mr_boot < 2) {
      if (c->mr_boot == 0)
        for (int g = 0; g < nlev; ++g) c->mr_slot[g][0] = 0, c->mr_slot[g][1] = 1, c->mr_slot[g][2] = 2;
      for (int k = 0; k < M; ++k) {
        const int nb = c->mr_boot * M + k;
        bool need = false;
        for (int g = 0; g < nlev; ++g) need = need || nb == 2 * M - (1 << g) || nb == 2 * M - (2 << g);
        if (need) {
          rhs_into(c, c->mr_tmp);
          for (int g = 0; g < nlev; ++g) {
            if (nb == 2 * M - (1 << g)) copy_level(g, c->mr_tmp, c->fh[c->mr_slot[g][1]]);
            if (nb == 2 * M - (2 << g)) copy_level(g, c->mr_tmp, c->fh[c->mr_slot[g][2]]);
          }
        }
        step_lserk(c, dt, 1);
      }
      if (++c->mr_boot == 2)
        PDG_CK(cudaMemcpyAsync(c->mr_u0, c->u[c->cur], nd * 8, cudaMemcpyDeviceToDevice, c->stream));
      continue;
    }
    for (int k = 0; k < M; ++k) {
      for (int g = 0; g < nlev; ++g) {
        if (k % (1 << g) != 0) continue;
        StageParams p = base_params(c);
        p.u_in = c->u[c->cur];
        p.rhs_out = c->fh[c->mr_slot[g][0]];
        p.mode = M_VOLUME | M_SURFACE | M_MEDIA;
        p.Kw_begin = c->mr_w[g];
        p.Kw_active = c->mr_w[g + 1];
        p.Kt_begin = c->mr_t[g];
        p.Kt_active = c->mr_t[g + 1];
        launch_checked(c, p, true);
        launch_checked(c, p, false);
      }
      for (int g = 0; g < nlev; ++g) {
        const int kk = k % (1 << g);
        const bool commit = kk + 1 == (1 << g);
        long long w0, w1, t0, t1;
        wr(g, w0, w1);
        tr(g, t0, t1);
        int* sl = c->mr_slot[g];
        PDG_CK(launch_mrab_update(w0, w1, t0, t1, c->u[c->cur], c->mr_u0, c->fh[sl[0]], c->fh[sl[1]], c->fh[sl[2]],
                                  std::ldexp(dt, g), (double)(kk + 1) / (1 << g), commit ? 1 : 0, c->stream));
        if (commit) {
          const int f2 = sl[2];
          sl[2] = sl[1];
          sl[1] = sl[0];
          sl[0] = f2;
        }
      }
    }
  }
}

void stage_lserk(pdg_ctx* c, double dt, int s, int part) {
  PDG_CK(cudaSetDevice(c->device));
  if (s < 0 || s > 4) throw prismdg::ConfigError("LSERK stage index must be in [0,5)");
  if (part < 0 || part > 2) throw prismdg::ConfigError("stage part must be 0 (all), 1 (interior) or 2 (boundary)");
  StageParams p = base_params(c);
  if (part == 1) {
    p.Kw_active = c->Kw_int;
    p.Kt_active = c->Kt_int;
  } else if (part == 2) {
    p.Kw_begin = c->Kw_int;
    p.Kt_begin = c->Kt_int;
  }
  p.res = c->res;
  p.dt = dt;
  p.u_in = c->u[c->cur];
  p.u_out = c->u[1 - c->cur];
  p.a = kRK4A[s];
  p.b = kRK4B[s];
  p.mode = M_VOLUME | M_SURFACE | M_MEDIA | M_LSERK | (s == 0 ? M_FIRST : 0);
  launch_checked(c, p, true);
  launch_checked(c, p, false);
  if (part == 1) return; // the boundary part completes the stage
  if (s == 0) ++c->stage_launches_first; else ++c->stage_launches_later;
  c->cur = 1 - c->cur;
}

SnapshotStream::SnapshotStream(pdg_ctx* c, Callback cb, void* user) : c_(c), cb_(cb), user_(user) {}

SnapshotStream::~SnapshotStream() {
  if (copy_) cudaStreamSynchronize(copy_);
  for (int k = 0; k < 2; ++k) {
    if (dev_[k]) cudaFree(dev_[k]);
    if (host_[k]) cudaFreeHost(host_[k]);
    if (done_[k]) cudaEventDestroy(done_[k]);
  }
  if (copy_) cudaStreamDestroy(copy_);
}

void SnapshotStream::deliver() {
  if (!pending_) return;
  const int k = (count_ - 1) & 1;
  PDG_CK(cudaEventSynchronize(done_[k]));
  pending_ = false;
  cb_(host_[k], pending_time_, count_ - 1, user_);
}

void SnapshotStream::take(double time) {
  PDG_CK(cudaSetDevice(c_->device));
  const std::size_t n = (std::size_t)c_->total_dofs;
  if (!copy_) {
    PDG_CK(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      dev_[k] = dalloc<double>(n);
      PDG_CK(cudaMallocHost(&host_[k], std::max<std::size_t>(n, 1) * 8));
      PDG_CK(cudaEventCreateWithFlags(&done_[k], cudaEventDisableTiming));
    }
  }
  deliver(); // the previous snapshot (other buffer pair) is handed over first
  const int k = count_ & 1;
  PDG_CK(launch_to_reference_layout(c_->N, c_->Kw, c_->Kt, c_->dev_to_ref, c_->ref_offset, c_->u[c_->cur], dev_[k],
                                    c_->stream));
  cudaEvent_t ready = nullptr;
  PDG_CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  PDG_CK(cudaEventRecord(ready, c_->stream));
  PDG_CK(cudaStreamWaitEvent(copy_, ready, 0));
  PDG_CK(cudaMemcpyAsync(host_[k], dev_[k], n * 8, cudaMemcpyDeviceToHost, copy_));
  PDG_CK(cudaEventRecord(done_[k], copy_));
  cudaEventDestroy(ready);
  pending_ = true;
  pending_time_ = time;
  ++count_;
}

void SnapshotStream::flush() {
  if (copy_) deliver();
}

void assemble_operator(pdg_ctx* c, double* A) {
  // A(:, j) = rhs(e_j).  A unit probe in element e only reaches the rows of e
  // and its face neighbours, and those rows only read e, its neighbours and
  // their neighbours: probes in elements at face-graph distance > 2 share one
  // rhs evaluation exactly (the per-row arithmetic is unchanged).  Greedy
  // distance-2 colouring in element order; 4*max(Np) evaluations per colour.
  require_unpartitioned(c, "operator assembly");
  const prismdg::Discretization& d = *c->disc;
  const int ne = d.num_elements();
  const std::size_t n = d.total_dofs;
  std::vector<std::vector<int>> nbr(ne);
  for (int e = 0; e < ne; ++e)
    for (int f = 0; f < d.mesh.num_faces(e); ++f) {
      const int q = d.conn.at(e, f).nbr;
      if (q >= 0) nbr[e].push_back(q);
    }
  std::vector<int> color(ne, -1);
  int ncolor = 0;
  std::vector<int> used;
  for (int e = 0; e < ne; ++e) {
    used.clear();
    auto visit = [&](int q) {
      if (color[q] >= 0) used.push_back(color[q]);
    };
    visit(e);
    for (int a : nbr[e]) {
      visit(a);
      for (int b : nbr[a]) visit(b);
    }
    std::sort(used.begin(), used.end());
    int cc = 0;
    for (int u : used)
      if (u == cc) ++cc;
      else if (u > cc) break;
    color[e] = cc;
    ncolor = std::max(ncolor, cc + 1);
  }
  std::vector<std::vector<int>> members(ncolor);
  for (int e = 0; e < ne; ++e) members[color[e]].push_back(e);
  int maxp = 0;
  for (int e = 0; e < ne; ++e) maxp = std::max(maxp, 4 * d.np(e));
  std::fill(A, A + n * n, 0.0);
  double *hu = nullptr, *hr = nullptr;
  PDG_CK(cudaMallocHost(&hu, n * 8));
  PDG_CK(cudaMallocHost(&hr, n * 8));
  std::fill(hu, hu + n, 0.0);
  try {
    for (int cc = 0; cc < ncolor; ++cc)
      for (int q = 0; q < maxp; ++q) {
        bool any = false;
        for (int e : members[cc])
          if (q < 4 * d.np(e)) {
            hu[d.elem_offset[e] + q] = 1.0;
            any = true;
          }
        if (!any) continue;
        compute_rhs(c, hu, hr, false);
        for (int e : members[cc]) {
          if (q >= 4 * d.np(e)) continue;
          const std::size_t col = d.elem_offset[e] + q;
          hu[col] = 0.0;
          double* Acol = A + col * n;
          auto copy_rows = [&](int r) {
            for (std::size_t k = d.elem_offset[r]; k < d.elem_offset[r + 1]; ++k) Acol[k] = hr[k];
          };
          copy_rows(e);
          for (int a : nbr[e]) copy_rows(a);
        }
      }
  } catch (...) {
    cudaFreeHost(hu);
    cudaFreeHost(hr);
    throw;
  }
  cudaFreeHost(hu);
  cudaFreeHost(hr);
}

long long trace_offsets(pdg_ctx* c, long long n, const long long* elems, const int* faces, long long* out) {
  const prismdg::Discretization& d = *c->disc;
  std::vector<long long> ref_to_dev(c->dev_to_ref_host.size());
  for (std::size_t q = 0; q < c->dev_to_ref_host.size(); ++q) ref_to_dev[c->dev_to_ref_host[q]] = (long long)q;
  long long m = 0;
  for (long long k = 0; k < n; ++k) {
    const long long r = elems[k];
    const int f = faces[k];
    if (r < 0 || r >= (long long)ref_to_dev.size()) throw prismdg::ConfigError("trace element out of range");
    const bool wedge = d.mesh.kind((int)r) == prismdg::ElemKind::wedge;
    if (f < 0 || f >= d.mesh.num_faces((int)r)) throw prismdg::ConfigError("trace face out of range");
    const long long dev = ref_to_dev[r];
    const long long base = wedge ? dev * 4 * npd_of(c->N) : c->tet_base + (dev - c->Kw) * 4 * c->npt;
    const int np = wedge ? npd_of(c->N) : c->npt;
    const auto& nodes = d.my_nodes((int)r, f);
    for (int fld = 0; fld < 4; ++fld)
      for (int nref : nodes) out[m++] = base + (long long)fld * np + dev_node_of(d, wedge, nref);
  }
  return m;
}

void gather_values(pdg_ctx* c, const long long* idx, long long n, double* buf, cudaStream_t s) {
  PDG_CK(cudaSetDevice(c->device));
  PDG_CK(launch_gather_values(idx, n, c->u[c->cur], buf, s ? s : c->stream));
}

void scatter_values(pdg_ctx* c, const long long* idx, long long n, const double* buf, cudaStream_t s) {
  PDG_CK(cudaSetDevice(c->device));
  PDG_CK(launch_scatter_values(idx, n, buf, c->u[c->cur], s ? s : c->stream));
}

void pack_states(pdg_ctx* c, const long long* dev_elems, long long n, double* buf) {
  PDG_CK(cudaSetDevice(c->device));
  PDG_CK(launch_pack_states(c->N, c->Kw, dev_elems, n, c->u[c->cur], buf, c->stream));
}

void unpack_states(pdg_ctx* c, const long long* dev_elems, long long n, const double* buf) {
  PDG_CK(cudaSetDevice(c->device));
  PDG_CK(launch_unpack_states(c->N, c->Kw, dev_elems, n, buf, c->u[c->cur], c->stream));
}

double energy(pdg_ctx* c) {
  PDG_CK(cudaSetDevice(c->device));
  const int NT = c->nt;
  const int E = (256 / NT) > 0 ? 256 / NT : 1;
  const int need = (int)((c->Kw_act + E - 1) / E + (c->Kw_act + 3) / 4 + c->Kt_act) + 1;
  if (need > c->partials_cap) {
    if (c->partials) cudaFree(c->partials);
    c->partials = dalloc<double>(need);
    c->partials_cap = need;
  }
  EnergyParams p{};
  p.Kw = c->Kw_act; // owned elements only (ghosts belong to another rank)
  p.Kt = c->Kt_act;
  p.tet_base = c->tet_base;
  p.u = c->u[c->cur];
  p.wgeo = c->wgeo;
  p.tgeo = c->tgeo;
  p.Mtri = c->Mtri;
  p.Xr = c->Xr;
  p.Xs = c->Xs;
  p.M1D = c->M1D;
  p.w1d = c->w1d;
  p.Mtet = c->Mtet;
  p.lumped = c->mass_mode == prismdg::MassMode::lumped;
  p.wadg = c->wadg;
  p.partials = c->partials;
  int nb = 0;
  if (c->wadg) {
    // wedges in the Mtilde norm (one partial per 4 wedges), then the tets
    int nbw = 0, nbt = 0;
    PDG_CK(launch_wadg_energy(c->N, p, &nbw, c->stream));
    EnergyParams pt = p;
    pt.Kw = 0;
    pt.partials = c->partials + nbw;
    PDG_CK(launch_energy(c->N, pt, &nbt, c->stream));
    nb = nbw + nbt;
  } else {
    PDG_CK(launch_energy(c->N, p, &nb, c->stream));
  }
  if (nb == 0) return 0.0;
  PDG_CK(launch_reduce_sum(c->partials, nb, c->scalar, c->stream));
  double e = 0.0;
  PDG_CK(cudaMemcpyAsync(&e, c->scalar, 8, cudaMemcpyDeviceToHost, c->stream));
  PDG_CK(cudaStreamSynchronize(c->stream));
  return e;
}

long long check_finite(pdg_ctx* c) {
  PDG_CK(cudaSetDevice(c->device));
  const unsigned long long none = std::numeric_limits<unsigned long long>::max();
  PDG_CK(cudaMemcpyAsync(c->badflag, &none, 8, cudaMemcpyHostToDevice, c->stream));
  PDG_CK(launch_check_finite(c->N, c->Kw, c->Kw_act, c->Kt_act, c->u[c->cur], c->dev_to_ref, c->badflag, c->stream));
  unsigned long long r = none;
  PDG_CK(cudaMemcpyAsync(&r, c->badflag, 8, cudaMemcpyDeviceToHost, c->stream));
  PDG_CK(cudaStreamSynchronize(c->stream));
  return r == none ? -1 : (long long)r;
}

void synchronize(pdg_ctx* c) {
  PDG_CK(cudaSetDevice(c->device));
  PDG_CK(cudaStreamSynchronize(c->stream));
  PDG_CK(cudaGetLastError());
}

void kernel_times(pdg_ctx* c, double* wms, long long* wl, double* tms, long long* tl, bool reset) {
  PDG_CK(cudaStreamSynchronize(c->stream));
  for (auto& pe : c->pending) {
    float ms = 0.0f;
    PDG_CK(cudaEventElapsedTime(&ms, pe.a, pe.b));
    if (pe.family == 0) {
      c->wedge_ms += ms;
      ++c->wedge_launches;
    } else {
      c->tet_ms += ms;
      ++c->tet_launches;
    }
    cudaEventDestroy(pe.a);
    cudaEventDestroy(pe.b);
  }
  c->pending.clear();
  *wms = c->wedge_ms;
  *wl = c->wedge_launches;
  *tms = c->tet_ms;
  *tl = c->tet_launches;
  if (reset) {
    c->wedge_ms = c->tet_ms = 0.0;
    c->wedge_launches = c->tet_launches = 0;
    c->stage_launches_first = c->stage_launches_later = 0;
  }
}

void stage_bytes(pdg_ctx* c, double* wb, double* tb) {
  // average over the 5 stages of a step (stage 0 does not read res)
  *wb = (c->wedge_bytes_first + 4.0 * c->wedge_bytes_later) / 5.0;
  *tb = (c->tet_bytes_first + 4.0 * c->tet_bytes_later) / 5.0;
}

} // namespace pdg
