#pragma once
// Device context behind the C ABI (pdg_ctx): owns every device buffer of one
// discretization on one GPU and issues all work on one stream.
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "pdg_device.cuh"
#include "prismdg/discretization.hpp"

struct pdg_ctx {
  const prismdg::Discretization* disc = nullptr; // must outlive the context
  int device = 0;
  cudaStream_t stream = nullptr;
  int flags = 0;
  int N = 0, nq = 0, nt = 0, npw = 0, npt = 0, fw = 0;
  long long Kw = 0, Kt = 0, total_dofs = 0, tet_base = 0;
  long long dev_dofs = 0; // device state size: wedge blocks padded to nts_of(N) per slice
  long long Kw_act = 0, Kt_act = 0; // owned (computed) elements; ghosts follow them
  long long Kw_int = 0, Kt_int = 0; // owned elements without ghost neighbours (they come first)
  prismdg::MassMode mass_mode = prismdg::MassMode::exact;

  double* u[2] = {nullptr, nullptr};
  int cur = 0;
  double* res = nullptr;
  double* rhs = nullptr;
  double* stage = nullptr; // reference-layout staging buffer (total_dofs)
  // AB3 history (TimeStepper fhist_, solver.cpp:527-532): fh[0] free slot for
  // f_n, fh[1] = f_{n-1}, fh[2] = f_{n-2}; allocated on first use
  double* fh[3] = {nullptr, nullptr, nullptr};
  int ab3_filled = 0;

  double* wgeo = nullptr;
  int* wconn = nullptr;
  double* Lt = nullptr;
  double* QL = nullptr;
  double* wadg = nullptr; // WADG shared tables (mass_mode == wadg)
  double* wadg_frag = nullptr; // fragment-major copy of the big WADG tables
  double* tet_frag = nullptr;  // fragment-major tet operators (N >= 6, read from L2/L1)
  bool wedge_simt = false; // low-order CUDA-core wedge kernel (compact L / quad-lift layout)
  double* tgeo = nullptr;
  int* tconn = nullptr;

  double *DrT = nullptr, *DsT = nullptr, *Dt = nullptr, *prof = nullptr;
  int* wface_dev = nullptr;
  double *tDrT = nullptr, *tDsT = nullptr, *tDtT = nullptr, *tLiftT = nullptr;
  int* tface = nullptr;
  int* nbr_nodes = nullptr;
  int max_nfp = 0;
  int nbr_nodes_len = 0;
  double *Mtri = nullptr, *Xr = nullptr, *Xs = nullptr, *M1D = nullptr, *w1d = nullptr,
         *Mtet = nullptr;
  double* partials = nullptr;
  int partials_cap = 0;
  double* scalar = nullptr;
  unsigned long long* badflag = nullptr;
  unsigned long long* ticket = nullptr;       // device work counter (never reset)
  unsigned long long ticket_next = 0;         // host copy of the next ticket base

  int* dev_to_ref = nullptr;      // device element -> reference element
  long long* ref_offset = nullptr; // reference elem_offset (K+1)
  std::vector<long long> dev_to_ref_host;

  // timing (PDG_CTX_TIMING)
  struct Pending {
    cudaEvent_t a, b;
    int family; // 0 wedge, 1 tet
  };
  std::vector<Pending> pending;
  double wedge_ms = 0.0, tet_ms = 0.0;
  long long wedge_launches = 0, tet_launches = 0;

  pdg::LaunchInfo last_launch[2]; // most recent wedge / tet stage launch

  // multi-rate AB3 (PDG_CTX_MRAB_LEVELS): rate level g steps with 2^g dt;
  // levels are contiguous in device order: wedges [mr_w[g], mr_w[g+1]),
  // tets Kw + [mr_t[g], mr_t[g+1])
  int mr_nlev = 0;
  std::vector<long long> mr_w, mr_t;
  std::vector<int> mr_level_ref;   // level of every reference element
  double* mr_u0 = nullptr;         // state at each level's current step start
  double* mr_tmp = nullptr;        // bootstrap rhs
  int mr_slot[16][3] = {};         // per level: fh index of f_n, f_{n-1}, f_{n-2}
  int mr_boot = 0;                 // bootstrap macro steps done (2 = running)

  double wedge_bytes_first = 0.0, wedge_bytes_later = 0.0;
  double tet_bytes_first = 0.0, tet_bytes_later = 0.0;
  long long stage_launches_first = 0, stage_launches_later = 0;
};

namespace pdg {

/// builds device buffers; throws prismdg::DeviceError on CUDA failures.  With
/// `owned` (one flag per reference element) only owned elements are computed;
/// ghosts are ordered after the owned elements of their kind.
pdg_ctx* create_context(const prismdg::Discretization& d, int device, int flags,
                        const unsigned char* owned = nullptr);
/// one LSERK stage over the owned elements (part 0), only the interior ones
/// (part 1: no ghost data needed, state not flipped) or only the boundary ones
/// (part 2: after the ghost refresh; flips the state)
void stage_lserk(pdg_ctx* c, double dt, int stage, int part = 0);
/// device-layout state offsets of the face traces (4 fields x face nodes) of
/// (reference element, face) pairs; returns the number written
long long trace_offsets(pdg_ctx* c, long long n, const long long* elems, const int* faces, long long* out);
/// Snapshot streaming of the run driver: the current state is converted to
/// the reference layout into one of two device buffers on the compute stream,
/// copied to one of two pinned host buffers on a copy stream (overlapping the
/// following steps), and handed to the callback once landed -- at the latest
/// when the next snapshot is taken or at flush().
class SnapshotStream {
 public:
  using Callback = void (*)(const double* u, double time, int index, void* user);
  SnapshotStream(pdg_ctx* c, Callback cb, void* user);
  ~SnapshotStream();
  void take(double time);
  void flush();

 private:
  void deliver();
  pdg_ctx* c_;
  Callback cb_;
  void* user_;
  cudaStream_t copy_ = nullptr;
  double* dev_[2] = {nullptr, nullptr};
  double* host_[2] = {nullptr, nullptr};
  cudaEvent_t done_[2] = {nullptr, nullptr};
  int count_ = 0;
  bool pending_ = false;
  double pending_time_ = 0.0;
};

/// dense RHS operator (assemble_global, analysis.cpp:12-40), column-major n x n
/// in the reference layout, from distance-2 colored batches of unit probes
void assemble_operator(pdg_ctx* c, double* A);
void gather_values(pdg_ctx* c, const long long* idx, long long n, double* buf, cudaStream_t s = nullptr);
void scatter_values(pdg_ctx* c, const long long* idx, long long n, const double* buf, cudaStream_t s = nullptr);
void pack_states(pdg_ctx* c, const long long* dev_elems, long long n, double* buf);
void unpack_states(pdg_ctx* c, const long long* dev_elems, long long n, const double* buf);
void destroy_context(pdg_ctx* c);
void set_state(pdg_ctx* c, const double* u, bool on_device);
void get_state(pdg_ctx* c, double* u, bool on_device);
void compute_rhs(pdg_ctx* c, const double* u, double* rhs, bool on_device);
void run_phase(pdg_ctx* c, bool wedge, bool volume);
void get_rhs(pdg_ctx* c, double* rhs, bool on_device);
void set_rhs(pdg_ctx* c, const double* rhs, bool on_device);
void step_lserk(pdg_ctx* c, double dt, int nsteps);
/// nsteps AB3 steps with the LSERK bootstrap of TimeStepper::step (solver.cpp:559-581)
void step_ab3(pdg_ctx* c, double dt, int nsteps);
/// nmacro multi-rate AB3 macro steps (2^L fine steps of dt each); the first two
/// macro steps after set_state are the LSERK45 bootstrap at dt
void step_mrab(pdg_ctx* c, double dt, int nmacro);
double energy(pdg_ctx* c);
long long check_finite(pdg_ctx* c);
void synchronize(pdg_ctx* c);
void kernel_times(pdg_ctx* c, double* wms, long long* wl, double* tms, long long* tl, bool reset);
void stage_bytes(pdg_ctx* c, double* wb, double* tb);

} // namespace pdg
