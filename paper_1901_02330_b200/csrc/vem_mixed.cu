// vem_mixed.cu — host driver of the C ABI declared in include/vem_mixed.h.
//
// Layout in HBM:
//   A        merged saddle CSR (n = n_u + n_p rows, int32 row pointer / column
//            index, fp64 values): velocity row i = [M row i | B^T row i (cols
//            shifted by n_u)], pressure row n_u + r = B row r.  x = [u; p] is
//            streamed once per SpMV.
//   S        S_D = B diag(M)^-1 B^T, CSR, built on the device at upload.
//   V        (m+1) x ldv Krylov basis, one contiguous vector per row,
//            ldv = n rounded up to 32 doubles; Z (FGMRES) m x ldv.
//   DevState GMRES/PCG scalars, Hessenberg, Givens, device-resident so a whole
//            GMRES(m) cycle runs without a host round trip (one CUDA graph).
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/vem_mixed.h"
#include "kernels.cuh"
#include "amg.cuh"
#include "assembly.cuh"
#include "amg_apply.cuh"
#include "blockreg_m.cuh"

namespace {

constexpr int NT = 256;

struct Timed {
  int cls;
  double bytes;
  cudaEvent_t a, b;
};

// one level of the S_D aggregation hierarchy (precond kind 3)
struct AmgLevel {
  long n = 0, nnz = 0;
  int *rp = nullptr, *ci = nullptr;            // CSR (setup)
  double *va = nullptr;
  long long *soff = nullptr;                   // SELL-32 (apply)
  int *sci = nullptr;
  double *sva = nullptr;
  long nnz_sell = 0;
  double *dinv = nullptr;
  double lmax = 0.0;
  int *agg = nullptr, *moff = nullptr, *mem = nullptr;  // restriction to the next level
  long nc = 0;
  double *b = nullptr, *x = nullptr, *t = nullptr, *y = nullptr, *sr = nullptr, *sd0 = nullptr, *sd1 = nullptr;
  bool owns_matrix = true;
  bool warp_rows = false;                      // coarse levels: long Galerkin rows -> G lanes per row (CSR)
  int group = 32;                              // lanes per row of the CSR level kernels (4 .. 32)
  // smoothed aggregation (level 0): P CSR (setup), P SELL (prolongation), P^T CSR (restriction)
  bool sa = false;
  int *prp = nullptr, *pci = nullptr, *ptrp = nullptr, *ptci = nullptr, *psci = nullptr;
  double *pva = nullptr, *ptva = nullptr, *psva = nullptr;
  long long *psoff = nullptr;
  long pnnz = 0, psnnz = 0;
  // FP32 mirror for precond kind 4 (values converted once after setup; own vectors)
  float *sva_f = nullptr, *va_f = nullptr, *dinv_f = nullptr, *psva_f = nullptr, *ptva_f = nullptr;
  float *b_f = nullptr, *x_f = nullptr, *t_f = nullptr, *sr_f = nullptr, *sd0_f = nullptr, *sd1_f = nullptr;
  // coarsest level without a dense inverse: one thread-block-cluster launch per smoother
  // (k_vc_coarse_cluster): rank row ranges, packed columns, shared bytes per precision
  int *vc_rs = nullptr;
  unsigned short *vc_c16 = nullptr;
  size_t vc_smem_d = 0, vc_smem_f = 0;
  bool vc_ok = false;
};

// one aggregation hierarchy: the S_D one of kinds 3/4 (Ctx::amg) or the S_D + eps W one that
// preconditions Block-Reg's inner PCG (Ctx::amge; on the element-mean block when n_p_dof > 1)
struct AmgHier {
  std::vector<AmgLevel> lv;
  double *cinv = nullptr;      // dense inverse of the coarsest level
  float *cinv_f = nullptr;     // its FP32 copy (kind 4)
  bool dense = false;
  int coarse_degree = 32;      // Chebyshev degree of a non-dense coarsest level
};

// level data of the V-cycle in precision T
template <typename T>
struct Lv;
template <>
struct Lv<double> {
  AmgLevel &L;
  const double *sva() const { return L.sva; }
  const double *va() const { return L.va; }
  const double *dinv() const { return L.dinv; }
  const double *psva() const { return L.psva; }
  const double *ptva() const { return L.ptva; }
  double *b() const { return L.b; }
  double *x() const { return L.x; }
  double *t() const { return L.t; }
  double *sr() const { return L.sr; }
  double *sd0() const { return L.sd0; }
  double *sd1() const { return L.sd1; }
};
template <>
struct Lv<float> {
  AmgLevel &L;
  const float *sva() const { return L.sva_f; }
  const float *va() const { return L.va_f; }
  const float *dinv() const { return L.dinv_f; }
  const float *psva() const { return L.psva_f; }
  const float *ptva() const { return L.ptva_f; }
  float *b() const { return L.b_f; }
  float *x() const { return L.x_f; }
  float *t() const { return L.t_f; }
  float *sr() const { return L.sr_f; }
  float *sd0() const { return L.sd0_f; }
  float *sd1() const { return L.sd1_f; }
};

struct Ctx {
  // sizes
  long nu = 0, np = 0, n = 0, ldv = 0;
  long nnzM = 0, nnzB = 0, nnzA = 0, nnzS = 0;
  vem_layout layout{};
  vem_opts opts{};
  cudaStream_t stream = nullptr;       // library-owned non-blocking work stream (capturable)
  cudaStream_t user_stream = nullptr;  // caller's stream; ordered against `stream` with events
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  int sm_count = 148;
  double eps = 0.0;
  bool has_reg = false;
  int nb = 1;                          // pressure DOFs per element (block-Jacobi size)
  double lmax = 0.0;                   // Gershgorin bound of diag(S)^-1 S (reported)
  double lmax_cheb = 2.0;              // Chebyshev interval top: lambda_max(D_B^-1 S_D) <= 2 (R15)
  double *dBinv = nullptr, *dBeinv = nullptr, *pz = nullptr;
  double *cheb_pool = nullptr;          // D^-1, r, d0, d1, x of the Chebyshev steps, contiguous
  double *h_rhs = nullptr, *h_u = nullptr, *h_p = nullptr;   // vem_mixed_solve_host staging
  AmgHier amg;                                   // S_D hierarchy (kinds 3, 4); empty when n_p_dof > 1
  AmgHier amge;                                  // S_D + eps W hierarchy (inner PCG of kinds 2, 5; R23)
  bool amg_f32 = false;                          // FP32 mirror built
  int amg_coarse_degree = 8;                     // Chebyshev degree of a non-dense coarsest level
  int amg_max_levels = 12;                       // AMG_MAX_LEVELS (VEM_AMG_MAX_LEVELS: tests only)
  long amg_warp_rows = 100000;                   // coarse levels below this many rows: CSR group kernels
  double amg_warp_nnz = 1e30;                    // ... or with at least this many nnz per row (off: r8 A/B,
                                                 // SELL-32 beats group CSR on C3's 35-nnz/row level 1)
  int amg_group = 8;                             // lanes per CSR row (0: by the mean row length; r8 A/B)
  double amg_group_div = 2.0;                    // ... G = power of two >= mean row length / this
  int pdl = 1;                                   // programmatic dependent launch of the V-cycle kernels
  int mdot_slots = 0;                            // >0: k_mdot grid = one full wave of this many resident CTAs
  int update_slots = 0;                          // >0: k_update grid = one full wave (VEM_UPDATE_WAVE)
  int mdot32_slots = 0, update32_slots = 0;      // the same for the compressed-basis kernels
  bool pdl_skip = false;                         // next launch follows an event record: plain edge
  int amg_cluster = 0;                           // coarsest smoother as one cluster launch (VEM_AMG_CLUSTER=1;
                                                 // off by default: slower than the per-step launches)
  float *f32_pool = nullptr;                     // kind 4 fine-level vectors (L2-persisting window)
  size_t f32_pool_bytes = 0;
  int l2_window_pool = -1;                       // pool under the window: 0 FP64 Chebyshev, 1 FP32
  size_t cheb_pool_bytes = 0;
  size_t l2_window_bytes = 0;           // bytes of the pool under a persisting L2 access window
  // device matrices
  int *a_rp = nullptr, *a_ci = nullptr;
  double *a_va = nullptr;
  int *s_rp = nullptr, *s_ci = nullptr;
  double *s_va = nullptr;
  // SELL-32 copies used by every hot-path kernel
  long long *a_soff = nullptr, *s_soff = nullptr;
  int *a_sci = nullptr, *s_sci = nullptr;
  double *a_sva = nullptr, *s_sva = nullptr;
  long nnzA_sell = 0, nnzS_sell = 0;
  // SELL-C-sigma reordering (build_reorder): perm[new] = old over [u; p], cmap = its inverse;
  // perm_p / cmap_p the pressure part in pressure numbering.  nullptr: identity.
  int *perm = nullptr, *cmap = nullptr, *perm_p = nullptr, *cmap_p = nullptr;
  // S_D SELL slot -> row (internal numbering): S_D rows sorted by length at row level
  // (element-block kernels need element-contiguous rows, so the symmetric permutation
  // moves whole elements; the SELL slots of S_D add a row-level sort on top)
  int *s_slot = nullptr, *s_slot_old = nullptr;
  int pcg_split = 0;   // block PCG: q = S p with block partials, then a one-block alpha kernel
  int pcg_persist = 1; // block PCG on small systems: one cooperative launch per inner solve
  int pcg_coop_grid = 0;
  double **pfinal = nullptr;   // persistent PCG: which p buffer holds the last direction (unused after)
  std::pair<long, long> reorder_pad{0, 0};
  double *dMinv = nullptr, *dSinv = nullptr, *dSepsinv = nullptr, *wdiag = nullptr, *sdiag = nullptr;
  // work vectors
  double *V = nullptr, *Z = nullptr;
  float *V32 = nullptr;                 // float copy of the basis (opts.basis_f32; the CGS kernels read it)
  int zcap = 0;
  double *x = nullptr, *b = nullptr, *z = nullptr, *t = nullptr;
  double *cr = nullptr, *cd0 = nullptr, *cd1 = nullptr, *cx = nullptr;           // Chebyshev
  double *px = nullptr, *pr = nullptr, *pp0 = nullptr, *pp1 = nullptr, *pq = nullptr, *pb = nullptr;  // PCG
  // MG-PCG (inner_precond = 1, R23): residual / preconditioned residual of the inner PCG
  // (n_p_dof = 1: the level-0 b / x of the S_eps hierarchy; else pr / pz), the S_eps matrix the
  // hierarchy `amge` starts from (n_p_dof = 1: S_D values with the shifted diagonal; else the CSR
  // of S_eps[0::n_p, 0::n_p] in the caller's element numbering)
  double *mg_r = nullptr, *mg_z = nullptr;
  int *se_rp = nullptr, *se_ci = nullptr;
  double *se_va = nullptr, *se_dinv = nullptr, *se_diag = nullptr;
  long se_n = 0, se_nnz = 0;
  cudaGraphExec_t pcgm_exec = nullptr;
  int pcgm_exec_chunk = 0;
  cudaEvent_t mg_samp_a = nullptr, mg_samp_b = nullptr;   // timing = 2: one fine-level pass per replay
  // K-PCG (kind 5, R24): p (velocity part of kx = [p; B p]), r, z, q
  double *kx = nullptr, *kr = nullptr, *kz = nullptr, *kq = nullptr;
  int64_t k_its_total = 0;
  std::string amg_unavailable;                   // why the S_D hierarchy of kinds 3 / 4 was not built
  int hist_steps = 0;                            // Arnoldi steps of the last cycle and the norms it started from
  double hist_beta = 0.0, hist_bnorm = 0.0;
  bool trace_k = false;                          // VEM_TRACE_K=1: one stderr line per kind-5 apply
  bool k_failed = false;
  double *part = nullptr;
  unsigned *counter = nullptr;
  DevState *st = nullptr;
  DevState *hst = nullptr;  // pinned mirror
  int *derr = nullptr;
  long part_cap = 0;
  // graphs
  cudaGraphExec_t cycle_exec[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};   // per precond kind
  cudaGraphExec_t pcg_exec = nullptr;
  int pcg_exec_chunk = 0;
  // timing
  std::vector<Timed> pending;
  std::vector<cudaEvent_t> free_events;
  vem_kernel_stats stats{};
  bool capturing = false;
  // timing = 2 (sampled, graph-compatible): one Chebyshev step per Arnoldi step
  // is bracketed by its own event pair (captured as event-record graph nodes);
  // the host reads the pairs of the executed steps after every cycle.
  int sample_slot = -1;
  bool sample_recorded = false;        // set when an enqueue recorded a sample pair
  bool sample_recorded_kind[6] = {false, false, false, false, false, false};
  std::vector<cudaEvent_t> samp_a, samp_b;
  // misc
  std::string err;
  double setup_ms = 0.0;
  int64_t device_bytes = 0;
  std::vector<void *> allocs;
  std::vector<size_t> alloc_bytes;
};

int fail(Ctx *c, int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(c, VEM_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                        \
  } while (0)

// status-only check for extern "C" helpers without a context in scope
#define CK_RET(call)                       \
  do {                                     \
    if ((call) != cudaSuccess) return VEM_ERR_CUDA; \
  } while (0)
#define CKL()                                                                                 \
  do {                                                                                        \
    cudaError_t e_ = cudaGetLastError();                                                      \
    if (e_ != cudaSuccess)                                                                    \
      return fail(c, VEM_ERR_CUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                        \
  } while (0)

template <typename T>
int dalloc(Ctx *c, T **p, size_t count) {
  size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  cudaError_t e = cudaMalloc((void **)p, bytes);
  if (e != cudaSuccess) return fail(c, VEM_ERR_CUDA, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
  c->allocs.push_back(*p);
  c->alloc_bytes.push_back(bytes);
  c->device_bytes += bytes;
  return 0;
}
#define DA(p, n)                        \
  do {                                  \
    int r_ = dalloc(c, &(p), (size_t)(n)); \
    if (r_) return r_;                  \
  } while (0)

void dfree(Ctx *c, void *p) {
  if (!p) return;
  auto it = std::find(c->allocs.begin(), c->allocs.end(), p);
  if (it != c->allocs.end()) {
    const size_t i = it - c->allocs.begin();
    c->device_bytes -= (int64_t)c->alloc_bytes[i];
    c->alloc_bytes.erase(c->alloc_bytes.begin() + i);
    c->allocs.erase(it);
  }
  cudaFree(p);
}

inline int grid_for(long work, int per_block = NT) {
  long g = (work + per_block - 1) / per_block;
  return (int)std::max<long>(1, std::min<long>(g, 1L << 30));
}
inline int grid_stream(Ctx *c, long n) {   // grid-stride kernels: a few waves of 148 SMs
  long g = (n + NT - 1) / NT;
  return (int)std::max<long>(1, std::min<long>(g, (long)c->sm_count * 32));
}

// ----------------------------------------------------------------------------
// timing: events around each launch when opts.timing (never inside a capture)
// ----------------------------------------------------------------------------
cudaEvent_t take_event(Ctx *c) {
  if (!c->free_events.empty()) {
    cudaEvent_t e = c->free_events.back();
    c->free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
struct TimeScope {
  Ctx *c;
  int cls;
  double bytes;
  cudaEvent_t a = nullptr;
  TimeScope(Ctx *c_, int cls_, double bytes_ = 0.0) : c(c_), cls(cls_), bytes(bytes_) {
    if (c->opts.timing == 1 && !c->capturing) {
      a = take_event(c);
      cudaEventRecord(a, c->stream);
    }
  }
  ~TimeScope() {
    if (a) {
      cudaEvent_t b = take_event(c);
      cudaEventRecord(b, c->stream);
      c->pending.push_back({cls, bytes, a, b});
    }
  }
};
int ensure_samples(Ctx *c) {
  const int m = c->opts.restart;
  while ((int)c->samp_a.size() < m) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    c->samp_a.push_back(a);
    c->samp_b.push_back(b);
  }
  return 0;
}
// after a cycle that executed `steps` Arnoldi steps (stream synchronised)
void collect_samples(Ctx *c, int steps, double bytes) {
  if (c->opts.timing != 2 || !c->sample_recorded) return;
  for (int j = 0; j < steps && j < (int)c->samp_a.size(); ++j) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->samp_a[j], c->samp_b[j]) == cudaSuccess) {
      c->stats.launches[VEM_K_CHEB] += 1;
      c->stats.ms[VEM_K_CHEB] += ms;
      c->stats.bytes[VEM_K_CHEB] += bytes;
    } else {
      (void)cudaGetLastError();   // never leave a query error for the next launch check
    }
  }
}

void flush_timing(Ctx *c) {   // call after a stream sync
  for (auto &t : c->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, t.a, t.b) == cudaSuccess) {
      c->stats.launches[t.cls] += 1;
      c->stats.ms[t.cls] += ms;
      c->stats.bytes[t.cls] += t.bytes;
    }
    c->free_events.push_back(t.a);
    c->free_events.push_back(t.b);
  }
  c->pending.clear();
}

// ----------------------------------------------------------------------------
// launch helpers (templated on the CSR lanes-per-row)
// ----------------------------------------------------------------------------

template <template <int> class F, typename... Args>
bool dispatch_nb(int nb, Args... a) {
  switch (nb) {
    case 2: F<2>::run(a...); return true;
    case 3: F<3>::run(a...); return true;
    case 4: F<4>::run(a...); return true;
    case 5: F<5>::run(a...); return true;
    case 6: F<6>::run(a...); return true;
    case 7: F<7>::run(a...); return true;
    case 8: F<8>::run(a...); return true;
    case 9: F<9>::run(a...); return true;
    case 10: F<10>::run(a...); return true;
    default: return false;
  }
}

template <int NB>
struct BlkInvL {
  static void run(Ctx *c, double shift, double *out);
};
template <int NB>
struct ChebBlkL {
  static void run(Ctx *c, const double *dold, double *dnew, double c1, double c2, int mode, int last, double *zp,
                  const int *gate);
};
template <int NB>
struct PcgInitBlkL {
  static void run(Ctx *c, double rtol, const int *gate);
};
template <int NB>
struct MgBlkL {
  static void run(Ctx *c, const double *r, const double *dold, double *dnew, double *x, double c1, double c2,
                  int init, int acc, const int *gate);
};
template <int NB>
struct PcgVecBlkL {
  static void run(Ctx *c, const double *p);
};

Sell sellA(Ctx *c) { return Sell{c->a_soff, c->a_sci, c->a_sva}; }
Sell sellS(Ctx *c) { return Sell{c->s_soff, c->s_sci, c->s_sva, c->s_slot}; }

void launch_spmv(Ctx *c, long row0, long nrows, const double *x, double *y, const double *b, int mode,
                 const int *gate) {
  k_spmv<<<grid_for(nrows), NT, 0, c->stream>>>(row0, nrows, sellA(c), x, y, b, mode, gate);
}
void launch_residual(Ctx *c, const double *x, const double *b, double *r, int use_x) {
  k_residual_start<<<grid_for(c->n), NT, 0, c->stream>>>(c->n, sellA(c), x, b, r, use_x, c->part, c->counter, c->st);
}
void launch_cheb(Ctx *c, double *dold, double *dnew, double c1, double c2, int last, double *zp, const int *gate) {
  k_cheb_step<<<grid_for(c->np), NT, 0, c->stream>>>(c->np, sellS(c), c->dSinv, c->cr, dold, dnew, c->cx, c1, c2,
                                                     last, zp, gate);
}
void launch_schur_spmv(Ctx *c, const double *x, double *y, const int *gate) {
  k_spmv<<<grid_for(c->np), NT, 0, c->stream>>>(0, c->np, sellS(c), x, y, nullptr, 0, gate);
}
void launch_br_finish(Ctx *c, double *z, const int *gate) {
  k_br_finish<<<grid_for(c->nu), NT, 0, c->stream>>>(c->nu, sellA(c), c->dMinv, c->px, z, gate);
}
void launch_pcg_spmv(Ctx *c, const double *pprev, double *pnew) {
  k_pcg_spmv<<<grid_for(c->np), NT, 0, c->stream>>>(c->np, sellS(c), c->dSepsinv, c->wdiag, c->eps, c->pr, pprev,
                                                    pnew, c->pq, c->part, c->counter, c->st);
}
void launch_cheb_resid(Ctx *c, const double *dold, const int *gate) {
  k_cheb_resid<<<grid_for(c->np), NT, 0, c->stream>>>(c->np, sellS(c), c->cr, dold, gate);
}

// algorithmic bytes per launch (include/vem_mixed.h)
double bytes_spmv(Ctx *c) { return 12.0 * c->nnzA + 16.0 * c->n; }
double bytes_cheb(Ctx *c) { return 12.0 * c->nnzS + 56.0 * c->np; }
double bytes_pcg_vec(Ctx *c) { return 64.0 * c->np; }
double bytes_vecs(Ctx *c, double nvec) { return 8.0 * c->n * nvec; }

// blocks for the element-block kernels (BlkWarp: 32 / NB elements per warp),
// grid-stride over warps with at most one resident wave (8 blocks of 256 per SM)
template <int NB>
int grid_blk(Ctx *c, long ne) {
  const long blocks = (blk_warps<NB>(ne) * 32 + 255) / 256;
  return (int)std::max<long>(1, std::min<long>(blocks, (long)c->sm_count * 8));
}

template <int NB>
void BlkInvL<NB>::run(Ctx *c, double shift, double *out) {
  const long ne = c->np / NB;
  k_block_extract_inv<NB><<<grid_stream(c, ne), 128, 0, c->stream>>>(ne, c->s_rp, c->s_ci, c->s_va, c->wdiag, shift,
                                                                     out, c->derr);
}
template <int NB>
void ChebBlkL<NB>::run(Ctx *c, const double *dold, double *dnew, double c1, double c2, int mode, int last, double *zp,
                       const int *gate) {
  const long ne = c->np / NB;
  k_cheb_block<NB><<<grid_blk<NB>(c, ne), 256, 0, c->stream>>>(ne, c->dBinv, c->cr, dold, dnew, c->cx, c1, c2, mode,
                                                              last, zp, gate);
}
template <int NB>
void PcgInitBlkL<NB>::run(Ctx *c, double rtol, const int *gate) {
  const long ne = c->np / NB;
  k_pcg_init_blk<NB><<<grid_blk<NB>(c, ne), 256, 0, c->stream>>>(ne, c->dBeinv, c->pb, c->px, c->pr, c->pz, c->pp0,
                                                               c->part, c->counter, c->st, rtol,
                                                               c->opts.inner_maxit, gate);
}
template <int NB>
void MgBlkL<NB>::run(Ctx *c, const double *r, const double *dold, double *dnew, double *x, double c1, double c2,
                     int init, int acc, const int *gate) {
  const long ne = c->np / NB;
  k_mg_blk<NB><<<grid_blk<NB>(c, ne), 256, 0, c->stream>>>(ne, c->dBeinv, r, dold, dnew, x, c1, c2, init, acc, gate);
}
template <int NB>
void PcgVecBlkL<NB>::run(Ctx *c, const double *p) {
  const long ne = c->np / NB;
  if (c->pcg_split) {   // full grid (one element group per warp), partials reduced by k_pcg_beta
    const int g = (int)((blk_warps<NB>(ne) * 32 + 255) / 256);
    k_pcg_vec_blk<NB><<<g, 256, 0, c->stream>>>(ne, c->dBeinv, p, c->pq, c->px, c->pr, c->pz, c->part, c->counter,
                                                c->st, 1);
    k_pcg_beta<<<1, 1024, 0, c->stream>>>(g, c->part, c->st);
  } else {
    k_pcg_vec_blk<NB><<<grid_blk<NB>(c, ne), 256, 0, c->stream>>>(ne, c->dBeinv, p, c->pq, c->px, c->pr, c->pz,
                                                                c->part, c->counter, c->st, 0);
  }
}

const int *gate_one(Ctx *c) { return &c->st->one_i; }
const int *gate_active(Ctx *c) { return &c->st->g.active; }
const int *gate_steps(Ctx *c) { return &c->st->g.has_steps; }

// ----------------------------------------------------------------------------
// preconditioner applications (enqueue only)
// ----------------------------------------------------------------------------
void cheb_coeffs(Ctx *c, double &inv_theta, std::vector<double> &c1, std::vector<double> &c2) {
  const double b = c->lmax_cheb, a = c->lmax_cheb / c->opts.cheb_ratio;
  const double theta = 0.5 * (b + a), delta = 0.5 * (b - a), sigma = theta / delta;
  double rho = 1.0 / sigma;
  inv_theta = 1.0 / theta;
  c1.clear();
  c2.clear();
  for (int i = 1; i < c->opts.cheb_degree; ++i) {
    const double rn = 1.0 / (2.0 * sigma - rho);
    c1.push_back(rn * rho);
    c2.push_back(2.0 * rn / delta);
    rho = rn;
  }
}

int enqueue_block_schur(Ctx *c, const double *v, const double *scale, double *z, const int *gate) {
  double inv_theta;
  std::vector<double> c1, c2;
  cheb_coeffs(c, inv_theta, c1, c2);
  const int deg = c->opts.cheb_degree;
  const bool blk = c->nb > 1;
  if (!blk && deg > 1) {
    // k = 0: init fused into the first Chebyshev step (one launch over all n rows)
    const bool sample = c->opts.timing == 2 && c->sample_slot >= 0 && deg / 2 == 1;
    if (sample) cudaEventRecordWithFlags(c->samp_a[c->sample_slot], c->stream, cudaEventRecordExternal);
    c->sample_recorded |= sample;
    {
      TimeScope ts(c, VEM_K_CHEB, bytes_cheb(c) - 16.0 * c->np + 24.0 * c->nu);
      k_cheb_first<<<grid_for(c->n), NT, 0, c->stream>>>(c->nu, c->np, sellS(c), v, scale, c->dMinv, c->dSinv,
                                                         inv_theta, c1[0], c2[0], c->cr, c->cd1, c->cx, z,
                                                         deg == 2 ? 1 : 0, gate);
    }
    if (sample) cudaEventRecordWithFlags(c->samp_b[c->sample_slot], c->stream, cudaEventRecordExternal);
    CKL();
    double *dold = c->cd1, *dnew = c->cd0;
    for (int i = 2; i < deg; ++i) {
      const int last = i == deg - 1 ? 1 : 0;
      const bool smp = c->opts.timing == 2 && c->sample_slot >= 0 && i == deg / 2;
      if (smp) {
      cudaEventRecordWithFlags(c->samp_a[c->sample_slot], c->stream, cudaEventRecordExternal);
      c->pdl_skip = true;
    }
      c->sample_recorded |= smp;
      {
        TimeScope ts(c, VEM_K_CHEB, bytes_cheb(c));
        launch_cheb(c, dold, dnew, c1[i - 1], c2[i - 1], last, z + c->nu, gate);
      }
      if (smp) {
      cudaEventRecordWithFlags(c->samp_b[c->sample_slot], c->stream, cudaEventRecordExternal);
      c->pdl_skip = true;
    }
      std::swap(dold, dnew);
    }
    CKL();
    return 0;
  }
  // k >= 1 (element-block Jacobi) or degree 1: separate init
  {
    TimeScope ts(c, VEM_K_PRECOND_VEC, 8.0 * (3 * c->nu + 5 * c->np));
    k_bs_init<<<grid_stream(c, c->n), NT, 0, c->stream>>>(c->nu, c->np, v, scale, c->dMinv, c->dSinv, inv_theta, z,
                                                          c->cr, c->cd0, c->cx, deg == 1, blk ? 1 : 0, gate);
  }
  if (blk) {
    TimeScope ts(c, VEM_K_PRECOND_VEC, 8.0 * c->np * (3 + c->nb));
    dispatch_nb<ChebBlkL>(c->nb, c, (const double *)nullptr, c->cd0, 0.0, inv_theta, 1, deg == 1 ? 1 : 0,
                          z + c->nu, gate);
  }
  CKL();
  double *dold = c->cd0, *dnew = c->cd1;
  for (int i = 1; i < deg; ++i) {
    const int last = i == deg - 1 ? 1 : 0;
    if (blk) {
      {
        TimeScope ts(c, VEM_K_CHEB, 12.0 * c->nnzS + 24.0 * c->np);
        launch_cheb_resid(c, (const double *)dold, gate);
      }
      TimeScope ts(c, VEM_K_PRECOND_VEC, 8.0 * c->np * (5 + c->nb));
      dispatch_nb<ChebBlkL>(c->nb, c, (const double *)dold, dnew, c1[i - 1], c2[i - 1], 0, last, z + c->nu, gate);
    } else {
      const bool sample = c->opts.timing == 2 && c->sample_slot >= 0 && i == deg / 2;
      // cudaEventRecordExternal: inside a capture this becomes a real event-record node
      if (sample) cudaEventRecordWithFlags(c->samp_a[c->sample_slot], c->stream, cudaEventRecordExternal);
      c->sample_recorded |= sample;
      {
        TimeScope ts(c, VEM_K_CHEB, bytes_cheb(c));
        launch_cheb(c, dold, dnew, c1[i - 1], c2[i - 1], last, z + c->nu, gate);
      }
      if (sample) cudaEventRecordWithFlags(c->samp_b[c->sample_slot], c->stream, cudaEventRecordExternal);
    }
    std::swap(dold, dnew);
  }
  CKL();
  return 0;
}

int run_pcg(Ctx *c, int64_t *inner_its);
int run_pcg_mg(Ctx *c, double rtol, const int *gate, int64_t *inner_its);

// Inner solve px = (S_D + eps W)^-1 pb by PCG from x0 = 0 to ||r|| <= rtol ||pb||, preconditioned by
// one V-cycle of S_eps (inner_precond = 1, reading R23) or its element-block Jacobi (0, R16)
int run_inner(Ctx *c, double rtol, const int *gate, int64_t *inner_its) {
  if (c->opts.inner_precond == 1) return run_pcg_mg(c, rtol, gate, inner_its);
  {
    TimeScope ts(c, VEM_K_PRECOND_VEC);
    if (c->nb > 1)
      dispatch_nb<PcgInitBlkL>(c->nb, c, rtol, gate);
    else
      k_pcg_init<<<grid_stream(c, c->np), NT, 0, c->stream>>>(c->np, c->pb, c->dSepsinv, c->px, c->pr, c->pp0,
                                                              c->part, c->counter, c->st, rtol,
                                                              c->opts.inner_maxit, gate);
  }
  CKL();
  return run_pcg(c, inner_its);
}

int enqueue_block_reg(Ctx *c, const double *v, const double *scale, double *z, const int *gate,
                      int64_t *inner_its) {
  {
    TimeScope ts(c, VEM_K_PRECOND_VEC);
    k_br_init<<<grid_stream(c, c->n), NT, 0, c->stream>>>(c->nu, c->np, v, scale, c->dMinv, c->wdiag,
                                                          1.0 / c->eps, z, gate);
  }
  {
    TimeScope ts(c, VEM_K_PRECOND_VEC);  // rhs = B t0 (pressure rows of A)
    launch_spmv(c, c->nu, c->np, (const double *)z, c->pb - c->nu, nullptr, 0, gate);
  }
  CKL();
  int rc = run_inner(c, c->opts.inner_rtol, gate, inner_its);
  if (rc) return rc;
  {
    TimeScope ts(c, VEM_K_PRECOND_VEC);
    launch_br_finish(c, z, gate);
  }
  CKL();
  return 0;
}

int enqueue_pcg_steps(Ctx *c, int nsteps) {
  for (int s = 0; s < nsteps; ++s) {
    double *pprev = (s % 2 == 0) ? c->pp0 : c->pp1;
    double *pnew = (s % 2 == 0) ? c->pp1 : c->pp0;
    if (c->nb > 1) {
      // block path: p materialised, q = S p with one gather, then p = z + beta p
      if (c->pcg_split == 2) {
        // plain product, then the p.q partials as a separate light pass (the fused kernel's block
        // barrier costs a third of its stall cycles: 172 vs 132 us on C5, ncu R2_27)
        {
          TimeScope ts(c, VEM_K_PCG_SPMV, 12.0 * c->nnzS + 32.0 * c->np);
          k_seps_mul<<<grid_for(c->np), NT, 0, c->stream>>>(c->np, sellS(c), c->wdiag, c->eps, c->pp0, c->pq,
                                                            &c->st->p.active);
        }
        TimeScope ts(c, VEM_K_PCG_VEC, 16.0 * c->np);
        const int gp = (int)std::max<long>(1, std::min<long>((c->np + NT - 1) / NT, (long)c->sm_count * 8));
        k_dot_part<<<gp, NT, 0, c->stream>>>(c->np, c->pp0, c->pq, c->part, &c->st->p.active);
        k_pcg_alpha<<<1, 1024, 0, c->stream>>>(gp, c->part, c->st);
      } else {
        TimeScope ts(c, VEM_K_PCG_SPMV, 12.0 * c->nnzS + 32.0 * c->np);
        const int g = grid_for(c->np);
        k_pcg_spmv_p<<<g, NT, 0, c->stream>>>(c->np, sellS(c), c->wdiag, c->eps, c->pp0, c->pq, c->part,
                                              c->counter, c->st, c->pcg_split);
        if (c->pcg_split) k_pcg_alpha<<<1, 1024, 0, c->stream>>>(g, c->part, c->st);
      }
      {
        TimeScope ts(c, VEM_K_PCG_VEC, bytes_pcg_vec(c) + 8.0 * c->np * c->nb);
        dispatch_nb<PcgVecBlkL>(c->nb, c, (const double *)c->pp0);
      }
      TimeScope ts(c, VEM_K_PCG_VEC, 24.0 * c->np);
      k_pcg_pupd<<<grid_stream(c, c->np), NT, 0, c->stream>>>(c->np, c->pz, c->pp0, c->st);
    } else {
      {
        TimeScope ts(c, VEM_K_PCG_SPMV, bytes_cheb(c));
        launch_pcg_spmv(c, (const double *)pprev, pnew);
      }
      TimeScope ts(c, VEM_K_PCG_VEC, bytes_pcg_vec(c));
      k_pcg_vec<<<grid_stream(c, c->np), NT, 0, c->stream>>>(c->np, c->dSepsinv, pnew, c->pq, c->px, c->pr,
                                                             c->part, c->counter, c->st);
    }
  }
  CKL();
  return 0;
}

// persistent cooperative form of the block PCG (k_pcg_persistent) for small systems
template <int NB>
struct PcgPersistK {
  static void run(void **f) { *f = (void *)k_pcg_persistent<NB>; }
};
constexpr long PCG_PERSIST_MAX_NP = 262144;
int ensure_part(Ctx *c, long need);

int run_pcg_persistent(Ctx *c, int64_t *inner_its) {
  void *fn = nullptr;
  dispatch_nb<PcgPersistK>(c->nb, &fn);
  if (!fn) return fail(c, VEM_ERR_PRECOND, "no persistent PCG for n_p_dof = %d", c->nb);
  if (!c->pfinal) DA(c->pfinal, 1);
  if (!c->pcg_coop_grid) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, 0));
    if (per_sm < 1) return fail(c, VEM_ERR_CUDA, "persistent PCG does not fit on an SM");
    c->pcg_coop_grid = (int)std::min<long>((long)per_sm * c->sm_count, (c->np + NT - 1) / NT);
    int rr = ensure_part(c, 4L * c->pcg_coop_grid + 64);
    if (rr) return rr;
  }
  long np = c->np;
  Sell S = sellS(c);
  const double *wd = c->wdiag;
  double eps = c->eps;
  const double *inv = c->dBeinv;
  double *x = c->px, *r = c->pr, *z = c->pz, *p0 = c->pp0, *p1 = c->pp1, *q = c->pq, *part = c->part;
  DevState *st = c->st;
  double **pf = c->pfinal;
  void *args[] = {&np, &S, &wd, &eps, &inv, &x, &r, &z, &p0, &p1, &q, &part, &st, &pf};
  {
    TimeScope ts(c, VEM_K_PCG_SPMV);
    CK(cudaLaunchCooperativeKernel(fn, dim3(c->pcg_coop_grid), dim3(NT), args, 0, c->stream));
  }
  CK(cudaMemcpyAsync(&c->hst->p, &c->st->p, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  flush_timing(c);
  if (inner_its) *inner_its += c->hst->p.its;
  if (c->hst->p.failed) return fail(c, VEM_ERR_INNER, "inner PCG did not reach %g in %d steps", c->opts.inner_rtol,
                                    c->opts.inner_maxit);
  return 0;
}

// Inner PCG: chunks of pcg_chunk (even) steps, graph-replayed, host polls the
// device state between chunks.
int run_pcg(Ctx *c, int64_t *inner_its) {
  if (c->nb > 1 && c->pcg_persist && c->np <= PCG_PERSIST_MAX_NP && !c->capturing)
    return run_pcg_persistent(c, inner_its);
  int chunk = std::max(2, c->opts.pcg_chunk);
  if (chunk % 2) ++chunk;
  const bool graphs = c->opts.use_graphs && c->opts.timing != 1;
  if (graphs && (!c->pcg_exec || c->pcg_exec_chunk != chunk)) {
    if (c->pcg_exec) cudaGraphExecDestroy(c->pcg_exec);
    c->pcg_exec = nullptr;
    cudaGraph_t g;
    c->capturing = true;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue_pcg_steps(c, chunk);
    cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    c->capturing = false;
    if (rc) return rc;
    if (e != cudaSuccess) return fail(c, VEM_ERR_CUDA, "PCG capture failed: %s", cudaGetErrorString(e));
    CK(cudaGraphInstantiate(&c->pcg_exec, g, 0));
    cudaGraphDestroy(g);
    c->pcg_exec_chunk = chunk;
  }
  for (;;) {
    if (graphs) {
      CK(cudaGraphLaunch(c->pcg_exec, c->stream));
    } else {
      int rc = enqueue_pcg_steps(c, chunk);
      if (rc) return rc;
    }
    CK(cudaMemcpyAsync(&c->hst->p, &c->st->p, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    flush_timing(c);
    if (!c->hst->p.active) break;
  }
  if (inner_its) *inner_its += c->hst->p.its;
  if (c->hst->p.failed) return fail(c, VEM_ERR_INNER, "inner PCG did not reach %g in %d steps", c->opts.inner_rtol,
                                    c->opts.inner_maxit);
  return 0;
}

// ----------------------------------------------------------------------------
// Block-Schur-AMG apply (kind 3): z_u = s v_u ./ diag(M), z_p = -V(s v_p)
// (oracle/amg.py AMG.vcycle, reading R22)
// ----------------------------------------------------------------------------
constexpr double AMG_THETA = 0.08, AMG_THETA_COARSE = 0.04, AMG_RATIO = 30.0, AMG_STAGNATION = 0.75;
constexpr int AMG_SA_LEVELS = 1;   // levels with the smoothed prolongator (oracle/amg.py SA_LEVELS)
constexpr int AMG_COARSE_SIZE = 2048, AMG_MAX_LEVELS = 12, AMG_DEGREE = 3, AMG_COARSE_DEGREE = 32;
// p-multigrid smoother of the inner V-cycle at n_p_dof > 1 (oracle/amg.py P_DEGREE, P_RATIO; R23)
constexpr int MG_P_DEGREE = 2;
constexpr double MG_P_RATIO = 6.0;
constexpr int MG_COARSE_DEGREE = 8;   // non-dense coarsest level of the S_eps hierarchy (P_COARSE_DEGREE)

void amg_cheb_coeffs(double lmax, int degree, double &inv_theta, std::vector<double> &c1, std::vector<double> &c2,
                     double ratio = AMG_RATIO) {
  const double b = lmax, a = lmax / ratio;
  const double theta = 0.5 * (b + a), delta = 0.5 * (b - a), sigma = theta / delta;
  double rho = 1.0 / sigma;
  inv_theta = 1.0 / theta;
  c1.clear();
  c2.clear();
  for (int i = 1; i < degree; ++i) {
    const double rn = 1.0 / (2.0 * sigma - rho);
    c1.push_back(rn * rho);
    c2.push_back(2.0 * rn / delta);
    rho = rn;
  }
}

// launch on the library stream, with programmatic dependent launch when c->pdl (the kernel
// must start with pdl_enter())
template <typename... KArgs, typename... Args>
void launch_pdl(Ctx *c, void (*k)(KArgs...), unsigned grid, unsigned block, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  // no programmatic edge right after an event node, nor under per-launch event timing
  cfg.numAttrs = c->pdl && !c->pdl_skip && c->opts.timing != 1 ? 1 : 0;
  c->pdl_skip = false;
  cudaLaunchKernelEx(&cfg, k, ((KArgs)args)...);
}

// the same launch without the PDL attribute: every V-cycle kernel but the coarse CSR ones (r13 A/B:
// PDL on every V-cycle kernel 151.2 / 151.2 ms vs 149.7 / 149.7 ms without)
template <typename... KArgs, typename... Args>
void launch_plain(Ctx *c, void (*k)(KArgs...), unsigned grid, unsigned block, Args... args) {
  k<<<grid, block, 0, c->stream>>>(((KArgs)args)...);
}

// CSR level kernels with L.group lanes per row
#define VC_GROUP_LAUNCH(KERNEL, L_, ...)                                                              \
  switch ((L_).group) {                                                                               \
    case 4: launch_pdl(c, KERNEL<T, 4>, grid_for((L_).n * 4), NT, __VA_ARGS__); break;                \
    case 8: launch_pdl(c, KERNEL<T, 8>, grid_for((L_).n * 8), NT, __VA_ARGS__); break;                \
    case 16: launch_pdl(c, KERNEL<T, 16>, grid_for((L_).n * 16), NT, __VA_ARGS__); break;             \
    default: launch_pdl(c, KERNEL<T, 32>, grid_for((L_).n * 32), NT, __VA_ARGS__); break;             \
  }

// out = C_degree(b) on level L (x0 = 0), in precision T; `sample`: bracket the second
// step with the sampled-timing events (fine-level pre-smoothing, timing = 2)
template <typename T>
void amg_smooth(Ctx *c, AmgLevel &L, const T *b, T *out, int degree, const int *gate, bool sample = false,
                int acc = 0) {
  const Lv<T> D{L};
  const double vb = sizeof(T) + 4.0;   // bytes per stored entry (value + index)
  double it;
  std::vector<double> c1, c2;
  amg_cheb_coeffs(L.lmax, degree, it, c1, c2);
  const SellT<T> A{L.soff, L.sci, D.sva()};
  T *dold = D.sd0(), *dnew = D.sd1();
  int first = 1;
  if (degree > 1) {   // init fused into the first step
    // degree 2: this launch is the whole smoother, so it is the one the sampled timing brackets
    const bool smp0 = sample && degree == 2 && c->opts.timing == 2 && c->sample_slot >= 0 && !L.warp_rows;
    if (smp0) cudaEventRecordWithFlags(c->samp_a[c->sample_slot], c->stream, cudaEventRecordExternal);
    c->sample_recorded |= smp0;
    struct SampleEnd {
      Ctx *c;
      bool on;
      ~SampleEnd() {
        if (on) cudaEventRecordWithFlags(c->samp_b[c->sample_slot], c->stream, cudaEventRecordExternal);
      }
    } sample_end{c, smp0};
    TimeScope ts(c, VEM_K_CHEB, vb * L.nnz + 6.0 * sizeof(T) * L.n);
    if (L.warp_rows)
      VC_GROUP_LAUNCH(k_vc_cheb_first_w, L, L.n, L.rp, L.ci, D.va(), D.dinv(), b, (T)it, (T)c1[0], (T)c2[0],
                      D.sr(), D.sd1(), out, acc, gate)
    else
      launch_plain(c, k_vc_cheb_first<T>, grid_for(L.n), NT, L.n, A, D.dinv(), b, (T)it, (T)c1[0], (T)c2[0],
                                                               D.sr(), D.sd1(), out, acc, gate);
    dold = D.sd1();
    dnew = D.sd0();
    first = 2;
  } else {
    TimeScope ts(c, VEM_K_PRECOND_VEC, 5.0 * sizeof(T) * L.n);
    launch_plain(c, k_vc_cheb_init<T>, grid_stream(c, L.n), NT, L.n, D.dinv(), b, (T)it, D.sr(), D.sd0(), out,
                                                                  acc, gate);
  }
  for (int i = first; i < degree; ++i) {
    const bool smp = sample && i == 2 && c->opts.timing == 2 && c->sample_slot >= 0 && !L.warp_rows;
    if (smp) cudaEventRecordWithFlags(c->samp_a[c->sample_slot], c->stream, cudaEventRecordExternal);
    c->sample_recorded |= smp;
    {
      TimeScope ts(c, VEM_K_CHEB, vb * L.nnz + 7.0 * sizeof(T) * L.n);
      if (L.warp_rows)
        VC_GROUP_LAUNCH(k_vc_cheb_step_w, L, L.n, L.rp, L.ci, D.va(), D.dinv(), D.sr(), dold, dnew, out,
                        (T)c1[i - 1], (T)c2[i - 1], gate)
      else
        launch_plain(c, k_vc_cheb_step<T>, grid_for(L.n), NT, L.n, A, D.dinv(), D.sr(), dold, dnew, out,
                                                               (T)c1[i - 1], (T)c2[i - 1], gate);
    }
    if (smp) cudaEventRecordWithFlags(c->samp_b[c->sample_slot], c->stream, cudaEventRecordExternal);
    std::swap(dold, dnew);
  }
}

// t = b - A x on level L
template <typename T>
void amg_residual(Ctx *c, AmgLevel &L, const int *gate) {
  const Lv<T> D{L};
  TimeScope ts(c, VEM_K_SPMV, (sizeof(T) + 4.0) * L.nnz + 3.0 * sizeof(T) * L.n);
  if (L.warp_rows)
    VC_GROUP_LAUNCH(k_vc_resid_w, L, L.n, L.rp, L.ci, D.va(), D.x(), D.b(), D.t(), gate)
  else
    launch_plain(c, k_vc_resid<T>, grid_for(L.n), NT, L.n, SellT<T>{L.soff, L.sci, D.sva()}, D.x(), D.b(), D.t(),
                                                        gate);
}

template <typename T>
const T *amg_cinv(const AmgHier &H);
template <>
const double *amg_cinv<double>(const AmgHier &H) { return H.cinv; }
template <>
const float *amg_cinv<float>(const AmgHier &H) { return H.cinv_f; }

// coarsest-level Chebyshev(d) from x0 = 0 as one 16-CTA cluster launch (k_vc_coarse_cluster)
template <typename T>
void amg_coarse_cluster(Ctx *c, AmgLevel &L, const int *gate) {
  const Lv<T> D{L};
  double it;
  std::vector<double> c1, c2;
  amg_cheb_coeffs(L.lmax, c->amg_coarse_degree, it, c1, c2);
  VcCheb cf{};
  cf.inv_theta = it;
  cf.degree = c->amg_coarse_degree;
  for (size_t i = 0; i < c1.size(); ++i) {
    cf.c1[i] = c1[i];
    cf.c2[i] = c2[i];
  }
  const VcCluster<T> P{L.vc_rs, L.rp, L.vc_c16, D.va(), D.dinv(), D.b(), D.x(), D.sd0(), D.sd1(), (int)L.n};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(VC_CLUSTER);
  cfg.blockDim = dim3(VC_CLUSTER_THREADS);
  cfg.dynamicSmemBytes = sizeof(T) == 8 ? L.vc_smem_d : L.vc_smem_f;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = VC_CLUSTER;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // bytes that move from memory: the level's CSR (16-bit columns) and the b, D^-1, x vectors once
  TimeScope ts(c, VEM_K_CHEB, (sizeof(T) + 2.0) * L.nnz + 4.0 * L.n + 3.0 * sizeof(T) * L.n);
  cudaLaunchKernelEx(&cfg, k_vc_coarse_cluster<T>, P, cf, gate);
}

template <typename T>
void amg_vcycle(Ctx *c, AmgHier &H, size_t l, const int *gate) {
  AmgLevel &L = H.lv[l];
  const Lv<T> D{L};
  if (l + 1 == H.lv.size()) {   // coarsest
    if (H.dense) {
      TimeScope ts(c, VEM_K_PRECOND_VEC, (double)sizeof(T) * L.n * L.n);
      launch_plain(c, k_vc_dense_mv<T>, grid_for(L.n * 32), NT, L.n, amg_cinv<T>(H), D.b(), D.x(), gate);
    } else if (L.vc_ok) {
      amg_coarse_cluster<T>(c, L, gate);
    } else {
      amg_smooth<T>(c, L, D.b(), D.x(), H.coarse_degree, gate);
    }
    return;
  }
  AmgLevel &C = H.lv[l + 1];
  const Lv<T> DC{C};
  amg_smooth<T>(c, L, D.b(), D.x(), AMG_DEGREE, gate, l == 0 && &H == &c->amg);
  amg_residual<T>(c, L, gate);
  if (L.sa) {
    TimeScope ts(c, VEM_K_PRECOND_VEC, (sizeof(T) + 4.0) * L.pnnz + sizeof(T) * (1.0 * L.n + C.n));
    launch_plain(c, k_vc_sa_restrict<T>, grid_for(C.n * 8), NT, C.n, L.ptrp, L.ptci, D.ptva(), D.t(), DC.b(), gate);
  } else {
    TimeScope ts(c, VEM_K_PRECOND_VEC, sizeof(T) * (2.0 * L.n + C.n));
    launch_plain(c, k_vc_restrict<T>, grid_stream(c, C.n), NT, C.n, L.moff, L.mem, D.t(), DC.b(), gate);
  }
  amg_vcycle<T>(c, H, l + 1, gate);
  if (L.sa) {
    TimeScope ts(c, VEM_K_PRECOND_VEC, (sizeof(T) + 4.0) * L.pnnz + sizeof(T) * (2.0 * L.n + C.n));
    launch_plain(c, k_vc_sa_prolong_add<T>, grid_for(L.n), NT, L.n, SellT<T>{L.psoff, L.psci, D.psva()}, DC.x(),
                                                                 D.x(), gate);
  } else {
    TimeScope ts(c, VEM_K_PRECOND_VEC, sizeof(T) * 3.0 * L.n);
    launch_plain(c, k_vc_prolong_add<T>, grid_stream(c, L.n), NT, L.n, L.agg, DC.x(), D.x(), gate);
  }
  amg_residual<T>(c, L, gate);
  amg_smooth<T>(c, L, D.t(), D.x(), AMG_DEGREE, gate, false, 1);   // x += C(b - A x)
}

// Block-Schur-AMG apply in precision T (kind 3: double, kind 4: float V-cycle).
// z_out = false: only the V-cycle runs (x0 = V(s v_p)); k_vc_spmv_z forms z on the fly
template <typename T>
int enqueue_block_schur_amg(Ctx *c, const double *v, const double *scale, double *z, const int *gate,
                            bool z_out = true) {
  if (c->amg.lv.empty())
    return fail(c, VEM_ERR_PRECOND, "Block-Schur-AMG is unavailable: %s",
                c->amg_unavailable.empty() ? "it needs n_p_dof = 1" : c->amg_unavailable.c_str());
  if (sizeof(T) == 4 && !c->amg_f32) return fail(c, VEM_ERR_PRECOND, "FP32 hierarchy not built");
  AmgLevel &L0 = c->amg.lv[0];
  const Lv<T> D0{L0};
  {
    TimeScope ts(c, VEM_K_PRECOND_VEC, z_out ? 24.0 * c->nu + (8.0 + sizeof(T)) * c->np : (8.0 + sizeof(T)) * c->np);
    if (z_out)
      launch_plain(c, k_vc_top<T>, grid_stream(c, c->n), NT, c->nu, c->np, v, scale, c->dMinv, z, D0.b(), gate);
    else   // pressure part only
      launch_plain(c, k_vc_top<T>, grid_stream(c, c->np), NT, 0, c->np, v + c->nu, scale, nullptr, nullptr, D0.b(),
                                                                gate);
  }
  amg_vcycle<T>(c, c->amg, 0, gate);
  if (z_out) {
    TimeScope ts(c, VEM_K_PRECOND_VEC, (8.0 + sizeof(T)) * c->np);
    launch_plain(c, k_vc_out<T>, grid_stream(c, c->np), NT, c->np, D0.x(), z + c->nu, gate);
  }
  CKL();
  return 0;
}

// ----------------------------------------------------------------------------
// MG-PCG: inner PCG on S_eps = S_D + eps W preconditioned by one V-cycle of S_eps
// (reading R23; oracle/amg.py SchurMG, oracle/solver.py pcg)
// ----------------------------------------------------------------------------
inline int grid_part(Ctx *c, long n) {   // fixed grid of the two-stage dot products
  return (int)std::max<long>(1, std::min<long>((n + NT - 1) / NT, (long)c->sm_count * 8));
}
const int *gate_pcg(Ctx *c) { return &c->st->p.active; }
const int *gate_k(Ctx *c) { return &c->st->k.active; }

// mg_z = V(mg_r)
int enqueue_schur_mg(Ctx *c, const int *gate) {
  AmgHier &H = c->amge;
  if (H.lv.empty()) return fail(c, VEM_ERR_PRECOND, "S_eps hierarchy not built (eps <= 0 at upload)");
  if (c->nb == 1) {   // mg_r / mg_z are the level-0 b / x
    amg_vcycle<double>(c, H, 0, gate);
    CKL();
    return 0;
  }
  const long np = c->np, ne = np / c->nb;
  double it;
  std::vector<double> c1, c2;
  amg_cheb_coeffs(2.0, MG_P_DEGREE, it, c1, c2, MG_P_RATIO);   // lambda_max(D_B^-1 S_eps) <= 2 (R15)
  const Sell S = sellS(c);
  const double blk_bytes = 8.0 * np * (4 + c->nb);
  auto smooth = [&](const double *b, int acc) {   // mg_z (+)= C(b), Chebyshev(MG_P_DEGREE)
    {
      TimeScope ts(c, VEM_K_PRECOND_VEC, blk_bytes);
      dispatch_nb<MgBlkL>(c->nb, c, b, (const double *)nullptr, c->cd0, c->mg_z, 0.0, it, 1, acc, gate);
    }
    double *dold = c->cd0, *dnew = c->cd1;
    const double *rb = b;
    for (int i = 1; i < MG_P_DEGREE; ++i) {
      {
        const bool smp = c->opts.timing == 2 && c->capturing && c->mg_samp_a && i == 1 && !acc;
        if (smp) cudaEventRecordWithFlags(c->mg_samp_a, c->stream, cudaEventRecordExternal);
        {
          TimeScope ts(c, VEM_K_MG_FINE, 12.0 * c->nnzS + 32.0 * np);
          k_seps_resid<<<grid_for(np), NT, 0, c->stream>>>(np, S, c->wdiag, c->eps, dold, rb, c->cr, gate);
        }
        if (smp) cudaEventRecordWithFlags(c->mg_samp_b, c->stream, cudaEventRecordExternal);
      }
      rb = c->cr;
      TimeScope ts(c, VEM_K_PRECOND_VEC, blk_bytes + 8.0 * np);
      dispatch_nb<MgBlkL>(c->nb, c, (const double *)c->cr, (const double *)dold, dnew, c->mg_z, c1[i - 1], c2[i - 1],
                          0, 1, gate);
      std::swap(dold, dnew);
    }
  };
  smooth(c->mg_r, 0);
  {
    TimeScope ts(c, VEM_K_MG_FINE, 12.0 * c->nnzS + 32.0 * np);
    k_seps_resid<<<grid_for(np), NT, 0, c->stream>>>(np, S, c->wdiag, c->eps, c->mg_z, c->mg_r, c->cx, gate);
  }
  {
    TimeScope ts(c, VEM_K_PRECOND_VEC, 20.0 * ne);
    k_mg_inject<<<grid_stream(c, ne), NT, 0, c->stream>>>(ne, c->nb, c->perm_p, c->cx, H.lv[0].b, gate);
  }
  amg_vcycle<double>(c, H, 0, gate);
  {
    TimeScope ts(c, VEM_K_PRECOND_VEC, 28.0 * ne);
    k_mg_prolong<<<grid_stream(c, ne), NT, 0, c->stream>>>(ne, c->nb, c->perm_p, H.lv[0].x, c->mg_z, gate);
  }
  {
    TimeScope ts(c, VEM_K_MG_FINE, 12.0 * c->nnzS + 32.0 * np);
    k_seps_resid<<<grid_for(np), NT, 0, c->stream>>>(np, S, c->wdiag, c->eps, c->mg_z, c->mg_r, c->cx, gate);
  }
  smooth(c->cx, 1);
  CKL();
  return 0;
}

int enqueue_pcgm_dir(Ctx *c, int first) {   // z = V(r); beta; p = z + beta p
  int rc = enqueue_schur_mg(c, gate_pcg(c));
  if (rc) return rc;
  const int gp = grid_part(c, c->np);
  TimeScope ts(c, VEM_K_PCG_VEC, 40.0 * c->np);
  k_dot_part<<<gp, NT, 0, c->stream>>>(c->np, c->mg_r, c->mg_z, c->part, gate_pcg(c));
  k_pcgm_beta<<<1, 1024, 0, c->stream>>>(gp, c->part, c->st, first);
  k_pcg_pupd<<<grid_stream(c, c->np), NT, 0, c->stream>>>(c->np, c->mg_z, c->pp0, c->st);
  return 0;
}

int enqueue_pcgm_steps(Ctx *c, int nsteps) {
  const int g = grid_for(c->np), gp = grid_part(c, c->np);
  for (int s = 0; s < nsteps; ++s) {
    {
      TimeScope ts(c, VEM_K_PCG_SPMV, 12.0 * c->nnzS + 32.0 * c->np);
      k_seps_mul<<<g, NT, 0, c->stream>>>(c->np, sellS(c), c->wdiag, c->eps, c->pp0, c->pq, gate_pcg(c));
    }
    {
      TimeScope ts(c, VEM_K_PCG_VEC, 16.0 * c->np);
      k_dot_part<<<gp, NT, 0, c->stream>>>(c->np, c->pp0, c->pq, c->part, gate_pcg(c));
      k_pcg_alpha<<<1, 1024, 0, c->stream>>>(gp, c->part, c->st);
    }
    {
      TimeScope ts(c, VEM_K_PCG_VEC, 48.0 * c->np);
      k_pcgm_xr<<<gp, NT, 0, c->stream>>>(c->np, c->pp0, c->pq, c->px, c->mg_r, c->part, c->st);
      k_pcgm_conv<<<1, 1024, 0, c->stream>>>(gp, c->part, c->st);
    }
    int rc = enqueue_pcgm_dir(c, 0);
    if (rc) return rc;
  }
  CKL();
  return 0;
}

int run_pcg_mg(Ctx *c, double rtol, const int *gate, int64_t *inner_its) {
  const int gp = grid_part(c, c->np);
  {
    TimeScope ts(c, VEM_K_PCG_VEC, 32.0 * c->np);
    k_pcgm_init<<<gp, NT, 0, c->stream>>>(c->np, c->pb, c->px, c->mg_r, c->pp0, c->part, gate);
    k_pcgm_init_fin<<<1, 1024, 0, c->stream>>>(gp, c->part, c->st, rtol, c->opts.inner_maxit, gate);
  }
  int rc = enqueue_pcgm_dir(c, 1);
  if (rc) return rc;
  CKL();
  int chunk = std::max(1, std::min(c->opts.pcg_chunk, c->opts.mg_chunk));
  const bool graphs = c->opts.use_graphs && c->opts.timing != 1 && !c->capturing;
  if (c->opts.timing == 2 && !c->mg_samp_a) {
    CK(cudaEventCreate(&c->mg_samp_a));
    CK(cudaEventCreate(&c->mg_samp_b));
  }
  if (graphs && (!c->pcgm_exec || c->pcgm_exec_chunk != chunk)) {
    if (c->pcgm_exec) cudaGraphExecDestroy(c->pcgm_exec);
    c->pcgm_exec = nullptr;
    cudaGraph_t g;
    c->capturing = true;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    rc = enqueue_pcgm_steps(c, chunk);
    cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    c->capturing = false;
    if (rc) return rc;
    if (e != cudaSuccess) return fail(c, VEM_ERR_CUDA, "MG-PCG capture failed: %s", cudaGetErrorString(e));
    CK(cudaGraphInstantiate(&c->pcgm_exec, g, 0));
    cudaGraphDestroy(g);
    c->pcgm_exec_chunk = chunk;
  }
  int its_prev = 0;
  for (;;) {
    if (graphs) {
      CK(cudaGraphLaunch(c->pcgm_exec, c->stream));
    } else {
      rc = enqueue_pcgm_steps(c, chunk);
      if (rc) return rc;
    }
    CK(cudaMemcpyAsync(&c->hst->p, &c->st->p, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    flush_timing(c);
    if (c->opts.timing == 2 && c->mg_samp_a && c->nb > 1 && (c->hst->p.active || c->hst->p.its - its_prev >= chunk)) {
      float ms = 0.f;   // every V-cycle of the replay ran: its last recorded pair is a live pass
      if (cudaEventElapsedTime(&ms, c->mg_samp_a, c->mg_samp_b) == cudaSuccess) {
        c->stats.launches[VEM_K_MG_FINE] += 1;
        c->stats.ms[VEM_K_MG_FINE] += ms;
        c->stats.bytes[VEM_K_MG_FINE] += 12.0 * c->nnzS + 32.0 * c->np;
      } else {
        (void)cudaGetLastError();
      }
    }
    its_prev = c->hst->p.its;
    if (!c->hst->p.active) break;
  }
  if (inner_its) *inner_its += c->hst->p.its;
  if (c->hst->p.failed) return fail(c, VEM_ERR_INNER, "inner MG-PCG did not reach %g in %d steps", rtol,
                                    c->opts.inner_maxit);
  return 0;
}

// ----------------------------------------------------------------------------
// Block-Reg-M apply (kind 5, reading R24; oracle/solver.py pcg_k): z_p = s v_p / (eps W),
// z_u = PCG on K = M + B^T (eps W)^-1 B from y0 = 0, preconditioned by the kind-2 Woodbury
// block (its inner solve to k_inner_rtol), until sqrt(r.z) <= k_rtol sqrt(r0.z0)
// ----------------------------------------------------------------------------
int enqueue_block_reg_m(Ctx *c, const double *v, const double *scale, double *z, const int *gate,
                        int64_t *inner_its) {
  if (!c->kx) {
    DA(c->kx, c->n);
    DA(c->kr, c->nu);
    DA(c->kz, c->nu);
    DA(c->kq, c->nu);
  }
  const long nu = c->nu, np = c->np;
  const int gu = grid_stream(c, nu), gp = grid_part(c, nu);
  const double inv_eps = 1.0 / c->eps;
  auto woodbury = [&](const int *g2) -> int {   // kz = (diag M + B^T (eps W)^-1 B)^-1 kr
    {
      TimeScope ts(c, VEM_K_PRECOND_VEC, 24.0 * nu);
      k_k_t0<<<gu, NT, 0, c->stream>>>(nu, c->kr, c->dMinv, c->kz, g2);
    }
    {
      TimeScope ts(c, VEM_K_PRECOND_VEC, 12.0 * c->nnzB + 8.0 * c->n);
      launch_spmv(c, nu, np, (const double *)c->kz, c->pb - nu, nullptr, 0, g2);
    }
    CKL();
    int rc = run_inner(c, c->opts.k_inner_rtol, g2, inner_its);
    if (rc) return rc;
    TimeScope ts(c, VEM_K_PRECOND_VEC, 12.0 * (c->nnzM + c->nnzB) + 8.0 * c->n + 16.0 * nu);
    launch_br_finish(c, c->kz, g2);
    return 0;
  };
  {
    TimeScope ts(c, VEM_K_PRECOND_VEC, 8.0 * (4 * nu + 2 * np));
    k_k_init<<<grid_stream(c, c->n), NT, 0, c->stream>>>(nu, np, v, scale, c->wdiag, inv_eps, c->kr, z, c->kx, gate);
  }
  int rc = woodbury(gate);
  if (rc) return rc;
  {
    TimeScope ts(c, VEM_K_PRECOND_VEC, 40.0 * nu);
    k_dot_part<<<gp, NT, 0, c->stream>>>(nu, c->kr, c->kz, c->part, gate);
    k_k_rz<<<1, 1024, 0, c->stream>>>(gp, c->part, c->st, 1, c->opts.k_rtol, c->opts.k_maxit, gate);
    k_k_pupd<<<gu, NT, 0, c->stream>>>(nu, c->kz, c->kx, c->st);
  }
  CKL();
  for (;;) {
    {
      TimeScope ts(c, VEM_K_SPMV, 12.0 * c->nnzA + 16.0 * c->n + 8.0 * nu);
      launch_spmv(c, nu, np, (const double *)c->kx, c->kx, nullptr, 0, gate_k(c));   // kx[nu:] = B p
      const int g = grid_for(nu);
      k_kmul<<<g, NT, 0, c->stream>>>(nu, sellA(c), c->kx, c->wdiag, inv_eps, c->kq, c->part, gate_k(c));
      k_k_alpha<<<1, 1024, 0, c->stream>>>(g, c->part, c->st);
    }
    {
      TimeScope ts(c, VEM_K_PRECOND_VEC, 48.0 * nu);
      k_k_xr<<<gu, NT, 0, c->stream>>>(nu, c->kx, c->kq, z, c->kr, c->st);
    }
    CKL();
    rc = woodbury(gate_k(c));
    if (rc) return rc;
    {
      TimeScope ts(c, VEM_K_PRECOND_VEC, 40.0 * nu);
      k_dot_part<<<gp, NT, 0, c->stream>>>(nu, c->kr, c->kz, c->part, gate_k(c));
      k_k_rz<<<1, 1024, 0, c->stream>>>(gp, c->part, c->st, 0, c->opts.k_rtol, c->opts.k_maxit, gate);
      k_k_pupd<<<gu, NT, 0, c->stream>>>(nu, c->kz, c->kx, c->st);
    }
    CKL();
    CK(cudaMemcpyAsync(&c->hst->k, &c->st->k, sizeof(KState), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    flush_timing(c);
    if (!c->hst->k.active) break;
  }
  c->k_its_total += c->hst->k.its;
  c->k_failed |= c->hst->k.failed != 0;
  if (c->trace_k)
    fprintf(stderr, "[vem kind 5] K-PCG: %d steps%s, sqrt(rz/rz0) = %.3e, inner steps so far %lld\n", c->hst->k.its,
            c->hst->k.failed ? " (cap reached)" : "", sqrt(fabs(c->hst->k.rz) / std::max(c->hst->k.rz0, 1e-300)),
            inner_its ? (long long)*inner_its : 0LL);
  return 0;
}

// FGMRES (Z stored) for the variable preconditioners: Block-Reg (inner PCG) and the
// FP32 V-cycle (its rounding makes P^-1 (V y) differ from sum y_j P^-1 v_j)
inline bool is_flexible(int kind) {
  return kind == VEM_PRECOND_BLOCK_REG || kind == VEM_PRECOND_BLOCK_SCHUR_AMG_F32 || kind == VEM_PRECOND_BLOCK_REG_M;
}
inline bool is_block_reg(int kind) { return kind == VEM_PRECOND_BLOCK_REG || kind == VEM_PRECOND_BLOCK_REG_M; }

int enqueue_precond(Ctx *c, int kind, const double *v, const double *scale, double *z, const int *gate,
                    int64_t *inner_its) {
  if (kind == VEM_PRECOND_BLOCK_SCHUR_AMG) return enqueue_block_schur_amg<double>(c, v, scale, z, gate);
  if (kind == VEM_PRECOND_BLOCK_SCHUR_AMG_F32) return enqueue_block_schur_amg<float>(c, v, scale, z, gate);
  if (kind == VEM_PRECOND_BLOCK_SCHUR) return enqueue_block_schur(c, v, scale, z, gate);
  if (kind == VEM_PRECOND_BLOCK_REG) return enqueue_block_reg(c, v, scale, z, gate, inner_its);
  if (kind == VEM_PRECOND_BLOCK_REG_M) return enqueue_block_reg_m(c, v, scale, z, gate, inner_its);
  // NONE: z = scale * v
  TimeScope ts(c, VEM_K_PRECOND_VEC);
  k_bs_init<<<grid_stream(c, c->n), NT, 0, c->stream>>>(c->n, 0, v, scale, nullptr, nullptr, 0.0, z, nullptr,
                                                        nullptr, nullptr, 0, 0, gate);
  CKL();
  return 0;
}

// ----------------------------------------------------------------------------
// GMRES(m) cycle
// ----------------------------------------------------------------------------
int ensure_part(Ctx *c, long need) {
  if (need <= c->part_cap) return 0;
  if (c->part) dfree(c, c->part);
  c->part = nullptr;
  DA(c->part, need);
  c->part_cap = need;
  return 0;
}

int enqueue_arnoldi_step(Ctx *c, int kind, int j, int64_t *inner_its) {
  const bool flex = is_flexible(kind);
  double *Vj = c->V + (size_t)j * c->ldv;
  double *w = c->V + (size_t)(j + 1) * c->ldv;
  double *zj = flex ? c->Z + (size_t)j * c->ldv : c->z;
  c->sample_slot = j;
  if (kind == VEM_PRECOND_BLOCK_SCHUR_AMG || kind == VEM_PRECOND_BLOCK_SCHUR_AMG_F32) {
    // z = P^-1 v_j formed inside the SpMV gather
    const bool f32 = kind == VEM_PRECOND_BLOCK_SCHUR_AMG_F32;
    int rc = f32 ? enqueue_block_schur_amg<float>(c, Vj, &c->st->vscale[j], nullptr, gate_active(c), false)
                 : enqueue_block_schur_amg<double>(c, Vj, &c->st->vscale[j], nullptr, gate_active(c), false);
    c->sample_slot = -1;
    if (rc) return rc;
    TimeScope ts(c, VEM_K_SPMV, bytes_spmv(c) + 8.0 * c->nu);
    if (f32)   // FGMRES: z_j is also stored (row by row, by the thread that owns the row)
      launch_plain(c, k_vc_spmv_z<float>, grid_for(c->n), NT, c->n, c->nu, sellA(c), Vj, &c->st->vscale[j],
                                                                c->dMinv, c->amg.lv[0].x_f, w, zj, gate_active(c));
    else
      launch_plain(c, k_vc_spmv_z<double>, grid_for(c->n), NT, c->n, c->nu, sellA(c), Vj, &c->st->vscale[j],
                                                                 c->dMinv, c->amg.lv[0].x, w, nullptr, gate_active(c));
  } else {
    int rc = enqueue_precond(c, kind, Vj, &c->st->vscale[j], zj, gate_active(c), inner_its);
    c->sample_slot = -1;
    if (rc) return rc;
    TimeScope ts(c, VEM_K_SPMV, bytes_spmv(c));
    launch_spmv(c, 0L, c->n, (const double *)zj, w, nullptr, 0, gate_active(c));
  }
  const int nv = j + 1;
  const int gx = c->sm_count * 2;
  // reorth: 1 CGS2, 0 CGS1, -1 auto = CGS1 for GMRES, CGS2 for FGMRES/Block-Reg (reading R17)
  const int npass = (c->opts.reorth == 1 || (c->opts.reorth < 0 && is_block_reg(kind))) ? 2 : 1;
  for (int pass = 1; pass <= npass; ++pass) {
    const int nout = nv + (pass == 1 ? 1 : 0);
    const int nchunk = (nout + VEM_DOT_CHUNK - 1) / VEM_DOT_CHUNK;
    // one full wave of resident CTAs over all chunks (a fixed 2 CTAs/SM per chunk leaves the
    // short-basis steps at a quarter of the SM slots and the long ones at 1.75 waves)
    dim3 grid(c->mdot_slots > 0 ? std::max(c->mdot_slots / nchunk, 1) : gx, nchunk);
    if (c->opts.basis_f32) {   // compressed basis: the CGS kernels stream the float copy (N4)
      {
        TimeScope ts(c, VEM_K_DOT, c->n * (4.0 * nv + 8.0));
        dim3 grid32(c->mdot32_slots > 0 ? std::max(c->mdot32_slots / nchunk, 1) : gx, nchunk);
        k_mdot32<<<grid32, NT, 0, c->stream>>>(c->n, c->V32, c->ldv, nv, pass == 1 ? 1 : 0, w, c->part, c->counter,
                                               c->st, pass);
      }
      TimeScope ts(c, VEM_K_UPDATE, c->n * (4.0 * nv + 16.0 + (pass == npass ? 4.0 : 0.0)));
      k_update32<<<c->update32_slots > 0 ? c->update32_slots : gx * 2, NT, 0, c->stream>>>(
          c->n, c->V32, c->ldv, nv, w, c->V32 + (size_t)(j + 1) * c->ldv, pass == npass ? 1 : 0, c->part, c->counter,
          c->st, j);
      continue;
    }
    {
      TimeScope ts(c, VEM_K_DOT, bytes_vecs(c, nv + 1));
      k_mdot<<<grid, NT, 0, c->stream>>>(c->n, c->V, c->ldv, nv, pass == 1 ? 1 : 0, w, c->part, c->counter, c->st,
                                         pass);
    }
    {
      TimeScope ts(c, VEM_K_UPDATE, bytes_vecs(c, nv + 2));
      k_update<<<c->update_slots > 0 ? c->update_slots : gx * 2, NT, 0, c->stream>>>(c->n, c->V, c->ldv, nv, w, pass == npass ? 1 : 0, c->part,
                                             c->counter, c->st, j);
    }
  }
  CKL();
  return 0;
}

int enqueue_cycle_end(Ctx *c, int kind, int64_t *inner_its) {
  const bool flex = is_flexible(kind);
  {
    TimeScope ts(c, VEM_K_CYCLE);
    k_backsolve<<<1, 32, 0, c->stream>>>(c->st, flex ? 0 : 1);
  }
  if (flex) {
    TimeScope ts(c, VEM_K_CYCLE);
    k_combine<<<grid_stream(c, c->n), NT, 0, c->stream>>>(c->n, c->Z, c->ldv, c->x, 1, c->st);
  } else {
    {
      TimeScope ts(c, VEM_K_CYCLE);
      k_combine<<<grid_stream(c, c->n), NT, 0, c->stream>>>(c->n, c->V, c->ldv, c->t, 0, c->st);
    }
    int rc = enqueue_precond(c, kind, c->t, &c->st->one, c->z, gate_steps(c), inner_its);
    if (rc) return rc;
    TimeScope ts(c, VEM_K_CYCLE);
    k_axpy_gated<<<grid_stream(c, c->n), NT, 0, c->stream>>>(c->n, c->z, c->x, gate_steps(c));
  }
  {
    TimeScope ts(c, VEM_K_SPMV, bytes_spmv(c) + 8.0 * c->n);
    launch_residual(c, c->x, c->b, c->V, 1);
  }
  if (c->opts.basis_f32) k_round_basis<<<grid_stream(c, c->n), NT, 0, c->stream>>>(c->n, c->V, c->V32);
  CKL();
  return 0;
}

int enqueue_cycle(Ctx *c, int kind, int64_t *inner_its) {
  for (int j = 0; j < c->opts.restart; ++j) {
    int rc = enqueue_arnoldi_step(c, kind, j, inner_its);
    if (rc) return rc;
  }
  return enqueue_cycle_end(c, kind, inner_its);
}

void destroy_graphs(Ctx *c) {
  for (auto &g : c->cycle_exec)
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
  if (c->pcg_exec) cudaGraphExecDestroy(c->pcg_exec);
  c->pcg_exec = nullptr;
  if (c->pcgm_exec) cudaGraphExecDestroy(c->pcgm_exec);
  c->pcgm_exec = nullptr;
}

int ensure_work(Ctx *c, int kind) {
  const int m = c->opts.restart;
  if (!c->V) {
    DA(c->V, (size_t)(m + 1) * c->ldv);
    CK(cudaMemsetAsync(c->V, 0, (size_t)(m + 1) * c->ldv * sizeof(double), c->stream));
  }
  if (c->opts.basis_f32 && !c->V32) {
    DA(c->V32, (size_t)(m + 1) * c->ldv);
    CK(cudaMemsetAsync(c->V32, 0, (size_t)(m + 1) * c->ldv * sizeof(float), c->stream));
  }
  if (is_flexible(kind) && c->zcap < m) {
    if (c->Z) dfree(c, c->Z);
    c->Z = nullptr;
    DA(c->Z, (size_t)m * c->ldv);
    c->zcap = m;
  }
  return ensure_part(c, (long)c->sm_count * 2 * ((m + 2 + VEM_DOT_CHUNK - 1) / VEM_DOT_CHUNK + 1) * VEM_DOT_CHUNK +
                            (long)(c->mdot_slots + c->sm_count * ((m + 2 + VEM_DOT_CHUNK - 1) / VEM_DOT_CHUNK)) *
                                VEM_DOT_CHUNK +
                            (long)c->sm_count * 64 * 2 + grid_for(c->n * 32) + 1024);
}

int apply_l2_window(Ctx *c, int which = 0);

// caller numbering <-> internal (SELL-C-sigma reordered) numbering of [u; p]
void to_internal(Ctx *c, const double *in, double *out) {
  if (c->perm)
    k_gather_rows<<<grid_stream(c, c->n), NT, 0, c->stream>>>(c->n, 1, c->perm, in, out);
  else
    cudaMemcpyAsync(out, in, c->n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream);
}
void from_internal(Ctx *c, const double *in, double *out_u, double *out_p) {
  if (c->perm) {
    k_scatter_split<<<grid_stream(c, c->n), NT, 0, c->stream>>>(c->n, c->nu, c->perm, in, out_u, out_p);
  } else {
    cudaMemcpyAsync(out_u, in, c->nu * sizeof(double), cudaMemcpyDeviceToDevice, c->stream);
    cudaMemcpyAsync(out_p, in + c->nu, c->np * sizeof(double), cudaMemcpyDeviceToDevice, c->stream);
  }
}

int solve_impl(Ctx *c, const double *rhs, double tol, int maxit, int kind, double *out_u, double *out_p,
               vem_solve_report *rep) {
  vem_solve_report R{};
  if (kind < 0 || kind > 5) return fail(c, VEM_ERR_PRECOND, "unsupported precond_kind %d", kind);
  if (is_block_reg(kind) && !c->has_reg)
    return fail(c, VEM_ERR_PRECOND, "Block-Reg needs eps > 0 at upload");
  c->k_its_total = 0;
  c->k_failed = false;
  if (!rhs || !out_u || !out_p || maxit < 0 || !(tol > 0)) return fail(c, VEM_ERR_INVALID, "invalid solve arguments");
  int rc = ensure_work(c, kind);
  if (rc) return rc;
  {  // the L2-persisting window covers the fine-level pool of the precision this kind runs in
    const int pool = kind == VEM_PRECOND_BLOCK_SCHUR_AMG_F32 ? 1 : 0;
    if (c->opts.l2_persist && c->l2_window_pool != pool) {
      rc = apply_l2_window(c, pool);
      if (rc) return rc;
    }
  }
  struct EvPair {   // destroyed on every exit path
    cudaEvent_t a = nullptr, b = nullptr;
    ~EvPair() {
      if (a) cudaEventDestroy(a);
      if (b) cudaEventDestroy(b);
    }
  } ev;
  CK(cudaEventCreate(&ev.a));
  CK(cudaEventCreate(&ev.b));
  cudaEvent_t e0 = ev.a, e1 = ev.b;
  CK(cudaEventRecord(e0, c->stream));
  to_internal(c, rhs, c->b);
  CK(cudaMemsetAsync(c->x, 0, c->n * sizeof(double), c->stream));
  // reset GMRES state
  GmresState g0{};
  g0.m = c->opts.restart;
  g0.maxit = maxit;
  g0.tol_abs = 0.0;
  g0.flexible = is_flexible(kind);
  CK(cudaMemcpyAsync(&c->hst->g, &g0, sizeof(g0), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(&c->st->g, &c->hst->g, sizeof(g0), cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  // beta0 = ||b||; V0 = b
  launch_residual(c, nullptr, c->b, c->V, 0);
  if (c->opts.basis_f32) k_round_basis<<<grid_stream(c, c->n), NT, 0, c->stream>>>(c->n, c->V, c->V32);
  CKL();
  CK(cudaMemcpyAsync(&c->hst->g, &c->st->g, sizeof(GmresState), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const double bnorm = c->hst->g.bnorm;
  int status = VEM_OK;
  int64_t inner = 0;
  if (bnorm > 0.0) {
    // tol_abs = tol * ||b||; re-run the start so conv/active use it
    GmresState gs = c->hst->g;
    gs.tol_abs = tol * bnorm;
    gs.active = (gs.its >= gs.maxit) ? 0 : 1;
    gs.conv_true = 0;
    CK(cudaMemcpyAsync(&c->st->g, &gs, sizeof(gs), cudaMemcpyHostToDevice, c->stream));
    const bool graphs = c->opts.use_graphs && c->opts.timing != 1 && !is_block_reg(kind);
    if (c->opts.timing == 2) {
      int rs = ensure_samples(c);
      if (rs) return rs;
    }
    // a replayed graph records its samples only if its capture did (kind 1, k = 0)
    c->sample_recorded = c->cycle_exec[kind] ? c->sample_recorded_kind[kind] : false;
    int restarts = 0, cycles = 0;
    int its_before = c->hst->g.its;
    while (c->hst->g.its < maxit || cycles == 0) {
      if (maxit == 0) break;
      c->hist_beta = c->hst->g.beta;   // residual norm this cycle starts from (vem_mixed_last_cycle_history)
      c->hist_bnorm = bnorm;
      if (graphs) {
        if (!c->cycle_exec[kind]) {
          cudaGraph_t gr;
          c->capturing = true;
          CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
          int r2 = enqueue_cycle(c, kind, &inner);
          cudaError_t e = cudaStreamEndCapture(c->stream, &gr);
          c->capturing = false;
          if (r2) return r2;
          if (e != cudaSuccess) return fail(c, VEM_ERR_CUDA, "cycle capture failed: %s", cudaGetErrorString(e));
          CK(cudaGraphInstantiate(&c->cycle_exec[kind], gr, 0));
          cudaGraphDestroy(gr);
          c->sample_recorded_kind[kind] = c->sample_recorded;
        }
        CK(cudaGraphLaunch(c->cycle_exec[kind], c->stream));
      } else {
        int r2 = enqueue_cycle(c, kind, &inner);
        if (r2) {
          status = r2;
          break;
        }
      }
      ++cycles;
      CK(cudaMemcpyAsync(&c->hst->g, &c->st->g, sizeof(GmresState), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      flush_timing(c);
      // the sampled launch: k_cheb_step (kind 1) or, with the degree-2 V-cycle smoother, the
      // fine-level k_vc_cheb_first (kinds 3, 4: one vector less than a later step)
      collect_samples(c, c->hst->g.its - its_before,
                      (kind == VEM_PRECOND_BLOCK_SCHUR_AMG && AMG_DEGREE == 2) ? bytes_cheb(c) - 8.0 * c->np
                                                                               : bytes_cheb(c));   // g.j was reset by the restart
      c->hist_steps = c->hst->g.its - its_before;
      its_before = c->hst->g.its;
      const GmresState &h = c->hst->g;
      if (h.conv_true) break;
      if (h.its >= maxit) {
        status = VEM_NOT_CONVERGED;
        break;
      }
      if (h.breakdown && h.j == 1) {
        status = VEM_BREAKDOWN;
        break;
      }
      ++restarts;
    }
    if (status == VEM_OK && !c->hst->g.conv_true) status = VEM_NOT_CONVERGED;
    R.restarts = restarts;
    R.cycles = cycles;
  }
  from_internal(c, c->x, out_u, out_p);
  CK(cudaEventRecord(e1, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  flush_timing(c);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const GmresState &h = c->hst->g;
  R.status = status;
  R.iterations = h.its;
  R.converged = bnorm == 0.0 ? 1 : h.conv_true;
  R.breakdown = h.breakdown;
  R.inner_iterations = inner;
  R.k_iterations = c->k_its_total;
  R.rel_residual_true = bnorm > 0 ? h.true_res / bnorm : 0.0;
  R.rel_residual_est = bnorm > 0 ? h.est / bnorm : 0.0;
  R.setup_ms = c->setup_ms;
  R.solve_ms = ms;
  if (rep) *rep = R;
  return status;
}

// ----------------------------------------------------------------------------
// upload
// ----------------------------------------------------------------------------
int check_csr(Ctx *c, const vem_csr *A, long nr, long nc, const char *name) {
  if (!A || !A->indptr || (A->nnz && (!A->indices || !A->values)))
    return fail(c, VEM_ERR_INVALID, "%s: NULL pointer", name);
  if (A->n_rows != nr || A->n_cols != nc)
    return fail(c, VEM_ERR_INVALID, "%s: shape %lld x %lld, expected %ld x %ld", name, (long long)A->n_rows,
                (long long)A->n_cols, nr, nc);
  if (A->indptr[0] != 0 || A->indptr[nr] != A->nnz) return fail(c, VEM_ERR_INVALID, "%s: bad indptr ends", name);
  for (long r = 0; r < nr; ++r) {
    const int64_t s = A->indptr[r], e = A->indptr[r + 1];
    if (e < s) return fail(c, VEM_ERR_INVALID, "%s: indptr decreasing at row %ld", name, r);
    for (int64_t k = s; k < e; ++k) {
      const int32_t j = A->indices[k];
      if (j < 0 || j >= nc) return fail(c, VEM_ERR_INVALID, "%s: column %d out of range in row %ld", name, j, r);
      if (k > s && A->indices[k - 1] >= j) return fail(c, VEM_ERR_INVALID, "%s: row %ld not sorted/unique", name, r);
    }
  }
  return 0;
}

template <typename T>
int upload_array(Ctx *c, T **dst, const T *src, size_t n) {
  int r = dalloc(c, dst, n);
  if (r) return r;
  if (n) CK(cudaMemcpyAsync(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  return 0;
}

int build_schur(Ctx *c, const int64_t *brp, const int *bci, const double *bva, const int *btrp, const int *btci,
                const double *btva) {
  // per-row expansion counts, processed in row chunks bounding the expansion buffer
  const long np = c->np;
  int64_t *cnt = nullptr;
  DA(cnt, np + 1);
  k_spgemm_count<<<grid_stream(c, np), NT, 0, c->stream>>>(0, np, brp, bci, btrp, cnt);
  CKL();
  std::vector<int64_t> hcnt(np);
  CK(cudaMemcpyAsync(hcnt.data(), cnt, np * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const int64_t cap = (int64_t)1 << 27;
  std::vector<std::pair<long, long>> chunks;
  {
    long r0 = 0;
    int64_t acc = 0;
    for (long r = 0; r < np; ++r) {
      if (acc + hcnt[r] > cap && r > r0) {
        chunks.push_back({r0, r});
        r0 = r;
        acc = 0;
      }
      acc += hcnt[r];
    }
    chunks.push_back({r0, np});
  }
  std::vector<int> hu(np);
  std::vector<int *> cci;
  std::vector<double *> cva;
  std::vector<long> cnnz;
  int *ucnt = nullptr, *urp = nullptr;
  DA(ucnt, np + 1);
  DA(urp, np + 1);
  int64_t *off = nullptr;
  DA(off, np + 1);
  int rcode = 0;
  for (auto &ch : chunks) {
    const long r0 = ch.first, nr = ch.second - ch.first;
    int64_t tot = 0;
    std::vector<int64_t> hoff(nr + 1);
    for (long t = 0; t < nr; ++t) {
      hoff[t] = tot;
      tot += hcnt[r0 + t];
    }
    hoff[nr] = tot;
    if (tot >= ((int64_t)1 << 31)) return fail(c, VEM_ERR_INVALID, "S_D expansion row chunk too large");
    CK(cudaMemcpyAsync(off, hoff.data(), (nr + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    int *k0 = nullptr, *k1 = nullptr;
    double *v0 = nullptr, *v1 = nullptr;
    DA(k0, tot);
    DA(k1, tot);
    DA(v0, tot);
    DA(v1, tot);
    k_spgemm_expand<<<grid_stream(c, nr), NT, 0, c->stream>>>(r0, nr, brp, bci, bva, c->dMinv, btrp, btci, btva, off,
                                                              k0, v0);
    CKL();
    size_t tb = 0;
    if (tot >= (1LL << 31)) return fail(c, VEM_ERR_INVALID, "S_D expansion chunk exceeds 2^31 entries");
    CK(cub::DeviceSegmentedSort::StableSortPairs(nullptr, tb, k0, k1, v0, v1, (int)tot, (int)nr, off, off + 1,
                                                 c->stream));
    char *tmp = nullptr;
    DA(tmp, tb);
    CK(cub::DeviceSegmentedSort::StableSortPairs(tmp, tb, k0, k1, v0, v1, (int)tot, (int)nr, off, off + 1,
                                                 c->stream));
    k_spgemm_unique<<<grid_stream(c, nr), NT, 0, c->stream>>>(nr, off, k1, ucnt);
    CKL();
    CK(cudaMemcpyAsync(hu.data() + r0, ucnt, nr * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    std::vector<int> hurp(nr + 1);
    long u = 0;
    for (long t = 0; t < nr; ++t) {
      hurp[t] = (int)u;
      u += hu[r0 + t];
    }
    hurp[nr] = (int)u;
    CK(cudaMemcpyAsync(urp, hurp.data(), (nr + 1) * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    int *sci = nullptr;
    double *sva = nullptr;
    DA(sci, u);
    DA(sva, u);
    k_spgemm_compact<<<grid_stream(c, nr), NT, 0, c->stream>>>(nr, off, k1, v1, urp, sci, sva);
    CKL();
    CK(cudaStreamSynchronize(c->stream));
    dfree(c, tmp);
    dfree(c, k0);
    dfree(c, k1);
    dfree(c, v0);
    dfree(c, v1);
    cci.push_back(sci);
    cva.push_back(sva);
    cnnz.push_back(u);
  }
  long nnzS = 0;
  for (long u : cnnz) nnzS += u;
  if (nnzS >= (1L << 31)) return fail(c, VEM_ERR_INVALID, "nnz(S_D) exceeds int32");
  c->nnzS = nnzS;
  std::vector<int> hrp(np + 1);
  long acc = 0;
  for (long r = 0; r < np; ++r) {
    hrp[r] = (int)acc;
    acc += hu[r];
  }
  hrp[np] = (int)acc;
  DA(c->s_rp, np + 1);
  DA(c->s_ci, nnzS);
  DA(c->s_va, nnzS);
  CK(cudaMemcpyAsync(c->s_rp, hrp.data(), (np + 1) * sizeof(int), cudaMemcpyHostToDevice, c->stream));
  long o = 0;
  for (size_t q = 0; q < cci.size(); ++q) {
    CK(cudaMemcpyAsync(c->s_ci + o, cci[q], cnnz[q] * sizeof(int), cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->s_va + o, cva[q], cnnz[q] * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    o += cnnz[q];
  }
  CK(cudaStreamSynchronize(c->stream));
  for (size_t q = 0; q < cci.size(); ++q) {
    dfree(c, cci[q]);
    dfree(c, cva[q]);
  }
  dfree(c, cnt);
  dfree(c, ucnt);
  dfree(c, urp);
  dfree(c, off);
  return rcode;
}

// Keep the Chebyshev vectors (5 x n_p doubles: 84 MB on C3) resident in the
// 126 MB L2 across the d-1 steps of an apply, so each step streams only S_D
// from HBM: a persisting access-policy window on the library stream (captured
// into the graph kernel nodes).  opts.l2_persist = 0 disables it.
// which = 0: the FP64 Chebyshev / AMG fine-level pool; 1: the FP32 pool of kind 4
int apply_l2_window(Ctx *c, int which) {
  cudaStreamAttrValue attr{};
  void *pool = which ? (void *)c->f32_pool : (void *)c->cheb_pool;
  const size_t pool_bytes = which ? c->f32_pool_bytes : c->cheb_pool_bytes;
  if (c->l2_window_pool >= 0 && c->l2_window_pool != which) cudaCtxResetPersistingL2Cache();
  c->l2_window_pool = which;
  if (!c->opts.l2_persist || !pool) {
    attr.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &attr);
    c->l2_window_bytes = 0;
    return 0;
  }
  int dev = 0, maxp = 0, maxw = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev));
  CK(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev));
  if (maxp <= 0 || maxw <= 0) return 0;
  const size_t win = std::min(pool_bytes, (size_t)maxw);
  const size_t setaside = std::min(win, (size_t)maxp);
  CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, setaside));
  attr.accessPolicyWindow.base_ptr = pool;
  attr.accessPolicyWindow.num_bytes = win;
  attr.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)setaside / (double)win);
  attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  CK(cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &attr));
  c->l2_window_bytes = win;
  return 0;
}

int build_sell(Ctx *c, long nrows, const int *rp, const int *ci, const double *va, long long **soff, int **sci,
               double **sva, long *nnz_sell, const int *perm = nullptr, const int *cmap = nullptr) {
  const long nsl = (nrows + 31) / 32;
  long long *w = nullptr;
  DA(w, nsl + 1);
  DA(*soff, nsl + 1);
  k_sell_width<<<grid_stream(c, nsl), NT, 0, c->stream>>>(nrows, rp, perm, w);
  CKL();
  CK(cudaMemsetAsync(w + nsl, 0, sizeof(long long), c->stream));
  size_t tb = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, w, *soff, (int)(nsl + 1), c->stream));
  char *tmp = nullptr;
  DA(tmp, tb);
  CK(cub::DeviceScan::ExclusiveSum(tmp, tb, w, *soff, (int)(nsl + 1), c->stream));
  long long tot = 0;
  CK(cudaMemcpyAsync(&tot, *soff + nsl, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  dfree(c, tmp);
  dfree(c, w);
  DA(*sci, tot);
  DA(*sva, tot);
  k_sell_fill<<<grid_stream(c, nsl * 32), NT, 0, c->stream>>>(nrows, rp, ci, va, perm, cmap, *soff, *sci, *sva);
  CKL();
  *nnz_sell = (long)tot;
  return 0;
}

// ----------------------------------------------------------------------------
// SELL-C-sigma reordering (k >= 1 layouts, no AMG): rows of different lengths
// (face / interior velocity rows, pair / cube elements) share SELL-32 slices and
// pad every slice to its longest row (C5: 1.8x the nonzeros of A, 2.1x of S_D).
// The unknowns are renumbered once at upload by a symmetric permutation that
// sorts velocity rows of A, and elements (all n_p DOFs together, so the
// element-block Jacobi structure is kept), by row length inside windows of
// REORDER_WINDOW rows (stable: equal lengths keep their order, locality of the
// column gathers is kept within a window).  The solve gathers rhs into the new
// order and scatters u, p back; every hot kernel is unchanged.
// ----------------------------------------------------------------------------
constexpr long REORDER_WINDOW = 4096;

long sell_padded(const std::vector<int> &len, const std::vector<int> &perm) {
  long tot = 0;
  const long n = (long)len.size();
  for (long s = 0; s < n; s += 32) {
    int w = 0;
    for (long r = s; r < std::min(n, s + 32); ++r) w = std::max(w, len[perm.empty() ? r : perm[r]]);
    tot += 32L * w;
  }
  return tot;
}

// stable sort of [first, last) of idx by key descending, in windows of `win` entries
void window_sort(std::vector<int> &idx, const std::vector<long long> &key, long win) {
  const long n = (long)idx.size();
  for (long w0 = 0; w0 < n; w0 += win) {
    auto b = idx.begin() + w0, e = idx.begin() + std::min(n, w0 + win);
    std::stable_sort(b, e, [&](int a, int c) { return key[a] > key[c]; });
  }
}

int build_reorder(Ctx *c) {
  if (c->nb <= 1 || c->opts.reorder == 0) return 0;
  const long nu = c->nu, np = c->np, n = c->n, nb = c->nb, ne = np / nb;
  std::vector<int> arp(n + 1), srp(np + 1);
  CK(cudaMemcpyAsync(arp.data(), c->a_rp, (n + 1) * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(srp.data(), c->s_rp, (np + 1) * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  std::vector<int> alen(n), slen(np);
  for (long i = 0; i < n; ++i) alen[i] = arp[i + 1] - arp[i];
  for (long i = 0; i < np; ++i) slen[i] = srp[i + 1] - srp[i];
  // velocity rows: element-major order (first element touching the row; counting sort,
  // stable), so a row's gathers of x stay near its own index, then sorted by A row
  // length inside the windows
  std::vector<int> pu(nu);
  std::vector<long long> ku(nu);
  const bool elem_major = !getenv("VEM_REORDER_ELEM") || atoi(getenv("VEM_REORDER_ELEM")) != 0;
  if (elem_major) {
    int *de = nullptr;
    DA(de, nu);
    k_first_elem<<<grid_stream(c, nu), NT, 0, c->stream>>>(nu, c->a_rp, c->a_ci, (int)nb, de);
    CKL();
    std::vector<int> el(nu);
    CK(cudaMemcpyAsync(el.data(), de, nu * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    dfree(c, de);
    std::vector<long> cnt(ne + 2, 0);
    for (long i = 0; i < nu; ++i) cnt[std::min<long>(el[i], ne) + 1]++;
    for (long e = 0; e <= ne; ++e) cnt[e + 1] += cnt[e];
    for (long i = 0; i < nu; ++i) pu[cnt[std::min<long>(el[i], ne)]++] = (int)i;
  } else {
    for (long i = 0; i < nu; ++i) pu[i] = (int)i;
  }
  for (long i = 0; i < nu; ++i) ku[i] = alen[i];
  window_sort(pu, ku, REORDER_WINDOW);
  // elements: key = (max B row length, max S_D row length) of the element's DOFs
  std::vector<int> pe(ne);
  std::vector<long long> ke(ne);
  for (long e = 0; e < ne; ++e) {
    int ls = 0, lb = 0;
    for (long a = 0; a < nb; ++a) {
      ls = std::max(ls, slen[e * nb + a]);
      lb = std::max(lb, alen[nu + e * nb + a]);
    }
    pe[e] = (int)e;
    ke[e] = ((long long)lb << 32) | (long long)ls;
  }
  window_sort(pe, ke, std::max(1L, REORDER_WINDOW / nb));
  std::vector<int> perm(n), cmap(n);
  for (long i = 0; i < nu; ++i) perm[i] = pu[i];
  for (long e = 0; e < ne; ++e)
    for (long a = 0; a < nb; ++a) perm[nu + e * nb + a] = (int)(nu + (long)pe[e] * nb + a);
  for (long i = 0; i < n; ++i) cmap[perm[i]] = (int)i;
  // keep it only where it removes padding
  const long pad0 = sell_padded(alen, {}) + sell_padded(slen, {});
  std::vector<int> permp(np);
  for (long i = 0; i < np; ++i) permp[i] = perm[nu + i] - (int)nu;
  // S_D slots: rows (internal numbering) sorted by length in windows; slot_old = the CSR row
  std::vector<int> sslot(np), sslot_old(np);
  {
    std::vector<long long> ks(np);
    for (long i = 0; i < np; ++i) {
      sslot[i] = (int)i;
      ks[i] = slen[permp[i]];
    }
    // window of the row-level sort of the S_D slots (VEM_SLOT_WINDOW, default 256 = one CTA): a small
    // window keeps the rows of neighbouring elements in the same CTA (gather locality) for a little more
    // padding; C5 fine-level pass, stored entries / time: 4096 -> 42.97M / 128.5 us, 1024 -> 43.19M / 128.5,
    // 256 -> 43.67M / 123.6, 64 -> 48.44M / 131.1 (R2_25)
    const long slot_win = getenv("VEM_SLOT_WINDOW") ? std::max(32L, atol(getenv("VEM_SLOT_WINDOW"))) : 256L;
    window_sort(sslot, ks, slot_win);
    // moment-major slices (VEM_SLOT_MOMENT=1): the slots of a group of 32 consecutive elements are
    // ordered moment by moment, so a SELL slice holds the same moment of 32 neighbouring elements
    // (similar row lengths: the elements are already sorted by length) and its vector accesses are a
    // fixed 8 n_p-byte stride that the sibling warps of the CTA share through L1, instead of a
    // scatter over the 4096-row window; kept when its padding is within 3% of the row-sorted one
    if (getenv("VEM_SLOT_MOMENT") && atoi(getenv("VEM_SLOT_MOMENT")) != 0) {
      std::vector<int> ms(np);
      long o = 0;
      for (long g0 = 0; g0 < ne; g0 += 32) {
        const long cnt = std::min<long>(32, ne - g0);
        for (long a = 0; a < nb; ++a)
          for (long l = 0; l < cnt; ++l) ms[o++] = (int)((g0 + l) * nb + a);
      }
      std::vector<int> ms_old(np);
      for (long i = 0; i < np; ++i) ms_old[i] = permp[ms[i]];
      std::vector<int> so_tmp(np);
      for (long i = 0; i < np; ++i) so_tmp[i] = permp[sslot[i]];
      const long pad_sorted = sell_padded(slen, so_tmp), pad_moment = sell_padded(slen, ms_old);
      if (getenv("VEM_SETUP_TRACE"))
        fprintf(stderr, "[vem setup] S_D slots: row-sorted %ld, moment-major %ld stored entries\n", pad_sorted,
                pad_moment);
      if ((double)pad_moment <= 1.03 * (double)pad_sorted || atoi(getenv("VEM_SLOT_MOMENT")) == 2) sslot = ms;
    }
    for (long i = 0; i < np; ++i) sslot_old[i] = permp[sslot[i]];
  }
  const long pad1 = sell_padded(alen, perm) + sell_padded(slen, sslot_old);
  if ((double)pad0 < 1.05 * (double)pad1) return 0;
  std::vector<int> cmapp(np);
  for (long i = 0; i < np; ++i) cmapp[i] = cmap[nu + i] - (int)nu;
  int r;
  if ((r = upload_array(c, &c->perm, perm.data(), n))) return r;
  if ((r = upload_array(c, &c->cmap, cmap.data(), n))) return r;
  if ((r = upload_array(c, &c->perm_p, permp.data(), np))) return r;
  if ((r = upload_array(c, &c->cmap_p, cmapp.data(), np))) return r;
  if ((r = upload_array(c, &c->s_slot, sslot.data(), np))) return r;
  if ((r = upload_array(c, &c->s_slot_old, sslot_old.data(), np))) return r;
  // permute the per-row vectors built in the original order
  double *tmp = nullptr;
  DA(tmp, np * nb);
  auto permute = [&](double *v, long len, const int *pm, int w) {
    k_gather_rows<<<grid_stream(c, len * w), NT, 0, c->stream>>>(len, w, pm, v, tmp);
    cudaMemcpyAsync(v, tmp, len * w * sizeof(double), cudaMemcpyDeviceToDevice, c->stream);
  };
  {
    double *tu = nullptr;
    DA(tu, nu);
    k_gather_rows<<<grid_stream(c, nu), NT, 0, c->stream>>>(nu, 1, c->perm, c->dMinv, tu);
    CK(cudaMemcpyAsync(c->dMinv, tu, nu * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    dfree(c, tu);
  }
  permute(c->dSinv, np, c->perm_p, 1);
  if (c->wdiag) permute(c->wdiag, np, c->perm_p, 1);
  if (c->dSepsinv) permute(c->dSepsinv, np, c->perm_p, 1);
  if (c->dBinv) permute(c->dBinv, np, c->perm_p, (int)nb);
  if (c->dBeinv) permute(c->dBeinv, np, c->perm_p, (int)nb);
  CKL();
  CK(cudaStreamSynchronize(c->stream));
  dfree(c, tmp);
  c->reorder_pad = {pad0, pad1};
  return 0;
}

// ----------------------------------------------------------------------------
// S_D aggregation hierarchy (upload; oracle/amg.py AMG.__init__)
// ----------------------------------------------------------------------------
template <typename T>
int scan_excl(Ctx *c, const T *in, T *out, long n) {
  if (n >= (1L << 31)) return fail(c, VEM_ERR_INVALID, "scan of %ld items exceeds the 32-bit CUB count", n);
  size_t tb = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)n, c->stream));
  char *tmp = nullptr;
  DA(tmp, tb);
  CK(cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, (int)n, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  dfree(c, tmp);
  return 0;
}

template <typename T>
T read_back(Ctx *c, const T *p) {
  T v{};
  cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, c->stream);
  cudaStreamSynchronize(c->stream);
  return v;
}

// aggregates of level L (device agg, returns nc); MIS-2 by repeated distance-2 maxima
int amg_aggregate(Ctx *c, AmgLevel &L, double *diag, double theta, long &nc_out) {
  const long n = L.n;
  unsigned char *strong = nullptr;
  signed char *state = nullptr;
  long long *kv = nullptr, *k1 = nullptr, *k2 = nullptr;
  int *flag = nullptr, *rank = nullptr, *agg0 = nullptr, *agg1 = nullptr;
  unsigned *cnt = nullptr;
  DA(strong, L.nnz);
  DA(state, n);
  DA(kv, n);
  DA(k1, n);
  DA(k2, n);
  DA(flag, n + 1);
  DA(rank, n + 1);
  DA(agg0, n);
  DA(agg1, n);
  DA(cnt, 1);
  DA(L.agg, n);
  const int g = grid_stream(c, n);
  k_amg_strong<<<g, NT, 0, c->stream>>>(n, L.rp, L.ci, L.va, diag, theta, strong);
  CK(cudaMemsetAsync(state, 0, n, c->stream));
  for (int it = 0; it < 1000; ++it) {
    k_amg_mis_keys<<<g, NT, 0, c->stream>>>(n, state, kv);
    k_amg_nbr_max<<<g, NT, 0, c->stream>>>(n, L.rp, L.ci, strong, kv, k1);
    k_amg_nbr_max<<<g, NT, 0, c->stream>>>(n, L.rp, L.ci, strong, k1, k2);
    CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned), c->stream));
    k_amg_mis_update<<<g, NT, 0, c->stream>>>(n, state, k2, cnt);
    CKL();
    if (read_back(c, cnt) == 0u) break;
  }
  k_amg_flag<<<g, NT, 0, c->stream>>>(n, state, flag);
  CK(cudaMemsetAsync(flag + n, 0, sizeof(int), c->stream));
  {
    int r = scan_excl(c, flag, rank, n + 1);
    if (r) return r;
  }
  const int nroot = read_back(c, rank + n);
  k_amg_roots<<<g, NT, 0, c->stream>>>(n, state, rank, agg0, kv);
  k_amg_nbr_max<<<g, NT, 0, c->stream>>>(n, L.rp, L.ci, strong, kv, k1);
  k_amg_join<<<g, NT, 0, c->stream>>>(n, agg0, k1, agg1);
  k_amg_assigned_keys<<<g, NT, 0, c->stream>>>(n, agg1, kv);
  k_amg_nbr_max<<<g, NT, 0, c->stream>>>(n, L.rp, L.ci, strong, kv, k1);
  k_amg_join<<<g, NT, 0, c->stream>>>(n, agg1, k1, L.agg);
  k_amg_free_flag<<<g, NT, 0, c->stream>>>(n, L.agg, flag);
  CKL();
  {
    int r = scan_excl(c, flag, rank, n + 1);
    if (r) return r;
  }
  const int nfree = read_back(c, rank + n);
  k_amg_singletons<<<g, NT, 0, c->stream>>>(n, rank, nroot, L.agg);
  CKL();
  CK(cudaStreamSynchronize(c->stream));
  for (void *p : {(void *)strong, (void *)state, (void *)kv, (void *)k1, (void *)k2, (void *)flag, (void *)rank,
                  (void *)agg0, (void *)agg1, (void *)cnt})
    dfree(c, p);
  nc_out = (long)nroot + nfree;
  return 0;
}

// (key, value) pairs with key = row * ncols + col -> CSR (nrows x ncols): stable radix
// sort, flags at run starts, in-order run sums (deterministic).  k0 / v0 are consumed
// (freed).  *row_out (optional) receives the row of every stored entry.
// m_valid >= 0: the keys hold m - m_valid dropped entries (ASM_DROPPED, sorted last)
int sort_reduce_csr(Ctx *c, unsigned long long *k0, double *v0, long m, long nrows, long ncols, int **rp_out,
                    int **ci_out, double **va_out, long *nnz_out, int **row_out = nullptr, long m_valid = -1) {
  unsigned long long *k1 = nullptr;
  double *v1 = nullptr;
  int *flag = nullptr, *pos = nullptr, *crow = nullptr, *cnt = nullptr;
  DA(k1, m);
  DA(v1, m);
  DA(flag, m + 1);
  DA(pos, m + 1);
  if (m >= (1L << 31)) return fail(c, VEM_ERR_INVALID, "Galerkin expansion of %ld entries exceeds the 32-bit CUB count", m);
  int bits = 1;
  while ((1ULL << bits) < (unsigned long long)nrows * (unsigned long long)ncols) ++bits;
  if (m_valid >= 0) bits = 64;   // the drop marker is the largest key
  {
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, v0, v1, (int)m, 0, bits, c->stream));
    char *tmp = nullptr;
    DA(tmp, tb);
    CK(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, (int)m, 0, bits, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    dfree(c, tmp);
  }
  dfree(c, k0);
  dfree(c, v0);
  if (m_valid >= 0) m = m_valid;
  k_amg_run_flags<<<grid_stream(c, m), NT, 0, c->stream>>>(m, k1, flag);
  CK(cudaMemsetAsync(flag + m, 0, sizeof(int), c->stream));
  {
    int r = scan_excl(c, flag, pos, m + 1);
    if (r) return r;
  }
  const long nnz = read_back(c, pos + m);
  DA(crow, nnz);
  DA(*ci_out, nnz);
  DA(*va_out, nnz);
  DA(*rp_out, nrows + 1);
  DA(cnt, nrows + 1);
  k_amg_run_reduce<<<grid_stream(c, m), NT, 0, c->stream>>>(m, k1, v1, flag, pos, ncols, crow, *ci_out, *va_out);
  CK(cudaMemsetAsync(cnt, 0, (nrows + 1) * sizeof(int), c->stream));
  k_amg_row_count<<<grid_stream(c, nnz), NT, 0, c->stream>>>(nnz, crow, cnt);
  CKL();
  {
    int r = scan_excl(c, cnt, *rp_out, nrows + 1);
    if (r) return r;
  }
  for (void *p : {(void *)k1, (void *)v1, (void *)flag, (void *)pos, (void *)cnt}) dfree(c, p);
  if (row_out)
    *row_out = crow;
  else
    dfree(c, crow);
  *nnz_out = nnz;
  return 0;
}

// Galerkin A_c = T^T A T for the piecewise-constant T (keys agg_i nc + agg_j)
int amg_galerkin(Ctx *c, const AmgLevel &L, long nc, AmgLevel &C) {
  const long m = L.nnz;
  unsigned long long *k0 = nullptr;
  double *v0 = nullptr;
  DA(k0, m);
  DA(v0, m);
  k_amg_expand<<<grid_stream(c, L.n), NT, 0, c->stream>>>(L.n, L.rp, L.ci, L.va, L.agg, nc, k0, v0);
  CKL();
  C.n = nc;
  return sort_reduce_csr(c, k0, v0, m, nc, nc, &C.rp, &C.ci, &C.va, &C.nnz);
}

// exclusive scan of per-row 64-bit counts -> offsets, returns the total
long long scan_counts(Ctx *c, long long *cnt, long long *off, long n) {
  CK(cudaMemsetAsync(cnt + n, 0, sizeof(long long), c->stream));
  if (scan_excl(c, cnt, off, n + 1)) return -1;
  return read_back(c, off + n);
}

// Smoothed aggregation level (oracle/amg.py smoothed_prolongator, SA_LEVELS = 1):
// P = T - omega D^-1 (A T), omega = 4 / (3 lmax); A_c = P^T (A P); P^T for the restriction.
int amg_sa_level(Ctx *c, AmgLevel &L, long nc, AmgLevel &C) {
  const long n = L.n;
  // A T
  {
    unsigned long long *k0 = nullptr;
    double *v0 = nullptr;
    DA(k0, L.nnz);
    DA(v0, L.nnz);
    k_sa_expand_at<<<grid_stream(c, n), NT, 0, c->stream>>>(n, L.rp, L.ci, L.va, L.agg, nc, k0, v0);
    CKL();
    int *prow = nullptr;
    int r = sort_reduce_csr(c, k0, v0, L.nnz, n, nc, &L.prp, &L.pci, &L.pva, &L.pnnz, &prow);
    if (r) return r;
    const double omega = 4.0 / (3.0 * L.lmax);
    k_sa_pvals<<<grid_stream(c, L.pnnz), NT, 0, c->stream>>>(L.pnnz, prow, L.pci, L.agg, L.dinv, omega, L.pva);
    CKL();
    CK(cudaStreamSynchronize(c->stream));
    dfree(c, prow);
  }
  // Q = A P
  int *qrp = nullptr, *qci = nullptr;
  double *qva = nullptr;
  long qnnz = 0;
  long long *cnt = nullptr, *off = nullptr;
  DA(cnt, n + 1);
  DA(off, n + 1);
  {
    k_sa_count_ap<<<grid_stream(c, n), NT, 0, c->stream>>>(n, L.rp, L.ci, L.prp, cnt);
    CKL();
    const long long m = scan_counts(c, cnt, off, n);
    if (m < 0) return VEM_ERR_CUDA;
    unsigned long long *k0 = nullptr;
    double *v0 = nullptr;
    DA(k0, m);
    DA(v0, m);
    k_sa_fill_ap<<<grid_stream(c, n), NT, 0, c->stream>>>(n, L.rp, L.ci, L.va, L.prp, L.pci, L.pva, off, nc, k0,
                                                          v0);
    CKL();
    int r = sort_reduce_csr(c, k0, v0, m, n, nc, &qrp, &qci, &qva, &qnnz);
    if (r) return r;
  }
  // A_c = P^T Q
  {
    k_sa_count_ptq<<<grid_stream(c, n), NT, 0, c->stream>>>(n, L.prp, qrp, cnt);
    CKL();
    const long long m = scan_counts(c, cnt, off, n);
    if (m < 0) return VEM_ERR_CUDA;
    unsigned long long *k0 = nullptr;
    double *v0 = nullptr;
    DA(k0, m);
    DA(v0, m);
    k_sa_fill_ptq<<<grid_stream(c, n), NT, 0, c->stream>>>(n, L.prp, L.pci, L.pva, qrp, qci, qva, off, nc, k0, v0);
    CKL();
    C.n = nc;
    int r = sort_reduce_csr(c, k0, v0, m, nc, nc, &C.rp, &C.ci, &C.va, &C.nnz);
    if (r) return r;
  }
  for (void *p : {(void *)qrp, (void *)qci, (void *)qva, (void *)cnt, (void *)off}) dfree(c, p);
  // P^T (restriction) and the SELL copy of P (prolongation)
  {
    unsigned long long *k0 = nullptr;
    double *v0 = nullptr;
    DA(k0, L.pnnz);
    DA(v0, L.pnnz);
    k_sa_expand_pt<<<grid_stream(c, n), NT, 0, c->stream>>>(n, L.prp, L.pci, L.pva, k0, v0);
    CKL();
    long tn = 0;
    int r = sort_reduce_csr(c, k0, v0, L.pnnz, nc, n, &L.ptrp, &L.ptci, &L.ptva, &tn);
    if (r) return r;
    r = build_sell(c, n, L.prp, L.pci, L.pva, &L.psoff, &L.psci, &L.psva, &L.psnnz);
    if (r) return r;
  }
  L.sa = true;
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int amg_members(Ctx *c, AmgLevel &L) {
  int *cnt = nullptr, *fill = nullptr;
  DA(cnt, L.nc + 1);
  DA(fill, L.nc + 1);
  DA(L.moff, L.nc + 1);
  DA(L.mem, L.n);
  CK(cudaMemsetAsync(cnt, 0, (L.nc + 1) * sizeof(int), c->stream));
  CK(cudaMemsetAsync(fill, 0, (L.nc + 1) * sizeof(int), c->stream));
  k_amg_row_count<<<grid_stream(c, L.n), NT, 0, c->stream>>>(L.n, L.agg, cnt);
  CKL();
  {
    int r = scan_excl(c, cnt, L.moff, L.nc + 1);
    if (r) return r;
  }
  k_amg_members<<<grid_stream(c, L.n), NT, 0, c->stream>>>(L.n, L.agg, L.moff, fill, L.mem);
  k_amg_sort_members<<<grid_stream(c, L.nc), NT, 0, c->stream>>>(L.nc, L.moff, L.mem);
  CKL();
  CK(cudaStreamSynchronize(c->stream));
  dfree(c, cnt);
  dfree(c, fill);
  return 0;
}

int amg_level_vectors(Ctx *c, AmgLevel &L) {
  DA(L.b, L.n);
  DA(L.x, L.n);
  DA(L.t, L.n);
  DA(L.sr, L.n);
  DA(L.sd0, L.n);
  DA(L.sd1, L.n);
  return 0;
}

// Hierarchy H on the level-0 matrix L0 (CSR + SELL + D^-1 + lmax set by the caller, not owned);
// diag0 = its diagonal.  share_pool: the level-0 smoother vectors live in the L2-resident
// Chebyshev pool (the users of the pool never overlap in time).
int build_amg(Ctx *c, AmgHier &H, const AmgLevel &L0, double *diag0, bool share_pool) {
  H.lv.clear();
  H.lv.push_back(L0);
  int r = amg_level_vectors(c, H.lv.back());
  if (r) return r;
  if (share_pool) {
    AmgLevel &F = H.lv.back();
    dfree(c, F.sr);
    dfree(c, F.sd0);
    dfree(c, F.sd1);
    dfree(c, F.x);
    F.sr = c->cr;
    F.sd0 = c->cd0;
    F.sd1 = c->cd1;
    F.x = c->cx;
  }
  double *diag = diag0;
  while (true) {
    AmgLevel &L = H.lv.back();
    if (L.n <= AMG_COARSE_SIZE || (int)H.lv.size() >= c->amg_max_levels) break;
    long nc = 0;
    const size_t lev = H.lv.size() - 1;
    r = amg_aggregate(c, L, diag, lev == 0 ? AMG_THETA : AMG_THETA_COARSE, nc);
    if (r) return r;
    if (nc > AMG_STAGNATION * L.n) {
      dfree(c, L.agg);
      L.agg = nullptr;
      break;
    }
    L.nc = nc;
    AmgLevel C;
    if ((int)lev < AMG_SA_LEVELS) {
      r = amg_sa_level(c, H.lv.back(), nc, C);
      if (r) return r;
    } else {
      r = amg_galerkin(c, L, nc, C);
      if (r) return r;
      r = amg_members(c, H.lv.back());
      if (r) return r;
    }
    // coarse diagonal, Gershgorin bound, SELL copy, vectors
    double *cdiag = nullptr;
    DA(C.dinv, C.n);
    DA(cdiag, C.n);
    k_diag_inv<<<grid_stream(c, C.n), NT, 0, c->stream>>>(C.n, C.rp, C.ci, C.va, 0, C.dinv, cdiag, c->derr);
    k_gershgorin<<<grid_stream(c, C.n), NT, 0, c->stream>>>(C.n, C.rp, C.ci, C.va, c->part, c->counter, c->st);
    CKL();
    C.lmax = read_back(c, &c->st->lmax);
    if (read_back(c, c->derr)) return fail(c, VEM_ERR_DIAG_S, "non-positive diagonal in a coarse S_D level");
    r = build_sell(c, C.n, C.rp, C.ci, C.va, &C.soff, &C.sci, &C.sva, &C.nnz_sell);
    if (r) return r;
    // small coarse levels (latency-bound): G lanes per CSR row, G = 8 (C3 levels 2 and 3, 24.5 and 15.5
    // nnz per row: 151.8 ms vs 158.0 ms with a warp per row, r8 A/B in DESIGN §5; VEM_AMG_GROUP=0 picks
    // the power of two >= mean row length / VEM_AMG_GROUP_DIV in [4, 32]); else SELL-32, one thread per row
    C.warp_rows = C.n < c->amg_warp_rows || (double)C.nnz / C.n >= c->amg_warp_nnz;
    {
      int g = 4;
      while (g < 32 && c->amg_group_div * g < (double)C.nnz / C.n) g *= 2;
      C.group = c->amg_group ? c->amg_group : g;
    }
    r = amg_level_vectors(c, C);
    if (r) return r;
    H.lv.push_back(C);
    diag = cdiag;
  }
  AmgLevel &Lc = H.lv.back();
  H.dense = Lc.n <= AMG_COARSE_SIZE;
  if (H.dense) {
    double *D = nullptr;
    DA(D, (size_t)Lc.n * 2 * Lc.n);
    DA(H.cinv, (size_t)Lc.n * Lc.n);
    k_amg_dense<<<grid_stream(c, Lc.n), NT, 0, c->stream>>>(Lc.n, Lc.rp, Lc.ci, Lc.va, D);
    auto tg = std::chrono::steady_clock::now();
    double *piv = nullptr, *col = nullptr;
    DA(piv, 2 * Lc.n);
    DA(col, Lc.n);
    const long n = Lc.n;
    for (long k = 0; k < n; ++k) {
      k_amg_gj_pivot<<<(unsigned)((2 * n + NT - 1) / NT), NT, 0, c->stream>>>(n, k, D, piv, col, c->derr);
      k_amg_gj_update<<<dim3((unsigned)((n + 1 + NT - 1) / NT), (unsigned)n), NT, 0, c->stream>>>(n, k, D, piv, col);
    }
    k_amg_gj_extract<<<grid_stream(c, n * n), NT, 0, c->stream>>>(n, D, H.cinv);
    CKL();
    CK(cudaStreamSynchronize(c->stream));
    dfree(c, piv);
    dfree(c, col);
    if (getenv("VEM_SETUP_TRACE"))
      fprintf(stderr, "[vem setup] coarsest Gauss-Jordan n=%ld %9.1f ms\n", n,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tg).count());
    CK(cudaStreamSynchronize(c->stream));
    dfree(c, D);
    if (read_back(c, c->derr)) return fail(c, VEM_ERR_DIAG_S, "coarsest S_D level not positive definite");
  }
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

// Coarsest level without a dense inverse: nnz-balanced row ranges of the 16 CTAs of
// k_vc_coarse_cluster.  Left off (the per-step
// warp kernels run instead) when the cluster cannot be launched or a rank's slice
// does not fit in shared memory.
int build_amg_cluster(Ctx *c) {
  if (c->amg.lv.empty() || c->amg.dense || !c->amg_cluster) return 0;
  AmgLevel &L = c->amg.lv.back();
  if (!L.rp || !L.ci || L.n < VC_CLUSTER || L.n > 65535 || L.nnz >= (1L << 31)) return 0;
  if (c->amg_coarse_degree < 1 || c->amg_coarse_degree > VC_MAX_DEGREE) return 0;
  std::vector<int> rp(L.n + 1);
  CK(cudaMemcpyAsync(rp.data(), L.rp, (L.n + 1) * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  std::vector<int> rs(VC_CLUSTER + 1);
  rs[0] = 0;
  rs[VC_CLUSTER] = (int)L.n;
  for (int g = 1; g < VC_CLUSTER; ++g) {
    const long target = (long)rp[L.n] * g / VC_CLUSTER;
    rs[g] = std::max(rs[g - 1], (int)(std::lower_bound(rp.begin(), rp.end(), (int)target) - rp.begin()));
    rs[g] = std::min(rs[g], (int)L.n);
  }
  size_t sd = 0, sf = 0;
  for (int g = 0; g < VC_CLUSTER; ++g) {
    const int nr = rs[g + 1] - rs[g];
    const long nz = rp[rs[g + 1]] - rp[rs[g]];
    if (nr > VC_CLUSTER_THREADS * VC_ROWS_PER_THREAD) return 0;
    sd = std::max(sd, vc_cluster_smem<double>(L.n, nr, nz));
    sf = std::max(sf, vc_cluster_smem<float>(L.n, nr, nz));
  }
  int dev = 0, optin = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (sd > (size_t)optin) return 0;
  auto prep = [&](const void *fn, size_t smem) -> bool {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(VC_CLUSTER);
    cfg.blockDim = dim3(VC_CLUSTER_THREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = VC_CLUSTER;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return nclusters >= 1;
  };
  if (!prep((const void *)k_vc_coarse_cluster<double>, sd)) return 0;
  if (c->amg_f32 && !prep((const void *)k_vc_coarse_cluster<float>, sf)) return 0;
  DA(L.vc_rs, VC_CLUSTER + 1);
  DA(L.vc_c16, L.nnz);
  CK(cudaMemcpyAsync(L.vc_rs, rs.data(), (VC_CLUSTER + 1) * sizeof(int), cudaMemcpyHostToDevice, c->stream));
  k_vc_cols16<<<grid_stream(c, L.nnz), NT, 0, c->stream>>>(L.nnz, L.ci, L.vc_c16);
  CKL();
  CK(cudaStreamSynchronize(c->stream));
  L.vc_smem_d = sd;
  L.vc_smem_f = sf;
  L.vc_ok = true;
  return 0;
}

// FP32 mirror of the hierarchy for precond kind 4 (values rounded once; own vectors)
int build_amg_f32(Ctx *c) {
  auto cvt = [&](const double *in, long n, float **out) -> int {
    if (!in || n <= 0) return 0;
    DA(*out, n);
    k_d2f<<<grid_stream(c, n), NT, 0, c->stream>>>(n, in, *out);
    return 0;
  };
  for (size_t l = 0; l < c->amg.lv.size(); ++l) {
    AmgLevel &L = c->amg.lv[l];
    int r;
    if ((r = cvt(L.sva, l == 0 ? c->nnzS_sell : L.nnz_sell, &L.sva_f))) return r;
    if ((r = cvt(L.va, L.nnz, &L.va_f))) return r;
    if ((r = cvt(L.dinv, L.n, &L.dinv_f))) return r;
    if (L.sa) {
      if ((r = cvt(L.psva, L.psnnz, &L.psva_f))) return r;
      if ((r = cvt(L.ptva, L.pnnz, &L.ptva_f))) return r;
    }
    if (l == 0) {   // fine level: one contiguous pool (D^-1, r, d0, d1, x, b, t) for the L2 window
      const long npad = (L.n + 63) / 64 * 64;
      DA(c->f32_pool, 7 * npad);
      c->f32_pool_bytes = (size_t)7 * npad * sizeof(float);
      float *q = c->f32_pool;
      CK(cudaMemcpyAsync(q, L.dinv_f, L.n * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      dfree(c, L.dinv_f);
      L.dinv_f = q;
      L.sr_f = q + npad;
      L.sd0_f = q + 2 * npad;
      L.sd1_f = q + 3 * npad;
      L.x_f = q + 4 * npad;
      L.b_f = q + 5 * npad;
      L.t_f = q + 6 * npad;
      continue;
    }
    DA(L.b_f, L.n);
    DA(L.x_f, L.n);
    DA(L.t_f, L.n);
    DA(L.sr_f, L.n);
    DA(L.sd0_f, L.n);
    DA(L.sd1_f, L.n);
  }
  if (c->amg.dense) {
    const long nc = c->amg.lv.back().n;
    int r = cvt(c->amg.cinv, nc * nc, &c->amg.cinv_f);
    if (r) return r;
  }
  CKL();
  CK(cudaStreamSynchronize(c->stream));
  c->amg_f32 = true;
  return 0;
}

// device CSR produced by vem_mixed_assemble (int64 row pointers, like vem_csr)
struct DevCsr {
  long nrows = 0, ncols = 0, nnz = 0;
  int64_t *rp = nullptr;
  int *ci = nullptr;
  double *va = nullptr;
};

// M, B: host CSR (copied), or dM, dB: device CSR from vem_mixed_assemble (read, not owned)
int upload_impl(Ctx *c, const vem_csr *M, const vem_csr *B, const vem_csr *W, double eps, const vem_layout *lay,
                const DevCsr *dM = nullptr, const DevCsr *dB = nullptr) {
  auto t0 = std::chrono::steady_clock::now();
  const bool trace = getenv("VEM_SETUP_TRACE") != nullptr;
  c->pcg_split = getenv("VEM_PCG_SPLIT") ? atoi(getenv("VEM_PCG_SPLIT")) : 2;
  c->pcg_persist = getenv("VEM_PCG_PERSIST") ? atoi(getenv("VEM_PCG_PERSIST")) : 1;
  c->amg_coarse_degree = getenv("VEM_AMG_COARSE_DEGREE") ? atoi(getenv("VEM_AMG_COARSE_DEGREE")) : AMG_COARSE_DEGREE;
  c->amg_max_levels = getenv("VEM_AMG_MAX_LEVELS") ? atoi(getenv("VEM_AMG_MAX_LEVELS")) : AMG_MAX_LEVELS;
  c->amg_cluster = getenv("VEM_AMG_CLUSTER") ? atoi(getenv("VEM_AMG_CLUSTER")) : 0;
  c->amg_warp_rows = getenv("VEM_AMG_WARP_ROWS") ? atol(getenv("VEM_AMG_WARP_ROWS")) : 100000;
  c->amg_warp_nnz = getenv("VEM_AMG_WARP_NNZ") ? atof(getenv("VEM_AMG_WARP_NNZ")) : 1e30;
  c->amg_group = getenv("VEM_AMG_GROUP") ? atoi(getenv("VEM_AMG_GROUP")) : 8;
  c->amg_group_div = getenv("VEM_AMG_GROUP_DIV") ? atof(getenv("VEM_AMG_GROUP_DIV")) : 2.0;
  c->pdl = getenv("VEM_PDL") ? atoi(getenv("VEM_PDL")) : 1;
  c->trace_k = getenv("VEM_TRACE_K") && atoi(getenv("VEM_TRACE_K")) != 0;
  auto phase = [&](const char *what) {
    if (!trace) return;
    cudaStreamSynchronize(c->stream);
    fprintf(stderr, "[vem setup] %-28s %9.1f ms\n", what,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  };
  const bool dev_in = dM && dB;
  if (!dev_in && (!M || !B)) return fail(c, VEM_ERR_INVALID, "M and B are required");
  c->nu = dev_in ? dM->nrows : M->n_rows;
  c->np = dev_in ? dB->nrows : B->n_rows;
  c->n = c->nu + c->np;
  if (c->nu <= 0 || c->np <= 0) return fail(c, VEM_ERR_INVALID, "empty system");
  if (c->n >= (1L << 31)) return fail(c, VEM_ERR_INVALID, "n exceeds int32 indexing");
  int r;
  if (dev_in) {   // assembled on the device: sorted, unique and in range by construction
    if (dM->ncols != c->nu || dB->ncols != c->nu) return fail(c, VEM_ERR_INVALID, "assembled shapes disagree");
  } else {
    if ((r = check_csr(c, M, c->nu, c->nu, "M"))) return r;
    if ((r = check_csr(c, B, c->np, c->nu, "B"))) return r;
  }
  if (lay) {
    c->layout = *lay;
    c->nb = std::max(1, (int)lay->n_p_dof);
    if (c->nb > 10) return fail(c, VEM_ERR_INVALID, "n_p_dof > 10 is not supported (k <= 2)");
    const long nu = (long)lay->n_faces * lay->n_face_dof + (long)lay->n_elems * lay->n_int_dof;
    const long np = (long)lay->n_elems * lay->n_p_dof;
    if (nu != c->nu || np != c->np) return fail(c, VEM_ERR_INVALID, "layout does not match M/B sizes");
  }
  c->nnzM = dev_in ? dM->nnz : M->nnz;
  c->nnzB = dev_in ? dB->nnz : B->nnz;
  c->nnzA = c->nnzM + 2 * c->nnzB;
  if (c->nnzA >= (1L << 31)) return fail(c, VEM_ERR_INVALID, "nnz(A) exceeds int32 indexing");
  if (W) {
    if ((r = check_csr(c, W, c->np, c->np, "W"))) return r;
    for (long i = 0; i < c->np; ++i)
      if (W->indptr[i + 1] - W->indptr[i] != 1 || W->indices[W->indptr[i]] != i || !(W->values[W->indptr[i]] > 0))
        return fail(c, VEM_ERR_INVALID, "W must be diagonal with positive entries");
  }
  c->ldv = (c->n + 127) / 128 * 128;   // 1 KB-aligned basis vectors
  cudaDeviceProp prop;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaGetDeviceProperties(&prop, dev));
  c->sm_count = prop.multiProcessorCount;
  if (!getenv("VEM_MDOT_WAVE") || atoi(getenv("VEM_MDOT_WAVE")) != 0) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mdot, NT, 0) == cudaSuccess && occ > 0)
      c->mdot_slots = occ * c->sm_count;
  }
  if (!getenv("VEM_UPDATE_WAVE") || atoi(getenv("VEM_UPDATE_WAVE")) != 0) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_update, NT, 0) == cudaSuccess && occ > 0)
      c->update_slots = occ * c->sm_count;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_update32, NT, 0) == cudaSuccess && occ > 0)
      c->update32_slots = occ * c->sm_count;
  }
  if (c->mdot_slots > 0) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mdot32, NT, 0) == cudaSuccess && occ > 0)
      c->mdot32_slots = occ * c->sm_count;
  }

  // raw uploads (freed after the merged formats are built)
  int64_t *mrp = nullptr, *brp = nullptr;
  int *mci = nullptr, *bci = nullptr;
  double *mva = nullptr, *bva = nullptr;
  if (dev_in) {
    mrp = dM->rp;
    mci = dM->ci;
    mva = dM->va;
    brp = dB->rp;
    bci = dB->ci;
    bva = dB->va;
  } else {
    if ((r = upload_array(c, &mrp, M->indptr, c->nu + 1))) return r;
    if ((r = upload_array(c, &mci, M->indices, M->nnz))) return r;
    if ((r = upload_array(c, &mva, M->values, M->nnz))) return r;
    if ((r = upload_array(c, &brp, B->indptr, c->np + 1))) return r;
    if ((r = upload_array(c, &bci, B->indices, B->nnz))) return r;
    if ((r = upload_array(c, &bva, B->values, B->nnz))) return r;
  }
  if (W) {
    std::vector<double> wd(c->np);
    for (long i = 0; i < c->np; ++i) wd[i] = W->values[W->indptr[i]];
    if ((r = upload_array(c, &c->wdiag, wd.data(), c->np))) return r;
    CK(cudaStreamSynchronize(c->stream));
  }
  phase("validate + upload");
  // B^T (CSR over velocity rows), deterministic order
  int *btrp = nullptr, *btci = nullptr, *fill = nullptr;
  double *btva = nullptr;
  DA(btrp, c->nu + 1);
  DA(fill, c->nu + 1);
  DA(btci, c->nnzB);
  DA(btva, c->nnzB);
  CK(cudaMemsetAsync(fill, 0, (c->nu + 1) * sizeof(int), c->stream));
  k_count_cols<<<grid_stream(c, c->nnzB), NT, 0, c->stream>>>(c->nnzB, bci, fill);
  CKL();
  {
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, fill, btrp, (int)(c->nu + 1), c->stream));
    char *tmp = nullptr;
    DA(tmp, tb);
    CK(cub::DeviceScan::ExclusiveSum(tmp, tb, fill, btrp, (int)(c->nu + 1), c->stream));
    CK(cudaStreamSynchronize(c->stream));
    dfree(c, tmp);
  }
  CK(cudaMemsetAsync(fill, 0, (c->nu + 1) * sizeof(int), c->stream));
  int *brp32 = nullptr;
  DA(brp32, c->np + 1);
  k_widen<<<grid_stream(c, c->np + 1), NT, 0, c->stream>>>(c->np + 1, brp, brp32);
  k_scatter_T<<<grid_stream(c, c->np), NT, 0, c->stream>>>(c->np, brp32, bci, bva, btrp, fill, btci, btva);
  k_sort_rows<<<grid_stream(c, c->nu), NT, 0, c->stream>>>(c->nu, btrp, btci, btva);
  CKL();
  // merged A
  int *len = nullptr;
  DA(len, c->n + 1);
  DA(c->a_rp, c->n + 1);
  DA(c->a_ci, c->nnzA);
  DA(c->a_va, c->nnzA);
  k_a_rowlen<<<grid_stream(c, c->n), NT, 0, c->stream>>>(c->nu, c->np, mrp, btrp, brp, len);
  CKL();
  {
    CK(cudaMemsetAsync(len + c->n, 0, sizeof(int), c->stream));
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, len, c->a_rp, (int)(c->n + 1), c->stream));
    char *tmp = nullptr;
    DA(tmp, tb);
    CK(cub::DeviceScan::ExclusiveSum(tmp, tb, len, c->a_rp, (int)(c->n + 1), c->stream));
    CK(cudaStreamSynchronize(c->stream));
    dfree(c, tmp);
  }
  k_a_fill<<<grid_stream(c, c->n), NT, 0, c->stream>>>(c->nu, c->np, mrp, mci, mva, btrp, btci, btva, brp, bci, bva,
                                                       c->a_rp, c->a_ci, c->a_va);
  CKL();
  // state
  DA(c->st, 1);
  CK(cudaMallocHost((void **)&c->hst, sizeof(DevState)));
  memset(c->hst, 0, sizeof(DevState));
  c->hst->one = 1.0;
  c->hst->one_i = 1;
  CK(cudaMemcpyAsync(c->st, c->hst, sizeof(DevState), cudaMemcpyHostToDevice, c->stream));
  DA(c->derr, 1);
  CK(cudaMemsetAsync(c->derr, 0, sizeof(int), c->stream));
  DA(c->counter, 1);
  CK(cudaMemsetAsync(c->counter, 0, sizeof(unsigned), c->stream));
  {
    int rr = ensure_part(c, (long)c->sm_count * 64 + grid_for(c->n * 32) + 1024);
    if (rr) return rr;
  }
  // diag(M)^-1
  DA(c->dMinv, c->nu);
  k_diag_inv<<<grid_stream(c, c->nu), NT, 0, c->stream>>>(c->nu, c->a_rp, c->a_ci, c->a_va, 0, c->dMinv, nullptr,
                                                          c->derr);
  CKL();
  int herr = 0;
  CK(cudaMemcpyAsync(&herr, c->derr, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (herr) return fail(c, VEM_ERR_DIAG_M, "non-positive diagonal entry in M");
  phase("merged A, diag(M)");
  // S_D
  r = build_schur(c, brp, bci, bva, btrp, btci, btva);
  if (r) return r;
  phase("S_D spgemm");
  {  // Chebyshev working set in one contiguous pool: D^-1, r, d0, d1, x (L2-persisting window)
    const long npad = (c->np + 31) / 32 * 32;
    DA(c->cheb_pool, 5 * npad);
    c->cheb_pool_bytes = (size_t)5 * npad * sizeof(double);
    c->dSinv = c->cheb_pool;
    c->cr = c->cheb_pool + npad;
    c->cd0 = c->cheb_pool + 2 * npad;
    c->cd1 = c->cheb_pool + 3 * npad;
    c->cx = c->cheb_pool + 4 * npad;
  }
  DA(c->sdiag, c->np);
  k_diag_inv<<<grid_stream(c, c->np), NT, 0, c->stream>>>(c->np, c->s_rp, c->s_ci, c->s_va, 0, c->dSinv, c->sdiag,
                                                          c->derr);
  CKL();
  CK(cudaMemcpyAsync(&herr, c->derr, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (herr) return fail(c, VEM_ERR_DIAG_S, "non-positive diagonal entry in S_D = B diag(M)^-1 B^T");
  k_gershgorin<<<grid_stream(c, c->np), NT, 0, c->stream>>>(c->np, c->s_rp, c->s_ci, c->s_va, c->part, c->counter,
                                                            c->st);
  CKL();
  double lm = 0.0;
  CK(cudaMemcpyAsync(&lm, &c->st->lmax, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->lmax = lm;
  c->eps = eps;
  c->has_reg = eps > 0.0;
  if (c->has_reg) {
    DA(c->dSepsinv, c->np);
    k_shift_inv<<<grid_stream(c, c->np), NT, 0, c->stream>>>(c->np, c->sdiag, c->wdiag, eps, c->dSepsinv);
    CKL();
  }
  if (c->nb > 1) {
    if (c->np % c->nb) return fail(c, VEM_ERR_INVALID, "n_p is not a multiple of n_p_dof");
    DA(c->dBinv, (size_t)c->np * c->nb);
    dispatch_nb<BlkInvL>(c->nb, c, 0.0, c->dBinv);
    if (c->has_reg) {
      DA(c->dBeinv, (size_t)c->np * c->nb);
      dispatch_nb<BlkInvL>(c->nb, c, eps, c->dBeinv);
      DA(c->pz, c->np);
    }
    CKL();
    CK(cudaMemcpyAsync(&herr, c->derr, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (herr) return fail(c, VEM_ERR_DIAG_S, "singular element block of S_D");
  }
  // work vectors
  DA(c->x, c->n);
  DA(c->b, c->n);
  DA(c->z, c->n);
  DA(c->t, c->n);
  if (c->has_reg) {
    DA(c->px, c->np);
    DA(c->pr, c->np);
    DA(c->pp0, c->np);
    DA(c->pp1, c->np);
    DA(c->pq, c->np);
    DA(c->pb, c->np);
  }
  if (c->has_reg) {   // matrix of the S_eps hierarchy (R23), in the caller's numbering (before the reordering)
    if (c->nb == 1) {
      c->se_n = c->np;
      c->se_nnz = c->nnzS;
      c->se_rp = c->s_rp;
      c->se_ci = c->s_ci;
      DA(c->se_va, c->nnzS);
      CK(cudaMemcpyAsync(c->se_va, c->s_va, c->nnzS * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
      k_shift_diag<<<grid_stream(c, c->np), NT, 0, c->stream>>>(c->np, c->s_rp, c->s_ci, c->se_va, c->wdiag, eps);
      CKL();
    } else {
      const long ne = c->np / c->nb;
      int *cnt = nullptr;
      DA(cnt, ne + 1);
      DA(c->se_rp, ne + 1);
      CK(cudaMemsetAsync(cnt, 0, (ne + 1) * sizeof(int), c->stream));
      k_mg_coarse_count<<<grid_stream(c, ne), NT, 0, c->stream>>>(ne, c->nb, c->s_rp, c->s_ci, cnt);
      CKL();
      int rr = scan_excl(c, cnt, c->se_rp, ne + 1);
      if (rr) return rr;
      int tot = 0;
      CK(cudaMemcpyAsync(&tot, c->se_rp + ne, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      dfree(c, cnt);
      c->se_n = ne;
      c->se_nnz = tot;
      DA(c->se_ci, tot);
      DA(c->se_va, tot);
      k_mg_coarse_fill<<<grid_stream(c, ne), NT, 0, c->stream>>>(ne, c->nb, c->s_rp, c->s_ci, c->s_va, c->wdiag, eps,
                                                                 c->se_rp, c->se_ci, c->se_va);
      CKL();
    }
  }
  {
    int rr = build_reorder(c);
    if (rr) return rr;
    rr = build_sell(c, c->n, c->a_rp, c->a_ci, c->a_va, &c->a_soff, &c->a_sci, &c->a_sva, &c->nnzA_sell, c->perm,
                    c->cmap);
    if (rr) return rr;
    rr = build_sell(c, c->np, c->s_rp, c->s_ci, c->s_va, &c->s_soff, &c->s_sci, &c->s_sva, &c->nnzS_sell,
                    c->s_slot_old, c->cmap_p);
    if (rr) return rr;
  }
  CK(cudaStreamSynchronize(c->stream));
  phase("block inverses, SELL");
  if (c->nb == 1) {   // S_D hierarchy for precond kinds 3 and 4 (k = 0)
    AmgLevel L0;
    L0.n = c->np;
    L0.nnz = c->nnzS;
    L0.rp = c->s_rp;
    L0.ci = c->s_ci;
    L0.va = c->s_va;
    L0.soff = c->s_soff;
    L0.sci = c->s_sci;
    L0.sva = c->s_sva;
    L0.dinv = c->dSinv;
    L0.lmax = c->lmax;
    L0.owns_matrix = false;
    c->amg.coarse_degree = c->amg_coarse_degree;
    int rr = build_amg(c, c->amg, L0, c->sdiag, true);
    if (rr == VEM_ERR_DIAG_S) {
      // a singular S_D (pure Neumann data: B^T annihilates the constant pressure) has no dense
      // coarsest inverse: kinds 3 and 4 are unavailable for this system (solve returns
      // VEM_ERR_PRECOND), kinds 1, 2 and 5 do not need the hierarchy
      c->amg.lv.clear();
      c->amg.dense = false;
      c->amg_unavailable = c->err;
      CK(cudaMemsetAsync(c->derr, 0, sizeof(int), c->stream));
      CK(cudaStreamSynchronize(c->stream));
      rr = 0;
    } else {
      if (rr) return rr;
      rr = build_amg_f32(c);
      if (rr) return rr;
      rr = build_amg_cluster(c);
      if (rr) return rr;
    }
  }
  if (c->has_reg) {   // S_eps hierarchy: the V-cycle preconditioner of Block-Reg's inner PCG (R23)
    AmgLevel L0;
    L0.n = c->se_n;
    L0.nnz = c->se_nnz;
    L0.rp = c->se_rp;
    L0.ci = c->se_ci;
    L0.va = c->se_va;
    L0.owns_matrix = false;
    DA(c->se_dinv, L0.n);
    DA(c->se_diag, L0.n);
    k_diag_inv<<<grid_stream(c, L0.n), NT, 0, c->stream>>>(L0.n, L0.rp, L0.ci, L0.va, 0, c->se_dinv, c->se_diag,
                                                           c->derr);
    k_gershgorin<<<grid_stream(c, L0.n), NT, 0, c->stream>>>(L0.n, L0.rp, L0.ci, L0.va, c->part, c->counter, c->st);
    CKL();
    L0.lmax = read_back(c, &c->st->lmax);
    if (read_back(c, c->derr)) return fail(c, VEM_ERR_DIAG_S, "non-positive diagonal in S_D + eps W");
    L0.dinv = c->se_dinv;
    int rr = build_sell(c, L0.n, L0.rp, L0.ci, L0.va, &L0.soff, &L0.sci, &L0.sva, &L0.nnz_sell);
    if (rr) return rr;
    c->amge.coarse_degree = getenv("VEM_MG_COARSE_DEGREE") ? atoi(getenv("VEM_MG_COARSE_DEGREE")) : MG_COARSE_DEGREE;
    rr = build_amg(c, c->amge, L0, c->se_diag, c->nb == 1);
    if (rr) return rr;
    if (c->nb == 1) {
      c->mg_r = c->amge.lv[0].b;
      c->mg_z = c->amge.lv[0].x;
    } else {
      c->mg_r = c->pr;
      c->mg_z = c->pz;
    }
  }
  phase("AMG hierarchy");
  {
    int rr = apply_l2_window(c);
    if (rr) return rr;
  }
  dfree(c, c->a_rp);
  dfree(c, c->a_ci);
  dfree(c, c->a_va);
  c->a_rp = nullptr;
  c->a_ci = nullptr;
  c->a_va = nullptr;
  if (!dev_in)
    for (void *p : {(void *)mrp, (void *)mci, (void *)mva, (void *)brp, (void *)bci, (void *)bva}) dfree(c, p);
  for (void *p : {(void *)btrp, (void *)btci, (void *)btva, (void *)fill, (void *)brp32, (void *)len}) dfree(c, p);
  c->setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  phase("done");
  return 0;
}

void destroy_ctx(Ctx *c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->l2_window_bytes) cudaCtxResetPersistingL2Cache();
  destroy_graphs(c);
  flush_timing(c);
  for (auto e : c->free_events) cudaEventDestroy(e);
  for (auto e : c->samp_a) cudaEventDestroy(e);
  for (auto e : c->samp_b) cudaEventDestroy(e);
  if (c->mg_samp_a) cudaEventDestroy(c->mg_samp_a);
  if (c->mg_samp_b) cudaEventDestroy(c->mg_samp_b);
  for (void *p : c->allocs) cudaFree(p);
  if (c->hst) cudaFreeHost(c->hst);
  if (c->ev_in) cudaEventDestroy(c->ev_in);
  if (c->ev_out) cudaEventDestroy(c->ev_out);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

// order the library stream after the caller's stream (entry) and vice versa (exit)
int enter(Ctx *c) {
  CK(cudaEventRecord(c->ev_in, c->user_stream));
  CK(cudaStreamWaitEvent(c->stream, c->ev_in, 0));
  return 0;
}
int leave(Ctx *c, int rc) {
  if (cudaEventRecord(c->ev_out, c->stream) == cudaSuccess) cudaStreamWaitEvent(c->user_stream, c->ev_out, 0);
  return rc;
}

// ----------------------------------------------------------------------------
// element-parallel assembly (vem_mixed_assemble, assembly.cuh)
// ----------------------------------------------------------------------------
int assemble_impl(Ctx *c, const vem_cell_class *cls, int ncls, long nu, long np, DevCsr &M, DevCsr &B,
                  double **f) {
  if (!cls || ncls <= 0 || nu <= 0 || np <= 0) return fail(c, VEM_ERR_INVALID, "empty assembly input");
  if (nu + np >= (1L << 31)) return fail(c, VEM_ERR_INVALID, "n exceeds int32 indexing");
  long mM = 0, mB = 0;
  for (int q = 0; q < ncls; ++q) {
    const vem_cell_class &k = cls[q];
    if (k.n_cells <= 0 || k.n_loc <= 0 || k.n_p <= 0 || k.n_t <= 0 || k.n_b <= 0 || !k.dof || !k.pdof || !k.ti ||
        !k.tj || !k.tA || !k.tS || !k.coef || !k.bi || !k.bj || !k.tB || !k.Hinv || !k.F || !k.vol)
      return fail(c, VEM_ERR_INVALID, "class %d: NULL pointer or empty size", q);
    for (long i = 0; i < k.n_cells * (long)k.n_loc; ++i)
      if (k.dof[i] < 0 || k.dof[i] >= nu) return fail(c, VEM_ERR_INVALID, "class %d: velocity DOF out of range", q);
    for (long i = 0; i < k.n_cells * (long)k.n_p; ++i)
      if (k.pdof[i] < 0 || k.pdof[i] >= np) return fail(c, VEM_ERR_INVALID, "class %d: pressure DOF out of range", q);
    for (int t = 0; t < k.n_t; ++t)
      if (k.ti[t] < 0 || k.ti[t] >= k.n_loc || k.tj[t] < 0 || k.tj[t] >= k.n_loc)
        return fail(c, VEM_ERR_INVALID, "class %d: template index out of range", q);
    for (int t = 0; t < k.n_b; ++t)
      if (k.bi[t] < 0 || k.bi[t] >= k.n_p || k.bj[t] < 0 || k.bj[t] >= k.n_loc)
        return fail(c, VEM_ERR_INVALID, "class %d: B template index out of range", q);
    mM += k.n_cells * (long)k.n_t;
    mB += k.n_cells * (long)k.n_b;
  }
  if (mM >= (1L << 31) || mB >= (1L << 31)) return fail(c, VEM_ERR_INVALID, "too many local entries");
  cudaDeviceProp prop;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaGetDeviceProperties(&prop, dev));
  c->sm_count = prop.multiProcessorCount;
  unsigned long long *kM = nullptr, *kB = nullptr;
  double *vM = nullptr, *vB = nullptr;
  DA(kM, mM);
  DA(vM, mM);
  DA(kB, mB);
  DA(vB, mB);
  DA(*f, np);
  CK(cudaMemsetAsync(*f, 0, np * sizeof(double), c->stream));
  long oM = 0, oB = 0;
  for (int q = 0; q < ncls; ++q) {
    const vem_cell_class &k = cls[q];
    const long ne = k.n_cells;
    int *dof = nullptr, *pdof = nullptr, *ti = nullptr, *tj = nullptr, *bi = nullptr, *bj = nullptr;
    double *tA = nullptr, *tS = nullptr, *coef = nullptr, *tB = nullptr, *Hinv = nullptr, *F = nullptr, *vol = nullptr;
    int r;
    if ((r = upload_array(c, &dof, k.dof, ne * k.n_loc))) return r;
    if ((r = upload_array(c, &pdof, k.pdof, ne * k.n_p))) return r;
    if ((r = upload_array(c, &ti, k.ti, k.n_t))) return r;
    if ((r = upload_array(c, &tj, k.tj, k.n_t))) return r;
    if ((r = upload_array(c, &tA, k.tA, 3L * k.n_t))) return r;
    if ((r = upload_array(c, &tS, k.tS, k.n_t))) return r;
    if ((r = upload_array(c, &coef, k.coef, 4 * ne))) return r;
    if ((r = upload_array(c, &bi, k.bi, k.n_b))) return r;
    if ((r = upload_array(c, &bj, k.bj, k.n_b))) return r;
    if ((r = upload_array(c, &tB, k.tB, k.n_b))) return r;
    if ((r = upload_array(c, &Hinv, k.Hinv, (long)k.n_p * k.n_p))) return r;
    if ((r = upload_array(c, &F, k.F, ne * k.n_p))) return r;
    if ((r = upload_array(c, &vol, k.vol, ne))) return r;
    k_asm_m<<<grid_stream(c, ne * k.n_t), NT, 0, c->stream>>>(ne, k.n_loc, k.n_t, dof, ti, tj, tA, tS, coef, nu,
                                                             kM + oM, vM + oM);
    k_asm_b<<<grid_stream(c, ne * k.n_b), NT, 0, c->stream>>>(ne, k.n_loc, k.n_p, k.n_b, dof, pdof, bi, bj, tB, nu,
                                                             kB + oB, vB + oB);
    k_asm_f<<<grid_stream(c, ne * k.n_p), NT, 0, c->stream>>>(ne, k.n_p, pdof, Hinv, F, vol, *f);
    CKL();
    CK(cudaStreamSynchronize(c->stream));
    for (void *p : {(void *)dof, (void *)pdof, (void *)ti, (void *)tj, (void *)tA, (void *)tS, (void *)coef,
                    (void *)bi, (void *)bj, (void *)tB, (void *)Hinv, (void *)F, (void *)vol})
      dfree(c, p);
    oM += ne * k.n_t;
    oB += ne * k.n_b;
  }
  int *rp32 = nullptr;
  int r = sort_reduce_csr(c, kM, vM, mM, nu, nu, &rp32, &M.ci, &M.va, &M.nnz);
  if (r) return r;
  DA(M.rp, nu + 1);
  k_widen64<<<grid_stream(c, nu + 1), NT, 0, c->stream>>>(nu + 1, rp32, M.rp);
  CK(cudaStreamSynchronize(c->stream));
  dfree(c, rp32);
  M.nrows = nu;
  M.ncols = nu;
  r = sort_reduce_csr(c, kB, vB, mB, np, nu, &rp32, &B.ci, &B.va, &B.nnz);
  if (r) return r;
  DA(B.rp, np + 1);
  k_widen64<<<grid_stream(c, np + 1), NT, 0, c->stream>>>(np + 1, rp32, B.rp);
  CK(cudaStreamSynchronize(c->stream));
  dfree(c, rp32);
  B.nrows = np;
  B.ncols = nu;
  return 0;
}

}  // namespace

struct vem_ctx {
  Ctx *impl;
};
struct vem_asm {
  Ctx *impl;   // allocations + stream
  DevCsr M, B;
  double *f = nullptr;
};

static thread_local std::string g_last_err;

extern "C" {

void vem_mixed_default_options(vem_opts *o) {
  if (!o) return;
  o->restart = 30;
  o->cheb_degree = 16;
  o->cheb_ratio = 30.0;
  o->inner_rtol = 1e-14;
  o->inner_maxit = 10000;
  o->use_graphs = 1;
  o->timing = 0;
  o->pcg_chunk = 16;
  o->reorth = -1;
  o->l2_persist = 1;
  o->reorder = 1;
  o->inner_precond = 1;
  o->k_maxit = 500;
  o->k_rtol = 0.1;
  o->k_inner_rtol = 1e-8;
  o->mg_chunk = 2;
  o->basis_f32 = 0;
}

static int validate_opts(Ctx *c, const vem_opts *o) {
  if (o->restart < 1 || o->restart > 100) return fail(c, VEM_ERR_INVALID, "restart must be in [1, 100]");
  if (o->cheb_degree < 1) return fail(c, VEM_ERR_INVALID, "cheb_degree must be >= 1");
  if (!(o->cheb_ratio > 1.0)) return fail(c, VEM_ERR_INVALID, "cheb_ratio must be > 1");
  if (!(o->inner_rtol > 0.0) || o->inner_maxit < 1) return fail(c, VEM_ERR_INVALID, "bad inner PCG options");
  if (o->reorth < -1 || o->reorth > 1) return fail(c, VEM_ERR_INVALID, "reorth must be -1, 0 or 1");
  if (o->reorder < 0 || o->reorder > 1) return fail(c, VEM_ERR_INVALID, "reorder must be 0 or 1");
  if (o->inner_precond < 0 || o->inner_precond > 1) return fail(c, VEM_ERR_INVALID, "inner_precond must be 0 or 1");
  if (o->k_maxit < 1 || !(o->k_rtol > 0.0) || !(o->k_inner_rtol > 0.0) || o->mg_chunk < 1)
    return fail(c, VEM_ERR_INVALID, "bad kind-5 / MG-PCG options");
  if (o->basis_f32 < 0 || o->basis_f32 > 1) return fail(c, VEM_ERR_INVALID, "basis_f32 must be 0 or 1");
  return 0;
}

__global__ void k_count_valid(long m, const unsigned long long *__restrict__ keys, unsigned long long *cnt) {
  unsigned long long local = 0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (long)gridDim.x * blockDim.x)
    local += keys[i] != ASM_DROPPED ? 1ULL : 0ULL;
  if (local) atomicAdd(cnt, local);
}

int assemble_tets_impl(Ctx *c, const vem_tet_class *cls, int ncls, long nu, long np, DevCsr &M, DevCsr &B,
                       double **f) {
  if (!cls || ncls <= 0 || nu <= 0 || np <= 0) return fail(c, VEM_ERR_INVALID, "empty assembly input");
  cudaDeviceProp prop;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaGetDeviceProperties(&prop, dev));
  c->sm_count = prop.multiProcessorCount;
  long mM = 0, mB = 0;
  for (int q = 0; q < ncls; ++q) {
    const vem_tet_class &t = cls[q];
    if (t.k < 0 || t.k > 1) return fail(c, VEM_ERR_INVALID, "device tetrahedral local operators: k = 0, 1 only");
    if (t.n_cells <= 0 || !t.cell || !t.faces || !t.signs || !t.coef || !t.dof || !t.pdof || !t.F || !t.vref ||
        !t.fref || t.n_qv <= 0 || t.n_qf <= 0 || !t.alphas1 || !t.betas || !t.rgrad || !t.rcross || !t.dgrad ||
        (t.k > 0 && !t.gens))
      return fail(c, VEM_ERR_INVALID, "tet class %d: NULL pointer or empty size", q);
    const int nk = dim_pk3(t.k), nloc = 4 * dim_pk2(t.k) + nk - 1 + dim_gp(t.k);
    for (long i = 0; i < t.n_cells * (long)nloc; ++i)
      if (t.dof[i] < 0 || t.dof[i] >= nu) return fail(c, VEM_ERR_INVALID, "tet class %d: velocity DOF out of range", q);
    for (long i = 0; i < t.n_cells * (long)nk; ++i)
      if (t.pdof[i] < 0 || t.pdof[i] >= np) return fail(c, VEM_ERR_INVALID, "tet class %d: pressure DOF out of range", q);
    mM += t.n_cells * (long)nloc * nloc;
    mB += t.n_cells * (long)nk * nloc;
  }
  if (mM >= (1L << 31) || mB >= (1L << 31)) return fail(c, VEM_ERR_INVALID, "too many local entries");
  unsigned long long *kM = nullptr, *kB = nullptr, *cnt = nullptr;
  double *vM = nullptr, *vB = nullptr;
  DA(kM, mM);
  DA(vM, mM);
  DA(kB, mB);
  DA(vB, mB);
  DA(cnt, 2);
  DA(*f, np);
  CK(cudaMemsetAsync(*f, 0, np * sizeof(double), c->stream));
  CK(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), c->stream));
  long oM = 0, oB = 0;
  for (int q = 0; q < ncls; ++q) {
    const vem_tet_class &t = cls[q];
    const long ne = t.n_cells;
    const int nk = dim_pk3(t.k), nk1 = dim_pk3(t.k + 1), nf = dim_pk2(t.k), ng = dim_gp(t.k);
    const int nloc = 4 * nf + nk - 1 + ng;
    double *cell = nullptr, *faces = nullptr, *signs = nullptr, *coef = nullptr, *F = nullptr, *vref = nullptr,
           *fref = nullptr, *al1 = nullptr, *bet = nullptr, *rg = nullptr, *rc = nullptr, *dg = nullptr,
           *gens = nullptr;
    int *dof = nullptr, *pdof = nullptr;
    int r;
    if ((r = upload_array(c, &cell, t.cell, ne * 17))) return r;
    if ((r = upload_array(c, &faces, t.faces, ne * 4 * 23))) return r;
    if ((r = upload_array(c, &signs, t.signs, ne * 4))) return r;
    if ((r = upload_array(c, &coef, t.coef, ne * 4))) return r;
    if ((r = upload_array(c, &F, t.F, ne * nk))) return r;
    if ((r = upload_array(c, &dof, t.dof, ne * nloc))) return r;
    if ((r = upload_array(c, &pdof, t.pdof, ne * nk))) return r;
    if ((r = upload_array(c, &vref, t.vref, 4L * t.n_qv))) return r;
    if ((r = upload_array(c, &fref, t.fref, 3L * t.n_qf))) return r;
    if ((r = upload_array(c, &al1, t.alphas1, 3L * nk1))) return r;
    if ((r = upload_array(c, &bet, t.betas, 2L * nf))) return r;
    if ((r = upload_array(c, &rg, t.rgrad, 6L * nk))) return r;
    if ((r = upload_array(c, &rc, t.rcross, 24L * nk))) return r;
    if ((r = upload_array(c, &dg, t.dgrad, 6L * std::max(nk - 1, 1)))) return r;
    if (ng > 0 && (r = upload_array(c, &gens, t.gens, 2L * ng))) return r;
    const int blocks = (int)((ne + 63) / 64);
    if (t.k == 0)
      k_local_tet<0><<<blocks, 64, 0, c->stream>>>(ne, cell, faces, signs, coef, dof, pdof, F, vref, t.n_qv, fref,
                                                    t.n_qf, al1, bet, rg, rc, dg, gens, nu, kM + oM, vM + oM,
                                                    kB + oB, vB + oB, *f);
    else
      k_local_tet<1><<<blocks, 64, 0, c->stream>>>(ne, cell, faces, signs, coef, dof, pdof, F, vref, t.n_qv, fref,
                                                    t.n_qf, al1, bet, rg, rc, dg, gens, nu, kM + oM, vM + oM,
                                                    kB + oB, vB + oB, *f);
    CKL();
    CK(cudaStreamSynchronize(c->stream));
    for (void *p : {(void *)cell, (void *)faces, (void *)signs, (void *)coef, (void *)F, (void *)dof, (void *)pdof,
                    (void *)vref, (void *)fref, (void *)al1, (void *)bet, (void *)rg, (void *)rc, (void *)dg,
                    (void *)gens})
      dfree(c, p);
    oM += ne * (long)nloc * nloc;
    oB += ne * (long)nk * nloc;
  }
  k_count_valid<<<grid_stream(c, mM), NT, 0, c->stream>>>(mM, kM, cnt);
  k_count_valid<<<grid_stream(c, mB), NT, 0, c->stream>>>(mB, kB, cnt + 1);
  CKL();
  unsigned long long nv[2];
  CK(cudaMemcpyAsync(nv, cnt, sizeof(nv), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  dfree(c, cnt);
  int *rp32 = nullptr;
  int r = sort_reduce_csr(c, kM, vM, mM, nu, nu, &rp32, &M.ci, &M.va, &M.nnz, nullptr, (long)nv[0]);
  if (r) return r;
  DA(M.rp, nu + 1);
  k_widen64<<<grid_stream(c, nu + 1), NT, 0, c->stream>>>(nu + 1, rp32, M.rp);
  CK(cudaStreamSynchronize(c->stream));
  dfree(c, rp32);
  M.nrows = nu;
  M.ncols = nu;
  r = sort_reduce_csr(c, kB, vB, mB, np, nu, &rp32, &B.ci, &B.va, &B.nnz, nullptr, (long)nv[1]);
  if (r) return r;
  DA(B.rp, np + 1);
  k_widen64<<<grid_stream(c, np + 1), NT, 0, c->stream>>>(np + 1, rp32, B.rp);
  CK(cudaStreamSynchronize(c->stream));
  dfree(c, rp32);
  B.nrows = np;
  B.ncols = nu;
  return 0;
}

static Ctx *new_ctx(const vem_opts *opts, void *stream, int *rc) {
  Ctx *c = new Ctx();
  vem_mixed_default_options(&c->opts);
  *rc = 0;
  if (opts) {
    int r = validate_opts(c, opts);
    if (r) {
      *rc = r;
      return c;
    }
    c->opts = *opts;
  }
  c->user_stream = (cudaStream_t)stream;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming) != cudaSuccess) {
    c->err = "failed to create the library stream (no CUDA device?)";
    *rc = VEM_ERR_CUDA;
  }
  return c;
}

static int upload_common(vem_ctx **out, const vem_csr *M, const vem_csr *B, const vem_csr *W, double eps,
                         const vem_layout *layout, const vem_opts *opts, void *stream, const DevCsr *dM,
                         const DevCsr *dB) {
  if (!out) return VEM_ERR_INVALID;
  *out = nullptr;
  int r = 0;
  Ctx *c = new_ctx(opts, stream, &r);
  if (!r) r = enter(c);
  if (!r) r = upload_impl(c, M, B, W, eps, layout, dM, dB);
  if (c->stream) leave(c, r);
  if (r) {
    g_last_err = c->err;
    destroy_ctx(c);
    return r;
  }
  vem_ctx *h = new vem_ctx{c};
  *out = h;
  return VEM_OK;
}

int vem_mixed_upload(vem_ctx **out, const vem_csr *M, const vem_csr *B, const vem_csr *W, double eps,
                     const vem_layout *layout, const vem_opts *opts, void *stream) {
  return upload_common(out, M, B, W, eps, layout, opts, stream, nullptr, nullptr);
}

int vem_mixed_upload_assembled(vem_ctx **out, const vem_asm *a, const vem_csr *W, double eps,
                               const vem_layout *layout, const vem_opts *opts, void *stream) {
  if (!a) return VEM_ERR_INVALID;
  CK_RET(cudaStreamSynchronize(a->impl->stream));
  return upload_common(out, nullptr, nullptr, W, eps, layout, opts, stream, &a->M, &a->B);
}

int vem_mixed_assemble(vem_asm **out, const vem_cell_class *classes, int32_t n_classes, int64_t n_u, int64_t n_p,
                       void *stream) {
  if (!out) return VEM_ERR_INVALID;
  *out = nullptr;
  int r = 0;
  Ctx *c = new_ctx(nullptr, stream, &r);
  vem_asm *a = new vem_asm();
  a->impl = c;
  if (!r) r = enter(c);
  if (!r) r = assemble_impl(c, classes, n_classes, n_u, n_p, a->M, a->B, &a->f);
  if (c->stream) leave(c, r);
  if (r) {
    g_last_err = c->err;
    destroy_ctx(c);
    delete a;
    return r;
  }
  *out = a;
  return VEM_OK;
}

int vem_mixed_assemble_tets(vem_asm **out, const vem_tet_class *classes, int32_t n_classes, int64_t n_u,
                            int64_t n_p, void *stream) {
  if (!out) return VEM_ERR_INVALID;
  *out = nullptr;
  int r = 0;
  Ctx *c = new_ctx(nullptr, stream, &r);
  vem_asm *a = new vem_asm();
  a->impl = c;
  if (!r) r = enter(c);
  if (!r) r = assemble_tets_impl(c, classes, n_classes, n_u, n_p, a->M, a->B, &a->f);
  if (c->stream) leave(c, r);
  if (r) {
    g_last_err = c->err;
    destroy_ctx(c);
    delete a;
    return r;
  }
  *out = a;
  return VEM_OK;
}

int vem_mixed_assembled_info(const vem_asm *a, int64_t *nnz_M, int64_t *nnz_B) {
  if (!a || !nnz_M || !nnz_B) return VEM_ERR_INVALID;
  *nnz_M = a->M.nnz;
  *nnz_B = a->B.nnz;
  return VEM_OK;
}

int vem_mixed_assembled_copy(const vem_asm *a, int64_t *mrp, int32_t *mci, double *mva, int64_t *brp, int32_t *bci,
                             double *bva, double *f) {
  if (!a || !mrp || !mci || !mva || !brp || !bci || !bva || !f) return VEM_ERR_INVALID;
  cudaStream_t s = a->impl->stream;
  CK_RET(cudaMemcpyAsync(mrp, a->M.rp, (a->M.nrows + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK_RET(cudaMemcpyAsync(mci, a->M.ci, a->M.nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CK_RET(cudaMemcpyAsync(mva, a->M.va, a->M.nnz * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK_RET(cudaMemcpyAsync(brp, a->B.rp, (a->B.nrows + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK_RET(cudaMemcpyAsync(bci, a->B.ci, a->B.nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CK_RET(cudaMemcpyAsync(bva, a->B.va, a->B.nnz * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK_RET(cudaMemcpyAsync(f, a->f, a->B.nrows * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK_RET(cudaStreamSynchronize(s));
  return VEM_OK;
}

void vem_mixed_assembled_free(vem_asm *a) {
  if (!a) return;
  destroy_ctx(a->impl);
  delete a;
}

int vem_mixed_solve(vem_ctx *h, const double *rhs, double tol, int32_t maxit, int32_t kind, double *out_u,
                    double *out_p, vem_solve_report *rep) {
  if (!h) return VEM_ERR_INVALID;
  Ctx *c = h->impl;
  int r = enter(c);
  if (r) return r;
  return leave(c, solve_impl(c, rhs, tol, maxit, kind, out_u, out_p, rep));
}

int vem_mixed_solve_host(vem_ctx *h, const double *rhs_host, double tol, int32_t maxit, int32_t kind,
                         double *u_host, double *p_host, vem_solve_report *rep) {
  if (!h || !rhs_host || !u_host || !p_host) return VEM_ERR_INVALID;
  Ctx *c = h->impl;
  {
    int r0 = enter(c);
    if (r0) return r0;
  }
  // device staging buffers for host solves, allocated once per context
  if (!c->h_rhs) {
    DA(c->h_rhs, c->n);
    DA(c->h_u, c->nu);
    DA(c->h_p, c->np);
  }
  CK(cudaMemcpyAsync(c->h_rhs, rhs_host, c->n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  int r = solve_impl(c, c->h_rhs, tol, maxit, kind, c->h_u, c->h_p, rep);
  if (r >= 0) {
    CK(cudaMemcpyAsync(u_host, c->h_u, c->nu * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(p_host, c->h_p, c->np * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  return leave(c, r);
}

int vem_mixed_spmv(vem_ctx *h, const double *x, double *y) {
  if (!h || !x || !y) return VEM_ERR_INVALID;
  Ctx *c = h->impl;
  int r = enter(c);
  if (r) return r;
  if (c->perm) {   // x, y in the caller's numbering
    to_internal(c, x, c->t);
    launch_spmv(c, 0L, c->n, c->t, c->z, nullptr, 0, gate_one(c));
    from_internal(c, c->z, y, y + c->nu);
  } else {
    launch_spmv(c, 0L, c->n, x, y, nullptr, 0, gate_one(c));
  }
  CKL();
  CK(cudaStreamSynchronize(c->stream));
  return leave(c, VEM_OK);
}

int vem_mixed_schur_spmv(vem_ctx *h, const double *x, double *y) {
  if (!h || !x || !y) return VEM_ERR_INVALID;
  Ctx *c = h->impl;
  int r = enter(c);
  if (r) return r;
  if (c->perm) {   // pressure vectors in the caller's numbering
    k_gather_rows<<<grid_stream(c, c->np), NT, 0, c->stream>>>(c->np, 1, c->perm_p, x, c->t);
    launch_schur_spmv(c, c->t, c->z, gate_one(c));
    k_gather_rows<<<grid_stream(c, c->np), NT, 0, c->stream>>>(c->np, 1, c->cmap_p, c->z, y);
  } else {
    launch_schur_spmv(c, x, y, gate_one(c));
  }
  CKL();
  CK(cudaStreamSynchronize(c->stream));
  return leave(c, VEM_OK);
}

int vem_mixed_precond_apply(vem_ctx *h, int32_t kind, const double *v, double *z, int64_t *inner_its) {
  if (!h || !v || !z) return VEM_ERR_INVALID;
  Ctx *c = h->impl;
  if (kind < 0 || kind > 5) return fail(c, VEM_ERR_PRECOND, "unsupported precond_kind %d", kind);
  if (is_block_reg(kind) && !c->has_reg) return fail(c, VEM_ERR_PRECOND, "Block-Reg needs eps > 0");
  int64_t its = 0;
  int r = enter(c);
  if (r) return r;
  if (c->perm) {   // v, z in the caller's numbering (staged through the solve vectors b, x)
    to_internal(c, v, c->b);
    r = enqueue_precond(c, kind, c->b, &c->st->one, c->x, gate_one(c), &its);
    if (r) return leave(c, r);
    from_internal(c, c->x, z, z + c->nu);
  } else {
    r = enqueue_precond(c, kind, v, &c->st->one, z, gate_one(c), &its);
    if (r) return leave(c, r);
  }
  CK(cudaStreamSynchronize(c->stream));
  flush_timing(c);
  if (inner_its) *inner_its = its;
  return leave(c, VEM_OK);
}

int vem_mixed_set_options(vem_ctx *h, const vem_opts *o) {
  if (!h || !o) return VEM_ERR_INVALID;
  Ctx *c = h->impl;
  int r = validate_opts(c, o);
  if (r) return r;
  const bool realloc_v = o->restart != c->opts.restart;
  c->opts = *o;
  destroy_graphs(c);
  {
    int rr = apply_l2_window(c);
    if (rr) return rr;
  }
  if (realloc_v) {
    if (c->V) dfree(c, c->V);
    c->V = nullptr;
    if (c->V32) dfree(c, c->V32);
    c->V32 = nullptr;
    if (c->Z) dfree(c, c->Z);
    c->Z = nullptr;
    c->zcap = 0;
  }
  return VEM_OK;
}

int vem_mixed_get_options(vem_ctx *h, vem_opts *o) {
  if (!h || !o) return VEM_ERR_INVALID;
  *o = h->impl->opts;
  return VEM_OK;
}

int vem_mixed_get_info(vem_ctx *h, vem_info *info) {
  if (!h || !info) return VEM_ERR_INVALID;
  Ctx *c = h->impl;
  info->n_u = c->nu;
  info->n_p = c->np;
  info->nnz_M = c->nnzM;
  info->nnz_B = c->nnzB;
  info->nnz_A = c->nnzA;
  info->nnz_S = c->nnzS;
  info->lambda_max = c->lmax;
  info->eps = c->eps;
  info->spmv_group = 1;      // SELL-32: one row per thread
  info->schur_group = 1;
  info->sm_count = c->sm_count;
  info->device_bytes = c->device_bytes;
  info->l2_window_bytes = (int64_t)c->l2_window_bytes;
  info->amg_levels = (int32_t)c->amg.lv.size();
  info->amg_coarsest = c->amg.lv.empty() ? 0 : c->amg.lv.back().n;
  info->amg_coarse_cluster = c->amg.lv.empty() ? 0 : (int32_t)c->amg.lv.back().vc_ok;
  info->reordered = c->perm ? 1 : 0;
  info->nnz_A_stored = c->nnzA_sell;
  info->nnz_S_stored = c->nnzS_sell;
  return VEM_OK;
}

int vem_mixed_get_schur(vem_ctx *h, int64_t *indptr, int32_t *indices, double *values) {
  if (!h || !indptr || !indices || !values) return VEM_ERR_INVALID;
  Ctx *c = h->impl;
  std::vector<int> rp(c->np + 1);
  CK(cudaMemcpyAsync(rp.data(), c->s_rp, (c->np + 1) * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(indices, c->s_ci, c->nnzS * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(values, c->s_va, c->nnzS * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (long i = 0; i <= c->np; ++i) indptr[i] = rp[i];
  return VEM_OK;
}

int vem_mixed_kernel_stats(vem_ctx *h, vem_kernel_stats *s, int32_t reset) {
  if (!h || !s) return VEM_ERR_INVALID;
  Ctx *c = h->impl;
  if (c->stream) cudaStreamSynchronize(c->stream);
  flush_timing(c);
  *s = c->stats;
  if (reset) memset(&c->stats, 0, sizeof(c->stats));
  return VEM_OK;
}

int vem_mixed_amg_level(vem_ctx *h, int32_t level, int64_t *n, int64_t *nnz) {
  if (!h || !n || !nnz) return VEM_ERR_INVALID;
  Ctx *c = h->impl;
  if (level < 0 || level >= (int)c->amg.lv.size()) return VEM_ERR_INVALID;
  *n = c->amg.lv[level].n;
  *nnz = c->amg.lv[level].nnz;
  return VEM_OK;
}

int vem_mixed_last_cycle_history(vem_ctx *h, double *hist, int32_t cap, int32_t *count) {
  if (!h || !hist || !count || cap < 0) return VEM_ERR_INVALID;
  Ctx *c = h->impl;
  const int k = std::min<int>(c->hist_steps, cap);
  *count = c->hist_steps;
  if (k <= 0 || !(c->hist_bnorm > 0.0)) return VEM_OK;
  std::vector<double> sn(k);
  CK(cudaMemcpy(sn.data(), c->st->sn, k * sizeof(double), cudaMemcpyDeviceToHost));
  double g = c->hist_beta;
  for (int j = 0; j < k; ++j) {   // |g_{j+1}| = |s_j| |g_j| (Givens, O8)
    g *= fabs(sn[j]);
    hist[j] = g / c->hist_bnorm;
  }
  return VEM_OK;
}

int vem_mixed_inner_amg_level(vem_ctx *h, int32_t level, int64_t *n, int64_t *nnz) {
  if (!h || !n || !nnz) return VEM_ERR_INVALID;
  Ctx *c = h->impl;
  if (level < 0 || level >= (int)c->amge.lv.size()) return VEM_ERR_INVALID;
  *n = c->amge.lv[level].n;
  *nnz = c->amge.lv[level].nnz;
  return VEM_OK;
}

void vem_mixed_destroy(vem_ctx *h) {
  if (!h) return;
  destroy_ctx(h->impl);
  delete h;
}

const char *vem_status_string(int s) {
  switch (s) {
    case VEM_OK: return "OK";
    case VEM_NOT_CONVERGED: return "NOT_CONVERGED";
    case VEM_BREAKDOWN: return "BREAKDOWN";
    case VEM_ERR_INVALID: return "ERR_INVALID";
    case VEM_ERR_DIAG_M: return "ERR_DIAG_M";
    case VEM_ERR_DIAG_S: return "ERR_DIAG_S";
    case VEM_ERR_CUDA: return "ERR_CUDA";
    case VEM_ERR_PRECOND: return "ERR_PRECOND";
    case VEM_ERR_INNER: return "ERR_INNER";
    default: return "UNKNOWN";
  }
}

const char *vem_last_error(vem_ctx *h) {
  if (!h) return g_last_err.c_str();   // last failed upload on this thread
  return h->impl->err.c_str();
}

}  // extern "C"
