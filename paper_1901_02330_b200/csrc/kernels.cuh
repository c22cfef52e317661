// kernels.cuh — sm_100a FP64 kernels of the block-preconditioned GMRES hot path.
//
// Every kernel is HBM-bound (0.1-0.25 flop/byte), so there are no
// tensor cores; the design levers are coalescing, one pass over each stream,
// fusion of the vector updates into the sparse products and deterministic
// two-stage reductions (per-block partials + last-block reduce, fixed order).
//
// Paper references (PAPER.md line numbers):
//   saddle operator A = [M B^T; B 0]
//   GMRES (PETSc) -> right-preconditioned GMRES(m)/FGMRES(m)
//   Block-Schur B_1 = diag(M), B_2 = -B diag(M)^-1 B^T
//   Block-Reg  B_1 ~ (M + B^T W^-1 B)^-1, B_2 = W^-1
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

#define VEM_MAXM 128
#define VEM_DOT_CHUNK 8

struct GmresState {
  int active;      // Arnoldi steps of the current cycle proceed while 1
  int j;           // steps done in the current cycle
  int its;         // total Arnoldi steps
  int maxit;
  int conv_est;    // |g_{j+1}| <= tol_abs
  int breakdown;   // h_{j+1,j} <= 1e-14 ||A z_j||
  int conv_true;   // ||b - A x|| <= tol_abs at the last cycle end
  int m;
  int flexible;
  int has_steps;   // gate for the cycle-end kernels
  int pad0, pad1;
  double bnorm, tol_abs, beta, est, true_res, wnorm0;
};

struct PcgState {
  int active, its, maxit, failed;
  double rz, alpha, beta, bn, tol_abs, rr;
};

// PCG on K = M + B^T (eps W)^-1 B (precond kind 5, blockreg_m.cuh)
struct KState {
  int active, its, maxit, failed;
  double rz, rz0, alpha, beta, rtol;
};

struct DevState {
  GmresState g;
  PcgState p;
  int one_i;       // constant 1 (always-open gate)
  int pad;
  double one;      // constant 1.0 (unit scale)
  double H[(VEM_MAXM + 1) * VEM_MAXM];   // column-major, leading dim m+1
  double cs[VEM_MAXM], sn[VEM_MAXM], gv[VEM_MAXM + 1];
  double h1[VEM_MAXM + 2], coef[VEM_MAXM + 2], vscale[VEM_MAXM + 1], y[VEM_MAXM];
  double lmax;
  int setup_err;
  int pad2;
  KState k;
};

// ---------------------------------------------------------------------------
// reduction helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Sum NV per-thread values over the block; result valid in thread 0 (out[i]).
template <int NV>
__device__ __forceinline__ void block_sum_n(double (&v)[NV], double *sh /* >= 32*NV */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) sh[warp * NV + i] = v[i];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double t = lane < nw ? sh[lane * NV + i] : 0.0;
      v[i] = warp_sum(t);
    }
  }
  __syncthreads();
}

// Last-block election after every block stored its partials (threadfence
// reduction pattern).  Returns true in every thread of the last block.
__device__ __forceinline__ bool elect_last_block(unsigned *counter) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned total = gridDim.x * gridDim.y;
    unsigned t = atomicAdd(counter, 1u);
    s_last = (t == total - 1);
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

// In the last block: out[o] = sum over blocks b < nb of part[(o / C) * nb * C + b * C + o % C]
// for o < nout (fixed order: lane-strided then xor tree => deterministic).
template <int C>
__device__ void reduce_partials(const double *part, int nb, int nout, double *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int o = warp; o < nout; o += nw) {
    const double *base = part + (size_t)(o / C) * nb * C + (o % C);
    double s = 0.0;
    for (int b = lane; b < nb; b += 32) s += __ldcg(base + (size_t)b * C);
    s = warp_sum(s);
    if (lane == 0) out[o] = s;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// SELL-32 sparse format (sliced ELLPACK, slice height 32 = one warp, sigma = 1:
// rows keep their order).  Slice s holds rows [32 s, 32 s + 32); entry j of
// row r sits at soff[s] + 32 j + (r & 31), so the 32 lanes of a warp read 32
// consecutive doubles (256 B) and 32 consecutive int32 columns per step:
// fully coalesced, one row per thread, no shuffles.  Rows shorter than the
// slice width are padded with (col = a valid column of the row, val = 0).
// ---------------------------------------------------------------------------
struct Sell {
  const long long *__restrict__ soff;
  const int *__restrict__ ci;
  const double *__restrict__ va;
  const int *__restrict__ perm;   // slot -> row (rows sorted by length in windows); nullptr: identity.
                                  // Only S_D at k >= 1 carries one (k_spmv, k_cheb_resid, k_pcg_spmv_p).
};
__device__ __forceinline__ long sell_row(const Sell &A, long slot) { return A.perm ? (long)A.perm[slot] : slot; }

// The matrix stream (values, column indices: read once per pass) uses __ldcs (evict-first).
// Tried and rejected (R2_06): L1::no_allocate for the stream, to keep the gathered sectors of x in
// L1: C5 fine-level pass 4.64 -> 4.11 TB/s, C3 solve 143.5 -> 157.5 ms.
template <typename Gather>
__device__ __forceinline__ double sell_dot(const Sell &A, long row, Gather g) {
  const long s = row >> 5;
  const int lane = (int)(row & 31);
  const long long b = A.soff[s];
  const int w = (int)((A.soff[s + 1] - b) >> 5);
  const int *__restrict__ c = A.ci + b + lane;
  const double *__restrict__ v = A.va + b + lane;
  double acc = 0.0;
#pragma unroll 4
  for (int j = 0; j < w; ++j) acc = fma(__ldcs(v + ((long)j << 5)), g(__ldcs(c + ((long)j << 5))), acc);
  return acc;
}

struct GatherX {
  const double *__restrict__ x;
  __device__ __forceinline__ double operator()(int c) const { return __ldg(x + c); }
};

// y[r] = (A x)[r] (mode 0) or b[r] - (A x)[r] (mode 1), rows [row0, row0 + nrows)
__global__ void __launch_bounds__(256) k_spmv(long row0, long nrows, Sell A, const double *__restrict__ x,
                                              double *__restrict__ y, const double *__restrict__ b, int mode,
                                              const int *gate) {
  if (!*gate) return;
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrows) return;
  const long slot = row0 + t;
  const long row = sell_row(A, slot);
  const double acc = sell_dot(A, slot, GatherX{x});
  y[row] = mode ? b[row] - acc : acc;
}

// Residual r = b - A x written to V0 with ||r||^2 partials; the last block
// starts a new GMRES cycle: beta = ||r||, vscale_0 = 1/beta, g = (beta, 0, ..).
__global__ void __launch_bounds__(256) k_residual_start(long n, Sell A, const double *__restrict__ x,
                                                        const double *__restrict__ b, double *__restrict__ r,
                                                        int use_x, double *part, unsigned *counter,
                                                        DevState *st) {
  __shared__ double sh[32];
  const long row = (long)blockIdx.x * blockDim.x + threadIdx.x;
  double v[1] = {0.0};
  if (row < n) {
    const double acc = use_x ? sell_dot(A, row, GatherX{x}) : 0.0;
    const double rv = b[row] - acc;
    r[row] = rv;
    v[0] = rv * rv;
  }
  block_sum_n<1>(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
  if (elect_last_block(counter)) {
    __shared__ double tot;
    reduce_partials<1>(part, gridDim.x, 1, &tot);
    if (threadIdx.x == 0) {
      GmresState &g = st->g;
      const double beta = sqrt(tot);
      if (!use_x) {               // first cycle: ||b||
        g.bnorm = beta;
      }
      g.beta = beta;
      g.true_res = beta;
      g.conv_true = beta <= g.tol_abs ? 1 : 0;
      g.j = 0;
      g.conv_est = 0;
      g.breakdown = 0;
      g.has_steps = 0;
      g.active = (g.conv_true || g.its >= g.maxit) ? 0 : 1;
      st->vscale[0] = beta > 0.0 ? 1.0 / beta : 0.0;
      st->gv[0] = beta;
      *counter = 0u;
    }
  }
}

// CSR -> SELL-32 conversion (upload only)
// SELL-C-sigma (C = 32): slot r of the stored matrix holds CSR row perm[r]
// (perm == nullptr: identity) with its columns renumbered through cmap
// (cmap == nullptr: unchanged), so a symmetric reordering that sorts rows by
// length inside sigma-row windows (upload_impl) removes the slice padding.
__global__ void k_sell_width(long nrows, const int *__restrict__ rp, const int *__restrict__ perm,
                             long long *__restrict__ wslice) {
  const long nsl = (nrows + 31) / 32;
  for (long s = (long)blockIdx.x * blockDim.x + threadIdx.x; s < nsl; s += (long)gridDim.x * blockDim.x) {
    int w = 0;
    for (long r = s * 32; r < s * 32 + 32 && r < nrows; ++r) {
      const long o = perm ? perm[r] : r;
      w = max(w, rp[o + 1] - rp[o]);
    }
    wslice[s] = 32LL * w;
  }
}
__global__ void k_sell_fill(long nrows, const int *__restrict__ rp, const int *__restrict__ ci,
                            const double *__restrict__ va, const int *__restrict__ perm,
                            const int *__restrict__ cmap, const long long *__restrict__ soff,
                            int *__restrict__ sci, double *__restrict__ sva) {
  const long nsl = (nrows + 31) / 32;
  for (long r = (long)blockIdx.x * blockDim.x + threadIdx.x; r < nsl * 32; r += (long)gridDim.x * blockDim.x) {
    const long s = r >> 5;
    const int lane = (int)(r & 31);
    const long long b = soff[s];
    const int w = (int)((soff[s + 1] - b) >> 5);
    const long o = r < nrows ? (perm ? perm[r] : r) : 0;
    const int st = r < nrows ? rp[o] : 0, len = r < nrows ? rp[o + 1] - rp[o] : 0;
    const int padc = len > 0 ? ci[st + len - 1] : 0;
    for (int j = 0; j < w; ++j) {
      const long long q = b + 32LL * j + lane;
      const int col = j < len ? ci[st + j] : padc;
      sci[q] = cmap ? cmap[col] : col;
      sva[q] = j < len ? va[st + j] : 0.0;
    }
  }
}
// first element touching velocity row i of the merged A (its B^T columns >= nu): the
// element-major key of the SELL-C-sigma velocity order
__global__ void k_first_elem(long nu, const int *__restrict__ rp, const int *__restrict__ ci, int nb,
                             int *__restrict__ elem) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nu; i += (long)gridDim.x * blockDim.x) {
    int m = 0x7fffffff;
    for (int k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] >= nu) m = min(m, (int)((ci[k] - nu) / nb));
    elem[i] = m;
  }
}
// out[i w + b] = in[perm[i] w + b]  (row gather of a row-major n x w array)
__global__ void k_gather_rows(long n, int w, const int *__restrict__ perm, const double *__restrict__ in,
                              double *__restrict__ out) {
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < n * w; t += (long)gridDim.x * blockDim.x) {
    const long i = t / w;
    out[t] = in[(long)perm[i] * w + (t - i * w)];
  }
}
// out[perm[i]] = in[i] for i < n, split at nu into out0 (rows < nu) and out1
__global__ void k_scatter_split(long n, long nu, const int *__restrict__ perm, const double *__restrict__ in,
                                double *__restrict__ out0, double *__restrict__ out1) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const long o = perm[i];
    if (o < nu)
      out0[o] = in[i];
    else
      out1[o - nu] = in[i];
  }
}

// ---------------------------------------------------------------------------
// Block-Schur apply:  z_u = s v_u ./ diag(M);
// z_p = -C_d(S_D) (s v_p): degree-d Jacobi Chebyshev (Saad Alg. 12.1, x0 = 0)
// init: r = s v_p, d = D^-1 r / theta, x = d   (degree 1: z_p = -d)
// ---------------------------------------------------------------------------
__global__ void k_bs_init(long nu, long np, const double *__restrict__ v, const double *scale,
                          const double *__restrict__ dMinv, const double *__restrict__ dSinv,
                          double inv_theta, double *__restrict__ z, double *__restrict__ cr,
                          double *__restrict__ cd, double *__restrict__ cx, int degree1, int blockmode,
                          const int *gate) {
  if (!*gate) return;
  const double s = *scale;
  const long n = nu + np;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    if (i < nu) {
      z[i] = dMinv ? s * v[i] * dMinv[i] : s * v[i];
    } else if (blockmode) {
      cr[i - nu] = s * v[i];
    } else {
      const long k = i - nu;
      const double r = s * v[i];
      const double d = dSinv[k] * r * inv_theta;
      if (degree1) {
        z[i] = -d;
      } else {
        cr[k] = r;
        cd[k] = d;
        cx[k] = d;
      }
    }
  }
}

// Block-Schur apply, first Chebyshev step fused with the init (k = 0 path):
// rows < nu:  z_u = s v_u ./ diag(M);  rows >= nu (pressure row k):
//   d0 = D^-1 (s v_p) / theta (recomputed at every gathered column),
//   r1 = s v_p - S d0;  d1 = c1 d0 + c2 D^-1 r1;  x = d0 + d1   (last: z_p = -x)
struct GatherD0 {
  const double *__restrict__ vp, *__restrict__ dinv;
  double f;  // s / theta
  __device__ __forceinline__ double operator()(int c) const { return dinv[c] * vp[c] * f; }
};
__global__ void __launch_bounds__(256) k_cheb_first(long nu, long np, Sell S, const double *__restrict__ v,
                                                    const double *scale, const double *__restrict__ dMinv,
                                                    const double *__restrict__ dSinv, double inv_theta, double c1,
                                                    double c2, double *__restrict__ r, double *__restrict__ d_new,
                                                    double *__restrict__ x, double *__restrict__ z, int last,
                                                    const int *gate) {
  if (!*gate) return;
  const double s = *scale;
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nu) {
    z[i] = s * v[i] * dMinv[i];
    return;
  }
  const long row = i - nu;
  if (row >= np) return;
  const double *vp = v + nu;
  const double f = s * inv_theta;
  const double sd = sell_dot(S, row, GatherD0{vp, dSinv, f});
  const double r0 = s * vp[row];
  const double d0 = dSinv[row] * r0 * inv_theta;
  const double rn = r0 - sd;
  const double dn = c1 * d0 + c2 * (dSinv[row] * rn);
  const double xn = d0 + dn;
  if (last) {
    z[nu + row] = -xn;
  } else {
    r[row] = rn;
    d_new[row] = dn;
    x[row] = xn;
  }
}

// one Chebyshev step:  r -= S d_old;  d_new = c1 d_old + c2 D^-1 r;  x += d_new
// last step writes z_p = -(x + d_new) instead of x.
__global__ void __launch_bounds__(256) k_cheb_step(long np, Sell S, const double *__restrict__ dSinv,
                                                   double *__restrict__ r, const double *__restrict__ d_old,
                                                   double *__restrict__ d_new, double *__restrict__ x, double c1,
                                                   double c2, int last, double *__restrict__ zp, const int *gate) {
  if (!*gate) return;
  const long row = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= np) return;
  const double sd = sell_dot(S, row, GatherX{d_old});
  const double rn = r[row] - sd;
  const double dn = c1 * d_old[row] + c2 * (dSinv[row] * rn);
  const double xn = x[row] + dn;
  if (last) {
    zp[row] = -xn;
  } else {
    r[row] = rn;
    d_new[row] = dn;
    x[row] = xn;
  }
}

// ---------------------------------------------------------------------------
// Block-Reg apply, W diagonal (wdiag == nullptr -> identity):
//   z_p = s v_p / (eps W);  t0 = s v_u ./ diag(M) -> z_u;  rhs = B t0 (k_spmv on B rows)
//   t = PCG(S_D + eps W, rhs);  z_u = t0 - diag(M)^-1 B^T t
// ---------------------------------------------------------------------------
__global__ void k_br_init(long nu, long np, const double *__restrict__ v, const double *scale,
                          const double *__restrict__ dMinv, const double *__restrict__ wdiag, double inv_eps,
                          double *__restrict__ z, const int *gate) {
  if (!*gate) return;
  const double s = *scale;
  const long n = nu + np;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    if (i < nu) {
      z[i] = s * v[i] * dMinv[i];
    } else {
      const double w = wdiag ? wdiag[i - nu] : 1.0;
      z[i] = s * v[i] * inv_eps / w;
    }
  }
}

// z_u[i] -= dMinv[i] * sum_{k in row i, col >= nu} A_ik t[col - nu]   (B^T t)
struct GatherBt {
  long nu;
  const double *__restrict__ tp;
  __device__ __forceinline__ double operator()(int c) const { return c >= nu ? tp[c - nu] : 0.0; }
};
__global__ void __launch_bounds__(256) k_br_finish(long nu, Sell A, const double *__restrict__ dMinv,
                                                   const double *__restrict__ tp, double *__restrict__ z,
                                                   const int *gate) {
  if (!*gate) return;
  const long row = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= nu) return;
  z[row] -= dMinv[row] * sell_dot(A, row, GatherBt{nu, tp});
}

// PCG init: x = 0, r = b, p_prev = 0, beta = 0; rz = r.D^-1 r, bn = ||b||
__global__ void k_pcg_init(long n, const double *__restrict__ b, const double *__restrict__ dinv,
                           double *__restrict__ x, double *__restrict__ r, double *__restrict__ p0,
                           double *part, unsigned *counter, DevState *st, double rtol, int maxit,
                           const int *gate) {
  __shared__ double sh[64];
  const bool on = *gate != 0;
  double v[2] = {0.0, 0.0};
  if (on) {
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
      const double bi = b[i];
      x[i] = 0.0;
      r[i] = bi;
      p0[i] = 0.0;
      v[0] += bi * dinv[i] * bi;
      v[1] += bi * bi;
    }
  }
  block_sum_n<2>(v, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x * 2 + 0] = v[0];
    part[blockIdx.x * 2 + 1] = v[1];
  }
  if (elect_last_block(counter)) {
    __shared__ double tot[2];
    reduce_partials<2>(part, gridDim.x, 2, tot);
    if (threadIdx.x == 0) {
      PcgState &p = st->p;
      p.rz = tot[0];
      p.bn = sqrt(tot[1]);
      p.tol_abs = rtol * p.bn;
      p.beta = 0.0;
      p.its = 0;
      p.maxit = maxit;
      p.failed = 0;
      p.active = (on && p.bn > 0.0) ? 1 : 0;
      *counter = 0u;
    }
  }
}

// PCG step part 1: p_new = D^-1 r + beta p_prev (on the fly at every gathered
// column), q = (S + eps W) p_new, partial p_new . q; last block: alpha = rz / pq
struct GatherPcg {
  double beta;
  const double *__restrict__ p_prev, *__restrict__ dinv, *__restrict__ r;
  __device__ __forceinline__ double operator()(int c) const { return fma(beta, p_prev[c], dinv[c] * r[c]); }
};
__global__ void __launch_bounds__(256) k_pcg_spmv(long n, Sell S, const double *__restrict__ dinv,
                                                  const double *__restrict__ wdiag, double eps,
                                                  const double *__restrict__ r, const double *__restrict__ p_prev,
                                                  double *__restrict__ p_new, double *__restrict__ q, double *part,
                                                  unsigned *counter, DevState *st) {
  __shared__ double sh[32];
  if (!st->p.active) return;
  const double beta = st->p.beta;
  const long row = (long)blockIdx.x * blockDim.x + threadIdx.x;
  double v[1] = {0.0};
  if (row < n) {
    const double acc = sell_dot(S, row, GatherPcg{beta, p_prev, dinv, r});
    const double pi = fma(beta, p_prev[row], dinv[row] * r[row]);
    const double w = wdiag ? wdiag[row] : 1.0;
    const double qi = fma(eps * w, pi, acc);
    p_new[row] = pi;
    q[row] = qi;
    v[0] += pi * qi;
  }
  block_sum_n<1>(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
  if (elect_last_block(counter)) {
    __shared__ double tot;
    reduce_partials<1>(part, gridDim.x, 1, &tot);
    if (threadIdx.x == 0) {
      st->p.alpha = st->p.rz / tot;
      *counter = 0u;
    }
  }
}

// PCG step part 2: x += alpha p; r -= alpha q; partial r.D^-1 r and r.r;
// last block: its++, convergence ||r|| <= rtol ||b||, beta = rz_new / rz
__global__ void k_pcg_vec(long n, const double *__restrict__ dinv, const double *__restrict__ p,
                          const double *__restrict__ q, double *__restrict__ x, double *__restrict__ r,
                          double *part, unsigned *counter, DevState *st) {
  __shared__ double sh[64];
  if (!st->p.active) return;
  const double alpha = st->p.alpha;
  double v[2] = {0.0, 0.0};
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    v[0] += ri * dinv[i] * ri;
    v[1] += ri * ri;
  }
  block_sum_n<2>(v, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x * 2 + 0] = v[0];
    part[blockIdx.x * 2 + 1] = v[1];
  }
  if (elect_last_block(counter)) {
    __shared__ double tot[2];
    reduce_partials<2>(part, gridDim.x, 2, tot);
    if (threadIdx.x == 0) {
      PcgState &p = st->p;
      p.its += 1;
      p.rr = tot[1];
      if (sqrt(tot[1]) <= p.tol_abs) {
        p.active = 0;
      } else if (p.its >= p.maxit) {
        p.active = 0;
        p.failed = 1;
      } else {
        p.beta = tot[0] / p.rz;
        p.rz = tot[0];
      }
      *counter = 0u;
    }
  }
}

// ---------------------------------------------------------------------------
// CGS2 Arnoldi (batched classical Gram-Schmidt, applied twice)
// ---------------------------------------------------------------------------
// partial dots: out index o < nv: V_o . w ; o == nv (if with_norm): w . w.
// grid (gx, ceil(nout / 8)); part layout [chunk][block][8]
// grid (nblk, nchunks): block b of chunk y dots basis vectors 8y..8y+7 with w
// over a grid-stride slice of the rows.
__global__ void __launch_bounds__(256) k_mdot(long n, const double *__restrict__ V, long ldv, int nv,
                                              int with_norm, const double *__restrict__ w, double *part,
                                              unsigned *counter, DevState *st, int pass) {
  __shared__ double sh[32 * VEM_DOT_CHUNK];
  if (!st->g.active) return;
  const int nout = nv + (with_norm ? 1 : 0);
  const int c0 = blockIdx.y * VEM_DOT_CHUNK;
  const int nb = gridDim.x, b = blockIdx.x;
  double acc[VEM_DOT_CHUNK];
#pragma unroll
  for (int c = 0; c < VEM_DOT_CHUNK; ++c) acc[c] = 0.0;
  const double *vp[VEM_DOT_CHUNK];
#pragma unroll
  for (int c = 0; c < VEM_DOT_CHUNK; ++c) {
    const int o = c0 + c;
    vp[c] = (o < nv) ? V + (size_t)o * ldv : w;
  }
  for (long i = (long)b * blockDim.x + threadIdx.x; i < n; i += (long)nb * blockDim.x) {
    const double wi = w[i];
#pragma unroll
    for (int c = 0; c < VEM_DOT_CHUNK; ++c)
      if (c0 + c < nout) acc[c] = fma(vp[c][i], wi, acc[c]);
  }
  block_sum_n<VEM_DOT_CHUNK>(acc, sh);
  if (threadIdx.x == 0) {
    double *dst = part + ((size_t)blockIdx.y * nb + b) * VEM_DOT_CHUNK;
#pragma unroll
    for (int c = 0; c < VEM_DOT_CHUNK; ++c) dst[c] = acc[c];
  }
  if (elect_last_block(counter)) {
    __shared__ double tot[VEM_MAXM + 2];
    reduce_partials<VEM_DOT_CHUNK>(part, nb, nout, tot);
    if (threadIdx.x == 0) {
      for (int o = 0; o < nv; ++o) {
        const double h = st->vscale[o] * tot[o];
        st->coef[o] = h * st->vscale[o];
        st->h1[o] = (pass == 1) ? h : st->h1[o] + h;
      }
      if (with_norm) st->g.wnorm0 = sqrt(tot[nv]);
      *counter = 0u;
    }
  }
}


// Givens step for column j, executed by one thread.
__device__ void givens_column(DevState *st, int j, double hn) {
  GmresState &g = st->g;
  const int ld = g.m + 1;
  double *Hc = st->H + (size_t)j * ld;
  for (int i = 0; i <= j; ++i) Hc[i] = st->h1[i];
  Hc[j + 1] = hn;
  for (int i = 0; i < j; ++i) {
    const double t = st->cs[i] * Hc[i] + st->sn[i] * Hc[i + 1];
    Hc[i + 1] = -st->sn[i] * Hc[i] + st->cs[i] * Hc[i + 1];
    Hc[i] = t;
  }
  const double rr = hypot(Hc[j], Hc[j + 1]);
  st->cs[j] = Hc[j] / rr;
  st->sn[j] = Hc[j + 1] / rr;
  Hc[j] = rr;
  Hc[j + 1] = 0.0;
  st->gv[j + 1] = -st->sn[j] * st->gv[j];
  st->gv[j] = st->cs[j] * st->gv[j];
  g.est = fabs(st->gv[j + 1]);
  g.its += 1;
  g.j = j + 1;
  g.has_steps = 1;
  st->vscale[j + 1] = 1.0 / hn;
  if (fabs(st->gv[j + 1]) <= g.tol_abs) {
    g.conv_est = 1;
    g.active = 0;
  } else if (hn <= 1e-14 * g.wnorm0) {
    g.breakdown = 1;
    g.active = 0;
  } else if (g.its >= g.maxit || j + 1 >= g.m) {
    g.active = 0;
  }
}

// w -= sum_{o < nv} coef_o V_o; optionally ||w||^2 partials and, in the last
// block, the Givens step of column j.
__global__ void __launch_bounds__(256) k_update(long n, const double *__restrict__ V, long ldv, int nv,
                                                double *__restrict__ w, int with_norm, double *part,
                                                unsigned *counter, DevState *st, int j) {
  __shared__ double sh[32];
  __shared__ double cf[VEM_MAXM + 1];
  if (!st->g.active) return;
  for (int o = threadIdx.x; o < nv; o += blockDim.x) cf[o] = st->coef[o];
  __syncthreads();
  double v[1] = {0.0};
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    double wi = w[i];
    for (int o = 0; o < nv; ++o) wi = fma(-cf[o], V[(size_t)o * ldv + i], wi);
    w[i] = wi;
    v[0] += wi * wi;
  }
  if (!with_norm) return;
  block_sum_n<1>(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
  if (elect_last_block(counter)) {
    __shared__ double tot;
    reduce_partials<1>(part, gridDim.x, 1, &tot);
    if (threadIdx.x == 0) {
      givens_column(st, j, sqrt(tot));
      *counter = 0u;
    }
  }
}

// ---------------------------------------------------------------------------
// Compressed Krylov basis (opts.basis_f32: traffic-reduced Krylov):
// every basis vector is the float32 rounding of the vector Arnoldi produced.  V (FP64) keeps
// the rounded values for its other readers (preconditioner input, SpMV, k_combine), V32 is
// the float copy the CGS kernels stream: 4 bytes per basis entry instead of 8.  Same
// arithmetic as k_mdot / k_update otherwise (FP64 accumulation, same reductions).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_mdot32(long n, const float *__restrict__ V32, long ldv, int nv,
                                                int with_norm, const double *__restrict__ w, double *part,
                                                unsigned *counter, DevState *st, int pass) {
  __shared__ double sh[32 * VEM_DOT_CHUNK];
  if (!st->g.active) return;
  const int nout = nv + (with_norm ? 1 : 0);
  const int c0 = blockIdx.y * VEM_DOT_CHUNK;
  const int nb = gridDim.x, b = blockIdx.x;
  double acc[VEM_DOT_CHUNK];
#pragma unroll
  for (int c = 0; c < VEM_DOT_CHUNK; ++c) acc[c] = 0.0;
  const float *vp[VEM_DOT_CHUNK];
#pragma unroll
  for (int c = 0; c < VEM_DOT_CHUNK; ++c) vp[c] = V32 + (size_t)min(c0 + c, nv - 1) * ldv;
  // two consecutive entries per thread (float2 / double2 loads: 8 bytes per basis vector and
  // thread in flight, as in the FP64 kernel); ldv and the vectors are 1 KB-aligned
  const long n2 = n >> 1;
  const int nvc = min(VEM_DOT_CHUNK, nv - c0);              // basis vectors of this chunk (block-uniform)
  const bool has_norm = with_norm && nv >= c0 && nv < c0 + VEM_DOT_CHUNK;   // the w.w slot lives here
  double accn = 0.0;
  for (long i = (long)b * blockDim.x + threadIdx.x; i < n2; i += (long)nb * blockDim.x) {
    const double2 wi = reinterpret_cast<const double2 *>(w)[i];
    float2 vv[VEM_DOT_CHUNK];
#pragma unroll
    for (int c = 0; c < VEM_DOT_CHUNK; ++c)
      if (c < nvc) vv[c] = reinterpret_cast<const float2 *>(vp[c])[i];
#pragma unroll
    for (int c = 0; c < VEM_DOT_CHUNK; ++c)
      if (c < nvc) acc[c] = fma((double)vv[c].y, wi.y, fma((double)vv[c].x, wi.x, acc[c]));
    if (has_norm) accn = fma(wi.y, wi.y, fma(wi.x, wi.x, accn));
  }
  if ((n & 1) && b == 0 && threadIdx.x == 0) {   // odd tail
    const double wi = w[n - 1];
#pragma unroll
    for (int c = 0; c < VEM_DOT_CHUNK; ++c)
      if (c < nvc) acc[c] = fma((double)vp[c][n - 1], wi, acc[c]);
    if (has_norm) accn = fma(wi, wi, accn);
  }
  if (has_norm) {
#pragma unroll
    for (int c = 0; c < VEM_DOT_CHUNK; ++c)
      if (c0 + c == nv) acc[c] = accn;
  }
  block_sum_n<VEM_DOT_CHUNK>(acc, sh);
  if (threadIdx.x == 0) {
    double *dst = part + ((size_t)blockIdx.y * nb + b) * VEM_DOT_CHUNK;
#pragma unroll
    for (int c = 0; c < VEM_DOT_CHUNK; ++c) dst[c] = acc[c];
  }
  if (elect_last_block(counter)) {
    __shared__ double tot[VEM_MAXM + 2];
    reduce_partials<VEM_DOT_CHUNK>(part, nb, nout, tot);
    if (threadIdx.x == 0) {
      for (int o = 0; o < nv; ++o) {
        const double h = st->vscale[o] * tot[o];
        st->coef[o] = h * st->vscale[o];
        st->h1[o] = (pass == 1) ? h : st->h1[o] + h;
      }
      if (with_norm) st->g.wnorm0 = sqrt(tot[nv]);
      *counter = 0u;
    }
  }
}

// w -= sum coef_o V32_o; the final pass (with_norm) rounds w to float32, stores the float copy as
// basis vector j + 1 and takes the norm of the ROUNDED vector (h_{j+1,j} = ||fl32(w)||)
__global__ void __launch_bounds__(256) k_update32(long n, const float *__restrict__ V32, long ldv, int nv,
                                                  double *__restrict__ w, float *__restrict__ w32, int with_norm,
                                                  double *part, unsigned *counter, DevState *st, int j) {
  __shared__ double sh[32];
  __shared__ double cf[VEM_MAXM + 1];
  if (!st->g.active) return;
  for (int o = threadIdx.x; o < nv; o += blockDim.x) cf[o] = st->coef[o];
  __syncthreads();
  double v[1] = {0.0};
  const long n2 = n >> 1;   // two consecutive entries per thread (float2 / double2)
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
    double2 wi = reinterpret_cast<double2 *>(w)[i];
    for (int o = 0; o < nv; ++o) {
      const float2 vv = reinterpret_cast<const float2 *>(V32 + (size_t)o * ldv)[i];
      wi.x = fma(-cf[o], (double)vv.x, wi.x);
      wi.y = fma(-cf[o], (double)vv.y, wi.y);
    }
    if (with_norm) {
      const float2 wf = make_float2((float)wi.x, (float)wi.y);
      reinterpret_cast<float2 *>(w32)[i] = wf;
      wi = make_double2((double)wf.x, (double)wf.y);
    }
    reinterpret_cast<double2 *>(w)[i] = wi;
    v[0] += wi.x * wi.x + wi.y * wi.y;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {   // odd tail
    double wi = w[n - 1];
    for (int o = 0; o < nv; ++o) wi = fma(-cf[o], (double)V32[(size_t)o * ldv + n - 1], wi);
    if (with_norm) {
      const float wf = (float)wi;
      w32[n - 1] = wf;
      wi = (double)wf;
    }
    w[n - 1] = wi;
    v[0] += wi * wi;
  }
  if (!with_norm) return;
  block_sum_n<1>(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
  if (elect_last_block(counter)) {
    __shared__ double tot;
    reduce_partials<1>(part, gridDim.x, 1, &tot);
    if (threadIdx.x == 0) {
      givens_column(st, j, sqrt(tot));
      *counter = 0u;
    }
  }
}

// first basis vector of a cycle: r -> fl32(r) in place, float copy to V32_0 (beta stays ||r||)
__global__ void k_round_basis(long n, double *__restrict__ v, float *__restrict__ v32) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const float f = (float)v[i];
    v32[i] = f;
    v[i] = (double)f;
  }
}

// y = R^-1 g (back substitution on the rotated Hessenberg), coef_i = y_i * scale_i
__global__ void k_backsolve(DevState *st, int use_vscale) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  GmresState &g = st->g;
  const int k = g.j;
  const int ld = g.m + 1;
  for (int i = k - 1; i >= 0; --i) {
    double s = st->gv[i];
    for (int c = i + 1; c < k; ++c) s -= st->H[(size_t)c * ld + i] * st->y[c];
    st->y[i] = s / st->H[(size_t)i * ld + i];
  }
  for (int i = 0; i < k; ++i) st->coef[i] = use_vscale ? st->y[i] * st->vscale[i] : st->y[i];
}

// out (+)= sum_{o < k} coef_o X_o, k = st->g.j
__global__ void __launch_bounds__(256) k_combine(long n, const double *__restrict__ X, long ldx,
                                                 double *__restrict__ out, int accumulate, DevState *st) {
  __shared__ double cf[VEM_MAXM];
  const int k = st->g.j;
  if (k == 0) return;
  for (int o = threadIdx.x; o < k; o += blockDim.x) cf[o] = st->coef[o];
  __syncthreads();
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    double s = accumulate ? out[i] : 0.0;
    for (int o = 0; o < k; ++o) s = fma(cf[o], X[(size_t)o * ldx + i], s);
    out[i] = s;
  }
}

__global__ void k_axpy_gated(long n, const double *__restrict__ z, double *__restrict__ x, const int *gate) {
  if (!*gate) return;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    x[i] += z[i];
}

// ---------------------------------------------------------------------------
// setup kernels (upload)
// ---------------------------------------------------------------------------
// count B entries per column (for B^T)
__global__ void k_count_cols(long nnz, const int *__restrict__ ci, int *__restrict__ cnt) {
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (long)gridDim.x * blockDim.x)
    atomicAdd(cnt + ci[k], 1);
}
// scatter B (rows p, cols u) into B^T rows (u) with atomic slots; sorted later
__global__ void k_scatter_T(long nrows, const int *__restrict__ rp, const int *__restrict__ ci,
                            const double *__restrict__ va, const int *__restrict__ trp, int *__restrict__ fill,
                            int *__restrict__ tci, double *__restrict__ tva) {
  for (long r = (long)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (long)gridDim.x * blockDim.x) {
    for (int k = rp[r]; k < rp[r + 1]; ++k) {
      const int c = ci[k];
      const int slot = trp[c] + atomicAdd(fill + c, 1);
      tci[slot] = (int)r;
      tva[slot] = va[k];
    }
  }
}
// insertion sort of each (short) row by column index: deterministic B^T
__global__ void k_sort_rows(long nrows, const int *__restrict__ rp, int *__restrict__ ci, double *__restrict__ va) {
  for (long r = (long)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (long)gridDim.x * blockDim.x) {
    const int s = rp[r], e = rp[r + 1];
    for (int a = s + 1; a < e; ++a) {
      const int key = ci[a];
      const double val = va[a];
      int b = a - 1;
      while (b >= s && ci[b] > key) {
        ci[b + 1] = ci[b];
        va[b + 1] = va[b];
        --b;
      }
      ci[b + 1] = key;
      va[b + 1] = val;
    }
  }
}
// merged saddle-matrix row lengths: velocity rows = M row + B^T row, pressure rows = B row
__global__ void k_a_rowlen(long nu, long np, const int64_t *__restrict__ mrp, const int *__restrict__ btrp,
                           const int64_t *__restrict__ brp, int *__restrict__ len) {
  const long n = nu + np;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    if (i < nu)
      len[i] = (int)(mrp[i + 1] - mrp[i]) + (btrp[i + 1] - btrp[i]);
    else
      len[i] = (int)(brp[i - nu + 1] - brp[i - nu]);
  }
}
__global__ void k_a_fill(long nu, long np, const int64_t *__restrict__ mrp, const int *__restrict__ mci,
                         const double *__restrict__ mva, const int *__restrict__ btrp, const int *__restrict__ btci,
                         const double *__restrict__ btva, const int64_t *__restrict__ brp,
                         const int *__restrict__ bci, const double *__restrict__ bva, const int *__restrict__ arp,
                         int *__restrict__ aci, double *__restrict__ ava) {
  const long n = nu + np;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    int o = arp[i];
    if (i < nu) {
      for (int64_t k = mrp[i]; k < mrp[i + 1]; ++k, ++o) {
        aci[o] = mci[k];
        ava[o] = mva[k];
      }
      for (int k = btrp[i]; k < btrp[i + 1]; ++k, ++o) {
        aci[o] = (int)(nu + btci[k]);
        ava[o] = btva[k];
      }
    } else {
      const long r = i - nu;
      for (int64_t k = brp[r]; k < brp[r + 1]; ++k, ++o) {
        aci[o] = bci[k];
        ava[o] = bva[k];
      }
    }
  }
}
// diag(M)^-1 from the merged rows; flags non-positive diagonals
__global__ void k_diag_inv(long n, const int *__restrict__ rp, const int *__restrict__ ci,
                           const double *__restrict__ va, long col_off, double *__restrict__ dinv,
                           double *__restrict__ diag, int *err) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    double d = 0.0;
    for (int k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] == i + col_off) d = va[k];
    if (diag) diag[i] = d;
    if (!(d > 0.0)) {
      atomicExch(err, 1);
      dinv[i] = 0.0;
    } else {
      dinv[i] = 1.0 / d;
    }
  }
}
// S_D expansion counts: cnt[i] = sum_{k in B row i} |B^T row col_k|
__global__ void k_spgemm_count(long r0, long nr, const int64_t *__restrict__ brp, const int *__restrict__ bci,
                               const int *__restrict__ btrp, int64_t *__restrict__ cnt) {
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < nr; t += (long)gridDim.x * blockDim.x) {
    const long i = r0 + t;
    int64_t c = 0;
    for (int64_t k = brp[i]; k < brp[i + 1]; ++k) c += btrp[bci[k] + 1] - btrp[bci[k]];
    cnt[t] = c;
  }
}
// expansion of row i of B D^-1 B^T in fixed order (k, then B^T row entries)
__global__ void k_spgemm_expand(long r0, long nr, const int64_t *__restrict__ brp, const int *__restrict__ bci,
                                const double *__restrict__ bva, const double *__restrict__ dMinv,
                                const int *__restrict__ btrp, const int *__restrict__ btci,
                                const double *__restrict__ btva, const int64_t *__restrict__ off,
                                int *__restrict__ keys, double *__restrict__ vals) {
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < nr; t += (long)gridDim.x * blockDim.x) {
    const long i = r0 + t;
    int64_t o = off[t];
    for (int64_t k = brp[i]; k < brp[i + 1]; ++k) {
      const int j = bci[k];
      const double a = bva[k] * dMinv[j];
      for (int q = btrp[j]; q < btrp[j + 1]; ++q, ++o) {
        keys[o] = btci[q];
        vals[o] = a * btva[q];
      }
    }
  }
}
// distinct keys per (sorted) segment
__global__ void k_spgemm_unique(long nr, const int64_t *__restrict__ off, const int *__restrict__ keys,
                                int *__restrict__ ucnt) {
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < nr; t += (long)gridDim.x * blockDim.x) {
    int c = 0;
    for (int64_t o = off[t]; o < off[t + 1]; ++o)
      if (o == off[t] || keys[o] != keys[o - 1]) ++c;
    ucnt[t] = c;
  }
}
// reduce runs of equal keys (in their stable-sorted expansion order)
__global__ void k_spgemm_compact(long nr, const int64_t *__restrict__ off, const int *__restrict__ keys,
                                 const double *__restrict__ vals, const int *__restrict__ urp,
                                 int *__restrict__ sci, double *__restrict__ sva) {
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < nr; t += (long)gridDim.x * blockDim.x) {
    int o = urp[t] - urp[0];
    int64_t a = off[t];
    const int64_t e = off[t + 1];
    while (a < e) {
      const int key = keys[a];
      double s = 0.0;
      while (a < e && keys[a] == key) s += vals[a++];
      sci[o] = key;
      sva[o] = s;
      ++o;
    }
  }
}
// Gershgorin: per-row sum |S_ij| / S_ii, block max partials + last block max
__global__ void k_gershgorin(long n, const int *__restrict__ rp, const int *__restrict__ ci,
                             const double *__restrict__ va, double *part, unsigned *counter, DevState *st) {
  __shared__ double sh[32];
  double m = 0.0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    double s = 0.0, d = 0.0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      s += fabs(va[k]);
      if (ci[k] == i) d = va[k];
    }
    if (d > 0.0) m = fmax(m, s / d);
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    t = warp_max(t);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
  }
  if (elect_last_block(counter)) {
    if (threadIdx.x == 0) {
      double mm = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) mm = fmax(mm, __ldcg(part + b));
      st->lmax = mm;
      *counter = 0u;
    }
  }
}
__global__ void k_shift_inv(long n, const double *__restrict__ diag, const double *__restrict__ wdiag, double eps,
                            double *__restrict__ out) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    out[i] = 1.0 / (diag[i] + eps * (wdiag ? wdiag[i] : 1.0));
}
// ---------------------------------------------------------------------------
// element-block Jacobi (reading R15/R16): D_B = n_p x n_p diagonal blocks of S_D
// (+ eps W), inverted at upload (Gauss-Jordan, partial pivoting), applied by
// one thread per element.  NB is a compile-time block size (k = 1: 4, k = 2: 10).
// ---------------------------------------------------------------------------
template <int NB>
__global__ void k_block_extract_inv(long ne, const int *__restrict__ rp, const int *__restrict__ ci,
                                    const double *__restrict__ va, const double *__restrict__ wdiag, double shift,
                                    double *__restrict__ inv, int *err) {
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += (long)gridDim.x * blockDim.x) {
    double a[NB][2 * NB];
    for (int i = 0; i < NB; ++i) {
      for (int j = 0; j < 2 * NB; ++j) a[i][j] = (j - NB == i) ? 1.0 : 0.0;
      const long row = e * NB + i;
      for (int k = rp[row]; k < rp[row + 1]; ++k) {
        const long c = ci[k] - e * NB;
        if (c >= 0 && c < NB) a[i][c] = va[k];
      }
      a[i][i] += shift * (wdiag ? wdiag[row] : 1.0);
    }
    bool ok = true;
    for (int col = 0; col < NB; ++col) {
      int piv = col;
      for (int i = col + 1; i < NB; ++i)
        if (fabs(a[i][col]) > fabs(a[piv][col])) piv = i;
      if (!(fabs(a[piv][col]) > 0.0)) {
        ok = false;
        break;
      }
      if (piv != col)
        for (int j = 0; j < 2 * NB; ++j) {
          const double t = a[col][j];
          a[col][j] = a[piv][j];
          a[piv][j] = t;
        }
      const double ip = 1.0 / a[col][col];
      for (int j = 0; j < 2 * NB; ++j) a[col][j] *= ip;
      for (int i = 0; i < NB; ++i) {
        if (i == col) continue;
        const double f = a[i][col];
        if (f != 0.0)
          for (int j = 0; j < 2 * NB; ++j) a[i][j] -= f * a[col][j];
      }
    }
    if (!ok) atomicExch(err, 1);
    double *o = inv + e * NB * NB;
    for (int i = 0; i < NB; ++i)
      for (int j = 0; j < NB; ++j) o[i * NB + j] = ok ? a[i][NB + j] : 0.0;
  }
}

template <int NB>
__device__ __forceinline__ void block_mv(const double *__restrict__ inv, long e, const double (&r)[NB],
                                         double (&t)[NB]) {
  const double *b = inv + e * NB * NB;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NB; ++j) s = fma(b[i * NB + j], r[j], s);
    t[i] = s;
  }
}

// r_new = r - S d_old (rows), the SpMV half of a block-Jacobi Chebyshev step
__global__ void __launch_bounds__(256) k_cheb_resid(long np, Sell S, double *__restrict__ r,
                                                    const double *__restrict__ d_old, const int *gate) {
  if (!*gate) return;
  const long slot = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= np) return;
  r[sell_row(S, slot)] -= sell_dot(S, slot, GatherX{d_old});
}

// ---------------------------------------------------------------------------
// Tiled element-block apply: a 256-thread block walks tiles of TE = 256 / NB
// elements; the tile's inverse blocks (TE NB^2 doubles) and its vector rows are
// staged in shared memory with coalesced loads, then thread t computes row t of
// D_B^-1 v for the tile and every vector update is a coalesced row access.
// ---------------------------------------------------------------------------
template <int NB>
struct BlkTile {
  static constexpr int TE = 256 / NB;
  static constexpr int ROWS = TE * NB;
};

// stage inverse blocks and one vector of the tile [e0, e0 + te) into shared memory
template <int NB>
__device__ __forceinline__ void stage_blk(const double *__restrict__ inv, const double *__restrict__ v, long e0,
                                          int te, double *sinv, double *sv) {
  const long base = e0 * NB;
  for (int q = threadIdx.x; q < te * NB * NB; q += blockDim.x) sinv[q] = inv[base * NB + q];
  for (int q = threadIdx.x; q < te * NB; q += blockDim.x) sv[q] = v[base + q];
}
template <int NB>
__device__ __forceinline__ double row_blk(const double *sinv, const double *sv, int t) {
  const int el = t / NB, i = t - el * NB;
  const double *a = sinv + el * NB * NB + i * NB;
  const double *x = sv + el * NB;
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < NB; ++j) s = fma(a[j], x[j], s);
  return s;
}

// Element blocks inside a warp: EPW = 32 / NB whole elements per warp (lane
// l -> element l / NB, row l % NB; lanes >= EPW NB idle).  The NB values of an
// element's vector are exchanged with shuffles, and each lane streams its own
// contiguous row of the block inverse, so a warp reads one contiguous span of
// the inverses and of every vector: no shared-memory staging, no barriers.
template <int NB>
struct BlkWarp {
  static constexpr int EPW = 32 / NB;
  long e, k;      // element, row
  int a, base;    // row inside the element, first lane of the element group
  bool valid;
  __device__ __forceinline__ BlkWarp(long gw, long ne) {
    const int lane = threadIdx.x & 31;
    a = lane % NB;
    base = lane - a;
    e = gw * EPW + lane / NB;
    valid = lane < EPW * NB && e < ne;
    k = e * NB + a;
  }
  // sum_b inv[e][a][b] v[e NB + b], v given per lane (vk = v[k])
  __device__ __forceinline__ double apply(const double *__restrict__ inv, double vk) const {
    const double *row = inv + k * NB;
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const double vb = __shfl_sync(0xffffffffu, vk, (base + b) & 31);
      if (valid) s = fma(__ldcs(row + b), vb, s);
    }
    return s;
  }
};
template <int NB>
__host__ __device__ __forceinline__ long blk_warps(long ne) { return (ne + BlkWarp<NB>::EPW - 1) / BlkWarp<NB>::EPW; }

// block half of a Chebyshev step (mode 0) or the init (mode 1: d = c2 D^-1 r, x = d)
//   d_new = c1 d_old + c2 D_B^-1 r ; x += d_new ; last -> z_p = -x
template <int NB>
__global__ void __launch_bounds__(256) k_cheb_block(long ne, const double *__restrict__ inv,
                                                    const double *__restrict__ r, const double *__restrict__ d_old,
                                                    double *__restrict__ d_new, double *__restrict__ x, double c1,
                                                    double c2, int mode, int last, double *__restrict__ zp,
                                                    const int *gate) {
  if (!*gate) return;
  const long nw = blk_warps<NB>(ne);
  for (long gw = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; gw < nw; gw += ((long)gridDim.x * blockDim.x) >> 5) {
    const BlkWarp<NB> w(gw, ne);
    const double rk = w.valid ? r[w.k] : 0.0;
    const double tv = w.apply(inv, rk);
    if (w.valid) {
      const long k = w.k;
      const double dn = mode ? c2 * tv : fma(c1, d_old[k], c2 * tv);
      const double xn = mode ? dn : x[k] + dn;
      if (last) {
        zp[k] = -xn;
      } else {
        d_new[k] = dn;
        x[k] = xn;
      }
    }
  }
}

// block PCG init: x = 0, r = b, p_prev = 0, z = D_B^-1 b; rz = r.z, bn = ||b||
template <int NB>
__global__ void __launch_bounds__(256) k_pcg_init_blk(long ne, const double *__restrict__ inv,
                                                      const double *__restrict__ b, double *__restrict__ x,
                                                      double *__restrict__ r, double *__restrict__ z,
                                                      double *__restrict__ p0, double *part, unsigned *counter,
                                                      DevState *st, double rtol, int maxit, const int *gate) {
  __shared__ double sh[64];
  const bool on = *gate != 0;
  double v[2] = {0.0, 0.0};
  if (on) {
    const long nw = blk_warps<NB>(ne);
    for (long gw = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; gw < nw;
         gw += ((long)gridDim.x * blockDim.x) >> 5) {
      const BlkWarp<NB> w(gw, ne);
      const double bk = w.valid ? b[w.k] : 0.0;
      const double tv = w.apply(inv, bk);
      if (w.valid) {
        const long k = w.k;
        x[k] = 0.0;
        r[k] = bk;
        z[k] = tv;
        p0[k] = tv;     // p_0 = z_0 (the block path materialises p, see k_pcg_pupd)
        v[0] += bk * tv;
        v[1] += bk * bk;
      }
    }
  }
  block_sum_n<2>(v, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x * 2 + 0] = v[0];
    part[blockIdx.x * 2 + 1] = v[1];
  }
  if (elect_last_block(counter)) {
    __shared__ double tot[2];
    reduce_partials<2>(part, gridDim.x, 2, tot);
    if (threadIdx.x == 0) {
      PcgState &p = st->p;
      p.rz = tot[0];
      p.bn = sqrt(tot[1]);
      p.tol_abs = rtol * p.bn;
      p.beta = 0.0;
      p.its = 0;
      p.maxit = maxit;
      p.failed = 0;
      p.active = (on && p.bn > 0.0) ? 1 : 0;
      *counter = 0u;
    }
  }
}

// block PCG step A (single gather): q = (S + eps W) p, p.q -> alpha
__global__ void __launch_bounds__(256) k_pcg_spmv_p(long n, Sell S, const double *__restrict__ wdiag, double eps,
                                                    const double *__restrict__ p, double *__restrict__ q,
                                                    double *part, unsigned *counter, DevState *st, int split) {
  __shared__ double sh[32];
  if (!st->p.active) return;
  double v[1] = {0.0};
  const long slot = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (slot < n) {
    const long row = sell_row(S, slot);
    const double pi = p[row];
    const double w = wdiag ? wdiag[row] : 1.0;
    const double qi = fma(eps * w, pi, sell_dot(S, slot, GatherX{p}));
    q[row] = qi;
    v[0] = pi * qi;
  }
  if (split) {   // partials only; k_pcg_alpha reduces them (no fence / atomic tail here).  One partial
    // per warp instead of per block was tried (R2_05, R2_09): the pass itself did not change and
    // the one-block sum of 8x the partials cost 20 us more
    block_sum_n<1>(v, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = v[0];
    return;
  }
  block_sum_n<1>(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
  if (elect_last_block(counter)) {
    __shared__ double tot;
    reduce_partials<1>(part, gridDim.x, 1, &tot);
    if (threadIdx.x == 0) {
      st->p.alpha = st->p.rz / tot;
      *counter = 0u;
    }
  }
}
// alpha = rz / sum(part[0 .. nb)): one block, fixed order (split form of k_pcg_spmv_p)
__global__ void __launch_bounds__(1024) k_pcg_alpha(int nb, const double *__restrict__ part, DevState *st) {
  __shared__ double sh[32];
  if (!st->p.active) return;
  double v[1] = {0.0};
  for (int b = threadIdx.x; b < nb; b += blockDim.x) v[0] += part[b];
  block_sum_n<1>(v, sh);
  if (threadIdx.x == 0) st->p.alpha = st->p.rz / v[0];
}

// split form of the k_pcg_vec_blk tail: one block sums the (r.z, r.r) partials in a
// fixed order, then its++, convergence ||r|| <= rtol ||b||, beta = rz_new / rz
__global__ void __launch_bounds__(1024) k_pcg_beta(int nb, const double *__restrict__ part, DevState *st) {
  __shared__ double sh[64];
  if (!st->p.active) return;
  double v[2] = {0.0, 0.0};
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    v[0] += part[2 * b];
    v[1] += part[2 * b + 1];
  }
  block_sum_n<2>(v, sh);
  if (threadIdx.x == 0) {
    PcgState &pp = st->p;
    pp.its += 1;
    pp.rr = v[1];
    if (sqrt(v[1]) <= pp.tol_abs) {
      pp.active = 0;
    } else if (pp.its >= pp.maxit) {
      pp.active = 0;
      pp.failed = 1;
    } else {
      pp.beta = v[0] / pp.rz;
      pp.rz = v[0];
    }
  }
}

// block PCG step C: p = z + beta p (after step B decided beta; skipped once converged)
__global__ void k_pcg_pupd(long n, const double *__restrict__ z, double *__restrict__ p, DevState *st) {
  if (!st->p.active) return;
  const double beta = st->p.beta;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
}

// block PCG step B: x += alpha p; r -= alpha q; z = D_B^-1 r; r.z, r.r -> beta, convergence
template <int NB>
__global__ void __launch_bounds__(256) k_pcg_vec_blk(long ne, const double *__restrict__ inv,
                                                     const double *__restrict__ p, const double *__restrict__ q,
                                                     double *__restrict__ x, double *__restrict__ r,
                                                     double *__restrict__ z, double *part, unsigned *counter,
                                                     DevState *st, int split) {
  __shared__ double sh[64];
  if (!st->p.active) return;
  const double alpha = st->p.alpha;
  double v[2] = {0.0, 0.0};
  const long nw = blk_warps<NB>(ne);
  for (long gw = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; gw < nw; gw += ((long)gridDim.x * blockDim.x) >> 5) {
    const BlkWarp<NB> w(gw, ne);
    double rk = 0.0;
    if (w.valid) {
      const long k = w.k;
      x[k] = fma(alpha, p[k], x[k]);
      rk = fma(-alpha, q[k], r[k]);
      r[k] = rk;
    }
    const double tv = w.apply(inv, rk);
    if (w.valid) {
      z[w.k] = tv;
      v[0] += rk * tv;
      v[1] += rk * rk;
    }
  }
  block_sum_n<2>(v, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x * 2 + 0] = v[0];
    part[blockIdx.x * 2 + 1] = v[1];
  }
  if (split) return;   // k_pcg_beta reduces the partials
  if (elect_last_block(counter)) {
    __shared__ double tot[2];
    reduce_partials<2>(part, gridDim.x, 2, tot);
    if (threadIdx.x == 0) {
      PcgState &pp = st->p;
      pp.its += 1;
      pp.rr = tot[1];
      if (sqrt(tot[1]) <= pp.tol_abs) {
        pp.active = 0;
      } else if (pp.its >= pp.maxit) {
        pp.active = 0;
        pp.failed = 1;
      } else {
        pp.beta = tot[0] / pp.rz;
        pp.rz = tot[0];
      }
      *counter = 0u;
    }
  }
}

__global__ void k_widen(long n, const int64_t *__restrict__ in, int *__restrict__ out) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    out[i] = (int)in[i];
}

// ---------------------------------------------------------------------------
// Persistent block PCG (small systems, latency-bound: C2): the whole inner solve
// in ONE cooperative launch, grid-wide barriers between the phases of a step
// instead of five kernel launches.  Same arithmetic as k_pcg_spmv_p /
// k_pcg_alpha / k_pcg_vec_blk / k_pcg_beta / k_pcg_pupd (split form): block
// partials, then EVERY block sums all partials in the same fixed order, so all
// blocks take identical decisions (alpha, beta, convergence) without another
// barrier.  Partial buffers of consecutive phases are disjoint (no read/write race).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void grid_sum_parts(const double *part, int nb, int nv, double *out, double *sh) {
  // out[0..nv) = sum over b < nb of part[b nv + i], lane-strided per warp then xor tree
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp < nv) {
    double s = 0.0;
    for (int b = lane; b < nb; b += 32) s += __ldcg(part + (size_t)b * nv + warp);
    s = warp_sum(s);
    if (lane == 0) sh[warp] = s;
  }
  __syncthreads();
  for (int i = 0; i < nv; ++i) out[i] = sh[i];
  __syncthreads();
}

// p_new = z + beta p_old formed at every gathered column (phase 3 folded into the
// next step's phase 1: two barriers per step instead of three)
struct GatherPz {
  double beta;
  const double *__restrict__ z, *__restrict__ p_old;
  __device__ __forceinline__ double operator()(int c) const { return fma(beta, p_old[c], z[c]); }
};

template <int NB>
__global__ void __launch_bounds__(256) k_pcg_persistent(long np, Sell S, const double *__restrict__ wdiag, double eps,
                                                        const double *__restrict__ inv, double *__restrict__ x,
                                                        double *__restrict__ r, double *__restrict__ z,
                                                        double *__restrict__ p0, double *__restrict__ p1,
                                                        double *__restrict__ q, double *part, DevState *st,
                                                        double **p_final) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[64];
  __shared__ double tot[2];
  double *part1 = part, *part2 = part + gridDim.x;
  const long nth = (long)gridDim.x * blockDim.x, tid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long ne = np / NB, nw = blk_warps<NB>(ne);
  int active = st->p.active, its = st->p.its, failed = 0;
  const int maxit = st->p.maxit;
  double rz = st->p.rz, rr = st->p.rr;
  const double tol = st->p.tol_abs;
  double beta = 0.0;            // first step: p = p0 (= z0, written by the init kernel)
  double *pold = p0, *pnew = p1;
  bool first = true;
  while (active) {
    // phase 1: p_new = z + beta p_old (own row, and on the fly at gathered columns);
    //          q = (S + eps W) p_new; partial p_new . q
    double v1[1] = {0.0};
    for (long slot = tid; slot < np; slot += nth) {
      const long row = sell_row(S, slot);
      double acc, pi;
      if (first) {
        acc = sell_dot(S, slot, GatherX{pold});
        pi = pold[row];
      } else {
        acc = sell_dot(S, slot, GatherPz{beta, z, pold});
        pi = fma(beta, pold[row], z[row]);
        pnew[row] = pi;
      }
      const double qi = fma(eps * (wdiag ? wdiag[row] : 1.0), pi, acc);
      q[row] = qi;
      v1[0] += pi * qi;
    }
    block_sum_n<1>(v1, sh);
    if (threadIdx.x == 0) part1[blockIdx.x] = v1[0];
    if (!first) {   // from here on the current direction is pnew
      double *t = pold;
      pold = pnew;
      pnew = t;
    }
    first = false;
    grid.sync();
    grid_sum_parts(part1, gridDim.x, 1, tot, sh);
    const double alpha = rz / tot[0];
    // phase 2: x += alpha p, r -= alpha q, z = D_B^-1 r, partial r.z and r.r
    double v[2] = {0.0, 0.0};
    for (long gw = tid >> 5; gw < nw; gw += nth >> 5) {
      const BlkWarp<NB> w(gw, ne);
      double rk = 0.0;
      if (w.valid) {
        x[w.k] = fma(alpha, pold[w.k], x[w.k]);
        rk = fma(-alpha, q[w.k], r[w.k]);
        r[w.k] = rk;
      }
      const double tv = w.apply(inv, rk);
      if (w.valid) {
        z[w.k] = tv;
        v[0] += rk * tv;
        v[1] += rk * rk;
      }
    }
    block_sum_n<2>(v, sh);
    if (threadIdx.x == 0) {
      part2[blockIdx.x * 2] = v[0];
      part2[blockIdx.x * 2 + 1] = v[1];
    }
    grid.sync();
    grid_sum_parts(part2, gridDim.x, 2, tot, sh);
    ++its;
    rr = tot[1];
    if (sqrt(tot[1]) <= tol) {
      active = 0;
    } else if (its >= maxit) {
      active = 0;
      failed = 1;
    } else {
      beta = tot[0] / rz;
      rz = tot[0];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->p.active = 0;
    st->p.its = its;
    st->p.failed = failed;
    st->p.rz = rz;
    st->p.rr = rr;
    *p_final = pold;
  }
}
