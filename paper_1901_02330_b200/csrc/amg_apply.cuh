// amg_apply.cuh — V-cycle kernels of the S_D aggregation multigrid (precond
// kinds 3 and 4, oracle/amg.py AMG.vcycle), templated on the value type T of
// the hierarchy: double (kind 3) or float (kind 4, the mixed-precision
// preconditioner of SURVEY.md §8(f) N4: the V-cycle runs in FP32 inside the
// FP64 GMRES).  Every kernel is gated by the Arnoldi-step flag.
#pragma once
#include "kernels.cuh"

// programmatic dependent launch (coarse-level chains of small kernels): wait for the
// previous kernel of the stream (all its writes visible), then let the next one be
// scheduled.  No-ops when the kernel was launched without the PDL attribute.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}


template <typename T>
struct SellT {
  const long long *__restrict__ soff;
  const int *__restrict__ ci;
  const T *__restrict__ va;
};

template <typename T, typename Gather>
__device__ __forceinline__ T sellt_dot(const SellT<T> &A, long row, Gather g) {
  const long s = row >> 5;
  const int lane = (int)(row & 31);
  const long long b = A.soff[s];
  const int w = (int)((A.soff[s + 1] - b) >> 5);
  const int *__restrict__ c = A.ci + b + lane;
  const T *__restrict__ v = A.va + b + lane;
  T acc = T(0);
#pragma unroll 4
  for (int j = 0; j < w; ++j) acc = fma(__ldcs(v + ((long)j << 5)), g(__ldcs(c + ((long)j << 5))), acc);
  return acc;
}

template <typename T>
__device__ __forceinline__ T warp_sum_t(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// one row per group of G lanes (G = 4 .. 32, a power of two): lane-strided CSR entries, xor-shuffle sum
template <typename T, int G, typename Gather>
__device__ __forceinline__ T warp_row_dot_t(const int *__restrict__ rp, const int *__restrict__ ci,
                                            const T *__restrict__ va, long row, Gather g) {
  const int lane = threadIdx.x & (G - 1);
  T acc = T(0);
  for (int k = rp[row] + lane; k < rp[row + 1]; k += G) acc = fma(va[k], g(ci[k]), acc);
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

template <typename T>
struct GatherT {
  const T *__restrict__ x;
  __device__ __forceinline__ T operator()(int c) const { return __ldg(x + c); }
};
// d0 = D^-1 b / theta at a gathered column (the Chebyshev init fused into the first step)
template <typename T>
struct GatherD0T {
  const T *__restrict__ b, *__restrict__ dinv;
  T it;
  __device__ __forceinline__ T operator()(int c) const { return dinv[c] * b[c] * it; }
};

// Chebyshev smoother init from x0 = 0: r = b, d = D^-1 b / theta, x = d (acc: x += d)
template <typename T>
__global__ void k_vc_cheb_init(long n, const T *__restrict__ dinv, const T *__restrict__ b, T inv_theta,
                               T *__restrict__ r, T *__restrict__ d, T *__restrict__ x, int acc, const int *gate) {
  if (!*gate) return;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const T bi = b[i];
    const T di = dinv[i] * bi * inv_theta;
    r[i] = bi;
    d[i] = di;
    x[i] = acc ? x[i] + di : di;
  }
}
// r -= A d_old; d_new = c1 d_old + c2 D^-1 r; x += d_new
template <typename T>
__global__ void __launch_bounds__(256) k_vc_cheb_step(long n, SellT<T> A, const T *__restrict__ dinv,
                                                      T *__restrict__ r, const T *__restrict__ d_old,
                                                      T *__restrict__ d_new, T *__restrict__ x, T c1, T c2,
                                                      const int *gate) {
  if (!*gate) return;
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const T rn = r[i] - sellt_dot(A, i, GatherT<T>{d_old});
  const T dn = c1 * d_old[i] + c2 * (dinv[i] * rn);
  r[i] = rn;
  d_new[i] = dn;
  x[i] += dn;
}
template <typename T, int G>
__global__ void __launch_bounds__(256) k_vc_cheb_step_w(long n, const int *__restrict__ rp, const int *__restrict__ ci,
                                                        const T *__restrict__ va, const T *__restrict__ dinv,
                                                        T *__restrict__ r, const T *__restrict__ d_old,
                                                        T *__restrict__ d_new, T *__restrict__ x, T c1, T c2,
                                                        const int *gate) {
  pdl_enter();
  if (!*gate) return;
  const long i = ((long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  if ((i & ~(long)(32 / G - 1)) >= n) return;   // whole warps only: the groups of a warp shuffle together
  const T ad = warp_row_dot_t<T, G>(rp, ci, va, i < n ? i : n - 1, GatherT<T>{d_old});
  if ((threadIdx.x & (G - 1)) == 0 && i < n) {
    const T rn = r[i] - ad;
    const T dn = c1 * d_old[i] + c2 * (dinv[i] * rn);
    r[i] = rn;
    d_new[i] = dn;
    x[i] += dn;
  }
}
// first step fused with the init: d0 = D^-1 b / theta gathered on the fly; r = b - A d0;
// d1 = c1 d0 + c2 D^-1 r; x = d0 + d1 (acc: x += d0 + d1)
template <typename T>
__global__ void __launch_bounds__(256) k_vc_cheb_first(long n, SellT<T> A, const T *__restrict__ dinv,
                                                       const T *__restrict__ b, T inv_theta, T c1, T c2,
                                                       T *__restrict__ r, T *__restrict__ d_new, T *__restrict__ x,
                                                       int acc, const int *gate) {
  if (!*gate) return;
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const T ad = sellt_dot(A, i, GatherD0T<T>{b, dinv, inv_theta});
  const T bi = b[i];
  const T d0 = dinv[i] * bi * inv_theta;
  const T rn = bi - ad;
  const T dn = c1 * d0 + c2 * (dinv[i] * rn);
  r[i] = rn;
  d_new[i] = dn;
  x[i] = acc ? x[i] + (d0 + dn) : d0 + dn;
}
template <typename T, int G>
__global__ void __launch_bounds__(256) k_vc_cheb_first_w(long n, const int *__restrict__ rp,
                                                         const int *__restrict__ ci, const T *__restrict__ va,
                                                         const T *__restrict__ dinv, const T *__restrict__ b,
                                                         T inv_theta, T c1, T c2, T *__restrict__ r,
                                                         T *__restrict__ d_new, T *__restrict__ x, int acc,
                                                         const int *gate) {
  pdl_enter();
  if (!*gate) return;
  const long i = ((long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  if ((i & ~(long)(32 / G - 1)) >= n) return;   // whole warps only: the groups of a warp shuffle together
  const T ad = warp_row_dot_t<T, G>(rp, ci, va, i < n ? i : n - 1, GatherD0T<T>{b, dinv, inv_theta});
  if ((threadIdx.x & (G - 1)) == 0 && i < n) {
    const T bi = b[i];
    const T d0 = dinv[i] * bi * inv_theta;
    const T rn = bi - ad;
    const T dn = c1 * d0 + c2 * (dinv[i] * rn);
    r[i] = rn;
    d_new[i] = dn;
    x[i] = acc ? x[i] + (d0 + dn) : d0 + dn;
  }
}
// t = b - A x
template <typename T>
__global__ void __launch_bounds__(256) k_vc_resid(long n, SellT<T> A, const T *__restrict__ x,
                                                  const T *__restrict__ b, T *__restrict__ t, const int *gate) {
  if (!*gate) return;
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const T acc = sellt_dot(A, i, GatherT<T>{x});
  t[i] = b[i] - acc;
}
template <typename T, int G>
__global__ void __launch_bounds__(256) k_vc_resid_w(long n, const int *__restrict__ rp, const int *__restrict__ ci,
                                                    const T *__restrict__ va, const T *__restrict__ x,
                                                    const T *__restrict__ b, T *__restrict__ t, const int *gate) {
  pdl_enter();
  if (!*gate) return;
  const long i = ((long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  if ((i & ~(long)(32 / G - 1)) >= n) return;   // whole warps only: the groups of a warp shuffle together
  const T ax = warp_row_dot_t<T, G>(rp, ci, va, i < n ? i : n - 1, GatherT<T>{x});
  if ((threadIdx.x & (G - 1)) == 0 && i < n) t[i] = b[i] - ax;
}
// plain aggregation transfers: bc[a] = sum over members (index order); x += xc[agg]
template <typename T>
__global__ void k_vc_restrict(long nc, const int *__restrict__ moff, const int *__restrict__ mem,
                              const T *__restrict__ r, T *__restrict__ bc, const int *gate) {
  if (!*gate) return;
  for (long a = (long)blockIdx.x * blockDim.x + threadIdx.x; a < nc; a += (long)gridDim.x * blockDim.x) {
    T s = T(0);
    for (int p = moff[a]; p < moff[a + 1]; ++p) s += r[mem[p]];
    bc[a] = s;
  }
}
template <typename T>
__global__ void k_vc_prolong_add(long n, const int *__restrict__ agg, const T *__restrict__ xc, T *__restrict__ x,
                                 const int *gate) {
  if (!*gate) return;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    x[i] += xc[agg[i]];
}
// smoothed-aggregation transfers: b_c = P^T r (8 lanes per coarse row, fixed order); x += P xc
template <typename T>
__global__ void __launch_bounds__(256) k_vc_sa_restrict(long nc, const int *__restrict__ trp,
                                                        const int *__restrict__ tci, const T *__restrict__ tva,
                                                        const T *__restrict__ r, T *__restrict__ bc, const int *gate) {
  if (!*gate) return;
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long a = t >> 3;
  const int g = (int)(t & 7);
  T acc = T(0);
  if (a < nc)
    for (int k = trp[a] + g; k < trp[a + 1]; k += 8) acc = fma(tva[k], r[tci[k]], acc);
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (a < nc && g == 0) bc[a] = acc;
}
template <typename T>
__global__ void __launch_bounds__(256) k_vc_sa_prolong_add(long n, SellT<T> P, const T *__restrict__ xc,
                                                           T *__restrict__ x, const int *gate) {
  if (!*gate) return;
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  x[i] += sellt_dot(P, i, GatherT<T>{xc});
}
// coarsest level: x = inv b, one warp per row
template <typename T>
__global__ void __launch_bounds__(256) k_vc_dense_mv(long n, const T *__restrict__ inv, const T *__restrict__ b,
                                                     T *__restrict__ x, const int *gate) {
  if (!*gate) return;
  const long i = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  const int lane = threadIdx.x & 31;
  T s = T(0);
  for (long j = lane; j < n; j += 32) s = fma(inv[i * n + j], b[j], s);
  s = warp_sum_t(s);
  if (lane == 0) x[i] = s;
}
// top of the Block-Schur-AMG apply: z_u = s v_u ./ diag(M) (FP64), b0 = s v_p (in T)
template <typename T>
__global__ void k_vc_top(long nu, long np, const double *__restrict__ v, const double *scale,
                         const double *__restrict__ dMinv, double *__restrict__ z, T *__restrict__ b0,
                         const int *gate) {
  if (!*gate) return;
  const double s = *scale;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nu + np; i += (long)gridDim.x * blockDim.x) {
    if (i < nu) {
      if (z) z[i] = s * v[i] * dMinv[i];
    } else {
      b0[i - nu] = (T)(s * v[i]);
    }
  }
}
// z_p = -x0 (FP64 output)
template <typename T>
__global__ void k_vc_out(long n, const T *__restrict__ x, double *__restrict__ out, const int *gate) {
  if (!*gate) return;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    out[i] = -1.0 * (double)x[i];
}
// Arnoldi-step form: w = A z with z = [s v_u ./ diag(M); -x0] formed in the gather
template <typename T>
struct GatherAmgZT {
  long nu;
  double s;
  const double *__restrict__ v, *__restrict__ dMinv;
  const T *__restrict__ x0;
  __device__ __forceinline__ double operator()(int c) const {
    return c < nu ? s * v[c] * dMinv[c] : -(double)x0[c - nu];
  }
};
template <typename T>
__global__ void __launch_bounds__(256) k_vc_spmv_z(long n, long nu, Sell A, const double *__restrict__ v,
                                                   const double *scale, const double *__restrict__ dMinv,
                                                   const T *__restrict__ x0, double *__restrict__ y,
                                                   double *__restrict__ zout, const int *gate) {
  if (!*gate) return;
  const long row = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  const GatherAmgZT<T> g{nu, *scale, v, dMinv, x0};
  y[row] = sell_dot(A, row, g);
  if (zout) zout[row] = g((int)row);   // FGMRES keeps z_j
}
__global__ void k_d2f(long n, const double *__restrict__ in, float *__restrict__ out) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    out[i] = (float)in[i];
}

// ---------------------------------------------------------------------------
// Coarsest level without a dense inverse (stagnated coarsening; C3: 11,794 rows):
// the degree-d Chebyshev smoother (oracle/amg.py AMG.vcycle -> smooth(lev, b,
// COARSE_DEGREE)) as ONE launch of a 16-CTA thread-block cluster instead of d
// launches.  Each CTA owns a contiguous nnz-balanced row range (at most two rows
// per thread, r, x, d, D^-1 of its rows in registers) and keeps its CSR slice in
// shared memory (16-bit columns) for all d-1 steps, together with a full copy of
// the current direction: the gathers of A d are shared-memory loads.  The new
// directions are exchanged through two global (L2-resident) buffers: each CTA
// writes its slice, one cluster barrier (release/acquire at cluster scope), then
// every CTA copies the whole vector into its shared memory with 16-byte loads.
// Gathering the directions from L2 or through distributed shared memory instead
// was bound by the per-SM rate of scattered 8-byte requests (~11k per SM per
// step on 16 SMs): 3x slower than the per-step launches.
// ---------------------------------------------------------------------------
constexpr int VC_CLUSTER = 16;          // CTAs per cluster (non-portable size, B200 allows 16)
constexpr int VC_CLUSTER_THREADS = 1024;
constexpr int VC_ROWS_PER_THREAD = 2;
constexpr int VC_MAX_DEGREE = 64;

struct VcCheb {
  double inv_theta;
  int degree;
  double c1[VC_MAX_DEGREE - 1], c2[VC_MAX_DEGREE - 1];
};

template <typename T>
struct VcCluster {
  const int *rs;              // [VC_CLUSTER + 1] first row of each rank
  const int *rp;              // level CSR row pointers
  const unsigned short *c16;  // level CSR columns as 16-bit (n <= 65535)
  const T *va;
  const T *dinv, *b;
  T *x;
  T *dg0, *dg1;               // direction exchange buffers (n each, global, 16-byte aligned)
  int n;
};

// shared-memory bytes of one CTA of the cluster kernel
template <typename T>
inline size_t vc_cluster_smem(long n, int rows, long nnz) {
  const size_t dv = ((size_t)n * sizeof(T) + 15) / 16 * 16;
  const size_t va = ((size_t)nnz * sizeof(T) + 15) / 16 * 16;
  const size_t rp = ((size_t)(rows + 1) * 4 + 15) / 16 * 16;
  return dv + va + rp + 2 * (size_t)nnz + 16;
}

template <typename T>
__global__ void __launch_bounds__(VC_CLUSTER_THREADS) k_vc_coarse_cluster(VcCluster<T> P, VcCheb cf,
                                                                          const int *gate) {
  if (!*gate) return;   // the gate is uniform: every CTA of the cluster leaves together
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int g = (int)cl.block_rank();
  const int r0 = P.rs[g], nr = P.rs[g + 1] - r0;
  const int z0 = P.rp[r0], nz = P.rp[r0 + nr] - z0;
  extern __shared__ __align__(16) unsigned char vc_smem[];
  T *sdv = reinterpret_cast<T *>(vc_smem);                                   // full direction
  T *sva = reinterpret_cast<T *>(vc_smem + ((size_t)P.n * sizeof(T) + 15) / 16 * 16);
  int *srp = reinterpret_cast<int *>(reinterpret_cast<unsigned char *>(sva) + ((size_t)nz * sizeof(T) + 15) / 16 * 16);
  unsigned short *scc = reinterpret_cast<unsigned short *>(srp + ((nr + 1 + 3) / 4) * 4);
  for (int k = threadIdx.x; k < nz; k += blockDim.x) {
    sva[k] = P.va[z0 + k];
    scc[k] = P.c16[z0 + k];
  }
  for (int i = threadIdx.x; i <= nr; i += blockDim.x) srp[i] = P.rp[r0 + i] - z0;
  const T it = (T)cf.inv_theta;
  // x0 = 0: r = b, d_0 = D^-1 b / theta, x = d_0 (Saad Alg. 12.1 as oracle.solver.chebyshev)
  T rr[VC_ROWS_PER_THREAD], xx[VC_ROWS_PER_THREAD], dd[VC_ROWS_PER_THREAD], di[VC_ROWS_PER_THREAD];
#pragma unroll
  for (int q = 0; q < VC_ROWS_PER_THREAD; ++q) {
    const int i = threadIdx.x + q * VC_CLUSTER_THREADS;
    rr[q] = xx[q] = dd[q] = di[q] = T(0);
    if (i < nr) {
      di[q] = P.dinv[r0 + i];
      rr[q] = P.b[r0 + i];
      dd[q] = di[q] * rr[q] * it;
      xx[q] = dd[q];
      P.dg0[r0 + i] = dd[q];
    }
  }
  cl.sync();
  using V4 = uint4;   // 16-byte copy of the exchanged direction into shared memory
  const int nv = (int)(((size_t)P.n * sizeof(T)) / 16), tail = (int)((size_t)P.n * sizeof(T) - 16 * (size_t)nv);
  for (int s = 0; s + 1 < cf.degree; ++s) {
    const T c1 = (T)cf.c1[s], c2 = (T)cf.c2[s];
    const T *dold = (s & 1) ? P.dg1 : P.dg0;
    T *dnew = (s & 1) ? P.dg0 : P.dg1;
    const V4 *src = reinterpret_cast<const V4 *>(dold);
    V4 *dst = reinterpret_cast<V4 *>(sdv);
    for (int k = threadIdx.x; k < nv; k += blockDim.x) dst[k] = __ldcg(src + k);
    if (tail && threadIdx.x < tail / (int)sizeof(T))
      sdv[16 * nv / sizeof(T) + threadIdx.x] = __ldcg(dold + 16 * nv / sizeof(T) + threadIdx.x);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < VC_ROWS_PER_THREAD; ++q) {
      const int i = threadIdx.x + q * VC_CLUSTER_THREADS;
      if (i < nr) {
        T acc = T(0);
        const int ke = srp[i + 1];
#pragma unroll 4
        for (int k = srp[i]; k < ke; ++k) acc = fma(sva[k], sdv[scc[k]], acc);
        const T rn = rr[q] - acc;          // r_i = r_{i-1} - A d_{i-1}
        const T dn = c1 * dd[q] + c2 * (di[q] * rn);
        rr[q] = rn;
        dd[q] = dn;
        xx[q] += dn;
        dnew[r0 + i] = dn;
      }
    }
    cl.sync();   // every slice of d_new written; every CTA done reading d_old and its shared copy
  }
#pragma unroll
  for (int q = 0; q < VC_ROWS_PER_THREAD; ++q) {
    const int i = threadIdx.x + q * VC_CLUSTER_THREADS;
    if (i < nr) P.x[r0 + i] = xx[q];
  }
}

__global__ void k_vc_cols16(long nnz, const int *__restrict__ ci, unsigned short *__restrict__ c16) {
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (long)gridDim.x * blockDim.x)
    c16[k] = (unsigned short)ci[k];
}
