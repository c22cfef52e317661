// blockreg_m.cuh — kernels of the two nested solves inside the Block-Reg preconditioners:
//
//   * MG-PCG: the inner PCG on S_eps = S_D + eps W preconditioned by one V-cycle of S_eps
//     (reading R23; oracle/amg.py SchurMG, oracle/solver.py pcg).  n_p_dof = 1: the
//     aggregation V-cycle of amg_apply.cuh on the S_eps hierarchy.  n_p_dof > 1: a p-multigrid
//     whose smoother is the element-block-Jacobi Chebyshev(2) on [2/6, 2] (k_mg_blk,
//     k_seps_resid) and whose coarse space is the element-mean moment (k_mg_inject,
//     k_mg_prolong) with the aggregation V-cycle on S_eps[0::n_p, 0::n_p].
//   * K-PCG (precond kind 5, reading R24; oracle/solver.py pcg_k): PCG on the paper's
//     regularised velocity block K = M + B^T (eps W)^-1 B,
//     preconditioned by the kind-2 Woodbury block, stopped on the preconditioned residual.
//
// All reductions are two-stage and deterministic: per-block partials in a fixed grid, then
// one block sums them in a fixed order and takes the scalar decisions (alpha, beta,
// convergence) on the device; the host only polls the state between graph replays.
#pragma once
#include "kernels.cuh"

// q-th partial of a grid-stride dot product, NV values per block at part[blockIdx.x * NV + i]
template <int NV>
__device__ __forceinline__ void store_partials(double (&v)[NV], double *sh, double *part) {
  block_sum_n<NV>(v, sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) part[blockIdx.x * NV + i] = v[i];
  }
}
// one block: out[i] = sum_b part[b * NV + i] in a fixed order (valid in thread 0)
template <int NV>
__device__ __forceinline__ void sum_partials(int nblk, const double *__restrict__ part, double (&v)[NV], double *sh) {
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] += part[b * NV + i];
  }
  block_sum_n<NV>(v, sh);
}

// ---------------------------------------------------------------------------
// S_eps = S_D + eps W pieces
// ---------------------------------------------------------------------------
// out = b - S_eps d on every row (b may alias out: the Chebyshev residual update r -= S_eps d)
__global__ void __launch_bounds__(256) k_seps_resid(long np, Sell S, const double *__restrict__ wdiag, double eps,
                                                    const double *__restrict__ d, const double *b, double *out,
                                                    const int *gate) {
  if (!*gate) return;
  const long slot = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= np) return;
  const long row = sell_row(S, slot);
  const double w = wdiag ? wdiag[row] : 1.0;
  out[row] = b[row] - fma(eps * w, d[row], sell_dot(S, slot, GatherX{d}));
}

// q = S_eps p on every row (the PCG product without its p.q partials: the block barrier of
// k_pcg_spmv_p costs a third of that kernel's stall cycles, ncu R2_27: 172 vs 132 us; the dot
// product is a separate light pass, k_dot_part)
__global__ void __launch_bounds__(256) k_seps_mul(long np, Sell S, const double *__restrict__ wdiag, double eps,
                                                  const double *__restrict__ p, double *__restrict__ q,
                                                  const int *gate) {
  if (!*gate) return;
  const long slot = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= np) return;
  const long row = sell_row(S, slot);
  const double w = wdiag ? wdiag[row] : 1.0;
  q[row] = fma(eps * w, p[row], sell_dot(S, slot, GatherX{p}));
}

// element-block half of a Chebyshev step of the p-multigrid smoother:
//   init: d_new = c2 D_B^-1 r           else: d_new = c1 d_old + c2 D_B^-1 r
//   acc_x: x += d_new                   else: x = d_new
template <int NB>
__global__ void __launch_bounds__(256) k_mg_blk(long ne, const double *__restrict__ inv, const double *__restrict__ r,
                                                const double *__restrict__ d_old, double *__restrict__ d_new,
                                                double *__restrict__ x, double c1, double c2, int init, int acc_x,
                                                const int *gate) {
  if (!*gate) return;
  const long nw = blk_warps<NB>(ne);
  for (long gw = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; gw < nw; gw += ((long)gridDim.x * blockDim.x) >> 5) {
    const BlkWarp<NB> w(gw, ne);
    const double rk = w.valid ? r[w.k] : 0.0;
    const double tv = w.apply(inv, rk);
    if (w.valid) {
      const long k = w.k;
      const double dn = init ? c2 * tv : fma(c1, d_old[k], c2 * tv);
      d_new[k] = dn;
      x[k] = acc_x ? x[k] + dn : dn;
    }
  }
}

// coarse right-hand side: the element-mean moment of t, in the caller's element numbering
// (the hierarchy of S_eps[0::n_p, 0::n_p] is built there so that its aggregation keys equal
// the oracle's); perm_p[new] = old pressure index, nullptr: identity
__global__ void k_mg_inject(long ne, int nb, const int *__restrict__ perm_p, const double *__restrict__ t,
                            double *__restrict__ bc, const int *gate) {
  if (!*gate) return;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += (long)gridDim.x * blockDim.x) {
    const long k = e * nb;
    const long eo = perm_p ? perm_p[k] / nb : e;
    bc[eo] = t[k];
  }
}
__global__ void k_mg_prolong(long ne, int nb, const int *__restrict__ perm_p, const double *__restrict__ xc,
                             double *__restrict__ x, const int *gate) {
  if (!*gate) return;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += (long)gridDim.x * blockDim.x) {
    const long k = e * nb;
    const long eo = perm_p ? perm_p[k] / nb : e;
    x[k] += xc[eo];
  }
}

// setup: rows / entries of S_c = S[0::nb, 0::nb] (+ eps W on its diagonal), CSR in, CSR out
__global__ void k_mg_coarse_count(long ne, int nb, const int *__restrict__ rp, const int *__restrict__ ci,
                                  int *__restrict__ cnt) {
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += (long)gridDim.x * blockDim.x) {
    int c = 0;
    for (int k = rp[e * nb]; k < rp[e * nb + 1]; ++k) c += (ci[k] % nb == 0) ? 1 : 0;
    cnt[e] = c;
  }
}
__global__ void k_mg_coarse_fill(long ne, int nb, const int *__restrict__ rp, const int *__restrict__ ci,
                                 const double *__restrict__ va, const double *__restrict__ wdiag, double eps,
                                 const int *__restrict__ crp, int *__restrict__ cci, double *__restrict__ cva) {
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += (long)gridDim.x * blockDim.x) {
    int o = crp[e];
    for (int k = rp[e * nb]; k < rp[e * nb + 1]; ++k) {
      const int c = ci[k];
      if (c % nb) continue;
      const int ce = c / nb;
      double v = va[k];
      if (ce == e) v += eps * (wdiag ? wdiag[e * nb] : 1.0);
      cci[o] = ce;
      cva[o] = v;
      ++o;
    }
  }
}
// va[diag of row i] += eps w_i (S_eps values from a copy of the S_D values, n_p_dof = 1)
__global__ void k_shift_diag(long n, const int *__restrict__ rp, const int *__restrict__ ci, double *__restrict__ va,
                             const double *__restrict__ wdiag, double eps) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    for (int k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] == i) va[k] += eps * (wdiag ? wdiag[i] : 1.0);
}

// ---------------------------------------------------------------------------
// MG-PCG on S_eps (oracle/solver.py pcg with a callable preconditioner)
// ---------------------------------------------------------------------------
// x = 0, r = b, p = 0; partial b.b
__global__ void k_pcgm_init(long n, const double *__restrict__ b, double *__restrict__ x, double *__restrict__ r,
                            double *__restrict__ p, double *part, const int *gate) {
  __shared__ double sh[32];
  double v[1] = {0.0};
  if (*gate) {
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
      const double bi = b[i];
      x[i] = 0.0;
      r[i] = bi;
      p[i] = 0.0;
      v[0] += bi * bi;
    }
  }
  store_partials<1>(v, sh, part);
}
__global__ void __launch_bounds__(1024) k_pcgm_init_fin(int nblk, const double *__restrict__ part, DevState *st,
                                                        double rtol, int maxit, const int *gate) {
  __shared__ double sh[32];
  double v[1];
  sum_partials<1>(nblk, part, v, sh);
  if (threadIdx.x == 0) {
    PcgState &p = st->p;
    p.bn = sqrt(v[0]);
    p.tol_abs = rtol * p.bn;
    p.beta = 0.0;
    p.rz = 1.0;        // beta = rz_new / rz is discarded at the first direction (p = 0)
    p.its = 0;
    p.maxit = maxit;
    p.failed = 0;
    p.active = (*gate && p.bn > 0.0) ? 1 : 0;
  }
}
// x += alpha p, r -= alpha q; partial r.r
__global__ void k_pcgm_xr(long n, const double *__restrict__ p, const double *__restrict__ q, double *__restrict__ x,
                          double *__restrict__ r, double *part, DevState *st) {
  __shared__ double sh[32];
  if (!st->p.active) return;
  const double alpha = st->p.alpha;
  double v[1] = {0.0};
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    v[0] += ri * ri;
  }
  store_partials<1>(v, sh, part);
}
// its++, ||r|| <= rtol ||b|| -> done; its == maxit -> failed
__global__ void __launch_bounds__(1024) k_pcgm_conv(int nblk, const double *__restrict__ part, DevState *st) {
  __shared__ double sh[32];
  if (!st->p.active) return;
  double v[1];
  sum_partials<1>(nblk, part, v, sh);
  if (threadIdx.x == 0) {
    PcgState &p = st->p;
    p.its += 1;
    p.rr = v[0];
    if (sqrt(v[0]) <= p.tol_abs) {
      p.active = 0;
    } else if (p.its >= p.maxit || !(v[0] == v[0])) {   // cap reached, or NaN: stop at once
      p.active = 0;
      p.failed = 1;
    }
  }
}
// partial a.b (gate: an int that is 1 while the owning solve runs)
__global__ void k_dot_part(long n, const double *__restrict__ a, const double *__restrict__ b, double *part,
                           const int *gate) {
  __shared__ double sh[32];
  if (!*gate) return;
  double v[1] = {0.0};
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    v[0] = fma(a[i], b[i], v[0]);
  store_partials<1>(v, sh, part);
}
// rz_new = r.z; beta = rz_new / rz; rz = rz_new  (first: rz = r.z, beta unused since p = 0)
__global__ void __launch_bounds__(1024) k_pcgm_beta(int nblk, const double *__restrict__ part, DevState *st,
                                                    int first) {
  __shared__ double sh[32];
  if (!st->p.active) return;
  double v[1];
  sum_partials<1>(nblk, part, v, sh);
  if (threadIdx.x == 0) {
    PcgState &p = st->p;
    p.beta = first ? 0.0 : v[0] / p.rz;
    p.rz = v[0];
  }
}

// ---------------------------------------------------------------------------
// K-PCG (kind 5): K = M + B^T (eps W)^-1 B on the velocity unknowns
// ---------------------------------------------------------------------------
// r = s v_u, y = 0, p = 0 (kx velocity part); z_p = s v_p / (eps W)
__global__ void k_k_init(long nu, long np, const double *__restrict__ v, const double *scale,
                         const double *__restrict__ wdiag, double inv_eps, double *__restrict__ r,
                         double *__restrict__ z, double *__restrict__ kx, const int *gate) {
  if (!*gate) return;
  const double s = *scale;
  const long n = nu + np;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    if (i < nu) {
      r[i] = s * v[i];
      z[i] = 0.0;
      kx[i] = 0.0;
    } else {
      const double w = wdiag ? wdiag[i - nu] : 1.0;
      z[i] = s * v[i] * inv_eps / w;
    }
  }
}
// t0 = r ./ diag(M)
__global__ void k_k_t0(long nu, const double *__restrict__ r, const double *__restrict__ dMinv,
                       double *__restrict__ t0, const int *gate) {
  if (!*gate) return;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nu; i += (long)gridDim.x * blockDim.x)
    t0[i] = r[i] * dMinv[i];
}
// q = M p + B^T ((eps W)^-1 B p) on the velocity rows of the merged matrix: kx = [p; B p]
struct GatherK {
  long nu;
  double inv_eps;
  const double *__restrict__ kx, *__restrict__ wdiag;
  __device__ __forceinline__ double operator()(int c) const {
    const double x = kx[c];
    if (c < nu) return x;
    return x * inv_eps / (wdiag ? wdiag[c - nu] : 1.0);
  }
};
__global__ void __launch_bounds__(256) k_kmul(long nu, Sell A, const double *__restrict__ kx,
                                              const double *__restrict__ wdiag, double inv_eps,
                                              double *__restrict__ q, double *part, const int *gate) {
  __shared__ double sh[32];
  if (!*gate) return;
  const long row = (long)blockIdx.x * blockDim.x + threadIdx.x;
  double v[1] = {0.0};
  if (row < nu) {
    const double qi = sell_dot(A, row, GatherK{nu, inv_eps, kx, wdiag});
    q[row] = qi;
    v[0] = kx[row] * qi;
  }
  store_partials<1>(v, sh, part);
}
__global__ void __launch_bounds__(1024) k_k_alpha(int nblk, const double *__restrict__ part, DevState *st) {
  __shared__ double sh[32];
  if (!st->k.active) return;
  double v[1];
  sum_partials<1>(nblk, part, v, sh);
  if (threadIdx.x == 0) st->k.alpha = st->k.rz / v[0];
}
// y += alpha p, r -= alpha q
__global__ void k_k_xr(long nu, const double *__restrict__ p, const double *__restrict__ q, double *__restrict__ y,
                       double *__restrict__ r, DevState *st) {
  if (!st->k.active) return;
  const double alpha = st->k.alpha;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nu; i += (long)gridDim.x * blockDim.x) {
    y[i] = fma(alpha, p[i], y[i]);
    r[i] = fma(-alpha, q[i], r[i]);
  }
}
// after z = P^-1 r: rz_new = r.z (partials summed here).
//   first: rz0 = rz = r.z; the solve runs iff the outer gate is open and r.z > 0
//   else : its++; sqrt|rz_new| <= rtol sqrt(rz0) -> done; its == maxit -> failed;
//          beta = rz_new / rz, rz = rz_new
__global__ void __launch_bounds__(1024) k_k_rz(int nblk, const double *__restrict__ part, DevState *st, int first,
                                               double rtol, int maxit, const int *gate) {
  __shared__ double sh[32];
  if (!first && !st->k.active) return;
  if (first && !*gate) {
    if (threadIdx.x == 0) {
      st->k.active = 0;
      st->k.its = 0;
      st->k.failed = 0;
    }
    return;
  }
  double v[1];
  sum_partials<1>(nblk, part, v, sh);
  if (threadIdx.x == 0) {
    KState &k = st->k;
    if (first) {
      k.rz = v[0];
      k.rz0 = v[0];
      k.beta = 0.0;
      k.its = 0;
      k.maxit = maxit;
      k.failed = 0;
      k.rtol = rtol;
      k.active = v[0] > 0.0 ? 1 : 0;
    } else {
      k.its += 1;
      if (sqrt(fabs(v[0])) <= k.rtol * sqrt(k.rz0)) {
        k.active = 0;
      } else if (k.its >= k.maxit || !(v[0] == v[0])) {   // cap reached, or NaN: stop at once
        k.active = 0;
        k.failed = 1;
      } else {
        k.beta = v[0] / k.rz;
        k.rz = v[0];
      }
    }
  }
}
// p = z + beta p
__global__ void k_k_pupd(long nu, const double *__restrict__ z, double *__restrict__ p, DevState *st) {
  if (!st->k.active) return;
  const double beta = st->k.beta;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nu; i += (long)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
}
