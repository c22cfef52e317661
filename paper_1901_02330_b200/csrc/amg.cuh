// amg.cuh — aggregation multigrid for S_D (precond kind 3, Block-Schur-AMG,
// DESIGN.md reading R22; oracle/amg.py is the step-by-step CPU definition).
//
// Setup (upload-time, all on the device): strength graph, deterministic MIS-2
// aggregation by repeated distance-2 maxima of a fixed splitmix64 key,
// Galerkin coarse operators P^T A P by a stable radix sort of (agg_i, agg_j)
// keys and an in-order run reduction, member lists for deterministic
// restriction, Gauss-Jordan inverse of the coarsest level.
// Apply: one symmetric V-cycle (Chebyshev(3) point-Jacobi smoothing).
#pragma once
#include "kernels.cuh"

#define AMG_KEY_BITS 30
#define AMG_ROOT_KEY 0x7fffffffffffffffLL

__device__ __forceinline__ long long amg_key(long long i) {
  unsigned long long z = (unsigned long long)i + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z = z ^ (z >> 31);
  return (long long)(((z >> 33) << AMG_KEY_BITS) | (unsigned long long)i);
}

// strong[k]: diagonal, or |a_ij| >= theta sqrt(|a_ii a_jj|)
__global__ void k_amg_strong(long n, const int *__restrict__ rp, const int *__restrict__ ci,
                             const double *__restrict__ va, const double *__restrict__ diag, double theta,
                             unsigned char *__restrict__ strong) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int j = ci[k];
      strong[k] = (j == i) || (fabs(va[k]) >= theta * sqrt(fabs(diag[i] * diag[j])));
    }
  }
}

// out[i] = max over strong N[i] of in[j]
__global__ void k_amg_nbr_max(long n, const int *__restrict__ rp, const int *__restrict__ ci,
                              const unsigned char *__restrict__ strong, const long long *__restrict__ in,
                              long long *__restrict__ out) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    long long m = LLONG_MIN;
    for (int k = rp[i]; k < rp[i + 1]; ++k)
      if (strong[k]) m = max(m, in[ci[k]]);
    out[i] = m;
  }
}

// state: 0 undecided, 1 root, 2 excluded.  key view for the next max sweep.
__global__ void k_amg_mis_keys(long n, const signed char *__restrict__ state, long long *__restrict__ kv) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    kv[i] = state[i] == 0 ? amg_key(i) : (state[i] == 1 ? AMG_ROOT_KEY : -1LL);
}
__global__ void k_amg_mis_update(long n, signed char *__restrict__ state, const long long *__restrict__ k2,
                                 unsigned *__restrict__ n_undecided) {
  unsigned cnt = 0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    if (state[i] != 0) continue;
    if (k2[i] == amg_key(i))
      state[i] = 1;
    else if (k2[i] == AMG_ROOT_KEY)
      state[i] = 2;
    else
      ++cnt;
  }
  if (cnt) atomicAdd(n_undecided, cnt);
}
__global__ void k_amg_flag(long n, const signed char *__restrict__ state, int *__restrict__ flag) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    flag[i] = state[i] == 1 ? 1 : 0;
}
// agg = root rank for roots, -1 otherwise; key view of roots for pass 1
__global__ void k_amg_roots(long n, const signed char *__restrict__ state, const int *__restrict__ rank,
                            int *__restrict__ agg, long long *__restrict__ kv) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const bool r = state[i] == 1;
    agg[i] = r ? rank[i] : -1;
    kv[i] = r ? amg_key(i) : -1LL;
  }
}
// pass 1/2: free nodes with best >= 0 take agg_src[best & mask]; writes agg_dst
__global__ void k_amg_join(long n, const int *__restrict__ agg_src, const long long *__restrict__ best,
                           int *__restrict__ agg_dst) {
  const long long mask = (1LL << AMG_KEY_BITS) - 1;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    int a = agg_src[i];
    if (a < 0 && best[i] >= 0) a = agg_src[best[i] & mask];
    agg_dst[i] = a;
  }
}
__global__ void k_amg_assigned_keys(long n, const int *__restrict__ agg, long long *__restrict__ kv) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    kv[i] = agg[i] >= 0 ? amg_key(i) : -1LL;
}
__global__ void k_amg_free_flag(long n, const int *__restrict__ agg, int *__restrict__ flag) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    flag[i] = agg[i] < 0 ? 1 : 0;
}
__global__ void k_amg_singletons(long n, const int *__restrict__ rank, int nroot, int *__restrict__ agg) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    if (agg[i] < 0) agg[i] = nroot + rank[i];
}
// Galerkin expansion: (agg_i * nc + agg_j, a_ij) in CSR order
__global__ void k_amg_expand(long n, const int *__restrict__ rp, const int *__restrict__ ci,
                             const double *__restrict__ va, const int *__restrict__ agg, long long nc,
                             unsigned long long *__restrict__ keys, double *__restrict__ vals) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const long long ai = agg[i];
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      keys[k] = (unsigned long long)(ai * nc + agg[ci[k]]);
      vals[k] = va[k];
    }
  }
}
// in-order reduction of runs of equal (sorted) keys: run starts are flagged
__global__ void k_amg_run_flags(long m, const unsigned long long *__restrict__ keys, int *__restrict__ flag) {
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (long)gridDim.x * blockDim.x)
    flag[k] = (k == 0 || keys[k] != keys[k - 1]) ? 1 : 0;
}
__global__ void k_amg_run_reduce(long m, const unsigned long long *__restrict__ keys, const double *__restrict__ vals,
                                 const int *__restrict__ flag, const int *__restrict__ pos, long long nc,
                                 int *__restrict__ crow, int *__restrict__ cci, double *__restrict__ cva) {
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (long)gridDim.x * blockDim.x) {
    if (!flag[k]) continue;
    double s = 0.0;
    long e = k;
    while (e < m && keys[e] == keys[k]) s += vals[e++];
    const int o = pos[k];
    crow[o] = (int)(keys[k] / nc);
    cci[o] = (int)(keys[k] % nc);
    cva[o] = s;
  }
}
__global__ void k_amg_row_count(long nnz, const int *__restrict__ row, int *__restrict__ cnt) {
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (long)gridDim.x * blockDim.x)
    atomicAdd(cnt + row[k], 1);
}
// members of each aggregate in index order: scatter i into slot off[agg]+fill, then sort slots
__global__ void k_amg_members(long n, const int *__restrict__ agg, const int *__restrict__ moff,
                              int *__restrict__ fill, int *__restrict__ mem) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const int a = agg[i];
    mem[moff[a] + atomicAdd(fill + a, 1)] = (int)i;
  }
}
__global__ void k_amg_sort_members(long nc, const int *__restrict__ moff, int *__restrict__ mem) {
  for (long a = (long)blockIdx.x * blockDim.x + threadIdx.x; a < nc; a += (long)gridDim.x * blockDim.x) {
    for (int p = moff[a] + 1; p < moff[a + 1]; ++p) {
      const int v = mem[p];
      int q = p - 1;
      while (q >= moff[a] && mem[q] > v) {
        mem[q + 1] = mem[q];
        --q;
      }
      mem[q + 1] = v;
    }
  }
}
// dense [A | I] of the coarsest level from CSR (n x 2n, row-major)
__global__ void k_amg_dense(long n, const int *__restrict__ rp, const int *__restrict__ ci,
                            const double *__restrict__ va, double *__restrict__ D) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    double *row = D + i * 2 * n;
    for (long j = 0; j < 2 * n; ++j) row[j] = (j - n == i) ? 1.0 : 0.0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) row[ci[k]] = va[k];
  }
}
// Gauss-Jordan without pivoting (SPD) on the augmented [A | I] (n x 2n, row-major),
// one pivot per launch pair: k_amg_gj_pivot copies the scaled pivot row and the
// pivot column into side buffers, k_amg_gj_update eliminates every other row from
// them (no reads of D that another thread writes in the same launch).
__global__ void k_amg_gj_pivot(long n, long k, const double *__restrict__ D, double *__restrict__ piv,
                               double *__restrict__ col, int *err) {
  const double p = D[k * 2 * n + k];
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 && !(p > 0.0)) atomicExch(err, 1);
  if (i < 2 * n) piv[i] = D[k * 2 * n + i] / p;
  if (i < n) col[i] = D[i * 2 * n + k];
}
__global__ void k_amg_gj_update(long n, long k, double *__restrict__ D, const double *__restrict__ piv,
                                const double *__restrict__ col) {
  const long i = blockIdx.y;
  // columns < k of the left half are already eliminated and columns > n + k of the
  // right half are still zero in every row: only [k, n + k] changes
  const long j = k + (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j > n + k) return;
  double *row = D + i * 2 * n;
  if (i == k)
    row[j] = piv[j];
  else
    row[j] = fma(-col[i], piv[j], row[j]);
}
__global__ void k_amg_gj_extract(long n, const double *__restrict__ D, double *__restrict__ inv) {
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < n * n; t += (long)gridDim.x * blockDim.x) {
    const long i = t / n, j = t % n;
    inv[t] = D[i * 2 * n + n + j];
  }
}

// ---------------------------------------------------------------------------
// Smoothed aggregation (level 0, oracle/amg.py smoothed_prolongator):
//   P = (I - omega D^-1 A) T,  A_c = P^T (A P); every product is expanded into
//   (key, value) pairs in a fixed order, stable-radix-sorted and run-reduced.
// ---------------------------------------------------------------------------
// A T: (i nc + agg_j, a_ij)
__global__ void k_sa_expand_at(long n, const int *__restrict__ rp, const int *__restrict__ ci,
                               const double *__restrict__ va, const int *__restrict__ agg, long long nc,
                               unsigned long long *__restrict__ keys, double *__restrict__ vals) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      keys[k] = (unsigned long long)(i * nc + agg[ci[k]]);
      vals[k] = va[k];
    }
  }
}
// P values from (A T) entries in place: p = [col == agg_row] - omega dinv_row (A T)
__global__ void k_sa_pvals(long nnz, const int *__restrict__ row, const int *__restrict__ col,
                           const int *__restrict__ agg, const double *__restrict__ dinv, double omega,
                           double *__restrict__ va) {
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (long)gridDim.x * blockDim.x) {
    const int i = row[k];
    va[k] = (col[k] == agg[i] ? 1.0 : 0.0) - omega * dinv[i] * va[k];
  }
}
// count / fill of the expansion of A P: row i emits sum_{j in A_i} |P_j| products
__global__ void k_sa_count_ap(long n, const int *__restrict__ arp, const int *__restrict__ aci,
                              const int *__restrict__ prp, long long *__restrict__ cnt) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    long long s = 0;
    for (int k = arp[i]; k < arp[i + 1]; ++k) s += prp[aci[k] + 1] - prp[aci[k]];
    cnt[i] = s;
  }
}
__global__ void k_sa_fill_ap(long n, const int *__restrict__ arp, const int *__restrict__ aci,
                             const double *__restrict__ ava, const int *__restrict__ prp,
                             const int *__restrict__ pci, const double *__restrict__ pva,
                             const long long *__restrict__ off, long long nc, unsigned long long *__restrict__ keys,
                             double *__restrict__ vals) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    long long o = off[i];
    for (int k = arp[i]; k < arp[i + 1]; ++k) {
      const int j = aci[k];
      const double a = ava[k];
      for (int q = prp[j]; q < prp[j + 1]; ++q) {
        keys[o] = (unsigned long long)(i * nc + pci[q]);
        vals[o] = a * pva[q];
        ++o;
      }
    }
  }
}
// count / fill of the expansion of P^T Q (Q = A P): row i emits |P_i| |Q_i| products (a nc + b, p_ia q_ib)
__global__ void k_sa_count_ptq(long n, const int *__restrict__ prp, const int *__restrict__ qrp,
                               long long *__restrict__ cnt) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    cnt[i] = (long long)(prp[i + 1] - prp[i]) * (qrp[i + 1] - qrp[i]);
}
__global__ void k_sa_fill_ptq(long n, const int *__restrict__ prp, const int *__restrict__ pci,
                              const double *__restrict__ pva, const int *__restrict__ qrp,
                              const int *__restrict__ qci, const double *__restrict__ qva,
                              const long long *__restrict__ off, long long nc, unsigned long long *__restrict__ keys,
                              double *__restrict__ vals) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    long long o = off[i];
    for (int a = prp[i]; a < prp[i + 1]; ++a)
      for (int b = qrp[i]; b < qrp[i + 1]; ++b) {
        keys[o] = (unsigned long long)((long long)pci[a] * nc + qci[b]);
        vals[o] = pva[a] * qva[b];
        ++o;
      }
  }
}
// P^T as (col n + row, p) pairs
__global__ void k_sa_expand_pt(long n, const int *__restrict__ prp, const int *__restrict__ pci,
                               const double *__restrict__ pva, unsigned long long *__restrict__ keys,
                               double *__restrict__ vals) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    for (int k = prp[i]; k < prp[i + 1]; ++k) {
      keys[k] = (unsigned long long)((long long)pci[k] * n + i);
      vals[k] = pva[k];
    }
}
