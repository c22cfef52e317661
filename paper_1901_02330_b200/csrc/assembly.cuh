// assembly.cuh — element-parallel assembly of M, B and f on the device
// (SURVEY.md §8(f) N2), for classes of congruent cells (cube grids, cube pairs)
// from their host shape cache (vemgen.assemble.class_template).
//
// a_h(u, v) = sum_P [consistency + stabilisation],
// b_h(v, q) = sum_P (div v, q)_P, (f, q)_P.  Cell e of a class contributes
//   M[dof[e][ti]] [dof[e][tj]] += ((c_e0 A0 + c_e1 A1) + c_e2 A2) + c_e3 S
//   B[pdof[e][bi]][dof[e][bj]] += Bt
//   f[pdof[e][a]] = -vol_e sum_b Hinv[a][b] F_e[b]
// with c_e = (1/K_x, 1/K_y, 1/K_z, s_P) (readings R4, R7).  Every
// product is rounded separately (no FMA contraction) so a value is the same
// double the host generator computes; duplicates are summed by the stable
// (key, value) radix sort + in-order run reduction of vem_mixed.cu in
// (class, cell, entry) order.
#pragma once
#include <cstdint>

__global__ void k_asm_m(long ne, int nloc, int nt, const int *__restrict__ dof, const int *__restrict__ ti,
                        const int *__restrict__ tj, const double *__restrict__ tA, const double *__restrict__ tS,
                        const double *__restrict__ coef, long long ncols, unsigned long long *__restrict__ keys,
                        double *__restrict__ vals) {
  const long m = ne * (long)nt;
  for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (long)gridDim.x * blockDim.x) {
    const long e = q / nt;
    const int t = (int)(q - e * nt);
    const long long row = dof[e * nloc + ti[t]], col = dof[e * nloc + tj[t]];
    const double *c4 = coef + e * 4;
    const double v = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(c4[0], tA[t]), __dmul_rn(c4[1], tA[nt + t])),
                                         __dmul_rn(c4[2], tA[2 * nt + t])),
                               __dmul_rn(c4[3], tS[t]));
    keys[q] = (unsigned long long)(row * ncols + col);
    vals[q] = v;
  }
}

__global__ void k_asm_b(long ne, int nloc, int np, int nb, const int *__restrict__ dof,
                        const int *__restrict__ pdof, const int *__restrict__ bi, const int *__restrict__ bj,
                        const double *__restrict__ tB, long long ncols, unsigned long long *__restrict__ keys,
                        double *__restrict__ vals) {
  const long m = ne * (long)nb;
  for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (long)gridDim.x * blockDim.x) {
    const long e = q / nb;
    const int t = (int)(q - e * nb);
    const long long row = pdof[e * np + bi[t]], col = dof[e * nloc + bj[t]];
    keys[q] = (unsigned long long)(row * ncols + col);
    vals[q] = tB[t];
  }
}

__global__ void k_asm_f(long ne, int np, const int *__restrict__ pdof, const double *__restrict__ Hinv,
                        const double *__restrict__ F, const double *__restrict__ vol, double *__restrict__ f) {
  const long m = ne * (long)np;
  for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (long)gridDim.x * blockDim.x) {
    const long e = q / np;
    const int a = (int)(q - e * np);
    double s = 0.0;
    for (int b = 0; b < np; ++b) s = __dadd_rn(s, __dmul_rn(Hinv[a * np + b], F[e * np + b]));
    f[pdof[e * np + a]] = __dmul_rn(-vol[e], s);
  }
}

__global__ void k_widen64(long n, const int *__restrict__ in, int64_t *__restrict__ out) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    out[i] = in[i];
}
