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

// ---------------------------------------------------------------------------
// Local operators of single tetrahedra on the device (the batched small dense
// Pi / Div solves of vemgen.local.local_operators, one thread per cell), for the
// non-congruent Kuhn classes (C2).  PAPER.md P:663-731 (face polynomial,
// divergence, Pi^0_k by Props. 1-3 and P:478-490), P:768-793 (consistency and
// dofi-dofi stabilisation), RT-type spaces of DESIGN.md reading R1.  The host
// (vemgen.assemble.tet_class_input) supplies geometry, the reference quadrature
// rules and the symbolic tables; every quadrature sum, small solve and product
// runs here.  Entries are emitted in the host generator's (cell, row, col) order
// after the same relative drop (reading R11); exact zeros are emitted with the
// marker key ~0 and removed after the sort.
// ---------------------------------------------------------------------------
constexpr unsigned long long ASM_DROPPED = ~0ULL;

__host__ __device__ constexpr int dim_pk3(int k) { return k < 0 ? 0 : (k + 1) * (k + 2) * (k + 3) / 6; }
__host__ __device__ constexpr int dim_pk2(int k) { return k < 0 ? 0 : (k + 1) * (k + 2) / 2; }
__host__ __device__ constexpr int dim_gp(int k) { return (2 * k * k * k + 9 * k * k + 7 * k) / 6; }

// in-place Gauss-Jordan inverse of a small SPD matrix (no pivoting), row-major n x n
template <int N>
__device__ void small_inv(double (&A)[N][N], double (&X)[N][N]) {
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) X[i][j] = (i == j) ? 1.0 : 0.0;
  for (int k = 0; k < N; ++k) {
    const double p = 1.0 / A[k][k];
    for (int j = 0; j < N; ++j) {
      A[k][j] *= p;
      X[k][j] *= p;
    }
    for (int i = 0; i < N; ++i) {
      if (i == k) continue;
      const double f = A[i][k];
      if (f == 0.0) continue;
      for (int j = 0; j < N; ++j) {
        A[i][j] -= f * A[k][j];
        X[i][j] -= f * X[k][j];
      }
    }
  }
}

__device__ __forceinline__ double ipow(double x, int p) {
  double r = 1.0;
  for (int i = 0; i < p; ++i) r *= x;
  return r;
}

template <int K>
__global__ void __launch_bounds__(64) k_local_tet(
    long E, const double *__restrict__ cell, const double *__restrict__ faces, const double *__restrict__ signs,
    const double *__restrict__ coef, const int *__restrict__ Lmap, const int *__restrict__ Pmap,
    const double *__restrict__ Fsrc, const double *__restrict__ vref, int nqv, const double *__restrict__ fref,
    int nqf, const double *__restrict__ alphas1, const double *__restrict__ betas, const double *__restrict__ rgrad,
    const double *__restrict__ rcross, const double *__restrict__ dgrad, const double *__restrict__ gens,
    long long nu, unsigned long long *__restrict__ mkeys, double *__restrict__ mvals,
    unsigned long long *__restrict__ bkeys, double *__restrict__ bvals, double *__restrict__ fout) {
  constexpr int NK = dim_pk3(K), NK1 = dim_pk3(K + 1), NF = dim_pk2(K), NG = dim_gp(K);
  constexpr int NLOC = 4 * NF + (NK - 1) + NG, OG = 4 * NF, OC = OG + NK - 1;
  const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const double *cg = cell + e * 17;
  const double xP[3] = {cg[0], cg[1], cg[2]}, hP = cg[3], vol = cg[4];
  const double *tv = cg + 5;
  double a3[3], b3[3], c3[3];
  for (int d = 0; d < 3; ++d) {
    a3[d] = tv[3 + d] - tv[d];
    b3[d] = tv[6 + d] - tv[d];
    c3[d] = tv[9 + d] - tv[d];
  }
  const double vol6 = fabs(a3[0] * (b3[1] * c3[2] - b3[2] * c3[1]) - a3[1] * (b3[0] * c3[2] - b3[2] * c3[0]) +
                           a3[2] * (b3[0] * c3[1] - b3[1] * c3[0]));
  int al1[NK1][3];
  for (int b = 0; b < NK1; ++b)
    for (int d = 0; d < 3; ++d) al1[b][d] = (int)alphas1[b * 3 + d];
  // ---- volume integrals: Hp, Hk_k1, and the cross-moment rows of D
  double Hp[NK][NK] = {}, Hk[NK][NK1] = {};
  double D[NLOC][3 * NK] = {};
  for (int q = 0; q < nqv; ++q) {
    const double S = vref[q * 4], T = vref[q * 4 + 1], R = vref[q * 4 + 2], w = vref[q * 4 + 3] * vol6;
    double s[3], mv[NK1];
    for (int d = 0; d < 3; ++d) s[d] = (tv[d] + S * a3[d] + T * b3[d] + R * c3[d] - xP[d]) / hP;
    for (int b = 0; b < NK1; ++b) mv[b] = ipow(s[0], al1[b][0]) * ipow(s[1], al1[b][1]) * ipow(s[2], al1[b][2]);
    for (int a = 0; a < NK; ++a) {
      for (int b = 0; b < NK; ++b) Hp[a][b] += w * mv[a] * mv[b];
      for (int b = 0; b < NK1; ++b) Hk[a][b] += w * mv[a] * mv[b];
    }
    for (int g = 0; g < NG; ++g) {   // field = (s x e_c2) m_al
      const int c2 = (int)gens[g * 2], ia = (int)gens[g * 2 + 1];
      double ec[3] = {0.0, 0.0, 0.0};
      ec[c2] = 1.0;
      const double fld[3] = {(s[1] * ec[2] - s[2] * ec[1]) * mv[ia], (s[2] * ec[0] - s[0] * ec[2]) * mv[ia],
                             (s[0] * ec[1] - s[1] * ec[0]) * mv[ia]};
      for (int c = 0; c < 3; ++c)
        for (int j = 0; j < NK; ++j) D[OC + g][c * NK + j] += w * mv[j] * fld[c] / vol;
    }
  }
  // ---- faces: boundary flux rows Bnd, face rows of D
  double Bnd[NK1][NLOC] = {};
  for (int lf = 0; lf < 4; ++lf) {
    const double *fgm = faces + (e * 4 + lf) * 23;
    const double *v0 = fgm, *v1 = fgm + 3, *v2 = fgm + 6, *nrm = fgm + 9, *e1 = fgm + 12, *e2 = fgm + 15,
                 *cen = fgm + 18;
    const double area = fgm[21], hf = fgm[22];
    const double sig = signs[e * 4 + lf];
    double fa[3], fb[3];
    for (int d = 0; d < 3; ++d) {
      fa[d] = v1[d] - v0[d];
      fb[d] = v2[d] - v0[d];
    }
    const double cx = fa[1] * fb[2] - fa[2] * fb[1], cy = fa[2] * fb[0] - fa[0] * fb[2],
                 cz = fa[0] * fb[1] - fa[1] * fb[0];
    const double area2 = sqrt(cx * cx + cy * cy + cz * cz);
    double Hf[NF][NF] = {}, Phi[NF][NK1] = {}, base[NF][NK] = {};
    for (int q = 0; q < nqf; ++q) {
      const double S = fref[q * 3], T = fref[q * 3 + 1], w = fref[q * 3 + 2] * area2;
      double p[3], dd[3], s[3], mf[NF], m3[NK1];
      for (int d = 0; d < 3; ++d) {
        p[d] = v0[d] + S * fa[d] + T * fb[d];
        dd[d] = p[d] - cen[d];
        s[d] = (p[d] - xP[d]) / hP;
      }
      const double t0 = (dd[0] * e1[0] + dd[1] * e1[1] + dd[2] * e1[2]) / hf;
      const double t1 = (dd[0] * e2[0] + dd[1] * e2[1] + dd[2] * e2[2]) / hf;
      for (int b = 0; b < NF; ++b) mf[b] = ipow(t0, (int)betas[b * 2]) * ipow(t1, (int)betas[b * 2 + 1]);
      for (int b = 0; b < NK1; ++b) m3[b] = ipow(s[0], al1[b][0]) * ipow(s[1], al1[b][1]) * ipow(s[2], al1[b][2]);
      for (int a = 0; a < NF; ++a) {
        for (int b = 0; b < NF; ++b) Hf[a][b] += w * mf[a] * mf[b];
        for (int b = 0; b < NK1; ++b) Phi[a][b] += w * mf[a] * m3[b];
        for (int b = 0; b < NK; ++b) base[a][b] += w * mf[a] * m3[b];
      }
    }
    double Hfi[NF][NF];
    small_inv<NF>(Hf, Hfi);
    for (int b = 0; b < NK1; ++b)
      for (int c = 0; c < NF; ++c) {
        double acc = 0.0;
        for (int a = 0; a < NF; ++a) acc += Phi[a][b] * (area * Hfi[a][c]);
        Bnd[b][lf * NF + c] += sig * acc;
      }
    for (int be = 0; be < NF; ++be)
      for (int c = 0; c < 3; ++c)
        for (int j = 0; j < NK; ++j) D[lf * NF + be][c * NK + j] = nrm[c] * (base[be][j] / area);
  }
  // ---- divergence: Hp Div = r
  double Hpc[NK][NK], Hpi[NK][NK];
  for (int a = 0; a < NK; ++a)
    for (int b = 0; b < NK; ++b) Hpc[a][b] = Hp[a][b];
  small_inv<NK>(Hpc, Hpi);
  double Div[NK][NLOC];
  {
    double r[NK][NLOC];
    for (int a = 0; a < NK; ++a)
      for (int l = 0; l < NLOC; ++l) r[a][l] = Bnd[a][l];
    for (int a = 1; a < NK; ++a) r[a][OG + a - 1] -= vol / hP;
    for (int a = 0; a < NK; ++a)
      for (int l = 0; l < NLOC; ++l) {
        double acc = 0.0;
        for (int b = 0; b < NK; ++b) acc += Hpi[a][b] * r[b][l];
        Div[a][l] = acc;
      }
  }
  // ---- G[b] . chi = int_P v . grad m_b
  double G[NK1][NLOC] = {};
  for (int b = 0; b < NK1; ++b) {
    const int deg = al1[b][0] + al1[b][1] + al1[b][2];
    if (deg == 0) continue;
    if (deg <= K) {
      G[b][OG + b - 1] = vol / hP;
    } else {
      for (int l = 0; l < NLOC; ++l) {
        double acc = 0.0;
        for (int a = 0; a < NK; ++a) acc += Hk[a][b] * Div[a][l];
        G[b][l] = -acc + Bnd[b][l];
      }
    }
  }
  // ---- R rows, Pi = (I3 x Hp)^-1 R
  double Pi[3 * NK][NLOC];
  {
    double R[3 * NK][NLOC] = {};
    for (int row = 0; row < 3 * NK; ++row) {
      const double gc = rgrad[row * 2];
      const int bi = (int)rgrad[row * 2 + 1];
      for (int l = 0; l < NLOC; ++l) R[row][l] += (gc * hP) * G[bi][l];
      for (int t = 0; t < 4; ++t) {
        const int g = (int)rcross[(row * 4 + t) * 2];
        if (g >= 0) R[row][OC + g] += rcross[(row * 4 + t) * 2 + 1] * vol;
      }
    }
    for (int c = 0; c < 3; ++c)
      for (int a = 0; a < NK; ++a)
        for (int l = 0; l < NLOC; ++l) {
          double acc = 0.0;
          for (int b = 0; b < NK; ++b) acc += Hpi[a][b] * R[c * NK + b][l];
          Pi[c * NK + a][l] = acc;
        }
  }
  // ---- gradient rows of D: (1/|P|) a_c int m_j m_{a - e_c}
  for (int a = 1; a < NK; ++a)
    for (int c = 0; c < 3; ++c) {
      const double ac = dgrad[((a - 1) * 3 + c) * 2];
      if (ac <= 0.0) continue;
      const int im = (int)dgrad[((a - 1) * 3 + c) * 2 + 1];
      for (int j = 0; j < NK; ++j) D[OG + a - 1][c * NK + j] = ac * Hp[j][im] / vol;
    }
  // ---- HPi_c = Hp Pi_c ; IDP = I - D Pi
  double HPi[3 * NK][NLOC];
  for (int c = 0; c < 3; ++c)
    for (int a = 0; a < NK; ++a)
      for (int l = 0; l < NLOC; ++l) {
        double acc = 0.0;
        for (int b = 0; b < NK; ++b) acc += Hp[a][b] * Pi[c * NK + b][l];
        HPi[c * NK + a][l] = acc;
      }
  double IDP[NLOC][NLOC];
  for (int i = 0; i < NLOC; ++i)
    for (int l = 0; l < NLOC; ++l) {
      double acc = 0.0;
      for (int m = 0; m < 3 * NK; ++m) acc += D[i][m] * Pi[m][l];
      IDP[i][l] = (i == l ? 1.0 : 0.0) - acc;
    }
  // A_c(i, j) = sum_a Pi_c[a][i] HPi_c[a][j];  S(i, j) = sum_m IDP[m][i] IDP[m][j]
  auto Aij = [&](int c, int i, int j) {
    double acc = 0.0;
    for (int a = 0; a < NK; ++a) acc += Pi[c * NK + a][i] * HPi[c * NK + a][j];
    return acc;
  };
  auto Sij = [&](int i, int j) {
    double acc = 0.0;
    for (int m = 0; m < NLOC; ++m) acc += IDP[m][i] * IDP[m][j];
    return acc;
  };
  double mxA[3] = {0.0, 0.0, 0.0}, mxS = 0.0, mxB = 0.0;
  for (int i = 0; i < NLOC; ++i)
    for (int j = 0; j < NLOC; ++j) {
      for (int c = 0; c < 3; ++c) mxA[c] = fmax(mxA[c], fabs(Aij(c, i, j)));
      mxS = fmax(mxS, fabs(Sij(i, j)));
    }
  for (int a = 0; a < NK; ++a)
    for (int l = 0; l < NLOC; ++l) mxB = fmax(mxB, fabs(-vol * Div[a][l]));
  const double *cf = coef + e * 4;
  const int *Le = Lmap + e * NLOC;
  const int *Pe = Pmap + e * NK;
  const long mo = e * (long)NLOC * NLOC;
  for (int i = 0; i < NLOC; ++i)
    for (int j = 0; j < NLOC; ++j) {
      double v = 0.0;
      for (int c = 0; c < 3; ++c) {
        double a = Aij(c, i, j);
        if (fabs(a) <= 1e-14 * mxA[c]) a = 0.0;
        v += cf[c] * a;
      }
      double sv = Sij(i, j);
      if (fabs(sv) <= 1e-14 * mxS) sv = 0.0;
      v += cf[3] * sv;
      const long q = mo + (long)i * NLOC + j;
      mkeys[q] = v != 0.0 ? (unsigned long long)((long long)Le[i] * nu + Le[j]) : ASM_DROPPED;
      mvals[q] = v;
    }
  const long bo = e * (long)NK * NLOC;
  for (int a = 0; a < NK; ++a)
    for (int l = 0; l < NLOC; ++l) {
      double v = -vol * Div[a][l];
      if (fabs(v) <= 1e-14 * mxB) v = 0.0;
      const long q = bo + (long)a * NLOC + l;
      bkeys[q] = v != 0.0 ? (unsigned long long)((long long)Pe[a] * nu + Le[l]) : ASM_DROPPED;
      bvals[q] = v;
    }
  for (int a = 0; a < NK; ++a) {
    double acc = 0.0;
    for (int b = 0; b < NK; ++b) acc += Hpi[a][b] * Fsrc[e * NK + b];
    fout[Pe[a]] = -vol * acc;
  }
}
