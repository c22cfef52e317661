/*
 * vem_mixed.h — C ABI of the B200 (sm_100a) block-preconditioned GMRES solver
 * for the mixed virtual element saddle-point system
 *
 *        [ M  B^T ] [u]   [g]
 *        [ B   0  ] [p] = [f]                         PAPER.md P:952-961 (C = 0)
 *
 * produced by the order-k mixed VEM of PAPER.md §4 (M = velocity mass matrix,
 * eqn a_{h,P}; B = discrete divergence).
 *
 * The solve is right-preconditioned GMRES(m) (FGMRES(m) for Block-Reg), the
 * Krylov method of P:962, with the two block-diagonal preconditioners of
 * P:963-985:
 *   Block-Schur: B_1 = diag(M); B_2 = S = -B diag(M)^-1 B^T, whose
 *     inverse is applied by a fixed-degree Jacobi-preconditioned Chebyshev
 *     iteration on S_D = B diag(M)^-1 B^T (reading R15; the paper
 *     uses an exact MUMPS solve).
 *   Block-Reg: B_2^-1 = (eps W)^-1; B_1^-1 = (diag(M) + B^T (eps W)^-1 B)^-1
 *     applied by the Woodbury identity with an inner PCG on S_D + eps W,
 *     preconditioned by one V-cycle of S_D + eps W or by its element-block Jacobi
 *     (readings R16, R23; the paper uses GAMG on A + B^T W^-1 B).
 *   Block-Reg-M (kind 5, reading R24): the same B_2, and B_1^-1 y = PCG on the
 *     paper's regularised velocity block K = M + B^T (eps W)^-1 B itself
 *     (P:981-984), preconditioned by the kind-2 B_1, to a relative tolerance
 *     k_rtol: the M-aware stand-in for GAMG where diag(M) is a poor model of M
 *     (anisotropic K, config C5).
 *
 * Everything runs in FP64 on the CUDA device; there is no CPU fallback.  A
 * host-side CSR input is copied to the device during upload; every later step
 * (format build, S_D product, preconditioners, Arnoldi, Givens, restarts)
 * runs in this library's kernels.
 *
 * Status codes (int return): see VEM_* below; vem_status_string() names them,
 * vem_last_error() returns the last detailed message of a context.
 */
#ifndef VEM_MIXED_H
#define VEM_MIXED_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  VEM_OK = 0,
  VEM_NOT_CONVERGED = 1,   /* maxit reached: the last iterate is written, report filled */
  VEM_BREAKDOWN = 2,       /* Arnoldi breakdown at the first step of a cycle            */
  VEM_ERR_INVALID = -1,    /* NULL / size mismatch / unsorted or out-of-range indices / eps<=0   */
  VEM_ERR_DIAG_M = -2,     /* non-positive diag(M)                                       */
  VEM_ERR_DIAG_S = -3,     /* non-positive diag(S_D) (B rank deficient)                          */
  VEM_ERR_CUDA = -4,       /* CUDA error or out of device memory                                 */
  VEM_ERR_PRECOND = -5,    /* unsupported precond_kind                                           */
  VEM_ERR_INNER = -6       /* Block-Reg inner PCG did not reach inner_rtol in inner_maxit        */
};

/* 3: Block-Schur with one aggregation V-cycle on S_D in place of the Chebyshev
 * iteration (the GPU-native stand-in for the exact MUMPS solve of S, P:978;
 * DESIGN.md reading R22; n_p_dof = 1 only, and only for a non-singular S_D: with pure
 * Neumann data B^T annihilates the constant pressure, the coarsest level has no dense
 * inverse, upload succeeds without the hierarchy and kinds 3 / 4 return VEM_ERR_PRECOND). */
enum { VEM_PRECOND_NONE = 0, VEM_PRECOND_BLOCK_SCHUR = 1, VEM_PRECOND_BLOCK_REG = 2, VEM_PRECOND_BLOCK_SCHUR_AMG = 3,
       /* kind 3 with the V-cycle in FP32 (hierarchy values and vectors), GMRES and the
        * saddle operator in FP64: the mixed-precision preconditioner of SURVEY.md §8(f) N4 */
       VEM_PRECOND_BLOCK_SCHUR_AMG_F32 = 4,
       /* Block-Reg with the M-aware velocity block: B_1^-1 = PCG on K = M + B^T (eps W)^-1 B
        * preconditioned by the kind-2 Woodbury block (reading R24) */
       VEM_PRECOND_BLOCK_REG_M = 5 };

typedef struct vem_ctx vem_ctx;    /* opaque; owns every device buffer it allocates */

/* Host CSR matrix, caller-owned, read during upload only.  Rows sorted by
 * column, no duplicates, 0-based.  indptr has n_rows + 1 entries. */
typedef struct {
  int64_t n_rows, n_cols, nnz;
  const int64_t *indptr;
  const int32_t *indices;
  const double *values;
} vem_csr;

/* DOF layout of the assembled system: velocity =
 * [n_faces * n_face_dof face moments | n_elems * n_int_dof interior moments],
 * pressure = n_elems * n_p_dof moments.  Used for validation and reporting. */
typedef struct {
  int32_t k, n_face_dof, n_int_dof, n_p_dof;
  int64_t n_faces, n_elems;
} vem_layout;

typedef struct {
  int32_t restart;        /* m, GMRES(m) restart length, 1..100 (default 30)              */
  int32_t cheb_degree;    /* d, Chebyshev degree of the Block-Schur B_2 apply (default 16) */
  double  cheb_ratio;     /* lambda_max / lambda_min of the Chebyshev interval (default 30) */
  double  inner_rtol;     /* Block-Reg inner PCG relative tolerance (default 1e-14)        */
  int32_t inner_maxit;    /* Block-Reg inner PCG iteration cap (default 10000)             */
  int32_t use_graphs;     /* 1: replay GMRES cycles / PCG chunks as CUDA graphs (default)  */
  int32_t timing;         /* 1: time every launch with CUDA events (no graphs);
                             2: sampled, graph-compatible: the middle Chebyshev step of
                                every Arnoldi step is bracketed by events (k = 0 path);
                                kinds 2 / 5 with the V-cycle inner PCG: one fine-level pass
                                (class MG_FINE) per graph replay of the inner PCG          */
  int32_t pcg_chunk;      /* PCG steps per host convergence poll (default 16)              */
  int32_t reorth;         /* -1 auto (default): CGS2 for the Block-Reg FGMRES (kinds 2, 5), CGS1
                             otherwise, including the FP32-V-cycle FGMRES (kind 4); 1: CGS2
                             always; 0: CGS1 always.  The CGS grids are sized to one wave of
                             resident CTAs (env VEM_MDOT_WAVE / VEM_UPDATE_WAVE = 0: fixed grids),
                             so the partial-sum tree depends on the device and the build    */
  int32_t l2_persist;     /* 1 (default): persisting L2 window over the Chebyshev vectors  */
  int32_t reorder;        /* 1 (default): SELL-C-sigma symmetric reordering of the unknowns
                             at upload when n_p_dof > 1 and it removes >= 5% slice padding
                             (rows sorted by length in 4096-row windows, element blocks
                             kept whole); invisible to the caller (rhs, u, p and every
                             operator entry point stay in the caller's numbering); 0: off */
  int32_t inner_precond;  /* Block-Reg inner PCG preconditioner: 1 (default) one V-cycle of
                             S_D + eps W (n_p_dof = 1: the kind-3 aggregation hierarchy built
                             on S_D + eps W; n_p_dof > 1: element-block-Jacobi Chebyshev(2) on [1/3, 2]
                             smoothing + injection of the element-mean moment + that hierarchy
                             on the mean-moment block; reading R23); 0: element-block Jacobi */
  int32_t k_maxit;        /* kind 5: iteration cap of the PCG on K per apply (default 500)  */
  double  k_rtol;         /* kind 5: the PCG on K stops at sqrt(r.z) <= k_rtol sqrt(r0.z0)
                             (default 0.1)                                                 */
  double  k_inner_rtol;   /* kind 5: tolerance of the inner PCG on S_D + eps W inside the
                             Woodbury preconditioner of the PCG on K (default 1e-8: errors of
                             that solve are amplified by lambda(S_D) / eps in K)            */
  int32_t mg_chunk;       /* MG-PCG steps per host convergence poll (default 2)             */
  int32_t basis_f32;      /* 1: compressed Krylov basis: every basis vector is
                             the float32 rounding of the vector Arnoldi produced, used as such by
                             every reader; the CGS kernels stream the float copy (half the bytes),
                             all arithmetic stays FP64, and the true-residual restart recovers the
                             full accuracy (a cycle reduces the residual by about 1e-6 at most, so
                             solves that converged inside one cycle need one more); 0 (default) */
} vem_opts;

typedef struct {
  int32_t status;                 /* same value as the return code                       */
  int32_t iterations;             /* total Arnoldi steps                          */
  int32_t restarts;
  int32_t converged;
  int32_t breakdown;
  int32_t cycles;
  int64_t inner_iterations;       /* Block-Reg: total inner PCG steps (on S_D + eps W)    */
  int64_t k_iterations;           /* kind 5: total steps of the PCG on K                   */
  double  rel_residual_true;      /* ||b - A x|| / ||b|| at exit                           */
  double  rel_residual_est;       /* last Givens estimate |g_{j+1}| / ||b||               */
  double  setup_ms;               /* upload + device format / S_D build                   */
  double  solve_ms;               /* CUDA-event time of the solve on the caller's stream  */
} vem_solve_report;

typedef struct {
  int64_t n_u, n_p, nnz_M, nnz_B, nnz_A, nnz_S;
  double  lambda_max;             /* Gershgorin bound of diag(S_D)^-1 S_D                 */
  double  eps;                    /* Block-Reg regularisation as uploaded                 */
  int32_t spmv_group, schur_group;/* lanes per row of the CSR kernels                     */
  int32_t sm_count;
  int64_t device_bytes;           /* device memory owned by the context                   */
  int64_t l2_window_bytes;        /* bytes under the persisting L2 access window          */
  int32_t amg_levels;             /* levels of the S_D hierarchy (0: kind 3 unavailable)   */
  int64_t amg_coarsest;           /* rows of its coarsest level                            */
  int32_t reordered;              /* 1 if the SELL-C-sigma reordering is active            */
  int32_t amg_coarse_cluster;     /* 1 if the non-dense coarsest level is smoothed by one
                                     16-CTA thread-block-cluster launch (k_vc_coarse_cluster) */
  int64_t nnz_A_stored, nnz_S_stored; /* stored SELL-32 slots (nonzeros + slice padding)   */
} vem_info;

/* Kernel classes for the per-launch CUDA-event statistics (opts.timing = 1). */
enum {
  VEM_K_SPMV = 0,       /* fused saddle SpMV y = A x (and residual b - A x)      */
  VEM_K_CHEB = 1,       /* Chebyshev step on S_D (Block-Schur B_2)               */
  VEM_K_PCG_SPMV = 2,   /* PCG step: p update + (S_D + eps W) p + p.q            */
  VEM_K_PCG_VEC = 3,    /* PCG step: x, r updates + r.z, r.r                     */
  VEM_K_DOT = 4,        /* CGS multi-dot V^T w                                   */
  VEM_K_UPDATE = 5,     /* CGS update w -= V h (+ norm, Givens)                  */
  VEM_K_PRECOND_VEC = 6,/* diagonal scalings, Woodbury pieces, Chebyshev init    */
  VEM_K_CYCLE = 7,      /* cycle end: back-substitution, x update                */
  VEM_K_MG_FINE = 8,    /* fine-level pass of the inner V-cycle: b - (S_D + eps W) d */
  VEM_NUM_KCLASS = 9
};

/* bytes[] is the ALGORITHMIC HBM traffic of the timed launches:
 *   SPMV      12 nnz(A) + 16 n                    (values+indices, x once, y)
 *   CHEB      12 nnz(S) + 56 n_p                  (S, D^-1, r rw, d_old, d_new, x rw)
 *   PCG_SPMV  12 nnz(S) + 56 n_p                  (S, D^-1, W, r, p_prev, p_new, q)
 *   PCG_VEC   64 n_p                               (D^-1, p, q, x rw, r rw)
 *   DOT       8 n (nv + 1)                         (nv basis vectors + w)
 *   UPDATE    8 n (nv + 2)                         (nv basis vectors + w rw)
 *   MG_FINE   12 nnz(S) + 32 n_p                   (S, W, d, b, out)
 * other classes count the vectors they stream once. */
typedef struct {
  int64_t launches[VEM_NUM_KCLASS];
  double  ms[VEM_NUM_KCLASS];
  double  bytes[VEM_NUM_KCLASS];
} vem_kernel_stats;

void vem_mixed_default_options(vem_opts *opts);

/* Copy M (n_u x n_u), B (n_p x n_u) and optionally a diagonal W (n_p x n_p,
 * NULL = identity) to the device on `cuda_stream` (a cudaStream_t, e.g.
 * torch.cuda.current_stream().cuda_stream; NULL = default stream), build the
 * device formats, diag(M)^-1, S_D = B diag(M)^-1 B^T (device SpGEMM), diag(S_D),
 * lambda_max and, if eps > 0, the Block-Reg pieces.  eps <= 0 disables
 * Block-Reg.  On success *ctx owns all device memory; on failure *ctx = NULL. */
int vem_mixed_upload(vem_ctx **ctx, const vem_csr *M, const vem_csr *B, const vem_csr *W,
                     double eps, const vem_layout *layout, const vem_opts *opts,
                     void *cuda_stream);

/* Solve A [u; p] = rhs from x0 = 0 to ||b - A x|| <= tol ||b|| (Givens estimate
 * checked every step, confirmed by the true residual at each cycle end).
 * rhs (n_u + n_p), out_u (n_u), out_p (n_p): caller-owned DEVICE pointers
 * (never freed by the library).  maxit caps the total Arnoldi steps.  The
 * stream is synchronised before return.  report (host) may be NULL.
 * precond_kind (readings R15-R17, R22):
 *   0 none; 1 Block-Schur, B_2^-1 by degree-d Chebyshev on S_D (GMRES);
 *   2 Block-Reg, Woodbury with an inner PCG (FGMRES, CGS2);
 *   3 Block-Schur, B_2^-1 by one smoothed-aggregation V-cycle on S_D (GMRES; n_p_dof = 1);
 *   4 kind 3 with the V-cycle in FP32 (FGMRES; n_p_dof = 1).
 * Errors: VEM_ERR_PRECOND for an unknown kind, kind 2 without eps > 0, kinds 3/4
 * without the hierarchy (n_p_dof > 1); VEM_ERR_INNER if the inner PCG fails. */
int vem_mixed_solve(vem_ctx *ctx, const double *rhs, double tol, int32_t maxit,
                    int32_t precond_kind, double *out_u, double *out_p,
                    vem_solve_report *report);

/* Same solve with HOST buffers: rhs is copied host->device and u, p
 * device->host inside the call (end-to-end path). */
int vem_mixed_solve_host(vem_ctx *ctx, const double *rhs_host, double tol, int32_t maxit,
                         int32_t precond_kind, double *u_host, double *p_host,
                         vem_solve_report *report);

/* y = A x for device x, y of length n_u + n_p (the fused saddle SpMV). */
int vem_mixed_spmv(vem_ctx *ctx, const double *x, double *y);

/* y = S_D x for device x, y of length n_p (checks the device S_D product). */
int vem_mixed_schur_spmv(vem_ctx *ctx, const double *x, double *y);

/* z = P^-1 v (device, length n_u + n_p) for precond_kind; inner_its (host,
 * may be NULL) receives the Block-Reg inner PCG step count. */
int vem_mixed_precond_apply(vem_ctx *ctx, int32_t precond_kind, const double *v, double *z,
                            int64_t *inner_its);

int vem_mixed_set_options(vem_ctx *ctx, const vem_opts *opts);
int vem_mixed_get_options(vem_ctx *ctx, vem_opts *opts);
int vem_mixed_get_info(vem_ctx *ctx, vem_info *info);

/* Copy S_D back to host CSR arrays sized from vem_info (n_p + 1, nnz_S, nnz_S). */
int vem_mixed_get_schur(vem_ctx *ctx, int64_t *indptr, int32_t *indices, double *values);

/* Per-kernel-class launch counts and CUDA-event milliseconds accumulated while
 * opts.timing = 1; reset != 0 clears them after copying. */
int vem_mixed_kernel_stats(vem_ctx *ctx, vem_kernel_stats *stats, int32_t reset);

/* Size of level `level` of the S_D aggregation hierarchy (kind 3): rows and
 * nonzeros; VEM_ERR_INVALID if the level does not exist. */
int vem_mixed_amg_level(vem_ctx *ctx, int32_t level, int64_t *n, int64_t *nnz);

/* The same for the S_D + eps W hierarchy that preconditions Block-Reg's inner PCG
 * (opts.inner_precond = 1, reading R23; level 0 is S_D + eps W itself when
 * n_p_dof = 1 and its element-mean block (S_D + eps W)[0::n_p, 0::n_p] otherwise).
 * VEM_ERR_INVALID if the level does not exist (always, when eps <= 0 at upload). */
int vem_mixed_inner_amg_level(vem_ctx *ctx, int32_t level, int64_t *n, int64_t *nnz);

/* Givens residual estimates |g_{j+1}| / ||rhs|| of the Arnoldi steps of
 * the LAST GMRES cycle the last vem_mixed_solve ran, rebuilt from the device-resident sines:
 * |g_{j+1}| = |s_j| |g_j|, g_0 = the residual norm the cycle started from.  hist (host, cap
 * doubles, caller-owned) receives min(cap, *count) values; *count = steps of that cycle. */
int vem_mixed_last_cycle_history(vem_ctx *ctx, double *hist, int32_t cap, int32_t *count);

/* ---------------------------------------------------------------------------
 * Element-parallel assembly on the device
 * for classes of congruent cells (translates of one cell: cube grids, cube pairs),
 * from each class's shape cache (host, vemgen.assemble.class_template).  Cell e of a
 * class contributes
 *   M[dof[e][ti[t]], dof[e][tj[t]]] += ((coef[e][0] tA[t] + coef[e][1] tA[n_t + t])
 *                                       + coef[e][2] tA[2 n_t + t]) + coef[e][3] tS[t]
 *   B[pdof[e][bi[t]], dof[e][bj[t]]] += tB[t]
 *   f[pdof[e][a]] = -vol[e] sum_b Hinv[a][b] F[e][b]
 * coef = (1/K_x, 1/K_y, 1/K_z, s_P) per cell (readings R4, R7); every product is
 * rounded separately (no FMA); duplicates are summed in (class, cell, entry) order.
 * All pointers are HOST arrays, copied during the call; row-major. */
typedef struct {
  int64_t n_cells;
  int32_t n_loc, n_p;          /* local velocity DOFs, pressure DOFs per cell          */
  const int32_t *dof;          /* n_cells x n_loc global velocity DOFs                 */
  const int32_t *pdof;         /* n_cells x n_p global pressure DOFs                    */
  int32_t n_t;                 /* M template entries                                    */
  const int32_t *ti, *tj;      /* n_t local (row, col)                                  */
  const double *tA;            /* 3 x n_t consistency components (K-independent)        */
  const double *tS;            /* n_t stabilisation                                     */
  const double *coef;          /* n_cells x 4                                           */
  int32_t n_b;                 /* B template entries                                    */
  const int32_t *bi, *bj;      /* n_b local (pressure row, velocity col)                */
  const double *tB;            /* n_b                                                   */
  const double *Hinv;          /* n_p x n_p inverse monomial mass (scaled coordinates)  */
  const double *F;             /* n_cells x n_p source moments int_P f m_a              */
  const double *vol;           /* n_cells                                               */
} vem_cell_class;

typedef struct vem_asm vem_asm;  /* opaque: device CSR of M (n_u x n_u), B (n_p x n_u), device f */

/* Assemble on the device (stream semantics as vem_mixed_upload; synchronised before
 * return).  Errors: VEM_ERR_INVALID (NULL pointer, DOF out of range, empty class),
 * VEM_ERR_CUDA.  On success *out owns the device arrays. */
int vem_mixed_assemble(vem_asm **out, const vem_cell_class *classes, int32_t n_classes, int64_t n_u,
                       int64_t n_p, void *cuda_stream);
/* Non-congruent single-tetrahedron classes (Kuhn meshes, C2), k = 0 or 1: the local
 * operators themselves (face polynomials, divergence, Pi^0_k via
 * Props. 1-3 and P:478-490, consistency + dofi-dofi stabilisation; the batched small
 * dense solves) are computed on the device, one thread per cell, then assembled as
 * above (same drop, reading R11; same (cell, row, col) emission order).  Host arrays
 * (vemgen.assemble.tet_class_input), row-major, copied during the call. */
typedef struct {
  int32_t k;
  int64_t n_cells;
  const double *cell;     /* n_cells x 17: centroid (3), h_P, |P|, the 4 vertices (12)            */
  const double *faces;    /* n_cells x 4 x 23: v0, v1, v2, normal, e1, e2, centroid, area, h_f     */
  const double *signs;    /* n_cells x 4 face orientation signs                                   */
  const double *coef;     /* n_cells x 4: 1/K_x, 1/K_y, 1/K_z, s_P                                */
  const int32_t *dof;     /* n_cells x n_loc                                                       */
  const int32_t *pdof;    /* n_cells x n_p                                                         */
  const double *F;        /* n_cells x n_p source moments                                          */
  int32_t n_qv;           /* reference tetrahedron rule: n_qv x 4 (s, t, r, weight)               */
  const double *vref;
  int32_t n_qf;           /* reference triangle rule: n_qf x 3 (s, t, weight)                     */
  const double *fref;
  const double *alphas1;  /* dim P_{k+1} x 3 graded-lex exponents                                 */
  const double *betas;    /* dim P_k(f) x 2                                                        */
  const double *rgrad;    /* 3 dim P_k x 2: (grad coefficient, index of beta in M_{k+1})          */
  const double *rcross;   /* 3 dim P_k x 4 x 2: (generator, coefficient), generator -1 = unused  */
  const double *dgrad;    /* max(dim P_k - 1, 1) x 3 x 2: (alpha_c, index of alpha - e_c), -1    */
  const double *gens;     /* dim G_k^perp x 2: (component, index of the exponent in M_{k-1})      */
} vem_tet_class;
int vem_mixed_assemble_tets(vem_asm **out, const vem_tet_class *classes, int32_t n_classes, int64_t n_u,
                            int64_t n_p, void *cuda_stream);
/* nnz of the assembled M and B. */
int vem_mixed_assembled_info(const vem_asm *a, int64_t *nnz_M, int64_t *nnz_B);
/* Copy the assembled CSR (int64 indptr, int32 indices, fp64 values; sorted, unique
 * columns) and f to caller-allocated HOST arrays sized from vem_mixed_assembled_info. */
int vem_mixed_assembled_copy(const vem_asm *a, int64_t *m_indptr, int32_t *m_indices, double *m_values,
                             int64_t *b_indptr, int32_t *b_indices, double *b_values, double *f);
/* vem_mixed_upload from an assembled system (device to device; `a` may be freed after). */
int vem_mixed_upload_assembled(vem_ctx **ctx, const vem_asm *a, const vem_csr *W, double eps,
                               const vem_layout *layout, const vem_opts *opts, void *cuda_stream);
void vem_mixed_assembled_free(vem_asm *a);

void vem_mixed_destroy(vem_ctx *ctx);
const char *vem_status_string(int status);
const char *vem_last_error(vem_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* VEM_MIXED_H */
