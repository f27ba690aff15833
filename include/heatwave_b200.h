/*
 * heatwave_b200.h -- C ABI of the B200 space-time PCG hot path.
 *
 * Drop-in boundary for the reference package `heatwave`
 * (/root/reference/pkg/src/heatwave).  The reference has no formal plugin
 * API: its hot path sits behind a duck-typed operator protocol consumed by
 * `pcg` and behind numba kernels on flat numpy arrays.  Each
 * entry point below replaces one of those call sites; the Python mirror in
 * paper_2009_08875_b200/ binds them with ctypes and maps return codes to the
 * reference's exceptions.
 *
 * Conventions
 *  - Space-time arrays are fp64, C-contiguous (rows, N_x): row j holds the
 *    spatial coefficients of temporal DOF j (sparse.py:132-175).
 *  - Every array pointer is a DEVICE pointer unless the name says `host`.
 *    The caller owns inputs and outputs; the context owns its workspaces
 *    (system.py:93-101: one solve per operator instance at a time).
 *  - `stream` is a cudaStream_t passed as void*; NULL = legacy default.
 *    All work is stream-ordered; calls return once the work is enqueued,
 *    except hwg_pcg (which reads two scalars back per iteration) and
 *    hwg_dot (which returns a host scalar).
 *  - Return codes: HWG_OK or one of the HWG_E* codes; hwg_last_error()
 *    gives a message for the calling thread.
 */
#ifndef HEATWAVE_B200_H
#define HEATWAVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    HWG_OK = 0,
    HWG_EINVAL = 1,     /* ValueError   (solver.py:185, system.py:190, wavelet.py:140, multigrid.py:49) */
    HWG_ENOTSPD = 2,    /* RuntimeError p^T S p <= 0 (solver.py:217-219) */
    HWG_EMAXIT = 3,     /* IterationLimitError (solver.py:132-137, 258-260) */
    HWG_ECUDA = 4,      /* CUDA runtime failure */
    HWG_ENOMEM = 5,     /* device allocation failed (cli.py:236-241 maps MemoryError) */
    HWG_EKEY = 6        /* KeyError: no preconditioner block for a level (system.py:253-255) */
};

/* Number of stencil slots per (operator, level) in the coefficient table. */
#define HWG_COEF_STRIDE 8

/*
 * Problem description.  Mirrors what assemble_system (solver.py:353-386)
 * builds: temporal trial/test matrices (temporal.py:82-144), per-level P1
 * stencils (spatial.py:202-229), the K_x solver (alpha=1, mu=0) and the
 * J+1 blocks C_j (alpha, mu=2^j) of K_X (solver.py:372-377).
 *
 * coef: table [(J + 2) operators][K + 1 levels][HWG_COEF_STRIDE] doubles
 *   (host memory, copied at create).  Operator 0 is K_x, operator 1 + j is
 *   C_j.  Level l in 1..K (slot 0 unused).  Slots:
 *     2D: 0 centre, 1 x-neighbours (i+-1), 2 y-neighbours (j+-1),
 *         3 diagonal (i+1,j+1)/(i-1,j-1), 4 1/centre, 5 coarse inverse (l=1)
 *     1D: 0 centre, 2 neighbours (i+-1), 4 1/centre, 5 coarse inverse
 *   Values are those of alpha*A_l + mu*M_l (multigrid.py:87-91).
 * stencil_M / stencil_A: the finest-level M_x / A_x stencils (4 doubles:
 *   centre, x, y, diagonal; 1D: centre, -, neighbour, -).
 * temporal: 11 doubles -- M_t (off, main, end), A_t (off, main, end),
 *   L (off = 0.5, end = 0.5), T_test (1/sqrt h), N_test (sqrt h / 2,
 *   sqrt(3h)/6) -- see temporal.py:82-144.
 * wavelet_scale: J doubles, s_j = 2^(j/2) for j = 1..J (wavelet.py:63).
 *
 * domain (ABI v4): 0 = [0,1]^dim (the reference's meshes, spatial.py:98-137);
 *   1 = the L-shaped domain of BASELINE config 5, [-1,1]^2 \ [0,1]^2 mapped
 *   to [0,1]^2 \ [1/2,1]^2 (pass D = I/4 in coef / stencils; the mapped S,
 *   f-hat are 1/4 and K_X 4x the unmapped ones, so PCG iterates agree).
 *   Level l (h = 2^-l) has the vertices of the square's level l minus the
 *   closed quadrant [1/2,1]^2; its dofs are the remaining interior vertices
 *   in lexicographic order (x slow, y fast): N_x = (2^K-1)^2 - 4^(K-1).
 *   The hierarchy starts at level 2 (5 dofs), inverted densely like the
 *   reference's coarsest level (multigrid.py:118): coarse_inv holds
 *   [(J + 2) operators][5][5] doubles (host), the inverse of the level-2
 *   matrix alpha*A_2 + mu*M_2 of each operator in dof order.  Full contexts
 *   take space-time arrays in the dof layout (rows of N_x); internally, and
 *   in the time-slab entry points of kernel contexts (rows_max > 0), rows
 *   use the embedded grid layout of (2^K-1)^2 points with the removed
 *   quadrant held at zero -- hwg_grid_scatter / hwg_grid_gather convert.
 */
typedef struct {
    int32_t dim;            /* 1 or 2 */
    int32_t J;              /* N_t = 2^J + 1 */
    int32_t K;              /* N_x = (2^K - 1)^dim */
    int32_t vcycles;        /* SolveConfig.vcycles (2) */
    int32_t smooth;         /* SolveConfig.smooth (3) */
    int32_t device;         /* CUDA device ordinal */
    double alpha;           /* SolveConfig.alpha (0.3) */
    const double *coef;     /* host, see above */
    const double *stencil_M;
    const double *stencil_A;
    const double *temporal;
    const double *wavelet_scale;
    /* 0: full context (operator workspaces for all N_t rows).  > 0: kernel
     * context for the distributed (time-slab) path -- multigrid and dot
     * workspaces for batches of up to rows_max rows, no N-sized operator
     * buffers (hwg_schur_apply, hwg_kx_apply, hwg_rhs, hwg_wavelet, hwg_pcg
     * and hwg_solve_host then return HWG_EINVAL). */
    int64_t rows_max;
    int32_t domain;         /* 0 square / cube, 1 L-shaped (dim 2, K in [2, 11]) */
    int32_t reserved;
    const double *coarse_inv;   /* domain 1: [(J + 2)][25] (host), else NULL */
} hwg_desc;

typedef struct hwg_ctx hwg_ctx;

/* PCG statistics (PCGResult, solver.py:140-148).  Arrays are host buffers
 * of capacity max_iterations + 1 supplied by the caller (may be NULL). */
typedef struct {
    int32_t iterations;
    int32_t capacity;
    double *residual_norms;   /* sqrt(rho_k), k = 0..iterations */
    double *alphas;           /* cg_alphas, iterations entries */
    double *betas;            /* cg_betas */
    double ms_schur, ms_precond, ms_vector, ms_total;  /* wall_times; the per-phase times
                                * are only measured when iterations run as plain launches
                                * (profiling on or HWG_GRAPH=0), else 0: by default each
                                * iteration replays one captured CUDA graph */
    double epsilon_used;      /* the absolute tolerance actually applied */
} hwg_pcg_stats;

/* Library / context lifetime. */
const char *hwg_last_error(void);
int hwg_version(void);
int hwg_create(const hwg_desc *desc, hwg_ctx **ctx);
int hwg_destroy(hwg_ctx *ctx);
/* Device bytes the context holds (workspaces only). */
int64_t hwg_workspace_bytes(const hwg_ctx *ctx);

/*
 * WaveletTransform.apply_array / transpose_apply_array (wavelet.py:114-149):
 * Y = (W_t (x) Id) X, or its transpose.  X, Y: (N_t, N_x); may not alias.
 */
int hwg_wavelet(hwg_ctx *ctx, const double *X, double *Y, int transpose, void *stream);

/*
 * Spatial factor on every row (system.py:48-51 `_spatial`, csr_rows_matvec
 * _kernels.py:25-34): Y[r] = M_x X[r] (which = 0) or A_x X[r] (which = 1).
 */
int hwg_spatial(hwg_ctx *ctx, int which, const double *X, double *Y, int64_t rows, void *stream);

/* SchurOperator.apply_array, five-term form (system.py:116-147, 182-187). */
int hwg_schur_apply(hwg_ctx *ctx, const double *X, double *Y, void *stream);

/* SchurOperator form (system.py:84-87, SolveConfig.form): 0 = "five_term"
 * (Lemma 2, the production path, default), 1 = "test_space" (Lemma 1:
 * B^T K_Y B + Gamma0 through the test-space matrices, system.py:149-180).
 * hwg_schur_apply and hwg_pcg apply the selected form. */
int hwg_set_schur_form(hwg_ctx *ctx, int form);

/* PreconditionerKX.apply_array (system.py:252-276). */
int hwg_kx_apply(hwg_ctx *ctx, const double *X, double *Y, void *stream);

/*
 * Batched V-cycles, MultigridSolver.apply_rows / apply_rows_indexed
 * (multigrid.py:58-68, _kernels.py:110-249): X[r] = MG_op(r)(B[r]) for
 * r in [0, rows).  op_host == NULL: every row uses operator `op`
 * (0 = K_x, 1 + j = C_j); otherwise op_host[r] (host int32 array) picks the
 * operator per row.  B and X must not alias.
 */
int hwg_mg_rows(hwg_ctx *ctx, int32_t op, const int32_t *op_host, const double *B,
                double *X, int64_t rows, void *stream);

/*
 * Right-hand side from nodal forcing (system.py:295-324 assemble_rhs with
 * the P1 x P1 interpolant load (N (x) M_x) F):
 *   fhat = W^T( B^T K_Y (N (x) M_x) F + e_0 (x) u0proj ).
 * F: (N_t, N_x) device or NULL (no forcing); u0proj: N_x device moments
 * <u0, phi_i> or NULL.  load: alternatively an already assembled test-space
 * load (2*2^J, N_x) on the device (pass F = NULL), e.g. from assemble_load
 * (spatial.py:269-300) for a callable forcing.
 */
int hwg_rhs(hwg_ctx *ctx, const double *F, const double *load, const double *u0proj,
            double *fhat, void *stream);

/* Deterministic inner product (solver.py:111-129): per-row partials, then
 * the fixed pairwise tree over rows.  Synchronises `stream`. */
int hwg_dot(hwg_ctx *ctx, const double *X, const double *Y, int64_t rows, double *result_host,
            void *stream);

/*
 * pcg (solver.py:181-263) on S-hat w = fhat, preconditioned by K_X.
 * Stops when r^T K_X r <= eps^2 with eps = epsilon (absolute) or, if
 * rtol > 0, eps = rtol * sqrt(f^T K_X f).  w is overwritten (zero start).
 * Returns HWG_EMAXIT after max_iterations (stats hold the history),
 * HWG_ENOTSPD if p^T S p <= 0, HWG_EINVAL if the tolerance is not positive.
 */
int hwg_pcg(hwg_ctx *ctx, const double *fhat, double *w, double epsilon, double rtol,
            int32_t max_iterations, int32_t recompute_every, hwg_pcg_stats *stats,
            void *stream);

/*
 * End-to-end call for host buffers (the e2e leg of bench.py): copies fhat
 * from host memory, solves with hwg_pcg, applies u = W w and copies u back.
 * For large problems (N >= 2^26) fhat is copied in up to 8 row chunks on a
 * context-owned stream and the row-local initial K_X starts on each chunk as
 * it lands (pinned host memory makes the copies asynchronous); results are
 * bit-identical to hwg_pcg followed by W.
 */
int hwg_solve_host(hwg_ctx *ctx, const double *fhat_host, double *u_host, double epsilon,
                   double rtol, int32_t max_iterations, int32_t recompute_every,
                   hwg_pcg_stats *stats, void *stream);

/* Kernel launches issued by this context since creation (bench evidence). */
int64_t hwg_launch_count(const hwg_ctx *ctx);

/*
 * Per-kernel-class timing for bench.py's roofline: CUDA events are recorded
 * on the launching stream around every multigrid launch while enabled
 * (enable != 0 also resets the totals).  Classes: 0 mg2d_stream DOWN on the
 * finest level, 1 mg2d_stream UP on the finest level, 2 DOWN on coarser
 * levels, 3 UP on coarser levels, 4 mg2d_coarse, 5 mg1d.  `bytes` is the
 * algorithmic HBM traffic of those launches (each input read once, each
 * output written once).  hwg_profile_read synchronises the context's events.
 */
int hwg_profile_enable(hwg_ctx *ctx, int enable);
int hwg_profile_read(hwg_ctx *ctx, int kclass, double *ms, double *bytes, int64_t *launches);

/* ------------------------------------------------------------------------
 * Time-slab building blocks (multi-GPU path).  The reference
 * distributes temporal rows over workers (ParallelPlan, solver.py:47-108)
 * with halo reads; these entry points compute one rank's share of an
 * operator given explicitly supplied halo rows.  Rows are named by their
 * GLOBAL temporal index; `x0`-style arguments give the global index of the
 * first row an array holds.
 * ------------------------------------------------------------------------ */

/* Synthesis stage j (wavelet.py:114-137 with M_j of :56-76): Y[f - f0] for
 * fine nodes f in [f0, f0 + nf) from coarse nodal rows C (C[i - c0] = node
 * i of level j-1) and level-j wavelet rows Dw (Dw[k - d0] = wavelet k).
 * Dhalo (nullable): wavelet d0 - 1 (a neighbour slab's halo row), so the
 * caller's own rows are read in place. */
int hwg_syn_stage(hwg_ctx *ctx, int j, const double *C, int64_t c0, const double *Dw, int64_t d0,
                  const double *Dhalo, double *Y, int64_t f0, int64_t nf, void *stream);

/* Transposed stage j: C[i - c0] = (P_j^T x)[i] for i in [c0, c0 + nc) and
 * Dw[k - d0] = (Q_j^T x)[k] for k in [d0, d0 + nd), from fine nodal rows X
 * (X[f - x0] = node f of level j). */
int hwg_ana_stage(hwg_ctx *ctx, int j, const double *X, int64_t x0, double *C, int64_t c0,
                  int64_t nc, double *Dw, int64_t d0, int64_t nd, void *stream);

/* B-side of the five-term S on nodal rows [r0, r0 + nr): t1 = A_t MxU + L^T
 * AxU, t1' = M_t AxU + L MxU (system.py:119-139).  U holds nodal rows
 * [u0, u0 + nu) including the halo rows the bands need.  If r0 == 0, E0
 * (N_x, may be NULL) receives M_x U[0] for the trace term. */
int hwg_bside_rows(hwg_ctx *ctx, const double *U, int64_t u0, int64_t nu, double *T1, double *T2,
                   int64_t r0, int64_t nr, double *E0, void *stream);

/* B^T-side: out = M_x G1 + A_x G2 on `rows` rows; E0 (or NULL) is added to
 * the first row (only the rank that owns global row 0 passes it). */
int hwg_bt_rows(hwg_ctx *ctx, const double *G1, const double *G2, const double *E0, double *out,
                int64_t rows, void *stream);

/* Temporal factor on a row range: Y[c - r0] = sum_k B[c,k] X[k - x0] for
 * c in [r0, r0 + nr) (temporal_apply, _kernels.py:37-52).  band: 0 M_t,
 * 1 A_t, 2 L, 3 L^T, 4 T, 5 T^T, 6 N, 7 N^T (temporal.py:82-144; T and N
 * have 2*2^J test rows).  X must hold every row the band touches. */
int hwg_temporal_rows(hwg_ctx *ctx, int band, const double *X, int64_t x0, double *Y, int64_t r0,
                      int64_t nr, void *stream);

/* L-shaped domain: dof-layout rows (N_x values each) -> embedded grid rows
 * ((2^K-1)^2 values, removed quadrant zero), and back.  For domain 0 both
 * are plain copies. */
int hwg_grid_scatter(hwg_ctx *ctx, const double *X, double *Y, int64_t rows, void *stream);
int hwg_grid_gather(hwg_ctx *ctx, const double *X, double *Y, int64_t rows, void *stream);

/* Batched V-cycles with a DEVICE array of per-row operator ids. */
int hwg_mg_rows_dev(hwg_ctx *ctx, const int32_t *ops, const double *B, double *X, int64_t rows,
                    void *stream);

/* hwg_mg_rows_dev plus the per-row partials part[r] = <Y row r, X row r> of
 * the result, fused into the last multigrid pass (the PCG's r.z after
 * z = K_X r; solver.py:233-236).  Deterministic; the same kernels on every
 * rank, so time slabs reproduce the single-GPU partials bit for bit. */
int hwg_mg_rows_dev_dot(hwg_ctx *ctx, const int32_t *ops, const double *B, double *X,
                        int64_t rows, const double *Y, double *part, void *stream);

/* Per-row partial inner products part[r] = sum_i X[r,i] Y[r,i] (device). */
int hwg_row_partials(hwg_ctx *ctx, const double *X, const double *Y, int64_t rows, double *part,
                     void *stream);

/* Fixed pairwise tree over n partials (solver.py:111-119) -> *result (device). */
int hwg_tree_sum(hwg_ctx *ctx, const double *part, int64_t n, double *result, void *stream);

/* Y += a X and Y = X + a Y over n values (axpy_rows / xpay_rows,
 * _kernels.py:64-76). */
int hwg_axpy(hwg_ctx *ctx, double a, const double *X, double *Y, int64_t n, void *stream);
int hwg_xpay(hwg_ctx *ctx, double a, const double *X, double *Y, int64_t n, void *stream);

/* Device-resident PCG scalars for the time-slab solver (solver.py:212-256),
 * the same kernels hwg_pcg runs.  scal (device, >= 5 doubles): [0] rho,
 * [1] p.q, [2] rho_new, [3] alpha, [4] beta.  step 0: alpha = rho / pq;
 * step 1: beta = rho_new / rho, rho = rho_new. */
int hwg_pcg_scalar(hwg_ctx *ctx, int step, double *scal, void *stream);

/* w += alpha p (if do_w); r -= alpha q (if do_r); alpha = scal[3]. */
int hwg_pcg_update_wr(hwg_ctx *ctx, double *w, double *r, const double *p, const double *q,
                      const double *scal, int64_t n, int do_w, int do_r, void *stream);

/* w += alpha p (if do_w, the deferred half of the step above) and
 * p = z + beta p in one pass over p; alpha = scal[3], beta = scal[4]. */
int hwg_pcg_update_wp(hwg_ctx *ctx, double *w, double *p, const double *z, const double *scal,
                      int64_t n, int do_w, void *stream);

/* r = f - t (the periodic residual recomputation, solver.py:227-229). */
int hwg_sub(hwg_ctx *ctx, const double *f, const double *t, double *r, int64_t n, void *stream);

/* *flag (device int) |= any(X[0:n] != 0)  (the zero right-hand side test,
 * solver.py:196-198; the caller zeroes *flag). */
int hwg_any_nonzero(hwg_ctx *ctx, const double *X, int64_t n, int32_t *flag, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HEATWAVE_B200_H */
