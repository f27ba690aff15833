// hw_internal.cuh -- argument structs and launchers shared between the
// kernel translation units and the C ABI (hw_capi.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hw {

// ---- hw_mg2d.cu ----------------------------------------------------------
struct MgStreamArgs {
    const double *B;   int64_t ldB;     // level right-hand sides
    double *X;         int64_t ldX;     // level iterates (in/out)
    double *Bc;        int64_t ldBc;    // DOWN: coarse right-hand sides (out)
    const double *Xc;  int64_t ldXc;    // UP: coarse iterates (in)
    const double *coef;                 // [op][K+1][8]
    int levels_p1;                      // K + 1
    int level;                          // l
    int n;                              // 2^l - 1
    const int32_t *row_op;              // per temporal row, or null
    int op;                             // default operator
    int zero_start;                     // DOWN: iterate starts at zero
    int reg_ok;                         // |beta| small enough for mg2d_reg
    int wide;                           // mg2d_reg: levels (bit l) run with the wide thread shape
    const double *dot_y;                // UP (mg2d_reg): dot_part[row] = <dot_y row, final X row>
    double *dot_part;
    int lshape;                         // mapped L-shaped domain (mg2d_reg only)
    int diag;                           // some row's operator has c_d != 0 on this level
};

struct MgCoarseArgs {
    const double *B;  int64_t ldB;
    double *X;        int64_t ldX;
    const double *coef;
    int levels_p1;
    int top;                 // top level handled here (<= kCoarseTop2d)
    int ncyc;                // V-cycles
    int zero_start;
    const int32_t *row_op;
    int op;
    int64_t rows;
    int lshape;              // mapped L-shaped domain: masked quadrant, level-2 dense solve
    const double *cinv;      // lshape: [op][25] inverse of the 5-dof level-2 operator
    int fast;                // below streamed levels: multiply by 1/c0, tree sums (not
                             // bit-exact); 0 = the reference's CSR-order arithmetic
};

constexpr int kCoarseTop2d = 5;
cudaError_t mg2d_stream_launch(const MgStreamArgs &a, bool down, int64_t rows, cudaStream_t st);
// register-resident variant (hw_mg2d_reg.cu), levels 6..11; cudaErrorNotSupported otherwise
cudaError_t mg2d_reg_launch(const MgStreamArgs &a, bool down, int64_t rows, cudaStream_t st);
// largest |beta| = |cy / c0| mg2d_reg accepts (8-chunk window: |beta|^32 <= 2^-60)
constexpr double kRegBetaMax = 0.2726;
// mg2d_reg: levels 7-9 run with twice the threads per row in contexts whose
// N_t-row batches have at most kWideWarps default-shape warps (~2 per SM)
constexpr int64_t kWideWarps = 320;
cudaError_t mg2d_coarse_launch(const MgCoarseArgs &a, cudaStream_t st);

// ---- hw_mg1d.cu ----------------------------------------------------------
struct Mg1dArgs {
    const double *B;  int64_t ldB;
    double *X;        int64_t ldX;
    const double *coef;
    int levels_p1;
    int K;
    int ncyc;
    const int32_t *row_op;
    int op;
    int64_t rows;
    // optional [op][15][15]: the V-cycle from level 4 (zero start) as a dense
    // operator, M[op][i][j] = (MG_4 e_i)_j (hwg_create builds it by running
    // this kernel with K = 4 on unit rows); mg1d_reg applies it instead of
    // the level-4..1 sub-cycle
    const double *cmat = nullptr;
    // mg1d_rr: [op][kRrCutN][64] the V-cycle from level kRrCut (zero start),
    // G[op][s][j] = (MG e_s)_j, columns padded to 64 with zeros
    const double *cmat_rr = nullptr;
    int rr_minb = 1;                              // 1: mg1d_rrp; 3 / 2: mg1d_rr CTAs (4 warps) per SM
};
constexpr int kMg1dCut = 4;                    // levels <= kMg1dCut: dense operator
constexpr int kMg1dCutN = (1 << kMg1dCut) - 1;  // 15
cudaError_t mg1d_launch(const Mg1dArgs &a, cudaStream_t st);
// register-resident hierarchy (hw_mg1d_rr.cu), 7 <= K <= 10, |beta| <= 1/2 on
// every level; cudaErrorNotSupported otherwise
constexpr int kRrCut = 6;                      // levels <= kRrCut: dense operator
constexpr int kRrCutN = (1 << kRrCut) - 1;     // 63
constexpr int kRrCutLd = 64;                   // padded row of the dense operator
cudaError_t mg1d_rr_launch(const Mg1dArgs &a, cudaStream_t st);


// ---- hw_wavelet.cu -------------------------------------------------------
// mask_n > 0: columns are points of an mask_n x mask_n grid whose quadrant
// a, b >= mask_lm is zero (the L-shaped domain): written, never read
cudaError_t wavelet_apply(const double *X, double *Y, double *S1, double *S2, int J,
                          const double *scale, int64_t nt, int64_t nx, bool transpose,
                          cudaStream_t st, int64_t *launches, int mask_n = 0, int mask_lm = 0);
// Dh (nullable): wavelet row d0 - 1 held apart from Dm (a slab's halo row)
cudaError_t launch_syn_stage(int j, double s, const double *C, int64_t c0, const double *Dm,
                             int64_t d0, const double *Dh, double *Y, int64_t f0, int64_t nf,
                             int64_t nx, cudaStream_t st);
cudaError_t launch_ana_stage(int j, double s, const double *X, int64_t x0, double *C, int64_t c0,
                             int64_t nc, double *Dm, int64_t d0, int64_t nd, int64_t nx,
                             cudaStream_t st);

// ---- hw_kron.cu ----------------------------------------------------------
struct Stencil {           // finest-level spatial stencil, see hwg_desc
    double c0, cx, cy, cd; // 1D: c0, -, cy (neighbour), -
};
struct Grid {
    int dim;
    int m;                 // points per direction
    int64_t nx;            // m^dim
    int lm;                // 2D: points with i >= lm and j >= lm are masked (held at
                           // zero; the L-shaped domain, lm = (m-1)/2), else > m
};
struct TCsr {              // temporal factor, CSR on the device
    const int32_t *ip, *ix;
    const double *v;
};
struct Tri4 {              // dense (lo, mid, hi) rows of A_t, L^T, M_t, L (device)
    const double *At, *LT, *Mt, *L;
};
struct BandOut {           // out = b1 x1 (+ b2 x2)
    TCsr b1, b2;
    const double *x1, *x2;
    double *out;
};
cudaError_t launch_stencil_rows(const double *X, double *YM, double *YA, Grid g, Stencil M,
                                Stencil A, int64_t rows, cudaStream_t st);
cudaError_t launch_bt_side(const double *G1, const double *G2, const double *E0, double *out,
                           Grid g, Stencil M, Stencil A, int64_t rows, cudaStream_t st);
cudaError_t launch_temporal_bands(BandOut o1, BandOut o2, int64_t rows, int64_t nx,
                                  cudaStream_t st);
// U holds nu temporal rows starting at global row u0 (the readable extent)
cudaError_t launch_bside_fused(const double *U, int64_t u0, int64_t nu, double *T1, double *T2,
                               double *E0, Grid g, Stencil M, Stencil A, Tri4 tri, int64_t r0,
                               int64_t nr, int64_t nt, cudaStream_t st);
cudaError_t launch_add(const double *X1, const double *X2, double *Y, int64_t total,
                       cudaStream_t st);
// L-shaped domain: rows of the lexicographic dof layout (nxu per row) <-> the
// embedded grid layout (g.nx per row, masked points zero)
cudaError_t launch_grid_scatter(const double *src, double *dst, int64_t rows, Grid g, int64_t nxu,
                                cudaStream_t st);
cudaError_t launch_grid_gather(const double *src, double *dst, int64_t rows, Grid g, int64_t nxu,
                               cudaStream_t st);
cudaError_t launch_temporal_rows(TCsr B, const double *X, int64_t x0, double *Y, int64_t r0,
                                 int64_t nr, int64_t nx, cudaStream_t st);

// ---- hw_vec.cu -----------------------------------------------------------
cudaError_t launch_dot(const double *X, const double *Y, int64_t rows, int64_t nx, double *part,
                       double *tmp, double *out, cudaStream_t st, int64_t *launches);
cudaError_t launch_pcg_alpha(double *s, cudaStream_t st);
cudaError_t launch_pcg_beta(double *s, cudaStream_t st);
cudaError_t launch_update_wr(double *w, double *r, const double *p, const double *q,
                             const double *s, int64_t n, int do_w, int do_r, cudaStream_t st);
cudaError_t launch_update_wp(double *w, double *p, const double *z, const double *s, int64_t n,
                             int do_w, cudaStream_t st);
cudaError_t launch_sub(const double *f, const double *t, double *r, int64_t n, cudaStream_t st);
cudaError_t launch_any_nonzero(const double *X, int64_t n, int *flag, cudaStream_t st);
cudaError_t launch_row_partials(const double *X, const double *Y, int64_t rows, int64_t nx,
                                double *part, cudaStream_t st);
cudaError_t launch_tree(const double *part, int64_t n, double *tmp, double *out, cudaStream_t st);
cudaError_t launch_axpy(double a, const double *X, double *Y, int64_t n, cudaStream_t st);
cudaError_t launch_xpay(double a, const double *X, double *Y, int64_t n, cudaStream_t st);

}  // namespace hw
