// hw_mg2d.cu -- batched geometric-multigrid V-cycles for alpha*A + mu*M, 2D.
//
// Restates _mg_core (/root/reference/pkg/src/heatwave/_kernels.py:110-199)
// for every temporal row of a space-time array at once.  The discrete
// operator is fixed by the reference's smoother ORDER (SURVEY.md §7 "hard
// parts"): lexicographic forward Gauss-Seidel before restriction, backward
// after prolongation, 3 sweeps each, 2 V-cycles from a zero start.  Both
// kernels below reproduce that order exactly (mathematically); only the
// rounding of individual updates can differ.
//
// Grid: level l has m = 2^l - 1 interior points per direction, numbered
// i (x, slow) then j (y, fast) -- spatial.py:105-111,131-135.  The operator
// is a 7-point stencil: centre c0, x-neighbours (i+-1,j) cx, y-neighbours
// (i,j+-1) cy, diagonal (i+1,j+1)/(i-1,j-1) cd (spatial.py:202-229).
//
// Two kernels:
//  * mg2d_stream<DOWN/UP>  -- one CTA per temporal row streams one fine
//    level through shared-memory row rings.  A forward GS sweep over grid
//    row i is, given rows i-1 (new) and i+1 (old), a first-order linear
//    recurrence along j; the CTA evaluates it as a block-wide affine scan.
//    The three sweeps are pipelined two grid rows apart, so the level is
//    read once and written once per pass (DOWN also fuses residual and
//    restriction; UP fuses prolongation and runs backward GS as forward GS
//    on the point-reversed grid, which maps the stencil onto itself).
//  * mg2d_coarse -- one warp per temporal row runs the remaining V-cycle on
//    levels <= 5 held in shared memory; GS is done by anti-diagonal
//    wavefronts in the reference's exact CSR arithmetic order.
#include "hw_common.cuh"
#include "hw_internal.cuh"

#include <type_traits>

namespace hw {

// ring sizes, see the lifetime analysis in DESIGN.md §MG
// ---------------------------------------------------------------------------
// streamed fine-level passes
// ---------------------------------------------------------------------------
// Ring slots: row i of a ring lives in slot (i mod R), R a power of two.  The
// step loop is unrolled by 4 so every slot offset is a compile-time constant
// (the 8-slot b ring needs one uniform select per block of 4 steps).
// Lifetimes (steps; row i is swept by sweep s at step i + 2(s-1), b is
// prefetched one step ahead):  V0 i-2..i (DOWN) / i-3..i (UP),  V1 i..i+2,
// V2 i+2..i+4,  V3 i+4..i+7,  b i-1..i+6,  residual i+6..i+7.
struct RingsDown { static constexpr int V0 = 4, V1 = 4, V2 = 4, V3 = 4, B = 8, R = 2, C = 0; };
struct RingsUp { static constexpr int V0 = 4, V1 = 4, V2 = 4, V3 = 4, B = 8, R = 0, C = 4; };
template <bool DOWN> using RingsOf = typename std::conditional<DOWN, RingsDown, RingsUp>::type;
constexpr int kMaxWarpCarry = 4;       // warp totals summed for a chunk carry (exact path)
constexpr int kChunkCarry = 8;         // chunk ends summed for a carry (truncated path)
// narrow rows (<= 2 warps) always use the exact scan: measured faster, and the
// chunk-end scratch would cost the n = 255 level one resident CTA per SM
template <int NT> constexpr bool trunc_carry_ok() { return NT >= 128; }
template <int NT> constexpr int chunk_end_words() { return trunc_carry_ok<NT>() ? 3 * (NT + kChunkCarry) : 0; }

template <int P, int NT, bool DOWN>
__host__ __device__ constexpr size_t stream_smem_words(int n)
{
    using G = RingsOf<DOWN>;
    const size_t W = (size_t)n + 2;
    const size_t Wc = (size_t)(n - 1) / 2 + 2;
    return W * (G::V0 + G::V1 + G::V2 + G::V3 + G::B + G::R + 1) + Wc * G::C +
           3 * (size_t)(NT / 32 + kMaxWarpCarry) + (size_t)chunk_end_words<NT>() + (P + 1) + 33 +
           (kMaxWarpCarry + 1) + (kChunkCarry + 1) + 8;
}

// Row recurrence.  Thread t owns P consecutive points of a grid row; y_k is
// the sweep recurrence x_j = p_j + beta x_{j-1} run over the chunk from a
// zero carry-in and S_t = y_{P-1}.  Within a warp the chunk carries are an
// exact inclusive scan of S with multiplier gamma = beta^P.  Across warps
// the carry into warp w is sum_{k>=1} Gamma^(k-1) T_{w-k} (T = warp totals,
// Gamma = gamma^32 = beta^(32P)); |beta| <= 1/4 for the 2D operators
// alpha A + mu M, so Gamma <= 2^-(64P) and the nearest warp already leaves a
// tail below 2^-70 relative -- 2^17 times smaller than one fp64 rounding:
// the lexicographic Gauss-Seidel result up to rounding.  (Kw, the number of
// warp totals summed, is computed per CTA and is at most kMaxWarpCarry.)
template <int P, int NT, bool DOWN>
__global__ void __launch_bounds__(NT, 1) mg2d_stream(MgStreamArgs a)
{
    using G = RingsOf<DOWN>;
    constexpr int NW = NT / 32;
    constexpr int KW = kMaxWarpCarry;
    constexpr int KC = kChunkCarry;
    constexpr int MJ = (NT * P / 2 + NT - 1) / NT;      // coarse columns per thread (DOWN)
    extern __shared__ __align__(16) double sm[];

    const int n = a.n;
    const int W = n + 2;                                // data at 1..n, zero pads at 0, n+1
    const int m = (n - 1) / 2;
    const int Wc = m + 2;
    const int64_t row = blockIdx.x;
    const int op = a.row_op ? a.row_op[row] : a.op;
    const double *cf = a.coef + ((int64_t)op * a.levels_p1 + a.level) * kCoefStride;
    const double c0 = cf[kC0], cx = cf[kCx], cy = cf[kCy], cd = cf[kCd], inv = cf[kInv];
    const double beta = -cy * inv;

    double *const v0 = sm;
    double *const v1 = v0 + G::V0 * W;
    double *const v2 = v1 + G::V1 * W;
    double *const v3 = v2 + G::V2 * W;
    double *const bs = v3 + G::V3 * W;
    double *const rs = bs + G::B * W;
    double *const zr = rs + G::R * W;                   // a row of zeros
    double *const cs = zr + W;                          // coarse ring (UP)
    double *const sc = cs + G::C * Wc;                  // warp totals [3][KW + NW]
    double *const se = sc + 3 * (NW + KW);              // chunk ends [3][KC + NT]
    double *const gp = se + chunk_end_words<NT>();             // beta^0..P, gamma^0..32, Gamma^0..KW, w^0..KC

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int j0 = tid * P;                             // first local column of this thread
    const int nvalid = n - j0 < 0 ? 0 : (n - j0 > P ? P : n - j0);
    const int jb = nvalid > 0 ? j0 : 0;                 // idle threads compute on row data
    const double *Bg = a.B + row * a.ldB;
    double *Xg = a.X + row * a.ldX;

    const double ab = fabs(beta);
    int Kw = 0;
    if (ab > 0.0) {
        Kw = ab >= 0.9 ? KW : (int)ceil(70.0 / (32.0 * P * -log2(ab)));
        Kw = Kw > KW ? KW : (Kw < 1 ? 1 : Kw);
    }
    // truncated chunk carries: the nearest Kc chunk ends, gamma^Kc <= 2^-70
    int Kc = 0;
    if (ab > 0.0) Kc = ab >= 0.9 ? KC + 1 : (int)ceil(70.0 / (P * -log2(ab)));
    constexpr bool kTruncOK = trunc_carry_ok<NT>();
    const bool trunc = kTruncOK && Kc <= KC;            // uniform per CTA
    if (tid == 0) {
        double bp = 1.0;
        for (int k = 0; k <= P; ++k) { gp[k] = bp; bp *= beta; }
        const double g = gp[P];
        double q = 1.0;
        for (int k = 0; k <= 32; ++k) { gp[P + 1 + k] = q; q *= g; }
        const double Gm = gp[P + 1 + 32];
        q = 1.0;
        for (int k = 0; k <= KW; ++k) { gp[P + 34 + k] = k < Kw ? q : 0.0; q *= Gm; }
        q = 1.0;
        for (int k = 0; k < KC; ++k) { gp[P + 35 + KW + k] = k < Kc ? q : 0.0; q *= g; }
    }
    {
        const int total = (int)(gp - sm);
        for (int k = tid; k < total; k += NT) sm[k] = 0.0;
    }
    __syncthreads();
    const double gl = gp[P + 1 + lane];                 // gamma^lane
    double Gw[KW];                                      // Gamma^(k) weights (0 beyond Kw)
#pragma unroll
    for (int k = 0; k < KW; ++k) Gw[k] = gp[P + 34 + k];
    double bpow[P];                                     // beta^(k+1)
#pragma unroll
    for (int k = 0; k < P; ++k) bpow[k] = gp[k + 1];
    double gscan[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) gscan[k] = gp[P + 1 + (1 << k)];
    double wc[KC];                                      // gamma^(k) weights, 0 beyond Kc
#pragma unroll
    for (int k = 0; k < KC; ++k) wc[k] = gp[P + 35 + KW + k];

    constexpr int gs = DOWN ? 1 : -1;                   // UP runs point-reversed
    auto grow = [&](const double *base, int i) -> const double * {
        return base + (DOWN ? (int64_t)i * n : (int64_t)(n - 1 - i) * n + (n - 1));
    };
    const bool zs = DOWN && a.zero_start;

    // loads of virtual step s: b row s+1; raw x row s+2 (DOWN) / s+3 (UP)
    // plus, UP, the coarse row it first needs.  Rows >= n get zeros.
    auto issue = [&](int s) {
        const int ib = s + 1;
        if (ib >= 0 && ib < n) {
            double *dst = bs + (ib & (G::B - 1)) * W + 1;
            const double *src = grow(Bg, ib);
            for (int e = tid; e < n; e += NT) cp_async8(dst + e, src + gs * e);
        }
        const int ix = DOWN ? s + 2 : s + 3;
        if (ix >= 0 && !zs) {
            double *dst = v0 + (ix & (G::V0 - 1)) * W + 1;
            if (ix < n) {
                const double *src = grow(Xg, ix);
                for (int e = tid; e < n; e += NT) cp_async8(dst + e, src + gs * e);
            } else {
                for (int e = tid; e < n; e += NT) dst[e] = 0.0;
            }
        }
        if (!DOWN && ix >= 0 && ix < n && !(ix & 1) && ix / 2 < m) {
            const int c = ix / 2;                       // coarse row first used by fine row 2c
            const double *Xc = a.Xc + row * a.ldXc;
            double *cdst = cs + (c & (G::C - 1)) * Wc + 1;
            for (int e = tid; e < m; e += NT)
                cp_async8(cdst + e, Xc + (int64_t)(m - 1 - c) * m + (m - 1 - e));
        }
        cp_async_commit();
    };

    // UP: V0[i] += P x_coarse (local = point-reversed coordinates)
    auto prolongate = [&](int i) {
        if (i < 0 || i >= n) return;
        double *xr = v0 + (i & (G::V0 - 1)) * W + 1;
        auto crow = [&](int c) -> const double * {
            return (c < 0 || c >= m) ? zr : cs + (c & (G::C > 0 ? G::C - 1 : 0)) * Wc;
        };
        const double *ca = (i & 1) ? crow((i - 1) / 2) : crow(i / 2 - 1);
        const double *cb = (i & 1) ? ca : crow(i / 2);
        for (int j = tid; j < n; j += NT) {
            double v;
            if (j & 1) {
                const int J = (j - 1) / 2 + 1;
                v = (i & 1) ? ca[J] : 0.5 * ca[J] + 0.5 * cb[J];
            } else {
                const int J = j / 2;                    // padded index of coarse j/2 - 1
                v = (i & 1) ? 0.5 * ca[J] + 0.5 * ca[J + 1] : 0.5 * ca[J] + 0.5 * cb[J + 1];
            }
            xr[j] += v;
        }
    };

    for (int s = DOWN ? -2 : -3; s < 0; ++s) issue(s);
    if (!DOWN) {
        cp_async_wait<1>();
        __syncthreads();
        prolongate(0);
        prolongate(1);
    }

    // coarse right-hand-side accumulator (DOWN): coarse row I collects the
    // restricted residual rows 2I (top), 2I+1 (centre), 2I+2 (bottom)
    // (R = P^T, spatial.py:140-173)
    double acc[MJ];
#pragma unroll
    for (int k = 0; k < MJ; ++k) acc[k] = 0.0;

    const int nsteps = DOWN ? n + 7 : n + 4;
    for (int t0 = 0; t0 < nsteps; t0 += 4) {
        const int h8 = (t0 >> 2) & 1;                   // b ring half for this block
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int t = t0 + u;
            if (t >= nsteps) break;
            cp_async_wait<0>();
            __syncthreads();                            // (#0) loads + last step's rows visible
            issue(t);

            // slot of row t - k in a ring of size R (compile-time for R <= 4)
#define SLOT(base, R, k) ((base) + (((u - (k)) & ((R) - 1))) * W)
#define BSLOT(k) (bs + ((((h8 << 2) + u - (k)) & 7)) * W)

            // ---- phase A: p_j = (b - known neighbours)/c0 and chunk recurrence ----
            double p[3][P];
            double S[3];
#pragma unroll
            for (int s = 0; s < 3; ++s) {
                const double *up, *cur, *dn;
                if (s == 0) {
                    up = SLOT(v1, G::V1, 1);
                    cur = zs ? zr : SLOT(v0, G::V0, 0);
                    dn = zs ? zr : SLOT(v0, G::V0, -1);
                } else if (s == 1) {
                    up = SLOT(v2, G::V2, 3);
                    cur = SLOT(v1, G::V1, 2);
                    dn = SLOT(v1, G::V1, 1);
                } else {
                    up = SLOT(v3, G::V3, 5);
                    cur = SLOT(v2, G::V2, 4);
                    dn = SLOT(v2, G::V2, 3);
                }
                const double *bb = BSLOT(2 * s) + 1 + jb;
                up += jb;
                cur += jb;
                dn += jb;
                double uu[P + 1], dd[P + 1], cc[P];
#pragma unroll
                for (int k = 0; k <= P; ++k) { uu[k] = up[k]; dd[k] = dn[k + 1]; }
#pragma unroll
                for (int k = 0; k < P; ++k) cc[k] = cur[k + 2];
                double y = 0.0;
#pragma unroll
                for (int k = 0; k < P; ++k) {
                    const double e1 = fma(-cd, uu[k], bb[k]);
                    const double e2 = uu[k + 1] + dd[k];
                    const double e3 = fma(cd, dd[k + 1], cy * cc[k]);
                    y = fma(beta, y, (fma(-cx, e2, e1) - e3) * inv);
                    p[s][k] = y;
                }
                S[s] = y;
            }
            // restriction (DOWN): residual row t-7 (written last step) into
            // the coarse accumulators; coarse row I completes with fine row 2I+2
            if (DOWN) {
                const int r = t - 7;
                if (r >= 0 && r < n) {
                    const double *rr = rs + (r & 1) * W;
                    double *bc = a.Bc + row * a.ldBc + (int64_t)(r / 2 - 1) * m;
#pragma unroll
                    for (int k = 0; k < MJ; ++k) {
                        const int J = tid + k * NT;
                        if (J < m) {
                            const int c = 2 * J;
                            if (r & 1) {          // centre row of coarse (r-1)/2
                                acc[k] += fma(0.5, rr[c] + rr[c + 2], rr[c + 1]);
                            } else {              // bottom of coarse r/2-1, top of r/2
                                if (r >= 2) bc[J] = acc[k] + 0.5 * (rr[c + 1] + rr[c + 2]);
                                acc[k] = 0.5 * (rr[c] + rr[c + 1]);
                            }
                        }
                    }
                }
            }

            double carry[3];
            auto exact_carry = [&]() {
                // ---- exact warp scan of chunk ends T_l = S_l + gamma T_{l-1} ----
#pragma unroll
                for (int o = 1, q = 0; o < 32; o <<= 1, ++q) {
#pragma unroll
                    for (int s = 0; s < 3; ++s) {
                        const double v = __shfl_up_sync(0xffffffffu, S[s], o);
                        if (lane >= o) S[s] = fma(gscan[q], v, S[s]);
                    }
                }
                if (lane == 31) {
#pragma unroll
                    for (int s = 0; s < 3; ++s) sc[s * (NW + KW) + KW + warp] = S[s];
                }
                __syncthreads();                        // (#1) warp totals visible
#pragma unroll
                for (int s = 0; s < 3; ++s) {
                    const double *sp = sc + s * (NW + KW) + KW + warp;
                    double Cw = 0.0;
#pragma unroll
                    for (int k = 0; k < KW; ++k) Cw = fma(Gw[k], sp[-1 - k], Cw);
                    const double prev = __shfl_up_sync(0xffffffffu, S[s], 1);
                    carry[s] = (lane == 0) ? Cw : fma(gl, Cw, prev);
                }
            };
            if constexpr (kTruncOK) {
                if (trunc) {
                // ---- truncated carries: c_t = sum_{k=1..Kc} gamma^(k-1) S_{t-k} ----
#pragma unroll
                for (int s = 0; s < 3; ++s) se[s * (NT + KC) + KC + tid] = S[s];
                __syncthreads();                        // (#1) chunk ends visible
#pragma unroll
                for (int s = 0; s < 3; ++s) {
                    const double *sp = se + s * (NT + KC) + KC + tid;
                    double part[KC / 2];
#pragma unroll
                    for (int k = 0; k < KC / 2; ++k)
                        part[k] = fma(wc[2 * k + 1], sp[-2 * k - 2], wc[2 * k] * sp[-2 * k - 1]);
#pragma unroll
                    for (int w = KC / 4; w >= 1; w >>= 1)
#pragma unroll
                        for (int k = 0; k < w; ++k) part[k] += part[k + w];
                    carry[s] = part[0];
                }
                } else {
                    exact_carry();
                }
            } else {
                exact_carry();
            }

            // ---- phase B: write the swept rows ----
            double *const Xrow = const_cast<double *>(grow(Xg, t - 4));
#pragma unroll
            for (int s = 0; s < 3; ++s) {
                const int i = t - 2 * s;
                if (i < 0 || i > n) continue;           // row n is written as zeros
                double *xr = (s == 0 ? SLOT(v1, G::V1, 0)
                                     : (s == 1 ? SLOT(v2, G::V2, 2) : SLOT(v3, G::V3, 4))) + 1 + j0;
                if (i == n) {
#pragma unroll
                    for (int k = 0; k < P; ++k) if (k < nvalid) xr[k] = 0.0;
                    continue;
                }
#pragma unroll
                for (int k = 0; k < P; ++k) {
                    if (k < nvalid) {
                        const double v = fma(bpow[k], carry[s], p[s][k]);
                        xr[k] = v;
                        if (s == 2) Xrow[gs * (j0 + k)] = v;
                    }
                }
            }

            if (DOWN) {
                // residual of grid row t-6 (final iterate rows t-7..t-5)
                const int ir = t - 6;
                if (ir >= 0 && ir < n) {
                    const double *up = SLOT(v3, G::V3, 7) + jb;
                    const double *cur = SLOT(v3, G::V3, 6) + jb;
                    const double *dn = SLOT(v3, G::V3, 5) + jb;
                    const double *bb = BSLOT(6) + 1 + jb;
                    double *rr = rs + (ir & 1) * W + jb;
#pragma unroll
                    for (int k = 0; k < P; ++k) {
                        const double e1 = fma(-cd, up[k], bb[k]);
                        const double e2 = up[k + 1] + dn[k + 1];
                        const double e3 = cur[k] + cur[k + 2];
                        const double e4 = fma(cd, dn[k + 2], c0 * cur[k + 1]);
                        const double acc = fma(-cy, e3, fma(-cx, e2, e1)) - e4;
                        if (k < nvalid) rr[k] = acc;
                    }
                }
            } else {
                prolongate(t + 2);
            }
#undef SLOT
#undef BSLOT
        }
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// coarse levels in shared memory, one warp per temporal row
// ---------------------------------------------------------------------------
// Level L (m = 2^L - 1 points per direction) is stored with row pitch 2^L so
// the anti-diagonal wavefront stride (pitch - 1 = m, odd) keeps a warp's
// 64-bit shared accesses bank-conflict free.
// Each level's block is a zero pad row, the m grid rows, a zero pad row; the
// pad column (j = m) of every row is zero too, so every neighbour of a grid
// point is an in-bounds word that reads 0 outside the grid (the FAST path
// needs no boundary tests).  off = row 0.
template <int L>
struct Lc {
    static constexpr int m = (1 << L) - 1;
    static constexpr int pitch = 1 << L;
    static constexpr int size = pitch * (m + 2);
    static constexpr int base = Lc<L - 1>::base + Lc<L - 1>::size;
    static constexpr int off = base + pitch;
};
template <>
struct Lc<0> { static constexpr int m = 0, pitch = 1, size = 0, base = 0, off = 0; };
constexpr int kCoarseStack = Lc<kCoarseTop2d>::base + Lc<kCoarseTop2d>::size;
constexpr int kCoarseWords = 2 * kCoarseStack;   // x, b

// level coefficients in registers
struct Cf {
    double c0, cx, cy, cd, inv;
    bool diag;
    HW_DEV Cf(const double *c)
        : c0(c[kC0]), cx(c[kCx]), cy(c[kCy]), cd(c[kCd]), inv(c[kInv]), diag(c[kCd] != 0.0) {}
};

// L-shaped domain (LSH): point (i, j) of level L lies in the removed closed
// quadrant -- not a dof, held at zero.  An unmasked point's neighbours in the
// quadrant contribute exact zeros, and they come last in its CSR row (they
// are "upper" neighbours), so the CSR-order arithmetic is unchanged.
template <int L, bool LSH>
__device__ __forceinline__ bool masked(int i, int j)
{
    constexpr int h = (Lc<L>::m - 1) / 2;
    return LSH && i >= h && j >= h;
}

// one point update.  Exact (FAST = false): CSR column order and the true
// division, bit-identical to the reference -- used when these levels are the
// whole hierarchy (K <= 5).  FAST: the symmetric neighbour pairs summed as a
// shallow tree and a multiply by 1/c0 (a ~5-deep dependent chain instead of
// 12 operations and a division on the wavefront's critical path) -- used
// below the streamed levels, whose results already differ from the
// reference by rounding.
template <int L, bool LSH, bool FAST>
__device__ __forceinline__ void gs_point(double *x, const double *b, const Cf &c, int i, int j)
{
    constexpr int m = Lc<L>::m, p = Lc<L>::pitch;
    if (masked<L, LSH>(i, j)) return;
    const int k = i * p + j;
    if constexpr (FAST) {
        const double xl = j > 0 ? x[k - 1] : 0.0, xr = j < m - 1 ? x[k + 1] : 0.0;
        const double xu = i > 0 ? x[k - p] : 0.0, xd = i < m - 1 ? x[k + p] : 0.0;
        double off = fma(c.cx, xu + xd, c.cy * (xl + xr));
        if (c.diag) {
            const double xa = (i > 0 && j > 0) ? x[k - p - 1] : 0.0;
            const double xb = (i < m - 1 && j < m - 1) ? x[k + p + 1] : 0.0;
            off = fma(c.cd, xa + xb, off);
        }
        x[k] = (b[k] - off) * c.inv;
        return;
    }
    double acc = b[k];
    if (i > 0 && j > 0 && c.diag) acc = sub_mul(acc, c.cd, x[k - p - 1]);
    if (i > 0) acc = sub_mul(acc, c.cx, x[k - p]);
    if (j > 0) acc = sub_mul(acc, c.cy, x[k - 1]);
    if (j < m - 1) acc = sub_mul(acc, c.cy, x[k + 1]);
    if (i < m - 1) acc = sub_mul(acc, c.cx, x[k + p]);
    if (i < m - 1 && j < m - 1 && c.diag) acc = sub_mul(acc, c.cd, x[k + p + 1]);
    x[k] = __ddiv_rn(acc, c.c0);
}

// Three lexicographic GS sweeps (forward) or three of their reverse, by
// anti-diagonal wavefronts with the sweeps PIPELINED three diagonals apart:
// at step tau sweep s updates diagonal tau - 3s.  A point reads the new
// values of its lower neighbours (diagonals d-1, d-2: this sweep, steps
// tau-1, tau-2) and the previous sweep's values of its upper neighbours
// (d+1, d+2: updated by sweep s-1 at steps tau-2, tau-1, not yet by sweep
// s), and within one step no sweep writes a diagonal another one reads --
// so every point sees exactly the operands of three sequential sweeps
// (bit-identical), in 2m+5 steps instead of 3(2m-1).  m <= 31: one grid row
// per lane.
// FAST path of coarse_sweep3: lane i owns grid row i (point (i, d - i) of
// diagonal d), every lane evaluates its three points every step with
// clamped in-range addresses and a predicated store -- no divergent
// branches on the wavefront (ncu: branch resolution was 30 % of the stalls)
template <int L, bool LSH, bool FWD, bool DIAG>
__device__ __forceinline__ void coarse_sweep3_fast(double *x, const double *b, const Cf &c, int lane)
{
    constexpr int m = Lc<L>::m, p = Lc<L>::pitch;
    constexpr int D = 2 * m - 1;
    const int i = lane < m ? lane : m - 1;
    const bool rowok = lane < m;
    double *xr = x + i * p;
    const double *br = b + i * p;
    // column of sweep s at step tau: j = d - i, d = tau - 3 s (forward) or
    // D - 1 - (tau - 3 s) (backward): one increment per step
    int js[3];
#pragma unroll
    for (int s = 0; s < 3; ++s) js[s] = FWD ? -3 * s - i : D - 1 + 3 * s - i;
    for (int tau = 0; tau < D + 6; ++tau) {
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            const int j = js[s];
            const bool ok = rowok && (unsigned)j < (unsigned)m && !masked<L, LSH>(i, j);
            const int jc = min(max(j, 0), m - 1);       // in-bounds address for idle lanes
            const double *xp = xr + jc;
            double off = fma(c.cx, xp[-p] + xp[p], c.cy * (xp[-1] + xp[1]));
            if constexpr (DIAG) off = fma(c.cd, xp[-p - 1] + xp[p + 1], off);
            const double v = (br[jc] - off) * c.inv;
            if (ok) xr[jc] = v;
            js[s] = FWD ? j + 1 : j - 1;
        }
        __syncwarp();
    }
}

template <int L, bool LSH, bool FAST>
__device__ __forceinline__ void coarse_sweep3(double *xw, const double *bw, const Cf &c,
                                              bool forward, int lane)
{
    constexpr int m = Lc<L>::m;
    if constexpr (FAST) {
        double *x = xw + Lc<L>::off;
        const double *b = bw + Lc<L>::off;
        if (forward) {
            if (c.diag) coarse_sweep3_fast<L, LSH, true, true>(x, b, c, lane);
            else coarse_sweep3_fast<L, LSH, true, false>(x, b, c, lane);
        } else {
            if (c.diag) coarse_sweep3_fast<L, LSH, false, true>(x, b, c, lane);
            else coarse_sweep3_fast<L, LSH, false, false>(x, b, c, lane);
        }
        return;
    }
    constexpr int D = 2 * m - 1;                       // diagonals per sweep
    static_assert(m <= 32, "one grid row per lane");
    double *x = xw + Lc<L>::off;
    const double *b = bw + Lc<L>::off;
    for (int tau = 0; tau < D + 6; ++tau) {
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            const int dd = tau - 3 * s;
            if (dd < 0 || dd >= D) continue;
            const int d = forward ? dd : D - 1 - dd;
            const int ilo = d - (m - 1) > 0 ? d - (m - 1) : 0;
            const int ihi = d < m - 1 ? d : m - 1;
            const int i = ilo + lane;
            if (i <= ihi) gs_point<L, LSH, FAST>(x, b, c, i, d - i);
        }
        __syncwarp();
    }
}

// the 5 dofs of the L's level 2 (3 x 3 grid, pitch 4): (0,0) (0,1) (0,2)
// (1,0) (2,0) in lexicographic order
__device__ __forceinline__ int lsh_dof2(int a) { return a < 3 ? a : (a - 2) * 4; }

template <int L, bool LSH, bool FAST>
__device__ __forceinline__ void coarse_vcycle(double *xw, double *bw, const double *coef,
                                              const double *cinv, int lane)
{
    if constexpr (LSH && L == 2) {
        // the L's coarsest level: dense inverse (multigrid.py:118,
        // _kernels.py:168-173: acc += inv[i, j] * b[j] in column order)
        double *x = xw + Lc<2>::off;
        const double *b = bw + Lc<2>::off;
        double acc = 0.0;
        if (lane < 5) {
#pragma unroll
            for (int q = 0; q < 5; ++q) acc = add_mul(acc, cinv[lane * 5 + q], b[lsh_dof2(q)]);
        }
        __syncwarp();
        if (lane < 5) x[lsh_dof2(lane)] = acc;
        __syncwarp();
    } else if constexpr (L >= 2) {
        constexpr int m = Lc<L>::m, p = Lc<L>::pitch, mc = Lc<L - 1>::m, pc = Lc<L - 1>::pitch;
        const double *c = coef + L * kCoefStride;
        const Cf cf(c);
        coarse_sweep3<L, LSH, FAST>(xw, bw, cf, true, lane);
        double *x = xw + Lc<L>::off;
        const double *b = bw + Lc<L>::off;
        // residual r = b - A x, evaluated where the restriction needs it (no r
        // array: the shared footprint per row drops to x and b, two rows per
        // SM more); the exact path keeps the reference's CSR order
        auto res = [&](int i, int j) -> double {
            if (masked<L, LSH>(i, j)) return 0.0;
            const int q = i * p + j;
            if constexpr (FAST) {                        // zero pads: no boundary tests
                double ax = fma(cf.cx, x[q - p] + x[q + p], fma(cf.c0, x[q], cf.cy * (x[q - 1] + x[q + 1])));
                if (cf.diag) ax = fma(cf.cd, x[q - p - 1] + x[q + p + 1], ax);
                return b[q] - ax;
            }
            double acc = b[q];
            if (i > 0 && j > 0 && c[kCd] != 0.0) acc = sub_mul(acc, c[kCd], x[q - p - 1]);
            if (i > 0) acc = sub_mul(acc, c[kCx], x[q - p]);
            if (j > 0) acc = sub_mul(acc, c[kCy], x[q - 1]);
            acc = sub_mul(acc, c[kC0], x[q]);
            if (j < m - 1) acc = sub_mul(acc, c[kCy], x[q + 1]);
            if (i < m - 1) acc = sub_mul(acc, c[kCx], x[q + p]);
            if (i < m - 1 && j < m - 1 && c[kCd] != 0.0) acc = sub_mul(acc, c[kCd], x[q + p + 1]);
            return acc;
        };
        double *xc = xw + Lc<L - 1>::off, *bc = bw + Lc<L - 1>::off;
        for (int k = lane; k < mc * mc; k += 32) {         // restrict, R = P^T in CSR order
            const int I = k / mc, J = k % mc, i0 = 2 * I, j0 = 2 * J;
            double acc = 0.0;
            acc = add_mul(acc, 0.5, res(i0, j0));
            acc = add_mul(acc, 0.5, res(i0, j0 + 1));
            acc = add_mul(acc, 0.5, res(i0 + 1, j0));
            acc = add_mul(acc, 1.0, res(i0 + 1, j0 + 1));
            acc = add_mul(acc, 0.5, res(i0 + 1, j0 + 2));
            acc = add_mul(acc, 0.5, res(i0 + 2, j0 + 1));
            acc = add_mul(acc, 0.5, res(i0 + 2, j0 + 2));
            bc[I * pc + J] = masked<L - 1, LSH>(I, J) ? 0.0 : acc;
        }
        __syncwarp();                                      // all reads of x_(L-1) region done
        for (int k = lane; k < mc * mc; k += 32) xc[(k / mc) * pc + k % mc] = 0.0;
        __syncwarp();
        coarse_vcycle<L - 1, LSH, FAST>(xw, bw, coef, cinv, lane);
        const double *xcc = xw + Lc<L - 1>::off;
        for (int k = lane; k < m * m; k += 32) {           // prolongate (spatial.py:140-173)
            const int gi = k / m + 1, gj = k % m + 1;      // 1-based fine grid coords
            auto cv = [&](int I, int J) -> double {        // 1-based coarse coords
                return (I < 1 || J < 1 || I > mc || J > mc) ? 0.0 : xcc[(I - 1) * pc + (J - 1)];
            };
            double acc = 0.0;
            const int pi = gi & 1, pj = gj & 1;
            if (!pi && !pj) {
                acc = add_mul(acc, 1.0, cv(gi / 2, gj / 2));
            } else {
                const int ai = (gi - pi) / 2, aj = (gj - pj) / 2;
                const int bi = (gi + pi) / 2, bj = (gj + pj) / 2;
                // CSR order: ascending coarse index (a precedes b)
                if (!(ai < 1 || aj < 1 || ai > mc || aj > mc)) acc = add_mul(acc, 0.5, cv(ai, aj));
                if (!(bi < 1 || bj < 1 || bi > mc || bj > mc)) acc = add_mul(acc, 0.5, cv(bi, bj));
            }
            const int q = (gi - 1) * p + (gj - 1);
            if (!masked<L, LSH>(gi - 1, gj - 1)) x[q] = add_rn(x[q], acc);
        }
        __syncwarp();
        coarse_sweep3<L, LSH, FAST>(xw, bw, cf, false, lane);
    } else {
        if (lane == 0)                                  // 1x1 solve
            xw[Lc<1>::off] = add_mul(0.0, coef[1 * kCoefStride + kCoarse], bw[Lc<1>::off]);
        __syncwarp();
    }
}

template <int TOP, int WPB, bool LSH, bool FAST>
__device__ __forceinline__ void coarse_row(const MgCoarseArgs &a, double *xw, int64_t row, int lane)
{
    constexpr int m = Lc<TOP>::m, p = Lc<TOP>::pitch;
    double *bw = xw + kCoarseStack;
    const int op = a.row_op ? a.row_op[row] : a.op;
    const double *coef = a.coef + (int64_t)op * a.levels_p1 * kCoefStride;
    const double *Bg = a.B + row * a.ldB;
    double *Xg = a.X + row * a.ldX;
    for (int k = lane; k < kCoarseWords; k += 32) xw[k] = 0.0;   // pads stay zero
    __syncwarp();
    for (int k = lane; k < m * m; k += 32) {
        const int q = Lc<TOP>::off + (k / m) * p + k % m;
        bw[q] = Bg[k];
        xw[q] = a.zero_start ? 0.0 : Xg[k];
    }
    __syncwarp();
    const double *cinv = LSH ? a.cinv + (int64_t)op * 25 : nullptr;
    for (int cyc = 0; cyc < a.ncyc; ++cyc) coarse_vcycle<TOP, LSH, FAST>(xw, bw, coef, cinv, lane);
    for (int k = lane; k < m * m; k += 32) Xg[k] = xw[Lc<TOP>::off + (k / m) * p + k % m];
}

template <int WPB, bool LSH, bool FAST>
__global__ void __launch_bounds__(32 * WPB) mg2d_coarse(MgCoarseArgs a)
{
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t row = (int64_t)blockIdx.x * WPB + w;
    if (row >= a.rows) return;
    double *xw = sm + (size_t)w * kCoarseWords;
    if constexpr (FAST) {                  // below the streamed levels: top = kCoarseTop2d
        coarse_row<kCoarseTop2d, WPB, LSH, FAST>(a, xw, row, lane);
        return;
    }
    switch (a.top) {
    case 1: if constexpr (!LSH) coarse_row<1, WPB, LSH, FAST>(a, xw, row, lane); break;
    case 2: coarse_row<2, WPB, LSH, FAST>(a, xw, row, lane); break;
    case 3: coarse_row<3, WPB, LSH, FAST>(a, xw, row, lane); break;
    case 4: coarse_row<4, WPB, LSH, FAST>(a, xw, row, lane); break;
    default: coarse_row<5, WPB, LSH, FAST>(a, xw, row, lane); break;
    }
}

// ---------------------------------------------------------------------------
// host-side launchers
// ---------------------------------------------------------------------------
template <int PPT, int NT, bool DOWN>
static cudaError_t launch_stream_t(const MgStreamArgs &a, int64_t rows, cudaStream_t st)
{
    const size_t smem = stream_smem_words<PPT, NT, DOWN>(a.n) * sizeof(double);
    auto k = mg2d_stream<PPT, NT, DOWN>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<(unsigned)rows, NT, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t mg2d_stream_launch(const MgStreamArgs &a, bool down, int64_t rows, cudaStream_t st)
{
    // one CTA per temporal row; P (odd) consecutive points per thread so a
    // warp's 64-bit shared loads at stride 8P bytes are bank-conflict free
    // (P = 5 measured faster than P = 3 with 11 warps at n = 1023)
    const int n = a.n;
    if (a.reg_ok) {
        const cudaError_t e = mg2d_reg_launch(a, down, rows, st);
        if (e != cudaErrorNotSupported) return e;
    }
    if (a.lshape) return cudaErrorNotSupported;   // masked levels: mg2d_reg only
    if (n <= 96)
        return down ? launch_stream_t<3, 32, true>(a, rows, st) : launch_stream_t<3, 32, false>(a, rows, st);
    if (n <= 160)
        return down ? launch_stream_t<5, 32, true>(a, rows, st) : launch_stream_t<5, 32, false>(a, rows, st);
    if (n <= 320)
        return down ? launch_stream_t<5, 64, true>(a, rows, st) : launch_stream_t<5, 64, false>(a, rows, st);
    if (n <= 640)
        return down ? launch_stream_t<5, 128, true>(a, rows, st) : launch_stream_t<5, 128, false>(a, rows, st);
    if (n <= 1120)
        return down ? launch_stream_t<5, 224, true>(a, rows, st) : launch_stream_t<5, 224, false>(a, rows, st);
    return cudaErrorInvalidValue;
}

cudaError_t mg2d_coarse_launch(const MgCoarseArgs &a, cudaStream_t st)
{
    constexpr int WPB = 4;
    const size_t smem = (size_t)WPB * kCoarseWords * sizeof(double);
    auto k = a.fast ? (a.lshape ? mg2d_coarse<WPB, true, true> : mg2d_coarse<WPB, false, true>)
                    : (a.lshape ? mg2d_coarse<WPB, true, false> : mg2d_coarse<WPB, false, false>);
    if (a.fast && a.top != kCoarseTop2d) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)((a.rows + WPB - 1) / WPB);
    k<<<grid, 32 * WPB, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace hw
