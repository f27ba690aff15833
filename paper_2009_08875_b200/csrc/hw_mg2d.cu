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

namespace hw {

// ring sizes, see the lifetime analysis in DESIGN.md §MG
template <bool DOWN> struct Rings;
template <> struct Rings<true> { static constexpr int RX = 11, RB = 9, RR = 4, RC = 0; };
template <> struct Rings<false> { static constexpr int RX = 10, RB = 7, RR = 0, RC = 4; };

template <int PPT, int NT, bool DOWN>
__host__ __device__ constexpr size_t stream_smem_words(int n)
{
    // x ring (padded n+2), b ring (n), r ring (n), coarse ring (m+2),
    // zero row (n+2), scan scratch (NW*3 + powers)
    return (size_t)Rings<DOWN>::RX * (n + 2) + (size_t)Rings<DOWN>::RB * n +
           (size_t)Rings<DOWN>::RR * n + (size_t)Rings<DOWN>::RC * ((n - 1) / 2 + 2) +
           (size_t)(n + 2) + 3 * (NT / 32) + 3 * 40;
}

template <int PPT, int NT, bool DOWN>
__global__ void __launch_bounds__(NT, 1) mg2d_stream(MgStreamArgs a)
{
    using R = Rings<DOWN>;
    constexpr int RRm = R::RR > 0 ? R::RR : 1;   // modulus guards for the
    constexpr int RCm = R::RC > 0 ? R::RC : 1;   // rings a pass does not use
    constexpr int NW = NT / 32;
    constexpr int D = 2;
    extern __shared__ double sm[];

    const int n = a.n;
    const int W = n + 2;
    const int m = (n - 1) / 2;
    const int64_t row = blockIdx.x;
    const int op = a.row_op ? a.row_op[row] : a.op;
    const double *cf = a.coef + ((int64_t)op * a.levels_p1 + a.level) * kCoefStride;
    const double c0 = cf[kC0], cx = cf[kCx], cy = cf[kCy], cd = cf[kCd], inv = cf[kInv];
    const double beta = -cy * inv;

    double *xs = sm;                                   // RX * W
    double *bs = xs + R::RX * W;                       // RB * n
    double *rs = bs + R::RB * n;                       // RR * n
    double *cs = rs + R::RR * n;                       // RC * (m+2)
    double *zr = cs + R::RC * (m + 2);                 // W zeros
    double *wt = zr + W;                               // NW * 3 warp totals
    double *gp = wt + 3 * NW;                          // powers: gamma^l (33), beta^k (PPT+1)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double *Bg = a.B + row * a.ldB;
    double *Xg = a.X + row * a.ldX;

    // powers of beta and gamma = beta^PPT (uniform per CTA)
    if (tid == 0) {
        double bp = 1.0;
        for (int k = 0; k <= PPT; ++k) { gp[33 + k] = bp; bp *= beta; }
        const double g = gp[33 + PPT];
        double q = 1.0;
        for (int l = 0; l <= 32; ++l) { gp[l] = q; q *= g; }
    }
    for (int k = tid; k < W; k += NT) zr[k] = 0.0;
    for (int s = 0; s < R::RX; ++s)
        for (int k = tid; k < W; k += NT) xs[s * W + k] = 0.0;
    if (!DOWN)
        for (int s = 0; s < R::RC; ++s)
            for (int k = tid; k < m + 2; k += NT) cs[s * (m + 2) + k] = 0.0;
    __syncthreads();

    auto xrow = [&](int i) -> double * { return (i < 0 || i >= n) ? zr : xs + (i % R::RX) * W; };
    auto brow = [&](int i) -> double * { return bs + (i % R::RB) * n; };
    auto crow = [&](int c) -> const double * {
        return (c < 0 || c >= m) ? zr : cs + (c % RCm) * (m + 2);
    };
    // global index of (grid row i, col j) in the pass's own (possibly
    // reversed) coordinates
    auto gidx = [&](int i, int j) -> int64_t {
        return DOWN ? (int64_t)i * n + j : (int64_t)(n - 1 - i) * n + (n - 1 - j);
    };

    // issue the loads of "virtual step" s: b row s+D; x row s+D+1 (DOWN,
    // unless zero start) or s+D+2 (UP) and the coarse row it first needs.
    auto issue = [&](int s) {
        const int ib = s + D;
        if (ib >= 0 && ib < n) {
            double *dst = brow(ib);
            for (int j = tid; j < n; j += NT) cp_async8(dst + j, Bg + gidx(ib, j));
        }
        const int ix = DOWN ? s + D + 1 : s + D + 2;
        if (ix >= 0 && ix < n) {
            double *dst = xs + (ix % R::RX) * W + 1;
            if (DOWN && a.zero_start) {
                for (int j = tid; j < n; j += NT) dst[j] = 0.0;
            } else {
                for (int j = tid; j < n; j += NT) cp_async8(dst + j, Xg + gidx(ix, j));
            }
            if (!DOWN && (ix % 2 == 0) && ix / 2 < m) {
                // coarse row c = ix/2 (reversed coordinates) first used by fine row 2c
                const int c = ix / 2;
                const double *Xc = a.Xc + row * a.ldXc;
                double *cdst = cs + (c % RCm) * (m + 2) + 1;
                for (int J = tid; J < m; J += NT)
                    cp_async8(cdst + J, Xc + (int64_t)(m - 1 - c) * m + (m - 1 - J));
            }
        }
        cp_async_commit();
    };

    // x[i] += P x_coarse (reversed coordinates, spatial.py:140-173)
    auto prolongate = [&](int i) {
        if (i < 0 || i >= n) return;
        double *xr = xs + (i % R::RX) * W + 1;
        const double *ca, *cb;
        if (i & 1) { ca = crow((i - 1) / 2); cb = nullptr; }
        else { ca = crow(i / 2 - 1); cb = crow(i / 2); }
        for (int j = tid; j < n; j += NT) {
            double v;
            if (i & 1) {
                if (j & 1) v = ca[1 + (j - 1) / 2];
                else v = 0.5 * ca[1 + j / 2 - 1] + 0.5 * ca[1 + j / 2];
            } else {
                if (j & 1) v = 0.5 * ca[1 + (j - 1) / 2] + 0.5 * cb[1 + (j - 1) / 2];
                else v = 0.5 * ca[1 + j / 2 - 1] + 0.5 * cb[1 + j / 2];
            }
            xr[j] += v;
        }
    };

    // prologue
    const int first = DOWN ? -D - 1 : -D - 2;
    for (int s = first; s < 0; ++s) issue(s);
    if (!DOWN) {
        cp_async_wait<D>();
        __syncthreads();
        prolongate(0);
        prolongate(1);
    }

    const int j0 = tid * PPT;
    const int nsteps = DOWN ? n + 7 : n + 4;

    for (int t = 0; t < nsteps; ++t) {
        cp_async_wait<D - 1>();
        __syncthreads();
        issue(t);

        // ---------------- phase A: right-hand sides from old values ----------
        double p[3][PPT];
        bool act[3];
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            const int i = t - 2 * s;
            act[s] = (i >= 0 && i < n);
            if (!act[s]) {
#pragma unroll
                for (int k = 0; k < PPT; ++k) p[s][k] = 0.0;
                continue;
            }
            const double *xu = xrow(i - 1) + 1, *xc = xrow(i) + 1, *xd = xrow(i + 1) + 1;
            const double *br = brow(i);
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                const int j = j0 + k;
                double acc = 0.0;
                if (j < n) {
                    acc = br[j];
                    acc -= cd * xu[j - 1];
                    acc -= cx * xu[j];
                    acc -= cy * xc[j + 1];
                    acc -= cx * xd[j];
                    acc -= cd * xd[j + 1];
                    acc *= inv;
                }
                p[s][k] = acc;
            }
        }
        if (DOWN) {
            const int ir = t - 6;
            if (ir >= 0 && ir < n) {
                const double *xu = xrow(ir - 1) + 1, *xc = xrow(ir) + 1, *xd = xrow(ir + 1) + 1;
                const double *br = brow(ir);
                double *rr = rs + (ir % RRm) * n;
                for (int j = tid; j < n; j += NT) {
                    double acc = br[j];
                    acc -= cd * xu[j - 1];
                    acc -= cx * xu[j];
                    acc -= cy * xc[j - 1];
                    acc -= c0 * xc[j];
                    acc -= cy * xc[j + 1];
                    acc -= cx * xd[j];
                    acc -= cd * xd[j + 1];
                    rr[j] = acc;
                }
            }
            if ((t & 1) && t >= 9) {
                const int I = (t - 9) / 2;
                if (I < m) {
                    const double *r0 = rs + ((2 * I) % RRm) * n;
                    const double *r1 = rs + ((2 * I + 1) % RRm) * n;
                    const double *r2 = rs + ((2 * I + 2) % RRm) * n;
                    double *bc = a.Bc + row * a.ldBc + (int64_t)I * m;
                    for (int J = tid; J < m; J += NT) {
                        const int c = 2 * J;
                        double acc = 0.5 * r0[c];
                        acc += 0.5 * r0[c + 1];
                        acc += 0.5 * r1[c];
                        acc += r1[c + 1];
                        acc += 0.5 * r1[c + 2];
                        acc += 0.5 * r2[c + 1];
                        acc += 0.5 * r2[c + 2];
                        bc[J] = acc;
                    }
                }
            }
        }
        __syncthreads();

        // ---------------- phase B: affine scans along the rows ---------------
        double S[3];
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            double y = 0.0;
#pragma unroll
            for (int k = 0; k < PPT; ++k) { y = fma(beta, y, p[s][k]); p[s][k] = y; }
            S[s] = y;
        }
        // inclusive warp scan of T_l = S_l + gamma T_{l-1}
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double g = gp[o];
#pragma unroll
            for (int s = 0; s < 3; ++s) {
                const double v = __shfl_up_sync(0xffffffffu, S[s], o);
                if (lane >= o) S[s] = fma(g, v, S[s]);
            }
        }
        if (lane == 31)
#pragma unroll
            for (int s = 0; s < 3; ++s) wt[warp * 3 + s] = S[s];
        __syncthreads();
        const double G32 = gp[32];
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            double Cw = 0.0;
            for (int v = 0; v < warp; ++v) Cw = fma(G32, Cw, wt[v * 3 + s]);
            const double prev = __shfl_up_sync(0xffffffffu, S[s], 1);
            const double carry = (lane == 0) ? Cw : fma(gp[lane], Cw, prev);
            if (act[s]) {
                const int i = t - 2 * s;
                double *xr = xs + (i % R::RX) * W + 1;
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    const int j = j0 + k;
                    if (j < n) {
                        const double v = fma(gp[33 + k + 1], carry, p[s][k]);
                        xr[j] = v;
                        if (s == 2) Xg[gidx(i, j)] = v;
                    }
                }
            }
        }
        if (!DOWN) prolongate(t + 2);
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// coarse levels in shared memory, one warp per temporal row
// ---------------------------------------------------------------------------
constexpr int kCoarseWords = 2 * (1 + 9 + 49 + 225 + 961) + 961;  // x, b, r

__device__ __forceinline__ int lvl_off(int l)
{
    // offset of level l (1-based) in the concatenated hierarchy
    int o = 0;
    for (int k = 1; k < l; ++k) o += ((1 << k) - 1) * ((1 << k) - 1);
    return o;
}

template <int WPB>
__global__ void __launch_bounds__(32 * WPB) mg2d_coarse(MgCoarseArgs a)
{
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t row = (int64_t)blockIdx.x * WPB + w;
    if (row >= a.rows) return;
    double *xw = sm + (size_t)w * kCoarseWords;
    double *bw = xw + (kCoarseWords - 961) / 2;
    double *rw = bw + (kCoarseWords - 961) / 2;
    const int op = a.row_op ? a.row_op[row] : a.op;
    const int top = a.top;
    const int mt = (1 << top) - 1;
    const int ot = lvl_off(top);
    const double *Bg = a.B + row * a.ldB;
    double *Xg = a.X + row * a.ldX;
    for (int k = lane; k < mt * mt; k += 32) {
        bw[ot + k] = Bg[k];
        xw[ot + k] = a.zero_start ? 0.0 : Xg[k];
    }
    __syncwarp();

    auto C = [&](int l) { return a.coef + ((int64_t)op * a.levels_p1 + l) * kCoefStride; };

    // one point update in CSR column order (the reference's arithmetic)
    auto gs_point = [&](double *x, const double *b, const double *c, int m, int i, int j) {
        double acc = b[i * m + j];
        if (i > 0 && j > 0 && c[kCd] != 0.0) acc = sub_mul(acc, c[kCd], x[(i - 1) * m + j - 1]);
        if (i > 0) acc = sub_mul(acc, c[kCx], x[(i - 1) * m + j]);
        if (j > 0) acc = sub_mul(acc, c[kCy], x[i * m + j - 1]);
        if (j < m - 1) acc = sub_mul(acc, c[kCy], x[i * m + j + 1]);
        if (i < m - 1) acc = sub_mul(acc, c[kCx], x[(i + 1) * m + j]);
        if (i < m - 1 && j < m - 1 && c[kCd] != 0.0) acc = sub_mul(acc, c[kCd], x[(i + 1) * m + j + 1]);
        x[i * m + j] = __ddiv_rn(acc, c[kC0]);
    };
    auto sweep = [&](int l, bool forward) {
        const int m = (1 << l) - 1;
        double *x = xw + lvl_off(l);
        const double *b = bw + lvl_off(l);
        const double *c = C(l);
        for (int dd = 0; dd <= 2 * m - 2; ++dd) {
            const int d = forward ? dd : 2 * m - 2 - dd;
            const int ilo = d - (m - 1) > 0 ? d - (m - 1) : 0;
            const int ihi = d < m - 1 ? d : m - 1;
            for (int i = ilo + lane; i <= ihi; i += 32) gs_point(x, b, c, m, i, d - i);
            __syncwarp();
        }
    };

    for (int cyc = 0; cyc < a.ncyc; ++cyc) {
        for (int l = top; l >= 2; --l) {
            const int m = (1 << l) - 1, mc = (1 << (l - 1)) - 1;
            for (int s = 0; s < 3; ++s) sweep(l, true);
            double *x = xw + lvl_off(l);
            const double *b = bw + lvl_off(l);
            const double *c = C(l);
            for (int k = lane; k < m * m; k += 32) {      // residual
                const int i = k / m, j = k % m;
                double acc = b[k];
                if (i > 0 && j > 0 && c[kCd] != 0.0) acc = sub_mul(acc, c[kCd], x[k - m - 1]);
                if (i > 0) acc = sub_mul(acc, c[kCx], x[k - m]);
                if (j > 0) acc = sub_mul(acc, c[kCy], x[k - 1]);
                acc = sub_mul(acc, c[kC0], x[k]);
                if (j < m - 1) acc = sub_mul(acc, c[kCy], x[k + 1]);
                if (i < m - 1) acc = sub_mul(acc, c[kCx], x[k + m]);
                if (i < m - 1 && j < m - 1 && c[kCd] != 0.0) acc = sub_mul(acc, c[kCd], x[k + m + 1]);
                rw[k] = acc;
            }
            __syncwarp();
            double *xc = xw + lvl_off(l - 1), *bc = bw + lvl_off(l - 1);
            for (int k = lane; k < mc * mc; k += 32) {    // restrict
                const int I = k / mc, J = k % mc;
                const double *r0 = rw + (2 * I) * m + 2 * J;
                const double *r1 = r0 + m, *r2 = r1 + m;
                double acc = 0.0;
                acc = add_mul(acc, 0.5, r0[0]);
                acc = add_mul(acc, 0.5, r0[1]);
                acc = add_mul(acc, 0.5, r1[0]);
                acc = add_mul(acc, 1.0, r1[1]);
                acc = add_mul(acc, 0.5, r1[2]);
                acc = add_mul(acc, 0.5, r2[1]);
                acc = add_mul(acc, 0.5, r2[2]);
                bc[k] = acc;
                xc[k] = 0.0;
            }
            __syncwarp();
        }
        if (lane == 0) xw[0] = add_mul(0.0, C(1)[kCoarse], bw[0]);  // 1x1 coarse solve
        __syncwarp();
        for (int l = 2; l <= top; ++l) {
            const int m = (1 << l) - 1, mc = (1 << (l - 1)) - 1;
            double *x = xw + lvl_off(l);
            const double *xc = xw + lvl_off(l - 1);
            for (int k = lane; k < m * m; k += 32) {       // prolongate
                const int gi = k / m + 1, gj = k % m + 1; // 1-based fine grid coords
                double acc = 0.0;
                auto cv = [&](int I, int J) -> double {   // 1-based coarse coords
                    return (I < 1 || J < 1 || I > mc || J > mc) ? 0.0 : xc[(I - 1) * mc + (J - 1)];
                };
                const int pi = gi & 1, pj = gj & 1;
                if (!pi && !pj) {
                    acc = add_mul(acc, 1.0, cv(gi / 2, gj / 2));
                } else {
                    const int ai = (gi - pi) / 2, aj = (gj - pj) / 2;
                    const int bi = (gi + pi) / 2, bj = (gj + pj) / 2;
                    const bool aok = !(ai < 1 || aj < 1 || ai > mc || aj > mc);
                    const bool bok = !(bi < 1 || bj < 1 || bi > mc || bj > mc);
                    // CSR order: ascending coarse index (a precedes b)
                    if (aok) acc = add_mul(acc, 0.5, cv(ai, aj));
                    if (bok) acc = add_mul(acc, 0.5, cv(bi, bj));
                }
                x[k] = add_rn(x[k], acc);
            }
            __syncwarp();
            for (int s = 0; s < 3; ++s) sweep(l, false);
        }
    }
    for (int k = lane; k < mt * mt; k += 32) Xg[k] = xw[ot + k];
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
    // NT * PPT >= n; one CTA per temporal row
    const int n = a.n;
    if (n <= 64)
        return down ? launch_stream_t<2, 32, true>(a, rows, st) : launch_stream_t<2, 32, false>(a, rows, st);
    if (n <= 128)
        return down ? launch_stream_t<4, 32, true>(a, rows, st) : launch_stream_t<4, 32, false>(a, rows, st);
    if (n <= 256)
        return down ? launch_stream_t<4, 64, true>(a, rows, st) : launch_stream_t<4, 64, false>(a, rows, st);
    if (n <= 512)
        return down ? launch_stream_t<4, 128, true>(a, rows, st) : launch_stream_t<4, 128, false>(a, rows, st);
    if (n <= 1024)
        return down ? launch_stream_t<4, 256, true>(a, rows, st) : launch_stream_t<4, 256, false>(a, rows, st);
    return cudaErrorInvalidValue;
}

cudaError_t mg2d_coarse_launch(const MgCoarseArgs &a, cudaStream_t st)
{
    constexpr int WPB = 4;
    const size_t smem = (size_t)WPB * kCoarseWords * sizeof(double);
    auto k = mg2d_coarse<WPB>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)((a.rows + WPB - 1) / WPB);
    k<<<grid, 32 * WPB, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace hw
