// hw_mg1d_rr.cu -- batched 1D V-cycles with the whole streamed hierarchy in
// registers (mg1d_rr), levels > kRrCut; the V-cycle from level kRrCut down
// applied as a dense operator.
//
// Restates _mg_core (/root/reference/pkg/src/heatwave/_kernels.py:110-199)
// for d = 1 (levels l = 1..K with 2^l - 1 points, spatial.py:98-103; P from
// spatial.py:140-173, R = P^T; 3 forward lexicographic GS sweeps before the
// restriction, 3 backward after the prolongation, 1x1 coarse inverse).
//
// One warp owns one temporal row.  At level l lane t owns the C = 2^(l-5)
// consecutive points [tC, tC + C) (the last point of lane 31 is a phantom
// held at zero), so the restriction of lane t's residuals lands exactly in
// lane t's coarse chunk and the prolongation reads lane t's coarse chunk
// plus one value of lane t - 1: every level's iterate stays in registers,
// only the right-hand sides b' = b / c0 live in shared memory (16-byte units,
// XOR-swizzled so a warp's LDS.128 of its chunks is conflict free).
//
// A GS sweep is the recurrence x_k = p_k + beta x_{k-1}, p_k = b'_k + beta
// x_{k+1}^old (beta = -c_y / c_0; backward sweeps mirrored).  A lane forms
// p, the zero-carry end of its chunk (NS independent sub-chunk chains), and
// then the recurrence again from the true carry.  |beta| < 1/2 for every
// alpha A + mu M in 1D (c_0 = 2a/h + 4mh/6 > 2|c_y|), so the carry into lane
// t, sum_k gamma^(k-1) S_(t-k) (gamma = beta^C, S = zero-carry chunk ends),
// is truncated after W = 64 / C chunks (gamma^W <= 2^-64, 11 bits below one
// fp64 rounding): lexicographic GS up to rounding, with a 1-3 step windowed
// shuffle scan instead of the exact 5-step scan (C <= 2 keeps the exact scan).
//
// Levels <= kRrCut (63 points): the zero-start V-cycle from that level is a
// fixed linear map, G[op][s][j] = (MG e_s)_j, built by hwg_create with the
// exact shared-memory kernel (mg1d_smem) on unit right-hand sides; lane t
// applies its two columns to the broadcast level right-hand side.
#include "hw_common.cuh"
#include "hw_internal.cuh"

namespace hw {
namespace rr {

template <int L>
struct RL {
    static constexpr int C = 1 << (L - 5);             // points per lane
    static constexpr int U = C / 2;                    // 16-byte units per lane
    static constexpr int off = 32 * (C - (1 << (kRrCut - 5)));   // doubles, level kRrCut at 0
    static constexpr int size = 32 * C;
    // unit u of lane t sits at unit t U + (u ^ swz(t)): the 8 lanes of an
    // LDS.128 phase touch 8 distinct 16-byte bank groups
    HW_DEV static int swz(int t)
    {
        if constexpr (U >= 8) return t & 7;
        else if constexpr (U == 4) return (t >> 1) & 3;
        else if constexpr (U == 2) return (t >> 2) & 1;
        else return 0;
    }
    HW_DEV static int unit(int t, int u) { return t * U + (u ^ swz(t)); }
    HW_DEV static int point(int j)                     // double index of point j
    {
        const int t = j / C, k = j % C;
        return off + 2 * unit(t, k >> 1) + (k & 1);
    }
};

template <int L>
HW_DEV void load_b(const double *s, int t, double (&v)[RL<L>::C])
{
#pragma unroll
    for (int u = 0; u < RL<L>::U; ++u) {
        const double2 d = *reinterpret_cast<const double2 *>(s + RL<L>::off + 2 * RL<L>::unit(t, u));
        v[2 * u] = d.x;
        v[2 * u + 1] = d.y;
    }
}

template <int L>
HW_DEV void store_b(double *s, int t, const double (&v)[RL<L>::C])
{
#pragma unroll
    for (int u = 0; u < RL<L>::U; ++u)
        *reinterpret_cast<double2 *>(s + RL<L>::off + 2 * RL<L>::unit(t, u)) =
            make_double2(v[2 * u], v[2 * u + 1]);
}

// carry into lane t from the zero-carry chunk ends S of the lanes before it
// (forward: t-1, t-2, ...; backward: t+1, t+2, ...), gamma = beta^C, truncated
// after W = 64 / C chunks: sum_{k=1..W} gamma^(k-1) S(t-k).  A 64-bit shuffle
// costs ~27 cycles and sits on the sweep's critical path (a DFMA 8), so for
// small chunks (C <= kPfMaxC, W >= 8: the scan is most of the sweep) the window
// is summed with few DEPENDENT shuffles: log2(W/4) doubling rounds build block
// sums of B = W/4 chunks, then the four blocks are fetched with independent
// shuffles and combined by Horner.  Larger chunks keep the plain doubling scan
// (fewer live registers where the level's iterate is large).
#ifndef RR_PF_MAXC
#define RR_PF_MAXC 8
#endif
constexpr int kPfMaxC = RR_PF_MAXC;
template <int C, bool FWD>
HW_DEV double lane_carry(double S, double gam, int lane)
{
    constexpr int W = (64 + C - 1) / C;                // chunks in the window
    auto sh = [&](double v, int o) {
        return FWD ? __shfl_up_sync(0xffffffffu, v, o) : __shfl_down_sync(0xffffffffu, v, o);
    };
    auto has = [&](int o) { return FWD ? lane >= o : lane + o < 32; };
    if constexpr (W == 2) {
        const double s1 = sh(S, 1), s2 = sh(S, 2);
        const double a = has(1) ? s1 : 0.0, b = has(2) ? s2 : 0.0;
        return fma(gam, b, a);
    } else if constexpr (C <= kPfMaxC && W >= 4 && W <= 32) {
        constexpr int B = W / 4;
        double T = S, g = gam;
#pragma unroll
        for (int o = 1; o < B; o <<= 1) {              // T(t) = sum_{k<2o} gamma^k S(t-k)
            const double v = sh(T, o);
            T = fma(g, has(o) ? v : 0.0, T);
            g *= g;
        }
        const double v0 = sh(T, 1), v1 = sh(T, 1 + B), v2 = sh(T, 1 + 2 * B), v3 = sh(T, 1 + 3 * B);
        const double a0 = has(1) ? v0 : 0.0, a1 = has(1 + B) ? v1 : 0.0;
        const double a2 = has(1 + 2 * B) ? v2 : 0.0, a3 = has(1 + 3 * B) ? v3 : 0.0;
        return fma(g, fma(g, fma(g, a3, a2), a1), a0);   // g = gamma^B
    } else {
        double T = S, g = gam;
#pragma unroll
        for (int o = 1; o < (W < 32 ? W : 32); o <<= 1) {
            const double v = sh(T, o);
            if (has(o)) T = fma(g, v, T);
            g *= g;
        }
        const double c = sh(T, 1);
        return has(1) ? c : 0.0;
    }
}

// one GS sweep on the lane's chunk x[C] (FWD: increasing j; else decreasing);
// ZS: the iterate is zero before the sweep.  bp: b' of the chunk
template <int L, bool FWD, bool ZS>
HW_DEV void sweep(double (&x)[RL<L>::C], const double *s, double beta, int lane)
{
    constexpr int C = RL<L>::C;
    constexpr int NS = C >= 16 ? 4 : (C >= 4 ? 2 : 1);
    constexpr int SC = C / NS;
    const bool tail = lane == 31;                      // owns the phantom point C - 1
    double bp[C];
    load_b<L>(s, lane, bp);
    // p in place (the neighbour is read before it is overwritten)
    if constexpr (ZS) {
#pragma unroll
        for (int k = 0; k < C; ++k) x[k] = bp[k];
    } else if constexpr (FWD) {
        const double xr = __shfl_down_sync(0xffffffffu, x[0], 1);
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const double xn = (k + 1 < C) ? x[k + 1] : (tail ? 0.0 : xr);
            x[k] = fma(beta, xn, bp[k]);
        }
    } else {
        const double xl = __shfl_up_sync(0xffffffffu, x[C - 1], 1);
#pragma unroll
        for (int k = C - 1; k >= 0; --k) {
            const double xn = (k > 0) ? x[k - 1] : (lane == 0 ? 0.0 : xl);
            x[k] = fma(beta, xn, bp[k]);
        }
    }
    if (!FWD && tail) x[C - 1] = 0.0;                  // the phantom starts lane 31's chain
    // zero-carry sub-chunk ends (sub-chunk q: the q-th SC points in sweep order)
    auto idx = [](int q, int i) { return FWD ? q * SC + i : C - 1 - (q * SC + i); };
    double e[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) {
        double y = x[idx(q, 0)];
#pragma unroll
        for (int i = 1; i < SC; ++i) y = fma(beta, y, x[idx(q, i)]);
        e[q] = y;
    }
    double bsc = beta;                                 // beta^SC
#pragma unroll
    for (int i = 1; i < SC; ++i) bsc *= beta;
    double T = e[0];
#pragma unroll
    for (int q = 1; q < NS; ++q) T = fma(bsc, T, e[q]);
    double gam = bsc;                                  // beta^C
#pragma unroll
    for (int q = 1; q < NS; ++q) gam *= bsc;
    double carry = lane_carry<C, FWD>(T, gam, lane);
#pragma unroll
    for (int q = 0; q < NS; ++q) {
        double y = carry;
#pragma unroll
        for (int i = 0; i < SC; ++i) {
            y = fma(beta, y, x[idx(q, i)]);
            x[idx(q, i)] = y;
        }
        carry = fma(bsc, carry, e[q]);
    }
    if (FWD && tail) x[C - 1] = 0.0;
}

// r' = b' - x + beta (x_l + x_r) (= r / c0) on level L, restricted into
// level L-1 right-hand sides kap * (r'_2i + r'_2i+2) / 2 + kap * r'_2i+1,
// stored in level L-1's shared-memory slots
template <int L>
HW_DEV void restrict_to(const double (&x)[RL<L>::C], double *s, double beta, double kap,
                        int lane)
{
    constexpr int C = RL<L>::C, NC = C / 2;
    const bool tail = lane == 31;
    double bp[C];
    load_b<L>(s, lane, bp);
    const double xl0 = __shfl_up_sync(0xffffffffu, x[C - 1], 1);
    const double xl = lane == 0 ? 0.0 : xl0;
    const double xr0 = __shfl_down_sync(0xffffffffu, x[0], 1);
    const double xr = tail ? 0.0 : xr0;
    double r[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
        const double a0 = k > 0 ? x[k - 1] : xl;
        const double a2 = k + 1 < C ? x[k + 1] : xr;
        r[k] = fma(beta, a0 + a2, bp[k] - x[k]);
    }
    const double rn = __shfl_down_sync(0xffffffffu, r[0], 1);
    double bc[NC > 0 ? NC : 1];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
        const double r2 = 2 * q + 2 < C ? r[2 * q + 2] : rn;
        bc[q] = kap * fma(0.5, r[2 * q] + r2, r[2 * q + 1]);
    }
    if (tail) bc[NC - 1] = 0.0;                        // the coarse phantom
    if constexpr (NC >= 2) {
        store_b<L - 1>(s, lane, bc);
    } else {
        s[RL<L - 1>::off + lane] = bc[0];
    }
}

// x (level L) += P xc (level L-1)
template <int L>
HW_DEV void prolongate(double (&x)[RL<L>::C], const double (&xc)[RL<L>::C / 2], int lane)
{
    constexpr int C = RL<L>::C, NC = C / 2;
    const double xcl0 = __shfl_up_sync(0xffffffffu, xc[NC - 1], 1);
    const double xcl = lane == 0 ? 0.0 : xcl0;
#pragma unroll
    for (int k = 0; k < C; ++k) {
        if (k & 1) {
            x[k] += xc[(k - 1) / 2];
        } else {
            const double lo = k == 0 ? xcl : xc[k / 2 - 1];
            x[k] += 0.5 * (lo + xc[k / 2]);
        }
    }
    if (lane == 31) x[C - 1] = 0.0;
}

// x (level kRrCut, C = 2 points per lane) = G b: b broadcast from shared
// memory; GS: G staged in shared memory by the CTA (mg1d_rrp), else read
// through L1
template <bool GS>
HW_DEV void dense_cut(double (&x)[RL<kRrCut>::C], const double *s, const double *G, int lane)
{
    constexpr int C = RL<kRrCut>::C, n = (1 << kRrCut) - 1, ld = 32 * C;
    static_assert(C == 2, "dense_cut assumes two points per lane at the cut level");
    double a0 = 0.0, a1 = 0.0, c0 = 0.0, c1 = 0.0;
    const double *g = G + 2 * lane;
    auto ldg2 = [](const double *p) {
        if constexpr (GS) return *reinterpret_cast<const double2 *>(p);
        else return __ldg(reinterpret_cast<const double2 *>(p));
    };
#pragma unroll 8
    for (int m = 0; m < (n + 1) / 2; ++m) {           // points 2m, 2m+1 (unit m, no swizzle at U = 1)
        const double2 bb = *reinterpret_cast<const double2 *>(s + RL<kRrCut>::off + 2 * m);
        const double2 g0 = ldg2(g + (2 * m) * ld);
        a0 = fma(g0.x, bb.x, a0);
        a1 = fma(g0.y, bb.x, a1);
        if (2 * m + 1 < n) {
            const double2 g1 = ldg2(g + (2 * m + 1) * ld);
            c0 = fma(g1.x, bb.y, c0);
            c1 = fma(g1.y, bb.y, c1);
        }
    }
    x[0] = a0 + c0;
    x[1] = a1 + c1;
}

struct Lv {
    double beta, kap;
};
HW_DEV Lv level_coef(const double *coef, int L)
{
    const double *c = coef + L * kCoefStride;
    const double *cc = coef + (L - 1) * kCoefStride;
    Lv v;
    v.beta = -c[kCy] * c[kInv];
    v.kap = (L - 1 == kRrCut) ? c[kC0] : c[kC0] * cc[kInv];   // the cut level keeps unscaled b
    return v;
}

template <int L, bool TOP, bool GS>
HW_DEV void vcycle(double (&x)[RL<L>::C], double *s, const double *coef, const double *G,
                   int lane, bool zs)
{
    constexpr int C = RL<L>::C;
    const Lv cf = level_coef(coef, L);
    if (!TOP || zs) sweep<L, true, true>(x, s, cf.beta, lane);
    else sweep<L, true, false>(x, s, cf.beta, lane);
    sweep<L, true, false>(x, s, cf.beta, lane);
    sweep<L, true, false>(x, s, cf.beta, lane);
    restrict_to<L>(x, s, cf.beta, cf.kap, lane);
    __syncwarp();
    double xc[C / 2];
    if constexpr (L - 1 == kRrCut) {
        dense_cut<GS>(xc, s, G, lane);
    } else {
        vcycle<L - 1, false, GS>(xc, s, coef, G, lane, true);
    }
    prolongate<L>(x, xc, lane);
    sweep<L, false, false>(x, s, cf.beta, lane);
    sweep<L, false, false>(x, s, cf.beta, lane);
    sweep<L, false, false>(x, s, cf.beta, lane);
}

}  // namespace rr

template <int K, int WPB, int MINB>
__global__ void __launch_bounds__(32 * WPB, MINB) mg1d_rr(Mg1dArgs a)
{
    using namespace rr;
    constexpr int C = RL<K>::C;
    constexpr int words = RL<K>::off + RL<K>::size;
    extern __shared__ double4 smraw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t row = (int64_t)blockIdx.x * WPB + w;
    if (row >= a.rows) return;                        // whole warps; no CTA barriers below
    double *s = reinterpret_cast<double *>(smraw) + (size_t)w * words;
    const int op = a.row_op ? a.row_op[row] : a.op;
    const double *coef = a.coef + (int64_t)op * a.levels_p1 * kCoefStride;
    const double *G = a.cmat_rr + (int64_t)op * kRrCutN * (32 * RL<kRrCut>::C);
    constexpr int nK = (1 << K) - 1;
    {   // warm L2 with the row the next CTA wave loads
        const int64_t ahead = row + 148LL * WPB * MINB;
        if (ahead < a.rows) {
            const char *p = reinterpret_cast<const char *>(a.B + ahead * a.ldB);
            for (int o = lane * 128; o < nK * 8; o += 32 * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(p + o));
        }
    }
    {   // b' = b / c0 of the finest level, coalesced row load into the swizzled slots
        const double inv = coef[K * kCoefStride + kInv];
        const double *Bg = a.B + row * a.ldB;
#pragma unroll 4
        for (int j = lane; j < 32 * C; j += 32) s[RL<K>::point(j)] = j < nK ? Bg[j] * inv : 0.0;
        __syncwarp();
    }
    double x[C];
#pragma unroll
    for (int k = 0; k < C; ++k) x[k] = 0.0;
    for (int cyc = 0; cyc < a.ncyc; ++cyc) vcycle<K, true, false>(x, s, coef, G, lane, cyc == 0);
    __syncwarp();
    store_b<K>(s, lane, x);                           // the row through the same slots
    __syncwarp();
    double *Xg = a.X + row * a.ldX;
#pragma unroll 4
    for (int j = lane; j < nK; j += 32) Xg[j] = s[RL<K>::point(j)];
}

// mg1d_rrp: the same per-row work as mg1d_rr in one persistent CTA of WPB
// warps per SM.  Rows are dealt out in tiles of WPB * TR consecutive rows;
// the dense cut-level operator of a tile's (first row's) multigrid operator
// is staged once in shared memory -- the rows of one wavelet level are
// contiguous, so it changes J + 1 times over the whole batch -- and every
// row of that operator applies it with LDS instead of 128 L1/L2 loads.  A row
// with another operator (a tile that straddles two levels) reads it through
// L1 as mg1d_rr does.  The row itself is loaded with 32 independent
// streaming loads per lane; the warp's next row is prefetched into L2.
template <int K, int WPB>
__global__ void __launch_bounds__(32 * WPB, 1) mg1d_rrp(Mg1dArgs a, int TR)
{
    using namespace rr;
    constexpr int C = RL<K>::C;
    constexpr int words = RL<K>::off + RL<K>::size;
    constexpr int gwords = kRrCutN * kRrCutLd;
    constexpr int nK = (1 << K) - 1;
    extern __shared__ double4 smraw[];
    double *Gs = reinterpret_cast<double *>(smraw);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double *s = Gs + kRrCutLd * kRrCutLd + (size_t)w * words;
    const int64_t tile_rows = (int64_t)WPB * TR;
    const int64_t ntiles = (a.rows + tile_rows - 1) / tile_rows;
    int cur_op = -1;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t row0 = tile * tile_rows;
        const int op_t = a.row_op ? a.row_op[row0] : a.op;
        if (op_t != cur_op) {                          // uniform over the CTA
            __syncthreads();                           // nobody still reads the old operator
            const double2 *src = reinterpret_cast<const double2 *>(a.cmat_rr + (int64_t)op_t * gwords);
            double2 *dst = reinterpret_cast<double2 *>(Gs);
            for (int q = threadIdx.x; q < gwords / 2; q += 32 * WPB) dst[q] = __ldg(src + q);
            cur_op = op_t;
            __syncthreads();
        }
        for (int i = 0; i < TR; ++i) {
            const int64_t row = row0 + (int64_t)i * WPB + w;
            if (row >= a.rows) break;
            {   // the row this warp handles next, into L2
                const int64_t nxt = i + 1 < TR ? row + WPB : row + (int64_t)gridDim.x * tile_rows - (int64_t)(TR - 1) * WPB;
                if (nxt < a.rows) {
                    const char *p = reinterpret_cast<const char *>(a.B + nxt * a.ldB);
                    for (int o = lane * 128; o < nK * 8; o += 32 * 128)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(p + o));
                }
            }
            const int op = a.row_op ? a.row_op[row] : a.op;
            const double *coef = a.coef + (int64_t)op * a.levels_p1 * kCoefStride;
            {   // b' = b / c0 of the finest level: all the lane's loads in flight at once
                const double inv = coef[K * kCoefStride + kInv];
                const double *Bg = a.B + row * a.ldB;
                double v[C];
#pragma unroll
                for (int k = 0; k < C; ++k) {
                    const int j = lane + 32 * k;
                    v[k] = j < nK ? __ldcs(Bg + j) : 0.0;
                }
#pragma unroll
                for (int k = 0; k < C; ++k) s[RL<K>::point(lane + 32 * k)] = v[k] * inv;
                __syncwarp();
            }
            double x[C];
#pragma unroll
            for (int k = 0; k < C; ++k) x[k] = 0.0;
            if (op == cur_op) {
                for (int cyc = 0; cyc < a.ncyc; ++cyc) vcycle<K, true, true>(x, s, coef, Gs, lane, cyc == 0);
            } else {
                const double *G = a.cmat_rr + (int64_t)op * gwords;
                for (int cyc = 0; cyc < a.ncyc; ++cyc) vcycle<K, true, false>(x, s, coef, G, lane, cyc == 0);
            }
            __syncwarp();
            store_b<K>(s, lane, x);                       // the row through the same slots
            __syncwarp();
            double *Xg = a.X + row * a.ldX;
#pragma unroll 8
            for (int j = lane; j < nK; j += 32) __stcs(Xg + j, s[RL<K>::point(j)]);
            __syncwarp();                                 // the slots are rewritten by the next row
        }
    }
}

template <int K, int MINB>
static cudaError_t launch_rr(const Mg1dArgs &a, cudaStream_t st)
{
    constexpr int WPB = 4;
    constexpr int words = rr::RL<K>::off + rr::RL<K>::size;
    const size_t smem = (size_t)WPB * words * sizeof(double);
    auto k = mg1d_rr<K, WPB, MINB>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t grid = (a.rows + WPB - 1) / WPB;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
    k<<<(unsigned)grid, 32 * WPB, smem, st>>>(a);
    return cudaGetLastError();
}

template <int K>
static cudaError_t launch_rrp(const Mg1dArgs &a, cudaStream_t st)
{
    constexpr int WPB = 12;
    constexpr int words = rr::RL<K>::off + rr::RL<K>::size;
    const size_t smem = ((size_t)kRrCutLd * kRrCutLd + (size_t)WPB * words) * sizeof(double);
    auto k = mg1d_rrp<K, WPB>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // rows per warp and tile: at least ~16 tiles per SM (strided tiles, <= 6 % imbalance)
    const int64_t per = a.rows / (148LL * WPB * 16);
    const int TR = per < 1 ? 1 : (per > 8 ? 8 : (int)per);
    const int64_t ntiles = (a.rows + (int64_t)WPB * TR - 1) / ((int64_t)WPB * TR);
    const int64_t grid = ntiles < 148 ? ntiles : 148;
    k<<<(unsigned)grid, 32 * WPB, smem, st>>>(a, TR);
    return cudaGetLastError();
}

cudaError_t mg1d_rr_launch(const Mg1dArgs &a, cudaStream_t st)
{
    if (a.rows <= 0) return cudaSuccess;
    // rr_minb = 1 (default): the persistent kernel, 12 warps/SM, the cut-level
    // operator in shared memory.  3: mg1d_rr, 12 warps/SM as 3 CTAs (A/B);
    // 2: mg1d_rr at 8 warps/SM and <= 255 registers (A/B)
    if (a.rr_minb == 1) {
        switch (a.K) {
        case 7: return launch_rrp<7>(a, st);
        case 8: return launch_rrp<8>(a, st);
        case 9: return launch_rrp<9>(a, st);
        case 10: return launch_rrp<10>(a, st);
        default: return cudaErrorNotSupported;
        }
    }
    if (a.rr_minb == 2) {
        switch (a.K) {
        case 7: return launch_rr<7, 2>(a, st);
        case 8: return launch_rr<8, 2>(a, st);
        case 9: return launch_rr<9, 2>(a, st);
        case 10: return launch_rr<10, 2>(a, st);
        default: return cudaErrorNotSupported;
        }
    }
    switch (a.K) {
    case 7: return launch_rr<7, 3>(a, st);
    case 8: return launch_rr<8, 3>(a, st);
    case 9: return launch_rr<9, 3>(a, st);
    case 10: return launch_rr<10, 3>(a, st);
    default: return cudaErrorNotSupported;
    }
}

}  // namespace hw
