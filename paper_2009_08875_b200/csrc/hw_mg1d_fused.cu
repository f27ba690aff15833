// hw_mg1d_fused.cu -- batched 1D V-cycles (K = 6..10), three Gauss-Seidel
// sweeps per pass fused into ONE carry scan.
//
// Same operator as hw_mg1d.cu (the reference's _mg_core,
// /root/reference/pkg/src/heatwave/_kernels.py:110-199, d = 1): per V-cycle
// and level 3 forward lexicographic GS sweeps, residual, restriction R = P^T,
// ..., the 1x1 coarse solve, prolongation, 3 backward sweeps.  One CTA of up
// to 128 threads owns one temporal row; every level lives in shared memory.
//
// A forward sweep over a line is x_j = bi_j + beta (x_{j-1}^new + x_{j+1}^old)
// (bi = b / c0, beta = -c_y / c0).  Thread t owns CF consecutive points and
// runs each sweep from a zero carry; the true values are affine in the three
// sweeps' carries c1, c2, c3 (the new values just before the chunk):
//   x1_k = y1_k + beta^(k+1) c1
//   x2_k = y2_k + (k+1) beta^(k+3) c1 + beta^(k+1) c2
//   x3_k = y3_k + beta^(k+1) (c3 + (k+1) beta^2 c2 + (k+1)(k+4)/2 beta^4 c1)
// (sweep s+1 reads sweep s's new value right of the point, whose carry part
// has the same beta; summing the geometric series gives the polynomials).
// The chunk-end values therefore obey C(t) = A C(t-1) + E(t-1) with the
// constant lower-triangular Toeplitz A = g (I + u S + v S^2), g = beta^CF,
// u = CF beta^2, v = CF (CF+3)/2 beta^4, whose powers have the closed form
// A^m = g^m (I + m u S + (m v + m(m-1)/2 u^2) S^2).  One Kogge-Stone scan of
// 3-vectors (warp shuffles, then the warp totals across the CTA) replaces
// the three sequential carry scans of hw_mg1d.cu, and the three sweeps'
// zero-carry recurrences are independent chains.  Exact algebra: the
// lexicographic GS iterates up to rounding.
//
// Layout F: thread t owns points j = t CF + k - 1 (k = 0..CF-1), so the extra
// slot (2^l points for 2^l - 1 unknowns) is the phantom j = -1.  Forward
// sweeps meet it first (its update is forced to zero: exact); backward sweeps
// meet it last.  The far boundary of a sweep (j = n forward, j = -1
// backward) breaks the uniform carry polynomials for the last two points in
// sweep order only; the last thread recomputes those three values (x2 of the
// last point, x3 of the last two) sequentially from exact neighbours.
// CF >= 4 on every level, so all of that stays inside one thread.
#include "hw_common.cuh"
#include "hw_internal.cuh"

namespace hw {
namespace {

constexpr int kPad = 2;            // doubles after each thread chunk: conflict-free LDS.128

template <int L>
struct Lv1 {
    static constexpr int NP = 1 << L;                               // slots incl. phantom
    static constexpr int CF = L == 1 ? 2 : ((NP / 128) > 4 ? NP / 128 : 4);
    static constexpr int A = NP / CF;                               // threads on this level
    static constexpr int S = CF + kPad;                             // chunk stride
    static constexpr int n = NP - 1;
    static constexpr int size = A * S;
    static constexpr int off = Lv1<L - 1>::off + Lv1<L - 1>::size;
    static HW_DEV int at(int j)                                      // j in [-1, n)
    {
        const int q = j + 1;
        return (q / CF) * S + (q % CF);
    }
};
template <>
struct Lv1<0> {
    static constexpr int off = 0, size = 0;
};

template <int K>
struct Fused {
    static constexpr int NT = Lv1<K>::A > 32 ? Lv1<K>::A : 32;
    static constexpr int total = Lv1<K>::off + Lv1<K>::size;         // per array (x or bi)
    static constexpr int words = 2 * total + 16;                     // + cross-warp totals
};

// A^m v for the Toeplitz A = g (I + u S + v S^2)
struct Tz {
    double g, u, w;          // g^m, m u, m v + m(m-1)/2 u^2
};
HW_DEV Tz tz_pow(double g1, double u1, double v1, int m)
{
    double gm = 1.0, gb = g1;
#pragma unroll
    for (int b = 0; b < 7; ++b) {
        if (m & (1 << b)) gm *= gb;
        gb *= gb;
    }
    const double md = (double)m;
    return Tz{gm, md * u1, fma(md * (md - 1.0) * 0.5, u1 * u1, md * v1)};
}
HW_DEV void tz_apply_add(const Tz &t, double v1, double v2, double v3, double &s1, double &s2,
                         double &s3)
{
    s3 = fma(t.g, fma(t.w, v1, fma(t.u, v2, v3)), s3);
    s2 = fma(t.g, fma(t.u, v1, v2), s2);
    s1 = fma(t.g, v1, s1);
}

// Three fused GS sweeps on level L (forward: pre-smoothing, ZS: the iterate
// starts at zero; backward: post-smoothing).  Ends with the chunk written
// back; the caller synchronises before anyone reads the level.
template <int L, bool FWD, bool ZS>
__device__ __noinline__ void triple(double *xs, const double *bs, double beta, double *tot, int tid)
{
    using V = Lv1<L>;
    constexpr int CF = V::CF, A = V::A, S = V::S;
    constexpr int AW = A < 32 ? A : 32;                  // threads per (active) warp
    constexpr int NWA = (A + 31) / 32;                   // active warps
    double *x = xs + V::off;
    const double *b = bs + V::off;
    const bool act = tid < A;
    const int lane = tid & 31, warp = tid >> 5;
    const bool lastr = FWD ? tid == A - 1 : tid == 0;    // last in sweep order
    const bool phf = FWD && tid == 0;                    // forward phantom: first point

    // ---- local zero-carry recurrences (order index o; k = FWD ? o : CF-1-o) ----
    double bo[CF + 2], xo[CF + 3];
    double y1[CF], y2[CF], y3[CF];
    if (act) {
        const double *bt = b + tid * S;
#pragma unroll
        for (int h = 0; h < CF / 2; ++h) {
            const double2 w = *reinterpret_cast<const double2 *>(bt + 2 * h);
            bo[FWD ? 2 * h : CF - 1 - 2 * h] = w.x;
            bo[FWD ? 2 * h + 1 : CF - 2 - 2 * h] = w.y;
        }
        if constexpr (!ZS) {
            const double *xt = x + tid * S;
#pragma unroll
            for (int h = 0; h < CF / 2; ++h) {
                const double2 w = *reinterpret_cast<const double2 *>(xt + 2 * h);
                xo[FWD ? 2 * h : CF - 1 - 2 * h] = w.x;
                xo[FWD ? 2 * h + 1 : CF - 2 - 2 * h] = w.y;
            }
        }
        // the next thread in sweep order: its first two right-hand sides and
        // first three old values (zero past the far boundary; fixed up below)
        if (!lastr) {
            const int tn = FWD ? tid + 1 : tid - 1;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const int k = FWD ? q : CF - 1 - q;
                if (q < 2) bo[CF + q] = b[tn * S + k];
                xo[CF + q] = ZS ? 0.0 : x[tn * S + k];
            }
        } else {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                if (q < 2) bo[CF + q] = 0.0;
                xo[CF + q] = 0.0;
            }
        }
        if constexpr (ZS) {
#pragma unroll
            for (int o = 0; o < CF; ++o) xo[o] = 0.0;
        }
        double acc = 0.0;
#pragma unroll
        for (int o = 0; o < CF; ++o) {                   // sweep 1
            const double p = (o == 0 && phf) ? 0.0 : fma(beta, xo[o + 1], bo[o]);
            acc = fma(beta, acc, p);
            y1[o] = acc;
        }
        const double y1n0 = fma(beta, xo[CF + 1], bo[CF]);
        const double y1n1 = fma(beta, y1n0, fma(beta, xo[CF + 2], bo[CF + 1]));
        const double Y1e = fma(beta, y1[CF - 1], y1n0);  // known part of x1 right of the chunk
        acc = 0.0;
#pragma unroll
        for (int o = 0; o < CF; ++o) {                   // sweep 2
            const double r = o + 1 < CF ? y1[o + 1] : Y1e;
            const double p = (o == 0 && phf) ? 0.0 : fma(beta, r, bo[o]);
            acc = fma(beta, acc, p);
            y2[o] = acc;
        }
        const double b3 = beta * beta * beta;
        const double Y2e = fma(beta, y2[CF - 1], fma(b3, y1[CF - 1], fma(beta, y1n1, bo[CF])));
        acc = 0.0;
#pragma unroll
        for (int o = 0; o < CF; ++o) {                   // sweep 3
            const double r = o + 1 < CF ? y2[o + 1] : Y2e;
            const double p = (o == 0 && phf) ? 0.0 : fma(beta, r, bo[o]);
            acc = fma(beta, acc, p);
            y3[o] = acc;
        }
    }

    // ---- carries: inclusive scan of the chunk ends in sweep order ----
    double g1 = beta;
#pragma unroll
    for (int k = 1; k < CF; ++k) g1 *= beta;            // beta^CF
    const double bt2 = beta * beta;
    const double u1 = CF * bt2;
    const double v1 = (CF * (CF + 3) / 2) * (bt2 * bt2);
    double s1 = act ? y1[CF - 1] : 0.0, s2 = act ? y2[CF - 1] : 0.0, s3 = act ? y3[CF - 1] : 0.0;
    const int rw = FWD ? lane : AW - 1 - lane;           // rank inside the warp
#pragma unroll
    for (int m = 1; m < AW; m <<= 1) {
        const double v1s = FWD ? __shfl_up_sync(0xffffffffu, s1, m) : __shfl_down_sync(0xffffffffu, s1, m);
        const double v2s = FWD ? __shfl_up_sync(0xffffffffu, s2, m) : __shfl_down_sync(0xffffffffu, s2, m);
        const double v3s = FWD ? __shfl_up_sync(0xffffffffu, s3, m) : __shfl_down_sync(0xffffffffu, s3, m);
        if (rw >= m && act) {
            const Tz t = tz_pow(g1, u1, v1, m);
            tz_apply_add(t, v1s, v2s, v3s, s1, s2, s3);
        }
    }
    // exclusive: the inclusive value one rank earlier in the warp
    double c1 = FWD ? __shfl_up_sync(0xffffffffu, s1, 1) : __shfl_down_sync(0xffffffffu, s1, 1);
    double c2 = FWD ? __shfl_up_sync(0xffffffffu, s2, 1) : __shfl_down_sync(0xffffffffu, s2, 1);
    double c3 = FWD ? __shfl_up_sync(0xffffffffu, s3, 1) : __shfl_down_sync(0xffffffffu, s3, 1);
    if (rw == 0) c1 = c2 = c3 = 0.0;
    if constexpr (NWA > 1) {
        // warp totals (at the warp's last rank) across the CTA, in sweep order
        if (act && rw == AW - 1) {
            tot[3 * warp] = s1;
            tot[3 * warp + 1] = s2;
            tot[3 * warp + 2] = s3;
        }
        __syncthreads();
        if (act) {
            const int wr = FWD ? warp : NWA - 1 - warp;  // warp rank
            const Tz t32 = tz_pow(g1, u1, v1, 32);
            double w1 = 0.0, w2 = 0.0, w3 = 0.0;
            for (int q = 0; q < wr; ++q) {                // warps before this one, in order
                const int wq = FWD ? q : NWA - 1 - q;
                double n1 = tot[3 * wq], n2 = tot[3 * wq + 1], n3 = tot[3 * wq + 2];
                tz_apply_add(t32, w1, w2, w3, n1, n2, n3);
                w1 = n1;
                w2 = n2;
                w3 = n3;
            }
            const Tz tr = tz_pow(g1, u1, v1, rw);
            tz_apply_add(tr, w1, w2, w3, c1, c2, c3);
        }
    } else {
        __syncwarp();
    }

    // ---- true values of sweep 3, far-boundary fix-up, write back ----
    if (act) {
        const double B2c2 = bt2 * c2, B4c1 = bt2 * bt2 * c1;
        double e = beta;
        double x3[CF];
#pragma unroll
        for (int o = 0; o < CF; ++o) {
            const double w = fma((double)((o + 1) * (o + 4) / 2), B4c1, fma((double)(o + 1), B2c2, c3));
            x3[o] = fma(e, w, y3[o]);
            e *= beta;
        }
        if (lastr) {
            constexpr int oL = FWD ? CF - 1 : CF - 2;    // last real point in sweep order
            double bp = 1.0;                             // beta^oL
#pragma unroll
            for (int k = 0; k < oL; ++k) bp *= beta;
            const double x2e = fma(bp, c2, fma((double)oL * bp * bt2, c1, y2[oL - 1]));  // x2 at oL-1
            const double x2L = fma(beta, x2e, bo[oL]);                                  // x2 at oL
            const double x3a = fma(beta, x3[oL - 2] + x2L, bo[oL - 1]);                 // x3 at oL-1
            x3[oL - 1] = x3a;
            x3[oL] = fma(beta, x3a, bo[oL]);
            if constexpr (!FWD) x3[CF - 1] = 0.0;        // the phantom
        }
        if (phf) x3[0] = 0.0;
        double *xt = x + tid * S;
#pragma unroll
        for (int h = 0; h < CF / 2; ++h) {
            const double lo = FWD ? x3[2 * h] : x3[CF - 1 - 2 * h];
            const double hi = FWD ? x3[2 * h + 1] : x3[CF - 2 - 2 * h];
            *reinterpret_cast<double2 *>(xt + 2 * h) = make_double2(lo, hi);
        }
    }
}

// scaled residual r / c0 = bi + beta (x_{j-1} + x_{j+1}) - x_j on level L,
// restricted (R = P^T) into level L-1's bi: bi_c = (c0_L / c0_{L-1}) P^T (r / c0)
template <int K, int L>
HW_DEV void restrict_level(double *xs, double *bs, double beta, double ratio, int tid)
{
    using F = Lv1<L>;
    using C = Lv1<L - 1>;
    constexpr int NT = Fused<K>::NT;
    const double *x = xs + F::off;
    const double *b = bs + F::off;
    double *bc = bs + C::off;
    auto X = [&](int j) { return j < F::n ? x[F::at(j)] : 0.0; };   // x(-1) = phantom = 0
    for (int i = tid; i < C::n; i += NT) {
        const int j = 2 * i;
        const double xm = X(j - 1), x0 = X(j), x1 = X(j + 1), x2 = X(j + 2), x3 = X(j + 3);
        const double r0 = fma(beta, xm + x1, b[F::at(j)]) - x0;
        const double r1 = fma(beta, x0 + x2, b[F::at(j + 1)]) - x1;
        const double r2 = fma(beta, x1 + x3, b[F::at(j + 2)]) - x2;
        bc[C::at(i)] = ratio * fma(0.5, r0 + r2, r1);
    }
}

// x_L += P x_{L-1}
template <int K, int L>
HW_DEV void prolongate_level(double *xs, int tid)
{
    using F = Lv1<L>;
    using C = Lv1<L - 1>;
    constexpr int NT = Fused<K>::NT;
    double *x = xs + F::off;
    const double *xc = xs + C::off;
    for (int j = tid; j < F::n; j += NT) {
        double v;
        if (j & 1) {
            v = xc[C::at((j - 1) / 2)];
        } else {
            const int lo = j / 2 - 1, hi = j / 2;        // lo = -1: the phantom slot (zero)
            v = 0.5 * (xc[C::at(lo)] + (hi < C::n ? xc[C::at(hi)] : 0.0));
        }
        x[F::at(j)] += v;
    }
}

template <int K, int L>
HW_DEV void vcycle(double *xs, double *bs, double *tot, const double *coef, bool zs_top, int tid)
{
    const double *cl = coef + L * kCoefStride;
    if constexpr (L == 1) {
        if (tid == 0) xs[Lv1<1>::off + Lv1<1>::at(0)] = bs[Lv1<1>::off + Lv1<1>::at(0)];  // x = b / c0
        __syncthreads();
    } else {
        const double beta = -cl[kCy] * cl[kInv];
        if (L < K || zs_top) triple<L, true, true>(xs, bs, beta, tot, tid);
        else triple<L, true, false>(xs, bs, beta, tot, tid);
        __syncthreads();
        const double ratio = cl[kC0] * coef[(L - 1) * kCoefStride + kInv];
        restrict_level<K, L>(xs, bs, beta, ratio, tid);
        __syncthreads();
        vcycle<K, L - 1>(xs, bs, tot, coef, true, tid);
        prolongate_level<K, L>(xs, tid);
        __syncthreads();
        triple<L, false, false>(xs, bs, beta, tot, tid);
        __syncthreads();
    }
}

template <int K>
__global__ void __launch_bounds__(Fused<K>::NT, 3) mg1d_fused(Mg1dArgs a)
{
    extern __shared__ __align__(16) double sm[];
    using T = Lv1<K>;
    constexpr int NT = Fused<K>::NT, tot_words = Fused<K>::total;
    const int tid = threadIdx.x;
    const int64_t row = blockIdx.x;
    double *xs = sm, *bs = sm + tot_words, *tot = bs + tot_words;
    const int op = a.row_op ? a.row_op[row] : a.op;
    const double *coef = a.coef + (int64_t)op * a.levels_p1 * kCoefStride;
    for (int w = tid; w < 2 * tot_words; w += NT) sm[w] = 0.0;   // phantoms and pads stay zero
    __syncthreads();
    const double inv = coef[K * kCoefStride + kInv];
    const double *Bg = a.B + row * a.ldB;
    for (int j = tid; j < T::n; j += NT) bs[T::off + T::at(j)] = Bg[j] * inv;
    __syncthreads();
    for (int cyc = 0; cyc < a.ncyc; ++cyc) vcycle<K, K>(xs, bs, tot, coef, cyc == 0, tid);
    double *Xg = a.X + row * a.ldX;
    for (int j = tid; j < T::n; j += NT) Xg[j] = xs[T::off + T::at(j)];
}

template <int K>
cudaError_t launch_fused(const Mg1dArgs &a, cudaStream_t st)
{
    const size_t smem = Fused<K>::words * sizeof(double);
    auto k = mg1d_fused<K>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (a.rows > 0x7fffffffLL) return cudaErrorInvalidValue;
    k<<<(unsigned)a.rows, Fused<K>::NT, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t mg1d_fused_launch(const Mg1dArgs &a, cudaStream_t st)
{
    if (a.rows <= 0) return cudaSuccess;
    switch (a.K) {
    case 6: return launch_fused<6>(a, st);
    case 7: return launch_fused<7>(a, st);
    case 8: return launch_fused<8>(a, st);
    case 9: return launch_fused<9>(a, st);
    case 10: return launch_fused<10>(a, st);
    default: return cudaErrorNotSupported;
    }
}

}  // namespace hw
