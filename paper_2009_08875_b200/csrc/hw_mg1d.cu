// hw_mg1d.cu -- batched V-cycles for alpha*A + mu*M in 1D (tridiagonal).
//
// Restates _mg_core (/root/reference/pkg/src/heatwave/_kernels.py:110-199)
// for d = 1: levels l = 1..K with 2^l - 1 interior points
// (spatial.py:98-103), P from spatial.py:140-173, R = P^T, 1x1 coarse
// inverse.  One warp owns one temporal row.  A lexicographic GS sweep over a
// line is the first-order recurrence x_j = p_j + beta x_{j-1} (forward) or
// x_j = p_j + beta x_{j+1} (backward) with p_j = (b_j - c x_{j+-1}^old)/c0;
// each lane runs it over a contiguous chunk and an exact 5-step warp scan
// supplies the chunk carries (same ordering as the reference, rounding may
// differ).
//
// mg1d_reg<K> (K >= 6): the finest level's x and b live in registers (lane
// owns CF = 2^(K-5) points; the last point of lane 31 is a phantom kept at
// zero), coarser levels in shared memory with compile-time chunk sizes.
// mg1d_smem: every level in shared memory (small K).
#include "hw_common.cuh"
#include "hw_internal.cuh"

namespace hw {

// Shared-memory layout of level l (n_l = 2^l - 1 points, chunk C_l per lane):
// point j is stored at j + j / C_l (one pad after every chunk) so lane
// chunks start at an odd multiple of 8 bytes and a warp's 64-bit accesses
// at chunk stride are bank-conflict free.
template <int L>
struct Lv {
    static constexpr int n = (1 << L) - 1;
    static constexpr int C = L >= 5 ? (1 << (L - 5)) : 1;
    static constexpr int size = C > 1 ? n + n / C + 1 : n;
    static constexpr int off = Lv<L - 1>::off + Lv<L - 1>::size;   // offset in a level stack
    __device__ __forceinline__ static int at(int j) { return C > 1 ? j + j / C : j; }
};
template <>
struct Lv<0> {
    static constexpr int n = 0, C = 1, size = 0, off = 0;
    __device__ __forceinline__ static int at(int j) { return j; }
};

// ---- one GS sweep on a shared-memory level (chunk split for ILP) ----------
template <int L>
__device__ __forceinline__ void sweep_smem(double *x, const double *b, double oc, double inv,
                                           double beta, bool forward, int lane)
{
    constexpr int C = Lv<L>::C, n = Lv<L>::n;
    constexpr int NS = C >= 8 ? 2 : 1;
    constexpr int SC = C / NS;
    double y[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
        const int jj = lane * C + k;
        double p = 0.0;
        if (jj < n) {
            const int j = forward ? jj : n - 1 - jj;
            const int jn = forward ? j + 1 : j - 1;
            const double xn = (jn >= 0 && jn < n) ? x[Lv<L>::at(jn)] : 0.0;
            p = fma(-oc, xn, b[Lv<L>::at(j)]) * inv;
        }
        y[k] = p;
    }
    double e[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) {
        double acc = 0.0;
#pragma unroll
        for (int k = q * SC; k < (q + 1) * SC; ++k) { acc = fma(beta, acc, y[k]); y[k] = acc; }
        e[q] = acc;
    }
    double bsc = beta;
#pragma unroll
    for (int k = 1; k < SC; ++k) bsc *= beta;               // beta^SC
    double T = e[0];
#pragma unroll
    for (int q = 1; q < NS; ++q) T = fma(bsc, T, e[q]);
    double g = bsc;
#pragma unroll
    for (int q = 1; q < NS; ++q) g *= bsc;                  // gamma = beta^C
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double v = __shfl_up_sync(0xffffffffu, T, o);
        if (lane >= o) T = fma(g, v, T);
        g *= g;
    }
    double carry = __shfl_up_sync(0xffffffffu, T, 1);
    if (lane == 0) carry = 0.0;
    __syncwarp();
#pragma unroll
    for (int q = 0; q < NS; ++q) {
        double bp = beta;
#pragma unroll
        for (int k = q * SC; k < (q + 1) * SC; ++k) {
            const int jj = lane * C + k;
            if (jj < n) x[Lv<L>::at(forward ? jj : n - 1 - jj)] = fma(bp, carry, y[k]);
            bp *= beta;
        }
        carry = fma(bsc, carry, e[q]);
    }
    __syncwarp();
}

// r = b - A x on level L; restrict to level L-1 (zeroing its iterate)
// (the three residuals a coarse point needs are evaluated where they are
// used: no r array in shared memory)
template <int L>
__device__ __forceinline__ void residual_restrict(double *xw, double *bw, const double *c, int lane)
{
    constexpr int n = Lv<L>::n, nc = Lv<L - 1>::n;
    const double *x = xw + Lv<L>::off, *b = bw + Lv<L>::off;
    auto res = [&](int j) -> double {
        double acc = b[Lv<L>::at(j)];
        if (j > 0) acc = fma(-c[kCy], x[Lv<L>::at(j - 1)], acc);
        acc = fma(-c[kC0], x[Lv<L>::at(j)], acc);
        if (j < n - 1) acc = fma(-c[kCy], x[Lv<L>::at(j + 1)], acc);
        return acc;
    };
    double *xc = xw + Lv<L - 1>::off, *bc = bw + Lv<L - 1>::off;
    for (int i = lane; i < nc; i += 32)
        bc[Lv<L - 1>::at(i)] = fma(0.5, res(2 * i) + res(2 * i + 2), res(2 * i + 1));
    __syncwarp();
    for (int i = lane; i < nc; i += 32) xc[Lv<L - 1>::at(i)] = 0.0;
    __syncwarp();
}

// x_L += P x_{L-1}
template <int L>
__device__ __forceinline__ void prolongate_smem(double *xw, int lane)
{
    constexpr int n = Lv<L>::n, nc = Lv<L - 1>::n;
    double *x = xw + Lv<L>::off;
    const double *xc = xw + Lv<L - 1>::off;
    for (int j = lane; j < n; j += 32) {
        double v;
        if (j & 1) {
            v = xc[Lv<L - 1>::at((j - 1) / 2)];            // fine j odd sits on coarse (j-1)/2
        } else {
            const int lo = j / 2 - 1, hi = j / 2;          // neighbours (0-based coarse)
            v = 0.5 * ((lo >= 0 ? xc[Lv<L - 1>::at(lo)] : 0.0) +
                       (hi < nc ? xc[Lv<L - 1>::at(hi)] : 0.0));
        }
        x[Lv<L>::at(j)] += v;
    }
    __syncwarp();
}

template <int L>
__device__ __forceinline__ void smooth_level(double *xw, double *bw, const double *coef,
                                             bool forward, int lane)
{
    const double *c = coef + L * kCoefStride;
    const double beta = -c[kCy] * c[kInv];
    for (int s = 0; s < 3; ++s)
        sweep_smem<L>(xw + Lv<L>::off, bw + Lv<L>::off, c[kCy], c[kInv], beta, forward, lane);
}

// pre-smoothing + restriction from level L down, the 1x1 coarse solve, then
// prolongation + post-smoothing back up to L (all in shared memory)
// x_4 = M b_4: the level-4 V-cycle (zero start) as a dense 15 x 15 operator
// staged in shared memory (cm: [i][j], lane j sums over i)
__device__ __forceinline__ void coarse_dense(double *xw, const double *bw, const double *cm, int lane)
{
    constexpr int n = kMg1dCutN;
    const double *b = bw + Lv<kMg1dCut>::off;
    double acc0 = 0.0, acc1 = 0.0;
    if (lane < n) {
#pragma unroll
        for (int i = 0; i < n; i += 2) {
            acc0 = fma(cm[i * n + lane], b[Lv<kMg1dCut>::at(i)], acc0);
            if (i + 1 < n) acc1 = fma(cm[(i + 1) * n + lane], b[Lv<kMg1dCut>::at(i + 1)], acc1);
        }
    }
    __syncwarp();
    if (lane < n) xw[Lv<kMg1dCut>::off + Lv<kMg1dCut>::at(lane)] = acc0 + acc1;
    __syncwarp();
}

template <int L>
__device__ __forceinline__ void down_from(double *xw, double *bw, const double *coef, int lane,
                                          const double *cm = nullptr)
{
    if (L == kMg1dCut && cm) {
        coarse_dense(xw, bw, cm, lane);
        return;
    }
    if constexpr (L >= 2) {
        smooth_level<L>(xw, bw, coef, true, lane);
        residual_restrict<L>(xw, bw, coef + L * kCoefStride, lane);
        down_from<L - 1>(xw, bw, coef, lane, cm);
        prolongate_smem<L>(xw, lane);
        smooth_level<L>(xw, bw, coef, false, lane);
    } else {
        if (lane == 0) xw[0] = 0.0 + coef[1 * kCoefStride + kCoarse] * bw[0];
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// all levels in shared memory (K <= 5, or as a fallback)
// ---------------------------------------------------------------------------
template <int K, int WPB>
__global__ void __launch_bounds__(32 * WPB) mg1d_smem(Mg1dArgs a, int words)
{
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t row = (int64_t)blockIdx.x * WPB + w;
    if (row >= a.rows) return;
    constexpr int ntot = Lv<K>::off + Lv<K>::size;
    double *xw = sm + (size_t)w * words;
    double *bw = xw + ntot;
    const int op = a.row_op ? a.row_op[row] : a.op;
    const double *coef = a.coef + (int64_t)op * a.levels_p1 * kCoefStride;
    constexpr int nK = Lv<K>::n;
    const double *Bg = a.B + row * a.ldB;
    double *Xg = a.X + row * a.ldX;
    for (int k = lane; k < nK; k += 32) {
        bw[Lv<K>::off + Lv<K>::at(k)] = Bg[k];
        xw[Lv<K>::off + Lv<K>::at(k)] = 0.0;
    }
    __syncwarp();
    for (int cyc = 0; cyc < a.ncyc; ++cyc) down_from<K>(xw, bw, coef, lane);
    for (int k = lane; k < nK; k += 32) Xg[k] = xw[Lv<K>::off + Lv<K>::at(k)];
}

// ---------------------------------------------------------------------------
// finest level in registers (K >= 6)
// ---------------------------------------------------------------------------
template <int K, int WPB>
__global__ void __launch_bounds__(32 * WPB, 1) mg1d_reg(Mg1dArgs a, int words)
{
    constexpr int CF = 1 << (K - 5);                    // points per lane, finest level
    constexpr int NC = CF / 2;                          // coarse points per lane (level K-1)
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t row = (int64_t)blockIdx.x * WPB + w;
    if (row >= a.rows) return;
    constexpr int ntot = Lv<K - 1>::off + Lv<K - 1>::size;   // levels 1..K-1
    double *xw = sm + (size_t)w * words;
    double *bw = xw + ntot;
    double *cm = a.cmat ? bw + ntot : nullptr;                // this row's dense coarse operator
    const int op = a.row_op ? a.row_op[row] : a.op;
    const double *coef = a.coef + (int64_t)op * a.levels_p1 * kCoefStride;
    if (cm) {
        const double *g = a.cmat + (int64_t)op * kMg1dCutN * kMg1dCutN;
        for (int e = lane; e < kMg1dCutN * kMg1dCutN; e += 32) cm[e] = g[e];
    }
    const double *cK = coef + K * kCoefStride;
    const double c0 = cK[kC0], oc = cK[kCy], inv = cK[kInv];
    const double beta = -oc * inv;
    const bool tail = lane == 31;                       // owns the phantom point 32 CF - 1
    const int nK = (1 << K) - 1;
    const int ncK = (1 << (K - 1)) - 1;

    // the row's b: coalesced loads staged through the (not yet used) level
    // storage with one pad per 32 points (a lane's chunk reads are then
    // bank-conflict free), instead of CF strided loads per lane
    static_assert(2 * ntot >= 32 * CF + CF, "staging fits in the coarse-level storage");
    // warm L2 with the row the next CTA wave will load (a cold row load at
    // kernel start is otherwise ~10 % of this kernel's stall samples)
    {
        const int64_t ahead = row + 148LL * WPB;        // one CTA per SM: a wave later
        if (ahead < a.rows) {
            const char *p = reinterpret_cast<const char *>(a.B + ahead * a.ldB);
            for (int o = lane * 128; o < nK * 8; o += 32 * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(p + o));
        }
    }
    double x[CF], b[CF];
    {
        const double *Bg = a.B + row * a.ldB;
        for (int j = lane; j < nK; j += 32) xw[j + j / CF] = Bg[j];
        __syncwarp();
#pragma unroll
        for (int k = 0; k < CF; ++k) {
            const int j = lane * CF + k;
            b[k] = (j < nK) ? xw[j + j / CF] : 0.0;
            x[k] = 0.0;
        }
        __syncwarp();
    }
    double gam = beta;                                  // beta^CF
#pragma unroll
    for (int k = 1; k < CF; ++k) gam *= beta;

    constexpr int NS = CF >= 16 ? 4 : (CF >= 4 ? 2 : 1);
    constexpr int SC = CF / NS;
    double bsc = beta;                                  // beta^SC
#pragma unroll
    for (int k = 1; k < SC; ++k) bsc *= beta;
    // GS sweep on the register-resident finest level, in three passes over
    // the lane's chunk: (1) p_k = (b_k - c x_k+-1^old) / c0 in place (the
    // neighbour is read before it is overwritten; no separate p array), (2) the
    // zero-carry chunk end from NS independent sub-chunk recurrences, (3)
    // after the lane carries (exact warp scan) the recurrence x_k = p_k +
    // beta x_k-+1 again from each sub-chunk's true carry-in.
    auto sweep = [&](bool forward) {
        double e[NS];                                   // sub-chunk end values (zero carry-in)
        if (forward) {
            const double xr = __shfl_down_sync(0xffffffffu, x[0], 1);    // next lane, old
#pragma unroll
            for (int k = 0; k < CF; ++k) {
                const double xn = (k + 1 < CF) ? x[k + 1] : (tail ? 0.0 : xr);
                x[k] = fma(-oc, xn, b[k]) * inv;
            }
#pragma unroll
            for (int q = 0; q < NS; ++q) {
                double y = 0.0;
#pragma unroll
                for (int k = q * SC; k < (q + 1) * SC; ++k) y = fma(beta, y, x[k]);
                e[q] = y;
            }
        } else {
            const double xl = __shfl_up_sync(0xffffffffu, x[CF - 1], 1);  // previous lane, old
#pragma unroll
            for (int k = CF - 1; k >= 0; --k) {
                const double xn = (k > 0) ? x[k - 1] : (lane == 0 ? 0.0 : xl);
                x[k] = fma(-oc, xn, b[k]) * inv;
            }
            if (tail) x[CF - 1] = 0.0;                  // phantom: x stays 0
#pragma unroll
            for (int q = 0; q < NS; ++q) {              // sub-chunk q = points CF-1-q*SC downwards
                double y = 0.0;
#pragma unroll
                for (int k = CF - 1 - q * SC; k > CF - 1 - (q + 1) * SC; --k) y = fma(beta, y, x[k]);
                e[q] = y;
            }
        }
        // lane end value with zero carry-in
        double T = e[0];
#pragma unroll
        for (int q = 1; q < NS; ++q) T = fma(bsc, T, e[q]);
        // chunk carries: exact scan over lanes (upward forward, downward backward)
        double g = gam;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double v = forward ? __shfl_up_sync(0xffffffffu, T, o)
                                     : __shfl_down_sync(0xffffffffu, T, o);
            if (forward ? lane >= o : lane + o < 32) T = fma(g, v, T);
            g *= g;
        }
        double carry = forward ? __shfl_up_sync(0xffffffffu, T, 1) : __shfl_down_sync(0xffffffffu, T, 1);
        if (forward ? lane == 0 : lane == 31) carry = 0.0;
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            double y = carry;
            if (forward) {
#pragma unroll
                for (int k = q * SC; k < (q + 1) * SC; ++k) { y = fma(beta, y, x[k]); x[k] = y; }
            } else {
#pragma unroll
                for (int k = CF - 1 - q * SC; k > CF - 1 - (q + 1) * SC; --k) {
                    y = fma(beta, y, x[k]);
                    x[k] = y;
                }
            }
            carry = fma(bsc, carry, e[q]);              // carry into sub-chunk q+1
        }
        if (tail) x[CF - 1] = 0.0;
    };

    for (int cyc = 0; cyc < a.ncyc; ++cyc) {
        for (int s = 0; s < 3; ++s) sweep(true);
        // residual r = b - A x on the fly, restricted into level K-1
        {
            const double xl = __shfl_up_sync(0xffffffffu, x[CF - 1], 1);
            const double xr = __shfl_down_sync(0xffffffffu, x[0], 1);
            auto res = [&](int k) -> double {
                const double a0 = (k > 0) ? x[k - 1] : (lane == 0 ? 0.0 : xl);
                const double a2 = (k + 1 < CF) ? x[k + 1] : (tail ? 0.0 : xr);
                return b[k] - fma(oc, a0, fma(c0, x[k], oc * a2));
            };
            double prev = res(0);
            const double rnext = __shfl_down_sync(0xffffffffu, prev, 1);
            double *bc = bw + Lv<K - 1>::off, *xc = xw + Lv<K - 1>::off;
#pragma unroll
            for (int q = 0; q < NC; ++q) {
                const int i = lane * NC + q;               // coarse index
                const double r1 = res(2 * q + 1);
                const double r2 = (2 * q + 2 < CF) ? res(2 * q + 2) : rnext;
                if (i < ncK) {
                    bc[Lv<K - 1>::at(i)] = fma(0.5, prev + r2, r1);
                    xc[Lv<K - 1>::at(i)] = 0.0;
                }
                prev = r2;
            }
            __syncwarp();
        }
        down_from<K - 1>(xw, bw, coef, lane, cm);
        // prolongate into the registers: fine j = lane CF + k
        {
            const double *xc = xw + Lv<K - 1>::off;
#pragma unroll
            for (int k = 0; k < CF; ++k) {
                const int j = lane * CF + k;
                double v;
                if (j & 1) {
                    v = (j < nK) ? xc[Lv<K - 1>::at((j - 1) / 2)] : 0.0;
                } else {
                    const int lo = j / 2 - 1, hi = j / 2;
                    v = 0.5 * ((lo >= 0 ? xc[Lv<K - 1>::at(lo)] : 0.0) +
                               (hi < ncK ? xc[Lv<K - 1>::at(hi)] : 0.0));
                }
                x[k] += v;
            }
            if (tail) x[CF - 1] = 0.0;
            __syncwarp();
        }
        for (int s = 0; s < 3; ++s) sweep(false);
    }
    // coalesced store through the same staging layout
    __syncwarp();
#pragma unroll
    for (int k = 0; k < CF; ++k) xw[lane * CF + k + lane] = x[k];     // j + j / CF, j = lane CF + k
    __syncwarp();
    double *Xg = a.X + row * a.ldX;
    for (int j = lane; j < nK; j += 32) Xg[j] = xw[j + j / CF];
}

template <int K, int WPB = 8>
static cudaError_t launch_reg(const Mg1dArgs &a, cudaStream_t st)
{
    const int ntot = Lv<K - 1>::off + Lv<K - 1>::size;
    const int words = 2 * ntot + 1 + (a.cmat ? kMg1dCutN * kMg1dCutN : 0);
    const size_t smem = (size_t)WPB * words * sizeof(double);
    auto k = mg1d_reg<K, WPB>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t grid = (a.rows + WPB - 1) / WPB;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
    k<<<(unsigned)grid, 32 * WPB, smem, st>>>(a, words);
    return cudaGetLastError();
}

template <int K>
static cudaError_t launch_smem(const Mg1dArgs &a, cudaStream_t st)
{
    constexpr int WPB = 4;
    const int ntot = Lv<K>::off + Lv<K>::size;
    const int words = 2 * ntot + 1;
    const size_t smem = (size_t)WPB * words * sizeof(double);
    auto k = mg1d_smem<K, WPB>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t grid = (a.rows + WPB - 1) / WPB;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
    k<<<(unsigned)grid, 32 * WPB, smem, st>>>(a, words);
    return cudaGetLastError();
}

cudaError_t mg1d_launch(const Mg1dArgs &a, cudaStream_t st)
{
    switch (a.K) {
    case 1: return launch_smem<1>(a, st);
    case 2: return launch_smem<2>(a, st);
    case 3: return launch_smem<3>(a, st);
    case 4: return launch_smem<4>(a, st);
    case 5: return launch_smem<5>(a, st);
    case 6: return launch_reg<6>(a, st);
    case 7: return launch_reg<7>(a, st);
    case 8: return launch_reg<8>(a, st);
    case 9: return launch_reg<9>(a, st);
    case 10: return launch_reg<10>(a, st);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace hw
