// hw_mg1d.cu -- batched V-cycles for alpha*A + mu*M in 1D (tridiagonal).
//
// Restates _mg_core (/root/reference/pkg/src/heatwave/_kernels.py:110-199)
// for d = 1: levels l = 1..K with 2^l - 1 interior points
// (spatial.py:98-103), P from spatial.py:140-173, R = P^T, 1x1 coarse
// inverse.  One warp owns one temporal row and keeps the whole level
// hierarchy in shared memory.  A lexicographic GS sweep over a line is a
// first-order linear recurrence x_j = p_j + beta x_{j-1}; each lane runs it
// over a contiguous chunk and a 5-step warp scan supplies the chunk
// carries (same ordering as the reference, rounding may differ).
#include "hw_common.cuh"
#include "hw_internal.cuh"

namespace hw {

template <int WPB>
__global__ void __launch_bounds__(32 * WPB) mg1d(Mg1dArgs a, int words)
{
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t row = (int64_t)blockIdx.x * WPB + w;
    if (row >= a.rows) return;
    const int K = a.K;
    const int ntot = (1 << (K + 1)) - K - 2;    // sum_{l=1..K} (2^l - 1)
    double *xw = sm + (size_t)w * words;
    double *bw = xw + ntot;
    double *rw = bw + ntot;                       // scratch, 2^K - 1
    const int op = a.row_op ? a.row_op[row] : a.op;
    auto C = [&](int l) { return a.coef + ((int64_t)op * a.levels_p1 + l) * kCoefStride; };
    auto off = [&](int l) { return (1 << l) - l - 1; };   // sum_{k<l} (2^k - 1)

    const int nK = (1 << K) - 1;
    const double *Bg = a.B + row * a.ldB;
    double *Xg = a.X + row * a.ldX;
    for (int k = lane; k < nK; k += 32) {
        bw[off(K) + k] = Bg[k];
        xw[off(K) + k] = 0.0;
    }
    __syncwarp();

    // one GS sweep on level l; forward (lexicographic) or backward
    auto sweep = [&](int l, bool forward) {
        const int n = (1 << l) - 1;
        double *x = xw + off(l);
        const double *b = bw + off(l);
        const double *c = C(l);
        const double oc = c[kCy], inv = c[kInv];
        const double beta = -oc * inv;
        const int ch = (n + 31) >> 5;             // chunk per lane
        const int s0 = lane * ch;
        // phase 1: p_j = (b_j - oc * x_next_old) * inv ; local recurrence
        double y = 0.0;
        for (int k = 0; k < ch; ++k) {
            const int jj = s0 + k;                // position in sweep order
            double p = 0.0;
            if (jj < n) {
                const int j = forward ? jj : n - 1 - jj;
                const int jn = forward ? j + 1 : j - 1;
                double acc = b[j];
                if (jn >= 0 && jn < n) acc -= oc * x[jn];
                p = acc * inv;
            }
            y = fma(beta, y, p);
            if (jj < n) rw[jj] = y;
        }
        // warp scan of chunk ends: T_l = y_l + gamma T_{l-1}, gamma = beta^ch
        double g = 1.0;
        for (int k = 0; k < ch; ++k) g *= beta;
        double T = y, gpow = g;
        for (int o = 1; o < 32; o <<= 1) {
            const double v = __shfl_up_sync(0xffffffffu, T, o);
            if (lane >= o) T = fma(gpow, v, T);
            gpow *= gpow;
        }
        const double prev = __shfl_up_sync(0xffffffffu, T, 1);
        const double carry = lane == 0 ? 0.0 : prev;
        __syncwarp();
        double bp = beta;
        for (int k = 0; k < ch; ++k) {
            const int jj = s0 + k;
            if (jj < n) {
                const int j = forward ? jj : n - 1 - jj;
                x[j] = fma(bp, carry, rw[jj]);
            }
            bp *= beta;
        }
        __syncwarp();
    };

    for (int cyc = 0; cyc < a.ncyc; ++cyc) {
        for (int l = K; l >= 2; --l) {
            const int n = (1 << l) - 1, nc = (1 << (l - 1)) - 1;
            for (int s = 0; s < 3; ++s) sweep(l, true);
            double *x = xw + off(l);
            const double *b = bw + off(l);
            const double *c = C(l);
            for (int j = lane; j < n; j += 32) {          // residual, CSR order
                double acc = b[j];
                if (j > 0) acc -= c[kCy] * x[j - 1];
                acc -= c[kC0] * x[j];
                if (j < n - 1) acc -= c[kCy] * x[j + 1];
                rw[j] = acc;
            }
            __syncwarp();
            double *xc = xw + off(l - 1), *bc = bw + off(l - 1);
            for (int i = lane; i < nc; i += 32) {         // restrict: R = P^T
                double acc = 0.0;
                acc += 0.5 * rw[2 * i];
                acc += 1.0 * rw[2 * i + 1];
                acc += 0.5 * rw[2 * i + 2];
                bc[i] = acc;
                xc[i] = 0.0;
            }
            __syncwarp();
        }
        if (lane == 0) xw[0] = 0.0 + C(1)[kCoarse] * bw[0];
        __syncwarp();
        for (int l = 2; l <= K; ++l) {
            const int n = (1 << l) - 1, nc = (1 << (l - 1)) - 1;
            double *x = xw + off(l);
            const double *xc = xw + off(l - 1);
            for (int j = lane; j < n; j += 32) {          // prolongate
                const int g = j + 1;                      // 1-based fine coordinate
                double acc = 0.0;
                if ((g & 1) == 0) {
                    acc += 1.0 * xc[g / 2 - 1];
                } else {
                    const int lo = (g - 1) / 2, hi = (g + 1) / 2;   // 1-based coarse
                    if (lo >= 1) acc += 0.5 * xc[lo - 1];
                    if (hi <= nc) acc += 0.5 * xc[hi - 1];
                }
                x[j] += acc;
            }
            __syncwarp();
            for (int s = 0; s < 3; ++s) sweep(l, false);
        }
    }
    for (int k = lane; k < nK; k += 32) Xg[k] = xw[off(K) + k];
}

cudaError_t mg1d_launch(const Mg1dArgs &a, cudaStream_t st)
{
    constexpr int WPB = 4;
    const int ntot = (1 << (a.K + 1)) - a.K - 2;
    const int words = 2 * ntot + (1 << a.K);
    const size_t smem = (size_t)WPB * words * sizeof(double);
    auto k = mg1d<WPB>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t grid = (a.rows + WPB - 1) / WPB;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
    k<<<(unsigned)grid, 32 * WPB, smem, st>>>(a, words);
    return cudaGetLastError();
}

}  // namespace hw
