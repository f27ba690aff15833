// hw_vec.cu -- PCG vector updates and deterministic inner products.
//
// Inner products follow _dot (/root/reference/pkg/src/heatwave/solver.py:
// 111-129): one partial per temporal row, then a FIXED pairwise tree over
// the rows (tree_reduce), so the value does not depend on how rows are
// split between CTAs or GPUs.  Within a row the partial is a fixed-shape
// block reduction (the reference sums left to right; the two differ only
// in rounding).  alpha/beta are formed on the device so the vector updates
// never wait for the host.
#include "hw_common.cuh"
#include "hw_internal.cuh"

namespace hw {

// one CTA per row: partial[r] = sum_i X[r,i] Y[r,i]
template <int BS>
__global__ void __launch_bounds__(BS) row_dots(const double *__restrict__ X,
                                               const double *__restrict__ Y,
                                               double *__restrict__ part, int64_t nx)
{
    __shared__ double red[BS / 32];
    const int64_t r = blockIdx.x;
    const double *x = X + r * nx, *y = Y + r * nx;
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < nx; i += BS) acc = fma(x[i], y[i], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < BS / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) part[r] = v;
    }
}

// tree_reduce (solver.py:111-119) by one CTA: level by level, pairs
// (2i, 2i+1) summed, an odd tail carried over unchanged.  Reads `in`,
// ping-pongs between two halves of `tmp` (>= n + 4 doubles).
__global__ void __launch_bounds__(1024) tree_reduce2(const double *__restrict__ in, int64_t n,
                                                     double *__restrict__ tmp,
                                                     double *__restrict__ out)
{
    const double *src = in;
    double *a = tmp, *b = tmp + (n + 1) / 2 + 1;
    double *dst = a;
    if (n <= 0) {
        if (threadIdx.x == 0) *out = 0.0;
        return;
    }
    while (n > 1) {
        const int64_t half = n / 2, nn = half + (n & 1);
        for (int64_t i = threadIdx.x; i < half; i += blockDim.x) dst[i] = src[2 * i] + src[2 * i + 1];
        if ((n & 1) && threadIdx.x == 0) dst[half] = src[n - 1];
        __syncthreads();
        src = dst;
        dst = (dst == a) ? b : a;
        n = nn;
    }
    if (threadIdx.x == 0) *out = src[0];
}

// PCG scalars: s[0] rho, s[1] pq, s[2] rho_new, s[3] alpha, s[4] beta
__global__ void pcg_alpha(double *s) { s[3] = s[0] / s[1]; }
__global__ void pcg_beta(double *s)
{
    s[4] = s[2] / s[0];
    s[0] = s[2];
}

// w += alpha p (if do_w) ; r -= alpha q (if do_r)  (axpy_rows, _kernels.py:64-68;
// solver.py:223-235)
__global__ void pcg_update_wr(double *__restrict__ w, double *__restrict__ r,
                              const double *__restrict__ p, const double *__restrict__ q,
                              const double *__restrict__ s, int64_t n, int do_w, int do_r)
{
    const double alpha = s[3];
    const double nalpha = -alpha;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (do_w) w[e] = add_rn(w[e], mul_rn(alpha, p[e]));
        if (do_r) r[e] = add_rn(r[e], mul_rn(nalpha, q[e]));
    }
}

// w += alpha p (deferred from the alpha step, if do_w) and p = z + beta p
// (xpay_rows, _kernels.py:71-76) in one pass over p: the same elementwise
// operations as the reference's two separate updates, one read of p saved
__global__ void pcg_update_wp(double *__restrict__ w, double *__restrict__ p,
                              const double *__restrict__ z, const double *__restrict__ s,
                              int64_t n, int do_w)
{
    const double alpha = s[3], beta = s[4];
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const double pe = p[e];
        if (do_w) w[e] = add_rn(w[e], mul_rn(alpha, pe));
        p[e] = add_rn(z[e], mul_rn(beta, pe));
    }
}

// r = f - t (periodic residual recomputation, solver.py:227-229)
__global__ void sub_arrays(const double *__restrict__ f, const double *__restrict__ t,
                           double *__restrict__ r, int64_t n)
{
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x)
        r[e] = f[e] - t[e];
}

// *flag |= any(X != 0)  (the zero-RHS early exit, solver.py:196-198)
__global__ void any_nonzero(const double *__restrict__ X, int64_t n, int *flag)
{
    int f = 0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x)
        f |= (X[e] != 0.0);
    if (__syncthreads_or(f) && threadIdx.x == 0) atomicOr(flag, 1);
}

static unsigned grid_for(int64_t total, int bs)
{
    int64_t g = (total + bs - 1) / bs;
    const int64_t cap = 148LL * 16;
    return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

// result -> *out (device); part/tmp: device scratch of >= rows and rows+4
cudaError_t launch_dot(const double *X, const double *Y, int64_t rows, int64_t nx, double *part,
                       double *tmp, double *out, cudaStream_t st, int64_t *launches)
{
    row_dots<256><<<(unsigned)rows, 256, 0, st>>>(X, Y, part, nx);
    tree_reduce2<<<1, 1024, 0, st>>>(part, rows, tmp, out);
    *launches += 2;
    return cudaGetLastError();
}

cudaError_t launch_row_partials(const double *X, const double *Y, int64_t rows, int64_t nx,
                                double *part, cudaStream_t st)
{
    if (rows <= 0) return cudaSuccess;
    row_dots<256><<<(unsigned)rows, 256, 0, st>>>(X, Y, part, nx);
    return cudaGetLastError();
}

cudaError_t launch_tree(const double *part, int64_t n, double *tmp, double *out, cudaStream_t st)
{
    tree_reduce2<<<1, 1024, 0, st>>>(part, n, tmp, out);
    return cudaGetLastError();
}

// Y += a X (axpy_rows) and Y = X + a Y (xpay_rows) with a host scalar
__global__ void axpy_h(double a, const double *__restrict__ X, double *__restrict__ Y, int64_t n)
{
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x)
        Y[e] = add_rn(Y[e], mul_rn(a, X[e]));
}
__global__ void xpay_h(double a, const double *__restrict__ X, double *__restrict__ Y, int64_t n)
{
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x)
        Y[e] = add_rn(X[e], mul_rn(a, Y[e]));
}

cudaError_t launch_axpy(double a, const double *X, double *Y, int64_t n, cudaStream_t st)
{
    axpy_h<<<grid_for(n, 256), 256, 0, st>>>(a, X, Y, n);
    return cudaGetLastError();
}

cudaError_t launch_xpay(double a, const double *X, double *Y, int64_t n, cudaStream_t st)
{
    xpay_h<<<grid_for(n, 256), 256, 0, st>>>(a, X, Y, n);
    return cudaGetLastError();
}

cudaError_t launch_pcg_alpha(double *s, cudaStream_t st)
{
    pcg_alpha<<<1, 1, 0, st>>>(s);
    return cudaGetLastError();
}

cudaError_t launch_pcg_beta(double *s, cudaStream_t st)
{
    pcg_beta<<<1, 1, 0, st>>>(s);
    return cudaGetLastError();
}

cudaError_t launch_update_wr(double *w, double *r, const double *p, const double *q,
                             const double *s, int64_t n, int do_w, int do_r, cudaStream_t st)
{
    pcg_update_wr<<<grid_for(n, 256), 256, 0, st>>>(w, r, p, q, s, n, do_w, do_r);
    return cudaGetLastError();
}

cudaError_t launch_update_wp(double *w, double *p, const double *z, const double *s, int64_t n,
                             int do_w, cudaStream_t st)
{
    pcg_update_wp<<<grid_for(n, 256), 256, 0, st>>>(w, p, z, s, n, do_w);
    return cudaGetLastError();
}

cudaError_t launch_any_nonzero(const double *X, int64_t n, int *flag, cudaStream_t st)
{
    any_nonzero<<<grid_for(n, 256), 256, 0, st>>>(X, n, flag);
    return cudaGetLastError();
}

cudaError_t launch_sub(const double *f, const double *t, double *r, int64_t n, cudaStream_t st)
{
    sub_arrays<<<grid_for(n, 256), 256, 0, st>>>(f, t, r, n);
    return cudaGetLastError();
}

}  // namespace hw
