// hw_kron.cu -- Kronecker pieces of S (B, B^T, gamma_0) and of the RHS.
//
// Spatial factors are the finest-level P1 stencils (spatial.py:202-229) on
// the lexicographic interior grid; temporal factors are the tridiagonal
// trial matrices M_t, A_t, L (temporal.py:82-115) and the test matrices
// T, N (temporal.py:118-144).  Every value is accumulated in the
// reference's CSR column order without FMA contraction (csr_rows_matvec
// _kernels.py:25-34, temporal_apply :37-52), so these kernels reproduce the
// reference bit for bit.
#include "hw_common.cuh"
#include "hw_internal.cuh"

namespace hw {



// y = S x at flattened interior index k of one row (CSR column order); the
// diagonal coupling exists in the CSR only where its value is nonzero
__device__ __forceinline__ double stencil_at(const double *__restrict__ x, int64_t k,
                                             const Grid &g, const Stencil &s)
{
    if (g.dim == 1) {
        const int i = (int)k;
        double acc = 0.0;
        bool first = true;
        auto add = [&](double v) { acc = first ? v : add_rn(acc, v); first = false; };
        if (i > 0) add(mul_rn(s.cy, x[k - 1]));
        add(mul_rn(s.c0, x[k]));
        if (i < g.m - 1) add(mul_rn(s.cy, x[k + 1]));
        return acc;
    }
    const int m = g.m;
    const bool HAS_DIAG = s.cd != 0.0;
    const int i = (int)(k / m), j = (int)(k - (int64_t)i * m);
    double acc = 0.0;
    bool first = true;
    auto add = [&](double v) { acc = first ? v : add_rn(acc, v); first = false; };
    if (HAS_DIAG && i > 0 && j > 0) add(mul_rn(s.cd, x[k - m - 1]));
    if (i > 0) add(mul_rn(s.cx, x[k - m]));
    if (j > 0) add(mul_rn(s.cy, x[k - 1]));
    add(mul_rn(s.c0, x[k]));
    if (j < m - 1) add(mul_rn(s.cy, x[k + 1]));
    if (i < m - 1) add(mul_rn(s.cx, x[k + m]));
    if (HAS_DIAG && i < m - 1 && j < m - 1) add(mul_rn(s.cd, x[k + m + 1]));
    return acc;
}

// Y1 = M X, Y2 = A X (either output may be null)
__global__ void stencil_rows(const double *__restrict__ X, double *__restrict__ YM,
                             double *__restrict__ YA, Grid g, Stencil M, Stencil A, int64_t rows)
{
    const int64_t total = rows * g.nx;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / g.nx, k = e - r * g.nx;
        const double *x = X + r * g.nx;
        if (YM) YM[e] = stencil_at(x, k, g, M);
        if (YA) YA[e] = stencil_at(x, k, g, A);
    }
}

// out = M G1 + A G2; row 0 additionally += E0 (the trace term Gamma0 (x) M_x)
// -- system.py:134,141-142,145
__global__ void bt_side(const double *__restrict__ G1, const double *__restrict__ G2,
                        const double *__restrict__ E0, double *__restrict__ out, Grid g,
                        Stencil M, Stencil A, int64_t rows)
{
    const int64_t total = rows * g.nx;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / g.nx, k = e - r * g.nx;
        double v = add_rn(stencil_at(G1 + r * g.nx, k, g, M),
                          stencil_at(G2 + r * g.nx, k, g, A));
        if (r == 0 && E0) v = add_rn(v, E0[k]);
        out[e] = v;
    }
}

// Temporal factor in CSR form (device arrays, <= 4 nnz per row).

__device__ __forceinline__ double tcsr_row(const TCsr &B, int64_t c, const double *__restrict__ X,
                                           int64_t i, int64_t nx)
{
    const int k0 = B.ip[c], k1 = B.ip[c + 1];
    if (k0 == k1) return 0.0;
    double acc = mul_rn(B.v[k0], X[(int64_t)B.ix[k0] * nx + i]);
    for (int k = k0 + 1; k < k1; ++k) acc = add_rn(acc, mul_rn(B.v[k], X[(int64_t)B.ix[k] * nx + i]));
    return acc;
}

// O1 = B1 X1 (+ B2 X2), O2 = B3 X3 (+ B4 X4); any B may be "absent" (ip null)
// -- t1 = A_t MxU + L^T AxU and t1' = M_t AxU + L MxU (system.py:130-139)

__global__ void temporal_bands(BandOut o1, BandOut o2, int64_t rows, int64_t nx)
{
    const int64_t total = rows * nx;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / nx, i = e - c * nx;
        {
            double v = tcsr_row(o1.b1, c, o1.x1, i, nx);
            if (o1.b2.ip) v = add_rn(v, tcsr_row(o1.b2, c, o1.x2, i, nx));
            o1.out[e] = v;
        }
        if (o2.out) {
            double v = tcsr_row(o2.b1, c, o2.x1, i, nx);
            if (o2.b2.ip) v = add_rn(v, tcsr_row(o2.b2, c, o2.x2, i, nx));
            o2.out[e] = v;
        }
    }
}

// Y = X1 + X2 (numpy add), rows*nx elements
__global__ void add_arrays(const double *__restrict__ X1, const double *__restrict__ X2,
                           double *__restrict__ Y, int64_t total)
{
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x)
        Y[e] = add_rn(X1[e], X2[e]);
}

static unsigned grid_for(int64_t total, int bs)
{
    int64_t g = (total + bs - 1) / bs;
    const int64_t cap = 148LL * 16;
    return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

cudaError_t launch_stencil_rows(const double *X, double *YM, double *YA, Grid g, Stencil M,
                                Stencil A, int64_t rows, cudaStream_t st)
{
    stencil_rows<<<grid_for(rows * g.nx, 256), 256, 0, st>>>(X, YM, YA, g, M, A, rows);
    return cudaGetLastError();
}

cudaError_t launch_bt_side(const double *G1, const double *G2, const double *E0, double *out,
                           Grid g, Stencil M, Stencil A, int64_t rows, cudaStream_t st)
{
    bt_side<<<grid_for(rows * g.nx, 256), 256, 0, st>>>(G1, G2, E0, out, g, M, A, rows);
    return cudaGetLastError();
}

cudaError_t launch_temporal_bands(BandOut o1, BandOut o2, int64_t rows, int64_t nx,
                                  cudaStream_t st)
{
    temporal_bands<<<grid_for(rows * nx, 256), 256, 0, st>>>(o1, o2, rows, nx);
    return cudaGetLastError();
}

cudaError_t launch_add(const double *X1, const double *X2, double *Y, int64_t total,
                       cudaStream_t st)
{
    add_arrays<<<grid_for(total, 256), 256, 0, st>>>(X1, X2, Y, total);
    return cudaGetLastError();
}

}  // namespace hw
