// hw_kron.cu -- Kronecker pieces of S (B, B^T, gamma_0) and of the RHS.
//
// Spatial factors are the finest-level P1 stencils (spatial.py:202-229) on
// the lexicographic interior grid; temporal factors are the tridiagonal
// trial matrices M_t, A_t, L (temporal.py:82-115) and the test matrices
// T, N (temporal.py:118-144) in CSR form.  Every value is accumulated in the
// reference's CSR column order without FMA contraction (csr_rows_matvec
// _kernels.py:25-34, temporal_apply :37-52), so these kernels reproduce the
// reference bit for bit.
//
// Geometry: a CTA of 64 x 4 threads covers 64 consecutive y-points (j) of 4
// grid rows (i) of one temporal row (2D), or 256 points (1D); temporal rows
// run over blockIdx.z with a grid-stride loop.  No integer division per
// element.  Neighbour reads go through the read-only cache (a tile's halo is
// reused by its 7-point stencils).
#include "hw_common.cuh"
#include "hw_internal.cuh"

namespace hw {

constexpr int TX = 64, TY = 4;

struct Pt {          // a grid point of one temporal row
    int i, j;        // 2D: (x index, y index); 1D: (0, index)
    bool ok;
};

__device__ __forceinline__ Pt point_of(const Grid &g)
{
    Pt p;
    if (g.dim == 2) {
        p.j = blockIdx.x * TX + threadIdx.x;
        p.i = blockIdx.y * TY + threadIdx.y;
        p.ok = p.i < g.m && p.j < g.m;
    } else {
        p.i = 0;
        p.j = (blockIdx.x * TY + threadIdx.y) * TX + threadIdx.x;
        p.ok = p.j < g.m;
    }
    return p;
}

// L-shaped domain: the removed closed quadrant is not part of the dof set;
// outputs there are zero (Grid::lm > m for the square, never masked)
__device__ __forceinline__ bool masked_pt(const Pt &p, const Grid &g)
{
    return p.i >= g.lm && p.j >= g.lm;
}

__device__ __forceinline__ int64_t pidx(const Pt &p, const Grid &g)
{
    return g.dim == 2 ? (int64_t)p.i * g.m + p.j : p.j;
}

// ---- point stencils with direct (read-only cached) loads -------------------
// x points at the grid point itself.  The interior path is straight-line
// (all seven couplings present); boundary points skip absent couplings.
// Arithmetic in the reference's CSR column order (csr_rows_matvec).
template <bool DIAG>
__device__ __forceinline__ double stencil2(const double *__restrict__ x, int i, int j, int m,
                                           bool interior, const Stencil &s)
{
    if (interior) {
        double acc;
        if (DIAG) {
            acc = mul_rn(s.cd, __ldg(x - m - 1));
            acc = add_rn(acc, mul_rn(s.cx, __ldg(x - m)));
        } else {
            acc = mul_rn(s.cx, __ldg(x - m));
        }
        acc = add_rn(acc, mul_rn(s.cy, __ldg(x - 1)));
        acc = add_rn(acc, mul_rn(s.c0, __ldg(x)));
        acc = add_rn(acc, mul_rn(s.cy, __ldg(x + 1)));
        acc = add_rn(acc, mul_rn(s.cx, __ldg(x + m)));
        if (DIAG) acc = add_rn(acc, mul_rn(s.cd, __ldg(x + m + 1)));
        return acc;
    }
    double acc = 0.0;
    bool first = true;
    auto add = [&](double v) { acc = first ? v : add_rn(acc, v); first = false; };
    if (DIAG && i > 0 && j > 0) add(mul_rn(s.cd, __ldg(x - m - 1)));
    if (i > 0) add(mul_rn(s.cx, __ldg(x - m)));
    if (j > 0) add(mul_rn(s.cy, __ldg(x - 1)));
    add(mul_rn(s.c0, __ldg(x)));
    if (j < m - 1) add(mul_rn(s.cy, __ldg(x + 1)));
    if (i < m - 1) add(mul_rn(s.cx, __ldg(x + m)));
    if (DIAG && i < m - 1 && j < m - 1) add(mul_rn(s.cd, __ldg(x + m + 1)));
    return acc;
}

__device__ __forceinline__ double stencil1(const double *__restrict__ x, int j, int m,
                                           const Stencil &s)
{
    double acc = mul_rn(s.c0, __ldg(x));
    if (j > 0) acc = add_rn(mul_rn(s.cy, __ldg(x - 1)), acc);
    if (j < m - 1) acc = add_rn(acc, mul_rn(s.cy, __ldg(x + 1)));
    return acc;
}

template <bool DIAG>
__device__ __forceinline__ double stencil_at(const double *__restrict__ x, const Pt &p,
                                             const Grid &g, bool interior, const Stencil &S)
{
    return g.dim == 2 ? stencil2<DIAG>(x, p.i, p.j, g.m, interior, S) : stencil1(x, p.j, g.m, S);
}

static dim3 spatial_grid(const Grid &g, int64_t rows)
{
    const unsigned z = (unsigned)(rows < 65535 ? (rows < 1 ? 1 : rows) : 65535);
    if (g.dim == 2) return dim3((g.m + TX - 1) / TX, (g.m + TY - 1) / TY, z);
    return dim3((g.m + TX * TY - 1) / (TX * TY), 1, z);
}

__device__ __forceinline__ bool interior_of(const Pt &p, const Grid &g)
{
    return p.i > 0 && p.j > 0 && p.i < g.m - 1 && p.j < g.m - 1;
}

// temporal rows per CTA of the row-streaming stencil kernels; the next
// rows' points are prefetched into L2 two rows ahead (these kernels are
// latency-bound on their 7-point loads otherwise)
constexpr int kBtRows = 16;

// YM = M X, YA = A X (either output may be null)
template <bool DM, bool DA>
__global__ void __launch_bounds__(TX * TY) stencil_rows(const double *__restrict__ X,
                                                        double *__restrict__ YM,
                                                        double *__restrict__ YA, Grid g,
                                                        Stencil M, Stencil A, int64_t rows)
{
    const Pt p = point_of(g);
    if (!p.ok) return;
    const int k = (int)pidx(p, g);
    const bool in = interior_of(p, g);
    const bool msk = masked_pt(p, g);
    for (int64_t r0 = (int64_t)blockIdx.z * kBtRows; r0 < rows; r0 += (int64_t)gridDim.z * kBtRows) {
        const int64_t r1 = r0 + kBtRows < rows ? r0 + kBtRows : rows;
        for (int64_t r = r0; r < r1; ++r) {
            const int64_t o = r * g.nx + k;
            if (msk) {
                if (YM) YM[o] = 0.0;
                if (YA) YA[o] = 0.0;
                continue;
            }
            if (r + 2 < r1) asm volatile("prefetch.global.L2 [%0];" ::"l"(X + o + 2 * g.nx));
            if (YM) YM[o] = stencil_at<DM>(X + o, p, g, in, M);
            if (YA) YA[o] = stencil_at<DA>(X + o, p, g, in, A);
        }
    }
}

// out = M G1 + A G2; row 0 additionally += E0 (the trace term Gamma0 (x) M_x)
// -- system.py:134,141-142,145
template <bool DM, bool DA>
__global__ void __launch_bounds__(TX * TY) bt_side(const double *__restrict__ G1,
                                                   const double *__restrict__ G2,
                                                   const double *__restrict__ E0,
                                                   double *__restrict__ out, Grid g, Stencil M,
                                                   Stencil A, int64_t rows)
{
    const Pt p = point_of(g);
    if (!p.ok) return;
    const int k = (int)pidx(p, g);
    const bool in = interior_of(p, g);
    const bool msk = masked_pt(p, g);
    for (int64_t r0 = (int64_t)blockIdx.z * kBtRows; r0 < rows; r0 += (int64_t)gridDim.z * kBtRows) {
        const int64_t r1 = r0 + kBtRows < rows ? r0 + kBtRows : rows;
        for (int64_t r = r0; r < r1; ++r) {
            const int64_t o = r * g.nx + k;
            if (msk) {
                out[o] = 0.0;
                continue;
            }
            if (r + 2 < r1) {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(G1 + o + 2 * g.nx));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(G2 + o + 2 * g.nx));
            }
            double v = add_rn(stencil_at<DM>(G1 + o, p, g, in, M), stencil_at<DA>(G2 + o, p, g, in, A));
            if (r == 0 && E0) v = add_rn(v, E0[k]);
            out[o] = v;
        }
    }
}

// a temporal band row as a dense (lo, mid, hi) triple; absent CSR entries
// are 0 (adding 0 * x leaves the CSR-order sum unchanged up to signed zeros)
__device__ __forceinline__ double band3(const double *__restrict__ tri, int64_t c, double vm,
                                        double v0, double vp)
{
    const double *b = tri + 3 * c;
    double acc = mul_rn(__ldg(b), vm);
    acc = add_rn(acc, mul_rn(__ldg(b + 1), v0));
    return add_rn(acc, mul_rn(__ldg(b + 2), vp));
}

constexpr int kBsidePf = 2;

// B-side, fused: t1 = A_t MxU + L^T AxU, t1' = M_t AxU + L MxU with
// MxU = M_x U, AxU = A_x U computed on the fly (system.py:119-139).  Each
// thread owns one grid point and a chunk of temporal rows and slides a 3-row
// window of (MxU, AxU) in registers, so U is read once and t1, t1' written
// once.  Output rows are the global temporal rows [r0, r0 + nr) (T1/T2
// indexed from r0); U holds global rows [u0, ...) including the halo rows
// the bands touch; nt is the global row count.  E0 (optional) receives
// M_x U[0].
template <bool DM, bool DA>
__global__ void __launch_bounds__(TX * TY) bside_fused(const double *__restrict__ U, int64_t u0,
                                                       double *__restrict__ T1,
                                                       double *__restrict__ T2,
                                                       double *__restrict__ E0, Grid g,
                                                       Stencil M, Stencil A, Tri4 tri,
                                                       int64_t r0, int64_t nr, int64_t nt,
                                                       int chunk)
{
    const Pt p = point_of(g);
    if (!p.ok) return;
    const int k = (int)pidx(p, g);
    const bool in = interior_of(p, g);
    const bool msk = masked_pt(p, g);
    const double *Uk = U + k;
    auto st = [&](int64_t c, double &mv, double &av) {
        if (msk) {                                 // zero rows -> zero bands
            mv = av = 0.0;
            return;
        }
        const double *x = Uk + (c - u0) * g.nx;
        mv = stencil_at<DM>(x, p, g, in, M);
        av = stencil_at<DA>(x, p, g, in, A);
    };
    for (int64_t c0 = r0 + (int64_t)blockIdx.z * chunk; c0 < r0 + nr;
         c0 += (int64_t)gridDim.z * chunk) {
        const int64_t c1 = c0 + chunk < r0 + nr ? c0 + chunk : r0 + nr;
        double mm = 0.0, am = 0.0;                     // row c-1
        if (c0 > 0) st(c0 - 1, mm, am);
        double m0, a0;
        st(c0, m0, a0);
        if (c0 == 0 && E0) E0[k] = m0;
        for (int64_t c = c0; c < c1; ++c) {
            // keep ~kBsidePf rows of U in flight: L2 prefetch of this thread's
            // point kBsidePf rows ahead (the 7-point halo lines come along)
            if (c + kBsidePf < nt && c + kBsidePf < c1 + 1)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(Uk + (c + kBsidePf - u0) * g.nx));
            double mp = 0.0, ap = 0.0;                 // row c+1
            if (c + 1 < nt) st(c + 1, mp, ap);
            const int64_t o = (c - r0) * g.nx + k;
            T1[o] = add_rn(band3(tri.At, c, mm, m0, mp), band3(tri.LT, c, am, a0, ap));
            T2[o] = add_rn(band3(tri.Mt, c, am, a0, ap), band3(tri.L, c, mm, m0, mp));
            mm = m0; am = a0;
            m0 = mp; a0 = ap;
        }
    }
}

// O1 = B1 X1 (+ B2 X2), O2 likewise; any B may be absent (ip null)
__device__ __forceinline__ double tcsr_row(const TCsr &B, int64_t c, const double *__restrict__ X,
                                           int64_t i, int64_t nx)
{
    const int k0 = B.ip[c], k1 = B.ip[c + 1];
    if (k0 == k1) return 0.0;
    double acc = mul_rn(B.v[k0], X[(int64_t)B.ix[k0] * nx + i]);
    for (int k = k0 + 1; k < k1; ++k) acc = add_rn(acc, mul_rn(B.v[k], X[(int64_t)B.ix[k] * nx + i]));
    return acc;
}

// Y[c - r0] = sum_k B[c,k] X[k - x0], c in [r0, r0 + nr)
__global__ void temporal_rows(TCsr B, const double *__restrict__ X, int64_t x0,
                              double *__restrict__ Y, int64_t r0, int64_t nr, int64_t nx)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nx) return;
    for (int64_t rr = blockIdx.y; rr < nr; rr += gridDim.y) {
        const int64_t c = r0 + rr;
        const int k0 = B.ip[c], k1 = B.ip[c + 1];
        double acc = 0.0;
        for (int k = k0; k < k1; ++k) {
            const double v = mul_rn(B.v[k], X[((int64_t)B.ix[k] - x0) * nx + i]);
            acc = (k == k0) ? v : add_rn(acc, v);
        }
        Y[rr * nx + i] = acc;
    }
}

__global__ void temporal_bands(BandOut o1, BandOut o2, int64_t rows, int64_t nx)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nx) return;
    for (int64_t c = blockIdx.y; c < rows; c += gridDim.y) {
        double v = tcsr_row(o1.b1, c, o1.x1, i, nx);
        if (o1.b2.ip) v = add_rn(v, tcsr_row(o1.b2, c, o1.x2, i, nx));
        o1.out[c * nx + i] = v;
        if (o2.out) {
            double w = tcsr_row(o2.b1, c, o2.x1, i, nx);
            if (o2.b2.ip) w = add_rn(w, tcsr_row(o2.b2, c, o2.x2, i, nx));
            o2.out[c * nx + i] = w;
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

// L-shaped domain layouts: dof row (lexicographic, grid row i holds n points
// for i < lm and lm points after) <-> embedded grid row (masked points 0)
__device__ __forceinline__ int64_t dof_offset(int i, const Grid &g)
{
    return i < g.lm ? (int64_t)i * g.m : (int64_t)g.lm * g.m + (int64_t)(i - g.lm) * g.lm;
}

__global__ void grid_scatter(const double *__restrict__ src, double *__restrict__ dst,
                             int64_t rows, Grid g, int64_t nxu)
{
    const Pt p = point_of(g);
    if (!p.ok) return;
    const bool msk = masked_pt(p, g);
    const int64_t k = pidx(p, g), ku = msk ? 0 : dof_offset(p.i, g) + p.j;
    for (int64_t r = blockIdx.z; r < rows; r += gridDim.z)
        dst[r * g.nx + k] = msk ? 0.0 : src[r * nxu + ku];
}

__global__ void grid_gather(const double *__restrict__ src, double *__restrict__ dst,
                            int64_t rows, Grid g, int64_t nxu)
{
    const Pt p = point_of(g);
    if (!p.ok || masked_pt(p, g)) return;
    const int64_t k = pidx(p, g), ku = dof_offset(p.i, g) + p.j;
    for (int64_t r = blockIdx.z; r < rows; r += gridDim.z) dst[r * nxu + ku] = src[r * g.nx + k];
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
    const bool dm = M.cd != 0.0, da = A.cd != 0.0;
    dim3 grid = spatial_grid(g, 1);
    const int64_t zb = (rows + kBtRows - 1) / kBtRows;
    grid.z = (unsigned)(zb < 65535 ? (zb < 1 ? 1 : zb) : 65535);
    const dim3 block(TX, TY);
    if (dm && da) stencil_rows<true, true><<<grid, block, 0, st>>>(X, YM, YA, g, M, A, rows);
    else if (dm) stencil_rows<true, false><<<grid, block, 0, st>>>(X, YM, YA, g, M, A, rows);
    else if (da) stencil_rows<false, true><<<grid, block, 0, st>>>(X, YM, YA, g, M, A, rows);
    else stencil_rows<false, false><<<grid, block, 0, st>>>(X, YM, YA, g, M, A, rows);
    return cudaGetLastError();
}

cudaError_t launch_bt_side(const double *G1, const double *G2, const double *E0, double *out,
                           Grid g, Stencil M, Stencil A, int64_t rows, cudaStream_t st)
{
    const bool dm = M.cd != 0.0, da = A.cd != 0.0;
    dim3 grid = spatial_grid(g, 1);
    const int64_t zb = (rows + kBtRows - 1) / kBtRows;
    grid.z = (unsigned)(zb < 65535 ? (zb < 1 ? 1 : zb) : 65535);
    const dim3 block(TX, TY);
    if (dm && da) bt_side<true, true><<<grid, block, 0, st>>>(G1, G2, E0, out, g, M, A, rows);
    else if (dm) bt_side<true, false><<<grid, block, 0, st>>>(G1, G2, E0, out, g, M, A, rows);
    else if (da) bt_side<false, true><<<grid, block, 0, st>>>(G1, G2, E0, out, g, M, A, rows);
    else bt_side<false, false><<<grid, block, 0, st>>>(G1, G2, E0, out, g, M, A, rows);
    return cudaGetLastError();
}

cudaError_t launch_bside_fused(const double *U, int64_t u0, double *T1, double *T2, double *E0,
                               Grid g, Stencil M, Stencil A, Tri4 tri, int64_t r0, int64_t nr,
                               int64_t nt, cudaStream_t st)
{
    // temporal chunks of 32 rows (2 halo rows of stencils recomputed per chunk)
    dim3 grid = spatial_grid(g, 1);
    const int chunk = 32;
    const int64_t chunks = (nr + chunk - 1) / chunk;
    grid.z = (unsigned)(chunks < 65535 ? (chunks < 1 ? 1 : chunks) : 65535);
    const bool dm = M.cd != 0.0, da = A.cd != 0.0;
    const dim3 block(TX, TY);
    if (dm && da)
        bside_fused<true, true><<<grid, block, 0, st>>>(U, u0, T1, T2, E0, g, M, A, tri, r0, nr, nt, chunk);
    else if (dm)
        bside_fused<true, false><<<grid, block, 0, st>>>(U, u0, T1, T2, E0, g, M, A, tri, r0, nr, nt, chunk);
    else if (da)
        bside_fused<false, true><<<grid, block, 0, st>>>(U, u0, T1, T2, E0, g, M, A, tri, r0, nr, nt, chunk);
    else
        bside_fused<false, false><<<grid, block, 0, st>>>(U, u0, T1, T2, E0, g, M, A, tri, r0, nr, nt, chunk);
    return cudaGetLastError();
}

cudaError_t launch_temporal_bands(BandOut o1, BandOut o2, int64_t rows, int64_t nx,
                                  cudaStream_t st)
{
    dim3 grid((unsigned)((nx + 255) / 256),
              (unsigned)(rows < 65535 ? (rows < 1 ? 1 : rows) : 65535));
    temporal_bands<<<grid, 256, 0, st>>>(o1, o2, rows, nx);
    return cudaGetLastError();
}

cudaError_t launch_temporal_rows(TCsr B, const double *X, int64_t x0, double *Y, int64_t r0,
                                 int64_t nr, int64_t nx, cudaStream_t st)
{
    if (nr <= 0) return cudaSuccess;
    dim3 grid((unsigned)((nx + 255) / 256), (unsigned)(nr < 65535 ? nr : 65535));
    temporal_rows<<<grid, 256, 0, st>>>(B, X, x0, Y, r0, nr, nx);
    return cudaGetLastError();
}

cudaError_t launch_grid_scatter(const double *src, double *dst, int64_t rows, Grid g, int64_t nxu,
                                cudaStream_t st)
{
    if (rows <= 0) return cudaSuccess;
    grid_scatter<<<spatial_grid(g, rows), dim3(TX, TY), 0, st>>>(src, dst, rows, g, nxu);
    return cudaGetLastError();
}

cudaError_t launch_grid_gather(const double *src, double *dst, int64_t rows, Grid g, int64_t nxu,
                               cudaStream_t st)
{
    if (rows <= 0) return cudaSuccess;
    grid_gather<<<spatial_grid(g, rows), dim3(TX, TY), 0, st>>>(src, dst, rows, g, nxu);
    return cudaGetLastError();
}

cudaError_t launch_add(const double *X1, const double *X2, double *Y, int64_t total,
                       cudaStream_t st)
{
    add_arrays<<<grid_for(total, 256), 256, 0, st>>>(X1, X2, Y, total);
    return cudaGetLastError();
}

}  // namespace hw
