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

#include <cstdio>
#include <cstdlib>

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

// ---------------------------------------------------------------------------
// TMA-staged row strips (2D, m >= 511).  The 7-point stencils above read
// every value seven times through L1/TEX (bside ran L1-bound at ~61 % of
// HBM).  Here a CTA of 512 threads owns FY complete grid rows of a chunk of
// temporal rows; one elected thread stages each temporal row's FY + 2 grid
// rows (the strip and its halo rows) into shared memory with 1D bulk copies
// (cp.async.bulk, the TMA engine) of the 16-byte-aligned superset of each
// row, completing on an mbarrier; NS temporal rows are in flight.  Whole
// rows keep the copies large (8 KB at m = 1023: the per-copy cost of small
// tiles made 64 x 4 tiles 2.6-4x slower than direct loads).  Warp
// specialised: a producer warp issues the copies as soon as a slot's
// "empty" mbarrier reports that all 16 consumer warps have read it, so the
// consumers never wait for the issue (a single leader thread issuing after a
// CTA barrier serialised every temporal row).  The stencils read shared
// memory in exactly the order of stencil2 (bit-identical).
// ---------------------------------------------------------------------------
constexpr int kStripT = 512;                  // consumer threads (16 warps)
constexpr int kStripW = kStripT / 32;
constexpr int kStripThreads = kStripT + 32;   // + the producer warp
constexpr size_t kStripSmemMax = 200 * 1024;

__device__ __forceinline__ unsigned sm_u32(const void *p)
{
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(sm_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            sm_u32(dst)),
        "l"(src), "r"(bytes), "r"(sm_u32(bar))
        : "memory");
}

// doubles per staged grid row: the aligned superset of columns 0..m-1 at
// index 2 (+ its lead), so column j of a staged row sits at 2 + lead + j
__host__ __device__ constexpr int strip_w(int m) { return (m + 5) & ~1; }

template <int NIN, int FY>
struct StripPipe {
    double *tiles;                      // [NS][NIN][FY + 2][W]
    uint64_t *full, *empty;             // [NS] each: data landed / slot read by all consumers
    const double *src[NIN];
    const double *beg[NIN], *end[NIN];  // readable extents
    int i0, m, W;

    __device__ __forceinline__ double *row(int slot, int a, int ii) const
    {
        return tiles + ((size_t)(slot * NIN + a) * (FY + 2) + ii) * W;
    }
    // one thread: copies of the temporal row at element offset rowoff into slot
    __device__ __forceinline__ void issue(int slot, int64_t rowoff) const
    {
        unsigned bytes = 0;
        for (int a = 0; a < NIN; ++a) {
            for (int ii = 0; ii < FY + 2; ++ii) {
                const int i = i0 - 1 + ii;
                if (i < 0 || i >= m) continue;
                const double *plo = src[a] + rowoff + (int64_t)i * m;
                const int lead = (int)((reinterpret_cast<uintptr_t>(plo) >> 3) & 1);
                const double *pa = plo - lead;
                double *d = row(slot, a, ii) + 2;
                int cnt = m + lead;
                if (pa < beg[a]) {              // (16-byte aligned allocations never get here)
                    d[1] = *plo;
                    pa += 2;
                    d += 2;
                    cnt -= 2;
                }
                cnt = (cnt + 1) & ~1;
                if (pa + cnt > end[a]) {        // the padding element lies past the array
                    cnt -= 2;
                    d[cnt] = pa[cnt];
                }
                if (cnt > 0) {
                    bulk_g2s(d, pa, (unsigned)cnt * 8u, &full[slot]);
                    bytes += (unsigned)cnt * 8u;
                }
            }
        }
        mbar_arrive_expect_tx(&full[slot], bytes);   // the slot's single arrival
    }
    // producer (one thread): the copies of use u of a slot, once use u - ns
    // has been read by every consumer warp
    __device__ __forceinline__ void produce(int u, int ns, int64_t rowoff) const
    {
        const int slot = u % ns;
        if (u >= ns) mbar_wait(&empty[slot], (unsigned)((u / ns - 1) & 1));
        issue(slot, rowoff);
    }
    // consumer: wait until use u of its slot has landed
    __device__ __forceinline__ int acquire(int u, int ns) const
    {
        const int slot = u % ns;
        mbar_wait(&full[slot], (unsigned)((u / ns) & 1));
        return slot;
    }
    // consumer warp: done reading the slot
    __device__ __forceinline__ void release(int slot) const
    {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[slot]);
    }
    // column 0 of tile row ii as staged for the temporal row at rowoff
    __device__ __forceinline__ const double *col0(int slot, int a, int ii, int64_t rowoff) const
    {
        const int i = i0 - 1 + ii;
        const int ic = i < 0 ? 0 : (i >= m ? m - 1 : i);    // never read when outside the grid
        const double *plo = src[a] + rowoff + (int64_t)ic * m;
        return row(slot, a, ii) + 2 + (int)((reinterpret_cast<uintptr_t>(plo) >> 3) & 1);
    }
    __device__ void setup(double *smem, int ns, const double *const *s, const double *const *b,
                          const double *const *e, int m_)
    {
        m = m_;
        W = strip_w(m_);
        tiles = smem;
        full = reinterpret_cast<uint64_t *>(smem + (size_t)ns * NIN * (FY + 2) * W);
        empty = full + ns;
        for (int a = 0; a < NIN; ++a) {
            src[a] = s[a];
            beg[a] = b[a];
            end[a] = e[a];
        }
        i0 = blockIdx.y * FY;
        if (threadIdx.x == 0) {
            for (int q = 0; q < ns; ++q) {
                mbar_init(&full[q], 1);
                mbar_init(&empty[q], kStripW);
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
};

template <int NIN, int FY>
static size_t strip_stage_bytes(int m)
{
    return (size_t)NIN * (FY + 2) * strip_w(m) * sizeof(double);
}

template <int NIN, int FY>
static int strip_stages(int m)
{
    const size_t st = strip_stage_bytes<NIN, FY>(m);
    const int ns = (int)((kStripSmemMax - 128) / st);
    return ns > 4 ? 4 : ns;
}

// the 2D stencil of stencil2 (same operation order) on staged rows
template <bool DIAG>
__device__ __forceinline__ double stencil_tile(const double *rm, const double *r0, const double *rp,
                                               int j, int i, int m, bool interior, const Stencil &s)
{
    if (interior) {
        double acc;
        if (DIAG) {
            acc = mul_rn(s.cd, rm[j - 1]);
            acc = add_rn(acc, mul_rn(s.cx, rm[j]));
        } else {
            acc = mul_rn(s.cx, rm[j]);
        }
        acc = add_rn(acc, mul_rn(s.cy, r0[j - 1]));
        acc = add_rn(acc, mul_rn(s.c0, r0[j]));
        acc = add_rn(acc, mul_rn(s.cy, r0[j + 1]));
        acc = add_rn(acc, mul_rn(s.cx, rp[j]));
        if (DIAG) acc = add_rn(acc, mul_rn(s.cd, rp[j + 1]));
        return acc;
    }
    double acc = 0.0;
    bool first = true;
    auto add = [&](double v) { acc = first ? v : add_rn(acc, v); first = false; };
    if (DIAG && i > 0 && j > 0) add(mul_rn(s.cd, rm[j - 1]));
    if (i > 0) add(mul_rn(s.cx, rm[j]));
    if (j > 0) add(mul_rn(s.cy, r0[j - 1]));
    add(mul_rn(s.c0, r0[j]));
    if (j < m - 1) add(mul_rn(s.cy, r0[j + 1]));
    if (i < m - 1) add(mul_rn(s.cx, rp[j]));
    if (DIAG && i < m - 1 && j < m - 1) add(mul_rn(s.cd, rp[j + 1]));
    return acc;
}

// a strip point: grid row i0 + r, column tid + kStripT c
struct SPt {
    int i, j;
    bool ok, in, msk;
};
__device__ __forceinline__ SPt strip_pt(int i0, int r, int c, const Grid &g)
{
    SPt p;
    p.i = i0 + r;
    p.j = (int)threadIdx.x + kStripT * c;
    p.ok = p.i < g.m && p.j < g.m;
    p.in = p.i > 0 && p.j > 0 && p.i < g.m - 1 && p.j < g.m - 1;
    p.msk = p.i >= g.lm && p.j >= g.lm;
    return p;
}

// ---- bside_stack: bside_fused with R vertically stacked points per thread --
// A thread owns column j of R consecutive grid rows, so the R 7-point
// stencils of one temporal row share their loads: (R + 2) x 3 values instead
// of 7 R (4.5 instead of 7 per point at R = 4).  The loads stay coalesced
// along j and the arithmetic per point is stencil2's (CSR column order,
// absent couplings skipped): bit-identical.  bside_fused is bound by L1
// wavefronts (rows of odd length: a warp's 256 bytes span three 128-byte
// lines per load) -- fewer loads per point is the lever.  2D only.
template <bool DIAG>
__device__ __forceinline__ double stencil_vals(const double (&a)[3], const double (&b)[3],
                                               const double (&c)[3], int i, int j, int m,
                                               bool interior, const Stencil &s)
{
    // a, b, c: grid rows i-1, i, i+1 at columns j-1, j, j+1
    if (interior) {
        double acc;
        if (DIAG) {
            acc = mul_rn(s.cd, a[0]);
            acc = add_rn(acc, mul_rn(s.cx, a[1]));
        } else {
            acc = mul_rn(s.cx, a[1]);
        }
        acc = add_rn(acc, mul_rn(s.cy, b[0]));
        acc = add_rn(acc, mul_rn(s.c0, b[1]));
        acc = add_rn(acc, mul_rn(s.cy, b[2]));
        acc = add_rn(acc, mul_rn(s.cx, c[1]));
        if (DIAG) acc = add_rn(acc, mul_rn(s.cd, c[2]));
        return acc;
    }
    double acc = 0.0;
    bool first = true;
    auto add = [&](double v) { acc = first ? v : add_rn(acc, v); first = false; };
    if (DIAG && i > 0 && j > 0) add(mul_rn(s.cd, a[0]));
    if (i > 0) add(mul_rn(s.cx, a[1]));
    if (j > 0) add(mul_rn(s.cy, b[0]));
    add(mul_rn(s.c0, b[1]));
    if (j < m - 1) add(mul_rn(s.cy, b[2]));
    if (i < m - 1) add(mul_rn(s.cx, c[1]));
    if (DIAG && i < m - 1 && j < m - 1) add(mul_rn(s.cd, c[2]));
    return acc;
}

template <bool DM, bool DA, int R>
__global__ void __launch_bounds__(TX * TY) bside_stack(const double *__restrict__ U, int64_t u0,
                                                       double *__restrict__ T1,
                                                       double *__restrict__ T2,
                                                       double *__restrict__ E0, Grid g,
                                                       Stencil M, Stencil A, Tri4 tri,
                                                       int64_t r0, int64_t nr, int64_t nt,
                                                       int chunk)
{
    const int m = g.m;
    const int j = blockIdx.x * TX + threadIdx.x;
    const int ib = (blockIdx.y * TY + threadIdx.y) * R;
    if (j >= m || ib >= m) return;
    const int64_t k0 = (int64_t)ib * m + j;              // point (ib, j)
    const double *Uk = U + k0;
    bool in[R], msk[R], ok[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const Pt p{ib + r, j, ib + r < m};
        ok[r] = p.ok;
        in[r] = interior_of(p, g);
        msk[r] = masked_pt(p, g);
    }
    // (M_x U, A_x U) of temporal row c at the R points
    auto st = [&](int64_t c, double (&mv)[R], double (&av)[R]) {
        const double *x = Uk + (c - u0) * g.nx;
        double v[R + 2][3];
#pragma unroll
        for (int rr = 0; rr < R + 2; ++rr) {
            const int i = ib - 1 + rr;
            const bool rowok = i >= 0 && i < m;
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                const int jj = j - 1 + cc;
                // the corners (ib-1, j+1) and (ib+R, j-1) couple to no owned point;
                // (ib-1, j-1) and (ib+R, j+1) only through the diagonal
                const bool need = rr == 0 ? (cc == 1 || (cc == 0 && (DM || DA)))
                                          : (rr == R + 1 ? (cc == 1 || (cc == 2 && (DM || DA))) : true);
                v[rr][cc] = (need && rowok && jj >= 0 && jj < m)
                                ? __ldg(x + (int64_t)(rr - 1) * m + (cc - 1))
                                : 0.0;
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (!ok[r] || msk[r]) {                       // zero rows -> zero bands
                mv[r] = av[r] = 0.0;
                continue;
            }
            mv[r] = stencil_vals<DM>(v[r], v[r + 1], v[r + 2], ib + r, j, m, in[r], M);
            av[r] = stencil_vals<DA>(v[r], v[r + 1], v[r + 2], ib + r, j, m, in[r], A);
        }
    };
    for (int64_t c0 = r0 + (int64_t)blockIdx.z * chunk; c0 < r0 + nr;
         c0 += (int64_t)gridDim.z * chunk) {
        const int64_t c1 = c0 + chunk < r0 + nr ? c0 + chunk : r0 + nr;
        double mm[R], am[R], m0[R], a0[R];
#pragma unroll
        for (int r = 0; r < R; ++r) mm[r] = am[r] = 0.0;  // row c-1
        if (c0 > 0) st(c0 - 1, mm, am);
        st(c0, m0, a0);
        if (c0 == 0 && E0) {
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (ok[r]) E0[k0 + (int64_t)r * m] = m0[r];
        }
        for (int64_t c = c0; c < c1; ++c) {
            if (c + kBsidePf < nt && c + kBsidePf < c1 + 1) {
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (ok[r])
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(Uk + (c + kBsidePf - u0) * g.nx +
                                                                      (int64_t)r * m));
            }
            double mp[R], ap[R];
#pragma unroll
            for (int r = 0; r < R; ++r) mp[r] = ap[r] = 0.0;  // row c+1
            if (c + 1 < nt) st(c + 1, mp, ap);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (!ok[r]) continue;
                const int64_t o = (c - r0) * g.nx + k0 + (int64_t)r * m;
                T1[o] = add_rn(band3(tri.At, c, mm[r], m0[r], mp[r]), band3(tri.LT, c, am[r], a0[r], ap[r]));
                T2[o] = add_rn(band3(tri.Mt, c, am[r], a0[r], ap[r]), band3(tri.L, c, mm[r], m0[r], mp[r]));
                mm[r] = m0[r]; am[r] = a0[r];
                m0[r] = mp[r]; a0[r] = ap[r];
            }
        }
    }
}

// bside_fused on TMA-staged strips: the same sliding window over temporal
// rows (FY x CJ points per consumer thread), stencils from shared memory
template <bool DM, bool DA, int FY, int CJ>
__global__ void __maxnreg__(96) bside_strip(const double *__restrict__ U,
                                                                 int64_t u0, int64_t nu,
                                                                 double *__restrict__ T1,
                                                                 double *__restrict__ T2,
                                                                 double *__restrict__ E0, Grid g,
                                                                 Stencil M, Stencil A, Tri4 tri,
                                                                 int64_t r0, int64_t nr, int64_t nt,
                                                                 int chunk, int ns)
{
    extern __shared__ __align__(16) double smem[];
    StripPipe<1, FY> sp;
    const double *srcs[1] = {U}, *begs[1] = {U}, *ends[1] = {U + nu * g.nx};
    sp.setup(smem, ns, srcs, begs, ends, g.m);
    const bool producer = threadIdx.x >= kStripT;
    int u = 0;                                                   // slot uses so far
    for (int64_t c0 = r0 + (int64_t)blockIdx.z * chunk; c0 < r0 + nr;
         c0 += (int64_t)gridDim.z * chunk) {
        const int64_t c1 = c0 + chunk < r0 + nr ? c0 + chunk : r0 + nr;
        const int64_t qs = c0 > 0 ? c0 - 1 : 0;
        const int64_t qe = c1 < nt - 1 ? c1 : nt - 1;           // inclusive
        const int nq = (int)(qe - qs + 1);
        if (producer) {
            if (threadIdx.x == kStripT)
                for (int qi = 0; qi < nq; ++qi) sp.produce(u + qi, ns, (qs + qi - u0) * g.nx);
            u += nq;
            continue;
        }
        double mm[FY][CJ], am[FY][CJ], m0[FY][CJ], a0[FY][CJ];
#pragma unroll
        for (int r = 0; r < FY; ++r)
#pragma unroll
            for (int c = 0; c < CJ; ++c) mm[r][c] = am[r][c] = m0[r][c] = a0[r][c] = 0.0;
        for (int qi = 0; qi < nq; ++qi, ++u) {
            const int64_t q = qs + qi;
            const int slot = sp.acquire(u, ns);
            double mp[FY][CJ], ap[FY][CJ];
            const int64_t roff = (q - u0) * g.nx;
#pragma unroll
            for (int r = 0; r < FY; ++r) {
                const double *rm = sp.col0(slot, 0, r, roff), *rz = sp.col0(slot, 0, r + 1, roff),
                             *rp = sp.col0(slot, 0, r + 2, roff);
#pragma unroll
                for (int c = 0; c < CJ; ++c) {
                    const SPt p = strip_pt(sp.i0, r, c, g);
                    mp[r][c] = ap[r][c] = 0.0;
                    if (p.ok && !p.msk) {
                        mp[r][c] = stencil_tile<DM>(rm, rz, rp, p.j, p.i, g.m, p.in, M);
                        ap[r][c] = stencil_tile<DA>(rm, rz, rp, p.j, p.i, g.m, p.in, A);
                    }
                }
            }
            sp.release(slot);
            const int64_t cc = q - 1;
            if (cc >= c0) {
                // band rows of cc (loaded once, shared by every point)
                const double *bA = tri.At + 3 * cc, *bT = tri.LT + 3 * cc;
                const double *bM = tri.Mt + 3 * cc, *bL = tri.L + 3 * cc;
                const double A0 = __ldg(bA), A1 = __ldg(bA + 1), A2 = __ldg(bA + 2);
                const double T0_ = __ldg(bT), T1_ = __ldg(bT + 1), T2_ = __ldg(bT + 2);
                const double M0 = __ldg(bM), M1 = __ldg(bM + 1), M2 = __ldg(bM + 2);
                const double L0 = __ldg(bL), L1 = __ldg(bL + 1), L2 = __ldg(bL + 2);
#pragma unroll
                for (int r = 0; r < FY; ++r)
#pragma unroll
                    for (int c = 0; c < CJ; ++c) {
                        const SPt p = strip_pt(sp.i0, r, c, g);
                        if (!p.ok) continue;
                        const int64_t o = (cc - r0) * g.nx + (int64_t)p.i * g.m + p.j;
                        // band3 (lo, mid, hi) order, as in bside_fused
                        const double t1a = add_rn(add_rn(mul_rn(A0, mm[r][c]), mul_rn(A1, m0[r][c])),
                                                  mul_rn(A2, mp[r][c]));
                        const double t1b = add_rn(add_rn(mul_rn(T0_, am[r][c]), mul_rn(T1_, a0[r][c])),
                                                  mul_rn(T2_, ap[r][c]));
                        const double t2a = add_rn(add_rn(mul_rn(M0, am[r][c]), mul_rn(M1, a0[r][c])),
                                                  mul_rn(M2, ap[r][c]));
                        const double t2b = add_rn(add_rn(mul_rn(L0, mm[r][c]), mul_rn(L1, m0[r][c])),
                                                  mul_rn(L2, mp[r][c]));
                        T1[o] = add_rn(t1a, t1b);
                        T2[o] = add_rn(t2a, t2b);
                    }
            }
            if (q == 0 && E0) {
#pragma unroll
                for (int r = 0; r < FY; ++r)
#pragma unroll
                    for (int c = 0; c < CJ; ++c) {
                        const SPt p = strip_pt(sp.i0, r, c, g);
                        if (p.ok) E0[(int64_t)p.i * g.m + p.j] = mp[r][c];
                    }
            }
#pragma unroll
            for (int r = 0; r < FY; ++r)
#pragma unroll
                for (int c = 0; c < CJ; ++c) {
                    mm[r][c] = m0[r][c];
                    am[r][c] = a0[r][c];
                    m0[r][c] = mp[r][c];
                    a0[r][c] = ap[r][c];
                }
        }
        if (c1 == nt) {                                         // last temporal row: no row c+1
            const int64_t cc = nt - 1;
#pragma unroll
            for (int r = 0; r < FY; ++r)
#pragma unroll
                for (int c = 0; c < CJ; ++c) {
                    const SPt p = strip_pt(sp.i0, r, c, g);
                    if (!p.ok) continue;
                    const int64_t o = (cc - r0) * g.nx + (int64_t)p.i * g.m + p.j;
                    T1[o] = add_rn(band3(tri.At, cc, mm[r][c], m0[r][c], 0.0),
                                   band3(tri.LT, cc, am[r][c], a0[r][c], 0.0));
                    T2[o] = add_rn(band3(tri.Mt, cc, am[r][c], a0[r][c], 0.0),
                                   band3(tri.L, cc, mm[r][c], m0[r][c], 0.0));
                }
        }
    }
}

// out = M G1 + A G2 (+ E0 on row 0) and YM = M X, YA = A X on TMA-staged
// strips: NIN = 2 (bt_side: src = G1, G2) or 1 (stencil_rows: src = X)
template <int NIN, bool DM, bool DA, int FY, int CJ>
__global__ void __maxnreg__(96) stencil_strip(const double *__restrict__ X1,
                                                                   const double *__restrict__ X2,
                                                                   const double *__restrict__ E0,
                                                                   double *__restrict__ Y1,
                                                                   double *__restrict__ Y2, Grid g,
                                                                   Stencil M, Stencil A,
                                                                   int64_t rows, int ns)
{
    extern __shared__ __align__(16) double smem[];
    StripPipe<NIN, FY> sp;
    const double *srcs[2] = {X1, X2}, *begs[2] = {X1, X2},
                 *ends[2] = {X1 + rows * g.nx, X2 ? X2 + rows * g.nx : nullptr};
    sp.setup(smem, ns, srcs, begs, ends, g.m);
    const bool producer = threadIdx.x >= kStripT;
    int u = 0;
    for (int64_t b0 = (int64_t)blockIdx.z * kBtRows; b0 < rows; b0 += (int64_t)gridDim.z * kBtRows) {
        const int nq = (int)((b0 + kBtRows < rows ? b0 + kBtRows : rows) - b0);
        if (producer) {
            if (threadIdx.x == kStripT)
                for (int qi = 0; qi < nq; ++qi) sp.produce(u + qi, ns, (b0 + qi) * g.nx);
            u += nq;
            continue;
        }
        for (int qi = 0; qi < nq; ++qi, ++u) {
            const int64_t rr = b0 + qi;
            const int slot = sp.acquire(u, ns);
            double v1[FY][CJ], v2[FY][CJ];
            const int64_t roff = rr * g.nx;
#pragma unroll
            for (int r = 0; r < FY; ++r) {
                const double *am_ = sp.col0(slot, 0, r, roff), *a0_ = sp.col0(slot, 0, r + 1, roff),
                             *ap_ = sp.col0(slot, 0, r + 2, roff);
                const double *bm_ = NIN == 2 ? sp.col0(slot, NIN - 1, r, roff) : am_;
                const double *b0_ = NIN == 2 ? sp.col0(slot, NIN - 1, r + 1, roff) : a0_;
                const double *bp_ = NIN == 2 ? sp.col0(slot, NIN - 1, r + 2, roff) : ap_;
#pragma unroll
                for (int c = 0; c < CJ; ++c) {
                    const SPt p = strip_pt(sp.i0, r, c, g);
                    v1[r][c] = v2[r][c] = 0.0;
                    if (p.ok && !p.msk) {
                        if (NIN == 2) {
                            v1[r][c] = add_rn(stencil_tile<DM>(am_, a0_, ap_, p.j, p.i, g.m, p.in, M),
                                              stencil_tile<DA>(bm_, b0_, bp_, p.j, p.i, g.m, p.in, A));
                        } else {
                            if (Y1) v1[r][c] = stencil_tile<DM>(am_, a0_, ap_, p.j, p.i, g.m, p.in, M);
                            if (Y2) v2[r][c] = stencil_tile<DA>(am_, a0_, ap_, p.j, p.i, g.m, p.in, A);
                        }
                    }
                }
            }
            sp.release(slot);
#pragma unroll
            for (int r = 0; r < FY; ++r)
#pragma unroll
                for (int c = 0; c < CJ; ++c) {
                    const SPt p = strip_pt(sp.i0, r, c, g);
                    if (!p.ok) continue;
                    const int64_t k = (int64_t)p.i * g.m + p.j;
                    const int64_t o = rr * g.nx + k;
                    if (NIN == 2) {
                        double v = v1[r][c];
                        if (rr == 0 && E0 && !p.msk) v = add_rn(v, E0[k]);
                        Y1[o] = v;
                    } else {
                        if (Y1) Y1[o] = v1[r][c];
                        if (Y2) Y2[o] = v2[r][c];
                    }
                }
        }
    }
}

// opt-in (HWG_TMA=1): measured slower than the cached-load kernels at cfg 4
// (bside 8.9 vs 6.7 ms, bt_side 7.1 vs 4.9 ms, A_x 4.0 vs 3.0 ms; DESIGN.md
// §3.3), kept for A/B measurements
static int tma_enabled()
{
    static int on = -1;
    if (on < 0) {
        const char *ev = getenv("HWG_TMA");
        on = (ev && ev[0] == '1') ? 1 : 0;
    }
    return on;
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

// row strips need 511 <= m <= 2047 (2D); smaller grids keep the cached-load kernels
static bool strip_ok(const Grid &g) { return g.dim == 2 && g.m >= 511 && g.m <= 2047 && tma_enabled(); }

template <typename KernelT>
static cudaError_t prep_smem(KernelT k, size_t bytes)
{
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    if (getenv("HWG_TMA_DEBUG")) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, k);
        int nb = -1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, kStripThreads, bytes);
        fprintf(stderr, "strip kernel: regs %d maxThreads %d local %zu static smem %zu dyn %zu -> %d blocks/SM\n",
                fa.numRegs, fa.maxThreadsPerBlock, fa.localSizeBytes, fa.sharedSizeBytes, bytes, nb);
    }
    return cudaSuccess;
}

template <int FY, int CJ>
static cudaError_t launch_bside_strip(const double *U, int64_t u0, int64_t nu, double *T1, double *T2,
                                      double *E0, Grid g, Stencil M, Stencil A, Tri4 tri, int64_t r0,
                                      int64_t nr, int64_t nt, int chunk, cudaStream_t st)
{
    const int ns = strip_stages<1, FY>(g.m);
    const size_t sm = ns * strip_stage_bytes<1, FY>(g.m) + 128;
    const int64_t chunks = (nr + chunk - 1) / chunk;
    const dim3 grid(1, (unsigned)((g.m + FY - 1) / FY),
                    (unsigned)(chunks < 65535 ? (chunks < 1 ? 1 : chunks) : 65535));
    const bool dm = M.cd != 0.0, da = A.cd != 0.0;
    auto k = dm ? (da ? bside_strip<true, true, FY, CJ> : bside_strip<true, false, FY, CJ>)
                : (da ? bside_strip<false, true, FY, CJ> : bside_strip<false, false, FY, CJ>);
    cudaError_t e = prep_smem(k, sm);
    if (e != cudaSuccess) return e;
    k<<<grid, kStripThreads, sm, st>>>(U, u0, nu, T1, T2, E0, g, M, A, tri, r0, nr, nt, chunk, ns);
    return cudaGetLastError();
}

template <int NIN, int FY, int CJ>
static cudaError_t launch_stencil_strip_t(const double *X1, const double *X2, const double *E0,
                                          double *Y1, double *Y2, Grid g, Stencil M, Stencil A,
                                          int64_t rows, cudaStream_t st)
{
    const int ns = strip_stages<NIN, FY>(g.m);
    const size_t sm = ns * strip_stage_bytes<NIN, FY>(g.m) + 128;
    const int64_t zb = (rows + kBtRows - 1) / kBtRows;
    const dim3 grid(1, (unsigned)((g.m + FY - 1) / FY),
                    (unsigned)(zb < 65535 ? (zb < 1 ? 1 : zb) : 65535));
    const bool dm = M.cd != 0.0, da = A.cd != 0.0;
    auto k = dm ? (da ? stencil_strip<NIN, true, true, FY, CJ> : stencil_strip<NIN, true, false, FY, CJ>)
                : (da ? stencil_strip<NIN, false, true, FY, CJ> : stencil_strip<NIN, false, false, FY, CJ>);
    cudaError_t e = prep_smem(k, sm);
    if (e != cudaSuccess) return e;
    k<<<grid, kStripThreads, sm, st>>>(X1, X2, E0, Y1, Y2, g, M, A, rows, ns);
    return cudaGetLastError();
}

template <int NIN>
static cudaError_t launch_stencil_strip(const double *X1, const double *X2, const double *E0,
                                        double *Y1, double *Y2, Grid g, Stencil M, Stencil A,
                                        int64_t rows, cudaStream_t st)
{
    // FY x CJ points per thread; two inputs halve the rows to keep 4 stages
    constexpr int F = 4;
    switch ((g.m + kStripT - 1) / kStripT) {
    case 1: return launch_stencil_strip_t<NIN, F, 1>(X1, X2, E0, Y1, Y2, g, M, A, rows, st);
    case 2: return launch_stencil_strip_t<NIN, F / 2, 2>(X1, X2, E0, Y1, Y2, g, M, A, rows, st);
    default: return launch_stencil_strip_t<NIN, F / 4, 4>(X1, X2, E0, Y1, Y2, g, M, A, rows, st);
    }
}

cudaError_t launch_stencil_rows(const double *X, double *YM, double *YA, Grid g, Stencil M,
                                Stencil A, int64_t rows, cudaStream_t st)
{
    const bool dm = M.cd != 0.0, da = A.cd != 0.0;
    dim3 grid = spatial_grid(g, 1);
    const int64_t zb = (rows + kBtRows - 1) / kBtRows;
    grid.z = (unsigned)(zb < 65535 ? (zb < 1 ? 1 : zb) : 65535);
    const dim3 block(TX, TY);
    if (rows <= 0) return cudaSuccess;
    if (strip_ok(g)) return launch_stencil_strip<1>(X, nullptr, nullptr, YM, YA, g, M, A, rows, st);
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
    if (rows <= 0) return cudaSuccess;
    if (strip_ok(g)) return launch_stencil_strip<2>(G1, G2, E0, out, nullptr, g, M, A, rows, st);
    if (dm && da) bt_side<true, true><<<grid, block, 0, st>>>(G1, G2, E0, out, g, M, A, rows);
    else if (dm) bt_side<true, false><<<grid, block, 0, st>>>(G1, G2, E0, out, g, M, A, rows);
    else if (da) bt_side<false, true><<<grid, block, 0, st>>>(G1, G2, E0, out, g, M, A, rows);
    else bt_side<false, false><<<grid, block, 0, st>>>(G1, G2, E0, out, g, M, A, rows);
    return cudaGetLastError();
}

cudaError_t launch_bside_fused(const double *U, int64_t u0, int64_t nu, double *T1, double *T2,
                               double *E0, Grid g, Stencil M, Stencil A, Tri4 tri, int64_t r0,
                               int64_t nr, int64_t nt, cudaStream_t st)
{
    // temporal chunks of 32 rows (2 halo rows of stencils recomputed per chunk)
    dim3 grid = spatial_grid(g, 1);
    const int chunk = 32;
    const int64_t chunks = (nr + chunk - 1) / chunk;
    grid.z = (unsigned)(chunks < 65535 ? (chunks < 1 ? 1 : chunks) : 65535);
    const bool dm = M.cd != 0.0, da = A.cd != 0.0;
    const dim3 block(TX, TY);
    if (nr <= 0) return cudaSuccess;
    if (strip_ok(g)) {
        switch ((g.m + kStripT - 1) / kStripT) {
        case 1: return launch_bside_strip<4, 1>(U, u0, nu, T1, T2, E0, g, M, A, tri, r0, nr, nt, chunk, st);
        case 2: return launch_bside_strip<2, 2>(U, u0, nu, T1, T2, E0, g, M, A, tri, r0, nr, nt, chunk, st);
        default: return launch_bside_strip<1, 4>(U, u0, nu, T1, T2, E0, g, M, A, tri, r0, nr, nt, chunk, st);
        }
    }
    static const bool stack = [] {                       // HWG_BSIDE_STACK=0: one point per thread (A/B)
        const char *ev = getenv("HWG_BSIDE_STACK");
        return !(ev && ev[0] == '0');
    }();
    if (g.dim == 2 && stack) {
        constexpr int R = 4;
        dim3 gs = grid;
        gs.y = (unsigned)((g.m + TY * R - 1) / (TY * R));
        if (dm && da)
            bside_stack<true, true, R><<<gs, block, 0, st>>>(U, u0, T1, T2, E0, g, M, A, tri, r0, nr, nt, chunk);
        else if (dm)
            bside_stack<true, false, R><<<gs, block, 0, st>>>(U, u0, T1, T2, E0, g, M, A, tri, r0, nr, nt, chunk);
        else if (da)
            bside_stack<false, true, R><<<gs, block, 0, st>>>(U, u0, T1, T2, E0, g, M, A, tri, r0, nr, nt, chunk);
        else
            bside_stack<false, false, R><<<gs, block, 0, st>>>(U, u0, T1, T2, E0, g, M, A, tri, r0, nr, nt, chunk);
        return cudaGetLastError();
    }
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
