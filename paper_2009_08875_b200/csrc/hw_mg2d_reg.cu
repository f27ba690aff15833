// hw_mg2d_reg.cu -- register-resident streamed multigrid level passes, 2D,
// levels l = 7..10 (n = 2^l - 1 = 4 NT - 1 points per direction).
//
// Same operator as mg2d_stream (hw_mg2d.cu; the reference's _mg_core,
// /root/reference/pkg/src/heatwave/_kernels.py:110-199): per temporal row,
// DOWN = 3 forward lexicographic Gauss-Seidel sweeps + residual + restriction
// (R = P^T, spatial.py:140-173), UP = prolongation + 3 backward sweeps (run
// as forward sweeps on the point-reversed grid).  One CTA streams one
// temporal row's grid, one grid row per step, the three sweeps pipelined two
// grid rows apart.  What differs from mg2d_stream is where the state lives:
//
//  * Thread t owns columns 4t..4t+3 of every grid row (n + 1 = 4 NT, so no
//    thread idles).  The swept rows each sweep still needs (two per sweep)
//    live in REGISTERS; only chunk-boundary values cross threads -- by
//    shuffles inside a warp and through a few shared-memory words between
//    neighbouring warps (written before a barrier, read after it).
//  * A sweep over grid row i is the recurrence x_j = p_j + beta x_{j-1}
//    (p_j: right-hand side minus the known neighbours, scaled by 1/c0).  Each
//    thread runs it over its 4 points from a zero carry (chunk end S); the
//    carry into chunk t is T_{t-1} = sum_k gamma^(k-1) S_{t-k}, gamma =
//    beta^4.  A 3-level shuffle scan sums the nearest 8 chunk ends inside the
//    warp; the previous warp's windowed total covers the rest.  |beta| <=
//    1/4 for alpha A + mu M in 2D (checked on the host, else mg2d_stream is
//    used), so the dropped tail is below gamma^8 = 2^-64 relative: the
//    lexicographic GS result up to rounding.
//  * DOWN's residual after the third sweep uses the GS identity
//      r(i,j) = -(cy d(i,j+1) + cx d(i+1,j) + cd d(i+1,j+1)),  d = x3 - x2,
//    (every point's equation held exactly when it was updated; only its
//    "upper" neighbours moved afterwards) -- 3 multiply-adds per point.
//  * b, the input iterate and (UP) the coarse correction are staged by
//    zero-filling cp.async into THREAD-PRIVATE shared-memory slots three
//    steps ahead, so they need no barrier; each step has two barriers
//    (halo exchange, carry exchange).
#include "hw_common.cuh"
#include "hw_internal.cuh"

namespace hw {
namespace {

constexpr int RP = 4;  // points per thread

HW_DEV void cp_async8z(void *smem, const void *gmem, bool valid)
{
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(valid ? 8 : 0));
}

// shared-memory words (doubles) of one CTA
template <int NT, bool DOWN, bool ZS>
struct RegSmem {
    static constexpr int NW = NT / 32;
    static constexpr int B = 8 * 2 * NT * 2;                 // b ring  [8][2][NT][2]
    static constexpr int X0 = (DOWN && ZS) ? 0 : 4 * 5 * NT;  // x0 ring [4][5][NT]
    static constexpr int C = DOWN ? 0 : 4 * 4 * NT;          // coarse  [4][4][NT]
    static constexpr int H = 11 * (NW + 1);                  // halos, carries
    static constexpr int total = B + X0 + C + H;
};

template <int NT, bool DOWN, bool ZS>
struct RegPass {
    static constexpr int P = RP;
    static constexpr int NW = NT / 32;
    static constexpr int n = P * NT - 1;
    static constexpr int m = (n - 1) / 2;
    using SM = RegSmem<NT, DOWN, ZS>;

    // ---- per-CTA constants ----
    const MgStreamArgs &a;
    int tid, lane, warp;
    bool last;                            // owns column n (a zero pad)
    double cx, cy, cd, inv, beta;
    double bp[4];                         // beta^(k+1)
    double w1, w2, w4, gl;                // scan weights, gamma^lane
    const double *Bg;
    double *Xg;
    const double *Xcg;
    double *Bcg;
    double *bsm, *x0sm, *csm;
    double *HL, *HR, *HRes, *tot;         // [3][NW+1], [3][NW+1], [2][NW+1], [3][NW+1]

    // ---- register state ----
    double X1[2][4], X1L, X1R[2];          // sweep-1 rows (slot = row & 1) + halos
    double X2[2][4], X2L, X2R[2];
    double X3[4], X3L;                     // last sweep-3 row
    double D[2][4], DR[2];                 // DOWN: x3 - x2 rows
    double X0n[5];                         // x0 row t (+ right halo)
    double acc[2];                         // DOWN: coarse accumulators

    HW_DEV RegPass(const MgStreamArgs &a_, double *sm) : a(a_)
    {
        tid = threadIdx.x;
        lane = tid & 31;
        warp = tid >> 5;
        last = tid == NT - 1;
        const int64_t row = blockIdx.x;
        const int op = a.row_op ? a.row_op[row] : a.op;
        const double *cf = a.coef + ((int64_t)op * a.levels_p1 + a.level) * kCoefStride;
        cx = cf[kCx];
        cy = cf[kCy];
        cd = cf[kCd];
        inv = cf[kInv];
        beta = -cy * inv;
        double q = 1.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) { q *= beta; bp[k] = q; }
        const double g = bp[3], g2 = g * g, g4 = g2 * g2;
        w1 = lane >= 1 ? g : 0.0;
        w2 = lane >= 2 ? g2 : 0.0;
        w4 = lane >= 4 ? g4 : 0.0;
        double gp = 1.0, gb = g;               // gamma^lane by binary powering
#pragma unroll
        for (int b = 0; b < 5; ++b) { if (lane & (1 << b)) gp *= gb; gb *= gb; }
        gl = gp;
        Bg = a.B + row * a.ldB;
        Xg = a.X + row * a.ldX;
        Xcg = DOWN ? nullptr : a.Xc + row * a.ldXc;
        Bcg = DOWN ? a.Bc + row * a.ldBc : nullptr;
        bsm = sm;
        x0sm = bsm + SM::B;
        csm = x0sm + SM::X0;
        HL = csm + SM::C;
        HR = HL + 3 * (NW + 1);
        HRes = HR + 3 * (NW + 1);
        tot = HRes + 2 * (NW + 1);
        for (int k = tid; k < SM::H; k += NT) HL[k] = 0.0;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
#pragma unroll
            for (int k = 0; k < 4; ++k) X1[s][k] = X2[s][k] = D[s][k] = 0.0;
            X1R[s] = X2R[s] = DR[s] = 0.0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) X3[k] = 0.0;
        X1L = X2L = X3L = 0.0;
#pragma unroll
        for (int e = 0; e < 5; ++e) X0n[e] = 0.0;
        acc[0] = acc[1] = 0.0;
    }

    // global element (grid row i, local column j) of a level array; UP runs
    // point-reversed
    HW_DEV int64_t gidx(int i, int j) const
    {
        return DOWN ? (int64_t)i * n + j : (int64_t)(n - 1 - i) * n + (n - 1 - j);
    }

    // zero-filling stages of b row ib, x0 row ix, (UP) coarse row ic
    HW_DEV void issue_b(int ib) const
    {
        const int j0 = P * tid;
        const bool vr = ib < n;
        double *dst = bsm + (size_t)(ib & 7) * 4 * NT;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const bool v = vr && (j0 + k < n);
            cp_async8z(dst + ((k >> 1) * NT + tid) * 2 + (k & 1), Bg + (v ? gidx(ib, j0 + k) : 0), v);
        }
    }
    HW_DEV void issue_x0(int ix) const
    {
        const int j0 = P * tid;
        const bool vr = ix < n;
        double *dst = x0sm + (size_t)(ix & 3) * 5 * NT + tid;
#pragma unroll
        for (int e = 0; e < 5; ++e) {
            const bool v = vr && (j0 + e < n);
            cp_async8z(dst + e * NT, Xg + (v ? gidx(ix, j0 + e) : 0), v);
        }
    }
    HW_DEV void issue_c(int ic) const
    {
        // coarse columns 2t-1 .. 2t+2, point-reversed like the fine grid
        const bool vr = ic >= 0 && ic < m;
        double *dst = csm + (size_t)(ic & 3) * 4 * NT + tid;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int J = 2 * tid - 1 + q;
            const bool v = vr && J >= 0 && J < m;
            cp_async8z(dst + q * NT, Xcg + (v ? (int64_t)(m - 1 - ic) * m + (m - 1 - J) : 0), v);
        }
    }
    // the group step t issues: b(t+3), x0(t+4) and the coarse row x0(t+4) adds
    HW_DEV void issue(int t) const
    {
        issue_b(t + 3);
        if constexpr (!(DOWN && ZS)) issue_x0(t + 4);
        if constexpr (!DOWN) {
            if (!((t + 4) & 1)) issue_c((t + 4) / 2);
        }
        cp_async_commit();
    }

    // x0 row i (5 values) from its slot; UP adds the prolongated coarse
    // correction (same arithmetic as mg2d_stream's prolongate)
    template <int IPAR, bool EDGE>
    HW_DEV void load_x0(int i, double v[5]) const
    {
        const double *src = x0sm + (size_t)(i & 3) * 5 * NT + tid;
#pragma unroll
        for (int e = 0; e < 5; ++e) v[e] = src[e * NT];
        if constexpr (!DOWN) {
            if (EDGE && i >= n) return;                  // row n stays a zero pad
            double ca[4], cb[4];
            const int c_a = IPAR ? (i - 1) / 2 : i / 2 - 1;
            const double *pa = csm + (size_t)(c_a & 3) * 4 * NT + tid;
#pragma unroll
            for (int q = 0; q < 4; ++q) ca[q] = pa[q * NT];
            double pv[5];
            if constexpr (IPAR) {
                pv[0] = 0.5 * ca[0] + 0.5 * ca[1];
                pv[1] = ca[1];
                pv[2] = 0.5 * ca[1] + 0.5 * ca[2];
                pv[3] = ca[2];
                pv[4] = 0.5 * ca[2] + 0.5 * ca[3];
            } else {
                const double *pb = csm + (size_t)((c_a + 1) & 3) * 4 * NT + tid;
#pragma unroll
                for (int q = 0; q < 4; ++q) cb[q] = pb[q * NT];
                pv[0] = 0.5 * ca[0] + 0.5 * cb[1];
                pv[1] = 0.5 * ca[1] + 0.5 * cb[1];
                pv[2] = 0.5 * ca[1] + 0.5 * cb[2];
                pv[3] = 0.5 * ca[2] + 0.5 * cb[2];
                pv[4] = 0.5 * ca[2] + 0.5 * cb[3];
            }
#pragma unroll
            for (int e = 0; e < 5; ++e) v[e] = v[e] + pv[e];
            if (last) v[3] = v[4] = 0.0;                 // columns n, n+1
        }
    }

    HW_DEV void load_b(int i, double b[4]) const
    {
        const double2 *src = reinterpret_cast<const double2 *>(bsm + (size_t)(i & 7) * 4 * NT);
        const double2 lo = src[tid], hi = src[NT + tid];
        b[0] = lo.x;
        b[1] = lo.y;
        b[2] = hi.x;
        b[3] = hi.y;
    }

    // zero-carry chunk recurrence of one sweep over the thread's 4 points
    HW_DEV void chunk(const double u[4], double uL, const double c[4], double cR,
                      const double d[4], double dR, const double b[4], double y[4]) const
    {
        double yy = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double ul = k ? u[k - 1] : uL;
            const double cr = k < 3 ? c[k + 1] : cR;
            const double dr = k < 3 ? d[k + 1] : dR;
            const double e1 = fma(-cd, ul, b[k]);
            const double e2 = u[k] + d[k];
            const double e3 = fma(cd, dr, cy * cr);
            yy = fma(beta, yy, (fma(-cx, e2, e1) - e3) * inv);
            y[k] = yy;
        }
    }

    HW_DEV double wscan(double s) const
    {
        s = fma(w1, __shfl_up_sync(0xffffffffu, s, 1), s);
        s = fma(w2, __shfl_up_sync(0xffffffffu, s, 2), s);
        s = fma(w4, __shfl_up_sync(0xffffffffu, s, 4), s);
        return s;
    }

    template <bool EDGE, int PAR>
    HW_DEV void step(int t)
    {
        constexpr int Q = PAR ^ 1;        // slot of rows t-1, t-3, t-5
        const bool v1 = !EDGE || t < n;
        const bool v2 = !EDGE || (t >= 2 && t - 2 < n);
        const bool v3 = !EDGE || (t >= 4 && t - 4 < n);
        const bool vr = DOWN && (!EDGE || (t >= 6 && t - 6 < n));

        cp_async_wait<2>();                              // own b(t), x0(t+1) landed
        __syncthreads();                                 // (A) halos of step t-1 visible
        issue(t);
        if (lane == 0) {
            X1L = HL[0 * (NW + 1) + warp];
            X2L = HL[1 * (NW + 1) + warp];
            X3L = HL[2 * (NW + 1) + warp];
        }
        if (lane == 31) {
            X1R[Q] = HR[0 * (NW + 1) + warp + 1];
            X2R[Q] = HR[1 * (NW + 1) + warp + 1];
            if constexpr (DOWN) DR[Q] = HR[2 * (NW + 1) + warp + 1];
        }

        // ---- phase A: chunk recurrences of the three sweeps ----
        double y[3][4], b[4];
        double dn0[5];
        if constexpr (DOWN && ZS) {
            const double z[4] = {0.0, 0.0, 0.0, 0.0};
            load_b(t, b);
            chunk(X1[Q], X1L, z, 0.0, z, 0.0, b, y[0]);
#pragma unroll
            for (int e = 0; e < 5; ++e) dn0[e] = 0.0;
        } else {
            load_x0<Q, EDGE>(t + 1, dn0);
            load_b(t, b);
            chunk(X1[Q], X1L, X0n, X0n[4], dn0, dn0[4], b, y[0]);
        }
        load_b(t - 2, b);
        chunk(X2[Q], X2L, X1[PAR], X1R[PAR], X1[Q], X1R[Q], b, y[1]);
        load_b(t - 4, b);
        chunk(X3, X3L, X2[PAR], X2R[PAR], X2[Q], X2R[Q], b, y[2]);

        // residual of grid row t-6 from d(t-6), d(t-5)
        double R[4];
        if constexpr (DOWN) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double d6r = k < 3 ? D[PAR][k + 1] : DR[PAR];
                const double d5r = k < 3 ? D[Q][k + 1] : DR[Q];
                R[k] = fma(-cy, d6r, fma(-cx, D[Q][k], -cd * d5r));
            }
            if (lane == 31) {
                HRes[warp + 1] = R[2];
                HRes[(NW + 1) + warp + 1] = R[3];
            }
        }

        double A[3];
#pragma unroll
        for (int s = 0; s < 3; ++s) A[s] = wscan(y[s][3]);
        if (lane == 31) {
#pragma unroll
            for (int s = 0; s < 3; ++s) tot[s * (NW + 1) + warp + 1] = A[s];
        }
        __syncthreads();                                 // (B) warp totals visible

        // ---- phase B: carries, new rows, halos ----
        double xn[3][4];
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            const double prev = __shfl_up_sync(0xffffffffu, A[s], 1);
            const double cin = fma(gl, tot[s * (NW + 1) + warp], lane ? prev : 0.0);
            const bool vs = s == 0 ? v1 : (s == 1 ? v2 : v3);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double v = fma(bp[k], cin, y[s][k]);
                xn[s][k] = (vs && !(k == 3 && last)) ? v : 0.0;
            }
        }
        double dl[4];
        if constexpr (DOWN) {
#pragma unroll
            for (int k = 0; k < 4; ++k) dl[k] = xn[2][k] - X2[PAR][k];
        }
        if (v3) {                                        // final values of row t-4
            const int j0 = P * tid;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k < 3 || !last) Xg[gidx(t - 4, j0 + k)] = xn[2][k];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            X1[PAR][k] = xn[0][k];
            X2[PAR][k] = xn[1][k];
            X3[k] = xn[2][k];
            if constexpr (DOWN) D[PAR][k] = dl[k];
        }
        X1L = __shfl_up_sync(0xffffffffu, xn[0][3], 1);
        X2L = __shfl_up_sync(0xffffffffu, xn[1][3], 1);
        X3L = __shfl_up_sync(0xffffffffu, xn[2][3], 1);
        X1R[PAR] = __shfl_down_sync(0xffffffffu, xn[0][0], 1);
        X2R[PAR] = __shfl_down_sync(0xffffffffu, xn[1][0], 1);
        if constexpr (DOWN) DR[PAR] = __shfl_down_sync(0xffffffffu, dl[0], 1);
        if (lane == 31) {
            HL[0 * (NW + 1) + warp + 1] = xn[0][3];
            HL[1 * (NW + 1) + warp + 1] = xn[1][3];
            HL[2 * (NW + 1) + warp + 1] = xn[2][3];
        }
        if (lane == 0) {
            HR[0 * (NW + 1) + warp] = xn[0][0];
            HR[1 * (NW + 1) + warp] = xn[1][0];
            if constexpr (DOWN) HR[2 * (NW + 1) + warp] = dl[0];
        }
        if constexpr (!(DOWN && ZS)) {
#pragma unroll
            for (int e = 0; e < 5; ++e) X0n[e] = dn0[e];
        }

        // ---- restriction of residual row r = t-6 (parity PAR) ----
        if constexpr (DOWN) {
            if (vr) {
                double RL2 = __shfl_up_sync(0xffffffffu, R[2], 1);
                double RL3 = __shfl_up_sync(0xffffffffu, R[3], 1);
                if (lane == 0) {
                    RL2 = HRes[warp];
                    RL3 = HRes[(NW + 1) + warp];
                }
                const int r = t - 6;
                if constexpr (PAR) {                     // centre row of coarse (r-1)/2
                    acc[0] += fma(0.5, RL2 + R[0], RL3);
                    acc[1] += fma(0.5, R[0] + R[2], R[1]);
                } else {                                 // bottom of r/2-1, top of r/2
                    if (r >= 2) {
                        double *bc = Bcg + (int64_t)(r / 2 - 1) * m + 2 * tid;
                        if (tid > 0) bc[-1] = acc[0] + 0.5 * (RL3 + R[0]);
                        bc[0] = acc[1] + 0.5 * (R[1] + R[2]);
                    }
                    acc[0] = 0.5 * (RL2 + RL3);
                    acc[1] = 0.5 * (R[0] + R[1]);
                }
            }
        }
    }

    HW_DEV void run()
    {
        // prologue: x0 row 0 (+ coarse rows -1, 0), then the groups steps
        // -3..-1 would have issued
        if constexpr (!(DOWN && ZS)) {
            issue_x0(0);
            if constexpr (!DOWN) {
                issue_c(-1);
                issue_c(0);
            }
            cp_async_commit();
        }
        issue(-3);
        issue(-2);
        issue(-1);
        if constexpr (!(DOWN && ZS)) {
            cp_async_wait<3>();
            load_x0<0, true>(0, X0n);
        }
        constexpr int nsteps = DOWN ? n + 6 : n + 4;
        int t = 0;
        for (; t < 6; t += 2) {
            step<true, 0>(t);
            step<true, 1>(t + 1);
        }
        for (; t + 2 < n; t += 2) {             // x0(t+2) < n: no edge cases
            step<false, 0>(t);
            step<false, 1>(t + 1);
        }
        for (; t < nsteps; t += 2) {
            step<true, 0>(t);
            if (t + 1 < nsteps) step<true, 1>(t + 1);
        }
        cp_async_wait<0>();
    }
};

template <int NT, bool DOWN, bool ZS>
__global__ void __launch_bounds__(NT, 1) mg2d_reg(MgStreamArgs a)
{
    extern __shared__ __align__(16) double sm[];
    RegPass<NT, DOWN, ZS> p(a, sm);
    p.run();
}

template <int NT, bool DOWN, bool ZS>
cudaError_t launch_reg_t(const MgStreamArgs &a, int64_t rows, cudaStream_t st)
{
    const size_t smem = RegSmem<NT, DOWN, ZS>::total * sizeof(double);
    auto k = mg2d_reg<NT, DOWN, ZS>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<(unsigned)rows, NT, smem, st>>>(a);
    return cudaGetLastError();
}

template <int NT>
cudaError_t launch_reg_n(const MgStreamArgs &a, bool down, int64_t rows, cudaStream_t st)
{
    if (!down) return launch_reg_t<NT, false, false>(a, rows, st);
    return a.zero_start ? launch_reg_t<NT, true, true>(a, rows, st)
                        : launch_reg_t<NT, true, false>(a, rows, st);
}

}  // namespace

cudaError_t mg2d_reg_launch(const MgStreamArgs &a, bool down, int64_t rows, cudaStream_t st)
{
    switch (a.n) {
    case 127: return launch_reg_n<32>(a, down, rows, st);
    case 255: return launch_reg_n<64>(a, down, rows, st);
    case 511: return launch_reg_n<128>(a, down, rows, st);
    case 1023: return launch_reg_n<256>(a, down, rows, st);
    default: return cudaErrorNotSupported;
    }
}

}  // namespace hw
