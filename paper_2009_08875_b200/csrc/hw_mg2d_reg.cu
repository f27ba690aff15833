// hw_mg2d_reg.cu -- register-resident streamed multigrid level passes, 2D,
// levels l = 6..11 (n = 2^l - 1 = P NT - 1 points per direction).
//
// Same operator as mg2d_stream (hw_mg2d.cu; the reference's _mg_core,
// /root/reference/pkg/src/heatwave/_kernels.py:110-199): per temporal row,
// DOWN = 3 forward lexicographic Gauss-Seidel sweeps + residual + restriction
// (R = P^T, spatial.py:140-173), UP = prolongation + 3 backward sweeps (run
// as forward sweeps on the point-reversed grid).  One CTA streams one
// temporal row's grid, one grid row per step, the three sweeps pipelined two
// grid rows apart.  What differs from mg2d_stream is where the state lives:
//
//  * Thread t owns columns P t .. P t + P-1 of every grid row (n + 1 = P NT,
//    no thread idles).  The swept rows each sweep still needs (two per sweep)
//    live in REGISTERS; only chunk-boundary values cross threads.
//  * A sweep over grid row i is the recurrence x_j = p_j + beta x_{j-1}
//    (p_j: right-hand side minus the known neighbours, scaled by 1/c0).  Each
//    thread runs it over its P points from a zero carry (chunk end S); the
//    carry into chunk t is T_{t-1} = sum_k gamma^(k-1) S_{t-k}, gamma =
//    beta^P.  A shuffle scan sums the nearest W = 32/P chunk ends inside the
//    warp; the previous warp's windowed total covers the rest.  |beta| <=
//    1/4 for alpha A + mu M in 2D (checked on the host, else mg2d_stream is
//    used), so the dropped tail is below gamma^W <= 2^-64 relative: the
//    lexicographic GS result up to rounding.
//  * The carry into chunk t IS the new value of the point left of the chunk,
//    so left halos cost nothing; right halos (the next chunk's first new
//    value) are one shuffle, or a shared word at a warp edge.
//  * DOWN's residual after the third sweep uses the GS identity
//      r(i,j) = -(cy d(i,j+1) + cx d(i+1,j) + cd d(i+1,j+1)),  d = x3 - x2,
//    (every point's equation held when it was updated; only its "upper"
//    neighbours moved afterwards) -- 3 multiply-adds per point.
//  * b, the input iterate and (UP) the coarse correction are staged by
//    zero-filling cp.async into THREAD-PRIVATE shared-memory slots three
//    steps ahead, so they need no barrier; each step has two barriers
//    (halo exchange, carry exchange).
//  * Scaled iterates: inside a pass every row the sweeps touch holds c0 x
//    (x0 rows are scaled once as they are loaded, final rows unscaled once
//    as they are staged for the store), so a point's update needs no b / c0:
//    c0 x = b - (cx/c0)(c0 u + c0 d) - ... + beta c0 x_left.  DOWN's GS-identity
//    residual of scaled differences is then the residual itself.
//  * LSH: the mapped L-shaped domain, embedded in the square grid with the
//    closed quadrant i, j >= m = (n-1)/2 (natural coordinates) held at zero.
//    Lexicographic GS on the L is GS on the square with those points reset
//    to zero: the recurrence restarts (y = 0) at a masked point, so masked
//    chunk ends are zero and carry nothing into the next unmasked chunk, and
//    the final values of masked points are forced to zero after the carry
//    (DOWN: the masked part of a row is a suffix; UP, point-reversed, a
//    prefix).  Masked residuals are zero before restriction; prolongation
//    needs nothing (masked fine points interpolate masked coarse zeros).
//  * Thread shapes: P = 8 points per thread by default; contexts with a short
//    time axis run levels 7-9 with twice the threads (mg2d_reg_launch).
//  * CL = 2 (opt-in, n = 2047): the grid row as two column strips on a
//    thread-block cluster; the strips exchange carry windows and halos as
//    st.async messages that complete the receiver's mbarrier (RegPass).
#include "hw_common.cuh"
#include "hw_internal.cuh"

#include <cstdint>
#include <cstdlib>

namespace hw {
namespace {

HW_DEV void cp_async8z(void *smem, const void *gmem, bool valid)
{
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(valid ? 8 : 0));
}

HW_DEV void cp_async8s(unsigned saddr, const void *gmem)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(gmem));
}
HW_DEV void cp_async16s(unsigned saddr, const void *gmem)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem));
}
HW_DEV unsigned smem_u32(const void *p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
// zero-filling variants: `skip` writes zeros without reading global memory
// (the L-shaped domain's removed quadrant, which holds zeros anyway)
HW_DEV void cp_async16s(unsigned saddr, const void *gmem, bool skip)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem),
                 "r"(skip ? 0 : 16));
}
HW_DEV void cp_async8s(unsigned saddr, const void *gmem, bool skip)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem),
                 "r"(skip ? 0 : 8));
}

constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v / 2); }

// ---- thread-block cluster helpers (CL = 2 column strips of one temporal row) ----
HW_DEV unsigned cluster_ctarank()
{
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
HW_DEV void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
HW_DEV unsigned mapa_u32(unsigned saddr, unsigned rank)
{
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
// store v at the address `local` has in CTA `rank` of the cluster (DSMEM)
HW_DEV void st_cluster(double *local, unsigned rank, double v)
{
    asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(mapa_u32(smem_u32(local), rank)), "d"(v)
                 : "memory");
}
// Per-step messages between the strips: the sender's st.async writes a
// double into the receiver's mailbox and completes 8 bytes of the receiver's
// mbarrier transaction count (STAS: no fence, no L1 invalidation -- a
// st.release.cluster costs MEMBAR.ALL.GPU, a barrier.cluster ~1.7k cycles
// here); the receiver arms the phase with arrive.expect_tx and polls
// try_wait.parity.
HW_DEV void mbar_init(unsigned mb, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mb), "r"(count) : "memory");
}
HW_DEV void mbar_expect(unsigned mb, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bytes)
                 : "memory");
}
HW_DEV void mbar_wait(unsigned mb, unsigned parity)
{
    unsigned done = 0;
    int spins = 0;
    while (!done) {
        asm volatile("{\n.reg .pred p;\n"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     "selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done)
                     : "r"(mb), "r"(parity)
                     : "memory");
        if (!done && ++spins > (1 << 22)) __trap();      // never hang the GPU on a lost message
    }
}
HW_DEV void st_async_f64(unsigned raddr, double v, unsigned rmbar)
{
    asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(raddr),
                 "d"(v), "r"(rmbar)
                 : "memory");
}

// shared-memory words (doubles) of one CTA.  Fine rows are staged whole
// (cooperative, coalesced copies) in slots of RS words with a 16-byte-unit
// XOR swizzle, so a thread's own chunk reads are conflict-free LDS.128.
template <int P, int NT, bool DOWN, bool ZS>
struct RegSmem {
    static constexpr int NW = NT / 32;
    static constexpr int RS = P * NT + 16;                  // fine row slot
    static constexpr int CS = P * NT / 2 + 8;               // coarse row slot
    // ring depths: copies are issued after the step's second barrier, when
    // the slot's previous row (b: t-4, x0: t+1) has been consumed
    static constexpr int NB = 7, NX = 3, NCR = 3;
    static constexpr int B = NB * RS;                       // b ring
    static constexpr int X0 = (DOWN && ZS) ? 0 : NX * RS;   // x0 ring
    static constexpr int C = DOWN ? 0 : NCR * CS;           // coarse ring (UP)
    static constexpr int O = RS;                            // output row
    static constexpr int H = 8 * (NW + 1) + 20;             // halos, carries, cluster dot share,
                                                            // strip mailboxes + mbarriers
    static constexpr int total = B + X0 + C + O + H;
};

// LB0 / LX0 (UP only): layout parity of grid row 0 of b / x0 (stage_row);
// row i has parity L0 ^ (i & 1) because a grid row is n (odd) words long
// DG: the operator has diagonal couplings (c_d != 0, every C_j = alpha A +
// mu M); DG = false (K_x = A_x, a 5-point stencil) drops them at compile time
// CL = 2: the grid row is split into two column strips of P NT columns, one
// per CTA of a thread-block cluster (n + 1 = 2 P NT; BASELINE cfg 5's n =
// 2047 with the footprint of the n = 1023 kernel, so two CTAs of different
// temporal rows share an SM instead of one phase-locked 256-thread CTA).
// The truncated carry into the right strip is the left strip's last-warp
// windowed total; the left strip's right halos are the right strip's first
// new values: six doubles per step cross the pair through distributed shared
// memory, ordered by the two per-step barriers (cluster-wide instead of
// CTA-wide).  Same chunks, windows and arithmetic as one CTA of 2 NT threads.
template <int P, int NT, bool DOWN, bool ZS, int LB0, int LX0, bool LSH, bool DG, int CL = 1>
struct RegPass {
    static constexpr int NW = NT / 32;
    static constexpr int n = CL * P * NT - 1;
    static constexpr int m = (n - 1) / 2;
    static constexpr int WIN = 32 / P;                 // chunk ends in the carry window
    static constexpr int LEV = ilog2c(WIN);            // shuffle-scan levels
    static constexpr int NC = (P / 2 + 3) & ~1;        // coarse columns a thread reads (even)
    static constexpr int HS = NW + 1;
    static constexpr int SWZ = P / 2 - 1;
    using SM = RegSmem<P, NT, DOWN, ZS>;
    static constexpr int RS = SM::RS, CS = SM::CS;
    static_assert(P % 2 == 0 && 32 % P == 0 && P >= 2 && CS >= (P / 2) * (NT - 1) + NC &&
                      CS >= (CL == 1 ? m + 2 : (P / 2) * NT + 4) && (CL == 1 || CL == 2),
                  "chunk layout");
    static constexpr int gs = DOWN ? 1 : -1;           // UP runs point-reversed

    // ---- per-CTA / per-thread constants ----
    int tid, lane, warp;
    int crank, col0, gt;                  // cluster rank, first column of the strip, chunk number in the row
    bool lstrip;                          // the strip that ends with column n
    bool last;                            // owns column n (a zero pad)
    double cxs, cds, c0, inv, beta;       // cx/c0, cd/c0, c0, 1/c0, -cy/c0
    double bp[P];                         // beta^(k+1)
    double wl[LEV];                       // scan weights gamma^(2^l) (0 below lane 2^l)
    double gl;                            // gamma^lane
    const double *Bg, *Xcg;               // row 0 of this temporal row's level arrays
    double *Xg, *Bcg;
    const double *Dg;                     // UP: fused inner-product operand (or null)
    double dsum;                          //     this thread's share of <Dg, X>
    double *bsm, *x0sm, *csm, *osm;
    double *HR, *HRes, *tot;              // [3][HS], [1][HS], [3][HS]
    double *box_tot, *box_hr, *box_res;   // CL > 1 mailboxes [2][3], [2][3], [2] (slot = step parity)
    unsigned mb_tot, mb_hr, mb_res;       //         their mbarriers (shared addresses)
    int cpo;                              // slot position of column tid (copy / flush lane)
    int hoff;                             // DOWN: slot position of the right-halo column P (t+1)
    int ooff[P / 2 + 1];                  // slot positions of units P t/2 .. P t/2 + P/2
    int sb, sx;                           // ring slots of b(t) and x0(t+1) at step t
    int sc;                               // UP: ring slot of coarse row floor(t/2) at step t
    double HC[NC];                        // UP: 0.5 x the latest coarse row this thread reads
    unsigned cm;                          // LSH: bit k = column P t + k lies in the masked range
    // column tid + k NT sits at cpo + k NT when the swizzle is periodic in NT
    static constexpr bool LIN = (NT / 16) % (P / 2) == 0;

    // ---- register state ----
    double X1[2][P], X1L, X1R[2];          // sweep-1 rows (slot = row & 1) + halos
    double X2[2][P], X2L, X2R[2];
    double X3[P], X3L;                     // last sweep-3 row
    double D[2][P], DR[2];                 // DOWN: x3 - x2 rows
    double X0n[P + 1];                     // x0 row t (+ right halo)
    double acc[P / 2];                     // DOWN: coarse accumulators

    // swizzled slot position of fine column j (16-byte units permuted within
    // groups of 8 so 8 consecutive threads' chunk units hit distinct banks)
    static HW_DEV int phys(int j)
    {
        const int u = j >> 1;
        return ((u ^ ((u >> 3) & SWZ)) << 1) | (j & 1);
    }

    // coarse slot position of index x (= local coarse column + 1): 16-byte
    // units XOR-swizzled by bit 3 so a thread's LDS.128 of its NC values
    // (units (P/4) t .. ) are bank-conflict free
    static HW_DEV int cphys(int x)
    {
        const int u = x >> 1;
        return ((u ^ ((u >> 3) & 1)) << 1) | (x & 1);
    }

    HW_DEV RegPass(const MgStreamArgs &a, double *sm)
    {
        tid = threadIdx.x;
        lane = tid & 31;
        warp = tid >> 5;
        crank = CL > 1 ? (int)cluster_ctarank() : 0;
        col0 = crank * P * NT;
        gt = crank * NT + tid;
        lstrip = crank == CL - 1;
        last = lstrip && tid == NT - 1;
        const int64_t row = blockIdx.x / CL;
        const int op = a.row_op ? a.row_op[row] : a.op;
        const double *cf = a.coef + ((int64_t)op * a.levels_p1 + a.level) * kCoefStride;
        inv = cf[kInv];
        c0 = cf[kC0];
        cxs = cf[kCx] * inv;
        cds = cf[kCd] * inv;
        beta = -cf[kCy] * inv;
        double q = 1.0;
#pragma unroll
        for (int k = 0; k < P; ++k) { q *= beta; bp[k] = q; }
        double g = bp[P - 1];
#pragma unroll
        for (int l = 0; l < LEV; ++l) { wl[l] = lane >= (1 << l) ? g : 0.0; g *= g; }
        double gp = 1.0, gb = bp[P - 1];       // gamma^lane by binary powering
#pragma unroll
        for (int b = 0; b < 5; ++b) { if (lane & (1 << b)) gp *= gb; gb *= gb; }
        gl = gp;
        Bg = a.B + row * a.ldB;
        Xg = a.X + row * a.ldX;
        Xcg = DOWN ? nullptr : a.Xc + row * a.ldXc;
        Bcg = DOWN ? a.Bc + row * a.ldBc + (P / 2) * gt : nullptr;
        Dg = (!DOWN && a.dot_y) ? a.dot_y + row * a.ldX : nullptr;
        dsum = 0.0;
        bsm = sm;
        x0sm = bsm + SM::B;
        csm = x0sm + SM::X0;
        osm = csm + SM::C;
        HR = osm + SM::O;
        HRes = HR + 3 * HS;
        tot = HRes + HS;
        box_tot = tot + 3 * HS + 2;                        // (+2: the cluster dot share)
        box_hr = box_tot + 6;
        box_res = box_hr + 6;
        mb_tot = smem_u32(box_res + 2);
        mb_hr = mb_tot + 8;
        mb_res = mb_hr + 8;
        for (int k = tid; k < SM::total; k += NT) sm[k] = 0.0;   // pads stay zero
        cpo = phys(tid);
        hoff = phys(P * (tid + 1));
        cm = 0u;
        if constexpr (LSH) {
#pragma unroll
            for (int k = 0; k < P; ++k)
                if (DOWN ? (P * gt + k >= m) : (P * gt + k <= m)) cm |= 1u << k;
        }
#pragma unroll
        for (int h = 0; h <= P / 2; ++h) ooff[h] = phys(P * tid + 2 * h);
        sb = 4;                                // step -3 (the prologue's first group)
        sx = 1;
        sc = 0;                                // coarse row 0 at steps 0, 1
#pragma unroll
        for (int s = 0; s < 2; ++s) {
#pragma unroll
            for (int k = 0; k < P; ++k) X1[s][k] = X2[s][k] = D[s][k] = 0.0;
            X1R[s] = X2R[s] = DR[s] = 0.0;
        }
#pragma unroll
        for (int k = 0; k < P; ++k) X3[k] = 0.0;
        X1L = X2L = X3L = 0.0;
#pragma unroll
        for (int e = 0; e <= P; ++e) X0n[e] = 0.0;
#pragma unroll
        for (int q2 = 0; q2 < P / 2; ++q2) acc[q2] = 0.0;
#pragma unroll
        for (int q = 0; q < NC; ++q) HC[q] = 0.0;          // coarse row -1
    }

    // global element of (grid row i, strip column j); UP is point-reversed
    HW_DEV int64_t gidx(int i, int j) const
    {
        return DOWN ? (int64_t)i * n + (col0 + j) : (int64_t)(n - 1 - i) * n + (n - 1 - col0 - j);
    }

    HW_DEV int koff(int k) const { return LIN ? k * NT : phys(tid + k * NT) - cpo; }

    // Cooperative coalesced stage of fine row i of src (columns 0..n-1; the
    // pad columns -1, n, n+1 are never written by a copy).  Rows >= n: ZERO
    // writes a zero row (x0 row n is the grid's zero boundary row), else the
    // copy is skipped (such b / x0 rows only feed discarded sweeps).
    //  DOWN: natural layout; rows whose column pairs (2p, 2p+1) are 16-byte
    //   units in global memory (half of them, n is odd) are copied 16 bytes
    //   at a time, the others 8 bytes.
    //  UP (LR = layout parity): the slot holds the row's global 16-byte
    //   units, columns (2u - LR, 2u + 1 - LR), in address order (so each
    //   unit's columns are swapped: UP reads point-reversed); every copy is
    //   16 bytes but the half-units at the row ends.  UP is bound by its
    //   copy-instruction count; DOWN is not (the parity variants cost it
    //   more than they saved).
    template <bool ZERO, int LR>
    HW_DEV void stage_row(double *slot, const double *src, int i) const
    {
        if (i >= n) {
            if constexpr (ZERO) {
#pragma unroll
                for (int k = 0; k < P; ++k) slot[tid + k * NT] = 0.0;
                if (CL > 1 && !lstrip && tid == 0) slot[phys(P * NT)] = slot[phys(P * NT) + 1] = 0.0;
            }
            return;
        }
        const double *row0 = src + gidx(i, 0);               // strip column 0
        // CL > 1: a strip that is not the last also stages the unit after it
        // (the next strip's first columns: the last thread's right halo)
        const bool xhalo = CL > 1 && !lstrip && tid == 0;
        const unsigned xs = smem_u32(slot + phys(P * NT));
        if constexpr (DOWN) {
            if ((reinterpret_cast<uintptr_t>(row0) & 15) == 0) {
                const unsigned sa = smem_u32(slot + phys(2 * tid));
#pragma unroll
                for (int k = 0; k < P / 2; ++k) {
                    const int q = tid + k * NT;              // pair (2q, 2q+1)
                    const bool skip = LSH && i >= m && col0 + 2 * q >= m;   // removed quadrant
                    if (k < P / 2 - 1 || tid < NT - 1 || !lstrip)
                        cp_async16s(sa + 16u * k * NT, row0 + 2 * q, skip);
                    else                                     // column n-1 only (n is a pad)
                        cp_async8s(sa + 16u * k * NT, row0 + 2 * q, skip);
                }
                if (xhalo) cp_async16s(xs, row0 + P * NT, LSH && i >= m && col0 + P * NT >= m);
            } else {
                const double *g = row0 + tid;
                const unsigned sa = smem_u32(slot + cpo);
#pragma unroll
                for (int k = 0; k < P; ++k)
                    if (k < P - 1 || tid < NT - 1 || !lstrip)
                        cp_async8s(sa + 8u * koff(k), g + k * NT,
                                   LSH && i >= m && col0 + tid + k * NT >= m);
                if (xhalo) cp_async8s(xs, row0 + P * NT, LSH && i >= m && col0 + P * NT >= m);
            }
        } else {
            const unsigned sa = smem_u32(slot + phys(2 * tid));
#pragma unroll
            for (int k = 0; k < P / 2; ++k) {
                const int q = tid + k * NT;                  // unit q
                const unsigned d = sa + 16u * k * NT;
                if constexpr (LR == 0) {                     // columns (2q, 2q+1)
                    if (k < P / 2 - 1 || tid < NT - 1 || !lstrip) {
                        cp_async16s(d, row0 - 2 * q - 1, LSH && i <= m && col0 + 2 * q + 1 <= m);
                    } else {                                 // (n-1, n): column n-1 only;
                        cp_async8s(d + 8u, row0 - 2 * q);
                        // the pad n: the slot may last have held a parity-1
                        // row, whose unit here was full
                        slot[phys(2 * q)] = 0.0;
                    }
                } else {                                     // columns (2q-1, 2q)
                    if (k > 0 || tid > 0 || crank > 0)
                        cp_async16s(d, row0 - 2 * q, LSH && i <= m && col0 + 2 * q <= m);
                    else cp_async8s(d, row0);                // (-1, 0): column 0 only
                }
            }
            if (xhalo) {
                if constexpr (LR == 0)                       // columns (P NT, P NT + 1)
                    cp_async16s(xs, row0 - P * NT - 1, LSH && i <= m && col0 + P * NT + 1 <= m);
                else                                         // columns (P NT - 1, P NT)
                    cp_async16s(xs, row0 - P * NT, LSH && i <= m && col0 + P * NT <= m);
            }
        }
    }
    // coarse row ic, local columns 0..m-1 at slot index J+1 (index 0 and m+1
    // stay zero); rows -1 and m are zero rows
    HW_DEV void stage_coarse(int ic, int slotno) const
    {
        if (ic > m) return;
        if constexpr (CL > 1) {
            // strip: slot index x holds coarse column (P/2) NT crank + x - 1;
            // indices whose column does not exist are never written (zero)
            double *slot = csm + (size_t)slotno * CS;
            constexpr int mc = (m - 1) / 2;
            for (int x = tid; x < (P / 2) * NT + 4; x += NT) {
                const int J = (P / 2) * NT * crank + x - 1;
                if (J < 0 || J >= m) continue;
                double *d = slot + cphys(x);
                if (ic < 0 || ic == m) *d = 0.0;
                else
                    cp_async8s(smem_u32(d), Xcg + (int64_t)(m - 1 - ic) * m + (m - 1 - J),
                               LSH && ic <= mc && J <= mc);
            }
            return;
        }
        static_assert((NT / 16) % 2 == 0, "coarse swizzle periodic in NT");
        double *slot = csm + (size_t)slotno * CS + cphys(1 + tid);
        if (ic < 0 || ic == m) {
#pragma unroll
            for (int k = 0; k < (m + NT - 1) / NT; ++k)
                if (tid + k * NT < m) slot[k * NT] = 0.0;
            return;
        }
        const double *g = Xcg + (int64_t)(m - 1 - ic) * m + (m - 1) - tid;
        const unsigned sa = smem_u32(slot);
        constexpr int mc = (m - 1) / 2;                      // coarse removed quadrant (reversed)
#pragma unroll
        for (int k = 0; k < (m + NT - 1) / NT; ++k)
            if (tid + k * NT < m)
                cp_async8s(sa + 8u * k * NT, g - k * NT, LSH && ic <= mc && tid + k * NT <= mc);
    }
    HW_DEV int bslot(int back) const { return sb >= back ? sb - back : sb + SM::NB - back; }
    // the group step t issues: b(t+3) (into b(t-4)'s slot), x0(t+4) (into
    // x0(t+1)'s slot) and the coarse row x0(t+4) adds
    template <int TPAR>                // TPAR = t & 1
    HW_DEV void issue(int t) const
    {
        stage_row<false, LB0 ^ TPAR ^ 1>(bsm + (size_t)bslot(4) * RS, Bg, t + 3);
        if constexpr (!(DOWN && ZS)) stage_row<true, LX0 ^ TPAR>(x0sm + (size_t)sx * RS, Xg, t + 4);
        if constexpr (!DOWN && TPAR == 0)    // coarse row floor(t/2) + 2 (even t)
            stage_coarse((t + 4) / 2, sc + 2 >= SM::NCR ? sc + 2 - SM::NCR : sc + 2);
        cp_async_commit();
    }

    // own chunk (v[0..P-1]) of a staged row; UP rows of layout parity 1 also
    // yield the right-halo column v[P] from the extra unit
    template <int LR>
    HW_DEV void load_chunk(const double *slot, double v[P + 1]) const
    {
        constexpr int L = DOWN ? 0 : LR;
#pragma unroll
        for (int h = 0; h < P / 2 + L; ++h) {
            const double2 w = *reinterpret_cast<const double2 *>(slot + ooff[h]);
            const double lo = DOWN ? w.x : w.y, hi = DOWN ? w.y : w.x;   // lower / upper column
            if constexpr (L == 0) {
                v[2 * h] = lo;
                v[2 * h + 1] = hi;
            } else {
                if (h > 0) v[2 * h - 1] = lo;
                v[2 * h] = hi;
            }
        }
    }

    // x0 row i (P+1 values) from its slot; UP adds the prolongated coarse
    // correction (same arithmetic as mg2d_stream's prolongate)
    template <int IPAR, bool EDGE, int LR>
    HW_DEV void load_x0(int i, int slotno, int cslot, double v[P + 1])
    {
        const double *slot = x0sm + (size_t)slotno * RS;
        load_chunk<LR>(slot, v);
        if constexpr (DOWN) v[P] = slot[hoff];                         // right halo
        else if constexpr (LR == 0) v[P] = slot[ooff[P / 2] + 1];
        if constexpr (!DOWN) {
            if (EDGE && i >= n) return;                  // row n stays a zero pad (no scaling)
            // coarse rows c_a = floor((i-1)/2) and, for even i, c_a + 1.  Row
            // c_a is the one the previous step loaded (kept as exact halves in
            // HC), so each pair of steps reads one new coarse row.  0.5 c is
            // exact, hence h_a + h_b == 0.5 c_a + 0.5 c_b and h + h == c:
            // the same rounding as the stream kernel's prolongation.
            double hb[NC];
            if constexpr (!IPAR) {
                const double *pb = csm + (size_t)(cslot + 1 == SM::NCR ? 0 : cslot + 1) * CS;
                if constexpr ((P / 2) % 2 == 0) {            // 16-byte aligned pairs
#pragma unroll
                    for (int q = 0; q < NC; q += 2) {
                        const double2 w = *reinterpret_cast<const double2 *>(pb + cphys((P / 2) * tid + q));
                        hb[q] = 0.5 * w.x;
                        hb[q + 1] = 0.5 * w.y;
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < NC; ++q) hb[q] = 0.5 * pb[cphys((P / 2) * tid + q)];
                }
            }
#pragma unroll
            for (int e = 0; e <= P; ++e) {
                double pv;
                if (e & 1) {
                    const int q = (e + 1) / 2;
                    pv = IPAR ? HC[q] + HC[q] : HC[q] + hb[q];
                } else {
                    const int q = e / 2;
                    pv = IPAR ? HC[q] + HC[q + 1] : HC[q] + hb[q + 1];
                }
                v[e] = v[e] + pv;
            }
            if constexpr (!IPAR) {
#pragma unroll
                for (int q = 0; q < NC; ++q) HC[q] = hb[q];
            }
            if (last) v[P - 1] = v[P] = 0.0;             // columns n, n+1
        }
#pragma unroll
        for (int e = 0; e <= P; ++e) v[e] *= c0;         // the pass works on c0 x
    }

    template <int LR>
    HW_DEV void load_b(int back, double b[P + 1]) const
    {
        load_chunk<LR>(bsm + (size_t)bslot(back) * RS, b);
    }

    // coalesced copy of the staged output row (grid row i) to global memory
    HW_DEV void flush(int i)
    {
        double *g = Xg + gidx(i, 0) + gs * tid;
        double v[P];
#pragma unroll
        for (int k = 0; k < P; ++k) v[k] = osm[cpo + koff(k)];
#pragma unroll
        for (int k = 0; k < P; ++k)
            if (k < P - 1 || tid < NT - 1 || !lstrip) g[gs * k * NT] = v[k];
        if (!DOWN && Dg) {                       // fused inner product, fixed order
            const double *d = Dg + gidx(i, 0) + gs * tid;
#pragma unroll
            for (int k = 0; k < P; ++k)
                if (k < P - 1 || tid < NT - 1 || !lstrip) dsum = fma(d[gs * k * NT], v[k], dsum);
        }
    }

    // per-row partial of the fused inner product: xor-butterfly in each warp,
    // then the warp totals in warp order (deterministic)
    HW_DEV void finish_dot(const MgStreamArgs &a)
    {
        if (DOWN || !Dg) return;
        double v = dsum;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        __syncthreads();
        if (lane == 0) tot[warp] = v;
        __syncthreads();
        if (warp == 0) {
            double u = lane < NW ? tot[lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
            if constexpr (CL == 1) {
                if (lane == 0) a.dot_part[blockIdx.x] = u;
            } else {
                double *xdot = tot + 3 * HS;               // [2], used only here
                if (lane == 0 && crank > 0) st_cluster(&xdot[1], 0, u);   // the right strip's share
                if (lane == 0) xdot[0] = u;
            }
        }
        if constexpr (CL > 1) {
            cluster_sync_all();
            const double *xdot = tot + 3 * HS;
            if (crank == 0 && tid == 0) a.dot_part[blockIdx.x / CL] = xdot[0] + xdot[1];
        }
    }

    // LSH: mask bits of grid row i (DOWN: rows >= m mask columns >= m; UP,
    // point-reversed: rows <= m mask columns <= m)
    HW_DEV unsigned rmask(int i) const
    {
        if constexpr (!LSH) return 0u;
        return (DOWN ? i >= m : i <= m) ? cm : 0u;
    }

    // zero-carry chunk recurrence of one sweep over the thread's P points
    // (masked points, bits of rm, restart it at zero)
    HW_DEV void chunk(const double u[P], double uL, const double c[P], double cR,
                      const double d[P], double dR, const double b[P], double y[P],
                      unsigned rm) const
    {
        double yy = 0.0;
#pragma unroll
        for (int k = 0; k < P; ++k) {
            const double ul = k ? u[k - 1] : uL;
            const double cr = k < P - 1 ? c[k + 1] : cR;
            const double dr = k < P - 1 ? d[k + 1] : dR;
            // c0 y = b - (cd/c0)(ul + dr) - (cx/c0)(u + d) - (cy/c0) cr on
            // rows scaled by c0 (6 FP64 operations per point)
            double pv = fma(beta, cr, b[k]);          // rows hold c0 x: no b / c0
            if constexpr (DG) pv = fma(-cds, ul + dr, pv);
            pv = fma(-cxs, u[k] + d[k], pv);
            yy = fma(beta, yy, pv);
            if (LSH && ((rm >> k) & 1u)) yy = 0.0;
            y[k] = yy;
        }
    }

    // the first sweep of a zero-start DOWN pass: the old rows (right and
    // below) are zero, so only the new row above and the left neighbour
    // remain (3 FP64 operations per point instead of 6)
    HW_DEV void chunk_zs(const double u[P], double uL, const double b[P], double y[P],
                         unsigned rm) const
    {
        double yy = 0.0;
#pragma unroll
        for (int k = 0; k < P; ++k) {
            const double ul = k ? u[k - 1] : uL;
            double pv = fma(-cxs, u[k], b[k]);
            if constexpr (DG) pv = fma(-cds, ul, pv);
            yy = fma(beta, yy, pv);
            if (LSH && ((rm >> k) & 1u)) yy = 0.0;
            y[k] = yy;
        }
    }

    HW_DEV double wscan(double s) const
    {
#pragma unroll
        for (int l = 0; l < LEV; ++l) s = fma(wl[l], __shfl_up_sync(0xffffffffu, s, 1 << l), s);
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
        const bool vo = !EDGE || (t >= 5 && t - 5 < n);

        cp_async_wait<2>();                              // own copies of step t-3 landed
        __syncthreads();                                 // (A) all copies, halos, output row visible
        if (vo) flush(t - 5);                            // row t-5, staged last step
        if (lane == 31) {
            X1R[Q] = HR[0 * HS + warp + 1];
            X2R[Q] = HR[1 * HS + warp + 1];
            if constexpr (DOWN) DR[Q] = HR[2 * HS + warp + 1];
        }
        if constexpr (CL > 1) {
            if (crank > 0 && tid == 0) mbar_expect(mb_tot, 24);          // this step's carry windows
            if (!lstrip && warp == NW - 1 && lane == 31) {
                if (t > 0) mbar_wait(mb_hr, Q);                          // the next strip's halos of step t-1
                X1R[Q] = box_hr[Q * 3 + 0];
                X2R[Q] = box_hr[Q * 3 + 1];
                if constexpr (DOWN) DR[Q] = box_hr[Q * 3 + 2];
                mbar_expect(mb_hr, DOWN ? 24 : 16);                      // ... and of this step
                if constexpr (DOWN) mbar_expect(mb_res, 8);
            }
        }

        // ---- phase A: chunk recurrences of the three sweeps ----
        double y[3][P], b[P + 1];
        const unsigned rm0 = rmask(t), rm1 = rmask(t - 2), rm2 = rmask(t - 4);
        constexpr int LBr = LB0 ^ PAR, LXr = LX0 ^ PAR ^ 1;   // UP parities of b(t), x0(t+1)
        double dn0[P + 1];
        if constexpr (DOWN && ZS) {
            load_b<LBr>(0, b);
            chunk_zs(X1[Q], X1L, b, y[0], rm0);
        } else {
            load_x0<Q, EDGE, LXr>(t + 1, sx, sc, dn0);
            load_b<LBr>(0, b);
            chunk(X1[Q], X1L, X0n, X0n[P], dn0, dn0[P], b, y[0], rm0);
        }
        load_b<LBr>(2, b);
        chunk(X2[Q], X2L, X1[PAR], X1R[PAR], X1[Q], X1R[Q], b, y[1], rm1);
        load_b<LBr>(4, b);
        chunk(X3, X3L, X2[PAR], X2R[PAR], X2[Q], X2R[Q], b, y[2], rm2);

        // residual of grid row t-6 from d(t-6), d(t-5)
        double R[P];
        if constexpr (DOWN) {
#pragma unroll
            for (int k = 0; k < P; ++k) {
                const double d6r = k < P - 1 ? D[PAR][k + 1] : DR[PAR];
                const double d5r = k < P - 1 ? D[Q][k + 1] : DR[Q];
                // the residual (differences of scaled rows: no c0 factor)
                R[k] = DG ? fma(beta, d6r, fma(-cxs, D[Q][k], -cds * d5r))
                          : fma(beta, d6r, -cxs * D[Q][k]);
            }
            if constexpr (LSH) {
                const unsigned rr = rmask(t - 6);
#pragma unroll
                for (int k = 0; k < P; ++k)
                    if ((rr >> k) & 1u) R[k] = 0.0;
            }
            if (lane == 0) HRes[warp] = R[0];
            if (CL > 1 && crank > 0 && tid == 0)
                st_async_f64(mapa_u32(smem_u32(box_res + PAR), crank - 1), R[0], mapa_u32(mb_res, crank - 1));
        }

        double A[3];
#pragma unroll
        for (int s = 0; s < 3; ++s) A[s] = wscan(y[s][P - 1]);
        if (lane == 31) {
#pragma unroll
            for (int s = 0; s < 3; ++s) tot[s * HS + warp + 1] = A[s];
            if (CL > 1 && !lstrip && warp == NW - 1) {   // the carry window into the next strip
                const unsigned rb = mapa_u32(smem_u32(box_tot + PAR * 3), crank + 1);
                const unsigned rm = mapa_u32(mb_tot, crank + 1);
#pragma unroll
                for (int s = 0; s < 3; ++s) st_async_f64(rb + 8u * s, A[s], rm);
            }
        }
        __syncthreads();                                 // (B) warp totals visible, output row
                                                         //     and the oldest ring slots free
        issue<PAR>(t);

        // ---- phase B: carries, new rows, halos ----
        double xn[3][P], cin[3];
        const bool inbox = CL > 1 && crank > 0 && warp == 0;    // the previous strip's windows
        if (inbox) mbar_wait(mb_tot, PAR);
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            const double prev = __shfl_up_sync(0xffffffffu, A[s], 1);
            const double tprev = inbox ? box_tot[PAR * 3 + s] : tot[s * HS + warp];
            cin[s] = fma(gl, tprev, lane ? prev : 0.0);
            const bool vs = s == 0 ? v1 : (s == 1 ? v2 : v3);
            const unsigned rms = s == 0 ? rm0 : (s == 1 ? rm1 : rm2);
#pragma unroll
            for (int k = 0; k < P; ++k) {
                const double v = fma(bp[k], cin[s], y[s][k]);
                xn[s][k] = (vs && !(k == P - 1 && last) && !(LSH && ((rms >> k) & 1u))) ? v : 0.0;
            }
            if (!vs) cin[s] = 0.0;
        }
        double dl[P];
        if constexpr (DOWN) {
#pragma unroll
            for (int k = 0; k < P; ++k) dl[k] = xn[2][k] - X2[PAR][k];
        }
        // stage the final values of row t-4 for next step's coalesced flush
#pragma unroll
        for (int h = 0; h < P / 2; ++h) {
            const int u = (P / 2) * tid + h;
            *reinterpret_cast<double2 *>(osm + ((u ^ ((u >> 3) & SWZ)) << 1)) =
                make_double2(xn[2][2 * h] * inv, xn[2][2 * h + 1] * inv);   // unscale
        }
#pragma unroll
        for (int k = 0; k < P; ++k) {
            X1[PAR][k] = xn[0][k];
            X2[PAR][k] = xn[1][k];
            X3[k] = xn[2][k];
            if constexpr (DOWN) D[PAR][k] = dl[k];
        }
        // left halo = the carry (the new value left of the chunk)
        X1L = cin[0];
        X2L = cin[1];
        X3L = cin[2];
        X1R[PAR] = __shfl_down_sync(0xffffffffu, xn[0][0], 1);
        X2R[PAR] = __shfl_down_sync(0xffffffffu, xn[1][0], 1);
        if constexpr (DOWN) DR[PAR] = __shfl_down_sync(0xffffffffu, dl[0], 1);
        if (lane == 0) {
            HR[0 * HS + warp] = xn[0][0];
            HR[1 * HS + warp] = xn[1][0];
            if constexpr (DOWN) HR[2 * HS + warp] = dl[0];
            if (CL > 1 && crank > 0 && warp == 0) {      // the previous strip's right halos
                const unsigned rb = mapa_u32(smem_u32(box_hr + PAR * 3), crank - 1);
                const unsigned rm = mapa_u32(mb_hr, crank - 1);
                st_async_f64(rb, xn[0][0], rm);
                st_async_f64(rb + 8u, xn[1][0], rm);
                if constexpr (DOWN) st_async_f64(rb + 16u, dl[0], rm);
            }
        }
        if constexpr (!(DOWN && ZS)) {
#pragma unroll
            for (int e = 0; e <= P; ++e) X0n[e] = dn0[e];
        }

        // ---- restriction of residual row r = t-6 (parity PAR) ----
        // coarse column J = (P/2) t + q collects fine columns 2J, 2J+1, 2J+2
        if constexpr (DOWN) {
            double rbox = 0.0;                           // CL > 1: consumed every step (phases stay in step)
            const bool rin = CL > 1 && !lstrip && warp == NW - 1 && lane == 31;
            if (rin) {
                mbar_wait(mb_res, PAR);
                rbox = box_res[PAR];
            }
            if (vr) {
                double RR = __shfl_down_sync(0xffffffffu, R[0], 1);
                if (lane == 31) RR = rin ? rbox : HRes[warp + 1];
                const int r = t - 6;
#pragma unroll
                for (int q = 0; q < P / 2; ++q) {
                    const double r0 = R[2 * q], r1 = R[2 * q + 1];
                    const double r2 = 2 * q + 2 < P ? R[2 * q + 2] : RR;
                    if constexpr (PAR) {                 // centre row of coarse (r-1)/2
                        acc[q] += fma(0.5, r0 + r2, r1);
                    } else {                             // bottom of r/2-1, top of r/2
                        if (r >= 2 && (q < P / 2 - 1 || !last))
                            Bcg[(int64_t)(r / 2 - 1) * m + q] = acc[q] + 0.5 * (r1 + r2);
                        acc[q] = 0.5 * (r0 + r1);
                    }
                }
            }
        }
        advance();
        if (PAR) sc = sc + 1 == SM::NCR ? 0 : sc + 1;
    }

    // the step barriers: CTA-wide, or cluster-wide when the row is split
    HW_DEV void sync_pair() const
    {
        if constexpr (CL > 1) cluster_sync_all();
        else __syncthreads();
    }

    HW_DEV void advance()
    {
        sb = sb + 1 == SM::NB ? 0 : sb + 1;
        sx = sx + 1 == SM::NX ? 0 : sx + 1;
    }

    HW_DEV void run()
    {
        // prologue: x0 row 0 (+ coarse rows -1, 0), then the groups steps
        // -3..-1 would have issued
        if constexpr (CL > 1) {                          // zeroed slots, then the mbarriers
            __syncthreads();
            if (threadIdx.x == 0) {
                mbar_init(mb_tot, 1);
                mbar_init(mb_hr, 1);
                mbar_init(mb_res, 1);
                asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
            }
        }
        sync_pair();                                     // zeroed slots before any copy lands
                                                         // (or any message of the other strip)
        if constexpr (!(DOWN && ZS)) {
            stage_row<true, LX0>(x0sm, Xg, 0);
            if constexpr (!DOWN) {
                stage_coarse(-1, SM::NCR - 1);
                stage_coarse(0, 0);
            }
            cp_async_commit();
        }
        issue<1>(-3);
        advance();
        sc = SM::NCR - 1;                                // coarse slot of row floor(-2/2) = -1
        issue<0>(-2);                                    // (stages coarse row 1)
        advance();
        if constexpr (!(DOWN && ZS)) {
            cp_async_wait<2>();
            __syncthreads();
            load_x0<0, true, LX0>(0, 0, SM::NCR - 1, X0n);
            __syncthreads();                             // x0(3) reuses x0(0)'s slot
        }
        issue<1>(-1);
        advance();
        sc = 0;
        constexpr int nsteps = DOWN ? n + 6 : n + 5;     // the last flush is step n+4
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
        if constexpr (CL > 1) {                          // the last halo message lands before exit
            if (!lstrip && warp == NW - 1 && lane == 31) mbar_wait(mb_hr, (nsteps - 1) & 1);
        }
        cp_async_wait<0>();
    }
};

template <int P, int NT, bool DOWN, bool ZS, int LB, int LX, bool LSH, bool DG, int CL>
HW_DEV void run_pass(const MgStreamArgs &a, double *sm)
{
    RegPass<P, NT, DOWN, ZS, LB, LX, LSH, DG, CL> p(a, sm);
    p.run();
    p.finish_dot(a);
    if constexpr (CL > 1) cluster_sync_all();            // no strip exits under the other's stores
}

template <int P, int NT, bool DOWN, bool ZS, int MINB, bool LSH, bool DG, int CL>
__global__ void __launch_bounds__(NT, MINB) mg2d_reg(MgStreamArgs a)
{
    extern __shared__ __align__(16) double sm[];
    if constexpr (DOWN) {
        run_pass<P, NT, DOWN, ZS, 0, 0, LSH, DG, CL>(a, sm);
    } else {
        // UP: layout parity of grid row 0 (stage_row) = 1 when local column 0
        // (global row n-1, column n-1) sits at a 16-byte boundary (the strips
        // of a split row start an even number of columns apart: same parity)
        constexpr int n = CL * P * NT - 1;
        const int64_t row = blockIdx.x / CL;
        auto parity = [&](const double *base, int64_t ld) -> int {
            const double *p0 = base + row * ld + (int64_t)(n - 1) * n + (n - 1);
            return 1 - (int)((reinterpret_cast<uintptr_t>(p0) >> 3) & 1);
        };
        const int lb = parity(a.B, a.ldB), lx = parity(a.X, a.ldX);
        if (lb) {
            if (lx) run_pass<P, NT, DOWN, ZS, 1, 1, LSH, DG, CL>(a, sm);
            else run_pass<P, NT, DOWN, ZS, 1, 0, LSH, DG, CL>(a, sm);
        } else {
            if (lx) run_pass<P, NT, DOWN, ZS, 0, 1, LSH, DG, CL>(a, sm);
            else run_pass<P, NT, DOWN, ZS, 0, 0, LSH, DG, CL>(a, sm);
        }
    }
}

template <int P, int NT, bool DOWN, bool ZS, int MINB, int CL>
cudaError_t launch_reg_t(const MgStreamArgs &a, int64_t rows, cudaStream_t st)
{
    const size_t smem = RegSmem<P, NT, DOWN, ZS>::total * sizeof(double);
    auto k = a.lshape ? mg2d_reg<P, NT, DOWN, ZS, MINB, true, true, CL>
                      : (a.diag ? mg2d_reg<P, NT, DOWN, ZS, MINB, false, true, CL>
                                : mg2d_reg<P, NT, DOWN, ZS, MINB, false, false, CL>);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if constexpr (CL == 1) {
        k<<<(unsigned)rows, NT, smem, st>>>(a);
        return cudaGetLastError();
    } else {                                             // one cluster of CL strips per temporal row
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(rows * CL), 1, 1);
        cfg.blockDim = dim3(NT, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, k, a);
    }
}

template <int P, int NT, int MINB, int CL = 1>
cudaError_t launch_reg_n(const MgStreamArgs &a, bool down, int64_t rows, cudaStream_t st)
{
    if (!down) return launch_reg_t<P, NT, false, false, MINB, CL>(a, rows, st);
    return a.zero_start ? launch_reg_t<P, NT, true, true, MINB, CL>(a, rows, st)
                        : launch_reg_t<P, NT, true, false, MINB, CL>(a, rows, st);
}

}  // namespace

// Thread shape per level.  The default shapes (P = 8 points per thread) are
// the HBM-efficient ones for batches of a wave or more.  A short time axis
// leaves each SM with one or two warps of a level <= 9 pass, each issuing a
// whole grid row's three sweeps alone (issue- and latency-bound); the WIDE
// shapes split the row over 2x the threads (P = 4 / 2, the same 32-column
// carry window, results equal up to rounding).  Measured
// (scripts/mg_wide_sweep.py, profiles/r02/mg_wide_sweep.txt): a gain while
// rows x default warps per row <= ~2 per SM (K = 8: -15 % at 129 rows, -11 %
// at 257; K = 10: -6 % at 136 rows), a loss above; level 10 only for the
// L-shaped variant at <= 1 row per SM (its P = 8 DOWN pass spills).  The
// choice (a.wide) is made once per context from N_t by hwg_create, so results
// never depend on a call's batch size.  HWG_REG_WIDE=<bitmask of levels>
// overrides it per launch (A/B and the parity tests of both shapes).
static int wide_mask(const MgStreamArgs &a)
{
    if (const char *ev = getenv("HWG_REG_WIDE")) return atoi(ev);
    return a.wide;
}

cudaError_t mg2d_reg_launch(const MgStreamArgs &a, bool down, int64_t rows, cudaStream_t st)
{
    const int wide = wide_mask(a);
    switch (a.n) {
    case 63: return launch_reg_n<2, 32, 1>(a, down, rows, st);
    case 127:
        if (wide & (1 << 7)) return launch_reg_n<2, 64, 1>(a, down, rows, st);
        return launch_reg_n<4, 32, 1>(a, down, rows, st);
    case 255:
        if (wide & (1 << 8)) return launch_reg_n<4, 64, 1>(a, down, rows, st);
        if (wide & (1 << 18)) return launch_reg_n<2, 128, 1>(a, down, rows, st);
        return launch_reg_n<8, 32, 1>(a, down, rows, st);
    case 511:
        if (wide & (1 << 9)) return launch_reg_n<4, 128, 1>(a, down, rows, st);
        return launch_reg_n<8, 64, 1>(a, down, rows, st);
    case 1023:
        // HWG_MG_REG=4: P = 4 for both passes; =5: P = 4 for UP only (A/B)
        if (a.reg_ok == 2 || (a.reg_ok == 3 && !down) || (wide & (1 << 10)))
            return launch_reg_n<4, 256, 1>(a, down, rows, st);
        return launch_reg_n<8, 128, 2>(a, down, rows, st);
    case 2047:
        // HWG_REG_CLUSTER=1 (A/B, bit-identical): the row as two 128-thread
        // strips on a CTA pair (RegPass CL = 2).  Measured slower
        // (profiles/r02/mg_cluster_strips.txt): a row still needs 256 x 255
        // registers, so an SM pair holds two rows either way, and the
        // per-step messages cost what the 8-warp barriers did
        if (const char *ev = getenv("HWG_REG_CLUSTER"))
            if (ev[0] == '1') return launch_reg_n<8, 128, 2, 2>(a, down, rows, st);
        if (wide & (1 << 11)) return launch_reg_n<4, 512, 1>(a, down, rows, st);
        return launch_reg_n<8, 256, 1>(a, down, rows, st);
    default: return cudaErrorNotSupported;
    }
}

}  // namespace hw
