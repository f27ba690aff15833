// hw_wavelet.cu -- three-point wavelet transform in time, W_t (x) Id_x.
//
// Restates WaveletTransform._apply_stages (/root/reference/pkg/src/heatwave/
// wavelet.py:114-137) with the two-scale matrices M_j = [P_j | Q_j] of
// wavelet.py:56-76 written out in closed form.  Every
// stage is one launch over (stage rows) x N_x with coalesced access along
// the spatial axis; each output value accumulates the same products in the
// same (CSR column) order as the reference's temporal_apply, without FMA
// contraction, so the transform is bit-identical to the reference.  A
// thread owns one column and a contiguous run of row pairs, so consecutive
// outputs share their inputs through registers and every input row is
// loaded once per thread.
//
// Synthesis (W): stage j maps the coarse nodal prefix c (rows 0..2^(j-1))
// and the level-j wavelet coefficients d (rows 2^(j-1)+1..2^j, read from the
// untouched input) to the fine nodal prefix (rows 0..2^j).  The ping-pong
// buffer choice puts stage J into the output; no copy-back pass is needed.
// Transpose (W^T): stage j reads the fine prefix and writes its wavelet
// part d' straight into the output rows, its coarse part c' into scratch.
#include "hw_common.cuh"
#include "hw_internal.cuh"

#include <algorithm>
#include <cstdlib>

namespace hw {

// a_k = -1 if k == 0 else -1/2 ; b_k = -1 if k == nw-1 else -1/2
// (wavelet.py:70-71); the stored CSR value is s * a_k, s = 2^(j/2).
__device__ __forceinline__ double qa(double s, int k) { return s * (k == 0 ? -1.0 : -0.5); }
__device__ __forceinline__ double qb(double s, int k, int nw) { return s * (k == nw - 1 ? -1.0 : -0.5); }

// ---------------------------------------------------------------------------
// Full-prefix stage kernels of the single-GPU transform: each thread owns
// one column and a contiguous run of QP row pairs (per-element kernels that
// reload every input 2-3 times and launch one CTA per output row took 1.9x
// as long at J = 10).
// ---------------------------------------------------------------------------
constexpr int kWavQP = 16, kWavBS = 256;

// L-shaped domain on the embedded grid (side mn, removed quadrant a, b >= lm):
// those columns are zero in and out, so they are written without being read
struct ColMask {
    int mn, lm;                       // mn = 0: no mask
    HW_DEV bool operator()(int64_t i) const
    {
        return mn > 0 && (int)(i / mn) >= lm && (int)(i % mn) >= lm;
    }
};

// synthesis stage j over the full prefix: pair q = fine nodes 2q, 2q+1
__global__ void __launch_bounds__(kWavBS) wav_syn_pairs(const double *__restrict__ C,
                                                        const double *__restrict__ Dm,
                                                        double *__restrict__ Y, int j, double s,
                                                        int64_t nx, ColMask msk)
{
    const int nw = 1 << (j - 1);
    const int64_t i = (int64_t)blockIdx.x * kWavBS + threadIdx.x;
    if (i >= nx) return;
    const int q0 = blockIdx.y * kWavQP;
    const int q1 = min(q0 + kWavQP, nw + 1);
    if (msk(i)) {
        for (int q = q0; q < q1; ++q) {
            if (q < nw) Y[(int64_t)(2 * q + 1) * nx + i] = 0.0;
            Y[(int64_t)(2 * q) * nx + i] = 0.0;
        }
        return;
    }
    double cq = C[(int64_t)q0 * nx + i];
    double dm = q0 >= 1 ? Dm[(int64_t)(q0 - 1) * nx + i] : 0.0;   // d[q-1]
#pragma unroll 4
    for (int q = q0; q < q1; ++q) {
        double acc = cq;
        if (q >= 1) acc = add_rn(acc, mul_rn(qb(s, q - 1, nw), dm));
        if (q < nw) {
            const double dq = Dm[(int64_t)q * nx + i];
            const double cn = C[(int64_t)(q + 1) * nx + i];
            acc = add_rn(acc, mul_rn(qa(s, q), dq));
            double od = mul_rn(0.5, cq);
            od = add_rn(od, mul_rn(0.5, cn));
            od = add_rn(od, mul_rn(s, dq));
            Y[(int64_t)(2 * q + 1) * nx + i] = od;
            cq = cn;
            dm = dq;
        }
        Y[(int64_t)(2 * q) * nx + i] = acc;
    }
}

// transposed stage j: pair r = coarse r (rows 2r-1..2r+1) and wavelet r
// (rows 2r..2r+2)
__global__ void __launch_bounds__(kWavBS) wav_ana_pairs(const double *__restrict__ X,
                                                        double *__restrict__ Cout,
                                                        double *__restrict__ Dout, int j,
                                                        double s, int64_t nx, ColMask msk)
{
    const int nw = 1 << (j - 1), nf = (1 << j) + 1;
    const int64_t i = (int64_t)blockIdx.x * kWavBS + threadIdx.x;
    if (i >= nx) return;
    const int r0 = blockIdx.y * kWavQP;
    const int r1 = min(r0 + kWavQP, nw + 1);
    if (msk(i)) {
        for (int r = r0; r < r1; ++r) {
            if (2 * r + 1 < nf) Dout[(int64_t)r * nx + i] = 0.0;
            Cout[(int64_t)r * nx + i] = 0.0;
        }
        return;
    }
    double xm = r0 >= 1 ? X[(int64_t)(2 * r0 - 1) * nx + i] : 0.0;   // x[2r-1]
    double x0 = X[(int64_t)(2 * r0) * nx + i];                      // x[2r]
#pragma unroll 4
    for (int r = r0; r < r1; ++r) {
        double acc;
        if (r >= 1) {
            acc = mul_rn(0.5, xm);
            acc = add_rn(acc, x0);
        } else {
            acc = x0;
        }
        if (2 * r + 1 < nf) {
            const double x1 = X[(int64_t)(2 * r + 1) * nx + i];
            const double x2 = X[(int64_t)(2 * r + 2) * nx + i];
            acc = add_rn(acc, mul_rn(0.5, x1));
            double dd = mul_rn(qa(s, r), x0);
            dd = add_rn(dd, mul_rn(s, x1));
            dd = add_rn(dd, mul_rn(qb(s, r, nw), x2));
            Dout[(int64_t)r * nx + i] = dd;
            xm = x1;
            x0 = x2;
        }
        Cout[(int64_t)r * nx + i] = acc;
    }
}

// ---------------------------------------------------------------------------
// Two stages in one pass (the top stages carry nearly all of a transform's
// bytes: stage J moves 2^J + 1 rows, J-1 half that).  Synthesis stages j and
// j+1: a thread computes a run of stage-j outputs F in registers and emits
// stage j+1's outputs as soon as their two F inputs exist, so F never goes
// through HBM (reads 4R + 4 and writes 4R rows per run of R stage-j pairs,
// instead of 6R + 4 and 6R).  Every output is the same sum in the same order
// as the single-stage kernels: bit-identical.
// ---------------------------------------------------------------------------
constexpr int kWavQP2 = 8;

__global__ void __launch_bounds__(kWavBS) wav_syn_pairs2(const double *__restrict__ C,
                                                         const double *__restrict__ Dm,
                                                         const double *__restrict__ Dm2,
                                                         double *__restrict__ Y, int j, double s,
                                                         double s2, int64_t nx, ColMask msk)
{
    const int nw = 1 << (j - 1), nw2 = 1 << j;          // wavelets of levels j, j+1
    const int64_t i = (int64_t)blockIdx.x * kWavBS + threadIdx.x;
    if (i >= nx) return;
    const int q0 = blockIdx.y * kWavQP2;
    const int q1 = min(q0 + kWavQP2, nw + 1);            // stage-j pairs [q0, q1)
    const int f0 = 2 * q0, f1 = min(2 * q1, 2 * nw + 1); // F rows this thread emits G for
    if (msk(i)) {
        for (int f = f0; f < f1; ++f) {
            if (f < nw2) Y[(int64_t)(2 * f + 1) * nx + i] = 0.0;
            Y[(int64_t)(2 * f) * nx + i] = 0.0;
        }
        return;
    }
    // every row the tile reads, loaded up front (37 independent loads in flight
    // per thread; read one by one inside the dependent recurrence below, the
    // kernel ran at 4.6 TB/s): c[u] = C[q0 + u], d1[u] = D_j[q0 - 1 + u],
    // d2[v] = D_{j+1}[f0 - 1 + v]; rows that do not exist are never used
    double c[kWavQP2 + 1], d1[kWavQP2 + 2], d2[2 * kWavQP2 + 2];
#pragma unroll
    for (int u = 0; u <= kWavQP2; ++u) c[u] = q0 + u <= nw ? C[(int64_t)(q0 + u) * nx + i] : 0.0;
#pragma unroll
    for (int u = 0; u <= kWavQP2 + 1; ++u) {
        const int k = q0 - 1 + u;
        d1[u] = (k >= 0 && k < nw) ? Dm[(int64_t)k * nx + i] : 0.0;
    }
#pragma unroll
    for (int v = 0; v <= 2 * kWavQP2 + 1; ++v) {
        const int k = f0 - 1 + v;
        d2[v] = (k >= 0 && k < nw2) ? Dm2[(int64_t)k * nx + i] : 0.0;
    }
    // F[2q] and F[2q+1] of stage j (wav_syn_pairs' arithmetic)
    auto Feven = [&](int q, double cq, double dm, double dq) {
        double acc = cq;
        if (q >= 1) acc = add_rn(acc, mul_rn(qb(s, q - 1, nw), dm));
        if (q < nw) acc = add_rn(acc, mul_rn(qa(s, q), dq));
        return acc;
    };
    auto Fodd = [&](double cq, double cn, double dq) {
        double od = mul_rn(0.5, cq);
        od = add_rn(od, mul_rn(0.5, cn));
        return add_rn(od, mul_rn(s, dq));
    };
    // G[2f], G[2f+1] of stage j+1 from F[f], F[f+1] (F[f+1] unused if f == nw2)
    double gdm = d2[0];                                   // d2[f-1]
    auto emit = [&](int f, double dq, double Ff, double Fn) {   // dq = D_{j+1}[f]
        double acc = Ff;
        if (f >= 1) acc = add_rn(acc, mul_rn(qb(s2, f - 1, nw2), gdm));
        if (f < nw2) {
            acc = add_rn(acc, mul_rn(qa(s2, f), dq));
            double od = mul_rn(0.5, Ff);
            od = add_rn(od, mul_rn(0.5, Fn));
            od = add_rn(od, mul_rn(s2, dq));
            Y[(int64_t)(2 * f + 1) * nx + i] = od;
            gdm = dq;
        }
        Y[(int64_t)(2 * f) * nx + i] = acc;
    };
    double cq = c[0];
    double dm = d1[0];
    double Fprev = 0.0;                                   // F[f-1], pending emission
    bool pending = false;
#pragma unroll
    for (int u = 0; u < kWavQP2; ++u) {
        const int q = q0 + u;
        if (q >= q1) break;
        const double dq = d1[u + 1];                      // D_j[q] (0 past the last wavelet)
        const double fe = Feven(q, cq, dm, dq);           // F[2q]
        if (pending) emit(2 * q - 1, d2[2 * u], Fprev, fe);
        if (q < nw) {
            const double cn = c[u + 1];
            const double fo = Fodd(cq, cn, dq);           // F[2q+1]
            emit(2 * q, d2[2 * u + 1], fe, fo);
            Fprev = fo;
            pending = true;
            cq = cn;
            dm = dq;
        } else {
            emit(2 * q, d2[2 * u + 1], fe, 0.0);          // F[2 nw] = the last fine node
            pending = false;
        }
    }
    if (pending) {                                        // F[2 q1 - 1] needs F[2 q1]; pending
        const double dq = d1[kWavQP2 + 1];                // implies q1 = q0 + kWavQP2 <= nw
        emit(2 * q1 - 1, d2[2 * kWavQP2], Fprev, Feven(q1, cq, dm, dq));
    }
}

// transposed stages j+1 and j in one pass: a thread owns stage-j outputs
// r in [r0, r1) (coarse C and wavelet d_j), computes the stage-(j+1) coarse
// values F it needs from the fine rows X in registers, and writes the
// stage-(j+1) wavelets d_{j+1} of F rows [2 r0, 2 r1) (wav_ana_pairs'
// arithmetic throughout: bit-identical)
__global__ void __launch_bounds__(kWavBS) wav_ana_pairs2(const double *__restrict__ X,
                                                         double *__restrict__ Cout,
                                                         double *__restrict__ Dout,
                                                         double *__restrict__ Dout2, int j,
                                                         double s, double s2, int64_t nx,
                                                         ColMask msk)
{
    const int nw = 1 << (j - 1), nf = (1 << j) + 1;      // stage j: fine prefix F of nf rows
    const int nw2 = 1 << j, nf2 = (1 << (j + 1)) + 1;    // stage j+1: fine prefix X of nf2 rows
    const int64_t i = (int64_t)blockIdx.x * kWavBS + threadIdx.x;
    if (i >= nx) return;
    const int r0 = blockIdx.y * kWavQP2;
    const int r1 = min(r0 + kWavQP2, nw + 1);
    const int f0 = 2 * r0, f1 = min(2 * r1, nf);         // d_{j+1} rows this thread writes
    if (msk(i)) {
        for (int f = f0; f < f1; ++f)
            if (2 * f + 1 < nf2) Dout2[(int64_t)f * nx + i] = 0.0;
        for (int r = r0; r < r1; ++r) {
            if (2 * r + 1 < nf) Dout[(int64_t)r * nx + i] = 0.0;
            Cout[(int64_t)r * nx + i] = 0.0;
        }
        return;
    }
    auto Xr = [&](int k) { return X[(int64_t)k * nx + i]; };
    // stage j+1 at F row f: coarse F[f] and (f < nw2, if write) wavelet
    // d2[f], from x[2f-1 .. 2f+2] (wav_ana_pairs' arithmetic)
    auto stage2 = [&](int f, double xm, double x0, double x1, double x2, bool write) {
        double acc;
        if (f >= 1) {
            acc = mul_rn(0.5, xm);
            acc = add_rn(acc, x0);
        } else {
            acc = x0;
        }
        if (2 * f + 1 < nf2) {
            acc = add_rn(acc, mul_rn(0.5, x1));
            if (write) {
                double dd = mul_rn(qa(s2, f), x0);
                dd = add_rn(dd, mul_rn(s2, x1));
                dd = add_rn(dd, mul_rn(qb(s2, f, nw2), x2));
                Dout2[(int64_t)f * nx + i] = dd;
            }
        }
        return acc;
    };
    // F[f] for f in [fs, fe], fs = 2 r0 - 1 (F[2 r0 - 1] is recomputed; its
    // wavelet belongs to the previous run), each x row read once
    constexpr int NFV = 2 * kWavQP2 + 2;
    const int fs = 2 * r0 - 1;
    const int fb = fs < 0 ? 0 : fs;
    const int fe = min(2 * r1, nw2);
    double F[NFV];
    // x rows 2 fs - 1 .. 2 (fs + NFV - 1) + 2, all loaded up front (independent
    // loads in flight instead of two per step of the loop below)
    double xr[2 * NFV + 2];
#pragma unroll
    for (int v = 0; v < 2 * NFV + 2; ++v) {
        const int k = 2 * fs - 1 + v;
        xr[v] = (k >= (fb >= 1 ? 2 * fb - 1 : 0) && k < nf2 && k <= 2 * fe + 2) ? Xr(k) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < NFV; ++t) {
        const int f = fs + t;
        F[t] = 0.0;
        if (f < fb || f > fe) continue;
        F[t] = stage2(f, xr[2 * t], xr[2 * t + 1], xr[2 * t + 2], xr[2 * t + 3], f >= f0 && f < f1);
    }
    // stage j (wav_ana_pairs on F): C[r], d_j[r]
#pragma unroll
    for (int u = 0; u < kWavQP2; ++u) {
        const int r = r0 + u;
        if (r >= r1) break;
        const int t = 2 * u + 1;                          // F[2r] = F[t]
        double acc;
        if (r >= 1) {
            acc = mul_rn(0.5, F[t - 1]);
            acc = add_rn(acc, F[t]);
        } else {
            acc = F[t];
        }
        if (2 * r + 1 < nf) {
            acc = add_rn(acc, mul_rn(0.5, F[t + 1]));
            double dd = mul_rn(qa(s, r), F[t]);
            dd = add_rn(dd, mul_rn(s, F[t + 1]));
            dd = add_rn(dd, mul_rn(qb(s, r, nw), F[t + 2]));
            Dout[(int64_t)r * nx + i] = dd;
        }
        Cout[(int64_t)r * nx + i] = acc;
    }
}

static dim3 pair_grid(int pairs, int64_t nx)
{
    return dim3((unsigned)((nx + kWavBS - 1) / kWavBS), (unsigned)((pairs + kWavQP - 1) / kWavQP));
}

// ---- general windows (the time-slab entries hwg_syn_stage / hwg_ana_stage):
// the same per-thread runs of pairs, every load guarded by what the in-range
// outputs need, register carries tracked with validity flags.

// Y[f - f0] <- (M_j [c ; d])[f], f in [f0, f0 + nf); C[i - c0], Dm[k - d0]
__global__ void __launch_bounds__(kWavBS) wav_syn_window(const double *__restrict__ C, int64_t c0,
                                                         const double *__restrict__ Dm, int64_t d0,
                                                         const double *__restrict__ Dh,
                                                         double *__restrict__ Y, int64_t f0,
                                                         int64_t nf, int j, double s, int64_t nx)
{
    const int nw = 1 << (j - 1);
    const int64_t i = (int64_t)blockIdx.x * kWavBS + threadIdx.x;
    if (i >= nx) return;
    const int64_t qlo = f0 >> 1, qhi = (f0 + nf - 1) >> 1;       // pairs touched
    const int64_t q0 = qlo + (int64_t)blockIdx.y * kWavQP;
    const int64_t q1 = q0 + kWavQP - 1 < qhi ? q0 + kWavQP - 1 : qhi;
    auto cr = [&](int64_t q) { return C[(q - c0) * nx + i]; };
    auto dr = [&](int64_t k) { return (Dh && k < d0) ? Dh[i] : Dm[(k - d0) * nx + i]; };
    double cq = 0.0, dm = 0.0;
    bool have_c = false, have_d = false;
    for (int64_t q = q0; q <= q1; ++q) {
        const bool ne = 2 * q >= f0 && 2 * q < f0 + nf;
        const bool no = q < nw && 2 * q + 1 >= f0 && 2 * q + 1 < f0 + nf;
        if (!have_c) cq = cr(q);
        if (ne && q >= 1 && !have_d) dm = dr(q - 1);
        const bool ldq = (ne && q < nw) || no;
        const double dq = ldq ? dr(q) : 0.0;
        if (ne) {
            double acc = cq;
            if (q >= 1) acc = add_rn(acc, mul_rn(qb(s, (int)q - 1, nw), dm));
            if (q < nw) acc = add_rn(acc, mul_rn(qa(s, (int)q), dq));
            Y[(2 * q - f0) * nx + i] = acc;
        }
        if (no) {
            const double cn = cr(q + 1);
            double od = mul_rn(0.5, cq);
            od = add_rn(od, mul_rn(0.5, cn));
            od = add_rn(od, mul_rn(s, dq));
            Y[(2 * q + 1 - f0) * nx + i] = od;
            cq = cn;
        }
        have_c = no;
        dm = dq;
        have_d = ldq;
    }
}

// Cout[r - c0] = (P_j^T x)[r], r in [c0, c0 + nc); Dout[k - d0] = (Q_j^T x)[k],
// k in [d0, d0 + nd); X[f - x0] = fine node f
__global__ void __launch_bounds__(kWavBS) wav_ana_window(const double *__restrict__ X, int64_t x0,
                                                         double *__restrict__ Cout, int64_t c0,
                                                         int64_t nc, double *__restrict__ Dout,
                                                         int64_t d0, int64_t nd, int j, double s,
                                                         int64_t nx)
{
    const int nw = 1 << (j - 1), nf = (1 << j) + 1;
    const int64_t i = (int64_t)blockIdx.x * kWavBS + threadIdx.x;
    if (i >= nx) return;
    const int64_t lo = nc && nd ? (c0 < d0 ? c0 : d0) : (nc ? c0 : d0);
    const int64_t hi = nc && nd ? (c0 + nc > d0 + nd ? c0 + nc : d0 + nd) : (nc ? c0 + nc : d0 + nd);
    const int64_t r0 = lo + (int64_t)blockIdx.y * kWavQP;
    const int64_t r1 = r0 + kWavQP < hi ? r0 + kWavQP : hi;
    auto xr = [&](int64_t f) { return X[(f - x0) * nx + i]; };
    double xm = 0.0, xa = 0.0;                          // x[2r-1], x[2r]
    bool have_m = false, have_a = false;
    for (int64_t r = r0; r < r1; ++r) {
        const bool cin = r >= c0 && r < c0 + nc;
        const bool din = r >= d0 && r < d0 + nd;
        if (!have_a) xa = xr(2 * r);
        const bool l1 = (cin && 2 * r + 1 < nf) || din;
        const double x1 = l1 ? xr(2 * r + 1) : 0.0;
        if (cin) {
            double acc;
            if (r >= 1) {
                if (!have_m) xm = xr(2 * r - 1);
                acc = mul_rn(0.5, xm);
                acc = add_rn(acc, xa);
            } else {
                acc = xa;
            }
            if (2 * r + 1 < nf) acc = add_rn(acc, mul_rn(0.5, x1));
            Cout[(r - c0) * nx + i] = acc;
        }
        double x2 = 0.0;
        if (din) {
            x2 = xr(2 * r + 2);
            double dd = mul_rn(qa(s, (int)r), xa);
            dd = add_rn(dd, mul_rn(s, x1));
            dd = add_rn(dd, mul_rn(qb(s, (int)r, nw), x2));
            Dout[(r - d0) * nx + i] = dd;
        }
        xm = x1;
        have_m = l1;
        xa = x2;
        have_a = din;
    }
}

cudaError_t launch_syn_stage(int j, double s, const double *C, int64_t c0, const double *Dm,
                             int64_t d0, const double *Dh, double *Y, int64_t f0, int64_t nf,
                             int64_t nx, cudaStream_t st)
{
    if (nf <= 0) return cudaSuccess;
    const int64_t pairs = ((f0 + nf - 1) >> 1) - (f0 >> 1) + 1;
    wav_syn_window<<<pair_grid((int)pairs, nx), kWavBS, 0, st>>>(C, c0, Dm, d0, Dh, Y, f0, nf, j, s,
                                                                 nx);
    return cudaGetLastError();
}

cudaError_t launch_ana_stage(int j, double s, const double *X, int64_t x0, double *C, int64_t c0,
                             int64_t nc, double *Dm, int64_t d0, int64_t nd, int64_t nx,
                             cudaStream_t st)
{
    if (nc + nd <= 0) return cudaSuccess;
    const int64_t lo = nc && nd ? std::min(c0, d0) : (nc ? c0 : d0);
    const int64_t hi = nc && nd ? std::max(c0 + nc, d0 + nd) : (nc ? c0 + nc : d0 + nd);
    wav_ana_window<<<pair_grid((int)(hi - lo), nx), kWavBS, 0, st>>>(X, x0, C, c0, nc, Dm, d0, nd,
                                                                     j, s, nx);
    return cudaGetLastError();
}

// A/B switch (HWG_WAV_FUSE=0: one launch per stage)
static bool wavelet_fuse_enabled()
{
    static int on = -1;
    if (on < 0) {
        const char *ev = getenv("HWG_WAV_FUSE");
        on = (ev && ev[0] == '0') ? 0 : 1;
    }
    return on != 0;
}

// Y = W X (transpose = 0) or W^T X (transpose = 1).  S1 (and S2 for the
// transpose) are scratch arrays with at least 2^(J-1)+1 rows.
cudaError_t wavelet_apply(const double *X, double *Y, double *S1, double *S2, int J,
                          const double *scale, int64_t nt, int64_t nx, bool transpose,
                          cudaStream_t st, int64_t *launches, int mask_n, int mask_lm)
{
    const ColMask msk{mask_n, mask_lm};
    if (J == 0) {
        return cudaMemcpyAsync(Y, X, (size_t)(nt * nx) * sizeof(double),
                               cudaMemcpyDeviceToDevice, st);
    }
    // the top two stages run fused (wav_*_pairs2); J = 1 has one stage
    const bool fuse = J >= 2 && wavelet_fuse_enabled();
    if (!transpose) {
        const double *src = X;
        const int jlast = fuse ? J - 2 : J;              // single stages 1..jlast
        for (int j = 1; j <= jlast; ++j) {
            double *dst = ((jlast - j) % 2 == 0) ? (fuse ? S1 : Y) : (fuse ? Y : S1);
            if (!fuse) dst = ((J - j) % 2 == 0) ? Y : S1;
            const int64_t nc = (1LL << (j - 1)) + 1;
            wav_syn_pairs<<<pair_grid((1 << (j - 1)) + 1, nx), kWavBS, 0, st>>>(
                src, X + nc * nx, dst, j, scale[j - 1], nx, msk);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
            ++*launches;
            src = dst;
        }
        if (fuse) {
            const int j = J - 1;                          // stages J-1 and J
            const int64_t nc = (1LL << (j - 1)) + 1, nc2 = (1LL << j) + 1;
            const dim3 g((unsigned)((nx + kWavBS - 1) / kWavBS),
                         (unsigned)(((1 << (j - 1)) + 1 + kWavQP2 - 1) / kWavQP2));
            wav_syn_pairs2<<<g, kWavBS, 0, st>>>(j == 1 ? X : src, X + nc * nx, X + nc2 * nx, Y, j,
                                                 scale[j - 1], scale[j], nx, msk);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
            ++*launches;
        }
    } else {
        const double *src = X;
        int jtop = J;
        if (fuse) {                                       // stages J and J-1
            const int j = J - 1;
            const int64_t nc = (1LL << (j - 1)) + 1, nc2 = (1LL << j) + 1;
            double *cdst = (j == 1) ? Y : S1;
            const dim3 g((unsigned)((nx + kWavBS - 1) / kWavBS),
                         (unsigned)(((1 << (j - 1)) + 1 + kWavQP2 - 1) / kWavQP2));
            wav_ana_pairs2<<<g, kWavBS, 0, st>>>(X, cdst, Y + nc * nx, Y + nc2 * nx, j,
                                                 scale[j - 1], scale[j], nx, msk);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
            ++*launches;
            src = cdst;
            jtop = J - 2;
        }
        for (int j = jtop; j >= 1; --j) {
            double *cdst = (j == 1) ? Y : (((jtop - j) % 2 == 0) ? (fuse ? S2 : S1) : (fuse ? S1 : S2));
            const int64_t nc = (1LL << (j - 1)) + 1;
            wav_ana_pairs<<<pair_grid((1 << (j - 1)) + 1, nx), kWavBS, 0, st>>>(
                src, cdst, Y + nc * nx, j, scale[j - 1], nx, msk);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
            ++*launches;
            src = cdst;
        }
    }
    return cudaGetLastError();
}

}  // namespace hw
