// hw_wavelet.cu -- three-point wavelet transform in time, W_t (x) Id_x.
//
// Restates WaveletTransform._apply_stages (/root/reference/pkg/src/heatwave/
// wavelet.py:114-137) with the two-scale matrices M_j = [P_j | Q_j] of
// wavelet.py:56-76 written out in closed form.  Every
// stage is one launch over (stage rows) x N_x with coalesced access along
// the spatial axis; each output value accumulates the same products in the
// same (CSR column) order as the reference's temporal_apply, without FMA
// contraction, so the transform is bit-identical to the reference.
//
// Synthesis (W): stage j maps the coarse nodal prefix c (rows 0..2^(j-1))
// and the level-j wavelet coefficients d (rows 2^(j-1)+1..2^j, read from the
// untouched input) to the fine nodal prefix (rows 0..2^j).  The ping-pong
// buffer choice puts stage J into the output; no copy-back pass is needed.
// Transpose (W^T): stage j reads the fine prefix and writes its wavelet
// part d' straight into the output rows, its coarse part c' into scratch.
#include "hw_common.cuh"
#include "hw_internal.cuh"

namespace hw {

// a_k = -1 if k == 0 else -1/2 ; b_k = -1 if k == nw-1 else -1/2
// (wavelet.py:70-71); the stored CSR value is s * a_k, s = 2^(j/2).
__device__ __forceinline__ double qa(double s, int k) { return s * (k == 0 ? -1.0 : -0.5); }
__device__ __forceinline__ double qb(double s, int k, int nw) { return s * (k == nw - 1 ? -1.0 : -0.5); }

// dst rows [0, nf) <- M_j [c ; d]; grid: (column blocks, stage rows)
__global__ void wav_syn_stage(const double *__restrict__ C, const double *__restrict__ Dm,
                              double *__restrict__ Y, int j, double s, int64_t nx)
{
    const int nc = (1 << (j - 1)) + 1, nf = (1 << j) + 1, nw = 1 << (j - 1);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nx) return;
    for (int r = blockIdx.y; r < nf; r += gridDim.y) {
        double acc;
        if ((r & 1) == 0) {
            const int q = r >> 1;                 // coarse index
            acc = C[(int64_t)q * nx + i];         // P: 1.0 * c[q]
            if (q >= 1)                           // Q col q-1: s * b_{q-1}
                acc = add_rn(acc, mul_rn(qb(s, q - 1, nw), Dm[(int64_t)(nc + q - 1) * nx + i]));
            if (q < nw)                           // Q col q: s * a_q
                acc = add_rn(acc, mul_rn(qa(s, q), Dm[(int64_t)(nc + q) * nx + i]));
        } else {
            const int k = r >> 1;
            acc = mul_rn(0.5, C[(int64_t)k * nx + i]);
            acc = add_rn(acc, mul_rn(0.5, C[(int64_t)(k + 1) * nx + i]));
            acc = add_rn(acc, mul_rn(s, Dm[(int64_t)(nc + k) * nx + i]));
        }
        Y[(int64_t)r * nx + i] = acc;
    }
}

// c' -> Cout rows [0, nc), d' -> Dout rows [nc, nf)   (M_j^T applied to X)
__global__ void wav_ana_stage(const double *__restrict__ X, double *__restrict__ Cout,
                              double *__restrict__ Dout, int j, double s, int64_t nx)
{
    const int nc = (1 << (j - 1)) + 1, nf = (1 << j) + 1, nw = 1 << (j - 1);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nx) return;
    for (int r = blockIdx.y; r < nf; r += gridDim.y) {
        if (r < nc) {
            // column r of P_j: rows 2r-1 (1/2), 2r (1), 2r+1 (1/2)
            double acc;
            if (r >= 1) {
                acc = mul_rn(0.5, X[(int64_t)(2 * r - 1) * nx + i]);
                acc = add_rn(acc, X[(int64_t)(2 * r) * nx + i]);
            } else {
                acc = X[i];
            }
            if (2 * r + 1 < nf) acc = add_rn(acc, mul_rn(0.5, X[(int64_t)(2 * r + 1) * nx + i]));
            Cout[(int64_t)r * nx + i] = acc;
        } else {
            const int k = r - nc;                 // column k of Q_j: rows 2k, 2k+1, 2k+2
            double acc = mul_rn(qa(s, k), X[(int64_t)(2 * k) * nx + i]);
            acc = add_rn(acc, mul_rn(s, X[(int64_t)(2 * k + 1) * nx + i]));
            acc = add_rn(acc, mul_rn(qb(s, k, nw), X[(int64_t)(2 * k + 2) * nx + i]));
            Dout[(int64_t)r * nx + i] = acc;
        }
    }
}

static dim3 stage_grid(int64_t rows, int64_t nx, int bs)
{
    return dim3((unsigned)((nx + bs - 1) / bs), (unsigned)(rows < 65535 ? rows : 65535));
}

// Y = W X (transpose = 0) or W^T X (transpose = 1).  S1 (and S2 for the
// transpose) are scratch arrays with at least 2^(J-1)+1 rows.
cudaError_t wavelet_apply(const double *X, double *Y, double *S1, double *S2, int J,
                          const double *scale, int64_t nt, int64_t nx, bool transpose,
                          cudaStream_t st, int64_t *launches)
{
    const int bs = 256;
    if (J == 0) {
        return cudaMemcpyAsync(Y, X, (size_t)(nt * nx) * sizeof(double),
                               cudaMemcpyDeviceToDevice, st);
    }
    if (!transpose) {
        const double *src = X;
        for (int j = 1; j <= J; ++j) {
            double *dst = ((J - j) % 2 == 0) ? Y : S1;
            wav_syn_stage<<<stage_grid((1LL << j) + 1, nx, bs), bs, 0, st>>>(src, X, dst, j,
                                                                          scale[j - 1], nx);
            ++*launches;
            src = dst;
        }
    } else {
        const double *src = X;
        for (int j = J; j >= 1; --j) {
            double *cdst = (j == 1) ? Y : (((J - j) % 2 == 0) ? S1 : S2);
            wav_ana_stage<<<stage_grid((1LL << j) + 1, nx, bs), bs, 0, st>>>(src, cdst, Y, j,
                                                                          scale[j - 1], nx);
            ++*launches;
            src = cdst;
        }
    }
    return cudaGetLastError();
}

}  // namespace hw
