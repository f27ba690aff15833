// hw_common.cuh -- shared definitions for the B200 space-time PCG kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define HW_DEV __device__ __forceinline__

namespace hw {

constexpr int kCoefStride = 8;       // HWG_COEF_STRIDE
enum CoefSlot { kC0 = 0, kCx = 1, kCy = 2, kCd = 3, kInv = 4, kCoarse = 5 };

// cp.async 8-byte global -> shared copy (LDGSTS); L1-bypass is not
// available for 8-byte copies, .ca keeps them coherent within the SM.
HW_DEV void cp_async8(void *smem, const void *gmem)
{
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
HW_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
HW_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Exactly-rounded products/sums where the reference's operation order is
// mirrored (no FMA contraction).
HW_DEV double mul_rn(double a, double b) { return __dmul_rn(a, b); }
HW_DEV double add_rn(double a, double b) { return __dadd_rn(a, b); }
HW_DEV double sub_mul(double acc, double a, double x) { return __dsub_rn(acc, __dmul_rn(a, x)); }
HW_DEV double add_mul(double acc, double a, double x) { return __dadd_rn(acc, __dmul_rn(a, x)); }

}  // namespace hw
