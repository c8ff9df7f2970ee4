// Instantiations of the ESC kernel for lane map VecMap<4, 4> (see esc_kernel.cuh).
#include "esc_kernel.cuh"
namespace escs {
namespace kern {
KernelFn get_b16(int h, int ufk, bool probe) {
    using M = VecMap<4, 4>;
    if (h == 1 && ufk == 2) return probe ? esc_spmm_kernel<1, M, 2, true> : esc_spmm_kernel<1, M, 2, false>;
    if (h == 1 && ufk == 4) return probe ? esc_spmm_kernel<1, M, 4, true> : esc_spmm_kernel<1, M, 4, false>;
    if (h == 2 && ufk == 2) return probe ? esc_spmm_kernel<2, M, 2, true> : esc_spmm_kernel<2, M, 2, false>;
    if (h == 2 && ufk == 4) return probe ? esc_spmm_kernel<2, M, 4, true> : esc_spmm_kernel<2, M, 4, false>;
    if (h == 3 && ufk == 2) return probe ? esc_spmm_kernel<3, M, 2, true> : esc_spmm_kernel<3, M, 2, false>;
    if (h == 3 && ufk == 4) return probe ? esc_spmm_kernel<3, M, 4, true> : esc_spmm_kernel<3, M, 4, false>;
    if (h == 4 && ufk == 2) return probe ? esc_spmm_kernel<4, M, 2, true> : esc_spmm_kernel<4, M, 2, false>;
    if (h == 4 && ufk == 4) return probe ? esc_spmm_kernel<4, M, 4, true> : esc_spmm_kernel<4, M, 4, false>;
    return nullptr;
}
}  // namespace kern
}  // namespace escs
