// Instantiations of the ESC kernel for lane map VecMap<1, 4> (see esc_kernel.cuh).
#include "esc_kernel.cuh"
namespace escs {
namespace kern {
KernelFn get_b4(int h, int ufk, bool probe) {
    using M = VecMap<1, 4>;
    if (h == 1 && ufk == 1) return probe ? esc_spmm_kernel<1, M, 1, true> : esc_spmm_kernel<1, M, 1, false>;
    if (h == 2 && ufk == 1) return probe ? esc_spmm_kernel<2, M, 1, true> : esc_spmm_kernel<2, M, 1, false>;
    if (h == 3 && ufk == 1) return probe ? esc_spmm_kernel<3, M, 1, true> : esc_spmm_kernel<3, M, 1, false>;
    if (h == 4 && ufk == 1) return probe ? esc_spmm_kernel<4, M, 1, true> : esc_spmm_kernel<4, M, 1, false>;
    return nullptr;
}
}  // namespace kern
}  // namespace escs
