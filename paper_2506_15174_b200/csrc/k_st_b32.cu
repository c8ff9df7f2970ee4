// Instantiations of the staged record walk (staged_kernel.cuh) for lane map
// VecMap<8, 4> (bCols 32): UFi 1, 2, 3, 4, 6, 8 (the record formats of
// esc_kernel.cuh RecFmt), panels per warp NPW with NPW x UFi x F <= 32
// accumulators per lane, UFk = 2 records per sub-warp in flight; each with
// its gather probe (same loads, no FMAs).
#include "staged_kernel.cuh"

namespace escs {
namespace kern {

StagedFn get_staged_b32(int h, int npw, bool probe) {
    using M = VecMap<8, 4>;
#ifdef ESC_ST_U
    constexpr int U = ESC_ST_U;
#else
    constexpr int U = 2;
#endif
#define ESC_ST_CASE(H_, NPW_)                                                             \
    if constexpr ((NPW_) * (H_) * M::F <= 32)                                             \
        if (h == (H_) && npw == (NPW_))                                                   \
            return probe ? esc_staged_kernel<H_, M, U, NPW_, true> : esc_staged_kernel<H_, M, U, NPW_, false>;
    ESC_ST_CASE(1, 1) ESC_ST_CASE(1, 2) ESC_ST_CASE(1, 4)
    ESC_ST_CASE(2, 1) ESC_ST_CASE(2, 2) ESC_ST_CASE(2, 4)
    ESC_ST_CASE(3, 1) ESC_ST_CASE(3, 2)
    ESC_ST_CASE(4, 1) ESC_ST_CASE(4, 2)
    ESC_ST_CASE(6, 1)
    ESC_ST_CASE(8, 1)
#undef ESC_ST_CASE
    return nullptr;
}

}  // namespace kern
}  // namespace escs
