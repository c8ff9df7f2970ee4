// launch.cu -- kernel selection and the single launch behind escs_spmm.
#include <cuda_runtime.h>

#include "esc_kernel.cuh"
#include "escs_internal.h"

namespace escs {
namespace kern {
KernelFn get_b32(int, int, bool);
KernelFn get_b64(int, int, bool);
KernelFn get_b128(int, int, bool);
KernelFn get_b256(int, int, bool);
KernelFn get_s1(int, int, bool);
KernelFn get_s2(int, int, bool);
KernelFn get_s4(int, int, bool);
KernelFn get_s8(int, int, bool);
}  // namespace kern

namespace {

kern::KernelFn select_kernel(int h, int n, bool vec, int ufk, bool probe) {
    if (vec) {
        switch (n) {
            case 32: return kern::get_b32(h, ufk, probe);
            case 64: return kern::get_b64(h, ufk, probe);
            case 128: return kern::get_b128(h, ufk, probe);
            case 256: return kern::get_b256(h, ufk, probe);
            default: return nullptr;
        }
    }
    if (probe) return nullptr;
    if (n <= 32) return kern::get_s1(h, 4, false);
    if (n <= 64) return kern::get_s2(h, 4, false);
    if (n <= 128) return kern::get_s4(h, 4, false);
    if (n <= 256) return kern::get_s8(h, 4, false);
    return nullptr;
}

kern::KParams make_params(const DevPlan& dp, const float* vals, const float* B, float* C) {
    kern::KParams p;
    p.grp = reinterpret_cast<const int4*>(dp.grp);
    p.gcol = dp.gcol;
    p.slot = dp.slot;
    p.items = reinterpret_cast<const int4*>(dp.items);
    p.item_aux = dp.item_aux;
    p.tiles = reinterpret_cast<const int4*>(dp.tiles);
    p.heavy = reinterpret_cast<const int4*>(dp.heavy);
    p.ws = dp.ws;
    p.counters = dp.counters;
    p.vals = vals;
    p.B = B;
    p.C = C;
    p.m = dp.m;
    p.n = dp.bcols;
    return p;
}

}  // namespace

bool kernel_supported(int h, int bcols, int variant, int ufk) {
    if (h < 1 || h > 4 || bcols < 1 || bcols > 256) return false;
    const bool vec = variant == 1;
    if (vec) return select_kernel(h, bcols, true, ufk, false) != nullptr;
    return select_kernel(h, bcols, false, 4, false) != nullptr;
}

size_t smem_bytes(const DevPlan& dp) {
    if (!dp.any_sync) return 0;
    return (size_t)dp.cta_warps * dp.h * dp.bcols * sizeof(float);
}

int prepare_kernels(const DevPlan& dp) {
    const size_t smem = smem_bytes(dp);
    for (int vec = 0; vec < 2; vec++) {
        if (vec && dp.variant != 1) continue;
        kern::KernelFn fn = select_kernel(dp.h, dp.bcols, vec == 1, vec ? dp.ufk : 4, false);
        if (!fn) continue;
        cudaError_t e = cudaFuncSetAttribute((const void*)fn,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return (int)e;
        // prefer L1 for the gathered B rows; leave enough carveout for the
        // combine buffers of resident tiles
        const int threads = 32 * dp.cta_warps;
        const int ctas = 2048 / threads;
        int pct = (int)((smem * ctas * 100 + 228 * 1024 - 1) / (228 * 1024));
        if (pct > 100) pct = 100;
        e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 pct);
        if (e != cudaSuccess) return (int)e;
        if (vec) {
            kern::KernelFn pf = select_kernel(dp.h, dp.bcols, true, dp.ufk, true);
            if (pf) cudaFuncSetAttribute((const void*)pf,
                                         cudaFuncAttributePreferredSharedMemoryCarveout, 0);
        }
    }
    return 0;
}

int launch_spmm(const DevPlan& dp, const float* vals, const float* B, float* C, void* stream,
                bool vec_ok) {
    const bool vec = vec_ok && dp.variant == 1;
    kern::KernelFn fn = select_kernel(dp.h, dp.bcols, vec, vec ? dp.ufk : 4, false);
    if (!fn) return (int)cudaErrorInvalidConfiguration;
    if (dp.n_tiles == 0) return 0;
    kern::KParams p = make_params(dp, vals, B, C);
    fn<<<dp.n_tiles, 32 * dp.cta_warps, smem_bytes(dp), (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}

int launch_probe(const DevPlan& dp, const float* B, float* sink, void* stream, bool vec_ok) {
    if (!(vec_ok && dp.variant == 1)) return (int)cudaErrorInvalidConfiguration;
    kern::KernelFn fn = select_kernel(dp.h, dp.bcols, true, dp.ufk, true);
    if (!fn) return (int)cudaErrorInvalidConfiguration;
    if (dp.n_tiles == 0) return 0;
    kern::KParams p = make_params(dp, nullptr, B, sink);
    fn<<<dp.n_tiles, 32 * dp.cta_warps, 0, (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace escs
