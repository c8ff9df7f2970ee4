// launch.cu -- kernel selection and the single launch behind escs_spmm.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <utility>
#include <vector>

#include "esc_kernel.cuh"
#include "escs_internal.h"
#include "k_table.h"

namespace escs {

namespace kern {
// escs_pack: packed[s] = vals[slot[s]] (the paper's ANNZ, §3.3.3).
__global__ void __launch_bounds__(256) esc_pack_kernel(const int* __restrict__ slot,
                                                       const float* __restrict__ vals,
                                                       float* __restrict__ out, int nnz) {
    grid_dep_wait();
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nnz; s += gridDim.x * blockDim.x)
        out[s] = vals[ld_stream(slot + s)];
}

// Busy-wait kernel for the plan-time tuner: occupies the stream while the
// host enqueues a batch of launches, so the timed batch measures GPU time,
// not host launch rate (microsecond-scale layers launch slower than they run).
__global__ void spin_kernel(long long cycles) {
    const long long t0 = clock64();
    while (clock64() - t0 < cycles) {
    }
}

}  // namespace kern

namespace {

kern::KernelFn select_kernel(int h, int n, bool vec, int ufk, bool probe, int colf) {
    if (vec) return kern::get_vec(n, colf > 0 ? colf : kern::default_colf(n), h, ufk, probe);
    if (probe) return nullptr;
    if (ufk < 2) ufk = 2;   // the scalar map has UFk 2/4/8 instances
    if (n <= 32) return kern::get_s1(h, ufk, false);
    if (n <= 64) return kern::get_s2(h, ufk, false);
    if (n <= 128) return kern::get_s4(h, ufk, false);
    if (n <= 256) return kern::get_s8(h, ufk, false);
    return nullptr;
}

kern::KParams make_params(const DevPlan& dp, const float* vals, const float* B, float* C,
                          bool packed = false) {
    kern::KParams p = {};
    p.packed = packed ? 1 : 0;
    p.gpk = dp.gpk;
    p.slot = dp.slot;
    p.items = reinterpret_cast<const int4*>(dp.items);
    p.item_aux = dp.item_aux;
    p.tile_heavy = reinterpret_cast<const int2*>(dp.tile_heavy);
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

// One launch; with programmatic stream serialization (PDL) unless disabled
// (ESCS_PDL=0), so that the launch's plan reads overlap the previous kernel.
int launch(kern::KernelFn fn, const DevPlan& dp, const kern::KParams& p, size_t smem,
           void* stream) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(dp.n_tiles);
    cfg.blockDim = dim3(32 * dp.cta_warps);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = dp.pdl ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, fn, p);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}

}  // namespace

int default_colf(int bcols) { return kern::default_colf(bcols); }

int launch_spin(void* stream, long long cycles) {
    kern::spin_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(cycles);
    return (int)cudaGetLastError();
}

bool kernel_supported(int h, int bcols, int variant, int ufk, int colf) {
    if (h < 1 || h > 4 || bcols < 1 || bcols > 256) return false;
    return select_kernel(h, bcols, variant == 1, ufk, false, colf) != nullptr &&
           select_kernel(h, bcols, false, ufk, false, 0) != nullptr;
}

// floats per lane-column slot F of the lane map the launch will use
static int lane_floats(int n, bool vec) {
    if (vec) return n < 32 ? 4 : n / 32;   // bCols < 32: L = bCols/4 lanes x float4
    return n <= 32 ? 1 : n <= 64 ? 2 : n <= 128 ? 4 : 8;
}

static size_t smem_for(const DevPlan& dp, bool vec) {
    const int F = lane_floats(dp.bcols, vec);
    const int hp = dp.h == 3 ? 4 : dp.h;
    const size_t stage = (size_t)2 * 32 * (1 + hp);           // Stage<H> floats
    const size_t part = (size_t)dp.h * 32 * F;   // kernel strides warps by max(stage, part)
    return (size_t)dp.cta_warps * (stage > part ? stage : part) * sizeof(float);
}

size_t smem_bytes(const DevPlan& dp) { return smem_for(dp, dp.variant == 1); }

int prepare_kernels(DevPlan& dp) {
    // Kernel attributes are per function and shared by every plan: only ever
    // raise the dynamic shared memory limit (never lower it under another plan).
    for (int vec = 0; vec < 2; vec++) {
        if (vec && dp.variant != 1) continue;
        const size_t smem = smem_for(dp, vec == 1);
        if (smem <= 48 * 1024) continue;
        kern::KernelFn fn = select_kernel(dp.h, dp.bcols, vec == 1, dp.ufk, false, vec ? dp.colf : 0);
        if (!fn) continue;
        cudaFuncAttributes attr;
        cudaError_t e = cudaFuncGetAttributes(&attr, (const void*)fn);
        if (e != cudaSuccess) return (int)e;
        if ((size_t)attr.maxDynamicSharedSizeBytes >= smem) continue;
        e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        if (e != cudaSuccess) return (int)e;
        if (vec) {
            kern::KernelFn pf = select_kernel(dp.h, dp.bcols, true, dp.ufk, true, dp.colf);
            if (pf) cudaFuncSetAttribute((const void*)pf,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        }
    }
    return 0;
}

int blocks_per_sm(const DevPlan& dp, bool vec, bool probe) {
    kern::KernelFn fn = select_kernel(dp.h, dp.bcols, vec, dp.ufk, probe, vec ? dp.colf : 0);
    if (!fn) return 1;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)fn, 32 * dp.cta_warps,
                                                      smem_for(dp, vec)) != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    return nb > 0 ? nb : 1;
}

int launch_pack(const DevPlan& dp, const float* vals, float* packed, void* stream) {
    if (dp.nnz == 0) return 0;
    const int threads = 256;
    const int blocks = (int)std::min<long>(((long)dp.nnz + threads - 1) / threads, 148L * 16);
    kern::esc_pack_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(dp.slot, vals, packed,
                                                                          dp.nnz);
    return (int)cudaGetLastError();
}

int launch_spmm(const DevPlan& dp, const float* vals, const float* B, float* C, void* stream,
                bool vec_ok, bool packed, float* const* extra, int n_extra, long long row_off,
                bool multicast) {
    const bool vec = vec_ok && dp.variant == 1;
    kern::KernelFn fn = select_kernel(dp.h, dp.bcols, vec, dp.ufk, false, vec ? dp.colf : 0);
    if (!fn) return (int)cudaErrorInvalidConfiguration;
    if (dp.n_tiles == 0) return 0;
    kern::KParams p = make_params(dp, vals, B, C, packed);
    p.n_extra = n_extra;
    p.mc = multicast ? 1 : 0;
    p.row_off = row_off;
    for (int d = 0; d < n_extra && d < kern::kMaxScatter; d++) p.extra[d] = extra[d];
    return launch(fn, dp, p, smem_for(dp, vec), stream);
}

int launch_group(int n, const DevPlan* const* dps, const float* const* vals,
                 const float* const* B, float* const* C, void* stream, bool packed) {
    auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
    // problems with a grouped instance (UFi = 1, vector map, aligned B/C),
    // keyed by kernel; everything else launches on its own, in input order
    std::vector<std::pair<kern::GroupFn, int>> keyed;
    for (int i = 0; i < n; i++) {
        const DevPlan& dp = *dps[i];
        if (dp.n_tiles == 0) continue;
        const bool vec = dp.variant == 1 && al16(B[i]) && al16(C[i]);
        kern::GroupFn g = nullptr;
        if (vec && dp.h == 1 && smem_for(dp, true) <= 48 * 1024)
            g = kern::get_vec_group(dp.bcols, dp.colf > 0 ? dp.colf : kern::default_colf(dp.bcols),
                                    dp.ufk);
        if (!g) {
            const int e = launch_spmm(dp, vals[i], B[i], C[i], stream, vec, packed);
            if (e) return e;
            continue;
        }
        keyed.emplace_back(g, i);
    }
    // one launch per (kernel, tile width): a CTA as wide as its problem's
    // tiles (idle warps would hold registers and shared memory for nothing)
    auto key = [&](const std::pair<kern::GroupFn, int>& x) {
        return std::make_pair(reinterpret_cast<uintptr_t>(x.first), dps[x.second]->cta_warps);
    };
    std::stable_sort(keyed.begin(), keyed.end(),
                     [&](const auto& a, const auto& b) { return key(a) < key(b); });
    for (size_t a = 0; a < keyed.size();) {
        size_t b = a;
        while (b < keyed.size() && b - a < (size_t)kern::kMaxGroup && key(keyed[b]) == key(keyed[a])) b++;
        kern::GroupParams gp = {};
        gp.n = (int)(b - a);
        int tiles = 0, maxw = 0;
        size_t warp_smem = 0;
        bool pdl = true;
        for (size_t j = a; j < b; j++) {
            const int i = keyed[j].second;
            const DevPlan& dp = *dps[i];
            kern::GProb& q = gp.prob[j - a];
            q.gpk = dp.gpk;
            q.slot = dp.slot;
            q.items = reinterpret_cast<const int4*>(dp.items);
            q.item_aux = dp.item_aux;
            q.tile_heavy = reinterpret_cast<const int2*>(dp.tile_heavy);
            q.heavy = reinterpret_cast<const int4*>(dp.heavy);
            q.ws = dp.ws;
            q.counters = dp.counters;
            q.vals = vals[i];
            q.B = B[i];
            q.C = C[i];
            q.m = dp.m;
            q.n = dp.bcols;
            q.W = dp.cta_warps;
            q.packed = packed ? 1 : 0;
            gp.tile_start[j - a] = tiles;
            tiles += dp.n_tiles;
            maxw = std::max(maxw, dp.cta_warps);
            warp_smem = std::max(warp_smem, smem_for(dp, true) / dp.cta_warps);
            pdl = pdl && dp.pdl;
        }
        gp.tile_start[gp.n] = tiles;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(tiles);
        cfg.blockDim = dim3(32 * maxw);
        cfg.dynamicSmemBytes = warp_smem * maxw;
        cfg.stream = (cudaStream_t)stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaError_t e = cudaLaunchKernelEx(&cfg, keyed[a].first, gp);
        if (e != cudaSuccess) return (int)e;
        e = cudaGetLastError();
        if (e != cudaSuccess) return (int)e;
        a = b;
    }
    return 0;
}

int launch_probe(const DevPlan& dp, const float* B, float* sink, void* stream, bool vec_ok) {
    if (!(vec_ok && dp.variant == 1)) return (int)cudaErrorInvalidConfiguration;
    kern::KernelFn fn = select_kernel(dp.h, dp.bcols, true, dp.ufk, true, dp.colf);
    if (!fn) return (int)cudaErrorInvalidConfiguration;
    if (dp.n_tiles == 0) return 0;
    kern::KParams p = make_params(dp, nullptr, B, sink);
    return launch(fn, dp, p, smem_for(dp, true), stream);
}

}  // namespace escs
