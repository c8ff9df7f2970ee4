// launch.cu -- kernel selection and the single launch behind escs_spmm.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <mutex>
#include <utility>
#include <vector>

#include "esc_kernel.cuh"
#include "escs_internal.h"
#include "k_table.h"

namespace escs {

namespace kern {
// escs_pack: the record stream of the packed walk (esc_kernel.cuh "records";
// the paper's value re-layout "ANNZ", §3.3.3).  One thread per gcol
// j: UFi = 1 writes {col, vals[j]} (the slot map is the identity); UFi > 1
// writes the gcol's packed word and its pattern rows' values by row, taking
// the p = popcount(mask) values from slots vbase[j] .. vbase[j] + p - 1
// (Reading R1: a gcol's values are contiguous in slot order, rows ascending).
// src != NULL (a staged plan): record q of the output is canonical gcol
// src[q] (-1: padding, written as zeros).
template <int H>
__global__ void __launch_bounds__(256) esc_pack_rec_kernel(const int* __restrict__ gpk,
                                                           const int* __restrict__ slot,
                                                           const int* __restrict__ vbase,
                                                           const float* __restrict__ vals,
                                                           const int* __restrict__ src,
                                                           const int* __restrict__ vmap,
                                                           int* __restrict__ out, int G) {
    constexpr int RW = RecFmt<H>::W;
    grid_dep_wait();
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < G; q += gridDim.x * blockDim.x) {
        const int j = src ? src[q] : q;
        if (j < 0) {
#pragma unroll
            for (int v = 0; v < RW; v++) out[(size_t)q * RW + v] = 0;
            continue;
        }
        const int pk = gpk[j];   // the plan's word: col | mask << RecFmt<H>::Shift
        if constexpr (H == 1) {
            *reinterpret_cast<int2*>(out + (size_t)q * 2) =
                make_int2(pk & RecFmt<1>::ColMask, __float_as_int(vals[vmap ? vmap[j] : j]));
        } else {
            int w[RW];
#pragma unroll
            for (int q = 0; q < RW; q++) w[q] = 0;
            w[0] = pk;
            const unsigned mk = (unsigned)pk >> RecFmt<H>::Shift;
            int s = vbase[j];
#pragma unroll
            for (int r = 0; r < H; r++)
                if ((mk >> r) & 1u) {
                    const int q = slot[s++];
                    w[1 + r] = __float_as_int(vals[vmap ? vmap[q] : q]);
                }
            int4* o = reinterpret_cast<int4*>(out + (size_t)q * RW);
#pragma unroll
            for (int v = 0; v < RW / 4; v++) o[v] = make_int4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]);
        }
    }
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

kern::KernelFn select_kernel(int h, int n, bool vec, int ufk, int mode, int colf) {
    if (vec) {
        kern::KernelFn f = kern::get_vec(n, colf > 0 ? colf : kern::default_colf(n), h, ufk, mode);
        // the CSR walk has the alternative coarsening factors at UFi = 1 only:
        // a record-tuned plan (UFi > 1, colf != default) runs escs_spmm on the
        // default lane map (same output layout, same per-warp smem)
        if (!f && mode < kern::kRec) f = kern::get_vec(n, kern::default_colf(n), h, ufk, mode);
        return f;
    }
    if (mode != kern::kCsr) return nullptr;   // probes and records: vector maps only
    if (ufk < 2) ufk = 2;   // the scalar map has UFk 2/4/8 instances
    if (n <= 32) return kern::get_s1(h, ufk, mode);
    if (n <= 64) return kern::get_s2(h, ufk, mode);
    if (n <= 128) return kern::get_s4(h, ufk, mode);
    if (n <= 256) return kern::get_s8(h, ufk, mode);
    return nullptr;
}

kern::KParams make_params(const DevPlan& dp, const float* vals, const float* B, float* C) {
    kern::KParams p = {};
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
    p.k = dp.k;
    p.rowmap = dp.rowmap;
    p.slot_ws = reinterpret_cast<const int4*>(dp.slot_ws);
    p.wsc = dp.wsc;
    p.wsc_counters = dp.wsc_counters;
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
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (dp.pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        na++;
    }
    if (dp.carveout >= 0) {   // the plan's L1 / shared split (DevPlan::carveout)
        attr[na].id = cudaLaunchAttributePreferredSharedMemoryCarveout;
        attr[na].val.sharedMemCarveout = (unsigned)dp.carveout;
        na++;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaError_t e = cudaLaunchKernelEx(&cfg, fn, p);
    if (e != cudaSuccess) {
        cudaGetLastError();   // consume it: a refused launch must not fail the next one
        return (int)e;
    }
    return (int)cudaGetLastError();
}

}  // namespace

int default_colf(int bcols) { return kern::default_colf(bcols); }

int launch_spin(void* stream, long long cycles) {
    kern::spin_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(cycles);
    return (int)cudaGetLastError();
}

bool kernel_supported(int h, int bcols, int variant, int ufk, int colf, bool packed) {
    if (h < 1 || h > 8 || bcols < 1 || bcols > 256) return false;
    if (packed)   // the record walk: vector lane map only; UFi 1-4, 6, 8
        return variant == 1 && select_kernel(h, bcols, true, ufk, kern::kRec, colf) != nullptr;
    if (h > 4) return false;   // the CSR-value walk: UFi 1-4
    return select_kernel(h, bcols, variant == 1, ufk, kern::kCsr, colf) != nullptr &&
           select_kernel(h, bcols, false, ufk, kern::kCsr, 0) != nullptr;
}

// floats per lane-column slot F of the lane map the launch will use
static int lane_floats(int n, bool vec) {
    if (vec) return n < 32 ? 4 : n / 32;   // bCols < 32: L = bCols/4 lanes x float4
    return n <= 32 ? 1 : n <= 64 ? 2 : n <= 128 ? 4 : 8;
}

// Dynamic shared memory of a launch: W warps x the kernel's per-warp area
// (esc_kernel.cuh warp_smem_floats: the CSR walk's staging area at UFi > 1
// and the H x bCols combine partial share it; the record walk needs only the
// partial).
static size_t smem_for(const DevPlan& dp, bool vec, bool rec = false) {
    const int F = lane_floats(dp.bcols, vec);
    const int hp = dp.h == 3 ? 4 : dp.h;
    const size_t stage = (!rec && dp.h > 1) ? (size_t)2 * 32 * (1 + hp) : 0;   // Stage<H> floats
    const size_t part = (size_t)dp.h * 32 * F;
    return (size_t)dp.cta_warps * (stage > part ? stage : part) * sizeof(float);
}

size_t smem_bytes(const DevPlan& dp, bool packed) { return smem_for(dp, dp.variant == 1, packed); }

// Kernel attributes are per function and shared by every plan: only ever
// raise the dynamic shared memory limit (never lower it under another plan);
// the read-and-raise is serialised so concurrent planners cannot lower it.
static std::mutex g_attr_mutex;
static int raise_smem(kern::KernelFn fn, size_t smem) {
    if (!fn || smem <= 32 * 1024) return 0;   // well under the 48 KB default (static smem included)
    std::lock_guard<std::mutex> lock(g_attr_mutex);
    cudaFuncAttributes attr;
    cudaError_t e = cudaFuncGetAttributes(&attr, (const void*)fn);
    if (e != cudaSuccess) return (int)e;
    if ((size_t)attr.maxDynamicSharedSizeBytes >= smem) return 0;
    return (int)cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem);
}

int prepare_kernels(DevPlan& dp) {
    for (int vec = 0; vec < 2; vec++) {
        if (vec && dp.variant != 1) continue;
        const int colf = vec ? dp.colf : 0;
        const int modes[4] = {kern::kCsr, kern::kProbe, kern::kRec, kern::kRecProbe};
        for (int md : modes) {
            const bool rec = md >= kern::kRec;
            if (rec && !vec) continue;
            if (int e = raise_smem(select_kernel(dp.h, dp.bcols, vec == 1, dp.ufk, md, colf),
                                   smem_for(dp, vec == 1, rec)))
                return e;
        }
    }
    return 0;
}

// The smallest shared-memory carveout (percent of the SM's 228 KB) that still
// holds the plan's full occupancy of the gather walk: the rest is L1, where the
// gathered B rows are re-read by the SM's other warps (2048x512@70% b128 hot:
// 10.4 -> 9.4 us at the maximum L1; a blanket minimum carveout instead lowers the
// occupancy of plans with wider tiles: 14.7 -> 17.5 us on 512x4608@80%).
int gather_carveout(const DevPlan& dp, bool packed) {
    const bool vec = dp.variant == 1;
    const int nb = blocks_per_sm(dp, vec, false, packed);
    const size_t per = smem_for(dp, vec, packed) + 1024;   // + the per-CTA reservation
    const size_t total = 228 * 1024;
    const size_t need = (size_t)nb * per;
    const int pct = (int)((need * 100 + total - 1) / total) + 2;   // rounded up, a small margin
    return pct > 100 ? 100 : pct;
}

int blocks_per_sm(const DevPlan& dp, bool vec, bool probe, bool packed) {
    const int mode = packed ? (probe ? kern::kRecProbe : kern::kRec) : (probe ? kern::kProbe : kern::kCsr);
    kern::KernelFn fn = select_kernel(dp.h, dp.bcols, vec, dp.ufk, mode, vec ? dp.colf : 0);
    if (!fn) return 1;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)fn, 32 * dp.cta_warps,
                                                      smem_for(dp, vec, packed)) != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    return nb > 0 ? nb : 1;
}

int64_t packed_words(const DevPlan& dp) {
    const int rw = dp.h == 1 ? 2 : (dp.h <= 3 ? 4 : (dp.h <= 7 ? 8 : 12));   // kern::RecFmt<h>::W
    // rounded to 16 bytes: bulk copies / prefetches of a range's last record
    // never reach past the buffer
    return ((int64_t)(dp.st_n_cta ? dp.st_n_rec : dp.G) * rw + 3) / 4 * 4;
}

// The record stream: canonical gcol order, or -- for a staged plan -- the
// staged schedule's order (record q = canonical gcol st_src[q]).
int launch_pack(const DevPlan& dp, const float* vals, float* packed, void* stream) {
    const int n = dp.st_n_cta ? dp.st_n_rec : dp.G;
    if (n == 0) return 0;
    const int* src = dp.st_n_cta ? dp.st_src : nullptr;
    const int threads = 256;
    const int blocks = (int)std::min<long>(((long)n + threads - 1) / threads, 148L * 16);
    int* out = reinterpret_cast<int*>(packed);
    cudaStream_t st = (cudaStream_t)stream;
    switch (dp.h) {
        case 1: kern::esc_pack_rec_kernel<1><<<blocks, threads, 0, st>>>(dp.gpk, dp.slot, dp.vbase, vals, src, dp.vmap, out, n); break;
        case 2: kern::esc_pack_rec_kernel<2><<<blocks, threads, 0, st>>>(dp.gpk, dp.slot, dp.vbase, vals, src, dp.vmap, out, n); break;
        case 3: kern::esc_pack_rec_kernel<3><<<blocks, threads, 0, st>>>(dp.gpk, dp.slot, dp.vbase, vals, src, dp.vmap, out, n); break;
        case 4: kern::esc_pack_rec_kernel<4><<<blocks, threads, 0, st>>>(dp.gpk, dp.slot, dp.vbase, vals, src, dp.vmap, out, n); break;
        case 6: kern::esc_pack_rec_kernel<6><<<blocks, threads, 0, st>>>(dp.gpk, dp.slot, dp.vbase, vals, src, dp.vmap, out, n); break;
        case 8: kern::esc_pack_rec_kernel<8><<<blocks, threads, 0, st>>>(dp.gpk, dp.slot, dp.vbase, vals, src, dp.vmap, out, n); break;
        default: return (int)cudaErrorInvalidConfiguration;
    }
    return (int)cudaGetLastError();
}

int launch_spmm(const DevPlan& dp, const float* vals, const float* B, float* C, void* stream,
                bool vec_ok, bool packed, float* const* extra, int n_extra, long long row_off,
                bool multicast) {
    const bool vec = vec_ok && dp.variant == 1;
    if (packed && !vec) return (int)cudaErrorInvalidConfiguration;   // records: vector map only
    kern::KernelFn fn = select_kernel(dp.h, dp.bcols, vec, dp.ufk, packed ? kern::kRec : kern::kCsr,
                                      vec ? dp.colf : 0);
    if (!fn) return (int)cudaErrorInvalidConfiguration;
    if (dp.n_tiles == 0) return 0;
    kern::KParams p = make_params(dp, vals, B, C);
    p.n_extra = n_extra;
    p.mc = multicast ? 1 : 0;
    p.row_off = row_off;
    for (int d = 0; d < n_extra && d < kern::kMaxScatter; d++) p.extra[d] = extra[d];
    return launch(fn, dp, p, smem_for(dp, vec, packed), stream);
}

int launch_group(int n, const DevPlan* const* dps, const float* const* vals,
                 const float* const* B, float* const* C, void* stream) {
    auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
    // problems with a grouped instance (UFi = 1, vector map, aligned B/C),
    // keyed by kernel; everything else launches on its own, in input order
    std::vector<std::pair<kern::GroupFn, int>> keyed;
    for (int i = 0; i < n; i++) {
        const DevPlan& dp = *dps[i];
        if (dp.n_tiles == 0) continue;
        const bool vec = dp.variant == 1 && al16(B[i]) && al16(C[i]);
        kern::GroupFn g = nullptr;
        if (vec && dp.h == 1 && !dp.slot_ws && smem_for(dp, true) <= 32 * 1024)   // no attribute raise for group kernels
            g = kern::get_vec_group(dp.bcols, dp.colf > 0 ? dp.colf : kern::default_colf(dp.bcols),
                                    dp.ufk);
        if (!g) {
            const int e = launch_spmm(dp, vals[i], B[i], C[i], stream, vec, false);
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
        if (e != cudaSuccess) {
            cudaGetLastError();
            return (int)e;
        }
        e = cudaGetLastError();
        if (e != cudaSuccess) return (int)e;
        a = b;
    }
    return 0;
}

int launch_probe(const DevPlan& dp, const float* B, float* sink, void* stream, bool vec_ok,
                 const float* packed) {
    if (!(vec_ok && dp.variant == 1)) return (int)cudaErrorInvalidConfiguration;
    const bool rec = packed != nullptr;
    kern::KernelFn fn = select_kernel(dp.h, dp.bcols, true, dp.ufk, rec ? kern::kRecProbe : kern::kProbe,
                                      dp.colf);
    if (!fn) return (int)cudaErrorInvalidConfiguration;
    if (dp.n_tiles == 0) return 0;
    kern::KParams p = make_params(dp, packed, B, sink);
    return launch(fn, dp, p, smem_for(dp, true, rec), stream);
}

}  // namespace escs
