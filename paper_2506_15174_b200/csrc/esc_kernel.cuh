// esc_kernel.cuh -- the enumerate-and-sparse-coarsen SpMM kernel for sm_100a.
//
// Paper mapping (arXiv 2506.15174):
//   * enumeration (§3.2): a warp works on one item of one row panel
//     (UFi = H rows); inside the item, every group (panel, pattern) is a run of
//     columns sharing one UFi-bit pattern, dispatched once to a body
//     specialised for that pattern, so the hot loop has no data-dependent
//     conditionals (the "enumerated blocks" of Listing 4);
//   * thread mapping map(j, W) (§3.3.1): lanes own consecutive
//     columns of B/C (float4 per lane on the vector map, 32-strided scalars on
//     the scalar map = the paper's WarpTile mapping, Listing 5);
//   * thread coarsening (§3.3.2): each lane keeps H x F
//     accumulators (pattern rows x its columns); a B element loaded once into a
//     register is reused for every row of the pattern, an A value for all the
//     lane's columns; UFK gathered B rows are in flight per sub-warp;
//   * data transformation (§3.3.3): columns ("Cols") and value
//     slots ("ANNZ" order, Reading R1) are staged 32 at a time by the warp with
//     coalesced loads and broadcast with __shfl_sync;
//   * safety: write-after-write between items of one panel is
//     resolved by a deterministic combine -- shared memory inside the CTA
//     tile, a global workspace + counter (last arriver sums in tile order)
//     across tiles -- instead of atomicAdd, so C is overwritten (beta = 0),
//     one launch, no memset, bitwise reproducible.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace escs {
namespace kern {

constexpr unsigned kFull = 0xffffffffu;

struct KParams {
    const int4* __restrict__ grp;      // col_begin, col_end, val_begin, mask
    const int* __restrict__ gcol;
    const int* __restrict__ slot;
    const int4* __restrict__ items;    // panel, group_begin, gcol_begin, gcol_end
    const int* __restrict__ item_aux;  // lead | cnt << 8
    const int4* __restrict__ tiles;    // item_begin, item_end, heavy_id, flags
    const int4* __restrict__ heavy;    // panel, ws_base, ntiles, 0
    float* ws;
    int* counters;
    const float* __restrict__ vals;
    const float* __restrict__ B;
    float* __restrict__ C;
    int m, n;
};

__device__ __forceinline__ float4 ldg_f4(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ int ldg_stream(const int* p) {
    int r;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

// Lane map with float4 lanes: L lanes cover one B row of N = 4*V*L floats,
// S = 32/L sub-warps process S gathered rows per warp step.
template <int L_, int V_>
struct VecMap {
    static constexpr int L = L_, S = 32 / L_, V = V_, F = 4 * V_;
    static constexpr bool kVec = true;
    __device__ static __forceinline__ int col(int lj, int f) { return (lj * V + (f >> 2)) * 4 + (f & 3); }
    __device__ static __forceinline__ void load(float (&b)[F], const float* row, int, int lj) {
        const float4* r4 = reinterpret_cast<const float4*>(row) + lj * V;
#pragma unroll
        for (int v = 0; v < V; v++) {
            const float4 x = ldg_f4(r4 + v);
            b[4 * v + 0] = x.x; b[4 * v + 1] = x.y; b[4 * v + 2] = x.z; b[4 * v + 3] = x.w;
        }
    }
    __device__ static __forceinline__ void store(float* row, const float (&a)[F], int, int lj) {
        float4* r4 = reinterpret_cast<float4*>(row) + lj * V;
#pragma unroll
        for (int v = 0; v < V; v++)
            r4[v] = make_float4(a[4 * v + 0], a[4 * v + 1], a[4 * v + 2], a[4 * v + 3]);
    }
};

// Scalar lane map (the paper's map(j, 32*WarpTile), Listing 5/6): lane owns
// columns lane + 32*f, f < WT, predicated on j < N.  Any N <= 32*WT, any
// alignment.
template <int WT>
struct ScalarMap {
    static constexpr int L = 32, S = 1, V = 0, F = WT;
    static constexpr bool kVec = false;
    __device__ static __forceinline__ int col(int lj, int f) { return lj + 32 * f; }
    __device__ static __forceinline__ void load(float (&b)[F], const float* row, int n, int lj) {
#pragma unroll
        for (int f = 0; f < F; f++) {
            const int j = lj + 32 * f;
            b[f] = (j < n) ? __ldg(row + j) : 0.f;
        }
    }
    __device__ static __forceinline__ void store(float* row, const float (&a)[F], int n, int lj) {
#pragma unroll
        for (int f = 0; f < F; f++) {
            const int j = lj + 32 * f;
            if (j < n) row[j] = a[f];
        }
    }
};

// One run of columns [pos, gend) of a group with pattern MASK.  The values of
// column ordinal ci sit at slots vbase + ci*P + rank (Reading R1).
template <int H, int MASK, class Map, int UFK, bool PROBE>
__device__ __forceinline__ void run_group(const KParams& p, float (&acc)[H][Map::F], int cbeg,
                                          int vbase, int pos, int gend, int lane, int sub, int lj) {
    constexpr int P = __builtin_popcount(MASK);
    constexpr int S = Map::S, F = Map::F;
    for (int c0 = pos; c0 < gend; c0 += 32) {
        const int n = min(32, gend - c0);
        const int myc = c0 + lane;
        int col = 0;
        float v[P];
        if (lane < n) {
            col = ldg_stream(p.gcol + myc);
            if constexpr (!PROBE) {
                const int* sp = p.slot + vbase + (myc - cbeg) * P;
#pragma unroll
                for (int r = 0; r < P; r++) v[r] = __ldg(p.vals + ldg_stream(sp + r));
            }
        }
        if (PROBE || lane >= n) {
#pragma unroll
            for (int r = 0; r < P; r++) v[r] = 0.f;
        }
        for (int t = 0; t < n; t += S * UFK) {
            float b[UFK][F];
            float a[UFK][P];
#pragma unroll
            for (int u = 0; u < UFK; u++) {
                const int tt = t + u * S + sub;
                const int src = tt & 31;
                const int cc = __shfl_sync(kFull, col, src);
#pragma unroll
                for (int r = 0; r < P; r++) a[u][r] = __shfl_sync(kFull, v[r], src);
                if (tt < n) {
                    Map::load(b[u], p.B + (size_t)cc * p.n, p.n, lj);
                } else {
#pragma unroll
                    for (int f = 0; f < F; f++) b[u][f] = 0.f;
                }
            }
#pragma unroll
            for (int u = 0; u < UFK; u++) {
                if constexpr (PROBE) {
#pragma unroll
                    for (int f = 0; f < F; f++) acc[0][f] += b[u][f];
                } else {
                    int rank = 0;
#pragma unroll
                    for (int row = 0; row < H; row++) {
                        if ((MASK >> row) & 1) {
#pragma unroll
                            for (int f = 0; f < F; f++)
                                acc[row][f] = fmaf(a[u][rank], b[u][f], acc[row][f]);
                            rank++;
                        }
                    }
                }
            }
        }
    }
}

// Warp-uniform pattern switch (one specialised body per enumerated block).
template <int H, class Map, int UFK, bool PROBE, int M = 1>
__device__ __forceinline__ void dispatch_mask(int mask, const KParams& p, float (&acc)[H][Map::F],
                                              int cbeg, int vbase, int pos, int gend, int lane,
                                              int sub, int lj) {
    if constexpr (M < (1 << H)) {
        if (mask == M)
            run_group<H, M, Map, UFK, PROBE>(p, acc, cbeg, vbase, pos, gend, lane, sub, lj);
        else
            dispatch_mask<H, Map, UFK, PROBE, M + 1>(mask, p, acc, cbeg, vbase, pos, gend, lane,
                                                     sub, lj);
    }
}

template <int H, class Map>
__device__ __forceinline__ void store_rows(const KParams& p, int panel, const float (&a)[H][Map::F],
                                           int sub, int lj) {
#pragma unroll
    for (int r = 0; r < H; r++) {
        const int row = panel * H + r;
        if ((r % Map::S) == sub && row < p.m) Map::store(p.C + (size_t)row * p.n, a[r], p.n, lj);
    }
}

template <int H, class Map, int UFK, bool PROBE>
__global__ void __launch_bounds__(512) esc_spmm_kernel(KParams p) {
    extern __shared__ float red[];   // [W][H][n] partials of split panels
    constexpr int F = Map::F, S = Map::S, L = Map::L;
    const int4 ti = p.tiles[blockIdx.x];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sub = lane / L, lj = lane % L;
    const int item = ti.x + w;
    const bool active = item < ti.y;

    float acc[H][F];
#pragma unroll
    for (int r = 0; r < H; r++)
#pragma unroll
        for (int f = 0; f < F; f++) acc[r][f] = 0.f;

    int panel = 0, aux = 0;
    if (active) {
        const int4 it = p.items[item];
        aux = p.item_aux[item];
        panel = it.x;
        int g = it.y, pos = it.z;
        const int end = it.w;
        while (pos < end) {
            const int4 gi = p.grp[g];
            const int gend = min(end, gi.y);
            dispatch_mask<H, Map, UFK, PROBE>(gi.w, p, acc, gi.x, gi.z, pos, gend, lane, sub, lj);
            pos = gend;
            ++g;
        }
        if constexpr (S > 1) {   // warp-level reduction of the sub-warps
#pragma unroll
            for (int r = 0; r < H; r++)
#pragma unroll
                for (int f = 0; f < F; f++)
#pragma unroll
                    for (int off = L; off < 32; off <<= 1)
                        acc[r][f] += __shfl_xor_sync(kFull, acc[r][f], off);
        }
    }

    if constexpr (PROBE) {
        if (active) {
            float s = 0.f;
#pragma unroll
            for (int f = 0; f < F; f++) s += acc[0][f];
            p.C[((size_t)blockIdx.x * blockDim.x) + threadIdx.x] = s;
        }
        return;
    } else {
        const int n = p.n;
        const bool heavy = ti.z >= 0;
        const int cnt = aux >> 8, lead = aux & 0xff;
        if (!(ti.w & 1)) {   // every panel of this tile has exactly one item here
            if (active) store_rows<H, Map>(p, panel, acc, sub, lj);
            return;
        }
        float* mine = red + (size_t)w * H * n;
        if (active && (cnt > 1 || heavy)) {
#pragma unroll
            for (int r = 0; r < H; r++)
                if ((r % S) == sub)
#pragma unroll
                    for (int f = 0; f < F; f++) {
                        const int j = Map::col(lj, f);
                        if (Map::kVec || j < n) mine[r * n + j] = acc[r][f];
                    }
        }
        __syncthreads();
        if (!active) return;
        if (cnt == 1 && !heavy) {
            store_rows<H, Map>(p, panel, acc, sub, lj);
            return;
        }
        if (w != lead) return;
        // combine the panel's partials in item order (deterministic)
        float tot[H][F];
#pragma unroll
        for (int r = 0; r < H; r++)
#pragma unroll
            for (int f = 0; f < F; f++) {
                const int j = Map::col(lj, f);
                float s = 0.f;
                if (Map::kVec || j < n)
                    for (int q = 0; q < cnt; q++) s += red[((size_t)(lead + q) * H + r) * n + j];
                tot[r][f] = s;
            }
        if (!heavy) {
            store_rows<H, Map>(p, panel, tot, sub, lj);
            return;
        }
        // heavy panel: tiles combine through the global workspace
        const int4 hv = p.heavy[ti.z];
        const int q = ti.w >> 1;
        float* wsq = p.ws + (size_t)(hv.y + q) * H * n;
#pragma unroll
        for (int r = 0; r < H; r++)
            if ((r % S) == sub)
#pragma unroll
                for (int f = 0; f < F; f++) {
                    const int j = Map::col(lj, f);
                    if (Map::kVec || j < n) __stcg(wsq + r * n + j, tot[r][f]);
                }
        __threadfence();
        __syncwarp();
        int last = 0;
        if (lane == 0) last = (atomicAdd(p.counters + ti.z, 1) == hv.z - 1);
        last = __shfl_sync(kFull, last, 0);
        if (!last) return;
        __threadfence();
#pragma unroll
        for (int r = 0; r < H; r++)
#pragma unroll
            for (int f = 0; f < F; f++) {
                const int j = Map::col(lj, f);
                float s = 0.f;
                if (Map::kVec || j < n)
                    for (int t = 0; t < hv.z; t++)
                        s += __ldcg(p.ws + ((size_t)(hv.y + t) * H + r) * n + j);
                tot[r][f] = s;
            }
        store_rows<H, Map>(p, hv.x, tot, sub, lj);
        if (lane == 0) p.counters[ti.z] = 0;   // self-reset: graph replay safe
    }
}

using KernelFn = void (*)(KParams);

}  // namespace kern
}  // namespace escs
