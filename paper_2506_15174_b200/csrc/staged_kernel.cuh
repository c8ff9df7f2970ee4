// staged_kernel.cuh -- the staged record walk: the enumerated, sparse-coarsened
// SpMM with the B rows of a CTA's column range staged in shared memory by
// TMA bulk copies (sm_100a).
//
// Why (profiles/r2_notes.md §1): the record walk of
// esc_kernel.cuh gathers every B row it multiplies from L2; on B200 an L2
// row gather costs ~7.6 clk per 512 bytes per SM, twice the L1/shared-memory
// data path (~4 clk), and the L1 hit rate of the walk is 7-15% because the
// warps of an SM walk unrelated panels across all k columns.  Here a CTA owns
// a row block (W warps x NPW panels of UFi rows) and one k-range ("split") of
// A; the B rows of that range and the CTA's records are copied into shared
// memory by cp.async.bulk (one elected lane per stage, mbarrier completion),
// and every gathered B row is then a shared-memory read reused for all
// nonzeros of the row block in that column -- the enumeration's register reuse
// (popcount(pattern) rows per loaded B element, §3.3.2) on top.
//
// Paper mapping (arXiv 2506.15174):
//   * enumeration (§3.2): a warp walks the records of its panels
//     (UFi rows each); record = (column, UFi-bit pattern, the pattern rows'
//     values) -- the packed record of escs_pack (esc_kernel.cuh RecFmt), so
//     each column runs the enumerated block of its pattern (Listing 4,
//     P:293-310), realised as predicates on the warp-uniform pattern bits;
//   * thread coarsening (§3.3.2): each lane keeps NPW x UFi x F accumulators,
//     a B element loaded once is reused for every row of the pattern;
//   * data transformation (§3.3.3): the records are stored by
//     (CTA, stage, warp slot) -- the canonical gcol order of each panel cut at
//     the stage boundaries -- so one bulk copy per stage brings them in;
//   * combine: the splits of a row block are summed in split order by a
//     second, tiny kernel (esc_staged_reduce_kernel): deterministic, C
//     overwritten (beta = 0), no atomics (Reading R10).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "esc_kernel.cuh"

namespace escs {
namespace kern {

constexpr int kStMaxStages = 16;   // mbarriers per CTA (stages of one k-range)

struct SParams {
    const int4* __restrict__ cta;     // per CTA: rb, split, stage_begin, n_stage
    const int4* __restrict__ stage;   // per stage: ks, ke, rec_begin (records, absolute), n_rec (padded)
    const int* __restrict__ hdr;      // per stage: HS ints: record offset of each warp slot (CTA-relative), end
    const int* __restrict__ rec;      // packed staged record stream (escs_pack)
    const float* __restrict__ B;
    float* __restrict__ C;            // nsplit == 1: C, else the split workspace [nsplit][m][n]
    int m, n, hs, nslot;              // hs: header ints per stage (nslot + 1 rounded to 4)
    int sb_floats;                    // shared floats reserved for B (max CTA k-range x n)
    int sr_words;                     // shared words reserved for records
    long long split_stride;           // floats between two splits' partials (m * n), 0 if nsplit == 1
    // in-kernel combine of the splits (coop = 1: the grid is co-resident,
    // launched cooperatively): the CTAs of a row block meet at counters[2*rb]
    // and each sums a slice of the block's partials into Cout
    float* Cout;
    int* counters;                    // 2 per row block: arrivals, departures (self-resetting)
    int nsplit, coop;
    int rows_per_block;               // nslot x UFi
    int max_st;                       // stages per CTA (stage table and header stride)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Bulk global -> shared copy completing on an mbarrier (TMA, non-tensor form:
// contiguous bytes, 16-byte aligned, size a multiple of 16).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         unsigned long long pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// Read the first NW words of a shared-memory record (stride RecFmt<H>::W, a
// multiple of 4 words beyond UFi = 1, so reading a pad word is harmless).
template <int NW, int RR>
__device__ __forceinline__ void lds_rec(int (&r)[RR], const int* q) {
    if constexpr (NW <= 2) {
        const int2 x = *reinterpret_cast<const int2*>(q);
        r[0] = x.x; r[1] = x.y;
    } else {
#pragma unroll
        for (int v = 0; v < (NW + 3) / 4; v++) {
            if (NW - 4 * v == 1) {
                r[4 * v] = q[4 * v];
            } else {
                const int4 x = *reinterpret_cast<const int4*>(q + 4 * v);
                r[4 * v] = x.x; r[4 * v + 1] = x.y; r[4 * v + 2] = x.z; r[4 * v + 3] = x.w;
            }
        }
    }
}

// One batch of U records per sub-warp (U*S per warp) from shared memory:
// record loads, then the U B rows (shared), then the pattern rows' FMAs.
// TAIL: slots past `end` re-read the last record and multiply nothing.
template <int H, class Map, int U, bool TAIL, bool PROBE>
__device__ __forceinline__ void st_batch(const int* sR, const float* sB, int k0, int i, int end,
                                         int sub, int lj, float (&acc)[H][Map::F]) {
    constexpr int F = Map::F, S = Map::S, RW = RecFmt<H>::W, NWR = RecFmt<H>::Words;
    constexpr int N = Map::L * Map::F;
    constexpr int RR = NWR > 2 ? (NWR + 3) / 4 * 4 : 2;
    int r[U][RR];
    float b[U][F];
#pragma unroll
    for (int u = 0; u < U; u++) {
        const int idx = i + u * S + sub;
        lds_rec<NWR, RR>(r[u], sR + (size_t)(TAIL ? min(idx, end - 1) : idx) * RW);
        if (TAIL && H > 1 && idx >= end) r[u][0] &= RecFmt<H>::ColMask;   // no pattern rows
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
        const int col = (H == 1 ? r[u][0] : (r[u][0] & RecFmt<H>::ColMask)) - k0;
        const float* row = sB + (size_t)col * N;
#pragma unroll
        for (int v = 0; v < F / 4; v++) {
            const float4 x = *reinterpret_cast<const float4*>(row + 4 * (F == 4 ? lj : v * Map::L + lj));
            b[u][4 * v] = x.x; b[u][4 * v + 1] = x.y; b[u][4 * v + 2] = x.z; b[u][4 * v + 3] = x.w;
        }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
        if constexpr (PROBE) {   // the gather probe: the same loads, no FMAs
#pragma unroll
            for (int f = 0; f < F; f++) acc[0][f] += b[u][f];
        } else if constexpr (H == 1) {
            if (!TAIL || i + u * S + sub < end) fma_row<F>(acc[0], __int_as_float(r[u][1]), b[u]);
        } else {
            const unsigned mk = (unsigned)r[u][0] >> RecFmt<H>::Shift;
            {
#pragma unroll
                for (int row = 0; row < H; row++)
                    if ((mk >> row) & 1u) fma_row<F>(acc[row], __int_as_float(r[u][1 + row]), b[u]);
            }
        }
    }
}

template <int H, class Map, int U, bool PROBE>
__device__ __forceinline__ void st_walk(const int* sR, const float* sB, int k0, int beg, int end,
                                        int sub, int lj, float (&acc)[H][Map::F]) {
    constexpr int US = U * Map::S;
    int i = beg;
#pragma unroll 1
    for (; i + US <= end; i += US) st_batch<H, Map, U, false, PROBE>(sR, sB, k0, i, end, sub, lj, acc);
    if (i < end) st_batch<H, Map, U, true, PROBE>(sR, sB, k0, i, end, sub, lj, acc);
}
// In-kernel combine of a row block's split partials (cooperative launch: all
// CTAs are resident, so the spin below cannot wait on an unscheduled CTA).
// Each CTA publishes its partial (release), waits until the block's nsplit
// CTAs have (acquire), then sums slice `sp` of the block's rows over all
// splits and writes C.  The order of every sum is fixed: deterministic.  The
// CTA's threads form G groups; group g sums splits [g*ns/G, (g+1)*ns/G) of
// the slice's float4s (several loads in flight per thread), the groups'
// results are added in group order through shared memory.  The last CTA to
// leave resets the block's counters (graph replay safe).
__device__ __forceinline__ void st_combine(const SParams& p, int rb, int sp) {
    const int tid = threadIdx.x, nth = blockDim.x;
    __shared__ float4 part[512];
    int* cnt = p.counters + 2 * rb;
    asm volatile("bar.sync 0;" ::: "memory");   // the CTA's partial stores precede the release
    if (tid == 0) {
        asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(cnt) : "memory");
        int v = 0;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
            if (v >= p.nsplit) break;
            __nanosleep(32);
        }
    }
    asm volatile("bar.sync 0;" ::: "memory");   // ... and the acquire precedes every thread's loads
    // this CTA's slice [a, b) of the block's rows, as float4s of C
    const long long n4 = p.n / 4;
    const long long e0 = (long long)rb * p.rows_per_block * n4;
    const long long e1 = min((long long)p.m, (long long)(rb + 1) * p.rows_per_block) * n4;
    const long long a = e0 + (e1 - e0) * sp / p.nsplit, b = e0 + (e1 - e0) * (sp + 1) / p.nsplit;
    const int ne = (int)(b - a);
    const float4* ws = reinterpret_cast<const float4*>(p.C);
    const long long stride4 = p.split_stride / 4;
    float4* c4 = reinterpret_cast<float4*>(p.Cout);
    const int per = min(nth, (ne + 31) / 32 * 32);          // threads per group
    const int G = per > 0 ? max(1, min(nth / per, p.nsplit)) : 1;
    const int g = per > 0 ? tid / per : G, e = per > 0 ? tid % per : 0;
    if (g < G) {
        const int s0 = g * p.nsplit / G, s1 = (g + 1) * p.nsplit / G;
        for (int x = e; x < ne; x += per) {
            float4 acc = __ldcg(ws + s0 * stride4 + a + x);
            int s = s0 + 1;
            for (; s + 4 <= s1; s += 4) {   // four splits' loads in flight, summed in split order
                float4 q[4];
#pragma unroll
                for (int d = 0; d < 4; d++) q[d] = __ldcg(ws + (s + d) * stride4 + a + x);
#pragma unroll
                for (int d = 0; d < 4; d++) {
                    acc.x += q[d].x; acc.y += q[d].y; acc.z += q[d].z; acc.w += q[d].w;
                }
            }
            for (; s < s1; s++) {
                const float4 q = __ldcg(ws + s * stride4 + a + x);
                acc.x += q.x; acc.y += q.y; acc.z += q.z; acc.w += q.w;
            }
            if (G == 1) c4[a + x] = acc;
            else part[g * ne + x] = acc;   // G > 1: ne <= per and G * per <= nth <= 512
        }
    }
    if (G > 1) {
        asm volatile("bar.sync 0;" ::: "memory");
        for (int x = tid; x < ne; x += nth) {
            float4 acc = part[x];
            for (int q = 1; q < G; q++) {
                const float4 y = part[q * ne + x];
                acc.x += y.x; acc.y += y.y; acc.z += y.z; acc.w += y.w;
            }
            c4[a + x] = acc;
        }
    }
    if (tid == 0) {
        int old;
        asm volatile("atom.relaxed.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(cnt + 1) : "memory");
        if (old == p.nsplit - 1) {   // every CTA of the block is past its spin: reset
            cnt[0] = 0;
            cnt[1] = 0;
        }
    }
}

// Register target: the accumulators, a batch of records and of B values with
// room for ptxas to keep the next batch's loads in flight, plus ~24 for
// addressing; capped at 128 (512 threads per SM at one CTA).  Without a
// target ptxas takes all 128 for every instance, which leaves the narrow
// tiles one CTA per SM.
template <int H, class Map, int U, int NPW>
struct StRegs {
    static constexpr int RR = RecFmt<H>::Words > 2 ? (RecFmt<H>::Words + 3) / 4 * 4 : 2;
    static constexpr int raw = NPW * H * Map::F + U * (2 * RR + Map::F) + 24;
    static constexpr int value = raw > 128 ? 128 : (raw + 7) / 8 * 8;
};
#ifndef ESC_ST_REGCAP
#define ESC_ST_REGCAP 1
#endif
#if ESC_ST_REGCAP
#define ESC_ST_BOUNDS __maxnreg__((StRegs<H, Map, U, NPW>::value))
#else
#define ESC_ST_BOUNDS __launch_bounds__(512, 1)
#endif
template <int H, class Map, int U, int NPW, bool PROBE>
__global__ void ESC_ST_BOUNDS esc_staged_kernel(const __grid_constant__ SParams p) {
    constexpr int F = Map::F, S = Map::S, N = Map::L * Map::F, RW = RecFmt<H>::W;
    static_assert(Map::kVec, "vector lane maps only");
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t bar[kStMaxStages];
    float* sB = smem;
    int* sR = reinterpret_cast<int*>(smem + p.sb_floats);
    int* sH = sR + p.sr_words;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    const int sub = lane / Map::L, lj = lane % Map::L;

    grid_dep_launch();
    // the plan (immutable): before the PDL wait, all loads independent --
    // this CTA's stages sit at blockIdx * max_stages (zero-padded)
    const int nst = p.max_st, sbase = blockIdx.x * nst;
    const int4 ci = p.cta[blockIdx.x];   // rb, split (for the output rows and the combine)
    const int k0 = p.stage[sbase].x;     // first column of the CTA's range
    if (tid == 0) {
        for (int s = 0; s < nst; s++) mbar_init(&bar[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (w == 0) {
        const unsigned long long pol_first = policy_first(), pol_last = policy_last();
        int4 st = make_int4(0, 0, 0, 0);
        if (lane < nst) st = p.stage[sbase + lane];
        const int rec0 = __shfl_sync(kFull, st.z, 0);
        uint32_t bbytes = 0;
        if (lane < nst) {
            const uint32_t rbytes = (uint32_t)st.w * RW * 4;
            bbytes = st.w > 0 ? (uint32_t)(st.y - st.x) * N * 4 : 0u;   // no records: no B rows needed
            const uint32_t hbytes = lane == 0 ? (uint32_t)nst * p.hs * 4 : 0u;
            mbar_arrive_expect_tx(&bar[lane], rbytes + bbytes + hbytes);
            // the plan headers and the record stream are immutable: fetched
            // before the programmatic-dependent-launch wait
            if (hbytes) bulk_g2s(sH, p.hdr + (size_t)sbase * p.hs, hbytes, &bar[0], pol_first);
            if (rbytes) bulk_g2s(sR + (size_t)(st.z - rec0) * RW, p.rec + (size_t)st.z * RW, rbytes, &bar[lane], pol_first);
            // B's stage rows into L2 already (a hint; L2 is coherent, L1 is not
            // filled), so the copies below, after the wait, hit L2 on a cold B
            if (bbytes) prefetch_l2_bulk(p.B + (size_t)st.x * N, bbytes);
        }
        grid_dep_wait();   // B is caller data written by the previous kernel
        if (lane < nst && bbytes)
            bulk_g2s(sB + (size_t)(st.x - k0) * N, p.B + (size_t)st.x * N, bbytes, &bar[lane], pol_last);
    } else {
        grid_dep_wait();   // C / workspace writes after the previous kernel
    }

    float acc[NPW][H][F];
#pragma unroll
    for (int q = 0; q < NPW; q++)
#pragma unroll
        for (int r = 0; r < H; r++)
#pragma unroll
            for (int f = 0; f < F; f++) acc[q][r][f] = 0.f;

#pragma unroll 1
    for (int s = 0; s < nst; s++) {
        mbar_wait(&bar[s], 0);
        const int* hs = sH + s * p.hs + w * NPW;
#pragma unroll
        for (int q = 0; q < NPW; q++) st_walk<H, Map, U, PROBE>(sR, sB, k0, hs[q], hs[q + 1], sub, lj, acc[q]);
    }
    if constexpr (S > 1) {   // warp-level reduction of the sub-warps
#pragma unroll
        for (int q = 0; q < NPW; q++)
#pragma unroll
            for (int r = 0; r < H; r++)
#pragma unroll
                for (int f = 0; f < F; f++)
#pragma unroll
                    for (int off = Map::L; off < 32; off <<= 1)
                        acc[q][r][f] += __shfl_xor_sync(kFull, acc[q][r][f], off);
    }
    if constexpr (PROBE) {   // one float per warp-lane into the sink (p.C): the loads are not dead
        float t = 0.f;
#pragma unroll
        for (int q = 0; q < NPW; q++)
#pragma unroll
            for (int f = 0; f < F; f++) t += acc[q][0][f];
        p.C[((size_t)blockIdx.x * (blockDim.x >> 5) + w) * 32 + lane] = t;
        return;
    }
    // every row of the row block is written (zeros where the split has no
    // nonzero): the reduction sums all splits
    float* out = p.C + (size_t)ci.y * p.split_stride;
#pragma unroll
    for (int q = 0; q < NPW; q++) {
        const int panel = ci.x * p.nslot + w * NPW + q;
#pragma unroll
        for (int r = 0; r < H; r++) {
            const int row = panel * H + r;
            if ((r % S) == sub && row < p.m) Map::store(out + (size_t)row * p.n, acc[q][r], p.n, lj);
        }
    }
    if (p.coop) st_combine(p, ci.x, ci.y);
}

// Fallback combine (a plan whose grid cannot be co-resident): C = sum over
// splits of the workspace partials, in split order (deterministic); one
// float4 per thread, four splits' loads in flight.
template <int kUnused = 0>
__global__ void __launch_bounds__(128) esc_staged_reduce_kernel(const float* __restrict__ ws, float* __restrict__ C,
                                                                long long n4, long long stride4, int nsplit) {
    grid_dep_launch();
    grid_dep_wait();
    const float4* w4 = reinterpret_cast<const float4*>(ws);
    float4* c4 = reinterpret_cast<float4*>(C);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        float4 a = __ldcg(w4 + i);
        int s = 1;
        for (; s + 4 <= nsplit; s += 4) {
            float4 q[4];
#pragma unroll
            for (int d = 0; d < 4; d++) q[d] = __ldcg(w4 + (s + d) * stride4 + i);
#pragma unroll
            for (int d = 0; d < 4; d++) {
                a.x += q[d].x; a.y += q[d].y; a.z += q[d].z; a.w += q[d].w;
            }
        }
        for (; s < nsplit; s++) {
            const float4 x = __ldcg(w4 + s * stride4 + i);
            a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
        }
        c4[i] = a;
    }
}

using StagedFn = void (*)(SParams);
StagedFn get_staged(int n, int F, int h, int npw, bool probe);

}  // namespace kern
}  // namespace escs
