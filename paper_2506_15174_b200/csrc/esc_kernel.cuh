// esc_kernel.cuh -- the enumerate-and-sparse-coarsen SpMM kernel for sm_100a.
//
// Paper mapping (arXiv 2506.15174):
//   * enumeration (§3.2): a warp works on one item (a balanced
//     slice of one UFi = H row panel's column stream).  The stream is sorted by
//     pattern, so consecutive columns share one UFi-bit pattern; every column
//     runs the enumerated block of its pattern (Listing 4): the
//     pattern is warp-uniform, its bits predicate the row FMAs, so exactly
//     popcount(pattern) rows accumulate and no lane diverges;
//   * thread mapping map(j, W) (§3.3.1): the 32 lanes own the
//     bCols columns of B/C (F consecutive floats per lane on the vector map,
//     32-strided scalars on the scalar map = the paper's WarpTile mapping);
//   * thread coarsening (§3.3.2): each lane keeps H x F
//     accumulators (pattern rows x its columns); a B element loaded once into a
//     register is reused for every row of the pattern, an A value for all the
//     lane's columns; columns are processed in batches of UFK gathered B rows
//     in flight per warp;
//   * data transformation (§3.3.3): columns ("Cols", packed with
//     their pattern) and value slots ("ANNZ" order, Reading R1) are staged 32
//     at a time by the warp with coalesced loads, one chunk ahead, and
//     broadcast with __shfl_sync;
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
constexpr int kColBits = 27;                       // packed gcol: col | mask << 27
constexpr int kColMask = (1 << kColBits) - 1;
constexpr int kMaxScatter = 8;
#ifndef ESC_MINB
#define ESC_MINB 1   // min resident 512-thread blocks per SM in __launch_bounds__ (0: none)
#endif
#if ESC_MINB > 0
#define ESC_CSR_BOUNDS __launch_bounds__(512, ESC_MINB)
#else
#define ESC_CSR_BOUNDS __launch_bounds__(512)
#endif

struct KParams {
    const int* __restrict__ gpk;       // packed gcols: column | pattern << 27
    const int* __restrict__ slot;      // value slot -> CSR position
    const int4* __restrict__ items;    // per slot: panel, gcol_begin, gcol_end, slot_begin
    const int* __restrict__ item_aux;  // per slot: lead | cnt<<8 | active<<16 | sync<<17 | heavy<<18
    const int2* __restrict__ tile_heavy; // per tile: heavy id, ordinal (heavy tiles only)
    const int4* __restrict__ heavy;    // panel, ws_base, ntiles, 0
    float* ws;
    int* counters;                     // heavy-panel arrival counters
    const float* __restrict__ vals;    // CSR values, or the packed record stream (kRec)
    const float* __restrict__ B;
    float* __restrict__ C;
    int m, n;
    int k;                             // rows of B (the walk's L2 prefetch of B)
    const int* __restrict__ rowmap;    // plan row -> row of C (a hybrid plan's part), NULL = identity
    const int4* __restrict__ slot_ws;  // column-window tiles: per slot {ws offset, counter, items, ordinal}
    float* wsc;                        // column-window tiles: per-item partials
    int* wsc_counters;
    // fused row-block all-gather (escs_spmm_scatter): every output row is
    // also stored to extra[d] + (row_off + row) * n, d < n_extra -- the peers'
    // C buffers (P2P / NVLink stores through mapped symmetric memory)
    int n_extra, mc;                               // mc: extra[0] is a multicast address
    long long row_off;
    float* extra[kMaxScatter];
    static constexpr bool kScatter = true;
};

// L2 cache policies: the plan and value streams are read once per call
// (evict_first); the gathered B rows are re-read by many panels and should
// stay L2-resident across the streams (evict_last).  createpolicy folds into
// the load's uniform descriptor (no per-load cost).
__device__ __forceinline__ unsigned long long policy_first() {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ unsigned long long policy_last() {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// Programmatic dependent launch (PDL): the plan is immutable, so a launch may
// read it while the previous kernel in the stream is still finishing; every
// read of caller data (vals, B) and every write of C happens after
// griddepcontrol.wait (the previous grid has completed and its writes are
// visible).  No-ops when the launch carries no programmatic dependency.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;"); }

// The plan and value streams are read front to back: each miss fetches 256 B
// into L2 (the next chunk's line rides along; C4 81.3 -> 80.3 us, suite
// +0.3-1.2%).  The same hint on the gathered B rows measured no gain.
#define ESC_STREAM_PF ".L2::256B"
__device__ __forceinline__ int ld_stream(const int* p) {
    int r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint" ESC_STREAM_PF ".s32 %0, [%1], %2;"
                 : "=r"(r) : "l"(p), "l"(policy_first()));
    return r;
}
__device__ __forceinline__ float ld_stream_f(const float* p) {
    float r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint" ESC_STREAM_PF ".f32 %0, [%1], %2;"
                 : "=f"(r) : "l"(p), "l"(policy_first()));
    return r;
}

// L1 eviction priorities of the gathered B rows and of the record loads
// (experiment hooks; empty = the default, evict_normal)
#ifndef ESC_B_L1
#define ESC_B_L1 ""
#endif
#ifndef ESC_REC_L1
#define ESC_REC_L1 ""
#endif

// Vector lane map: L lanes own one gathered B row of N = L*F floats (F
// consecutive floats per lane, 128-bit loads for F >= 4), so a warp gathers
// S = 32/L rows per step ("sub-warps"); sub-warp partial sums are reduced
// with shfl_xor at the end of the item (the warp-level reduction of P:450).
// acc[f] += a * b[f] for f < F.  Pairs go through FFMA2 (fma.rn.f32x2,
// sm_100): per element the same correctly rounded fma as fmaf, so results are
// bit-identical, at half the FMA instructions (the 3-register FFMA issues at
// half rate per SMSP on Blackwell, B300_MICROARCH "Pipe rates").
template <int F>
__device__ __forceinline__ void fma_row(float (&acc)[F], float a, const float (&b)[F]) {
#pragma unroll
    for (int f = 0; f + 1 < F; f += 2) {
        const float2 r = __ffma2_rn(make_float2(b[f], b[f + 1]), make_float2(a, a),
                                    make_float2(acc[f], acc[f + 1]));
        acc[f] = r.x;
        acc[f + 1] = r.y;
    }
    if constexpr (F % 2) acc[F - 1] = fmaf(a, b[F - 1], acc[F - 1]);
}

template <int L_, int F_>
struct VecMap {
    static constexpr int L = L_, F = F_, S = 32 / L_;
    static constexpr bool kVec = true;
    // F > 4: float4 v of lane lj sits at column (v*L + lj)*4, so each 128-bit
    // load instruction of the L lanes reads one contiguous L*16-byte span (one
    // L1 wavefront per 128-byte line, no strided replays)
    __device__ static __forceinline__ int col(int lj, int f) {
        return F <= 4 ? lj * F + f : (((f >> 2) * L + lj) << 2) + (f & 3);
    }
    __device__ static __forceinline__ void load(float (&b)[F], const float* row, int, int lj) {
        load_pol(b, row, lj, policy_last());
    }
    __device__ static __forceinline__ void load_pol(float (&b)[F], const float* row, int lj,
                                                    unsigned long long pol) {
        const float* q = row + (F <= 4 ? lj * F : 4 * lj);
        if constexpr (F == 1) {
            asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;"
                         : "=f"(b[0]) : "l"(q), "l"(pol));
        } else if constexpr (F == 2) {
            asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
                         : "=f"(b[0]), "=f"(b[1]) : "l"(q), "l"(pol));
        } else {
#pragma unroll
            for (int v = 0; v < F / 4; v++)
                asm volatile("ld.global.nc" ESC_B_L1 ".L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                             : "=f"(b[4 * v]), "=f"(b[4 * v + 1]), "=f"(b[4 * v + 2]),
                               "=f"(b[4 * v + 3])
                             : "l"(q + 4 * v * L), "l"(pol));
        }
    }
    __device__ static __forceinline__ void store(float* row, const float (&a)[F], int, int lj) {
        float* q = row + (F <= 4 ? lj * F : 4 * lj);
        if constexpr (F == 1) {
            q[0] = a[0];
        } else if constexpr (F == 2) {
            *reinterpret_cast<float2*>(q) = make_float2(a[0], a[1]);
        } else {
#pragma unroll
            for (int v = 0; v < F / 4; v++)
                *reinterpret_cast<float4*>(q + 4 * v * L) =
                    make_float4(a[4 * v], a[4 * v + 1], a[4 * v + 2], a[4 * v + 3]);
        }
    }
    // Store through an NVLS multicast address (one store lands in every
    // GPU's copy of C; escs_spmm_scatter with ESCS_SCATTER_MULTICAST).
    __device__ static __forceinline__ void store_mc(float* row, const float (&a)[F], int, int lj) {
        float* q = row + (F <= 4 ? lj * F : 4 * lj);
        if constexpr (F == 1) {
            asm volatile("multimem.st.weak.global.f32 [%0], %1;" :: "l"(q), "f"(a[0]) : "memory");
        } else if constexpr (F == 2) {
            asm volatile("multimem.st.weak.global.v2.f32 [%0], {%1,%2};"
                         :: "l"(q), "f"(a[0]), "f"(a[1]) : "memory");
        } else {
#pragma unroll
            for (int v = 0; v < F / 4; v++)
                asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1,%2,%3,%4};"
                             :: "l"(q + 4 * v * L), "f"(a[4 * v]), "f"(a[4 * v + 1]),
                                "f"(a[4 * v + 2]), "f"(a[4 * v + 3]) : "memory");
        }
    }
};

// Scalar lane map (the paper's map(j, 32*WarpTile), Listings 5-6): lane owns
// columns lane + 32*f, f < WT, predicated on j < N.  Any N <= 32*WT, any
// alignment.  One gathered row per warp step.
template <int WT>
struct ScalarMap {
    static constexpr int L = 32, F = WT, S = 1;
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
    __device__ static __forceinline__ void store_mc(float* row, const float (&a)[F], int n, int lj) {
#pragma unroll
        for (int f = 0; f < F; f++) {
            const int j = lj + 32 * f;
            if (j < n)
                asm volatile("multimem.st.weak.global.f32 [%0], %1;" :: "l"(row + j), "f"(a[f])
                             : "memory");
        }
    }
};

// Per-warp staging area in shared memory, double-buffered by chunk: the 32
// packed words of a chunk and, per column, the value of every pattern row
// (0 for rows outside the pattern), so one broadcast LDS gives a column's
// pattern and all its row values.
template <int H>
struct Stage {
    static constexpr int HP = H == 3 ? 4 : H;   // row values padded to a vector
    int pk[2][32];
    float w[2][32][HP];
};

template <int H>
__device__ __forceinline__ void put_chunk(Stage<H>& st, int buf, int lane, int pk,
                                          const float (&w)[H]) {
    st.pk[buf][lane] = pk;
    if constexpr (Stage<H>::HP == 4) {
        float x[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int r = 0; r < H; r++) x[r] = w[r];
        *reinterpret_cast<float4*>(&st.w[buf][lane][0]) = make_float4(x[0], x[1], x[2], x[3]);
    } else if constexpr (H == 2) {
        *reinterpret_cast<float2*>(&st.w[buf][lane][0]) = make_float2(w[0], w[1]);
    } else {
        st.w[buf][lane][0] = w[0];
    }
}

template <int H>
__device__ __forceinline__ void get_vals(const Stage<H>& st, int buf, int s, float (&a)[H]) {
    if constexpr (Stage<H>::HP == 4) {
        const float4 x = *reinterpret_cast<const float4*>(&st.w[buf][s][0]);
        const float y[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int r = 0; r < H; r++) a[r] = y[r];
    } else if constexpr (H == 2) {
        const float2 x = *reinterpret_cast<const float2*>(&st.w[buf][s][0]);
        a[0] = x.x; a[1] = x.y;
    } else {
        a[0] = st.w[buf][s][0];
    }
}

// UFi = 1: every column has the single pattern 0b1 and the slot map is the
// identity (a panel is one CSR row, its value slots are that row's CSR
// positions in order), so column i of an item reads vals[sbase + i]
// directly -- contiguous, no second indirection.  Column index and value of
// the current and next chunk live in registers and are broadcast with
// __shfl_sync (each sub-warp reads its own column).  Full batches run
// unpredicated; the last partial batch of an item predicates its FMAs
// (structural zeros are never multiplied).
template <class Map, int U, bool PROBE, class PP>
__device__ __forceinline__ void walk1(const PP& p, int beg, int end, int sbase,
                                      float (&acc)[1][Map::F], int lane) {
    constexpr int F = Map::F, S = Map::S, US = U * S;
    static_assert(32 % US == 0, "UFK * sub-warps must divide 32");
    const int sub = lane / Map::L, lj = lane % Map::L;
    const int n = end - beg;
    const int* gp = p.gpk + beg;
    const float* vp = p.vals + sbase;
    int pk0 = 0, pk1 = 0;
    float v0 = 0.f, v1 = 0.f;
    if (lane < n) pk0 = ld_stream(gp + lane);          // plan: before the PDL wait
    if (32 + lane < n) pk1 = ld_stream(gp + 32 + lane);
    grid_dep_wait();
    if constexpr (!PROBE) {
        if (lane < n) v0 = ld_stream_f(vp + lane);
        if (32 + lane < n) v1 = ld_stream_f(vp + 32 + lane);
    }
#pragma unroll 1
    for (int c0 = 0; c0 < n; c0 += 32) {
        int pk2 = 0;
        float v2 = 0.f;
        if (c0 + 64 + lane < n) {
            pk2 = ld_stream(gp + c0 + 64 + lane);
            if constexpr (!PROBE) v2 = ld_stream_f(vp + c0 + 64 + lane);
        }
        const int cn = min(32, n - c0);
        int s = 0;
#pragma unroll 1
        for (; s + US <= cn; s += US) {
            float b[U][F];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int c = __shfl_sync(kFull, pk0, s + u * S + sub) & kColMask;
                Map::load(b[u], p.B + (size_t)c * p.n, p.n, lj);
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const float a = PROBE ? 1.f : __shfl_sync(kFull, v0, s + u * S + sub);
#pragma unroll
                fma_row<F>(acc[0], a, b[u]);
            }
        }
        if (s < cn) {   // partial batch
            float b[U][F];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int c = __shfl_sync(kFull, pk0, (s + u * S + sub) & 31) & kColMask;
                Map::load(b[u], p.B + (size_t)c * p.n, p.n, lj);
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int ci = s + u * S + sub;
                const float a = PROBE ? 1.f : __shfl_sync(kFull, v0, ci & 31);
                if (ci < cn) fma_row<F>(acc[0], a, b[u]);
            }
        }
        pk0 = pk1; v0 = v1;
        pk1 = pk2; v1 = v2;
    }
}

// Walk one item: columns [beg, end) of the gcol stream, values from sbase.
// Columns are processed in batches of U: U gathered B rows in flight (thread
// coarsening over k, "UFk"), then for every column the rows of its
// pattern accumulate a*b -- the enumerated block of Listing 4,
// realised as predicates on the pattern bits (uniform within a sub-warp),
// so structural zeros are never multiplied and the code stays one compact
// body for all 2^UFi - 1 patterns.  The next chunk's columns and values are
// fetched while the current chunk computes.
// Operand pipeline of the UFi > 1 walk, three chunks deep: while chunk c
// computes, the values of chunk c+1 (addresses known), the slot-map entries
// of chunk c+2 (packed words known) and the packed words of chunk c+3 are in
// flight, so no dependent global round trip sits between two chunks' FMAs.
// slot_addr: this lane's value positions for a chunk (exclusive warp scan of
// the popcounts, Reading R1 order) -- the slot-map loads for CSR-ordered
// values.
template <int H, class PP>
__device__ __forceinline__ int slot_addr(const PP& p, int pk, int sbase, int lane,
                                         int (&sl)[H]) {
    const unsigned mask = (unsigned)pk >> kColBits;
    const unsigned lt = (1u << lane) - 1u;
    int excl = 0, total = 0;
#pragma unroll
    for (int bit = 0; bit < 3; bit++) {
        const unsigned bal = __ballot_sync(kFull, (__popc(mask) >> bit) & 1);
        excl += __popc(bal & lt) << bit;
        total += __popc(bal) << bit;
    }
#pragma unroll
    for (int r = 0; r < H; r++) {
        const int pos = sbase + excl + __popc(mask & ((1u << r) - 1u));
        sl[r] = ((mask >> r) & 1u) ? ld_stream(p.slot + pos) : -1;
    }
    return sbase + total;
}

template <int H, class PP>
__device__ __forceinline__ void load_vals(const PP& p, const int (&sl)[H], float (&w)[H]) {
#pragma unroll
    for (int r = 0; r < H; r++) w[r] = sl[r] >= 0 ? ld_stream_f(p.vals + sl[r]) : 0.f;
}

template <int H, class Map, int U, bool PROBE, class PP>
__device__ __forceinline__ void walk(const PP& p, Stage<H>& st, int beg, int end, int sbase,
                                     float (&acc)[H][Map::F], int lane) {
    constexpr int F = Map::F, S = Map::S, US = U * S;
    static_assert(32 % US == 0, "UFK * sub-warps must divide 32");
    const int sub = lane / Map::L, lj = lane % Map::L;
    const int n = end - beg;
    const int* gp = p.gpk + beg;
    // plan words of chunks 0..2 (immutable plan: before the PDL wait)
    int pkA = lane < n ? ld_stream(gp + lane) : 0;
    int pkB = 32 + lane < n ? ld_stream(gp + 32 + lane) : 0;
    int pkC = 64 + lane < n ? ld_stream(gp + 64 + lane) : 0;
    grid_dep_wait();
    float w[H];
    int slA[H], slB[H];
    if constexpr (PROBE) {
#pragma unroll
        for (int r = 0; r < H; r++) { w[r] = 0.f; slB[r] = -1; }
    } else {
        sbase = slot_addr<H, PP>(p, pkA, sbase, lane, slA);
        sbase = slot_addr<H, PP>(p, pkB, sbase, lane, slB);
        load_vals<H, PP>(p, slA, w);
    }
    put_chunk<H>(st, 0, lane, pkA, w);
    __syncwarp();
    int buf = 0;
#pragma unroll 1
    for (int c0 = 0; c0 < n; c0 += 32) {
        const bool more = c0 + 32 < n;
        if (more) {
            if constexpr (!PROBE) {
                load_vals<H, PP>(p, slB, w);                        // chunk c+1
                if (c0 + 64 < n) sbase = slot_addr<H, PP>(p, pkC, sbase, lane, slB);   // chunk c+2
            }
        }
        const int pkN = pkB;
        pkB = pkC;
        pkC = c0 + 96 + lane < n ? ld_stream(gp + c0 + 96 + lane) : 0;   // chunk c+3
        const int cn = min(32, n - c0);
        // columns past the item end have pk = 0: row 0 is loaded, pattern 0
        // predicates every FMA off
#pragma unroll 1
        for (int s = 0; s < cn; s += US) {
            float b[U][F];
            int pq[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                pq[u] = st.pk[buf][s + u * S + sub];
                Map::load(b[u], p.B + (size_t)(pq[u] & kColMask) * p.n, p.n, lj);
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const unsigned mk = (unsigned)pq[u] >> kColBits;
                if constexpr (PROBE) {
#pragma unroll
                    for (int f = 0; f < F; f++)
                        if (mk) acc[0][f] += b[u][f];
                } else {
                    float a[H];
                    get_vals<H>(st, buf, s + u * S + sub, a);
#pragma unroll
                    for (int row = 0; row < H; row++) {
                        if ((mk >> row) & 1u) fma_row<F>(acc[row], a[row], b[u]);
                    }
                }
            }
        }
        if (more) {
            put_chunk<H>(st, buf ^ 1, lane, pkN, w);
            __syncwarp();
            buf ^= 1;
        }
    }
}

// ---------------------------------------------------------------- records
// Kernel modes: the CSR-value walks above (kCsr, and their gather probe), or
// the record walk below over the packed stream written by escs_pack (kRec,
// and its probe).
enum Mode { kCsr = 0, kProbe = 1, kRec = 2, kRecProbe = 3 };

// The packed record stream (escs_pack; the paper's data transformation that
// stores the nonzeros in kernel traversal order, "ANNZ", §3.3.3 P:455-493,
// built once per weight matrix and reused across calls): one record
// per gcol j, in canonical gcol order, values stored BY PATTERN ROW (0.0 for
// the rows outside the pattern; they are never multiplied, the FMAs are
// predicated on the pattern bits):
//   UFi = 1      int2 {col, value}                              ( 8 bytes)
//   UFi = 2, 3   int4 {col | mask << 27, w_0, .., w_{h-1}, 0..}  (16 bytes)
//   UFi = 4      2 x int4 {col | mask << 27, w_0, w_1, w_2}, {w_3, 0, 0, 0}
//   UFi = 6      2 x int4 {col | mask << 24, w_0 .. w_5, 0}      (32 bytes)
//   UFi = 8      3 x int4 {col | mask << 24, w_0 .. w_7, 0, 0, 0} (48 bytes)
// A (sub-)warp reads its column's record with ONE broadcast load (all lanes
// of the sub-warp the same address: one L1 wavefront), so the column index,
// the pattern and every value arrive together: no shuffles, no slot map, no
// shared-memory staging.  The B row is then gathered with 128-bit loads and
// reused in registers for every row of the pattern (§3.3.2).
template <int H>
struct RecFmt {
    // int words per record: {word0, w_0 .. w_{h-1}} padded to 2, 4, 8 or 12
    static constexpr int W = H == 1 ? 2 : (H <= 3 ? 4 : (H <= 7 ? 8 : 12));
    // word0 = col | mask << Shift: 27 for UFi <= 4 (the plan's packed gcol
    // word, k < 2^27), 24 for UFi 5..8 (k < 2^24)
    static constexpr int Shift = H <= 4 ? kColBits : 24;
    static constexpr int ColMask = (1 << Shift) - 1;
    static constexpr int Words = H == 1 ? 2 : 1 + H;   // words the walk reads
};

template <int RW, int NW>
__device__ __forceinline__ void ld_rec(int (&r)[RW], const int* q) {
    if constexpr (RW == 2) {
        asm volatile("ld.global.nc" ESC_REC_L1 ".v2.s32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "l"(q));
    } else {
#pragma unroll
        for (int v = 0; v < NW / 4; v++)
            asm volatile("ld.global.nc" ESC_REC_L1 ".v4.s32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(r[4 * v]), "=r"(r[4 * v + 1]), "=r"(r[4 * v + 2]), "=r"(r[4 * v + 3])
                         : "l"(q + 4 * v));
        constexpr int R = NW % 4, B0 = NW - R;
        if constexpr (R >= 2)
            asm volatile("ld.global.nc.v2.s32 {%0,%1}, [%2];" : "=r"(r[B0]), "=r"(r[B0 + 1]) : "l"(q + B0));
        if constexpr (R == 1 || R == 3)
            asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(r[NW - 1]) : "l"(q + NW - 1));
    }
}

// One batch of U records per sub-warp (U*S records per warp): record loads,
// then the U gathered B rows, then the pattern rows' FMAs.  TAIL: the batch
// crosses the item end; a past-the-end slot re-reads the item's last record
// (a valid address) and multiplies nothing (pattern cleared, or the UFi = 1
// FMA predicated off).  The records are read with plain L1-allocating loads:
// a 128-byte line holds the next 4-16 records of the (sub-)warp.
template <int H, class Map, int U, bool TAIL, bool PROBE, class PP>
__device__ __forceinline__ void rec_batch(const PP& p, const int* rec, int i, int end, int sub,
                                          int lj, int lane, float (&acc)[H][Map::F],
                                          unsigned long long pol_b) {
    constexpr int F = Map::F, S = Map::S, RW = RecFmt<H>::W, N = Map::L * Map::F;
    int r[U][RW];
    float b[U][F];
#pragma unroll
    for (int u = 0; u < U; u++) {
        const int idx = i + u * S + sub;
        ld_rec<RW, RecFmt<H>::Words>(r[u], rec + (size_t)(TAIL ? min(idx, end - 1) : idx) * RW);
        if (TAIL && H > 1 && idx >= end) r[u][0] &= RecFmt<H>::ColMask;   // no pattern rows
    }
    if constexpr (!TAIL) {
        // the record lines two batches ahead into L1: with a cold L2 (the
        // bench flushes it per step) a record line is a DRAM round trip that
        // would otherwise sit between two batches' B gathers
        constexpr int kLines = (U * S * RW * 4 + 127) / 128;
        const int ahead = i + 2 * U * S;
        if (lane < kLines && ahead + lane * (128 / (RW * 4)) < end)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(rec + (size_t)ahead * RW + lane * 32));
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
        const int col = H == 1 ? r[u][0] : (r[u][0] & RecFmt<H>::ColMask);
        Map::load_pol(b[u], p.B + (size_t)col * N, lj, pol_b);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
        if constexpr (PROBE) {
#pragma unroll
            for (int f = 0; f < F; f++) acc[0][f] += b[u][f];
        } else if constexpr (H == 1) {
            if (!TAIL || i + u * S + sub < end) fma_row<F>(acc[0], __int_as_float(r[u][1]), b[u]);
        } else {
            const unsigned mk = (unsigned)r[u][0] >> RecFmt<H>::Shift;
#pragma unroll
            for (int row = 0; row < H; row++)
                if ((mk >> row) & 1u) fma_row<F>(acc[row], __int_as_float(r[u][1 + row]), b[u]);
        }
    }
}

// Fire-and-forget bulk prefetch of [q, q + bytes) into L2 (TMA; no
// completion to wait for).  q 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void prefetch_l2_bulk(const void* q, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(q), "r"(bytes) : "memory");
}

#ifndef ESC_REC_BPF
#define ESC_REC_BPF 1
#endif
#ifndef ESC_REC_L2PF
#define ESC_REC_L2PF 0   // measured: no gain on the cold step, +0.2-0.4 us on the small hot layers
#endif
// Walk one item's records [beg, end) (record j = canonical gcol j).
template <int H, class Map, int U, bool PROBE, class PP>
__device__ __forceinline__ void walk_rec(const PP& p, int beg, int end, float (&acc)[H][Map::F],
                                         int lane) {
    static_assert(Map::kVec, "the record walk uses the vector lane maps");
    constexpr int US = U * Map::S;
    static_assert(32 % US == 0, "UFK * sub-warps must divide 32");
    const int sub = lane / Map::L, lj = lane % Map::L;
    const int* rec = reinterpret_cast<const int*>(p.vals);
    const unsigned long long pol_b = policy_last();
    // The record stream is immutable once escs_pack has returned (escs_pack
    // synchronises its stream, include/escs.h), so -- like the plan -- its
    // first lines may be fetched before the programmatic-dependent-launch wait,
    // overlapping the previous kernel's tail; B is caller data written by that
    // kernel and is read only after the wait.
    {
        constexpr int kLines = (2 * US * RecFmt<H>::W * 4 + 127) / 128;   // the first two batches
        if (lane < kLines && beg + lane * (128 / (RecFmt<H>::W * 4)) < end)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(rec + (size_t)beg * RecFmt<H>::W + lane * 32));
    }
#if ESC_REC_L2PF
    // the item's whole record range into L2 in one bulk request (on a cold L2
    // the walk's later batches then wait on an L2 hit, not a DRAM round trip)
    if (lane == 0 && end > beg) {
        const char* a = reinterpret_cast<const char*>(rec + (size_t)beg * RecFmt<H>::W);
        const char* a0 = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(a) & ~uintptr_t(15));
        const char* b1 = reinterpret_cast<const char*>(rec + (size_t)end * RecFmt<H>::W);
        prefetch_l2_bulk(a0, (uint32_t)(((b1 - a0) + 15) & ~15));
    }
#endif
#if ESC_REC_BPF
    // This CTA's share of B into L2, BEFORE the programmatic-dependent-launch
    // wait: an L2 prefetch is only a hint and L2 is the device's point of
    // coherence, so a line the previous kernel is still writing is never seen
    // stale (L1 is not filled); the DRAM fetch of a cold B then overlaps the
    // previous kernel's tail instead of the walk's first gathers.
    if (lane == 0 && (threadIdx.x >> 5) == 0 && p.k > 0) {
        const size_t total = (size_t)p.k * p.n * 4;
        const size_t chunk = ((total + gridDim.x - 1) / gridDim.x + 255) & ~size_t(255);
        const size_t off = (size_t)blockIdx.x * chunk;
        if (off < total) {
            const size_t len = (total - off < chunk ? total - off : chunk);
            prefetch_l2_bulk(reinterpret_cast<const char*>(p.B) + off, (uint32_t)((len + 15) & ~size_t(15)));
        }
    }
#endif
    grid_dep_wait();
#if ESC_REC_L2PF && !ESC_REC_BPF
    // this CTA's share of B into L2 (B is caller data: after the wait); every
    // row is gathered by many warps, most of them on other SMs
    if (lane == 0 && (threadIdx.x >> 5) == 0 && p.k > 0) {
        const size_t total = (size_t)p.k * p.n * 4;
        const size_t chunk = ((total + gridDim.x - 1) / gridDim.x + 255) & ~size_t(255);
        const size_t off = (size_t)blockIdx.x * chunk;
        if (off < total) {
            const size_t len = (total - off < chunk ? total - off : chunk);
            prefetch_l2_bulk(reinterpret_cast<const char*>(p.B) + off, (uint32_t)((len + 15) & ~size_t(15)));
        }
    }
#endif
    int i = beg;
#pragma unroll 1
    for (; i + US <= end; i += US)
        rec_batch<H, Map, U, false, PROBE, PP>(p, rec, i, end, sub, lj, lane, acc, pol_b);
    if (i < end) rec_batch<H, Map, U, true, PROBE, PP>(p, rec, i, end, sub, lj, lane, acc, pol_b);
}

// Row r of a panel tile is written by sub-warp r % S (after the sub-warp
// reduction every sub-warp holds the totals).
template <int H, class Map, class PP>
__device__ __forceinline__ void store_rows(const PP& p, int panel, const float (&a)[H][Map::F],
                                           int sub, int lj) {
#pragma unroll
    for (int r = 0; r < H; r++) {
        const int prow = panel * H + r;
        if ((r % Map::S) == sub && prow < p.m) {
            const int row = p.rowmap ? p.rowmap[prow] : prow;
            if (p.C) Map::store(p.C + (size_t)row * p.n, a[r], p.n, lj);
            if constexpr (PP::kScatter) {
                for (int d = 0; d < p.n_extra; d++) {   // fused all-gather epilogue
                    float* q = p.extra[d] + (size_t)(p.row_off + row) * p.n;
                    if (p.mc) Map::store_mc(q, a[r], p.n, lj);
                    else Map::store(q, a[r], p.n, lj);
                }
            }
        }
    }
}

// Per-warp shared memory: the CSR walk's staging area (UFi > 1) and the
// combine partial (H x bCols floats) share it; the record walk needs only the
// partial.
template <int H, class Map, int MODE = kCsr>
__host__ __device__ constexpr int warp_smem_floats() {
    return (MODE < kRec && H > 1 && (int)(sizeof(Stage<H>) / 4) > H * Map::L * Map::F)
               ? (int)(sizeof(Stage<H>) / 4) : H * Map::L * Map::F;
}

// Store one value group of an output row: C and the fused all-gather
// destinations (escs_spmm_scatter), V = 4 (float4) or 1 consecutive floats.
template <int V, class PP>
__device__ __forceinline__ void store_out(const PP& p, int prow, int c, const float (&v)[V]) {
    const int row = p.rowmap ? p.rowmap[prow] : prow;
    if (p.C) {
        if constexpr (V == 4) *reinterpret_cast<float4*>(p.C + (size_t)row * p.n + c) = make_float4(v[0], v[1], v[2], v[3]);
        else p.C[(size_t)row * p.n + c] = v[0];
    }
    if constexpr (PP::kScatter) {
        for (int d = 0; d < p.n_extra; d++) {
            float* q = p.extra[d] + (size_t)(p.row_off + row) * p.n + c;
            if constexpr (V == 4) {
                if (p.mc)
                    asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1,%2,%3,%4};"
                                 :: "l"(q), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]) : "memory");
                else *reinterpret_cast<float4*>(q) = make_float4(v[0], v[1], v[2], v[3]);
            } else {
                if (p.mc) asm volatile("multimem.st.weak.global.f32 [%0], %1;" :: "l"(q), "f"(v[0]) : "memory");
                else q[0] = v[0];
            }
        }
    }
}

// Heavy panel (more items than the tile's warps; power-law rows, long rows
// split for parallelism): its tiles combine through the global workspace.
// Every warp of the tile takes part (the slots of the H x bCols output are
// spread over the CTA's threads): the tile's item partials are summed from
// shared memory in item order into the tile's workspace slice; the
// last-arriving tile (counter) sums the tiles' slices in tile order and
// writes C.  The order of every sum is fixed -- deterministic -- and each
// thread keeps all the tiles' loads of its slots in flight (one round trip
// for the last tile instead of one per tile).  The barriers are named
// (barrier 1, the tile's W warps only) so that the idle warps of a grouped
// launch's wider CTA need not take part.
template <int H, class Map, class PP>
__device__ __forceinline__ void heavy_combine(const PP& p, const float* smem, int tile, int w, int lane,
                                           int W, int cnt, int lead, int WS) {
    constexpr int NR = Map::L * Map::F;   // floats per tile row in shared memory
    constexpr int V = Map::kVec ? 4 : 1;
    __shared__ int s_last;
    const int n = p.n, nv = n / V, slots = H * nv;
    const int tid = w * 32 + lane, nth = W * 32;
    const int2 th = p.tile_heavy[tile];      // heavy id, ordinal
    const int4 hv = p.heavy[th.x];           // panel, ws_base, ntiles
    float* wsq = p.ws + (size_t)(hv.y + th.y) * H * n;
    {   // the tile's item count and lead from its first slot (always an item)
        const int a0 = p.item_aux[tile * W];
        cnt = (a0 >> 8) & 0xff;
        lead = a0 & 0xff;
    }
    for (int s = tid; s < slots; s += nth) {
        const int r = s / nv, c = (s - r * nv) * V;
        float a[V];
#pragma unroll
        for (int v = 0; v < V; v++) a[v] = 0.f;
        for (int q = 0; q < cnt; q++) {
            const float* part = smem + (size_t)(lead + q) * WS + r * NR + c;
#pragma unroll
            for (int v = 0; v < V; v++) a[v] += part[v];
        }
        if constexpr (V == 4) __stcg(reinterpret_cast<float4*>(wsq + r * n + c), make_float4(a[0], a[1], a[2], a[3]));
        else __stcg(wsq + r * n + c, a[0]);
    }
    // release/acquire through one thread (the CTA barrier orders the other
    // threads' partial stores before thread 0's release, and thread 0's
    // acquire before their loads): no per-thread fence.sc (__threadfence),
    // whose latency under a full load of gathers cost ~35% of the kernel
    asm volatile("bar.sync 1, %0;" :: "r"(nth) : "memory");
    if (tid == 0) {
        int old;
        asm volatile("atom.release.gpu.global.add.s32 %0, [%1], 1;"
                     : "=r"(old) : "l"(p.counters + th.x) : "memory");
        s_last = old == hv.z - 1;
        // the last arriver acquires (the non-last tiles skip the acquire's L1
        // invalidation, which would evict the gathered B rows of every CTA on
        // the SM)
        if (s_last) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    asm volatile("bar.sync 1, %0;" :: "r"(nth) : "memory");
    if (!s_last) return;
    const float* base = p.ws + (size_t)hv.y * H * n;
    for (int s = tid; s < slots; s += nth) {
        const int r = s / nv, c = (s - r * nv) * V;
        const int row = hv.x * H + r;
        float a[V];
#pragma unroll
        for (int v = 0; v < V; v++) a[v] = 0.f;
        int t = 0;
        for (; t + 4 <= hv.z; t += 4) {   // four tiles' loads in flight, summed in tile order
            float q[4][V];
#pragma unroll
            for (int d = 0; d < 4; d++) {
                const float* src = base + (size_t)(t + d) * H * n + r * n + c;
                if constexpr (V == 4) {
                    const float4 x = __ldcg(reinterpret_cast<const float4*>(src));
                    q[d][0] = x.x; q[d][1] = x.y; q[d][2] = x.z; q[d][3] = x.w;
                } else {
                    q[d][0] = __ldcg(src);
                }
            }
#pragma unroll
            for (int d = 0; d < 4; d++)
#pragma unroll
                for (int v = 0; v < V; v++) a[v] += q[d][v];
        }
        for (; t < hv.z; t++) {
            const float* src = base + (size_t)t * H * n + r * n + c;
#pragma unroll
            for (int v = 0; v < V; v++) a[v] += __ldcg(src + v);
        }
        if (row < p.m) store_out<V, PP>(p, row, c, a);
    }
    if (tid == 0) p.counters[th.x] = 0;   // self-reset: graph replay safe
}

// Column-window tiles (tile_order 3): the warps of a CTA hold item j of W
// different panels -- one column window of W panels, whose B rows the SM
// re-reads from L1.  A split panel's items therefore sit in different CTAs:
// each warp stores its item's partial (h x bCols) in the workspace slot of
// (panel, item), releases it on the panel's counter, and the last item to
// arrive sums the panel's partials in item order and writes C (deterministic;
// per warp, no CTA barrier; the counter resets itself).
template <int H, class Map, class PP>
__device__ __forceinline__ void item_ws_combine(const PP& p, float (&acc)[H][Map::F], int slot, int panel,
                                                int sub, int lj, int lane) {
    constexpr int F = Map::F, S = Map::S;
    const int n = p.n;
    const int4 sw = p.slot_ws[slot];   // ws offset, counter, items of the panel, this item's ordinal
    float* mine = p.wsc + sw.x;
#pragma unroll
    for (int r = 0; r < H; r++)
        if ((r % S) == sub) Map::store(mine + (size_t)r * n, acc[r], n, lj);
    __threadfence();
    __syncwarp();
    int last = 0;
    if (lane == 0) last = atomicAdd(p.wsc_counters + sw.y, 1) == sw.z - 1;
    last = __shfl_sync(kFull, last, 0);
    if (!last) return;
    __threadfence();
    const float* base = p.wsc + sw.x - (size_t)sw.w * H * n;   // the panel's item 0
#pragma unroll
    for (int r = 0; r < H; r++) {
        if ((r % S) != sub) continue;
        float a[F];
#pragma unroll
        for (int f = 0; f < F; f++) a[f] = 0.f;
        for (int q = 0; q < sw.z; q++) {
            const float* row = base + (size_t)q * H * n + (size_t)r * n;
#pragma unroll
            for (int v = 0; v < F / 4; v++) {
                const float4 x = __ldcg(reinterpret_cast<const float4*>(row + 4 * (F <= 4 ? lj : v * Map::L + lj)));
                a[4 * v] += x.x; a[4 * v + 1] += x.y; a[4 * v + 2] += x.z; a[4 * v + 3] += x.w;
            }
        }
#pragma unroll
        for (int f = 0; f < F; f++) acc[r][f] = a[f];
    }
    store_rows<H, Map, PP>(p, panel, acc, sub, lj);
    if (lane == 0) p.wsc_counters[sw.y] = 0;   // graph replay safe
}

// One CTA tile.  Item slots are tile-major: tile t owns slots [t*W, t*W + W),
// W = warps per CTA; slot aux = lead | cnt << 8 | active << 16 | tile_sync << 17
// | tile_heavy << 18 (lead: warp of the panel's first item in this tile, cnt:
// the panel's items in this tile).  Every warp of the CTA calls this; the
// __syncthreads below is reached by all of them when the tile needs a combine
// (the flag is tile-uniform).
template <int H, class Map, int U, int MODE, class PP>
__device__ __forceinline__ void process_tile(const PP& p, float* smem, int tile, int w,
                                             int lane, int W) {
    constexpr int F = Map::F, S = Map::S, NR = Map::L * Map::F;   // NR: floats per tile row
    constexpr bool PROBE = MODE == kProbe || MODE == kRecProbe;
    constexpr int WS = warp_smem_floats<H, Map, MODE>();
    const int sub = lane / Map::L, lj = lane % Map::L;
    const int slot = tile * W + w;
    const int aux = p.item_aux[slot];
    const int4 it = p.items[slot];   // independent of aux: both loads in flight together
    const bool active = (aux >> 16) & 1;

    float acc[H][F];
#pragma unroll
    for (int r = 0; r < H; r++)
#pragma unroll
        for (int f = 0; f < F; f++) acc[r][f] = 0.f;

    const int panel = it.x;
    if (active) {
        if constexpr (MODE >= kRec) {
            walk_rec<H, Map, U, PROBE, PP>(p, it.y, it.z, acc, lane);
        } else if constexpr (H == 1) {
            walk1<Map, U, PROBE, PP>(p, it.y, it.z, it.w, acc, lane);
        } else {
            walk<H, Map, U, PROBE, PP>(p, *reinterpret_cast<Stage<H>*>(smem + (size_t)w * WS), it.y,
                                   it.z, it.w, acc, lane);
        }
        if constexpr (S > 1) {   // warp-level reduction of the sub-warps
#pragma unroll
            for (int r = 0; r < H; r++)
#pragma unroll
                for (int f = 0; f < F; f++)
#pragma unroll
                    for (int off = Map::L; off < 32; off <<= 1)
                        acc[r][f] += __shfl_xor_sync(kFull, acc[r][f], off);
        }
    }
    if constexpr (!(MODE == kProbe || MODE == kRecProbe)) {
        if ((aux >> 19) & 1) {   // column-window tile: this item's partial through the workspace
            item_ws_combine<H, Map, PP>(p, acc, slot, it.x, sub, lj, lane);
            return;
        }
    }
    __syncwarp();   // staging reads done before the area holds the partial
#ifdef ESC_TEST_ATOMIC   // A/B experiment only: atomics into a pre-zeroed C instead of the combine
    if constexpr (MODE == kRec) {
        if (active && sub == 0)
            for (int r = 0; r < H; r++)
                if (panel * H + r < p.m)
                    for (int v = 0; v < F / 4; v++)
                        atomicAdd(reinterpret_cast<float4*>(p.C + (size_t)(panel * H + r) * p.n + Map::col(lj, 4 * v)),
                                  make_float4(acc[r][4 * v], acc[r][4 * v + 1], acc[r][4 * v + 2], acc[r][4 * v + 3]));
        return;
    }
#endif

    if constexpr (PROBE) {
        if (active) {
            float s = 0.f;
#pragma unroll
            for (int f = 0; f < F; f++) s += acc[0][f];
            p.C[(size_t)slot * 32 + lane] += s;
        }
        return;
    } else {
        const int n = p.n;
        const bool heavy = (aux >> 18) & 1;
        const int cnt = (aux >> 8) & 0xff, lead = aux & 0xff;
        if (!((aux >> 17) & 1)) {   // every panel of this tile has exactly one item here
            if (active) store_rows<H, Map, PP>(p, panel, acc, sub, lj);
            return;
        }
        float* mine = smem + (size_t)w * WS;
        if (active && (cnt > 1 || heavy)) {
#pragma unroll
            for (int r = 0; r < H; r++)
                if ((r % S) == sub)
#pragma unroll
                    for (int f = 0; f < F; f++) {
                        const int j = Map::col(lj, f);
                        if (Map::kVec || j < n) mine[r * NR + j] = acc[r][f];
                    }
        }
        __syncthreads();
        if (heavy) {   // tile-uniform: every warp of a heavy tile combines (more barriers)
            heavy_combine<H, Map, PP>(p, smem, tile, w, lane, W, cnt, lead, WS);
            return;
        }
        if (!active) return;
        if (cnt == 1) {
            store_rows<H, Map, PP>(p, panel, acc, sub, lj);
            return;
        }
        if (w != lead) return;
        // combine the panel's partials in item order (deterministic)
#pragma unroll
        for (int r = 0; r < H; r++)
#pragma unroll
            for (int f = 0; f < F; f++) acc[r][f] = 0.f;
#pragma unroll 1
        for (int q = 0; q < cnt; q++) {
            const float* part = smem + (size_t)(lead + q) * WS;
#pragma unroll
            for (int r = 0; r < H; r++)
                if ((r % S) == sub)
#pragma unroll
                    for (int f = 0; f < F; f++) {
                        const int j = Map::col(lj, f);
                        if (Map::kVec || j < n) acc[r][f] += part[r * NR + j];
                    }
        }
        store_rows<H, Map, PP>(p, panel, acc, sub, lj);
    }
}

// One CTA per tile.  (A persistent variant with a dynamic tile counter was
// measured and dropped: the hardware block scheduler already dispatches CTAs
// dynamically, and the counter atomics and extra barriers cost 0.2-1.5 us per
// launch on the latency-bound suite -- profiles/r1_notes.md.)
template <int H, class Map, int U, int MODE>
__global__ void ESC_CSR_BOUNDS esc_spmm_kernel(KParams p) {
    extern __shared__ __align__(16) float smem[];
    grid_dep_launch();   // the next launch may start reading its plan
    process_tile<H, Map, U, MODE, KParams>(p, smem, blockIdx.x, threadIdx.x >> 5, threadIdx.x & 31,
                                           blockDim.x >> 5);
}

// The record walk (kRec / kRecProbe) as its own kernel: its register budget
// sets both the resident warps per SM and how many record / B-row loads ptxas
// keeps in flight per warp -- the two quantities that decide a gather-bound,
// latency-bound walk.  With "__launch_bounds__(512, 1)" ptxas takes all 128
// registers (16 warps/SM); with "(512)" alone it settles near 55 and
// interleaves each record's loads with the previous record's FMAs (4 loads in
// flight); a register target of 72 keeps 8 loads in flight at 7 CTAs of 4
// warps per SM: 512x4608@70% bCols 128, UFi 3: 24.6 us -> 19.1 us
// (profiles/r2_notes.md, "record walk register target").
// Wider register tiles (H x F accumulators beyond 32) get the target raised
// with them (UFi 6/8, 16 columns per lane), up to 128.
#ifndef ESC_REC_MAXREG
#define ESC_REC_MAXREG 72
#endif
template <int H, class Map>
struct RecRegs {
    static constexpr int acc = H * Map::F;
    static constexpr int value = acc <= 32 ? ESC_REC_MAXREG
                                           : ((acc + 48 + 7) / 8 * 8 > 128 ? 128 : (acc + 48 + 7) / 8 * 8);
};
#if ESC_REC_MAXREG > 0
#define ESC_REC_BOUNDS __maxnreg__((RecRegs<H, Map>::value))
#else
#define ESC_REC_BOUNDS __launch_bounds__(512)
#endif
template <int H, class Map, int U, int MODE>
__global__ void ESC_REC_BOUNDS esc_rec_kernel(KParams p) {
    static_assert(MODE == kRec || MODE == kRecProbe, "record modes only");
    extern __shared__ __align__(16) float smem[];
    grid_dep_launch();
    process_tile<H, Map, U, MODE, KParams>(p, smem, blockIdx.x, threadIdx.x >> 5, threadIdx.x & 31,
                                           blockDim.x >> 5);
}

using KernelFn = void (*)(KParams);

// Grouped launch (escs_spmm_group): up to kMaxGroup independent problems
// whose plans select the same kernel instance run as ONE grid -- the
// concatenation of their CTA tiles -- so a suite of small, latency-bound
// layers pays one launch and one ramp/tail instead of one per layer.  The
// per-problem operands travel in the kernel's parameter space (no per-call
// copy, graph capturable).  A CTA finds its problem by binary search over the
// tile prefix; a problem whose tiles are narrower than the launch's block
// (W < blockDim/32) leaves the extra warps idle (they still meet the tile's
// combine barrier).  Each tile is processed exactly as by esc_spmm_kernel, so
// results are bitwise identical to separate escs_spmm calls.
constexpr int kMaxGroup = 32;
struct GProb {
    const int* gpk;
    const int* slot;
    const int4* items;
    const int* item_aux;
    const int2* tile_heavy;
    const int4* heavy;
    float* ws;
    int* counters;
    const float* vals;
    const float* B;
    float* C;
    int m, n, W;
    const int* rowmap;                        // always NULL (hybrid plans are not grouped)
    const int4* slot_ws;                      // always NULL (column-window tiles are not grouped)
    float* wsc;
    int* wsc_counters;
    static constexpr bool kScatter = false;   // no fused all-gather in grouped launches
};
struct GroupParams {
    int n;
    int tile_start[kMaxGroup + 1];
    GProb prob[kMaxGroup];
};

template <int H, class Map, int U>
__global__ void ESC_CSR_BOUNDS esc_spmm_group_kernel(const __grid_constant__ GroupParams gp) {
    extern __shared__ __align__(16) float smem[];
    grid_dep_launch();
    const int t = blockIdx.x;
    int lo = 0, hi = gp.n - 1;          // last problem with tile_start <= t
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (gp.tile_start[mid] <= t) lo = mid;
        else hi = mid - 1;
    }
    const GProb& q = gp.prob[lo];       // read in place from the parameter space
    const int tile = t - gp.tile_start[lo], w = threadIdx.x >> 5;
    if (w >= q.W) {                     // idle warp: only the tile's combine barrier
        if ((q.item_aux[tile * q.W] >> 17) & 1) __syncthreads();
        return;
    }
    process_tile<H, Map, U, kCsr, GProb>(q, smem, tile, w, threadIdx.x & 31, q.W);
}

using GroupFn = void (*)(GroupParams);

}  // namespace kern
}  // namespace escs
