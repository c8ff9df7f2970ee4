/*
 * escs.h -- C ABI of the B200-native enumerate-and-sparse-coarsen (ESC) SpMM.
 *
 * Method: arXiv 2506.15174, "A Novel Compiler Transformation for Fast Sparse
 * Matrix Multiplication in GPUs".  Citations: P:n = PAPER.md line n (section
 * named), S:n = SPEC.md line n, R<k> = a reading recorded in DESIGN.md.
 *
 * Problem (§2 Motivation): C = A x B with A sparse M x K (CSR), B dense
 * K x N, C dense M x N; N is "bCols" (32..128 in the paper's evaluation,
 * P:31).  Everything is fp32 (§4.2).
 *
 * Life cycle (Listing 2, §3.1): the sparsity pattern of A is
 * enumerated once on the host into a plan ("TA = dataTransformer(A, UFi, UFk)",
 * reused across inference calls, §3.6); each product is then one
 * kernel launch ("spmmOpt<<<...>>>").
 *
 * Conventions
 *   - All functions are thread-safe; errors are reported per calling thread
 *     through escs_last_error().
 *   - Return codes: ESCS_OK (0) or one of the ESCS_ERR_* values below
 *     (error convention of S:551: 1 = user error; higher = library/CUDA).
 *   - "HOST" pointers are read only during the call; the caller keeps
 *     ownership.  "DEVICE" pointers must be CUDA device memory on the plan's
 *     device; the caller keeps ownership.
 *   - Streams are passed as `void*` holding a cudaStream_t (NULL = legacy
 *     default stream), so this header needs no CUDA include.
 */
#ifndef ESCS_H
#define ESCS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    ESCS_OK = 0,
    ESCS_ERR_ARG = 1,          /* bad argument (sizes, NULL, host-only plan)        */
    ESCS_ERR_CSR = 2,          /* CSR violates an invariant (message names the row) */
    ESCS_ERR_UNSUPPORTED = 3,  /* valid input outside what the kernels implement    */
    ESCS_ERR_OOM = 4,          /* host or device allocation failed                  */
    ESCS_ERR_CUDA = 5,         /* a CUDA runtime call failed (message has the name) */
    ESCS_ERR_INTERNAL = 6      /* internal invariant violated (a bug)               */
};

#define ESCS_PLAN_VERSION 1
#define ESCS_MAX_BCOLS 256     /* largest supported N (bCols)                    */
#define ESCS_MAX_UFI 8         /* largest UFi of the device kernels: 4 for the CSR-value
                                  walk (escs_spmm), 8 for the packed record walk
                                  (escs_spmm_packed; UFi 1-4, 6 and 8 are built)    */

typedef struct escs_plan_impl *escs_plan_t;   /* opaque, library-owned */

/*
 * escs_plan -- enumerate A's sparsity pattern (§3.2 Enumeration)
 * and upload the plan to the current CUDA device.
 *
 *   m, k      rows / columns of A.  1 <= m, k < 2^31.
 *   nnz       number of stored entries, 0 <= nnz < 2^31.
 *   rowptr    HOST int32[m+1]: rowptr[0] = 0, non-decreasing, rowptr[m] = nnz.
 *   colidx    HOST int32[nnz]: 0 <= colidx < k, strictly increasing per row.
 *             Explicitly stored zeros count as structural nonzeros.
 *   bCols     N, the number of columns of B and C: 1 <= N <= ESCS_MAX_BCOLS,
 *             and m*N, k*N < 2^31.
 *
 * The plan records the panel height UFi (=h), the item size T and the kernel
 * variant, chosen from a per-bCols parameter table (§3.5 Scheduler & Tuner,
 * P:510-526; env override ESCS_PARAMS="ufi=4,T=64,warps=8").
 * Synchronous, deterministic (identical inputs give byte-identical plans
 * regardless of planner thread count).  Returns NULL on failure; the reason
 * is in escs_last_error().  Allocates device memory with cudaMalloc on the
 * current device; the plan is bound to that device.
 */
escs_plan_t escs_plan(int64_t m, int64_t k, int64_t nnz,
                      const int32_t *rowptr, const int32_t *colidx,
                      int32_t bCols);

/*
 * escs_spmm -- C = A x B (beta = 0: every element of C is written) with the
 * enumerated, sparse-coarsened kernel (§3.3 Sparse Coarsen).
 *
 *   plan   a device plan from escs_plan / escs_plan_ex (host_only = 0).
 *   vals   DEVICE float[nnz], A's values in CSR order (the values may change
 *          between calls; the pattern may not).
 *   B      DEVICE float[k * bCols], row-major (ld = bCols).
 *   C      DEVICE float[m * bCols], row-major, overwritten.  Must not alias
 *          vals or B.
 *   stream cudaStream_t (as void*), may be NULL.
 *
 * Exactly one kernel launch, enqueue-only: no host synchronisation, no
 * allocation, no memset -- capturable in a CUDA graph.  The launch uses
 * programmatic dependent launch: it may start reading its (immutable) plan
 * while the previous kernel in `stream` finishes, but reads vals/B and writes
 * C only after that kernel has completed (stream order is preserved for the
 * caller's data; set ESCS_PDL=0 to launch without the attribute).  Two calls on the same
 * plan must not be in flight concurrently (they share the plan's fixup
 * workspace).  Asynchronous device faults surface at the next synchronising
 * CUDA call, as with cuBLAS.  Pointers that are not 16-byte aligned take the
 * scalar (generic) kernel.  Returns ESCS_OK, ESCS_ERR_ARG (NULL pointer,
 * host-only plan, wrong device) or ESCS_ERR_CUDA (launch failure).
 */
int escs_spmm(escs_plan_t plan, const float *vals, const float *B, float *C,
              void *stream);

/*
 * escs_spmm_group -- n independent SpMMs C[i] = A_i x B[i] (a layer suite,
 * the experts of a layer, Q/K/V projections) in as few launches as possible:
 * the problems whose plans select the same kernel instance (UFi = 1, vector
 * lane map, 16-byte aligned B/C) run as one grid -- the concatenation of their
 * CTA tiles, up to 32 problems per launch -- so small latency-bound layers
 * share one launch, ramp and tail; any other problem is launched on its own.
 * Each CTA tile computes exactly what escs_spmm computes for it: results are
 * bitwise identical to n separate escs_spmm calls.
 *   n       number of problems, >= 0 (0: no-op).
 *   plans   HOST array of n device plans on the current device; a plan may
 *           appear at most once (its fixup workspace is per plan).
 *   vals, B, C   HOST arrays of n DEVICE pointers with escs_spmm's meaning,
 *           layout and ownership per problem; no C[i] may alias another
 *           problem's vals, B or C.
 * Enqueue-only on `stream` (no host sync, no allocation, graph capturable:
 * the per-problem operands travel in the kernel parameters).  The problem
 * order inside a launch is unspecified.  Returns ESCS_OK, ESCS_ERR_ARG
 * (naming the offending problem) or ESCS_ERR_CUDA.
 */
int escs_spmm_group(int32_t n, const escs_plan_t *plans, const float *const *vals,
                    const float *const *B, float *const *C, void *stream);

/*
 * escs_pack -- the value half of the paper's data transformation: the
 * nonzeros re-stored in kernel traversal order ("ANNZ", §3.3.3),
 * built once per weight matrix and reused across inference calls
 * ("TA = dataTransformer(A, UFi, UFk)").  Writes the plan's RECORD
 * STREAM: one record per gcol j (a (panel, column) pair with a nonzero, in the
 * canonical gcol order of escs_plan_export), holding the column, the UFi-bit
 * pattern and the pattern rows' values (Reading R1 slots, stored by row):
 *   UFi = 1      int32 {col, value}                               2 words
 *   UFi = 2, 3   int32 {col | mask << 27, w_0 .. w_{h-1}, 0 ..}    4 words
 *   UFi = 4      int32 {col | mask << 27, w_0, w_1, w_2, w_3, 0, 0, 0}  8 words
 * (w_r = the value of A(panel*h + r, col), 0.0 for rows outside the pattern;
 * values are copied bit for bit).  One kernel launch on `stream`; SYNCHRONOUS
 * (returns after the stream has finished it): like the plan, the record
 * stream is then immutable input -- escs_spmm_packed may read it before the
 * previous kernel in its stream has finished (programmatic dependent
 * launch); rewrite it only through escs_pack.
 *   vals    DEVICE float[nnz], CSR order.
 *   packed  DEVICE buffer of escs_plan_stats.packed_words 32-bit words,
 *           16-byte aligned, caller-owned output; must not alias vals.
 * Returns ESCS_OK, ESCS_ERR_ARG or ESCS_ERR_CUDA.
 */
int escs_pack(escs_plan_t plan, const float *vals, float *packed, void *stream);

/*
 * escs_spmm_packed -- C = A x B from the record stream of escs_pack: each
 * (sub-)warp reads its column's record with one broadcast load (column,
 * pattern and every row value together), gathers the B row once with 128-bit
 * loads and reuses it in registers for every row of the pattern (the
 * enumerated, sparse-coarsened kernel of §3.3 without the slot-map
 * indirection).  Same contract as escs_spmm (one launch, beta = 0, PDL, graph
 * capturable); B and C must be 16-byte aligned and the plan must use the
 * vector kernel (bCols in {4,8,16,32,64,128,256}), else ESCS_ERR_UNSUPPORTED.
 * For finite B the result is bitwise identical to escs_spmm on the CSR values
 * (same per-lane FMA order, same combine).
 */
int escs_spmm_packed(escs_plan_t plan, const float *packed, const float *B, float *C,
                     void *stream);

/*
 * escs_spmm_scatter -- escs_spmm whose epilogue stores every output row i of
 * the plan's A into each of the n_dst destination buffers at row
 * row_offset + i (row-major, ld = bCols): with the destinations being the
 * peers' C buffers of a row-block-sharded SpMM (mapped through CUDA IPC /
 * symmetric memory over NVLink), this is the SpMM fused with the optional
 * all-gather of C: each C tile crosses NVLink once, as it
 * is produced, with no separate collective.  One launch; same contract as
 * escs_spmm otherwise.
 *   dsts        HOST array of n_dst DEVICE pointers (1 <= n_dst <= 8), each a
 *               float[(row_offset + m) * bCols] buffer reachable from this
 *               device (local or peer-mapped); not aliasing vals or B.
 *   row_offset  first row of this plan's block in the destinations (>= 0).
 *   flags       0, or ESCS_SCATTER_MULTICAST: n_dst must be 1 and dsts[0] an
 *               NVLS multicast address (CUDA multicast object bound to every
 *               rank's C); the epilogue then issues multimem.st, one store
 *               per element reaching all GPUs through the NVSwitch.
 * Errors: ESCS_ERR_ARG for NULL pointers, n_dst outside 1..8, negative
 * row_offset, unknown flags or a device other than the plan's.
 */
#define ESCS_SCATTER_MULTICAST 1u
int escs_spmm_scatter(escs_plan_t plan, const float *vals, const float *B,
                      float *const *dsts, int32_t n_dst, int64_t row_offset, uint32_t flags,
                      void *stream);

/* escs_free -- release the plan's host and device memory (the plan owns them,
 * "TA" of Listing 2, kept until the caller drops it).  NULL is a
 * no-op.  No call on the plan may be in flight (the caller synchronises the
 * streams that used it, as with cudaFree).  Autotuned plans take their device
 * memory from a private stream-ordered pool (up to 1 GiB of freed memory is
 * kept for later plans); escs_free then waits for the device, like cudaFree. */
void escs_free(escs_plan_t plan);

/* Code and message of the last failed call on this thread (ESCS_OK and ""
 * if none).  The message pointer stays valid until the next ESCS call on the
 * same thread.  msg may be NULL. */
int escs_last_error(const char **msg);

/* ------------------------------------------------------------------ *
 * Test / tuning / benchmarking entry points                           *
 * ------------------------------------------------------------------ */

typedef struct {
    int32_t ufi;          /* panel height h = UFi, 0 = auto; 1..16 for
                             host-only plans; device plans: 1..4 (escs_spmm),
                             1..4, 6, 8 with packed = 1 (escs_spmm_packed)     */
    int32_t T;            /* max gcols per item (balanced tiles), 0 = auto      */
    int32_t host_only;    /* 1: build host arrays only (no CUDA), for parity     */
    int32_t cta_warps;    /* warps per CTA tile, 0 = auto, else 1..16            */
    int32_t variant;      /* 0 = auto, 1 = vector (float4) kernel, 2 = scalar    */
    int32_t ufk;          /* B-row loads in flight per warp (UFk: 4 or 8), 0 = auto */
    int32_t nthreads;     /* planner threads, 0 = hardware concurrency           */
    int32_t autotune;     /* 1: time candidate (T, tile width, UFk) plans on the
                             device at plan time and keep the fastest (the
                             paper's profiling-based tuner, §3.5);
                             parameters given explicitly are not searched.
                             Adds a few ms to escs_plan; the plan arrays are
                             still the canonical plan of the chosen (UFi, T).
                             Also enabled by ESCS_AUTOTUNE=1.
                             2: same search, throughput objective: each
                             candidate is timed as 8 concurrent chains of
                             its launches on 8 streams (ESCS_TUNE_STREAMS,
                             2..16; each chain with its own
                             fixup workspace; for callers that overlap
                             independent SpMMs on several streams; prefers
                             plans that leave SMs to the other streams;
                             such plans launch without programmatic
                             dependent launch).
                             Candidates are timed as CUDA-graph replays of
                             back-to-back launches (ESCS_TUNE_GRAPH=0: eager).
                             The chosen parameters are cached per problem
                             class (escs_plan_stats.autotuned).
                             Any other value: ESCS_ERR_ARG.                   */
    int32_t colf;         /* B columns per lane of the vector kernel: the bCols
                             coarsening factor (register tile of B columns,
                             §3.4).  0 = default (4; 8 at bCols 256); 8 or 16
                             at bCols 32..256 (UFi = 1 only).  Searched by the
                             autotuner when 0.                                  */
    int32_t tile_order;   /* CTA tile formation: 0 = auto (by item length when the
                             panel work is skewed, p99 >= 2x median), 1 = panel
                             order, 2 = panels ordered by their longest item
                             (similar work per tile, long tiles first), 3 =
                             column windows (UFi 1 only): a tile holds item j
                             of W consecutive panels, so an SM walks one
                             column window of many rows; a split panel's items
                             combine through per-item workspace slots and a
                             per-panel counter (last arriver sums in item
                             order).  1 and 2 are searched by the autotuner
                             when 0.                                         */
    int32_t packed;       /* 1: the plan will run through escs_pack +
                             escs_spmm_packed (the record walk): the parameter
                             table and the autotuner target that walk, and
                             the tuner also searches UFi in 1..4
                             unless ufi is given.  0: escs_spmm (CSR values).
                             Either way any call works on the plan.           */
    int32_t staged;       /* the packed walk's B-row source: 0 = auto (the
                             autotuner times both walks when it runs; the L2
                             gather walk otherwise), 1 = gather B rows from
                             L2 (esc_kernel.cuh record walk), 2 = staged: a
                             CTA owns a row block (st_warps x st_npw panels)
                             and one of st_nsplit column ranges of A; TMA bulk
                             copies bring that range's B rows and the CTA's
                             records into shared memory and every B row is
                             read there (staged_kernel.cuh); with st_nsplit >
                             1 a second launch sums the ranges' partials in
                             range order.  Staged plans need packed = 1 and
                             bCols 32, 64 or 128.                            */
    int32_t st_warps;     /* staged: warps per CTA (1..16), 0 = auto           */
    int32_t st_npw;       /* staged: panels per warp (1, 2, 4), 0 = auto        */
    int32_t st_nsplit;    /* staged: column ranges per row block, 0 = auto (fit
                             227 KB of shared memory, ~1 CTA per SM)          */
    int32_t st_kb;        /* staged: columns per pipeline stage (one mbarrier
                             each, <= 16 stages per CTA), 0 = auto             */
    int32_t hybrid_rows;  /* packed walk on skewed row lengths: 0 = auto (off;
                             with ESCS_TUNE_HYBRID=1 the autotuner tries a
                             hybrid plan when the rows of at least twice the
                             mean length hold >= 25% of the nonzeros -- on
                             B200 it has not won: DESIGN.md §7), -1 = off, X > 0:
                             a hybrid plan whose part 0 is the X longest rows
                             (in descending length order, ties by row index)
                             planned as their own matrix -- dense rows share
                             panels, so the enumeration's B-row reuse p is
                             large there -- and whose part 1 is the other
                             rows in row order.  Each part is an ordinary
                             plan (escs_plan_part); escs_pack writes part 0's
                             record stream then part 1's; escs_spmm_packed
                             launches part 0 then part 1, each writing its
                             rows of C.  Only escs_pack / escs_spmm_packed
                             accept a hybrid plan.                            */
    int32_t carveout;     /* the gather walk's preferred shared-memory carveout
                             per launch: 0 = auto (the smallest that holds the
                             plan's occupancy -- the rest of the SM's 228 KB is
                             L1 for re-read B rows; the autotuner also times
                             smaller carveouts, trading occupancy for L1),
                             1..100 = that percent, -1 = the driver's choice,
                             -2 = 0 percent (maximum L1)                      */
    int32_t reserved[1];  /* must be zero                                        */
} escs_params;

/* escs_plan with explicit parameters; p may be NULL (= all auto). */
escs_plan_t escs_plan_ex(int64_t m, int64_t k, int64_t nnz,
                         const int32_t *rowptr, const int32_t *colidx,
                         int32_t bCols, const escs_params *p);

/*
 * The canonical plan (DESIGN.md "Canonical plan" P1-P8), host copies owned by
 * the plan and valid until escs_free.  Array lengths: grp_* NG (+1 for the
 * *_ptr arrays), gcol G, slot_src nnz, item_* n_items (+1 for item_gcol_ptr).
 *   grp_panel[g], grp_mask[g]  group g = (row panel, UFi-bit pattern)
 *   grp_col_ptr                prefix of group widths       (paper "RPP")
 *   grp_val_ptr                prefix of popcount*width     (paper "NPP")
 *   gcol                       group columns, ascending     (paper "Cols")
 *   slot_src[s]                CSR position of the value at slot s (paper
 *                              "ANNZ" order, Reading R1)
 *   item_panel, item_group_begin, item_gcol_ptr   balanced items (Reading R7)
 */
typedef struct escs_plan_view {
    int32_t header[11];   /* version, m, k, nnz, bCols, h, T, nP, NG, G, n_items */
    const int32_t *grp_panel, *grp_mask, *grp_col_ptr, *grp_val_ptr, *gcol, *slot_src,
                  *item_panel, *item_group_begin, *item_gcol_ptr;
} escs_plan_view;

int escs_plan_export(escs_plan_t plan, escs_plan_view *out);

/* Derived, device-side facts about a plan (for tests and the bench). */
typedef struct {
    int32_t h, T, bcols, variant, cta_warps, ufk;
    int32_t n_tiles;        /* CTA tiles = grid size of one escs_spmm launch     */
    int32_t n_heavy;        /* panels split across CTA tiles (global fixup)       */
    int32_t n_split_items;  /* items whose panel has more than one item           */
    int32_t device;         /* CUDA ordinal, -1 for host-only plans               */
    int64_t nP, NG, G, n_items, nnz;
    int64_t device_bytes;   /* plan arrays + workspace resident on the device     */
    int64_t workspace_bytes;
    double plan_seconds;    /* host enumeration time                              */
    int32_t ctas_per_sm;    /* resident CTAs per SM of the launch (occupancy), 0 host-only */
    int32_t autotuned;      /* 1 if the parameters were chosen by plan-time timing,
                               2 if taken from the process's tuning cache (the
                               tuned parameters of an earlier matrix with the
                               same m, k, nnz, bCols and requested parameters;
                               ESCS_TUNE_CACHE=0 disables the cache)           */
    int32_t colf;           /* B columns per lane of the launch's lane map (0 scalar map) */
    int32_t tile_order;     /* 1 panel order, 2 by item length (resolved)          */
    int32_t pdl;            /* 1 if launches carry programmatic dependent launch    */
    int32_t packed;         /* 1 if planned (and tuned) for escs_spmm_packed         */
    int64_t packed_words;   /* size of the buffer escs_pack fills, in 32-bit words
                               (the record stream rounded up to 16 bytes)         */
    int32_t staged;         /* 1 if escs_spmm_packed runs the staged walk          */
    int32_t st_ctas;        /* staged: CTAs of the walk launch (row blocks x ranges) */
    int32_t st_warps, st_npw, st_nsplit, st_kb;
    int32_t st_smem_bytes;  /* staged: dynamic shared memory per CTA               */
    int32_t st_launches;    /* staged: kernel launches per escs_spmm_packed (1, 2)  */
    int32_t carveout;       /* the gather walk's launch carveout in percent (-1: driver) */
    int32_t hybrid_rows;    /* hybrid plan: rows in part 0 (0: not a hybrid plan);
                               the other fields then describe part 0, except
                               nnz, G, packed_words and device_bytes (totals) */
} escs_plan_stats;

int escs_plan_info(escs_plan_t plan, escs_plan_stats *out);

/*
 * escs_gather_probe -- measurement only (SURVEY §8(d) t_probe): the same CTA,
 * warp and lane walk as escs_spmm with the same 128-bit B-row loads, but no
 * values and no FMAs; writes one float per warp-lane sum into
 * `sink` (DEVICE float[n_tiles * 32 * cta_warps]) so the loads are not dead.
 * Its duration is the empirical gather ceiling of this plan.
 */
int escs_gather_probe(escs_plan_t plan, const float *B, float *sink, void *stream);

/*
 * escs_gather_probe_packed -- the same for escs_spmm_packed: the record walk
 * (one broadcast record load per column, the 128-bit B-row gathers) without
 * the FMAs.  `packed` is the record stream of escs_pack (only the column
 * words are used).  Same sink contract; for a staged plan the staged walk's
 * probe (the same bulk copies and shared-memory reads, no FMAs) with `sink`
 * float[st_ctas * 32 * st_warps].  Hybrid plans: ESCS_ERR_UNSUPPORTED.
 */
int escs_gather_probe_packed(escs_plan_t plan, const float *packed, const float *B, float *sink,
                             void *stream);

/*
 * escs_staged_export -- the staged walk's schedule (host copies owned by the
 * plan, valid until escs_free; plans built with staged = 2, host-only plans
 * included).  It is derived from the canonical plan: CTA c = (row block rb,
 * column range sp) owns panels [rb*nslot, (rb+1)*nslot) (nslot = st_warps x
 * st_npw) and columns [sp*k/nsplit, (sp+1)*k/nsplit), cut into stages of
 * st_kb columns; record r of the stream escs_pack writes for the plan is the
 * canonical gcol src[r] (-1: padding), stored by (CTA, stage, slot) and, in a
 * slot, in canonical order.
 *   cta[4c..]    rb, sp, first stage, stage count
 *   stage[4s..]  first column, end column, first record, records (padded)
 *   hdr[hs*s+j]  record offset (from the CTA's first record) of slot j's
 *                records in stage s; hdr[hs*s + nslot] = the stage's end
 */
typedef struct escs_staged_view {
    int32_t n_cta, n_stage, n_rec, hs, nslot, max_k, max_rec, max_stages;
    const int32_t *cta, *stage, *hdr, *src;
} escs_staged_view;
int escs_staged_export(escs_plan_t plan, escs_staged_view *out);
/* escs_plan_part -- part i (0 or 1) of a hybrid plan as a plan handle
 * (borrowed: owned by `plan`, valid until escs_free(plan); do not free it),
 * for escs_plan_export / escs_plan_info; NULL if `plan` is not hybrid. */
escs_plan_t escs_plan_part(escs_plan_t plan, int32_t i);
/* Library version string ("escs <ver> sm_100a"). */
const char *escs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ESCS_H */
