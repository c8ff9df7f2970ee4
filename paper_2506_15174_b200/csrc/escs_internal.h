// escs_internal.h -- shared between the host planner/ABI (C++) and the
// sm_100a kernels (CUDA).  Not part of the public ABI (include/escs.h).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace escs {

// Parameters recorded in the plan (§3.5 Scheduler & Tuner).
struct Params {
    int h = 4;          // UFi: rows per panel
    int T = 64;         // max gcols per item
    int cta_warps = 8;  // warps per CTA tile
    int variant = 1;    // 1 = vector (float4) lane map, 2 = scalar lane map
    int ufk = 4;        // B-row loads in flight per sub-warp step (UFk)
    int packed = 0;     // 1: tuned for the packed-record walk (escs_spmm_packed)
    int colf = 0;       // B columns per lane of the vector map (bCols coarsening), 0 = default
    int tile_order = 0; // 0 auto, 1 panel order, 2 by longest item, 3 column windows
    int nthreads = 0;   // planner threads
    // staged record walk (staged_kernel.cuh): B rows of a CTA's k-range in
    // shared memory.  staged: 0 = auto, 1 = off (record walk gathers from L2),
    // 2 = on; st_*: compute warps per CTA, panels per warp, k-splits per row
    // block, columns per pipeline stage
    int staged = 0;
    int st_warps = 0, st_npw = 0, st_nsplit = 0, st_kb = 0;
};

// The staged walk's derived schedule (deterministic; a permutation of the
// canonical record stream cut by row block, k-split, stage and warp slot).
struct StagedHost {
    int warps = 0, npw = 0, nsplit = 0, kb = 0, nslot = 0, hs = 0, rw = 0;
    int n_cta = 0, max_k = 0, max_rec = 0, max_stages = 0;
    std::vector<int32_t> cta;     // 4 per CTA: rb, split, stage_begin, n_stage
    std::vector<int32_t> stage;   // 4 per stage: ks, ke, rec_begin, n_rec (padded to 16 bytes)
    std::vector<int32_t> hdr;     // hs per stage: CTA-relative record offset of each slot, end
    std::vector<int32_t> src;     // per record: canonical gcol, -1 = padding
};

// Host plan: the canonical arrays (P1-P8) plus the device-only
// derived CTA-tile schedule.
struct PlanHost {
    int32_t header[11] = {0};
    std::vector<int32_t> grp_panel, grp_mask, grp_col_ptr, grp_val_ptr, gcol, slot_src;
    std::vector<int32_t> item_panel, item_group_begin, item_gcol_ptr;
    // derived CTA-tile schedule (not part of plan parity; deterministic):
    // W item slots per tile, tile-major
    std::vector<int32_t> slot_item;   // canonical item of each slot, -1 = empty
    std::vector<int32_t> slot_aux;    // lead | cnt<<8 | active<<16 | tile_sync<<17 | tile_heavy<<18
    std::vector<int32_t> tile_heavy;  // 2 per tile: heavy id (-1), ordinal
    std::vector<int32_t> heavy_info;  // 4 per heavy panel: panel, ws_base, ntiles, 0
    // column-window tiles (tile_order 3): per slot {ws offset (floats), panel
    // counter, the panel's item count, the item's ordinal}; counters, ws floats
    std::vector<int32_t> slot_ws;
    int n_wsc_counters = 0;
    int64_t wsc_floats = 0;
    int n_tiles = 0, n_heavy = 0, n_heavy_tiles = 0, n_split_items = 0;
    bool any_sync = false;
    double plan_seconds = 0.0;
    StagedHost st;                    // empty unless the plan runs the staged walk
};

// Validate the CSR.  Returns "" when valid, else a message.
std::string validate_csr(int64_t m, int64_t k, int64_t nnz, const int32_t* rowptr,
                         const int32_t* colidx);

// Build the canonical plan + tiles.  Throws std::runtime_error on bad params.
void build_plan(int64_t m, int64_t k, int64_t nnz, const int32_t* rowptr,
                const int32_t* colidx, int32_t bcols, const Params& p, PlanHost& out);

// Auto parameters from the per-bCols table and the problem size; h_req > 0
// fixes UFi, packed selects the table of the record walk.
Params choose_params(int64_t m, int64_t k, int64_t nnz, int32_t bcols, int n_sm, int h_req = 0,
                     bool packed = false);

// Build the staged walk's schedule from the canonical plan: row blocks of
// warps x npw panels, nsplit even column splits, stages of kb columns, record
// words rw per record.  Returns "" or why the configuration does not fit
// (shared-memory budget smem_cap bytes, at most kStMaxStages stages).
std::string build_staged(const PlanHost& ph, int bcols, int warps, int npw, int nsplit, int kb,
                         size_t smem_cap, StagedHost& st);
int rec_words(int h);   // record stride in 32-bit words (esc_kernel.cuh RecFmt<h>::W)

// Pick cta_warps from the item distribution and build the tile schedule.
void build_tiles(PlanHost& ph, int cta_warps, bool by_length = true);
// Column-window tiles: tile = item j of W consecutive panels (the same column
// window of W panels on one SM, so their B rows are re-read from L1); a split
// panel's items combine through a per-item workspace slot and a per-panel
// counter (the last item to arrive sums them in item order).
void build_tiles_cols(PlanHost& ph, int cta_warps, int bcols);

// Device-side view used by the kernels.
struct DevPlan {
    const int32_t* gpk = nullptr;       // int32[G]: column | pattern << 27
    const int32_t* slot = nullptr;      // int32[nnz]
    const int32_t* vbase = nullptr;     // int32[G]: slot of each gcol's first value (UFi > 1, escs_pack)
    const int32_t* items = nullptr;     // int4[n_slots]: panel, gcol_begin, gcol_end, slot_begin
    const int32_t* item_aux = nullptr;  // int32[n_slots]
    const int32_t* tile_heavy = nullptr;  // int2[n_tiles]
    const int32_t* heavy = nullptr;     // int4[n_heavy]
    const int32_t* slot_ws = nullptr;   // int4[n_slots] (column-window tiles)
    float* wsc = nullptr;               // column-window tiles: per-item partials
    int32_t* wsc_counters = nullptr;
    float* ws = nullptr;                // float[n_heavy_tiles * h * bcols]
    int32_t* counters = nullptr;        // int32[n_heavy]
    int m = 0, k = 0, nnz = 0, bcols = 0, h = 0, n_tiles = 0, cta_warps = 0, variant = 1, ufk = 4, colf = 0;
    int G = 0;
    bool any_sync = false;
    bool pdl = true;                    // programmatic dependent launch (ESCS_PDL=0 disables)
    int carveout = -1;                  // preferred shared-memory carveout (percent) of the gather
                                        // walk's launches, -1 = the driver's choice
    // a hybrid plan's part: plan row -> row of C, plan CSR position -> CSR
    // position of the caller's values (NULL: identity)
    const int32_t* rowmap = nullptr;
    const int32_t* vmap = nullptr;
    // staged walk (st_n_cta > 0): schedule arrays and the split workspace
    const int32_t* st_cta = nullptr;
    const int32_t* st_stage = nullptr;
    const int32_t* st_hdr = nullptr;
    const int32_t* st_src = nullptr;
    float* st_ws = nullptr;             // float[nsplit * m * bcols] when nsplit > 1
    int32_t* st_counters = nullptr;     // 2 per row block (in-kernel split combine)
    bool st_coop = false;               // grid co-resident: combine in the walk kernel
    int st_n_cta = 0, st_warps = 0, st_npw = 0, st_nsplit = 0, st_hs = 0, st_max_stages = 0;
    int st_sb_floats = 0, st_sr_words = 0, st_n_rec = 0;
};

// Launch the ESC SpMM kernel (one launch).  packed: `vals` is the record
// stream of escs_pack (record walk).  Returns a cudaError_t value.
int launch_spmm(const DevPlan& dp, const float* vals, const float* B, float* C, void* stream,
                bool vec_ok, bool packed = false, float* const* extra = nullptr,
                int n_extra = 0, long long row_off = 0, bool multicast = false);
// escs_spmm_group: n independent SpMMs, grouped into one launch per kernel
// instance (UFi = 1 vector plans; the rest launch one by one).
int launch_group(int n, const DevPlan* const* dps, const float* const* vals,
                 const float* const* B, float* const* C, void* stream);
// escs_pack: the record stream (packed_words(dp) int32 words).
int launch_pack(const DevPlan& dp, const float* vals, float* packed, void* stream);
int64_t packed_words(const DevPlan& dp);
// The staged walk: kernel instance exists?  Launch (1 or 2 kernels), shared
// memory per CTA, kernel attributes.
bool staged_supported(int h, int bcols, int colf, int npw);
int launch_staged(const DevPlan& dp, const float* rec, const float* B, float* C, void* stream,
                  bool probe = false);
size_t staged_smem_bytes(const DevPlan& dp);
int prepare_staged(const DevPlan& dp);
int staged_blocks_per_sm(const DevPlan& dp);
// Launch the gather probe (same walk, loads only); packed != NULL: the record walk.
int launch_probe(const DevPlan& dp, const float* B, float* sink, void* stream, bool vec_ok,
                 const float* packed = nullptr);
// Prepare kernel attributes (dynamic smem limits) once per plan.
int prepare_kernels(DevPlan& dp);
// Does a kernel instance exist for this configuration (packed: the record walk)?
bool kernel_supported(int h, int bcols, int variant, int ufk, int colf, bool packed = false);
int default_colf(int bcols);
int launch_spin(void* stream, long long cycles);   // tuner: busy-wait on the stream
size_t smem_bytes(const DevPlan& dp, bool packed = false);
// Resident CTAs per SM for this plan's launch configuration.
int blocks_per_sm(const DevPlan& dp, bool vec, bool probe, bool packed = false);
// The gather walk's preferred carveout for this plan (percent shared memory).
int gather_carveout(const DevPlan& dp, bool packed);

}  // namespace escs
