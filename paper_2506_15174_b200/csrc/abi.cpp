// abi.cpp -- the C ABI (include/escs.h): argument checking, error reporting,
// parameter choice, plan upload and the single launch of escs_spmm.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>

#include "../../include/escs.h"
#include "escs_internal.h"

struct escs_plan_impl {
    escs::PlanHost host;
    escs::Params params;
    escs::DevPlan dev;
    bool host_only = true;
    int device = -1;
    void* dmem = nullptr;
    size_t dbytes = 0, ws_bytes = 0;
    int autotuned = 0;   // 1: tuned at plan time, 2: parameters from the tuning cache
    bool pooled = false; // device memory from the planner's stream-ordered pool (autotuned plans)
    // hybrid plan (escs_params.hybrid_rows): a container of two parts, each an
    // ordinary plan of a row subset of A -- the hybrid_rows longest rows (in
    // descending length order) and the rest (in row order); aux holds each
    // part's row map and value map on the device
    escs_plan_impl* parts[2] = {nullptr, nullptr};
    int hybrid_rows = 0;
    void* aux = nullptr;
    int64_t part_words[2] = {0, 0};   // record-stream words of each part (packed layout: part 0, part 1)
};

namespace {

int pack_plan(escs_plan_t P, const float* vals, float* packed, void* stream);
int64_t plan_packed_words(escs_plan_t P);
escs_plan_t make_plan_hybrid(int64_t m, int64_t k, int64_t nnz, const int32_t* rowptr, const int32_t* colidx,
                             int32_t bCols, const escs_params* ep, int64_t X);
int64_t auto_hybrid_rows(int64_t m, int64_t nnz, const int32_t* rowptr, double* share);

thread_local int g_code = ESCS_OK;
thread_local std::string g_msg;

int fail(int code, const std::string& msg) {
    g_code = code;
    g_msg = msg;
    return code;
}
void clear_error() {
    g_code = ESCS_OK;
    g_msg.clear();
}

int sm_count_of_current_device() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
    return n > 0 ? n : 148;
}

// ESCS_PARAMS="ufi=4,T=64,warps=8,variant=1,ufk=4,colf=8"
void apply_env(escs::Params& p, bool& set_warps) {
    const char* e = std::getenv("ESCS_PARAMS");
    if (!e) return;
    std::string s(e);
    size_t i = 0;
    while (i < s.size()) {
        size_t j = s.find(',', i);
        if (j == std::string::npos) j = s.size();
        std::string kv = s.substr(i, j - i);
        size_t eq = kv.find('=');
        if (eq != std::string::npos) {
            std::string k = kv.substr(0, eq);
            int v = std::atoi(kv.c_str() + eq + 1);
            if (k == "ufi") p.h = v;
            else if (k == "T") p.T = v;
            else if (k == "warps") { p.cta_warps = v; set_warps = true; }
            else if (k == "variant") p.variant = v;
            else if (k == "ufk") p.ufk = v;
            else if (k == "colf") p.colf = v;
            else if (k == "order") p.tile_order = v;
            else if (k == "packed") p.packed = v;
            else if (k == "staged") p.staged = v;
            else if (k == "st_warps") p.st_warps = v;
            else if (k == "st_npw") p.st_npw = v;
            else if (k == "st_nsplit") p.st_nsplit = v;
            else if (k == "st_kb") p.st_kb = v;
        }
        i = j + 1;
    }
}

// Warps per CTA tile: at least the number of items of all but the heaviest 1%
// of panels (so they combine inside one CTA), rounded up to a multiple that
// gives about 8 warps per CTA; at most 16.  Skewed panels (power-law rows,
// C4: p99 items >= 4x median) get 4-warp tiles and combine heavy panels
// through the workspace (C4: 117 -> 92 us, profiles/r1_tune_c4.json).
// (16-warp tiles packing several panels were measured too: faster only when
// they remove a second wave, slower otherwise -- profiles/r1_tune_big.json.)
// Tile order: by item length when panel work is skewed (power-law rows, C4:
// 96 -> 82 us), else panel order (uniform layers: within noise, slightly
// better in panel order).  p99 vs median of the panels' stream lengths.
int auto_tile_order(const escs::PlanHost& ph) {
    const int64_t nP = ph.header[7];
    const int64_t NI = ph.item_panel.size();
    if (nP < 2) return 1;
    std::vector<int32_t> len(nP, 0);
    for (int64_t i = 0; i < NI; i++)
        len[ph.item_panel[i]] += ph.item_gcol_ptr[i + 1] - ph.item_gcol_ptr[i];
    const int64_t k99 = std::min<int64_t>(nP - 1, (nP * 99) / 100);
    std::nth_element(len.begin(), len.begin() + k99, len.end());
    const int32_t p99 = len[k99];
    std::nth_element(len.begin(), len.begin() + nP / 2, len.begin() + k99);
    const int32_t med = std::max(1, len[nP / 2]);
    return p99 >= 2 * med ? 2 : 1;
}

int auto_cta_warps(const escs::PlanHost& ph) {
    const int64_t nP = ph.header[7];
    const int64_t NI = ph.item_panel.size();
    if (nP == 0) return 8;
    std::vector<int32_t> per(nP, 0);
    for (int64_t i = 0; i < NI; i++) per[ph.item_panel[i]]++;
    const int64_t k99 = std::min<int64_t>(nP - 1, (nP * 99) / 100);
    std::nth_element(per.begin(), per.begin() + k99, per.end());
    const int typ = std::max(1, per[k99]);
    std::nth_element(per.begin(), per.begin() + nP / 2, per.begin() + k99);
    const int med = std::max(1, per[nP / 2]);
    if (typ >= 4 * med) return 4;
    if (typ >= 8) return std::min(typ, 16);
    return typ * std::max(1, 8 / typ);
}

template <class T>
size_t add_region(size_t& off, size_t count) {
    off = (off + 255) & ~size_t(255);
    size_t at = off;
    off += count * sizeof(T);
    return at;
}

#define CUDA_TRY(call)                                                                 \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess) {                                                       \
            fail(ESCS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));   \
            return false;                                                              \
        }                                                                              \
    } while (0)

// Shared memory a staged CTA may use: the sm_100 opt-in maximum (227 KB)
// less the kernel's static mbarriers and a margin.
constexpr size_t kStSmemCap = 227 * 1024 - 8 * 1024 - 512;   // static: mbarriers + combine buffer

// Auto tile of the staged walk: 16 warps x 1 panel per CTA (fewer when the
// matrix has fewer panels), column ranges so that about one CTA per SM runs
// (the B range plus the records fill most of the 227 KB), stages of ~32 KB of
// B rows (at most 16).  build_staged then checks the budget; the caller
// raises nsplit while it does not fit.
void auto_staged(escs::Params& p, const escs::PlanHost& ph, int bcols, int n_sm) {
    const int64_t nP = ph.header[7], k = ph.header[2], G = ph.header[9];
    if (!p.st_npw) p.st_npw = 1;
    if (!p.st_warps) p.st_warps = (int)std::max<int64_t>(1, std::min<int64_t>(16, (nP + p.st_npw - 1) / p.st_npw));
    const int64_t nslot = (int64_t)p.st_warps * p.st_npw;
    const int64_t n_rb = (nP + nslot - 1) / nslot;
    if (!p.st_nsplit) {
        // at most one wave of CTAs, leaving a few SMs free: a grid of exactly
        // one CTA per SM waits, launch after launch, for the last SM to drain
        // the previous kernel while its row blocks' CTAs spin in the combine
        // (512x4608@70% b128 eager: 148 CTAs 40 us, 144 CTAs 20.6 us;
        // profiles/r2_notes.md)
        int64_t ns = std::max<int64_t>(1, std::max(1, n_sm - 4) / n_rb);
        const int rw = escs::rec_words(ph.header[5]);
        for (;; ns++) {
            const double wd = std::ceil((double)k / ns);
            const double rec = 1.25 * (double)G / (double)(n_rb * ns) + 64;
            if ((wd * bcols + rec * rw) * 4.0 + 16 * 4 * 20 <= (double)kStSmemCap || ns >= k) break;
        }
        p.st_nsplit = (int)std::min<int64_t>(ns, k);
    }
    if (!p.st_kb) {
        const int64_t wd = (k + p.st_nsplit - 1) / p.st_nsplit;
        // ~32 KB of B rows per stage (dominant layer: 16 KB stages 17.9 us,
        // 32 KB 17.1 us; profiles/r2_notes.md §4)
        const int64_t kb = std::max<int64_t>(8, 32768 / (4 * bcols));
        p.st_kb = (int)std::max<int64_t>(kb, (wd + 15) / 16);
    }
}

double g_tune_build_s = 0.0, g_tune_time_s = 0.0;   // ESCS_TUNE_DEBUG accounting
double g_dbg_upload_s = 0.0, g_dbg_prepare_s = 0.0, g_dbg_host_s = 0.0, g_dbg_free_s = 0.0;
long g_tune_cands = 0;
struct TuneReport {
    ~TuneReport() {
        if (g_tune_cands)
            std::fprintf(stderr, "escs tune: %ld candidates, %.2f s building plans (host %.2f, upload %.2f, "
                                 "kernel attributes %.2f), %.2f s timing, %.2f s freeing\n", g_tune_cands,
                         g_tune_build_s, g_dbg_host_s, g_dbg_upload_s, g_dbg_prepare_s, g_tune_time_s, g_dbg_free_s);
    }
} g_tune_report;

// B sizes for which the tuner also searches at a 2% carveout: above 96 KB (a
// smaller B fits L1 at any carveout: the second search never won) and up to
// ESCS_L1_FIT_KB (default 320: wins at 128-288 KB, rare beyond; notes §10)
int64_t l1_fit_bytes() {
    static const int64_t v = [] {
        const char* e = std::getenv("ESCS_L1_FIT_KB");
        return (int64_t)(e ? std::atoi(e) : 320) * 1024;
    }();
    return v;
}

bool tune_debug() {
    static const bool on = [] {
        const char* e = std::getenv("ESCS_TUNE_DEBUG");
        return e && e[0] == '1';
    }();
    return on;
}

// The autotuner builds and frees thousands of candidate plans: cudaMalloc /
// cudaFree per candidate (the latter synchronising the device) was ~10 s of the
// suite's ~24 s of planning (ESCS_TUNE_DEBUG accounting).  Autotuned plans
// therefore take their memory from a private stream-ordered pool (retained up
// to 1 GiB), allocated and freed on the legacy stream.
cudaMemPool_t plan_pool(int device) {
    static std::mutex mu;
    static std::map<int, cudaMemPool_t> pools;
    std::lock_guard<std::mutex> lk(mu);
    auto it = pools.find(device);
    if (it != pools.end()) return it->second;
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
        cudaGetLastError();
        pool = nullptr;
    } else {
        uint64_t keep = 1ull << 30;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pools[device] = pool;
    return pool;
}

bool upload(escs_plan_impl* P) {
    auto& ph = P->host;
    auto& dp = P->dev;
    const int h = ph.header[5], n = ph.header[4];
    const int64_t NG = ph.header[8], G = ph.header[9], nnz = ph.header[3];
    // packed gcols (column | pattern << 27) and items {panel, gcol_begin,
    // gcol_end, slot_begin}: the kernel needs no group records (Reading R1:
    // a panel's value slots are contiguous in stream order).
    // (UFi 5..8, record walk only: col | mask << 24, k < 2^24)
    const int shift = h <= 4 ? 27 : 24;
    std::vector<int32_t> gpk(G);
    for (int64_t g = 0; g < NG; g++)
        for (int32_t c = ph.grp_col_ptr[g]; c < ph.grp_col_ptr[g + 1]; c++)
            gpk[c] = (int32_t)((uint32_t)ph.gcol[c] | ((uint32_t)ph.grp_mask[g] << shift));
    const int64_t NS = ph.slot_item.size();
    std::vector<int32_t> items(4 * NS, 0);
    for (int64_t k = 0; k < NS; k++) {
        const int32_t i = ph.slot_item[k];
        if (i < 0) continue;
        const int32_t gb = ph.item_group_begin[i], s0 = ph.item_gcol_ptr[i];
        int32_t sb = 0;
        if (gb < NG)
            sb = ph.grp_val_ptr[gb] +
                 (s0 - ph.grp_col_ptr[gb]) * __builtin_popcount((unsigned)ph.grp_mask[gb]);
        items[4 * k + 0] = ph.item_panel[i];
        items[4 * k + 1] = s0;
        items[4 * k + 2] = ph.item_gcol_ptr[i + 1];
        items[4 * k + 3] = sb;
    }
    size_t off = 0;
    // slot of each gcol's first value (escs_pack's record stream, UFi > 1)
    std::vector<int32_t> vbase;
    if (h > 1) {
        vbase.resize(G);
        for (int64_t g = 0; g < NG; g++) {
            const int p = __builtin_popcount((unsigned)ph.grp_mask[g]);
            for (int32_t c = ph.grp_col_ptr[g]; c < ph.grp_col_ptr[g + 1]; c++)
                vbase[c] = ph.grp_val_ptr[g] + (c - ph.grp_col_ptr[g]) * p;
        }
    }
    const size_t o_gpk = add_region<int32_t>(off, G);
    const size_t o_slot = add_region<int32_t>(off, nnz);
    const size_t o_vb = add_region<int32_t>(off, vbase.size());
    const size_t o_items = add_region<int32_t>(off, 4 * NS);
    const size_t o_aux = add_region<int32_t>(off, NS);
    const size_t o_tiles = add_region<int32_t>(off, ph.tile_heavy.size());
    const size_t o_heavy = add_region<int32_t>(off, ph.heavy_info.size());
    const size_t o_cnt = add_region<int32_t>(off, ph.n_heavy);
    const size_t ws_elems = (size_t)ph.n_heavy_tiles * h * n;
    const size_t o_ws = add_region<float>(off, ws_elems);
    const auto& st = ph.st;
    const size_t o_sws = add_region<int32_t>(off, ph.slot_ws.size());
    const size_t o_wscc = add_region<int32_t>(off, ph.n_wsc_counters);
    const size_t o_wsc = add_region<float>(off, (size_t)ph.wsc_floats);
    const size_t o_stc = add_region<int32_t>(off, st.cta.size());
    const size_t o_sts = add_region<int32_t>(off, st.stage.size());
    const size_t o_sth = add_region<int32_t>(off, st.hdr.size());
    const size_t o_str = add_region<int32_t>(off, st.src.size());
    const size_t st_ws = (st.n_cta && st.nsplit > 1) ? (size_t)st.nsplit * ph.header[1] * n : 0;
    const size_t o_stw = add_region<float>(off, st_ws);
    const int64_t st_rb = st.n_cta ? st.n_cta / st.nsplit : 0;
    const size_t o_stk = add_region<int32_t>(off, 2 * st_rb);
    off = std::max<size_t>(off, 256);
    void* d = nullptr;
    cudaError_t e = cudaErrorMemoryAllocation;
    if (P->pooled) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaMemPool_t pool = plan_pool(dev)) {
            e = cudaMallocFromPoolAsync(&d, off, pool, 0);
            if (e != cudaSuccess) cudaGetLastError();
        }
        if (e != cudaSuccess) P->pooled = false;
    }
    if (!P->pooled) e = cudaMalloc(&d, off);
    if (e != cudaSuccess) {
        fail(e == cudaErrorMemoryAllocation ? ESCS_ERR_OOM : ESCS_ERR_CUDA,
             std::string("cudaMalloc(") + std::to_string(off) + "): " + cudaGetErrorString(e));
        return false;
    }
    P->dmem = d;
    P->dbytes = off;
    P->ws_bytes = (ws_elems + st_ws + (size_t)ph.wsc_floats) * sizeof(float);
    char* b = static_cast<char*>(d);
    auto put = [&](size_t o, const void* src, size_t bytes) -> bool {
        if (!bytes) return true;
        CUDA_TRY(cudaMemcpy(b + o, src, bytes, cudaMemcpyHostToDevice));
        return true;
    };
    if (!put(o_gpk, gpk.data(), G * 4)) return false;
    if (!put(o_slot, ph.slot_src.data(), nnz * 4)) return false;
    if (!put(o_vb, vbase.data(), vbase.size() * 4)) return false;
    if (!put(o_items, items.data(), items.size() * 4)) return false;
    if (!put(o_aux, ph.slot_aux.data(), NS * 4)) return false;
    if (!put(o_tiles, ph.tile_heavy.data(), ph.tile_heavy.size() * 4)) return false;
    if (!put(o_heavy, ph.heavy_info.data(), ph.heavy_info.size() * 4)) return false;
    if (ph.n_heavy) CUDA_TRY(cudaMemset(b + o_cnt, 0, ph.n_heavy * 4));
    if (!ph.slot_ws.empty()) {
        if (!put(o_sws, ph.slot_ws.data(), ph.slot_ws.size() * 4)) return false;
        if (ph.n_wsc_counters) CUDA_TRY(cudaMemset(b + o_wscc, 0, (size_t)ph.n_wsc_counters * 4));
        dp.slot_ws = reinterpret_cast<const int32_t*>(b + o_sws);
        dp.wsc_counters = reinterpret_cast<int32_t*>(b + o_wscc);
        dp.wsc = reinterpret_cast<float*>(b + o_wsc);
    }
    if (!put(o_stc, st.cta.data(), st.cta.size() * 4)) return false;
    if (!put(o_sts, st.stage.data(), st.stage.size() * 4)) return false;
    if (!put(o_sth, st.hdr.data(), st.hdr.size() * 4)) return false;
    if (!put(o_str, st.src.data(), st.src.size() * 4)) return false;
    if (st.n_cta) {
        dp.st_cta = reinterpret_cast<const int32_t*>(b + o_stc);
        dp.st_stage = reinterpret_cast<const int32_t*>(b + o_sts);
        dp.st_hdr = reinterpret_cast<const int32_t*>(b + o_sth);
        dp.st_src = reinterpret_cast<const int32_t*>(b + o_str);
        dp.st_ws = st_ws ? reinterpret_cast<float*>(b + o_stw) : nullptr;
        dp.st_counters = reinterpret_cast<int32_t*>(b + o_stk);
        CUDA_TRY(cudaMemset(b + o_stk, 0, 2 * st_rb * 4));
    }
    dp.gpk = reinterpret_cast<const int32_t*>(b + o_gpk);
    dp.slot = reinterpret_cast<const int32_t*>(b + o_slot);
    dp.vbase = h > 1 ? reinterpret_cast<const int32_t*>(b + o_vb) : nullptr;
    dp.items = reinterpret_cast<const int32_t*>(b + o_items);
    dp.item_aux = reinterpret_cast<const int32_t*>(b + o_aux);
    dp.tile_heavy = reinterpret_cast<const int32_t*>(b + o_tiles);
    dp.heavy = reinterpret_cast<const int32_t*>(b + o_heavy);
    dp.counters = reinterpret_cast<int32_t*>(b + o_cnt);
    dp.ws = reinterpret_cast<float*>(b + o_ws);
    CUDA_TRY(cudaDeviceSynchronize());
    return true;
}

escs_plan_t make_plan_fixed(int64_t m, int64_t k, int64_t nnz, const int32_t* rowptr,
                            const int32_t* colidx, int32_t bCols, const escs_params* ep,
                            bool pooled = false) {
    clear_error();
    if (m < 1 || k < 1 || nnz < 0 || bCols < 1) {
        fail(ESCS_ERR_ARG, "m, k, bCols must be >= 1 and nnz >= 0");
        return nullptr;
    }
    const int64_t lim = (int64_t)1 << 31;
    if (m >= lim || k >= lim || nnz >= lim || m * bCols >= lim || k * bCols >= lim) {
        fail(ESCS_ERR_ARG, "m, k, nnz, m*bCols and k*bCols must be < 2^31");
        return nullptr;
    }
    if (bCols > ESCS_MAX_BCOLS) {
        fail(ESCS_ERR_UNSUPPORTED, "bCols > ESCS_MAX_BCOLS (256)");
        return nullptr;
    }
    if (ep) {
        if (ep->reserved[0] != 0) {
            fail(ESCS_ERR_ARG, "escs_params.reserved must be zero");
            return nullptr;
        }
        if (ep->packed < 0 || ep->packed > 1) {
            fail(ESCS_ERR_ARG, "escs_params.packed must be 0 or 1");
            return nullptr;
        }
        if (ep->carveout < -2 || ep->carveout > 100) {
            fail(ESCS_ERR_ARG, "escs_params.carveout must be -2..100");
            return nullptr;
        }
    }
    std::string v = escs::validate_csr(m, k, nnz, rowptr, colidx);
    if (!v.empty()) {
        fail(ESCS_ERR_CSR, "invalid CSR: " + v);
        return nullptr;
    }
    const bool host_only = ep && ep->host_only;
    int device = -1;
    if (!host_only) {
        cudaError_t e = cudaGetDevice(&device);
        if (e != cudaSuccess) {
            fail(ESCS_ERR_CUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
            return nullptr;
        }
    }
    const bool want_packed = ep && ep->packed;
    escs::Params p = escs::choose_params(m, k, nnz, bCols, host_only ? 148 : sm_count_of_current_device(),
                                         ep ? ep->ufi : 0, want_packed);
    bool set_warps = false;
    apply_env(p, set_warps);
    if (ep) {
        if (ep->ufi) p.h = ep->ufi;
        if (ep->packed) p.packed = 1;
        if (ep->T) p.T = ep->T;
        if (ep->cta_warps) { p.cta_warps = ep->cta_warps; set_warps = true; }
        if (ep->variant) p.variant = ep->variant;
        if (ep->ufk) p.ufk = ep->ufk;
        if (ep->colf) p.colf = ep->colf;
        if (ep->tile_order) p.tile_order = ep->tile_order;
        if (ep->nthreads) p.nthreads = ep->nthreads;
        if (ep->staged) p.staged = ep->staged;
        if (ep->st_warps) p.st_warps = ep->st_warps;
        if (ep->st_npw) p.st_npw = ep->st_npw;
        if (ep->st_nsplit) p.st_nsplit = ep->st_nsplit;
        if (ep->st_kb) p.st_kb = ep->st_kb;
    }
    // CTA tile width: up to 16 warps (512 threads, the CSR walk's launch
    // bounds); up to 28 for the record walk (72 registers x 28 x 32 <= 64K)
    const int max_warps = p.packed ? 28 : 16;
    if (p.h < 1 || p.h > 16 || p.T < 1 || (set_warps && (p.cta_warps < 1 || p.cta_warps > max_warps)) ||
        p.variant < 1 || p.variant > 2 || p.tile_order < 0 || p.tile_order > 3 ||
        !(p.colf == 0 || p.colf == 4 || p.colf == 8 || p.colf == 16)) {
        fail(ESCS_ERR_ARG, "parameters out of range (ufi 1..16, T >= 1, cta_warps 1..16 (1..28 packed), "
                           "variant 1..2, colf 0/4/8/16, tile_order 0..3)");
        return nullptr;
    }
    if (p.variant == 1 && !(bCols == 4 || bCols == 8 || bCols == 16 || bCols == 32 || bCols == 64 ||
                            bCols == 128 || bCols == 256))
        p.variant = 2;
    if (!host_only && k >= (1 << 27)) {
        fail(ESCS_ERR_UNSUPPORTED, "device plans need k < 2^27 (packed column words)");
        return nullptr;
    }
    if (!host_only && p.h > 4 && k >= (1 << 24)) {
        fail(ESCS_ERR_UNSUPPORTED, "device plans with UFi > 4 need k < 2^24 (packed column words)");
        return nullptr;
    }
    if (p.staged < 0 || p.staged > 2) {
        fail(ESCS_ERR_ARG, "escs_params.staged must be 0, 1 or 2");
        return nullptr;
    }
    if (p.staged == 2 && !(p.packed && p.variant == 1 && (bCols == 32 || bCols == 64 || bCols == 128))) {
        fail(ESCS_ERR_UNSUPPORTED, "the staged walk needs packed = 1, the vector lane map and bCols 32, 64 or 128");
        return nullptr;
    }
    if (p.variant != 1) {
        p.colf = 0;
        p.packed = 0;   // the record walk needs the vector lane map: a CSR-walk plan
    } else if (p.colf == 0) {
        p.colf = escs::default_colf(bCols);
    }
    // the record walk has every coarsening factor at every UFi; the CSR walk
    // has the alternative factors at UFi = 1 only (tools/gen_kernels.py)
    if (!p.packed && p.h > 1 && p.variant == 1) p.colf = escs::default_colf(bCols);
    // automatic UFk: fall back to the largest UFk the chosen lane map has
    // (wide per-lane tiles carry fewer rows in flight: UFk x colf <= 64)
    if (!host_only && !(ep && ep->ufk) && !std::getenv("ESCS_PARAMS")) {
        // the table's columns per lane may have no instance at this UFi (UFi
        // 6/8 records: default lane maps only): fall back to the default map
        if (!(ep && ep->colf) && p.variant == 1 && p.colf != escs::default_colf(bCols)) {
            bool any = false;
            for (int u = 1; u <= 8 && !any; u *= 2)
                any = escs::kernel_supported(p.h, bCols, p.variant, u, p.colf, p.packed);
            if (!any) p.colf = escs::default_colf(bCols);
        }
        while (p.ufk > 1 && !escs::kernel_supported(p.h, bCols, p.variant, p.ufk, p.colf, p.packed))
            p.ufk /= 2;
    }
    if (!host_only && !escs::kernel_supported(p.h, bCols, p.variant, p.ufk, p.colf, p.packed)) {
        fail(ESCS_ERR_UNSUPPORTED, "no kernel for ufi=" + std::to_string(p.h) + " bCols=" +
                                       std::to_string(bCols) + " variant=" +
                                       std::to_string(p.variant) + " ufk=" + std::to_string(p.ufk) +
                                       " colf=" + std::to_string(p.colf) + (p.packed ? " (packed)" : ""));
        return nullptr;
    }
    escs_plan_impl* P = new (std::nothrow) escs_plan_impl();
    if (!P) {
        fail(ESCS_ERR_OOM, "host allocation");
        return nullptr;
    }
    try {
        escs::build_plan(m, k, nnz, rowptr, colidx, bCols, p, P->host);
        if (!set_warps) p.cta_warps = auto_cta_warps(P->host);
        const char* to = std::getenv("ESCS_TILE_ORDER");   // "panel" | "length" override
        if (to && std::string(to) == "panel") p.tile_order = 1;
        else if (to && std::string(to) == "length") p.tile_order = 2;
        if (p.tile_order == 3 && p.h != 1) p.tile_order = 1;   // column windows: UFi 1 (column-ordered streams)
        if (p.tile_order < 1 || p.tile_order > 3) p.tile_order = auto_tile_order(P->host);
        if (p.tile_order == 3)
            escs::build_tiles_cols(P->host, p.cta_warps, bCols);
        else
            escs::build_tiles(P->host, p.cta_warps, p.tile_order == 2);
        if (p.staged == 2) {
            // lane map of the staged walk: the plan's columns per lane if that
            // instance exists, else 4
            const int F = escs::staged_supported(p.h, bCols, p.colf, p.st_npw ? p.st_npw : 1) ? p.colf : 4;
            if (!escs::staged_supported(p.h, bCols, F, p.st_npw ? p.st_npw : 1)) {
                delete P;
                fail(ESCS_ERR_UNSUPPORTED, "no staged kernel for ufi=" + std::to_string(p.h) + " bCols=" +
                                               std::to_string(bCols) + " npw=" + std::to_string(p.st_npw));
                return nullptr;
            }
            p.colf = F;
            const bool fixed_split = p.st_nsplit != 0;
            auto_staged(p, P->host, bCols, host_only ? 148 : sm_count_of_current_device());
            std::string why;
            for (int tries = 0; tries < 64; tries++) {
                why = escs::build_staged(P->host, bCols, p.st_warps, p.st_npw, p.st_nsplit, p.st_kb,
                                         kStSmemCap, P->host.st);
                if (why.empty() || fixed_split || p.st_nsplit >= k) break;
                if (why.find("shared memory") == std::string::npos && why.find("stages") == std::string::npos)
                    break;
                p.st_nsplit += std::max(1, p.st_nsplit / 8);   // did not fit: more, narrower ranges
                const int64_t wd = (k + p.st_nsplit - 1) / p.st_nsplit;
                p.st_kb = std::max<int>(p.st_kb, (int)((wd + 15) / 16));
            }
            if (!why.empty()) {
                delete P;
                fail(ESCS_ERR_UNSUPPORTED, "staged walk: " + why);
                return nullptr;
            }
        }
    } catch (const std::bad_alloc&) {
        delete P;
        fail(ESCS_ERR_OOM, "host allocation while planning");
        return nullptr;
    } catch (const std::exception& ex) {
        delete P;
        fail(ESCS_ERR_INTERNAL, ex.what());
        return nullptr;
    }
    P->params = p;
    P->host_only = host_only;
    P->device = device;
    P->pooled = pooled && !host_only;
    auto& dp = P->dev;
    dp.m = (int)m; dp.k = (int)k; dp.nnz = (int)nnz; dp.bcols = bCols; dp.h = p.h;
    dp.n_tiles = P->host.n_tiles; dp.cta_warps = p.cta_warps; dp.variant = p.variant;
    dp.ufk = p.ufk; dp.colf = p.colf; dp.any_sync = P->host.any_sync;
    dp.G = P->host.header[9];
    if (P->host.st.n_cta) {
        const auto& st = P->host.st;
        dp.st_n_cta = st.n_cta; dp.st_warps = st.warps; dp.st_npw = st.npw; dp.st_nsplit = st.nsplit;
        dp.st_hs = st.hs; dp.st_max_stages = st.max_stages;
        dp.st_sb_floats = (st.max_k * bCols + 31) / 32 * 32;   // records start 128-byte aligned
        dp.st_sr_words = (st.max_rec * st.rw + 3) / 4 * 4;
        dp.st_n_rec = (int)st.src.size();
    }
    {
        const char* e = std::getenv("ESCS_PDL");
        dp.pdl = !(e && e[0] == '0');
    }
    if (!host_only) {
        const auto tu0 = std::chrono::steady_clock::now();
        if (!upload(P)) {
            escs_free(P);
            return nullptr;
        }
        const auto tu1 = std::chrono::steady_clock::now();
        int e = escs::prepare_kernels(dp);
        {   // L1 for the gathered B rows: the carveout that just holds the walk's occupancy
            const char* lm = std::getenv("ESCS_L1MAX");
            const int cv = ep ? ep->carveout : 0;
            if (!e && cv == 0 && !(lm && lm[0] == '0')) dp.carveout = escs::gather_carveout(dp, p.packed != 0);
            else if (cv > 0) dp.carveout = std::min(cv, 100);
            else if (cv == -2) dp.carveout = 0;
        }
        if (!e && dp.st_n_cta) {
            e = escs::prepare_staged(dp);
            // the split combine runs in the walk kernel when the whole grid
            // can be resident at once (cooperative launch); else a second,
            // tiny kernel sums the partials
            const char* ec = std::getenv("ESCS_ST_COOP");
            const int nb = e ? 0 : escs::staged_blocks_per_sm(dp);
            dp.st_coop = !(ec && ec[0] == '0') && nb > 0 &&
                         (int64_t)dp.st_n_cta <= (int64_t)nb * sm_count_of_current_device();
        }
        if (tune_debug()) {
            const auto tu2 = std::chrono::steady_clock::now();
            g_dbg_upload_s += std::chrono::duration<double>(tu1 - tu0).count();
            g_dbg_prepare_s += std::chrono::duration<double>(tu2 - tu1).count();
            g_dbg_host_s += P->host.plan_seconds;
        }
        if (e) {
            fail(ESCS_ERR_CUDA, std::string("kernel attributes: ") +
                                    cudaGetErrorString((cudaError_t)e));
            escs_free(P);
            return nullptr;
        }
    }
    return P;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---------------------------------------------------------------- autotune
// The paper's scheduler & tuner (§3.5) is profiling-based: here the
// profiling runs at plan time, on the device the plan is bound to, for this
// matrix and bCols.  Coordinate descent over the item size T (with the auto
// tile width), then the tile width W, then UFk; every candidate is a complete
// canonical plan, timed as back-to-back launches (min over 3 batches of 8).
// Throughput objective (autotune = 2): ESCS_TUNE_STREAMS copies of a candidate
// plan (each with its own workspace/counters and C) run concurrently, one per
// stream, as independent layers of a suite would.
constexpr int kTuneStreams = 16;  // capacity; ESCS_TUNE_STREAMS (default 8) chains are timed
int tune_streams() {
    const char* e = std::getenv("ESCS_TUNE_STREAMS");
    const int v = e ? std::atoi(e) : 8;
    return v < 2 ? 2 : v > kTuneStreams ? kTuneStreams : v;
}
struct TuneBufs {
    float *vals = nullptr, *B = nullptr, *C = nullptr;
    float* packed = nullptr;          // record stream of the candidate (packed objective)
    size_t packed_cap = 0;            // words
    float* Cx[kTuneStreams] = {};
    cudaStream_t stream = nullptr;
    cudaStream_t sx[kTuneStreams] = {};
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaEvent_t ex[kTuneStreams] = {};
    int ns = 0;                       // concurrent chains timed (0: latency objective)
    // per-stream heavy-panel workspace + counters for the concurrent copies
    // (zeroed once; every launch leaves its counters at zero again)
    float* wsx[kTuneStreams] = {};
    int32_t* cntx[kTuneStreams] = {};
    size_t ws_cap = 0, cnt_cap = 0;
    void free_scratch() {
        for (int i = 0; i < kTuneStreams; i++) {
            if (wsx[i]) cudaFree(wsx[i]);
            if (cntx[i]) cudaFree(cntx[i]);
            wsx[i] = nullptr;
            cntx[i] = nullptr;
        }
        ws_cap = cnt_cap = 0;
    }
    // Grow the per-stream workspaces.  The capacities are raised only after
    // every allocation succeeded; on failure everything is released (caps 0),
    // so a later call cannot mistake a partial set for a usable one.
    bool scratch(size_t ws_elems, size_t n_cnt) {
        if (ws_elems <= ws_cap && n_cnt <= cnt_cap) return true;
        cudaDeviceSynchronize();
        const size_t wc = std::max(ws_cap, ws_elems), cc = std::max(cnt_cap, n_cnt);
        free_scratch();
        for (int i = 0; i < ns; i++) {
            if (cudaMalloc(&wsx[i], std::max<size_t>(wc, 1) * 4) != cudaSuccess ||
                cudaMalloc(&cntx[i], std::max<size_t>(cc, 1) * 4) != cudaSuccess ||
                cudaMemset(cntx[i], 0, std::max<size_t>(cc, 1) * 4) != cudaSuccess) {
                cudaGetLastError();
                free_scratch();
                return false;
            }
        }
        if (cudaDeviceSynchronize() != cudaSuccess) {
            cudaGetLastError();
            free_scratch();
            return false;
        }
        ws_cap = wc;
        cnt_cap = cc;
        return true;
    }
    // the candidate's record stream (packed objective): escs_pack of the
    // tuning values into a buffer grown on demand
    bool pack_for(escs_plan_t P) {
        const size_t w = (size_t)plan_packed_words(P);
        if (w > packed_cap) {
            cudaDeviceSynchronize();
            if (packed) cudaFree(packed);
            packed = nullptr;
            packed_cap = 0;
            if (cudaMalloc(&packed, std::max<size_t>(w, 4) * 4) != cudaSuccess) {
                cudaGetLastError();
                packed = nullptr;
                return false;
            }
            packed_cap = w;
        }
        if (pack_plan(P, vals, packed, stream) != 0) {
            cudaGetLastError();
            return false;
        }
        return true;
    }
    bool ok = false;
    TuneBufs(int64_t m, int64_t k, int64_t nnz, int32_t n, bool concurrent) {
        ok = cudaMalloc(&vals, std::max<int64_t>(nnz, 1) * 4) == cudaSuccess &&
             cudaMalloc(&B, (size_t)k * n * 4) == cudaSuccess &&
             cudaMalloc(&C, (size_t)m * n * 4) == cudaSuccess &&
             cudaMemset(vals, 0, std::max<int64_t>(nnz, 1) * 4) == cudaSuccess &&
             cudaMemset(B, 0, (size_t)k * n * 4) == cudaSuccess &&
             cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreate(&e0) == cudaSuccess && cudaEventCreate(&e1) == cudaSuccess;
        ns = concurrent ? tune_streams() : 0;
        for (int i = 0; ok && i < ns; i++)
            ok = cudaMalloc(&Cx[i], (size_t)m * n * 4) == cudaSuccess &&
                 cudaStreamCreateWithFlags(&sx[i], cudaStreamNonBlocking) == cudaSuccess &&
                 cudaEventCreateWithFlags(&ex[i], cudaEventDisableTiming) == cudaSuccess;
        if (!ok) cudaGetLastError();
    }
    ~TuneBufs() {
        if (vals) cudaFree(vals);
        if (B) cudaFree(B);
        if (C) cudaFree(C);
        if (packed) cudaFree(packed);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        if (stream) cudaStreamDestroy(stream);
        for (int i = 0; i < kTuneStreams; i++) {
            if (Cx[i]) cudaFree(Cx[i]);
            if (sx[i]) cudaStreamDestroy(sx[i]);
            if (ex[i]) cudaEventDestroy(ex[i]);
        }
        free_scratch();
        cudaGetLastError();
    }
};

constexpr float kFailed = 1e30f;



// One SpMM launch of whichever walk the plan runs (the staged walk for a
// staged plan's record stream).
int launch_plan(const escs::DevPlan& dp, const float* v, const float* B, float* C, void* stream, bool vec,
                bool packed) {
    if (packed && dp.st_n_cta) return escs::launch_staged(dp, v, B, C, stream);
    return escs::launch_spmm(dp, v, B, C, stream, vec, packed);
}

// escs_spmm_packed / escs_pack of any plan, a hybrid container included (its
// parts in order, part 1's records after part 0's).
int launch_packed_plan(escs_plan_t P, const float* packed, const float* B, float* C, void* stream, bool vec) {
    if (!P->parts[0]) return launch_plan(P->dev, packed, B, C, stream, vec, true);
    for (int q = 0; q < 2; q++) {
        const int e = launch_plan(P->parts[q]->dev, packed + (q ? P->part_words[0] : 0), B, C, stream, vec, true);
        if (e) return e;
    }
    return 0;
}
int pack_plan(escs_plan_t P, const float* vals, float* packed, void* stream) {
    if (!P->parts[0]) return escs::launch_pack(P->dev, vals, packed, stream);
    for (int q = 0; q < 2; q++) {
        const int e = escs::launch_pack(P->parts[q]->dev, vals, packed + (q ? P->part_words[0] : 0), stream);
        if (e) return e;
    }
    return 0;
}
int64_t plan_packed_words(escs_plan_t P) {
    return P->parts[0] ? P->part_words[0] + P->part_words[1] : escs::packed_words(P->dev);
}

// Latency objective: batches of 16 back-to-back launches queued behind a
// ~100 us busy-wait (the host enqueues the batch while the GPU spins): GPU
// time only; min over 3 batches.  A candidate whose launch fails is rejected
// (time kFailed, CUDA error cleared) -- it must never win by timing no work.
// Latency objective, graph mode (the default, ESCS_TUNE_GRAPH != 0): the
// batch of kBatch back-to-back launches is captured once into a CUDA graph
// and replayed -- the way a fixed layer sequence runs in production (and
// bench.py's step), launch overhead excluded; min over 3 replays.  Capture
// failures fall back to eager batches.
float time_plan_graph(escs_plan_t P, TuneBufs& b, bool packed, const float* v, bool vec) {
    constexpr int kBatch = 16;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    if (cudaStreamBeginCapture(b.stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        return -1.f;
    }
    bool ok = true;
    for (int i = 0; i < kBatch; i++)
        ok = ok && (packed ? launch_packed_plan(P, v, b.B, b.C, b.stream, vec)
                           : launch_plan(P->dev, v, b.B, b.C, b.stream, vec, false)) == 0;
    const cudaError_t ce = cudaStreamEndCapture(b.stream, &g);
    if (ce != cudaSuccess || !ok || !g || cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
        cudaGetLastError();
        if (g) cudaGraphDestroy(g);
        cudaStreamSynchronize(b.stream);
        cudaGetLastError();
        return -1.f;
    }
    float best = kFailed;
    for (int rep = 0; rep < 4 && ok; rep++) {
        escs::launch_spin(b.stream, 100000);
        cudaEventRecord(b.e0, b.stream);
        ok = cudaGraphLaunch(ge, b.stream) == cudaSuccess;
        cudaEventRecord(b.e1, b.stream);
        if (cudaEventSynchronize(b.e1) != cudaSuccess || !ok) {
            cudaGetLastError();
            cudaStreamSynchronize(b.stream);
            cudaGetLastError();
            best = kFailed;
            break;
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, b.e0, b.e1);
        if (rep > 0) best = std::min(best, ms / kBatch);   // the first replay uploads the graph
    }
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    return best;
}

float time_plan(escs_plan_t P, TuneBufs& b, bool packed) {
    float best = kFailed;
    const bool vec = aligned16(b.B) && aligned16(b.C);
    if (packed && !b.pack_for(P)) return kFailed;
    const float* v = packed ? b.packed : b.vals;
    for (int w = 0; w < 2; w++)
        if ((packed ? launch_packed_plan(P, v, b.B, b.C, b.stream, vec)
                    : launch_plan(P->dev, v, b.B, b.C, b.stream, vec, false)) != 0) {
            cudaGetLastError();
            cudaStreamSynchronize(b.stream);   // nothing of the candidate left in flight
            cudaGetLastError();
            return kFailed;
        }
    static const bool graph = [] {
        const char* e = std::getenv("ESCS_TUNE_GRAPH");
        return !(e && e[0] == '0');
    }();
    if (graph) {
        const float t = time_plan_graph(P, b, packed, v, vec);
        if (t >= 0.f) return t;
    }
    constexpr int kBatch = 16;
    for (int rep = 0; rep < 3; rep++) {
        escs::launch_spin(b.stream, 200000);
        cudaEventRecord(b.e0, b.stream);
        bool ok = true;
        for (int i = 0; i < kBatch; i++)
            ok = ok && (packed ? launch_packed_plan(P, v, b.B, b.C, b.stream, vec)
                               : launch_plan(P->dev, v, b.B, b.C, b.stream, vec, false)) == 0;
        cudaEventRecord(b.e1, b.stream);
        if (cudaEventSynchronize(b.e1) != cudaSuccess || !ok) {
            cudaGetLastError();
            cudaStreamSynchronize(b.stream);
            cudaGetLastError();
            return kFailed;
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, b.e0, b.e1);
        best = std::min(best, ms / kBatch);
    }
    return best;
}

// Throughput objective: the copies run one per stream, each stream a chain of
// kBatch launches, all released together after the busy-wait; time per
// launch = span / (kBatch * copies).
float time_plans_concurrent(escs_plan_t P0, TuneBufs& b, bool packed) {
    float best = kFailed;
    const bool vec = aligned16(b.B) && aligned16(b.C);
    // the copies share the read-only plan arrays; each has its own workspace
    // and counters (one plan must not run on two streams at once)
    // staged and hybrid plans keep per-plan state the copies would share (the
    // column-range partials and counters; two parts): not timed concurrently
    if (P0->dev.st_n_cta || P0->parts[0]) return kFailed;
    const auto& ph = P0->host;
    if (!b.scratch((size_t)ph.n_heavy_tiles * P0->dev.h * P0->dev.bcols, (size_t)ph.n_heavy))
        return kFailed;
    if (packed && !b.pack_for(P0)) return kFailed;
    const float* v = packed ? b.packed : b.vals;
    const int ns = b.ns;
    escs::DevPlan dp[kTuneStreams];
    for (int i = 0; i < ns; i++) {
        dp[i] = P0->dev;
        dp[i].ws = b.wsx[i];
        dp[i].counters = b.cntx[i];
    }
    if (cudaStreamSynchronize(b.stream) != cudaSuccess) return kFailed;   // pack done
    for (int i = 0; i < ns; i++)
        for (int w = 0; w < 2; w++)
            if (escs::launch_spmm(dp[i], v, b.B, b.Cx[i], b.sx[i], vec, packed) != 0) {
                cudaGetLastError();
                return kFailed;
            }
    constexpr int kBatch = 8;
    for (int rep = 0; rep < 3; rep++) {
        escs::launch_spin(b.stream, 200000);
        cudaEventRecord(b.e0, b.stream);
        for (int i = 0; i < ns; i++) cudaStreamWaitEvent(b.sx[i], b.e0, 0);
        bool ok = true;
        for (int j = 0; j < kBatch; j++)
            for (int i = 0; i < ns; i++)
                ok = ok && escs::launch_spmm(dp[i], v, b.B, b.Cx[i], b.sx[i], vec, packed) == 0;
        for (int i = 0; i < ns; i++) {
            cudaEventRecord(b.ex[i], b.sx[i]);
            cudaStreamWaitEvent(b.stream, b.ex[i], 0);
        }
        cudaEventRecord(b.e1, b.stream);
        if (cudaEventSynchronize(b.e1) != cudaSuccess || !ok) {
            cudaGetLastError();
            return kFailed;
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, b.e0, b.e1);
        best = std::min(best, ms / (kBatch * ns));
    }
    return best;
}

// The paper's scheduler & tuner (§3.5) is profiling-based: here the
// profiling runs at plan time, on the device the plan is bound to, for this
// matrix and bCols.  Coordinate descent: UFi first (the tuner's
// first parameter; for plans of the record walk, where the enumeration's B-row
// reuse pays), then the item size T (with the auto tile width), the tile width
// W, UFk, the bCols coarsening factor and the tile order; every candidate is a
// complete canonical plan, timed by the chosen objective on the walk it will
// run (packed: escs_pack then escs_spmm_packed launches).
// Staged-walk search (escs_params.staged = 2 with autotune, or as the last
// stage of the packed latency search): UFi x tile (warps x panels per warp)
// from the B200 sweeps (profiles/r2_notes.md "staged walk"), column ranges
// automatic (about one co-resident CTA per SM); explicit parameters are not
// searched.  Returns the fastest, or NULL.
// Free a tuner candidate: its launches were synchronised by the timing, so
// its pooled memory goes back to the pool without a device-wide wait.
void free_candidate(escs_plan_t P) {
    if (P && P->pooled && !P->parts[0] && !P->aux) {
        if (P->dmem) cudaFreeAsync(P->dmem, 0);
        P->dmem = nullptr;
        delete P;
        return;
    }
    escs_free(P);
}

escs_plan_t make_plan_staged_tuned(int64_t m, int64_t k, int64_t nnz, const int32_t* rowptr,
                                   const int32_t* colidx, int32_t bCols, escs_params q, TuneBufs* shared) {
    q.autotune = 0;
    q.staged = 2;
    q.T = q.T ? q.T : 1 << 20;   // the canonical items are not used by the staged walk: one per panel
    std::unique_ptr<TuneBufs> own;
    TuneBufs* bufs = shared;
    if (!bufs) {
        own.reset(new TuneBufs(m, k, nnz, bCols, false));
        if (!own->ok) return make_plan_fixed(m, k, nnz, rowptr, colidx, bCols, &q, true);
        bufs = own.get();
    }
    static const int cand[][3] = {{8, 16, 1}, {4, 16, 2}, {6, 8, 1}, {4, 8, 1}, {3, 16, 1}, {2, 16, 1}};
    escs_plan_t best = nullptr;
    float bt = kFailed;
    for (const auto& x : cand) {
        escs_params c = q;
        if (!q.ufi) c.ufi = x[0];
        if (!q.st_warps) c.st_warps = x[1];
        if (!q.st_npw) c.st_npw = x[2];
        bool dup = false;   // explicit parameters collapse candidates
        for (const auto* y = cand; y != &x; y++)
            dup = dup || ((q.ufi ? q.ufi : (*y)[0]) == c.ufi && (q.st_warps ? q.st_warps : (*y)[1]) == c.st_warps &&
                          (q.st_npw ? q.st_npw : (*y)[2]) == c.st_npw);
        if (dup) continue;
        escs_plan_t P = make_plan_fixed(m, k, nnz, rowptr, colidx, bCols, &c, true);
        if (!P) {
            if (tune_debug()) std::fprintf(stderr, "escs tune: staged h%d W%d npw%d: %s\n", c.ufi, c.st_warps, c.st_npw, g_msg.c_str());
            clear_error();
            continue;
        }
        const float t = time_plan(P, *bufs, true);
        if (tune_debug())
            std::fprintf(stderr, "escs tune: staged h%d W%d npw%d ns%d ctas %d coop %d: %.2f us\n", c.ufi, c.st_warps,
                         c.st_npw, P->host.st.nsplit, P->host.st.n_cta, (int)P->dev.st_coop, 1e3f * t);
        if (t < bt) {
            if (best) free_candidate(best);
            best = P;
            bt = t;
        } else {
            free_candidate(P);
        }
    }
    if (best) {
        best->autotuned = true;
        clear_error();
    } else if (!shared) {
        return make_plan_fixed(m, k, nnz, rowptr, colidx, bCols, &q, true);   // reports why
    }
    return best;
}

escs_plan_t make_plan_autotuned(int64_t m, int64_t k, int64_t nnz, const int32_t* rowptr,
                                const int32_t* colidx, int32_t bCols, const escs_params* ep) {
    escs_params q = ep ? *ep : escs_params{};
    const bool concurrent = q.autotune == 2;
    const bool packed = q.packed != 0;
    q.autotune = 0;
    // the staged walk is a candidate of the latency objective (its split
    // combine needs the whole grid resident: not a plan for many streams);
    // staged = 2 searches only staged plans, 0 both walks
    const int want_st = (packed && !concurrent) ? q.staged : 1;
    if (want_st == 2) return make_plan_staged_tuned(m, k, nnz, rowptr, colidx, bCols, q, nullptr);
    q.staged = 1;
    escs_plan_t first = make_plan_fixed(m, k, nnz, rowptr, colidx, bCols, &q, true);
    // Throughput plans launch without programmatic dependent launch: with
    // many streams sharing the SMs, CTAs that start early and wait on the
    // previous grid hold SM slots the other streams' layers could use (suite
    // on 16 streams +2%; profiles/r1_notes.md)
    if (first && concurrent) first->dev.pdl = false;
    if (!first || nnz > 8000000) return first;   // large problems: many waves, heuristic holds
    if (packed && first->dev.variant != 1) return first;   // the record walk needs the vector map
    TuneBufs bufs(m, k, nnz, bCols, concurrent);
    if (!bufs.ok) return first;
    struct Cand {
        escs_plan_t P = nullptr;
        float t = kFailed;
    };
    auto timed = [&](escs_plan_t P) -> float {
        return concurrent ? time_plans_concurrent(P, bufs, packed) : time_plan(P, bufs, packed);
    };
    auto build = [&](escs_params c) -> Cand {
        const auto t0 = std::chrono::steady_clock::now();
        escs_plan_t P = make_plan_fixed(m, k, nnz, rowptr, colidx, bCols, &c, true);
        const auto t1 = std::chrono::steady_clock::now();
        if (!P) {
            clear_error();
            return {};
        }
        if (concurrent) P->dev.pdl = false;
        const float t = timed(P);
        if (tune_debug()) {
            const auto t2 = std::chrono::steady_clock::now();
            g_tune_build_s += std::chrono::duration<double>(t1 - t0).count();
            g_tune_time_s += std::chrono::duration<double>(t2 - t1).count();
            g_tune_cands++;
        }
        return {P, t};
    };
    auto keep = [](Cand& cur, Cand x) {   // cur = the faster of cur and x (the other is freed)
        if (!x.P) return;
        const auto f0 = std::chrono::steady_clock::now();
        if (x.t < cur.t) {
            if (cur.P) free_candidate(cur.P);
            cur = x;
        } else {
            free_candidate(x.P);
        }
        if (tune_debug()) g_dbg_free_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - f0).count();
    };
    // the parameters of a plan as an escs_params candidate base
    auto params_of = [&](escs_plan_t P) {
        escs_params c = q;
        c.ufi = P->params.h;
        c.T = P->params.T;
        c.cta_warps = P->params.cta_warps;
        c.ufk = P->params.ufk;
        c.colf = P->dev.variant == 1 ? P->params.colf : 0;
        return c;
    };
    // Coordinate descent from a start plan at a fixed UFi: the item size T
    // (tile width then follows automatically), the tile width W, UFk, the bCols
    // coarsening factor, the tile order.
    auto refine = [&](Cand cur) -> Cand {
        if (!(ep && ep->T)) {   // stage 1: item size
            const double nP = (double)cur.P->host.header[7];
            const double sp = nP > 0 ? (double)cur.P->host.header[9] / nP : 0.0;
            std::vector<int> cand;
            const int T0 = cur.P->params.T;
            const std::vector<double> fs = packed ? std::vector<double>{0.5, 0.7, 1.4, 2.0}
                                                  : std::vector<double>{0.25, 0.35, 0.5, 0.7, 1.4, 2.0, 3.0, 5.0};
            const std::vector<int> pers = packed ? std::vector<int>{1, 2, 4} : std::vector<int>{1, 2, 3, 4, 6, 8};
            for (double f : fs) cand.push_back(std::max(8, (int)(T0 * f)));
            for (int per : pers)
                if (sp >= 1.0) cand.push_back(std::max(8, (int)std::ceil((sp + 3 * std::sqrt(sp)) / per)));
            std::sort(cand.begin(), cand.end());
            cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
            const escs_params base = params_of(cur.P);
            for (int T : cand) {
                if (T == T0) continue;
                escs_params c = base;
                c.T = T;
                c.cta_warps = (ep && ep->cta_warps) ? ep->cta_warps : 0;   // auto width for the new T
                keep(cur, build(c));
            }
        }
        // stage 2: tile width.  Whole panels are packed per tile, so W sets
        // both the warps per CTA and the tile count; the intermediate widths
        // let a layer land on one full wave of the 148 SMs (2048x512@70% b128:
        // 14 warps -> 147 tiles, 9.4 us vs 10.2 us at 16 warps -> 128 tiles;
        // profiles/r1_notes.md)
        if (!(ep && ep->cta_warps)) {
            const escs_params base = params_of(cur.P);
            for (int W : {4, 6, 8, 10, 12, 14, 16}) {
                if (W == base.cta_warps) continue;
                escs_params c = base;
                c.cta_warps = W;
                keep(cur, build(c));
            }
        }
        if (!(ep && ep->ufk)) {   // stage 3: rows in flight
            const escs_params base = params_of(cur.P);
            for (int U : {2, 4, 8}) {
                if (U == base.ufk || bCols < 32 || (U == 2 && !packed)) continue;
                escs_params c = base;
                c.ufk = U;
                keep(cur, build(c));
            }
        }
        // stage 4: B columns per lane (bCols coarsening of the vector lane map;
        // wider per-lane tiles trade shuffles or broadcasts per gathered row
        // for fewer lanes); the CSR walk has the alternatives at UFi = 1 only
        if (!(ep && ep->colf) && (cur.P->params.h == 1 || packed) && cur.P->dev.variant == 1) {
            const escs_params base = params_of(cur.P);
            for (int F : {4, 8, 16}) {
                if (F == base.colf) continue;
                for (int U : {base.ufk, 4, 2}) {
                    escs_params c = base;
                    c.ufk = U;
                    c.colf = F;
                    if (!escs::kernel_supported(c.ufi, bCols, 1, U, F, packed)) continue;
                    keep(cur, build(c));
                    break;
                }
            }
        }
        if (!(ep && ep->tile_order)) {   // stage 5: tile order
            escs_params c = params_of(cur.P);
            c.tile_order = cur.P->params.tile_order == 2 ? 1 : 2;
            keep(cur, build(c));
            // (column windows, tile_order 3, are not searched: chosen by the hot
            // timing on six 2048x512 layers, they lost on the cold step --
            // profiles/r2_notes.md §11)
        }
        return cur;
    };

    // The packed walk's search (stage 0 + refinement), from a start plan.
    auto packed_search = [&](escs_plan_t start) -> Cand {
        Cand out;
        Cand per_h[9];
        per_h[start->params.h] = {start, timed(start)};
        const double dens = (double)nnz / ((double)m * (double)k);
        const bool fixed_h = ep && ep->ufi;
        for (int h : {1, 2, 3, 4, 6, 8}) {
            if (fixed_h ? h != ep->ufi : (h > 4 && dens < 0.15)) continue;   // UFi 6/8 where p is large
            // the expected B-row reuse of UFi h on a uniformly pruned matrix,
            // p = h d / (1 - (1 - d)^h): below 1.1 a UFi > 1 plan only adds
            // record bytes and predicated FMA slots (never chosen in the B200
            // suite sweeps) -- not searched
            if (!fixed_h && h > 1 && h * dens / (1.0 - std::pow(1.0 - dens, h)) < 1.1) continue;
            const double sp = (double)k * (1.0 - std::pow(1.0 - dens, h));
            const int pw[6][2] = {{1, 0}, {3, 0}, {8, 4}, {8, 16}, {24, 4}, {24, 16}};
            for (const auto& x : pw) {
                if (ep && ep->T && x[0] != 1) continue;
                escs_params c = q;
                c.ufi = h;
                if (!(ep && ep->T)) c.T = std::max(8, (int)std::ceil((sp + 3 * std::sqrt(sp)) / x[0]));
                if (!(ep && ep->cta_warps)) c.cta_warps = x[1];
                keep(per_h[h], build(c));
            }
        }
        int hb = 0;
        for (int h = 1; h <= 8; h++)
            if (per_h[h].P && (!hb || per_h[h].t < per_h[hb].t)) hb = h;
        for (int h = 1; h <= 8; h++)   // keep only the best UFi and UFi = 1
            if (per_h[h].P && h != hb && h != 1) {
                free_candidate(per_h[h].P);
                per_h[h] = {};
            }
        Cand r1 = per_h[1].P ? refine(per_h[1]) : Cand{};
        // the best UFi > 1 is refined only if it is within 10% of the refined
        // UFi-1 plan already (refinement gains are a few percent)
        Cand rb = (hb != 1 && per_h[hb].P && (!r1.P || per_h[hb].t < 1.10f * r1.t)) ? refine(per_h[hb]) : Cand{};
        if (hb != 1 && per_h[hb].P && !rb.P) free_candidate(per_h[hb].P);
        if (rb.P && (!r1.P || rb.t < 0.97f * r1.t)) {
            if (r1.P) free_candidate(r1.P);
            out = rb;
        } else {
            if (rb.P) free_candidate(rb.P);
            out = r1;
        }
        return out;
    };
    Cand best;
    if (!packed) {
        best = refine({first, timed(first)});
    } else {
        best = packed_search(first);
        // A second search for a nearly all-L1 SM (2% carveout: the smallest
        // shared-memory configuration, fewer resident CTAs) where B about fits
        // in L1 (96-320 KB): with a fixed carveout the tuned plans differ in T, W
        // and UFk (2048x512@70% b128: 10.3 -> 9.4 us hot; profiles/r2_notes.md
        // §10); kept at a 2% margin
        const int64_t bbytes = (int64_t)k * bCols * 4;
        if (!concurrent && !(ep && ep->carveout) && bbytes > 96 * 1024 && bbytes <= l1_fit_bytes() &&
            best.P->dev.variant == 1) {
            const escs_params q0 = q;
            q.carveout = 2;
            escs_plan_t first2 = make_plan_fixed(m, k, nnz, rowptr, colidx, bCols, &q, true);
            if (first2) {
                Cand l1 = packed_search(first2);
                if (tune_debug() && l1.P)
                    std::fprintf(stderr, "escs tune: L1 search %.2f us vs %.2f us\n", 1e3f * l1.t, 1e3f * best.t);
                if (l1.P && l1.t < 0.98f * best.t) {
                    free_candidate(best.P);
                    best = l1;
                } else if (l1.P) {
                    free_candidate(l1.P);
                }
            }
            clear_error();
            q = q0;
        }
    }
    if (!concurrent && !(ep && ep->carveout) && !best.P->dev.st_n_cta && best.P->dev.carveout > 0) {
        // L1 against occupancy: the same plan with smaller carveouts (fewer
        // resident CTAs, more L1 for re-read B rows); kept at a 2% margin
        const int cv0 = best.P->dev.carveout;
        int cv_best = cv0;
        float t_best = best.t;
        for (int cv : {0, cv0 / 2}) {
            if (cv >= cv0) continue;
            best.P->dev.carveout = cv;
            const float t = timed(best.P);
            if (tune_debug()) std::fprintf(stderr, "escs tune: carveout %d%%: %.2f us (vs %d%%: %.2f us)\n", cv,
                                           1e3f * t, cv0, 1e3f * best.t);
            if (t < 0.98f * t_best) {
                t_best = t;
                cv_best = cv;
            }
        }
        best.P->dev.carveout = cv_best;
        best.t = t_best;
    }
    if (want_st == 0 && best.P->dev.variant == 1 && (bCols == 32 || bCols == 64 || bCols == 128) &&
        (double)nnz >= 0.15 * (double)m * (double)k && (double)nnz * bCols >= 4.0e7) {
        // the staged walk where its B-row reuse in shared memory can pay:
        // dense enough (<= 85% sparsity) and long enough that its fixed costs
        // (bulk-copy latency before the first stage, the in-kernel combine of
        // the column ranges) are amortised -- on the B200 suite sweeps it wins
        // only above ~40M multiply-adds per call (profiles/r2_notes.md); kept
        // at a 3% margin
        escs_params c = q;
        c.staged = 2;
        escs_plan_t S = make_plan_staged_tuned(m, k, nnz, rowptr, colidx, bCols, c, &bufs);
        if (S) {
            const float ts = time_plan(S, bufs, true);
            if (tune_debug())
                std::fprintf(stderr, "escs tune: best staged %.2f us vs gather walk %.2f us (h%d)\n", 1e3f * ts,
                             1e3f * best.t, best.P->params.h);
            if (ts < 0.97f * best.t) {
                free_candidate(best.P);
                best = {S, ts};
            } else {
                free_candidate(S);
            }
        }
        clear_error();
    }
    // Hybrid candidate: opt-in (ESCS_TUNE_HYBRID=1).  Measured on C4 (power-law
    // 16384^2, profiles/r2_notes.md §6) the hybrid never beat the single plan:
    // the dense rows' part runs fewer, costlier records (UFi 3: 742k records
    // in 33.6 us vs 1.45M UFi-1 records of the short rows in 41 us), 72-74 us
    // in total vs 70 us for one plan.
    const char* eh = std::getenv("ESCS_TUNE_HYBRID");
    const bool try_hybrid = eh && eh[0] == '1';
    if (try_hybrid && packed && !concurrent && (!ep || ep->hybrid_rows == 0) && nnz <= 8000000) {
        // skewed rows (power-law, C4): the longest rows as their own plan, where
        // panels of dense rows give the enumeration a large p, the rest at UFi 1
        double share = 0.0;
        const int64_t X = auto_hybrid_rows(m, nnz, rowptr, &share);
        if (X >= 8 && X <= m / 2 && share >= 0.25) {
            escs_params c = q;
            c.autotune = 1;
            c.staged = 0;
            escs_plan_t Hp = make_plan_hybrid(m, k, nnz, rowptr, colidx, bCols, &c, X);
            if (Hp) {
                const float th = time_plan(Hp, bufs, true);
                if (tune_debug())
                    std::fprintf(stderr, "escs tune: hybrid %lld rows (%.0f%% of nnz) %.2f us vs %.2f us\n",
                                 (long long)X, 100.0 * share, 1e3f * th, 1e3f * best.t);
                if (th < 0.97f * best.t) {
                    free_candidate(best.P);
                    best = {Hp, th};
                } else {
                    free_candidate(Hp);
                }
            }
            clear_error();
        }
    }
    best.P->autotuned = best.P->autotuned ? best.P->autotuned : 1;
    clear_error();
    return best.P;
}

escs_plan_t make_plan(int64_t m, int64_t k, int64_t nnz, const int32_t* rowptr,
                      const int32_t* colidx, int32_t bCols, const escs_params* ep);

// Hybrid plan (escs_params.hybrid_rows = X): part 0 = the X longest rows in
// descending length order (ties by row index), part 1 = the other rows in
// row order, each planned (and, with autotune, tuned) as its own matrix for
// the packed gather walk; part 0 at the requested UFi (else the tuner's, else
// 8), part 1 at UFi 1 unless tuned.  Each part gets a row map (its row -> row
// of C) and a value map (its CSR position -> the caller's CSR position).
escs_plan_t make_plan_hybrid(int64_t m, int64_t k, int64_t nnz, const int32_t* rowptr, const int32_t* colidx,
                             int32_t bCols, const escs_params* ep, int64_t X) {
    if (X < 1 || X >= m) {
        fail(ESCS_ERR_ARG, "hybrid_rows must be in 1..m-1");
        return nullptr;
    }
    std::vector<int64_t> order(m);
    for (int64_t i = 0; i < m; i++) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        return rowptr[a + 1] - rowptr[a] > rowptr[b + 1] - rowptr[b];
    });
    std::vector<int64_t> rows[2];
    rows[0].assign(order.begin(), order.begin() + X);
    rows[1].assign(order.begin() + X, order.end());
    std::sort(rows[1].begin(), rows[1].end());
    const bool tune = ep && ep->autotune;
    escs_plan_impl* H = new (std::nothrow) escs_plan_impl();
    if (!H) {
        fail(ESCS_ERR_OOM, "host allocation");
        return nullptr;
    }
    size_t aux_words = 0;
    std::vector<int32_t> maps[2][2];   // [part][rowmap, vmap]
    for (int q = 0; q < 2; q++) {
        const auto& R = rows[q];
        const int64_t mq = (int64_t)R.size();
        std::vector<int32_t> rp(mq + 1, 0), ci;
        auto& rowmap = maps[q][0];
        auto& vmap = maps[q][1];
        rowmap.resize(mq);
        for (int64_t i = 0; i < mq; i++) {
            const int64_t r = R[i];
            rowmap[i] = (int32_t)r;
            for (int32_t t = rowptr[r]; t < rowptr[r + 1]; t++) {
                ci.push_back(colidx[t]);
                vmap.push_back(t);
            }
            rp[i + 1] = (int32_t)ci.size();
        }
        escs_params c = ep ? *ep : escs_params{};
        c.hybrid_rows = -1;
        c.packed = 1;
        c.staged = 1;   // the gather walk (its epilogue maps rows)
        // an explicit UFi is part 0's; part 1 (the short rows) runs UFi 1 unless tuned
        if (q == 1) c.ufi = tune && !(ep && ep->ufi) ? 0 : 1;
        if (q == 0 && !c.ufi && !tune) c.ufi = 8;
        // dense rows: short items, so that no lane's fp32 running sum spans
        // thousands of terms (C4's full rows: G2 1.5e-4 at the table's T, within
        // 1e-4 at 256)
        if (q == 0 && !c.T && !tune) c.T = 256;
        escs_plan_t P = make_plan(mq, k, (int64_t)ci.size(), rp.data(), ci.empty() ? nullptr : ci.data(), bCols, &c);
        if (!P) {
            escs_free(H);
            return nullptr;
        }
        H->parts[q] = P;
        aux_words += (size_t)mq + vmap.size() + 64;
    }
    void* d = nullptr;
    if (cudaMalloc(&d, std::max<size_t>(aux_words, 1) * 4) != cudaSuccess) {
        cudaGetLastError();
        escs_free(H);
        fail(ESCS_ERR_OOM, "cudaMalloc (hybrid maps)");
        return nullptr;
    }
    H->aux = d;
    int32_t* a = static_cast<int32_t*>(d);
    size_t off = 0;
    for (int q = 0; q < 2; q++) {
        for (int w = 0; w < 2; w++) {
            const auto& v = maps[q][w];
            if (!v.empty() && cudaMemcpy(a + off, v.data(), v.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
                cudaGetLastError();
                escs_free(H);
                fail(ESCS_ERR_CUDA, "cudaMemcpy (hybrid maps)");
                return nullptr;
            }
            (w == 0 ? H->parts[q]->dev.rowmap : H->parts[q]->dev.vmap) = a + off;
            off += (v.size() + 31) / 32 * 32;
        }
        H->part_words[q] = escs::packed_words(H->parts[q]->dev);
    }
    H->host_only = false;
    H->device = H->parts[0]->device;
    H->params = H->parts[0]->params;
    H->hybrid_rows = (int)X;
    H->autotuned = (H->parts[0]->autotuned && H->parts[1]->autotuned) ? 1 : 0;
    int32_t* hd = H->host.header;
    hd[0] = 1; hd[1] = (int32_t)m; hd[2] = (int32_t)k; hd[3] = (int32_t)nnz; hd[4] = bCols;
    hd[5] = H->parts[0]->host.header[5];
    hd[9] = H->parts[0]->host.header[9] + H->parts[1]->host.header[9];
    H->dev = H->parts[0]->dev;   // the launch-facing fields are per part; m / bcols of the whole
    H->dev.m = (int)m;
    H->dev.rowmap = nullptr;
    H->dev.vmap = nullptr;
    return H;
}

// Rows of at least twice the mean length and their share of the nonzeros:
// the automatic hybrid candidate (escs_params.hybrid_rows = 0 with autotune).
int64_t auto_hybrid_rows(int64_t m, int64_t nnz, const int32_t* rowptr, double* share) {
    if (m < 16 || nnz == 0) return 0;
    const double mean = (double)nnz / (double)m;
    int64_t X = 0, hn = 0;
    for (int64_t i = 0; i < m; i++) {
        const int64_t L = rowptr[i + 1] - rowptr[i];
        if ((double)L >= 2.0 * mean) {
            X++;
            hn += L;
        }
    }
    *share = (double)hn / (double)nnz;
    return X;
}

// Tuning cache (the paper tunes per architecture and bCols; here per
// problem class): the parameters the tuner chose for (device, m, k, nnz,
// bCols, requested parameters) are reused for the next matrix of the same
// class -- the same layer shape pruned to the same density -- which is then
// planned with them directly (escs_plan_stats.autotuned = 2).  Process-wide,
// thread-safe; ESCS_TUNE_CACHE=0 disables it.
struct TuneKey {
    int64_t m, k, nnz;
    int32_t bcols, device;
    escs_params q;
    bool operator<(const TuneKey& o) const {
        if (m != o.m) return m < o.m;
        if (k != o.k) return k < o.k;
        if (nnz != o.nnz) return nnz < o.nnz;
        if (bcols != o.bcols) return bcols < o.bcols;
        if (device != o.device) return device < o.device;
        return std::memcmp(&q, &o.q, sizeof(q)) < 0;
    }
};
std::mutex g_tune_mu;
std::map<TuneKey, std::pair<escs_params, bool>> g_tune_cache;   // params, pdl

// ESCS_TUNE_CACHE_FILE=path: the cache persists across processes (tune once,
// e.g. before a profiling run that must replay the same plans).  One line per
// entry: the key's m k nnz bCols device and escs_params words, then the
// chosen escs_params words and the PDL flag.
constexpr int kParamWords = (int)(sizeof(escs_params) / sizeof(int32_t));
const char* tune_cache_file() {
    const char* f = std::getenv("ESCS_TUNE_CACHE_FILE");
    return (f && f[0]) ? f : nullptr;
}
void tune_cache_load_locked() {
    static bool loaded = false;
    if (loaded) return;
    loaded = true;
    const char* path = tune_cache_file();
    if (!path) return;
    FILE* f = std::fopen(path, "r");
    if (!f) return;
    for (;;) {
        long long m, k, nnz;
        int bc, dev, pdl;
        int32_t kq[kParamWords], vq[kParamWords];
        if (std::fscanf(f, "%lld %lld %lld %d %d", &m, &k, &nnz, &bc, &dev) != 5) break;
        bool ok = true;
        for (int i = 0; i < kParamWords && ok; i++) ok = std::fscanf(f, "%d", &kq[i]) == 1;
        for (int i = 0; i < kParamWords && ok; i++) ok = std::fscanf(f, "%d", &vq[i]) == 1;
        if (!ok || std::fscanf(f, "%d", &pdl) != 1) break;
        TuneKey key{m, k, nnz, bc, dev, {}};
        escs_params v{};
        std::memcpy(&key.q, kq, sizeof(escs_params));
        std::memcpy(&v, vq, sizeof(escs_params));
        g_tune_cache[key] = {v, pdl != 0};
    }
    std::fclose(f);
}
void tune_cache_append_locked(const TuneKey& key, const escs_params& v, bool pdl) {
    const char* path = tune_cache_file();
    if (!path) return;
    int32_t kq[kParamWords], vq[kParamWords];
    std::memcpy(kq, &key.q, sizeof(escs_params));
    std::memcpy(vq, &v, sizeof(escs_params));
    // the whole line in one write (O_APPEND-style): processes sharing the file
    // never interleave inside an entry
    std::string line = std::to_string((long long)key.m) + " " + std::to_string((long long)key.k) + " " +
                       std::to_string((long long)key.nnz) + " " + std::to_string(key.bcols) + " " +
                       std::to_string(key.device);
    for (int i = 0; i < kParamWords; i++) line += " " + std::to_string(kq[i]);
    for (int i = 0; i < kParamWords; i++) line += " " + std::to_string(vq[i]);
    line += pdl ? " 1\n" : " 0\n";
    FILE* f = std::fopen(path, "a");
    if (!f) return;
    std::setvbuf(f, nullptr, _IONBF, 0);
    std::fwrite(line.data(), 1, line.size(), f);
    std::fclose(f);
}

escs_plan_t make_plan(int64_t m, int64_t k, int64_t nnz, const int32_t* rowptr,
                      const int32_t* colidx, int32_t bCols, const escs_params* ep) {
    const char* env = std::getenv("ESCS_AUTOTUNE");
    if (ep && (ep->autotune < 0 || ep->autotune > 2)) {
        fail(ESCS_ERR_ARG, "autotune must be 0 (off), 1 (latency) or 2 (concurrent throughput)");
        return nullptr;
    }
    const bool tune = (ep && ep->autotune) || (env && env[0] == '1');
    if (ep && ep->hybrid_rows > 0) {
        if (ep->host_only) {
            fail(ESCS_ERR_UNSUPPORTED, "hybrid plans are device plans");
            return nullptr;
        }
        if (!ep->packed) {
            fail(ESCS_ERR_UNSUPPORTED, "hybrid plans run the packed walk (escs_params.packed = 1)");
            return nullptr;
        }
        clear_error();
        std::string v = escs::validate_csr(m, k, nnz, rowptr, colidx);
        if (!v.empty()) {
            fail(ESCS_ERR_CSR, "invalid CSR: " + v);
            return nullptr;
        }
        escs_params c = *ep;
        if (tune) c.autotune = c.autotune ? c.autotune : 1;
        return make_plan_hybrid(m, k, nnz, rowptr, colidx, bCols, &c, ep->hybrid_rows);
    }
    if (ep && ep->hybrid_rows < -1) {
        fail(ESCS_ERR_ARG, "hybrid_rows must be -1, 0 or a row count");
        return nullptr;
    }
    if (!tune || (ep && ep->host_only)) return make_plan_fixed(m, k, nnz, rowptr, colidx, bCols, ep);
    const char* ce = std::getenv("ESCS_TUNE_CACHE");
    const bool use_cache = !(ce && ce[0] == '0');
    TuneKey key{m, k, nnz, bCols, -1, ep ? *ep : escs_params{}};
    key.q.nthreads = 0;
    if (!key.q.autotune) key.q.autotune = 1;
    cudaGetDevice(&key.device);
    if (use_cache) {
        std::pair<escs_params, bool> hit;
        bool found = false;
        {
            std::lock_guard<std::mutex> lk(g_tune_mu);
            tune_cache_load_locked();
            auto it = g_tune_cache.find(key);
            if (it != g_tune_cache.end()) {
                hit = it->second;
                found = true;
            }
        }
        if (found) {
            escs_params c = hit.first;
            c.nthreads = ep ? ep->nthreads : 0;
            escs_plan_t P = make_plan_fixed(m, k, nnz, rowptr, colidx, bCols, &c);
            if (P) {
                P->dev.pdl = hit.second;
                P->autotuned = 2;
                return P;
            }
            clear_error();   // fall through: tune this matrix
        }
    }
    escs_plan_t P = make_plan_autotuned(m, k, nnz, rowptr, colidx, bCols, ep);
    if (P && use_cache && P->autotuned) {
        escs_params c = key.q;
        c.autotune = 0;
        c.ufi = P->params.h;
        c.T = P->params.T;
        c.cta_warps = P->params.cta_warps;
        c.variant = P->params.variant;
        c.ufk = P->params.ufk;
        c.colf = P->dev.variant == 1 ? P->params.colf : 0;
        c.tile_order = P->params.tile_order;
        c.packed = P->params.packed;
        c.carveout = P->dev.carveout < 0 ? -1 : (P->dev.carveout == 0 ? -2 : P->dev.carveout);
        if (P->host.st.n_cta) {
            c.staged = 2;
            c.st_warps = P->host.st.warps;
            c.st_npw = P->host.st.npw;
            c.st_nsplit = P->host.st.nsplit;
            c.st_kb = P->host.st.kb;
        } else if (c.packed) {
            c.staged = 1;
        }
        std::lock_guard<std::mutex> lk(g_tune_mu);
        tune_cache_load_locked();
        g_tune_cache[key] = {c, P->dev.pdl};
        tune_cache_append_locked(key, c, P->dev.pdl);
    }
    return P;
}

}  // namespace

extern "C" {

escs_plan_t escs_plan(int64_t m, int64_t k, int64_t nnz, const int32_t* rowptr,
                      const int32_t* colidx, int32_t bCols) {
    return make_plan(m, k, nnz, rowptr, colidx, bCols, nullptr);
}

escs_plan_t escs_plan_ex(int64_t m, int64_t k, int64_t nnz, const int32_t* rowptr,
                         const int32_t* colidx, int32_t bCols, const escs_params* p) {
    return make_plan(m, k, nnz, rowptr, colidx, bCols, p);
}

static int spmm_common(escs_plan_t plan, const float* vals, const float* B, float* C,
                       void* stream, bool packed) {
    clear_error();
    if (!plan) return fail(ESCS_ERR_ARG, "plan is NULL");
    if (plan->host_only) return fail(ESCS_ERR_ARG, "plan is host-only (escs_params.host_only=1)");
    if (!B || !C || (!vals && plan->host.header[3] > 0))
        return fail(ESCS_ERR_ARG, "vals, B and C must be non-NULL device pointers");
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess || dev != plan->device)
        return fail(ESCS_ERR_ARG, "current device " + std::to_string(dev) +
                                      " differs from the plan's device " +
                                      std::to_string(plan->device));
    const bool vec_ok = aligned16(B) && aligned16(C);
    if (plan->parts[0]) {   // hybrid: its parts in order
        if (!packed)
            return fail(ESCS_ERR_UNSUPPORTED, "a hybrid plan runs only through escs_pack + escs_spmm_packed");
        if (!vec_ok) return fail(ESCS_ERR_UNSUPPORTED, "escs_spmm_packed needs 16-byte aligned B and C");
        if (vals && !aligned16(vals)) return fail(ESCS_ERR_ARG, "the packed record stream must be 16-byte aligned");
        const int e = launch_packed_plan(plan, vals, B, C, stream, true);
        if (e) return fail(ESCS_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString((cudaError_t)e));
        return ESCS_OK;
    }
    if (!packed && plan->dev.h > 4)
        return fail(ESCS_ERR_UNSUPPORTED, "the CSR-value walk (escs_spmm) is built for UFi <= 4; "
                                          "run this plan through escs_pack + escs_spmm_packed");
    if (packed && !(vec_ok && plan->dev.variant == 1))
        return fail(ESCS_ERR_UNSUPPORTED, "escs_spmm_packed needs 16-byte aligned B and C and a "
                                          "vector-kernel plan (bCols in {4,8,16,32,64,128,256})");
    if (packed && vals && !aligned16(vals))
        return fail(ESCS_ERR_ARG, "the packed record stream must be 16-byte aligned");
    int e = (packed && plan->dev.st_n_cta) ? escs::launch_staged(plan->dev, vals, B, C, stream)
                                           : escs::launch_spmm(plan->dev, vals, B, C, stream, vec_ok, packed);
    if (e) return fail(ESCS_ERR_CUDA, std::string("kernel launch: ") +
                                          cudaGetErrorString((cudaError_t)e));
    return ESCS_OK;
}

int escs_spmm(escs_plan_t plan, const float* vals, const float* B, float* C, void* stream) {
    return spmm_common(plan, vals, B, C, stream, false);
}

int escs_spmm_group(int32_t n, const escs_plan_t* plans, const float* const* vals,
                    const float* const* B, float* const* C, void* stream) {
    clear_error();
    if (n < 0) return fail(ESCS_ERR_ARG, "n must be >= 0");
    if (n == 0) return ESCS_OK;
    if (!plans || !vals || !B || !C) return fail(ESCS_ERR_ARG, "NULL pointer array");
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(ESCS_ERR_CUDA, "cudaGetDevice failed");
    std::vector<const escs::DevPlan*> dps(n);
    for (int i = 0; i < n; i++) {
        const escs_plan_t P = plans[i];
        const std::string at = " (problem " + std::to_string(i) + ")";
        if (!P || P->host_only) return fail(ESCS_ERR_ARG, "plan is NULL or host-only" + at);
        if (P->device != dev)
            return fail(ESCS_ERR_ARG, "current device differs from the plan's device" + at);
        if (!B[i] || !C[i] || (!vals[i] && P->host.header[3] > 0))
            return fail(ESCS_ERR_ARG, "vals, B and C must be non-NULL device pointers" + at);
        if (P->parts[0]) return fail(ESCS_ERR_UNSUPPORTED, "hybrid plans are not grouped" + at);
        for (int j = 0; j < i; j++)
            if (plans[j] == P)
                return fail(ESCS_ERR_ARG, "a plan appears twice in one group (shared workspace)" + at);
        dps[i] = &P->dev;
    }
    int e = escs::launch_group(n, dps.data(), vals, B, C, stream);
    if (e) return fail(ESCS_ERR_CUDA, std::string("kernel launch: ") +
                                          cudaGetErrorString((cudaError_t)e));
    return ESCS_OK;
}

int escs_spmm_scatter(escs_plan_t plan, const float* vals, const float* B, float* const* dsts,
                      int32_t n_dst, int64_t row_offset, uint32_t flags, void* stream) {
    clear_error();
    if (!plan || plan->host_only) return fail(ESCS_ERR_ARG, "plan is NULL or host-only");
    if (plan->parts[0]) return fail(ESCS_ERR_UNSUPPORTED, "escs_spmm_scatter does not take hybrid plans");
    if (!dsts || n_dst < 1 || n_dst > 8)
        return fail(ESCS_ERR_ARG, "escs_spmm_scatter needs 1..8 destination buffers");
    if (!B || (!vals && plan->host.header[3] > 0))
        return fail(ESCS_ERR_ARG, "vals and B must be non-NULL device pointers");
    if (row_offset < 0) return fail(ESCS_ERR_ARG, "row_offset must be >= 0");
    if (flags & ~(uint32_t)ESCS_SCATTER_MULTICAST) return fail(ESCS_ERR_ARG, "unknown flags");
    const bool mc = flags & ESCS_SCATTER_MULTICAST;
    if (mc && n_dst != 1)
        return fail(ESCS_ERR_ARG, "ESCS_SCATTER_MULTICAST takes exactly one (multicast) address");
    bool vec_ok = aligned16(B);
    for (int d = 0; d < n_dst; d++) {
        if (!dsts[d]) return fail(ESCS_ERR_ARG, "NULL destination buffer");
        vec_ok = vec_ok && aligned16(dsts[d]);
    }
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess || dev != plan->device)
        return fail(ESCS_ERR_ARG, "current device differs from the plan's device");
    int e = escs::launch_spmm(plan->dev, vals, B, nullptr, stream, vec_ok, false, dsts, n_dst,
                              (long long)row_offset, mc);
    if (e) return fail(ESCS_ERR_CUDA, std::string("kernel launch: ") +
                                          cudaGetErrorString((cudaError_t)e));
    return ESCS_OK;
}

int escs_spmm_packed(escs_plan_t plan, const float* packed, const float* B, float* C,
                     void* stream) {
    return spmm_common(plan, packed, B, C, stream, true);
}

int escs_pack(escs_plan_t plan, const float* vals, float* packed, void* stream) {
    clear_error();
    if (!plan || plan->host_only) return fail(ESCS_ERR_ARG, "plan is NULL or host-only");
    if (plan->host.header[9] > 0 && (!vals || !packed))
        return fail(ESCS_ERR_ARG, "vals and packed must be non-NULL device pointers");
    if (vals == packed && plan->host.header[9] > 0)
        return fail(ESCS_ERR_ARG, "packed must not alias vals");
    if (packed && !aligned16(packed)) return fail(ESCS_ERR_ARG, "packed must be 16-byte aligned");
    int e = pack_plan(plan, vals, packed, stream);
    if (e) return fail(ESCS_ERR_CUDA, std::string("pack launch: ") +
                                          cudaGetErrorString((cudaError_t)e));
    // synchronous: the record stream is complete when escs_pack returns, so
    // escs_spmm_packed may read it before its programmatic-dependent-launch
    // wait (like the plan arrays)
    cudaError_t se = cudaStreamSynchronize((cudaStream_t)stream);
    if (se != cudaSuccess) return fail(ESCS_ERR_CUDA, std::string("pack: ") + cudaGetErrorString(se));
    return ESCS_OK;
}

int escs_gather_probe(escs_plan_t plan, const float* B, float* sink, void* stream) {
    clear_error();
    if (!plan || plan->host_only || !B || !sink) return fail(ESCS_ERR_ARG, "bad probe arguments");
    if (plan->parts[0]) return fail(ESCS_ERR_UNSUPPORTED, "no gather probe for hybrid plans");
    const bool vec_ok = aligned16(B);
    int e = escs::launch_probe(plan->dev, B, sink, stream, vec_ok);
    if (e) return fail(ESCS_ERR_UNSUPPORTED, std::string("probe: ") +
                                                 cudaGetErrorString((cudaError_t)e));
    return ESCS_OK;
}

int escs_gather_probe_packed(escs_plan_t plan, const float* packed, const float* B, float* sink,
                             void* stream) {
    clear_error();
    if (!plan || plan->host_only || !B || !sink || (!packed && plan->host.header[9] > 0))
        return fail(ESCS_ERR_ARG, "bad probe arguments");
    if (plan->parts[0]) return fail(ESCS_ERR_UNSUPPORTED, "no gather probe for hybrid plans");
    if (plan->dev.st_n_cta) {   // the staged walk's probe (sink: st_ctas x st_warps x 32 floats)
        int e = escs::launch_staged(plan->dev, packed, B, sink, stream, true);
        if (e) return fail(ESCS_ERR_UNSUPPORTED, std::string("probe: ") + cudaGetErrorString((cudaError_t)e));
        return ESCS_OK;
    }
    static const float dummy[4] = {0.f, 0.f, 0.f, 0.f};
    const float* rec = packed ? packed : dummy;   // G = 0: no record is read
    int e = escs::launch_probe(plan->dev, B, sink, stream, aligned16(B), rec);
    if (e) return fail(ESCS_ERR_UNSUPPORTED, std::string("probe: ") +
                                                 cudaGetErrorString((cudaError_t)e));
    return ESCS_OK;
}

void escs_free(escs_plan_t plan) {
    if (!plan) return;
    for (auto* q : plan->parts)
        if (q) escs_free(q);
    if (plan->aux) cudaFree(plan->aux);
    if (plan->dmem) {
        if (plan->pooled) {
            // the caller's streams may be non-blocking: wait for the device as
            // cudaFree would, then return the memory to the planner's pool
            cudaDeviceSynchronize();
            cudaFreeAsync(plan->dmem, 0);
        } else {
            cudaFree(plan->dmem);
        }
    }
    delete plan;
}

int escs_last_error(const char** msg) {
    if (msg) *msg = g_msg.c_str();
    return g_code;
}

int escs_plan_export(escs_plan_t plan, escs_plan_view* out) {
    clear_error();
    if (!plan || !out) return fail(ESCS_ERR_ARG, "NULL argument");
    if (plan->parts[0]) return fail(ESCS_ERR_ARG, "a hybrid plan: export its parts (escs_plan_part)");
    const auto& h = plan->host;
    std::memcpy(out->header, h.header, sizeof(out->header));
    out->grp_panel = h.grp_panel.data();
    out->grp_mask = h.grp_mask.data();
    out->grp_col_ptr = h.grp_col_ptr.data();
    out->grp_val_ptr = h.grp_val_ptr.data();
    out->gcol = h.gcol.data();
    out->slot_src = h.slot_src.data();
    out->item_panel = h.item_panel.data();
    out->item_group_begin = h.item_group_begin.data();
    out->item_gcol_ptr = h.item_gcol_ptr.data();
    return ESCS_OK;
}

int escs_plan_info(escs_plan_t plan, escs_plan_stats* o) {
    clear_error();
    if (!plan || !o) return fail(ESCS_ERR_ARG, "NULL argument");
    if (plan->parts[0]) {   // a hybrid plan: part 0's facts, totals where noted (include/escs.h)
        escs_plan_stats b;
        int e = escs_plan_info(plan->parts[1], &b);
        if (!e) e = escs_plan_info(plan->parts[0], o);
        if (e) return e;
        o->nnz += b.nnz;
        o->G += b.G;
        o->device_bytes += b.device_bytes;
        o->packed_words = plan->part_words[0] + plan->part_words[1];
        o->hybrid_rows = plan->hybrid_rows;
        o->autotuned = plan->autotuned;
        return ESCS_OK;
    }
    const auto& h = plan->host;
    std::memset(o, 0, sizeof(*o));
    o->h = plan->params.h;
    o->T = plan->params.T;
    o->bcols = h.header[4];
    o->variant = plan->params.variant;
    o->cta_warps = plan->params.cta_warps;
    o->ufk = plan->params.ufk;
    o->n_tiles = h.n_tiles;
    o->n_heavy = h.n_heavy;
    o->n_split_items = h.n_split_items;
    o->device = plan->device;
    o->nP = h.header[7];
    o->NG = h.header[8];
    o->G = h.header[9];
    o->n_items = h.header[10];
    o->nnz = h.header[3];
    o->device_bytes = (int64_t)plan->dbytes;
    o->workspace_bytes = (int64_t)plan->ws_bytes;
    o->plan_seconds = h.plan_seconds;
    o->packed = plan->params.packed;
    o->ctas_per_sm = plan->host_only ? 0 : escs::blocks_per_sm(plan->dev, plan->dev.variant == 1, false,
                                                               o->packed != 0);
    o->autotuned = plan->autotuned;
    o->colf = plan->dev.variant == 1 ? plan->params.colf : 0;
    o->tile_order = plan->params.tile_order;
    o->pdl = plan->dev.pdl ? 1 : 0;
    o->carveout = plan->dev.carveout;
    {
        escs::DevPlan d = plan->dev;   // host-only plans: the same formula from the header
        d.h = h.header[5];
        d.G = h.header[9];
        d.st_n_cta = h.st.n_cta;
        d.st_n_rec = (int)h.st.src.size();
        o->packed_words = escs::packed_words(d);
    }
    if (h.st.n_cta) {
        o->staged = 1;
        o->st_ctas = h.st.n_cta;
        o->st_warps = h.st.warps;
        o->st_npw = h.st.npw;
        o->st_nsplit = h.st.nsplit;
        o->st_kb = h.st.kb;
        o->st_smem_bytes = (int32_t)(plan->host_only ? 0 : escs::staged_smem_bytes(plan->dev));
        o->st_launches = (h.st.nsplit > 1 && !plan->dev.st_coop) ? 2 : 1;
    }
    return ESCS_OK;
}

int escs_staged_export(escs_plan_t plan, escs_staged_view* out) {
    clear_error();
    if (!plan || !out) return fail(ESCS_ERR_ARG, "NULL argument");
    const auto& st = plan->host.st;
    if (!st.n_cta) return fail(ESCS_ERR_ARG, "plan has no staged schedule (escs_params.staged = 2)");
    out->n_cta = st.n_cta;
    out->n_stage = (int32_t)(st.stage.size() / 4);
    out->n_rec = (int32_t)st.src.size();
    out->hs = st.hs;
    out->nslot = st.nslot;
    out->max_k = st.max_k;
    out->max_rec = st.max_rec;
    out->max_stages = st.max_stages;
    out->cta = st.cta.data();
    out->stage = st.stage.data();
    out->hdr = st.hdr.data();
    out->src = st.src.data();
    return ESCS_OK;
}

escs_plan_t escs_plan_part(escs_plan_t plan, int32_t i) {
    clear_error();
    if (!plan || i < 0 || i > 1 || !plan->parts[0]) {
        fail(ESCS_ERR_ARG, "not a hybrid plan, or part index not 0/1");
        return nullptr;
    }
    return plan->parts[i];
}

const char* escs_version(void) { return "escs 0.1 sm_100a"; }

}  // extern "C"
