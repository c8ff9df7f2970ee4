// plan.cpp -- host enumeration planner (§3.2 Enumeration) and the
// data transformation of §3.3.3, built from CSR in O(nnz * UFi)
// by an UFi-way merge of each panel's sorted rows.  The paper's own
// dataTransformer scans dense A in O(M*K); that form is the
// oracle's (oracle/escs_oracle.c) and shares no code with this file.  The two
// must agree byte for byte (tests/test_plan_parity.py).
//
// Canonical plan (P1-P8):
//   panel P = rows [P*h, min(m,(P+1)*h))                      (R2)
//   gcol    = (panel, column) with >= 1 nonzero, pattern = UFi-bit row mask
//   groups  = (panel, mask) ordered by panel then mask ascending   (R3, Fig. 4)
//   slots   = column-major over a group's columns, pattern rows ascending
//             (Listing 7's t_nnz cursor, Reading R1)
//   items   = panel stream cut into n_P = max(1, ceil(S_P/T)) even pieces (R7)
#include <algorithm>
#include <atomic>
#include <cmath>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <thread>

#include "escs_internal.h"

namespace escs {

std::string validate_csr(int64_t m, int64_t k, int64_t nnz, const int32_t* rowptr,
                         const int32_t* colidx) {
    if (!rowptr) return "rowptr is NULL";
    if (nnz > 0 && !colidx) return "colidx is NULL";
    if (rowptr[0] != 0) return "rowptr[0] != 0";
    if ((int64_t)rowptr[m] != nnz) return "rowptr[m] != nnz";
    for (int64_t i = 0; i < m; i++) {
        int64_t a = rowptr[i], b = rowptr[i + 1];
        if (b < a) return "rowptr decreases at row " + std::to_string(i);
        if (b > nnz) return "rowptr exceeds nnz at row " + std::to_string(i);
        for (int64_t t = a; t < b; t++) {
            int32_t c = colidx[t];
            if (c < 0 || c >= k)
                return "column index out of range at row " + std::to_string(i) + " position " +
                       std::to_string(t);
            if (t > a && c <= colidx[t - 1])
                return "column indices not strictly increasing at row " + std::to_string(i) +
                       " position " + std::to_string(t);
        }
    }
    return "";
}

namespace {

// One chunk of consecutive panels, planned independently then concatenated.
struct Chunk {
    int64_t p0 = 0, p1 = 0;
    std::vector<int32_t> grp_panel, grp_mask, grp_w, grp_vw;   // widths, value widths
    std::vector<int32_t> gcol, slot;
    std::vector<int32_t> item_panel, item_gb_local, item_s1_local;
};

void plan_chunk(const int32_t* rowptr, const int32_t* colidx, int64_t m, int h, int T,
                Chunk& ch) {
    const int nmask = 1 << h;
    std::vector<int32_t> cur(h), end(h);
    std::vector<int32_t> e_col, e_mask, e_pos;   // merged entries and their CSR positions
    std::vector<int32_t> e_off;
    std::vector<int64_t> cnt(nmask), gstart(nmask), vstart(nmask), gslot(nmask);
    std::vector<int32_t> gidx(nmask);

    for (int64_t P = ch.p0; P < ch.p1; P++) {
        const int64_t r0 = P * h;
        const int rows = (int)std::min<int64_t>(h, m - r0);
        for (int r = 0; r < h; r++) {
            if (r < rows) {
                cur[r] = rowptr[r0 + r];
                end[r] = rowptr[r0 + r + 1];
            } else {
                cur[r] = end[r] = 0;
            }
        }
        e_col.clear(); e_mask.clear(); e_pos.clear(); e_off.clear();
        // UFi-way merge: smallest pending column across the panel's rows.
        for (;;) {
            int32_t c = INT32_MAX;
            for (int r = 0; r < rows; r++)
                if (cur[r] < end[r] && colidx[cur[r]] < c) c = colidx[cur[r]];
            if (c == INT32_MAX) break;
            int32_t mask = 0;
            e_off.push_back((int32_t)e_pos.size());
            for (int r = 0; r < rows; r++)
                if (cur[r] < end[r] && colidx[cur[r]] == c) {
                    mask |= 1 << r;
                    e_pos.push_back(cur[r]++);   // ranks ascend with r
                }
            e_col.push_back(c);
            e_mask.push_back(mask);
        }
        const int64_t ne = (int64_t)e_col.size();
        // stable counting sort of entries by mask -> groups
        std::fill(cnt.begin(), cnt.end(), 0);
        for (int64_t e = 0; e < ne; e++) cnt[e_mask[e]]++;
        const int64_t g_first = (int64_t)ch.grp_panel.size();
        const int64_t col_base = (int64_t)ch.gcol.size();
        const int64_t val_base = (int64_t)ch.slot.size();
        int64_t s = 0, v = 0;
        for (int mu = 1; mu < nmask; mu++) {
            if (!cnt[mu]) continue;
            const int p = __builtin_popcount((unsigned)mu);
            gidx[mu] = (int32_t)ch.grp_panel.size();
            gstart[mu] = s;
            vstart[mu] = v;
            gslot[mu] = 0;
            ch.grp_panel.push_back((int32_t)P);
            ch.grp_mask.push_back(mu);
            ch.grp_w.push_back((int32_t)cnt[mu]);
            ch.grp_vw.push_back((int32_t)(cnt[mu] * p));
            s += cnt[mu];
            v += cnt[mu] * p;
        }
        ch.gcol.resize(col_base + s);
        ch.slot.resize(val_base + v);
        for (int64_t e = 0; e < ne; e++) {
            const int mu = e_mask[e];
            const int p = __builtin_popcount((unsigned)mu);
            const int64_t ci = gslot[mu]++;
            ch.gcol[col_base + gstart[mu] + ci] = e_col[e];
            int32_t* dst = &ch.slot[val_base + vstart[mu] + ci * p];
            for (int j = 0; j < p; j++) dst[j] = e_pos[e_off[e] + j];
        }
        // balanced items over the panel stream of length s
        const int64_t SP = s;
        int64_t n = (SP + T - 1) / T;
        if (n < 1) n = 1;
        const int64_t ng = (int64_t)ch.grp_panel.size() - g_first;
        int64_t gb = 0;   // monotone pointer: last group with stream start <= s0
        for (int64_t q = 0; q < n; q++) {
            const int64_t s0 = (q * SP) / n, s1 = ((q + 1) * SP) / n;
            while (gb + 1 < ng && gstart[ch.grp_mask[g_first + gb + 1]] <= s0) gb++;
            ch.item_panel.push_back((int32_t)P);
            ch.item_gb_local.push_back((int32_t)(g_first + gb));
            ch.item_s1_local.push_back((int32_t)(col_base + s1));
        }
    }
}

}  // namespace

void build_plan(int64_t m, int64_t k, int64_t nnz, const int32_t* rowptr, const int32_t* colidx,
                int32_t bcols, const Params& p, PlanHost& out) {
    auto t0 = std::chrono::steady_clock::now();
    const int h = p.h, T = p.T;
    if (h < 1 || h > 16) throw std::runtime_error("ufi must be in 1..16");
    if (T < 1) throw std::runtime_error("T must be >= 1");
    const int64_t nP = (m + h - 1) / h;

    // chunks of consecutive panels balanced by nnz
    int nth = p.nthreads > 0 ? p.nthreads : (int)std::max(1u, std::thread::hardware_concurrency());
    if (nnz < 200000) nth = 1;
    const int64_t nchunks = std::min<int64_t>(nP, (int64_t)nth * 8);
    std::vector<Chunk> chunks(nchunks);
    {
        int64_t P = 0;
        for (int64_t c = 0; c < nchunks; c++) {
            const int64_t target = (nnz * (c + 1)) / nchunks;
            int64_t P1 = P + 1;
            if (c == nchunks - 1) {
                P1 = nP;
            } else {
                // advance until the chunk's cumulative nnz reaches target, leaving
                // at least one panel for each remaining chunk
                while (P1 < nP - (nchunks - 1 - c) &&
                       rowptr[std::min<int64_t>(m, P1 * h)] < target)
                    P1++;
            }
            chunks[c].p0 = P;
            chunks[c].p1 = P1;
            P = P1;
        }
    }
    if (nth <= 1 || nchunks <= 1) {
        for (auto& ch : chunks) plan_chunk(rowptr, colidx, m, h, T, ch);
    } else {
        std::vector<std::thread> th;
        std::atomic<int64_t> next{0};
        for (int t = 0; t < nth; t++)
            th.emplace_back([&] {
                for (;;) {
                    int64_t c = next.fetch_add(1);
                    if (c >= nchunks) break;
                    plan_chunk(rowptr, colidx, m, h, T, chunks[c]);
                }
            });
        for (auto& x : th) x.join();
    }

    // deterministic concatenation in panel order
    int64_t NG = 0, G = 0, V = 0, NI = 0;
    for (auto& ch : chunks) {
        NG += ch.grp_panel.size();
        G += ch.gcol.size();
        V += ch.slot.size();
        NI += ch.item_panel.size();
    }
    if (V != nnz) throw std::runtime_error("internal: slot count != nnz");
    if (NG >= INT32_MAX || G >= INT32_MAX || NI >= INT32_MAX)
        throw std::runtime_error("plan too large for int32 indices");
    out.grp_panel.resize(NG); out.grp_mask.resize(NG);
    out.grp_col_ptr.resize(NG + 1); out.grp_val_ptr.resize(NG + 1);
    out.gcol.resize(G); out.slot_src.resize(nnz);
    out.item_panel.resize(NI); out.item_group_begin.resize(NI); out.item_gcol_ptr.resize(NI + 1);
    out.grp_col_ptr[0] = 0; out.grp_val_ptr[0] = 0; out.item_gcol_ptr[0] = 0;
    int64_t og = 0, oc = 0, ov = 0, oi = 0;
    for (auto& ch : chunks) {
        const int64_t ng = ch.grp_panel.size();
        for (int64_t g = 0; g < ng; g++) {
            out.grp_panel[og + g] = ch.grp_panel[g];
            out.grp_mask[og + g] = ch.grp_mask[g];
            out.grp_col_ptr[og + g + 1] = out.grp_col_ptr[og + g] + ch.grp_w[g];
            out.grp_val_ptr[og + g + 1] = out.grp_val_ptr[og + g] + ch.grp_vw[g];
        }
        if (!ch.gcol.empty()) std::memcpy(&out.gcol[oc], ch.gcol.data(), ch.gcol.size() * 4);
        if (!ch.slot.empty()) std::memcpy(&out.slot_src[ov], ch.slot.data(), ch.slot.size() * 4);
        const int64_t ni = ch.item_panel.size();
        for (int64_t i = 0; i < ni; i++) {
            out.item_panel[oi + i] = ch.item_panel[i];
            out.item_group_begin[oi + i] = (int32_t)(og + ch.item_gb_local[i]);
            out.item_gcol_ptr[oi + i + 1] = (int32_t)(oc + ch.item_s1_local[i]);
        }
        og += ng; oc += ch.gcol.size(); ov += ch.slot.size(); oi += ni;
    }
    int32_t* hd = out.header;
    hd[0] = 1; hd[1] = (int32_t)m; hd[2] = (int32_t)k; hd[3] = (int32_t)nnz; hd[4] = bcols;
    hd[5] = h; hd[6] = T; hd[7] = (int32_t)nP; hd[8] = (int32_t)NG; hd[9] = (int32_t)G;
    hd[10] = (int32_t)NI;
    out.plan_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// CTA tiles: whole panels are packed greedily (in panel order) into tiles of
// W item slots, so that a panel split into several items is combined in
// shared memory by one CTA.  A panel with more than W items ("heavy", the
// power-law case C4) gets ceil(n/W) exclusive tiles that are combined through
// a global workspace in tile order (deterministic fixup).
void build_tiles(PlanHost& ph, int W, bool by_length) {
    const int64_t NI = ph.item_panel.size();
    const int64_t nP = ph.header[7];
    ph.slot_item.clear();
    ph.slot_aux.clear();
    ph.tile_heavy.clear();
    ph.heavy_info.clear();
    ph.n_heavy = ph.n_heavy_tiles = ph.n_split_items = 0;
    ph.any_sync = false;
    std::vector<int32_t> lc(NI, 0);      // lead | cnt << 8 per item
    auto emit = [&](const std::vector<int64_t>& its, bool sync, int hid, int q) {
        for (int k = 0; k < W; k++) {
            if (k < (int)its.size()) {
                ph.slot_item.push_back((int32_t)its[k]);
                ph.slot_aux.push_back(lc[its[k]] | (1 << 16) | (sync ? 1 << 17 : 0) |
                                      (hid >= 0 ? 1 << 18 : 0));
            } else {
                // empty slot: inactive; in a heavy tile it still carries the
                // tile's heavy flag and item count (all warps of a heavy tile
                // take part in its combine, esc_kernel.cuh heavy_combine)
                ph.slot_item.push_back(-1);
                ph.slot_aux.push_back((sync ? 1 << 17 : 0) |
                                      (hid >= 0 ? (1 << 18) | ((int32_t)its.size() << 8) : 0));
            }
        }
        ph.tile_heavy.push_back(hid);
        ph.tile_heavy.push_back(q);
        ph.any_sync |= sync;
    };
    // panels' item ranges (items are ordered by panel)
    std::vector<int64_t> first(nP + 1, NI);
    for (int64_t i = NI - 1; i >= 0; i--) first[ph.item_panel[i]] = i;
    first[nP] = NI;
    for (int64_t P = nP - 1; P >= 0; P--)
        if (first[P] > first[P + 1]) first[P] = first[P + 1];
    // heavy panels (more items than warps): their own tiles, combined through
    // the workspace; emitted first -- they are the longest chains
    std::vector<int64_t> light;
    light.reserve(nP);
    for (int64_t P = 0; P < nP; P++) {
        const int64_t a = first[P], n = first[P + 1] - a;
        if (n > 1) ph.n_split_items += (int32_t)n;
        if (n <= W) {
            light.push_back(P);
            continue;
        }
        const int64_t nt = (n + W - 1) / W;
        const int hid = ph.n_heavy++;
        ph.heavy_info.insert(ph.heavy_info.end(), {(int32_t)P, ph.n_heavy_tiles, (int32_t)nt, 0});
        for (int64_t q = 0; q < nt; q++) {
            const int64_t b0 = a + (q * n) / nt, b1 = a + ((q + 1) * n) / nt;
            std::vector<int64_t> its;
            for (int64_t j = b0; j < b1; j++) {
                lc[j] = 0 | ((int32_t)(b1 - b0) << 8);
                its.push_back(j);
            }
            emit(its, true, hid, (int)q);
        }
        ph.n_heavy_tiles += (int32_t)nt;
    }
    // light panels: whole panels packed W item slots per tile.  With
    // by_length, panels are ordered by their longest item (descending, ties by
    // panel) so that a tile's warps carry similar work -- a CTA holds its SM
    // slot until its longest warp finishes -- and long tiles start first.
    if (by_length) {
        std::vector<int32_t> len(nP, 0);
        for (int64_t P : light)
            for (int64_t j = first[P]; j < first[P + 1]; j++)
                len[P] = std::max(len[P], ph.item_gcol_ptr[j + 1] - ph.item_gcol_ptr[j]);
        std::stable_sort(light.begin(), light.end(),
                         [&](int64_t x, int64_t y) { return len[x] > len[y]; });
    }
    std::vector<int64_t> cur;
    bool cur_sync = false;
    for (int64_t P : light) {
        const int64_t a = first[P], n = first[P + 1] - a;
        if ((int64_t)cur.size() + n > W) {
            emit(cur, cur_sync, -1, 0);
            cur.clear();
            cur_sync = false;
        }
        const int32_t lead = (int32_t)cur.size();
        for (int64_t j = a; j < a + n; j++) {
            lc[j] = lead | ((int32_t)n << 8);
            cur.push_back(j);
        }
        if (n > 1) cur_sync = true;
    }
    if (!cur.empty()) emit(cur, cur_sync, -1, 0);
    ph.n_tiles = (int)(ph.tile_heavy.size() / 2);
}

void build_tiles_cols(PlanHost& ph, int W, int bcols) {
    const int64_t NI = ph.item_panel.size();
    const int64_t nP = ph.header[7];
    const int h = ph.header[5];
    ph.slot_item.clear();
    ph.slot_aux.clear();
    ph.tile_heavy.clear();
    ph.heavy_info.clear();
    ph.slot_ws.clear();
    ph.n_heavy = ph.n_heavy_tiles = ph.n_split_items = 0;
    ph.any_sync = false;
    ph.n_wsc_counters = 0;
    ph.wsc_floats = 0;
    std::vector<int64_t> first(nP + 1, NI);
    for (int64_t i = NI - 1; i >= 0; i--) first[ph.item_panel[i]] = i;
    first[nP] = NI;
    for (int64_t P = nP - 1; P >= 0; P--)
        if (first[P] > first[P + 1]) first[P] = first[P + 1];
    // per split panel: a counter and a workspace range of n x h x bcols floats
    std::vector<int32_t> ctr(nP, -1);
    std::vector<int64_t> wsb(nP, 0);
    int64_t maxn = 0;
    for (int64_t P = 0; P < nP; P++) {
        const int64_t n = first[P + 1] - first[P];
        maxn = std::max(maxn, n);
        if (n > 1) {
            ctr[P] = ph.n_wsc_counters++;
            wsb[P] = ph.wsc_floats;
            ph.wsc_floats += n * (int64_t)h * bcols;
            ph.n_split_items += (int32_t)n;
        }
    }
    std::vector<int64_t> grp;
    auto emit = [&]() {
        for (int k = 0; k < W; k++) {
            if (k < (int)grp.size()) {
                const int64_t it = grp[k], P = ph.item_panel[it], n = first[P + 1] - first[P];
                const int64_t q = it - first[P];
                ph.slot_item.push_back((int32_t)it);
                ph.slot_aux.push_back((1 << 16) | (n > 1 ? (1 << 19) : 0));
                if (wsb[P] + q * h * bcols >= INT32_MAX) throw std::runtime_error("column-window workspace too large");
                ph.slot_ws.insert(ph.slot_ws.end(), {(int32_t)(wsb[P] + q * h * bcols), ctr[P], (int32_t)n, (int32_t)q});
            } else {
                ph.slot_item.push_back(-1);
                ph.slot_aux.push_back(0);
                ph.slot_ws.insert(ph.slot_ws.end(), {0, -1, 0, 0});
            }
        }
        ph.tile_heavy.push_back(-1);
        ph.tile_heavy.push_back(0);
        grp.clear();
    };
    // item index j of consecutive panels, j-major: the tiles of one column
    // window are launched together
    for (int64_t j = 0; j < maxn; j++) {
        for (int64_t P = 0; P < nP; P++) {
            if (first[P + 1] - first[P] <= j) continue;
            grp.push_back(first[P] + j);
            if ((int)grp.size() == W) emit();
        }
        if (!grp.empty()) emit();
    }
    ph.n_tiles = (int)(ph.tile_heavy.size() / 2);
}

int rec_words(int h) { return h == 1 ? 2 : (h <= 3 ? 4 : (h <= 7 ? 8 : 12)); }

// The staged walk's schedule.  Row block rb = panels [rb*nslot, (rb+1)*nslot)
// (nslot = warps x npw; warp w owns slots w*npw .. w*npw + npw - 1), split sp
// = columns [sp*k/nsplit, (sp+1)*k/nsplit), stage = kb columns of a split.
// CTA (rb, sp) = rb*nsplit + sp.  Its records: for each stage, for each slot,
// the slot panel's gcols whose column lies in the stage, in canonical gcol
// order (a stable counting sort by (stage, slot) of the panels' streams), each
// stage padded to 16 bytes.  Every canonical gcol lands in exactly one record
// (tests/test_staged.py checks the permutation against the exported plan).
std::string build_staged(const PlanHost& ph, int bcols, int warps, int npw, int nsplit, int kb,
                         size_t smem_cap, StagedHost& st) {
    const int64_t k = ph.header[2], nP = ph.header[7], NG = ph.header[8];
    const int h = ph.header[5];
    if (warps < 1 || warps > 16 || npw < 1 || npw > 4 || nsplit < 1 || kb < 1)
        return "staged parameters out of range (warps 1..16, npw 1..4, nsplit >= 1, kb >= 1)";
    if (nsplit > k) return "more k-splits than columns";
    st = StagedHost();
    st.warps = warps; st.npw = npw; st.nsplit = nsplit; st.kb = kb;
    st.nslot = warps * npw;
    st.hs = (st.nslot + 1 + 3) & ~3;
    st.rw = rec_words(h);
    const int64_t pad = st.rw >= 4 ? 1 : 16 / (4 * st.rw);   // records per 16 bytes
    const int64_t nslot = st.nslot;
    const int64_t n_rb = (nP + nslot - 1) / nslot;
    if (n_rb * nsplit >= INT32_MAX) return "too many CTAs";
    auto ks = [&](int64_t sp) { return (sp * k) / nsplit; };
    int max_st = 0;
    for (int64_t sp = 0; sp < nsplit; sp++) {
        const int64_t wd = ks(sp + 1) - ks(sp);
        max_st = std::max<int>(max_st, (int)((wd + kb - 1) / kb));
        st.max_k = std::max<int>(st.max_k, (int)wd);
    }
    if (max_st > 16) return "more than 16 stages per CTA (raise kb or nsplit)";
    st.max_stages = max_st;
    // first group of each panel (groups are ordered by panel)
    std::vector<int64_t> pg(nP + 1, NG);
    for (int64_t g = NG - 1; g >= 0; g--) pg[ph.grp_panel[g]] = g;
    for (int64_t P = nP - 1; P >= 0; P--) pg[P] = std::min(pg[P], pg[P + 1]);
    const int64_t nkey = (int64_t)nsplit * max_st * nslot;
    std::vector<int64_t> cnt(nkey + 1), pos(nkey);
    std::vector<int32_t> keyed;   // gcols of the row block by key
    int64_t R = 0;                // records emitted (absolute)
    for (int64_t rb = 0; rb < n_rb; rb++) {
        std::fill(cnt.begin(), cnt.end(), 0);
        auto key_of = [&](int64_t j, int32_t col) {
            const int64_t sp = (((int64_t)col + 1) * nsplit - 1) / k;
            const int64_t s = (col - ks(sp)) / kb;
            return (sp * max_st + s) * nslot + j;
        };
        for (int64_t j = 0; j < nslot; j++) {
            const int64_t P = rb * nslot + j;
            if (P >= nP) break;
            for (int64_t c = ph.grp_col_ptr[pg[P]]; c < ph.grp_col_ptr[pg[P + 1]]; c++)
                cnt[key_of(j, ph.gcol[c]) + 1]++;
        }
        for (int64_t x = 0; x < nkey; x++) cnt[x + 1] += cnt[x];
        keyed.assign(cnt[nkey], 0);
        for (int64_t x = 0; x < nkey; x++) pos[x] = cnt[x];
        for (int64_t j = 0; j < nslot; j++) {
            const int64_t P = rb * nslot + j;
            if (P >= nP) break;
            for (int64_t c = ph.grp_col_ptr[pg[P]]; c < ph.grp_col_ptr[pg[P + 1]]; c++)
                keyed[pos[key_of(j, ph.gcol[c])]++] = (int32_t)c;
        }
        for (int64_t sp = 0; sp < nsplit; sp++) {
            const int64_t k0 = ks(sp), k1 = ks(sp + 1);
            const int nst = (int)((k1 - k0 + kb - 1) / kb);
            const int64_t rec0 = R;
            // stage entries and headers at a fixed stride of max_stages per
            // CTA (zero padding): a CTA finds its stages from blockIdx alone,
            // so its first loads are independent of each other
            st.cta.insert(st.cta.end(), {(int32_t)rb, (int32_t)sp, (int32_t)(st.stage.size() / 4), nst});
            for (int s = 0; s < nst; s++) {
                const int64_t a = k0 + (int64_t)s * kb, b = std::min<int64_t>(k1, a + kb);
                const int64_t r0 = R;
                const size_t hb = st.hdr.size();
                st.hdr.resize(hb + st.hs, 0);
                for (int64_t j = 0; j < nslot; j++) {
                    const int64_t x = (sp * max_st + s) * nslot + j;
                    st.hdr[hb + j] = (int32_t)(R - rec0);
                    for (int64_t q = cnt[x]; q < cnt[x + 1]; q++) st.src.push_back(keyed[q]);
                    R += cnt[x + 1] - cnt[x];
                }
                st.hdr[hb + nslot] = (int32_t)(R - rec0);
                while (R % pad) {
                    st.src.push_back(-1);
                    R++;
                }
                st.stage.insert(st.stage.end(), {(int32_t)a, (int32_t)b, (int32_t)r0, (int32_t)(R - r0)});
                if (R >= INT32_MAX) return "staged record stream too large";
            }
            for (int s = nst; s < max_st; s++) {
                st.stage.insert(st.stage.end(), {0, 0, 0, 0});
                st.hdr.resize(st.hdr.size() + st.hs, 0);
            }
            st.max_rec = std::max<int>(st.max_rec, (int)(R - rec0));
        }
    }
    st.n_cta = (int)(st.cta.size() / 4);
    const size_t need = ((size_t)st.max_k * bcols + (size_t)st.max_rec * st.rw + (size_t)st.max_stages * st.hs) * 4;
    if (need > smem_cap)
        return "staged CTA needs " + std::to_string(need) + " bytes of shared memory (cap " +
               std::to_string(smem_cap) + "): raise nsplit";
    return "";
}

// Parameter table (§3.5 Scheduler & Tuner), fitted to the
// profiling sweeps of tools/tune.py on B200 (profiles/r1_tune_*.json,
// profiles/r2_notes.md):
//  * UFi, CSR-value walk (escs_spmm): UFi = 1 -- every pattern row costs a
//    slot-map indirection and staged values, which outweighs the B rows the
//    enumeration saves (r1 sweeps).  Packed-record walk (escs_spmm_packed,
//    packed = 1): the record carries the column, the pattern and the row values
//    in one broadcast load, so the p = h(1-s)/(1-s^h) B-row reuse of the
//    enumeration pays where p is large: UFi 4 below 75% sparsity, 2 below 85%,
//    1 above (the plan-time tuner searches UFi 1..4 either way).
//  * UFk = 8 B rows in flight per sub-warp on the layer suites; 4 on large
//    problems (occupancy) and at bCols 256 (registers).
//  * T: about 1536 items per launch (~10 warps per SM on 148 SMs: each item
//    long enough to amortise its dependent round trips), at least 16 columns,
//    rounded (with a 3-sigma margin on the panel stream) so that a typical
//    panel splits into equal items.
Params choose_params(int64_t m, int64_t k, int64_t nnz, int32_t bcols, int n_sm, int h_req,
                     bool packed) {
    Params p;
    const double d = (double)nnz / ((double)m * (double)k);
    const double s = 1.0 - d;
    p.packed = packed ? 1 : 0;
    p.h = h_req > 0 ? h_req : (!packed ? 1 : s < 0.75 ? 4 : s < 0.85 ? 2 : 1);
    p.variant = (bcols == 4 || bcols == 8 || bcols == 16 || bcols == 32 || bcols == 64 ||
                 bcols == 128 || bcols == 256) ? 1 : 2;
    // more rows in flight per warp on the small, latency-bound layers; more
    // resident warps (fewer registers) on the large, L2-bandwidth-bound ones
    // (C4: 183 -> 135 us, C5: 2.63 -> 2.28 ms with UFk 4; profiles/r1_notes.md)
    const double g_est = (double)nnz;   // gcols at UFi = 1
    p.ufk = (bcols > 128 || g_est > 1.5e6) ? 4 : 8;
    if (bcols < 32) p.ufk = bcols == 4 ? 1 : bcols == 8 ? 2 : 4;   // UFk x (32 / (bCols/4)) <= 32
    // bCols coarsening (columns per lane): on the large L1-wavefront-bound
    // problems a 16-column register tile per lane (8 lanes per B row, 4 rows
    // per warp instruction) halves the per-row broadcasts and issue
    // (C4: 91.5 -> 83.6 us hot-L2, C5: 2.25 -> 2.14 ms; profiles/r1_notes.md);
    // the packed walk takes 8 columns per lane at bCols 128 (two records per
    // warp load instruction; exp sweeps in profiles/r2_notes.md)
    p.colf = (bcols == 128 && g_est > 1.5e6) ? 16 : (packed && bcols == 128) ? 8 : 0;
    const double sp = (double)k * (1.0 - std::pow(s, p.h));   // expected panel stream
    const double G = std::ceil((double)m / p.h) * sp;
    const double target_items = 1536.0 * (double)n_sm / 148.0;
    const int64_t Tmin = 16;
    int64_t T = std::max<int64_t>(Tmin, (int64_t)std::ceil(G / target_items));
    if (sp >= 1.0) {
        // panel streams vary around sp (binomial, sigma ~ sqrt(sp)): leave a
        // 3-sigma margin so that typical panels really split into `per` items
        const int64_t per = std::max<int64_t>(1, (int64_t)std::ceil(sp / (double)T));
        T = std::max<int64_t>(Tmin, (int64_t)std::ceil((sp + 3.0 * std::sqrt(sp)) / (double)per));
    }
    T = std::min<int64_t>(T, 1 << 20);
    p.T = (int)T;
    p.cta_warps = 0;   // auto from the item distribution
    return p;
}

}  // namespace escs
