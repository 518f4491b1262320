// bc_tmem_plan.cpp -- schedule of the Tensor-Memory kernel (bc_tmem.cuh).
//
// The kernel's SpMV cost is shared-memory wavefronts (ncu: the LSU data pipe
// is the bound).  Per SpMV a warp (team) issues, besides the TMEM reads:
//   * one LDS.64 gather per step          -- wavefronts = sum over the
//     half-warps of the largest number of distinct 8-byte slots that fall in
//     one of the 16 bank pairs (measured exactly, tools/bank_probe.py);
//   * one STS.64 per row-end position      -- lane-major Y makes each half-
//     warp's stores conflict-free (1 wavefront per half with an end);
//   * R*RV publishes of x into the gather vector copies and RV reads of Y.
// The gather vector is kept in R (2) copies; every access picks the copy
// whose bank is free (an exact small b-matching per half-warp).  Copy 0 is
// the identity placement and copy 1 rotates each 16-column group, so the
// owners' publishes are conflict-free.  Rows are packed into 32W lanes x ST
// row streams (first-fit decreasing / LPT), then a simulated annealing over
// copy 1's rotations and over which lane runs which (padded) row, in which
// order, minimises the weighted total.  BiCG's pair schedule holds A's rows on
// stream 0 and A^T's rows on stream 1.  Row entries keep their CSR order (A^T:
// ascending source row) and rows their values, so this changes speed only.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <string>
#include <mutex>
#include <map>
#include <stdexcept>

#include "bc_plan.hpp"

namespace bc {

namespace {

constexpr int kLanes = 32;

struct TmOpt {
    int S = 0, ncol = 0, nrow = 0, R = 1, NS = 16;
    // pair: A rows on stream 0 and A^T rows (outputs nrow + j, gathering
    // columns nrow + i) on stream 1, one pass for BiCG's two products
    bool pair = false;
    // ST interleaved row streams per lane: virtual lane v = s*32 + L runs on
    // physical lane L, its virtual step u on physical step u*ST + s
    int ST = 1;
    // LW lanes per group: a team of LW/32 warps shares one cell (rows spread
    // over all its lanes; half-warps are lanes [16h, 16h+16), H of them)
    int LW = kLanes;
    // stream s's Y region starts s * ybank_shift banks further round (ystream
    // = 8 mod 16 for two streams), so owner reads of rows computed on
    // different streams by lanes L and L+16 no longer collide
    int ybank_shift = 0;
    int H() const { return LW / 16; }
    int VL() const { return LW * ST; }
    int cap() const { return S / ST; }
    const std::vector<int>* seg_len;
    const std::vector<std::vector<int>>* seg_cols;
    const std::vector<int>* seg_row;
    std::vector<std::vector<int>> lane_segs;
    std::vector<int> pos;    // [r * ncol + c] slot within copy r
    std::vector<int> owner;  // [r * NS + slot] -> column, -1 free
    std::vector<int> col_at; // [t * 32 + L] column read, -1 = idle tail
    std::vector<uint8_t> end_at;
    std::vector<int> row_lane;  // row -> lane computing it
    std::vector<int> load;
    std::vector<int> gcost;  // [t * H() + h]
    int gsum = 0, pub = 0, yrd = 0, yst = 0;

    int bank(int r, int c) const { return pos[r * ncol + c] & 15; }

    // min over copy choices of the max bank load of distinct columns cols[0..m)
    int match_cost(const int* cols, int m, int* choice) const {
        if (m == 0) return 0;
        for (int cap = (m + 15) / 16; cap <= m; ++cap) {
            int load_b[16] = {0};
            int assign[16];
            for (int i = 0; i < m; ++i) assign[i] = -1;
            bool ok = true;
            for (int i = 0; i < m && ok; ++i) {
                bool vis[16] = {false};
                ok = augment(i, cols, m, cap, load_b, assign, vis);
            }
            if (ok) {
                if (choice)
                    for (int i = 0; i < m; ++i) {
                        choice[i] = 0;
                        for (int r = 0; r < R; ++r)
                            if (bank(r, cols[i]) == assign[i]) {
                                choice[i] = r;
                                break;
                            }
                    }
                return cap;
            }
        }
        return m;
    }
    bool augment(int i, const int* cols, int m, int cap, int* load_b, int* assign, bool* vis) const {
        for (int r = 0; r < R; ++r) {
            const int b = bank(r, cols[i]);
            if (vis[b]) continue;
            vis[b] = true;
            if (load_b[b] < cap) {
                load_b[b]++;
                assign[i] = b;
                return true;
            }
            for (int i2 = 0; i2 < m; ++i2)
                if (assign[i2] == b && augment(i2, cols, m, cap, load_b, assign, vis)) {
                    assign[i] = b;
                    return true;
                }
        }
        return false;
    }
    int distinct(int t, int h, int* cols) const {
        int m = 0;
        for (int L = 16 * h; L < 16 * h + 16; ++L) {
            const int c = col_at[t * LW + L];
            if (c < 0) continue;
            bool dup = false;
            for (int q = 0; q < m; ++q) dup |= cols[q] == c;
            if (!dup) cols[m++] = c;
        }
        return m;
    }
    int group_cost(int t, int h) const {
        int cols[16];
        const int m = distinct(t, h, cols);
        return match_cost(cols, m, nullptr);
    }
    int at(int v, int u) const { return (u * ST + v / LW) * LW + v % LW; }
    void lay_lane(int v) {
        for (int u = 0; u < cap(); ++u) {
            col_at[at(v, u)] = -1;
            end_at[at(v, u)] = 0;
        }
        int u = 0;
        for (int sg : lane_segs[v]) {
            const auto& cols = (*seg_cols)[sg];
            for (size_t q = 0; q < cols.size(); ++q, ++u) col_at[at(v, u)] = cols[q];
            // the row's Y bank (mod 16): lane and stream shift
            const int bank = (v % LW + (v / LW) * ybank_shift) & 15;
            end_at[at(v, u - 1)] = static_cast<uint8_t>(1 + bank);
            row_lane[(*seg_row)[sg]] = bank;
        }
        load[v] = u;
    }
    int publish_cost() const {  // R*RV STS.64 by the owner lanes (rows 32j+L), twice for a pair
        int tot = 0;
        for (int part = 0; part < (pair ? 2 : 1); ++part)
            for (int r = 0; r < R; ++r)
                for (int j = 0; j * 32 < nrow; ++j)
                    for (int h = 0; h < 2; ++h) {
                        int cnt[16] = {0};
                        for (int q = 0; q < 16; ++q) {
                            const int row = 32 * j + 16 * h + q;
                            if (row < nrow) cnt[bank(r, part * nrow + row)]++;
                        }
                        tot += *std::max_element(cnt, cnt + 16);
                    }
        return tot;
    }
    int yread_cost() const {  // RV LDS.64 of Y[..+k*32+lane(row)]: bank = lane(row) & 15
        int tot = 0;
        for (int part = 0; part < (pair ? 2 : 1); ++part)
            for (int j = 0; j * 32 < nrow; ++j)
                for (int h = 0; h < 2; ++h) {
                    int cnt[16] = {0};
                    for (int q = 0; q < 16; ++q) {
                        const int row = 32 * j + 16 * h + q;
                        if (row < nrow && row_lane[part * nrow + row] >= 0) cnt[row_lane[part * nrow + row] & 15]++;
                    }
                    tot += *std::max_element(cnt, cnt + 16);
                }
        return tot;
    }
    int ystore_cost() const {  // per half-warp with row ends: the largest bank multiplicity
        int tot = 0;
        for (int t = 0; t < S; ++t)
            for (int h = 0; h < H(); ++h) {
                int cnt[16] = {0}, mx = 0;
                for (int L = 16 * h; L < 16 * h + 16; ++L)
                    if (const int e = end_at[t * LW + L]) mx = std::max(mx, ++cnt[e - 1]);
                tot += mx;
            }
        return tot;
    }
    // weights of the wavefront kinds in the annealing objective (BC_PUB_WEIGHT,
    // BC_YST_WEIGHT): the model counts wavefronts, weights bias the search
    // (B200, 100k M156: Y stores weighted 3 -> BiCGSTAB 584k vs 574k with 2, 538k with 1)
    int wpub = 1, wyst = 3, wyrd = 1;
    bool copy0_fixed = false;
    // copy1_shift (default): copy 0 keeps the identity placement and copy 1
    // rotates each 16-column group by a shift (bank = (column + shift[group])
    // mod 16), so the owners' publishes are conflict-free in both copies (20
    // wavefronts per M156 SpMV, the floor, vs 37) while the shifts still give
    // every column a second bank for the gathers (111 vs 104 wavefronts):
    // 538k vs 515k cell-solves/s (B200, 100k M156, BiCGSTAB)
    bool copy1_shift = true;
    std::vector<int> shift1;
    void place_group1(int g) {
        for (int c = 16 * g; c < std::min(ncol, 16 * g + 16); ++c) {
            const int slot = 16 * g + ((c % 16 + shift1[g]) % 16);
            pos[ncol + c] = slot;
            owner[NS + slot] = c;
        }
    }
    int total() const { return gsum + wpub * pub + wyrd * yrd + wyst * yst; }
    void full_eval() {
        gsum = 0;
        for (int t = 0; t < S; ++t)
            for (int h = 0; h < H(); ++h) gsum += (gcost[t * H() + h] = group_cost(t, h));
        pub = publish_cost();
        yrd = yread_cost();
        yst = ystore_cost();
    }
    // re-evaluate the gather groups of the halves holding lanes A and B
    int regather_lanes(int A, int B) {
        int g = gsum;
        const int ha = (A % LW) / 16, hb = (B % LW) / 16;
        for (int t = 0; t < S; ++t) {
            const int id = t * H() + ha;
            const int c = group_cost(t, ha);
            g += c - gcost[id];
            gcost[id] = c;
            if (hb != ha) {
                const int id2 = t * H() + hb;
                const int c2 = group_cost(t, hb);
                g += c2 - gcost[id2];
                gcost[id2] = c2;
            }
        }
        return g;
    }
};

}  // namespace

namespace {

TmemSchedule build_uncached(const Pattern& pat, int k, bool pair, int team, bool optimize, bool quick) {
    if (const char* e = std::getenv("BC_SCHED_OPT")) optimize = optimize && std::atoi(e) != 0;
    // two placements of the gather vector: 448k vs 409k cell-solves/s with one,
    // 413k with three (B200, 100k M156, P regime; BC_GATHER_COPIES=1 overrides)
    int copies = 2;
    if (const char* e = std::getenv("BC_GATHER_COPIES")) copies = std::atoi(e) == 1 ? 1 : 2;
    if (!optimize) copies = 1;
    // rows padded to an even number of (virtual) steps, so that rows end only
    // on steps 1, 3 (one stream) or 2, 3 (two streams) of a 4-step chunk
    constexpr int d = 2;
    // two interleaved accumulator chains per lane (BC_TMEM_STREAMS); four-warp
    // teams on groups of <= 512 rows use one, as their rows are already short
    // (the longest row would set the step count).  Coupled groups above 512
    // rows (Block-cells(N): 936) take two: B200, 100k M156 cells, BiCGSTAB P,
    // 412k vs 394k cell-solves/s
    const int n_rows = k * pat.species;
    int streams = team >= 4 && n_rows <= 512 ? 1 : 2;
    if (const char* e = std::getenv("BC_TMEM_STREAMS")) streams = std::atoi(e) == 1 ? 1 : 2;
    if (pair) streams = 2;  // A on stream 0, A^T on stream 1
    const int s = pat.species, nnz = pat.nnz, n = k * s;
    const int nx = pair ? 2 * n : n;  // gathered columns: p (and p~ at n + i)
    const int zero_col = nx;          // pseudo-row whose slots always hold +0.0
    // rows as segments padded to a multiple of d (csr.cpp:90-101 order kept)
    std::vector<int> seg_row, seg_len;
    std::vector<std::vector<int>> seg_cols, seg_vals;
    for (int c = 0; c < k; ++c)
        for (int r = 0; r < s; ++r) {
            if (pat.row_ptr[r + 1] == pat.row_ptr[r]) continue;
            std::vector<int> cols, vals;
            for (int e = pat.row_ptr[r]; e < pat.row_ptr[r + 1]; ++e) {
                cols.push_back(c * s + pat.col_idx[e]);
                vals.push_back(c * nnz + e);
            }
            while (cols.size() % d) {
                cols.push_back(zero_col);
                vals.push_back(-1);
            }
            seg_row.push_back(c * s + r);
            seg_len.push_back(static_cast<int>(cols.size()));
            seg_cols.push_back(std::move(cols));
            seg_vals.push_back(std::move(vals));
        }
    const int n_a_segs = static_cast<int>(seg_row.size());
    if (pair) {  // A^T row j = column j of A in ascending source row i (csr.cpp:129-142)
        for (int c = 0; c < k; ++c) {
            std::vector<std::vector<int>> tcols(s), tvals(s);
            for (int i = 0; i < s; ++i)
                for (int e = pat.row_ptr[i]; e < pat.row_ptr[i + 1]; ++e) {
                    tcols[pat.col_idx[e]].push_back(n + c * s + i);
                    tvals[pat.col_idx[e]].push_back(c * nnz + e);
                }
            for (int j = 0; j < s; ++j) {
                if (tcols[j].empty()) continue;
                while (tcols[j].size() % d) {
                    tcols[j].push_back(zero_col);
                    tvals[j].push_back(-1);
                }
                seg_row.push_back(n + c * s + j);
                seg_len.push_back(static_cast<int>(tcols[j].size()));
                seg_cols.push_back(std::move(tcols[j]));
                seg_vals.push_back(std::move(tvals[j]));
            }
        }
    }
    TmOpt o;
    o.LW = kLanes * std::max(1, team);
    if (const char* e = std::getenv("BC_PUB_WEIGHT")) o.wpub = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("BC_YST_WEIGHT")) o.wyst = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("BC_YRD_WEIGHT")) o.wyrd = std::max(1, std::atoi(e));
    if (!optimize) o.copy1_shift = false;
    if (const char* e = std::getenv("BC_COPY0_FIXED")) o.copy0_fixed = std::atoi(e) != 0;
    if (const char* e = std::getenv("BC_COPY1_SHIFT")) o.copy1_shift = std::atoi(e) != 0;
    if (o.copy1_shift && copies == 2) o.copy0_fixed = true;
    o.seg_len = &seg_len;
    o.seg_cols = &seg_cols;
    o.seg_row = &seg_row;
    o.ncol = nx + 1;
    o.nrow = n;
    o.R = copies;
    o.ST = streams;
    o.ybank_shift = o.ST == 2 ? 8 : 0;
    if (const char* e = std::getenv("BC_YBANK_SHIFT")) o.ybank_shift = std::atoi(e) ? o.ybank_shift : 0;
    o.pair = pair;
    o.lane_segs.assign(o.VL(), {});
    o.load.assign(o.VL(), 0);
    // lane groups a segment may use: everything, or (pair) stream 0 / stream 1
    auto group_of_seg = [&](int sg) { return pair && sg >= n_a_segs ? 1 : 0; };
    auto group_of_lane = [&](int v) { return pair && v >= o.LW ? 1 : 0; };
    {  // longest-processing-time start
        std::vector<int> order(seg_row.size());
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return seg_len[a] > seg_len[b]; });
        for (int idx : order) {
            int best = -1;
            for (int L = 0; L < o.VL(); ++L)
                if (group_of_lane(L) == group_of_seg(idx) && (best < 0 || o.load[L] < o.load[best])) best = L;
            o.load[best] += seg_len[idx];
            o.lane_segs[best].push_back(idx);
        }
        // lower the longest lane: move a segment off it, or swap it for a
        // shorter one, whenever the other lane stays below the current maximum
        for (int guard = 0; guard < 10000; ++guard) {
            const int M = *std::max_element(o.load.begin(), o.load.end());
            bool moved = false;
            for (int b = 0; b < o.VL() && !moved; ++b) {
                if (o.load[b] != M) continue;
                for (size_t i = 0; i < o.lane_segs[b].size() && !moved; ++i) {
                    const int sa = o.lane_segs[b][i];
                    for (int c = 0; c < o.VL() && !moved; ++c) {
                        if (c == b || group_of_lane(c) != group_of_lane(b)) continue;
                        if (o.load[c] + seg_len[sa] < M) {
                            o.lane_segs[b].erase(o.lane_segs[b].begin() + i);
                            o.lane_segs[c].push_back(sa);
                            o.load[b] -= seg_len[sa];
                            o.load[c] += seg_len[sa];
                            moved = true;
                            break;
                        }
                        for (size_t j = 0; j < o.lane_segs[c].size(); ++j) {
                            const int sc = o.lane_segs[c][j];
                            const int dlt = seg_len[sa] - seg_len[sc];
                            if (dlt > 0 && o.load[c] + dlt < M) {
                                std::swap(o.lane_segs[b][i], o.lane_segs[c][j]);
                                o.load[b] -= dlt;
                                o.load[c] += dlt;
                                moved = true;
                                break;
                            }
                        }
                    }
                }
            }
            if (!moved) break;
        }
        // first-fit decreasing into the smallest lane capacity it fits, if that
        // beats the balanced start (S = ST * capacity must stay a multiple of 4)
        const int unit = 4 / o.ST;
        int total = 0;
        for (int l : seg_len) total += l;
        const int lpt_max = *std::max_element(o.load.begin(), o.load.end());
        int cap = std::max(order.empty() ? 0 : seg_len[order[0]], (total + o.VL() - 1) / o.VL());
        if (pair) {  // each stream's lanes carry their own rows
            int ta = 0;
            for (int sg = 0; sg < n_a_segs; ++sg) ta += seg_len[sg];
            cap = std::max({cap, (ta + o.LW - 1) / o.LW, (total - ta + o.LW - 1) / o.LW});
        }
        cap = (cap + unit - 1) / unit * unit;
        for (; cap < lpt_max; cap += unit) {
            std::vector<std::vector<int>> segs(o.VL());
            std::vector<int> load(o.VL(), 0);
            bool ok = true;
            for (int idx : order) {
                int b = 0;
                while (b < o.VL() && (group_of_lane(b) != group_of_seg(idx) || load[b] + seg_len[idx] > cap)) ++b;
                if (b == o.VL()) {
                    ok = false;
                    break;
                }
                load[b] += seg_len[idx];
                segs[b].push_back(idx);
            }
            if (ok) {
                o.lane_segs = segs;
                o.load = load;
                break;
            }
        }
    }
    const int S0 = std::max(4, o.ST * *std::max_element(o.load.begin(), o.load.end()));
    o.S = (S0 + 3) & ~3;  // the kernel walks 8 steps per TMEM load pair, then a 4-step tail
    // slots per copy: the rotated placements need no slack; free placement gets 25%
    o.NS = optimize && !(o.copy1_shift && o.R == 2) ? ((o.ncol + o.ncol / 4 + 15) / 16) * 16
                                                  : ((o.ncol + 15) / 16) * 16;
    o.pos.resize(static_cast<size_t>(o.R) * o.ncol);
    o.owner.assign(static_cast<size_t>(o.R) * o.NS, -1);
    uint64_t rng = 0x243F6A8885A308D3ull ^ static_cast<uint64_t>(n * 977 + nnz);
    auto rnd = [&]() {
        rng ^= rng << 13;
        rng ^= rng >> 7;
        rng ^= rng << 17;
        return rng;
    };
    for (int r = 0; r < o.R; ++r) {
        std::vector<int> perm(o.NS);
        std::iota(perm.begin(), perm.end(), 0);
        if (r > 0)
            for (int i = o.NS - 1; i > 0; --i) std::swap(perm[i], perm[rnd() % (i + 1)]);
        for (int c = 0; c < o.ncol; ++c) {
            o.pos[r * o.ncol + c] = perm[c];
            o.owner[r * o.NS + perm[c]] = c;
        }
    }
    if (o.copy1_shift && o.R == 2) {
        std::fill(o.owner.begin() + o.NS, o.owner.begin() + 2 * o.NS, -1);
        o.shift1.assign((o.ncol + 15) / 16, 0);
        for (size_t g = 0; g < o.shift1.size(); ++g) {
            o.shift1[g] = static_cast<int>(rnd() % 16);
            o.place_group1(static_cast<int>(g));
        }
    }
    o.col_at.assign(static_cast<size_t>(o.S) * o.LW, -1);
    o.end_at.assign(static_cast<size_t>(o.S) * o.LW, 0);
    o.row_lane.assign(pair ? 2 * n : n, -1);
    o.gcost.assign(static_cast<size_t>(o.S) * o.H(), 0);
    for (int v = 0; v < o.VL(); ++v) o.lay_lane(v);
    o.full_eval();

    if (optimize) {
        auto urand = [&]() { return static_cast<double>(rnd() >> 11) * 0x1.0p-53; };
        // ~128 moves per scheduled entry, 2k..200k: at M156 (200k) 511k vs
        // 503k cell-solves/s with 24k (B200, 100k cells), a few seconds once
        // per pattern (schedules are cached per process); small patterns stay
        // cheap
        long entries = 0;
        for (int l : seg_len) entries += l;
        long iters = std::max<long>(2000, std::min<long>(200000, 128 * entries));
        if (quick) iters = std::min<long>(iters, 10000);  // small batches: latency-bound, placement matters less
        if (o.LW > kLanes) iters = std::min<long>(iters, 50000);  // teams: latency-bound small batches
        if (const char* e = std::getenv("BC_ANNEAL_ITERS")) iters = std::atol(e);
        double T = 1.0;
        const double cool = std::pow(0.01 / T, 1.0 / static_cast<double>(iters));
        int cur = o.total(), best = cur;
        TmOpt best_o = o;
        std::vector<int> touched;
        for (long it = 0; it < iters; ++it, T *= cool) {
            const int kind = static_cast<int>(rnd() % 4);
            if (kind <= 1) {  // move one column's slot within one copy
                // copy0_fixed: copy 0 keeps the identity placement (bank = column mod 16,
                // so the owners' publishes into it are conflict-free); copy 1 moves
                const int r = o.copy0_fixed && o.R > 1 ? 1 + static_cast<int>(rnd() % (o.R - 1))
                                                       : static_cast<int>(rnd() % o.R);
                if (o.copy1_shift && r == 1) {  // re-rotate one 16-column group of copy 1
                    const int gi = static_cast<int>(rnd() % o.shift1.size());
                    const int old_sh = o.shift1[gi];
                    o.shift1[gi] = static_cast<int>(rnd() % 16);
                    if (o.shift1[gi] == old_sh) continue;
                    o.place_group1(gi);
                    touched.clear();
                    for (size_t q = 0; q < o.col_at.size(); ++q)
                        if (o.col_at[q] >= 16 * gi && o.col_at[q] < 16 * gi + 16)
                            touched.push_back(static_cast<int>((q / o.LW) * o.H() + (q % o.LW) / 16));
                    std::sort(touched.begin(), touched.end());
                    touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
                    int g = o.gsum;
                    std::vector<int> nc(touched.size());
                    for (size_t q = 0; q < touched.size(); ++q) {
                        nc[q] = o.group_cost(touched[q] / o.H(), touched[q] % o.H());
                        g += nc[q] - o.gcost[touched[q]];
                    }
                    const int nt = g + o.wpub * o.pub + o.wyrd * o.yrd + o.wyst * o.yst;
                    if (nt - cur <= 0 || urand() < std::exp(-(nt - cur) / T)) {
                        for (size_t q = 0; q < touched.size(); ++q) o.gcost[touched[q]] = nc[q];
                        o.gsum = g;
                        cur = nt;
                    } else {
                        o.shift1[gi] = old_sh;
                        o.place_group1(gi);
                    }
                    continue;
                }
                const int c = static_cast<int>(rnd() % o.ncol);
                const int slot = static_cast<int>(rnd() % o.NS);
                const int other = o.owner[r * o.NS + slot];
                if (other == c) continue;
                const int old = o.pos[r * o.ncol + c];
                auto apply = [&](int a_slot, int b_slot) {
                    o.pos[r * o.ncol + c] = a_slot;
                    o.owner[r * o.NS + a_slot] = c;
                    o.owner[r * o.NS + b_slot] = other;
                    if (other >= 0) o.pos[r * o.ncol + other] = b_slot;
                };
                apply(slot, old);
                touched.clear();
                for (size_t q = 0; q < o.col_at.size(); ++q)
                    if (o.col_at[q] == c || (other >= 0 && o.col_at[q] == other))
                        touched.push_back(static_cast<int>((q / o.LW) * o.H() + (q % o.LW) / 16));
                std::sort(touched.begin(), touched.end());
                touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
                int g = o.gsum;
                std::vector<int> nc(touched.size());
                for (size_t q = 0; q < touched.size(); ++q) {
                    nc[q] = o.group_cost(touched[q] / o.H(), touched[q] % o.H());
                    g += nc[q] - o.gcost[touched[q]];
                }
                const int npub = o.publish_cost();
                const int nt = g + o.wpub * npub + o.wyrd * o.yrd + o.wyst * o.yst;
                if (nt - cur <= 0 || urand() < std::exp(-(nt - cur) / T)) {
                    for (size_t q = 0; q < touched.size(); ++q) o.gcost[touched[q]] = nc[q];
                    o.gsum = g;
                    o.pub = npub;
                    cur = nt;
                } else {
                    apply(old, slot);
                }
            } else {
                // segment moves: reorder within a lane, move or exchange between lanes
                const int A = static_cast<int>(rnd() % o.VL());
                int B = kind == 2 ? A
                        : pair    ? (A / o.LW) * o.LW + static_cast<int>(rnd() % o.LW)
                                  : static_cast<int>(rnd() % o.VL());
                if (o.lane_segs[A].empty()) continue;
                const auto saveA = o.lane_segs[A], saveB = o.lane_segs[B];
                if (kind == 2) {
                    const int m = static_cast<int>(o.lane_segs[A].size());
                    if (m < 2) continue;
                    const int i = static_cast<int>(rnd() % m), j = static_cast<int>(rnd() % m);
                    if (i == j) continue;
                    std::swap(o.lane_segs[A][i], o.lane_segs[A][j]);
                } else {
                    if (A == B) continue;
                    const int ia = static_cast<int>(rnd() % o.lane_segs[A].size());
                    const int sa = o.lane_segs[A][ia];
                    if (o.lane_segs[B].empty() || (rnd() & 1)) {
                        if (o.load[B] + seg_len[sa] > o.cap()) continue;
                        const int ib = static_cast<int>(rnd() % (o.lane_segs[B].size() + 1));
                        o.lane_segs[A].erase(o.lane_segs[A].begin() + ia);
                        o.lane_segs[B].insert(o.lane_segs[B].begin() + ib, sa);
                    } else {
                        const int ib = static_cast<int>(rnd() % o.lane_segs[B].size());
                        const int sb = o.lane_segs[B][ib];
                        if (o.load[A] - seg_len[sa] + seg_len[sb] > o.cap() ||
                            o.load[B] - seg_len[sb] + seg_len[sa] > o.cap())
                            continue;
                        std::swap(o.lane_segs[A][ia], o.lane_segs[B][ib]);
                    }
                }
                const int old_g = o.gsum, old_y = o.yrd, old_s = o.yst;
                const auto old_gc = o.gcost;
                o.lay_lane(A);
                if (B != A) o.lay_lane(B);
                o.gsum = o.regather_lanes(A, B);
                o.yrd = o.yread_cost();
                o.yst = o.ystore_cost();
                const int nt = o.total();
                if (nt - cur <= 0 || urand() < std::exp(-(nt - cur) / T)) {
                    cur = nt;
                } else {
                    o.lane_segs[A] = saveA;
                    o.lane_segs[B] = saveB;
                    o.lay_lane(A);
                    if (B != A) o.lay_lane(B);
                    o.gsum = old_g;
                    o.gcost = old_gc;
                    o.yrd = old_y;
                    o.yst = old_s;
                }
            }
            if (cur < best) {
                best = cur;
                best_o = o;
            }
        }
        o = best_o;
    }

    // emission
    TmemSchedule ts;
    ts.steps = o.S;
    ts.copies = o.R;
    ts.xslots = o.R * o.NS;
    ts.zero_slot = o.pos[zero_col];
    ts.pair = pair ? 1 : 0;
    ts.xpos.assign(static_cast<size_t>(o.R) * nx, 0);
    for (int r = 0; r < o.R; ++r)
        for (int i = 0; i < nx; ++i) ts.xpos[static_cast<size_t>(r) * nx + i] = r * o.NS + o.pos[r * o.ncol + i];
    ts.words.assign(static_cast<size_t>(o.S) * o.LW, 0);
    ts.vidx.assign(static_cast<size_t>(o.S) * o.LW, -1);
    ts.yslot.assign(pair ? 2 * n : n, -1);
    std::vector<int> vals_at(static_cast<size_t>(o.S) * o.LW, -1);
    int kmax = 1;
    for (int v = 0; v < o.VL(); ++v) kmax = std::max(kmax, static_cast<int>(o.lane_segs[v].size()));
    // stream s's k-th row of lane L -> Y[s*kmax*32 + k*32 + L] (lane-major per stream)
    for (int v = 0; v < o.VL(); ++v) {
        int u = 0, kk = 0;
        for (int sg : o.lane_segs[v]) {
            for (size_t q = 0; q < seg_cols[sg].size(); ++q, ++u) vals_at[o.at(v, u)] = seg_vals[sg][q];
            ts.yslot[seg_row[sg]] = (v / o.LW) * (kmax * o.LW + o.ybank_shift) + kk * o.LW + v % o.LW;
            ++kk;
        }
    }
    ts.streams = o.ST;
    ts.ystream = kmax * o.LW + o.ybank_shift;
    ts.yslots = o.ST * ts.ystream;
    ts.team = o.LW / kLanes;
    for (int& y : ts.yslot)
        if (y < 0) y = ts.yslots;  // empty rows read the zero slot after the last row slot
    int cost = 0;
    for (int t = 0; t < o.S; ++t)
        for (int h = 0; h < o.H(); ++h) {
            int cols[16], choice[16];
            const int m = o.distinct(t, h, cols);
            cost += o.match_cost(cols, m, choice);
            for (int L = 16 * h; L < 16 * h + 16; ++L) {
                const int id = t * o.LW + L;
                int c = o.col_at[id], r = 0;
                if (c < 0) {  // idle tail: broadcast a column the half already reads
                    c = m > 0 ? cols[0] : zero_col;
                    r = m > 0 ? choice[0] : 0;
                } else {
                    for (int q = 0; q < m; ++q)
                        if (cols[q] == c) r = choice[q];
                }
                const int slot = r * o.NS + o.pos[r * o.ncol + c];
                uint16_t w = static_cast<uint16_t>(slot * 8);
                // a row ending on step 4c+3 is flagged on step 4c+2, one ending on
                // step 4c+1 (one stream) or 4c+2 (two streams) on step 4c: the low
                // halves of the chunk's two 32-bit TMEM words, masked off by the
                // address LOP3
                if ((t & 3) == 2 && o.end_at[id + o.LW]) w |= 0x8000u;
                if ((t & 3) == 0 && o.end_at[id + (o.ST == 1 ? 1 : 2) * o.LW]) w |= 0x8000u;
                ts.words[id] = w;
                ts.vidx[id] = vals_at[id];
            }
        }
    ts.conflict_cost = cost;
    ts.model_total = o.total();
    if (std::getenv("BC_PLAN_VERBOSE"))  // the model's unweighted terms
        std::fprintf(stderr, "tmem plan n=%d k=%d pair=%d team=%d S=%d: gathers %d publishes %d yreads %d ystores %d "
                     "total(weighted) %d\n", n, k, pair ? 1 : 0, team, o.S, o.gsum, o.pub, o.yrd, o.yst, o.total());
    if (ts.xslots * 8 > 0x7FFF) throw std::invalid_argument("TMEM schedule: gather vector too large");
    return ts;
}

}  // namespace

// Schedules are deterministic functions of (pattern, k, pair, team) and the
// tuning knobs, and cost seconds of annealing: built once per process.
TmemSchedule build_tmem_schedule(const Pattern& pat, int k, bool pair, int team, bool optimize, bool quick) {
    static std::mutex mu;
    static std::map<std::string, TmemSchedule> cache;
    std::string key;
    auto put = [&](const void* p, size_t n) { key.append(static_cast<const char*>(p), n); };
    const int head[6] = {pat.species, k, pair ? 1 : 0, team, optimize ? 1 : 0, quick ? 1 : 0};
    put(head, sizeof head);
    for (const char* env : {"BC_SCHED_OPT", "BC_GATHER_COPIES", "BC_TMEM_STREAMS", "BC_ANNEAL_ITERS", "BC_PUB_WEIGHT",
                            "BC_YST_WEIGHT", "BC_YRD_WEIGHT", "BC_COPY0_FIXED", "BC_COPY1_SHIFT",
                            "BC_YBANK_SHIFT"}) {
        const char* e = std::getenv(env);
        key += e ? e : "-";
        key += '|';
    }
    put(pat.row_ptr.data(), sizeof(int32_t) * pat.row_ptr.size());
    put(pat.col_idx.data(), sizeof(int32_t) * pat.col_idx.size());
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    TmemSchedule ts = build_uncached(pat, k, pair, team, optimize, quick);
    std::lock_guard<std::mutex> lock(mu);
    return cache.emplace(key, std::move(ts)).first->second;
}

}  // namespace bc
