// bc_plan.cpp -- see bc_plan.hpp.
#include "bc_plan.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <stdexcept>

namespace bc {

void optimize_gathers(int S, int lanes, int n, const std::vector<int>& seg_len,
                      const std::vector<std::vector<int>>& seg_cols, std::vector<std::vector<int>>* lane_segs,
                      int* xslots, std::vector<int32_t>* xpos);
int gather_cost(int steps, int lanes, const std::vector<uint32_t>& words);

Geometry choose_geometry(int n) {
    Geometry g;
    g.n = n;
    g.P = static_cast<int>(padded_len(n));
    g.Q = g.P >= 32 ? g.P / 32 : 1;
    // Up to 8 register slots per lane, then widen the team.
    g.W = g.Q <= 8 ? 1 : g.Q / 8;
    g.R = g.Q / g.W;
    const int m_count = (n + 31) / 32;        // 32-row columns holding real rows
    g.RV = (m_count + g.W - 1) / g.W;          // slots warp 0 may own
    if (g.RV < 1) g.RV = 1;
    if (g.RV > g.R) g.RV = g.R;
    return g;
}

Schedule build_schedule(const Pattern& pat, int k, int lanes, bool transpose, bool optimize) {
    const int s = pat.species, nnz = pat.nnz, n = k * s;
    // segments: output index + ordered list of (value index, gather index)
    struct Seg {
        int out;
        std::vector<std::pair<int, int>> ent;
    };
    std::vector<Seg> segs;
    if (!transpose) {
        // csr.cpp:90-101: row i accumulates its entries in storage order
        for (int c = 0; c < k; ++c)
            for (int r = 0; r < s; ++r) {
                Seg sg{c * s + r, {}};
                for (int e = pat.row_ptr[r]; e < pat.row_ptr[r + 1]; ++e)
                    sg.ent.push_back({c * nnz + e, c * s + pat.col_idx[e]});
                if (!sg.ent.empty()) segs.push_back(std::move(sg));
            }
    } else {
        // csr.cpp:129-142: y[col] accumulates rows in ascending order
        std::vector<Seg> cols(n);
        for (int j = 0; j < n; ++j) cols[j].out = j;
        for (int c = 0; c < k; ++c)
            for (int r = 0; r < s; ++r)
                for (int e = pat.row_ptr[r]; e < pat.row_ptr[r + 1]; ++e)
                    cols[c * s + pat.col_idx[e]].ent.push_back({c * nnz + e, c * s + r});
        for (auto& sg : cols)
            if (!sg.ent.empty()) segs.push_back(std::move(sg));
    }
    // Longest-processing-time assignment to lanes.
    std::vector<int> order(segs.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        return segs[a].ent.size() > segs[b].ent.size();
    });
    std::vector<int> load(lanes, 0);
    std::vector<std::vector<int>> lane_segs(lanes);
    for (int idx : order) {
        int best = 0;
        for (int L = 1; L < lanes; ++L)
            if (load[L] < load[best]) best = L;
        load[best] += static_cast<int>(segs[idx].ent.size());
        lane_segs[best].push_back(idx);
    }
    for (int L = 0; L < lanes; ++L)
        std::sort(lane_segs[L].begin(), lane_segs[L].end(),
                  [&](int a, int b) { return segs[a].out < segs[b].out; });
    Schedule sc;
    sc.steps = *std::max_element(load.begin(), load.end());
    sc.xslots = ((n + 15) / 16) * 16;
    sc.xpos.resize(n);
    std::iota(sc.xpos.begin(), sc.xpos.end(), 0);

    std::vector<int> seg_len(segs.size());
    std::vector<std::vector<int>> seg_cols(segs.size());
    for (size_t i = 0; i < segs.size(); ++i) {
        seg_len[i] = static_cast<int>(segs[i].ent.size());
        for (const auto& e : segs[i].ent) seg_cols[i].push_back(e.second);
    }
    if (optimize && sc.steps > 0)
        optimize_gathers(sc.steps, lanes, n, seg_len, seg_cols, &lane_segs, &sc.xslots, &sc.xpos);

    sc.words.assign(static_cast<size_t>(sc.steps) * lanes, 0u);
    sc.vpos.assign(static_cast<size_t>(k) * nnz, -1);
    sc.vidx.assign(static_cast<size_t>(sc.steps) * lanes, 0);
    std::vector<int> col_at(static_cast<size_t>(sc.steps) * lanes, -1);
    for (int L = 0; L < lanes; ++L) {
        int t = 0;
        for (int idx : lane_segs[L]) {
            const Seg& sg = segs[idx];
            for (size_t q = 0; q < sg.ent.size(); ++q, ++t) {
                const int slot = sc.xpos[sg.ent[q].second];
                uint32_t w = static_cast<uint32_t>(slot) | (static_cast<uint32_t>(sg.out) << kColBits);
                if (q + 1 == sg.ent.size()) w |= kEndBit;
                sc.words[static_cast<size_t>(t) * lanes + L] = w;
                col_at[static_cast<size_t>(t) * lanes + L] = slot;
                sc.vpos[sg.ent[q].first] = t * lanes + L;
                sc.vidx[static_cast<size_t>(t) * lanes + L] = sg.ent[q].first;
            }
        }
    }
    // Padding steps gather a slot another lane of the same half-warp already
    // reads (a broadcast, no extra wavefront); their sums are never stored.
    for (int t = 0; t < sc.steps; ++t)
        for (int g0 = 0; g0 < lanes; g0 += 16) {
            int any = -1;
            for (int L = g0; L < g0 + 16; ++L)
                if (col_at[static_cast<size_t>(t) * lanes + L] >= 0) any = col_at[static_cast<size_t>(t) * lanes + L];
            if (any < 0) any = 0;
            for (int L = g0; L < g0 + 16; ++L)
                if (col_at[static_cast<size_t>(t) * lanes + L] < 0)
                    sc.words[static_cast<size_t>(t) * lanes + L] = static_cast<uint32_t>(any);
        }
    sc.conflict_cost = gather_cost(sc.steps, lanes, sc.words);
    return sc;
}

// Shared-memory wavefronts of the gather loads of one schedule under the
// LDS.64 bank model (two half-warp phases; a phase costs the largest number
// of distinct 8-byte slots mapped to one of the 16 bank pairs).
int gather_cost(int steps, int lanes, const std::vector<uint32_t>& words) {
    int total = 0;
    for (int t = 0; t < steps; ++t)
        for (int g0 = 0; g0 < lanes; g0 += 16) {
            int cnt[16] = {0};
            int seen[16];
            int ns = 0;
            for (int L = g0; L < g0 + 16; ++L) {
                const int slot = static_cast<int>(words[static_cast<size_t>(t) * lanes + L] & kColMask);
                bool dup = false;
                for (int q = 0; q < ns; ++q) dup |= seen[q] == slot;
                if (dup) continue;
                seen[ns++] = slot;
                cnt[slot & 15]++;
            }
            total += *std::max_element(cnt, cnt + 16);
        }
    return total;
}

// Simulated annealing over (a) the shared-memory slot of every gathered
// vector entry and (b) which lane runs which row segment and in what order,
// minimising gather bank conflicts.  The step count S is kept (no lane may
// exceed it), each row's entries stay in CSR order, so the arithmetic -- and
// every result bit -- is unchanged; only the schedule's speed changes.
void optimize_gathers(int S, int lanes, int n, const std::vector<int>& seg_len,
                      const std::vector<std::vector<int>>& seg_cols, std::vector<std::vector<int>>* lane_segs_p,
                      int* xslots, std::vector<int32_t>* xpos_p) {
    auto& lane_segs = *lane_segs_p;
    auto& pos = *xpos_p;
    const int NS = ((n + n / 4 + 15) / 16) * 16;  // 25% spare slots
    *xslots = NS;
    std::vector<int> owner(NS, -1);
    for (int i = 0; i < n; ++i) owner[pos[i]] = i;
    const int groups = lanes / 16;
    // col_at[t][L]: gathered vector index at step t of lane L, -1 when idle
    std::vector<int> col_at(static_cast<size_t>(S) * lanes, -1);
    std::vector<int> load(lanes, 0);
    auto lay_lane = [&](int L) {
        for (int t = 0; t < S; ++t) col_at[static_cast<size_t>(t) * lanes + L] = -1;
        int t = 0;
        for (int sg : lane_segs[L])
            for (int c : seg_cols[sg]) col_at[static_cast<size_t>(t++) * lanes + L] = c;
        load[L] = t;
    };
    for (int L = 0; L < lanes; ++L) lay_lane(L);
    auto group_cost = [&](int t, int g) {
        int cnt[16] = {0}, seen[16], ns = 0;
        for (int L = g * 16; L < g * 16 + 16; ++L) {
            const int c = col_at[static_cast<size_t>(t) * lanes + L];
            if (c < 0) continue;
            const int slot = pos[c];
            bool dup = false;
            for (int q = 0; q < ns; ++q) dup |= seen[q] == slot;
            if (dup) continue;
            seen[ns++] = slot;
            cnt[slot & 15]++;
        }
        return *std::max_element(cnt, cnt + 16);
    };
    std::vector<int> gcost(static_cast<size_t>(S) * groups);
    int total = 0;
    for (int t = 0; t < S; ++t)
        for (int g = 0; g < groups; ++g) total += (gcost[static_cast<size_t>(t) * groups + g] = group_cost(t, g));
    // columns -> (t, g) occurrences are recomputed lazily by full rescans of
    // the affected lanes' groups; sizes here are small (S*lanes <= ~20k).
    auto rescan_lanes = [&](int La, int Lb) {
        int tot = total;
        const int ga = La / 16, gb = Lb / 16;
        const int ng = ga == gb ? 1 : 2;
        const int gs[2] = {ga, gb};
        for (int t = 0; t < S; ++t)
            for (int q = 0; q < ng; ++q) {
                const size_t id = static_cast<size_t>(t) * groups + gs[q];
                const int c = group_cost(t, gs[q]);
                tot += c - gcost[id];
                gcost[id] = c;
            }
        return tot;
    };
    uint64_t rng = 0x9E3779B97F4A7C15ull ^ static_cast<uint64_t>(n * 131 + lanes * 7 + S);
    auto rnd = [&]() {
        rng ^= rng << 13;
        rng ^= rng >> 7;
        rng ^= rng << 17;
        return rng;
    };
    auto urand = [&]() { return static_cast<double>(rnd() >> 11) * 0x1.0p-53; };
    // bounded host work: a slot move rescans the S*lanes step table once
    const long iters = std::max<long>(4000, std::min<long>(60000, 60000000L / (static_cast<long>(S) * lanes)));
    double T = 0.6;
    const double cool = std::pow(0.005 / T, 1.0 / static_cast<double>(iters));
    int best_total = total;
    std::vector<int> touched;
    std::vector<std::vector<int>> best_segs = lane_segs;
    std::vector<int32_t> best_pos = pos;
    for (long it = 0; it < iters; ++it, T *= cool) {
        const int kind = static_cast<int>(rnd() % 4);
        if (kind <= 1) {  // slot move / swap of one vector entry
            const int c = static_cast<int>(rnd() % n);
            const int slot = static_cast<int>(rnd() % NS);
            const int other = owner[slot];
            if (other == c) continue;
            const int old = pos[c];
            pos[c] = slot;
            owner[slot] = c;
            owner[old] = other;
            if (other >= 0) pos[other] = old;
            // only the (step, half-warp) groups that read c or other change
            touched.clear();
            for (size_t q = 0; q < col_at.size(); ++q)
                if (col_at[q] == c || (other >= 0 && col_at[q] == other))
                    touched.push_back(static_cast<int>((q / lanes) * groups + (q % lanes) / 16));
            std::sort(touched.begin(), touched.end());
            touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
            int nt = total;
            for (int id : touched) nt += group_cost(id / groups, id % groups) - gcost[id];
            const int d = nt - total;
            if (d <= 0 || urand() < std::exp(-d / T)) {
                for (int id : touched) gcost[id] = group_cost(id / groups, id % groups);
                total = nt;
            } else {
                pos[c] = old;
                owner[old] = c;
                owner[slot] = other;
                if (other >= 0) pos[other] = slot;
            }
        } else if (kind == 2) {  // reorder two segments within a lane
            const int L = static_cast<int>(rnd() % lanes);
            const int m = static_cast<int>(lane_segs[L].size());
            if (m < 2) continue;
            const int i = static_cast<int>(rnd() % m), j = static_cast<int>(rnd() % m);
            if (i == j) continue;
            std::swap(lane_segs[L][i], lane_segs[L][j]);
            lay_lane(L);
            const int nt = rescan_lanes(L, L);
            const int d = nt - total;
            if (d <= 0 || urand() < std::exp(-d / T)) {
                total = nt;
            } else {
                std::swap(lane_segs[L][i], lane_segs[L][j]);
                lay_lane(L);
                total = rescan_lanes(L, L);
            }
        } else {  // exchange (or move) segments between two lanes
            const int A = static_cast<int>(rnd() % lanes), B = static_cast<int>(rnd() % lanes);
            if (A == B || lane_segs[A].empty()) continue;
            const int ia = static_cast<int>(rnd() % lane_segs[A].size());
            const int sa = lane_segs[A][ia];
            const bool move = lane_segs[B].empty() || (rnd() & 1);
            if (move) {
                if (load[B] + seg_len[sa] > S) continue;
                const int ib = static_cast<int>(rnd() % (lane_segs[B].size() + 1));
                lane_segs[A].erase(lane_segs[A].begin() + ia);
                lane_segs[B].insert(lane_segs[B].begin() + ib, sa);
                lay_lane(A);
                lay_lane(B);
                const int nt = rescan_lanes(A, B);
                const int d = nt - total;
                if (d <= 0 || urand() < std::exp(-d / T)) {
                    total = nt;
                } else {
                    lane_segs[B].erase(lane_segs[B].begin() + ib);
                    lane_segs[A].insert(lane_segs[A].begin() + ia, sa);
                    lay_lane(A);
                    lay_lane(B);
                    total = rescan_lanes(A, B);
                }
            } else {
                const int ib = static_cast<int>(rnd() % lane_segs[B].size());
                const int sb = lane_segs[B][ib];
                if (load[A] - seg_len[sa] + seg_len[sb] > S || load[B] - seg_len[sb] + seg_len[sa] > S) continue;
                std::swap(lane_segs[A][ia], lane_segs[B][ib]);
                lay_lane(A);
                lay_lane(B);
                const int nt = rescan_lanes(A, B);
                const int d = nt - total;
                if (d <= 0 || urand() < std::exp(-d / T)) {
                    total = nt;
                } else {
                    std::swap(lane_segs[A][ia], lane_segs[B][ib]);
                    lay_lane(A);
                    lay_lane(B);
                    total = rescan_lanes(A, B);
                }
            }
        }
        if (total < best_total) {
            best_total = total;
            best_segs = lane_segs;
            best_pos = pos;
        }
    }
    lane_segs = best_segs;
    pos = best_pos;
}

GroupPlan build_group_plan(const Pattern& pat, int k, bool with_transpose, bool optimize) {
    GroupPlan gp;
    gp.k = k;
    if (const char* e = std::getenv("BC_SCHED_OPT")) optimize = optimize && std::atoi(e) != 0;
    const int n = k * pat.species;
    if (n > kMaxGroupRows) throw std::invalid_argument("group exceeds 2048 rows");
    gp.geo = choose_geometry(n);
    const int lanes = gp.geo.W * 32;
    gp.a = build_schedule(pat, k, lanes, false, optimize);
    if (with_transpose) gp.at = build_schedule(pat, k, lanes, true, optimize);
    gp.dpos.assign(n, -1);
    gp.didx.assign(n, -1);
    for (int c = 0; c < k; ++c)
        for (int r = 0; r < pat.species; ++r)
            if (pat.diag[r] >= 0) {
                gp.dpos[c * pat.species + r] = gp.a.vpos[c * pat.nnz + pat.diag[r]];
                gp.didx[c * pat.species + r] = c * pat.nnz + pat.diag[r];
            }
    return gp;
}

}  // namespace bc
