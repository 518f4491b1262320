// bc_plan.cpp -- see bc_plan.hpp.
#include "bc_plan.hpp"

#include <algorithm>
#include <numeric>
#include <stdexcept>

namespace bc {

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

Schedule build_schedule(const Pattern& pat, int k, int lanes, bool transpose) {
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
    Schedule sc;
    sc.steps = *std::max_element(load.begin(), load.end());
    sc.words.assign(static_cast<size_t>(sc.steps) * lanes, 0u);
    sc.vpos.assign(static_cast<size_t>(k) * nnz, -1);
    sc.vidx.assign(static_cast<size_t>(sc.steps) * lanes, 0);
    for (int L = 0; L < lanes; ++L) {
        std::sort(lane_segs[L].begin(), lane_segs[L].end(),
                  [&](int a, int b) { return segs[a].out < segs[b].out; });
        int t = 0;
        for (int idx : lane_segs[L]) {
            const Seg& sg = segs[idx];
            for (size_t q = 0; q < sg.ent.size(); ++q, ++t) {
                uint32_t w = static_cast<uint32_t>(sg.ent[q].second) |
                             (static_cast<uint32_t>(sg.out) << kColBits);
                if (q + 1 == sg.ent.size()) w |= kEndBit;
                sc.words[static_cast<size_t>(t) * lanes + L] = w;
                sc.vpos[sg.ent[q].first] = t * lanes + L;
                sc.vidx[static_cast<size_t>(t) * lanes + L] = sg.ent[q].first;
            }
        }
    }
    return sc;
}

GroupPlan build_group_plan(const Pattern& pat, int k, bool with_transpose) {
    GroupPlan gp;
    gp.k = k;
    const int n = k * pat.species;
    if (n > kMaxGroupRows) throw std::invalid_argument("group exceeds 2048 rows");
    gp.geo = choose_geometry(n);
    const int lanes = gp.geo.W * 32;
    gp.a = build_schedule(pat, k, lanes, false);
    if (with_transpose) gp.at = build_schedule(pat, k, lanes, true);
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
