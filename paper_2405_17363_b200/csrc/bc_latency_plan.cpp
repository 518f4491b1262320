// bc_latency_plan.cpp -- schedule of the latency-mode kernel (bc_latency.cuh).
//
// One thread per row; which thread runs which row is free (the reduction
// slot of row j is written to red[j] whoever computes it, the vector entries
// of a row live with its thread), so rows are sorted by length (BiCG: the
// longer of the row and its A^T row) and dealt to threads in that order: the
// longest rows share warp 0, the shortest the last warp, and every warp runs
// only as many gather/multiply-add steps as its own longest row.  A row's
// entries keep their CSR order (A^T: ascending source row), so every sum is
// the reference's.
//
// The cost is shared-memory wavefronts of the gathers (an LDS.64 per step per
// warp; per half-warp the largest number of distinct 8-byte slots in one of
// the 16 bank pairs).  All warps gather from the one copy the leader warp
// publishes; padding steps read one of 16 zero slots (one per bank pair), picked per
// half-warp step as the least-loaded bank.
//
// The gather region (doubles): [0, P) the vector (slot = row), [P, P + 16)
// zero slots, and for BiCG p~ at [P + 16, 2P + 16).
#include <algorithm>
#include <numeric>
#include <stdexcept>

#include "bc_plan.hpp"

namespace bc {

namespace {

// Smallest cap such that the m distinct items (each with its bank in copy 0
// and copy 1) can be placed with at most cap per bank; choice[i] = copy.
int match_items(const int (*banks)[2], int m, int* choice, int* load_out) {
    if (m == 0) {
        if (load_out) std::fill(load_out, load_out + 16, 0);
        return 0;
    }
    for (int cap = (m + 15) / 16; cap <= m; ++cap) {
        int load[16] = {0}, assign[16];
        std::fill(assign, assign + 16, -1);
        bool ok = true;
        for (int i = 0; i < m && ok; ++i) {
            bool vis[16] = {false};
            // augmenting path over banks
            struct Aug {
                const int (*bk)[2];
                int m, cap;
                int* load;
                int* assign;
                bool run(int it, bool* v) {
                    for (int r = 0; r < 2; ++r) {
                        const int b = bk[it][r];
                        if (v[b]) continue;
                        v[b] = true;
                        if (load[b] < cap) {
                            load[b]++;
                            assign[it] = b;
                            return true;
                        }
                        for (int i2 = 0; i2 < m; ++i2)
                            if (assign[i2] == b && run(i2, v)) {
                                assign[it] = b;
                                return true;
                            }
                    }
                    return false;
                }
            } aug{banks, m, cap, load, assign};
            ok = aug.run(i, vis);
        }
        if (ok) {
            for (int i = 0; i < m; ++i) choice[i] = banks[i][0] == assign[i] ? 0 : 1;
            if (load_out) std::copy(load, load + 16, load_out);
            return cap;
        }
    }
    return m;
}

struct Half {  // one half-warp's accesses at one step: entries (column, lane) and padding lanes
    int cols[16], lanes[16], n = 0;
    int pad[16], npad = 0;
};

}  // namespace

LatencySchedule build_latency_schedule(const Pattern& pat, int k, bool bicg, int threads) {
    LatencySchedule ls;
    const int s = pat.species, nnz = pat.nnz;
    const int n = k * s;
    ls.n = n;
    ls.P = static_cast<int>(padded_len(n));
    ls.T = std::max(threads, 32 * ((n + 31) / 32));
    const int P = ls.P, T = ls.T;
    // rows of one cell (CSR) and its A^T rows (ascending source row)
    std::vector<std::vector<int>> acol(s), aent(s), tsrc(s), tent(s);
    for (int i = 0; i < s; ++i)
        for (int e = pat.row_ptr[i]; e < pat.row_ptr[i + 1]; ++e) {
            acol[i].push_back(pat.col_idx[e]);
            aent[i].push_back(e);
            tsrc[pat.col_idx[e]].push_back(i);
            tent[pat.col_idx[e]].push_back(e);
        }
    auto len = [&](int j) {
        const int i = j % s;
        return std::max<int>(static_cast<int>(acol[i].size()), bicg ? static_cast<int>(tsrc[i].size()) : 0);
    };
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return len(a) > len(b); });
    ls.rowof.assign(T, -1);
    for (int t = 0; t < n; ++t) ls.rowof[t] = order[t];
    int lmax = 0;
    for (int j = 0; j < n; ++j) lmax = std::max(lmax, len(j));
    ls.lmax = lmax;
    ls.L = lmax <= 16 ? 16 : lmax <= 24 ? 24 : 32;
    if (lmax > 32) return ls;  // no kernel instance: the throughput kernels take this group
    ls.steps.assign(T, 0);
    for (int w = 0; w < T / 32; ++w) {
        int mx = 0;
        for (int l = 0; l < 32; ++l)
            if (ls.rowof[w * 32 + l] >= 0) mx = std::max(mx, len(ls.rowof[w * 32 + l]));
        for (int l = 0; l < 32; ++l) ls.steps[w * 32 + l] = mx;
    }
    const int zero0 = P, t0base = P + 16;
    ls.xslots = bicg ? 2 * P + 16 : P + 16;
    if (8 * ls.xslots > 65535) throw std::invalid_argument("latency schedule: gather offsets beyond 16 bits");


    // one matrix pass (A or A^T) of the schedule: fills vi/xo when given, returns modelled wavefronts
    auto pass = [&](bool transposed, std::vector<int32_t>* vi, std::vector<uint16_t>* xo) {
        const int base0 = transposed ? t0base : 0;
        int total = 0;
        for (int w = 0; w < T / 32; ++w) {
            const int steps = ls.steps[w * 32];
            for (int e = 0; e < steps; ++e)
                for (int h = 0; h < 2; ++h) {
                    Half hf;
                    for (int l = 16 * h; l < 16 * h + 16; ++l) {
                        const int t = w * 32 + l, j = ls.rowof[t];
                        const int i = j >= 0 ? j % s : 0, c = j >= 0 ? j / s : 0;
                        const auto& cl = transposed ? tsrc[i] : acol[i];
                        if (j < 0 || e >= static_cast<int>(cl.size())) {
                            hf.pad[hf.npad++] = l;
                            continue;
                        }
                        hf.cols[hf.n] = c * s + cl[e];  // gather index (row of the group)
                        hf.lanes[hf.n++] = l;
                    }
                    // distinct gather indices -> items
                    int items[16], nit = 0, item_of[16];
                    for (int q = 0; q < hf.n; ++q) {
                        int f = -1;
                        for (int u = 0; u < nit; ++u)
                            if (items[u] == hf.cols[q]) f = u;
                        if (f < 0) {
                            f = nit;
                            items[nit++] = hf.cols[q];
                        }
                        item_of[q] = f;
                    }
                    int banks[16][2], choice[16], load[16];
                    for (int u = 0; u < nit; ++u) banks[u][0] = banks[u][1] = (base0 + items[u]) & 15;
                    int cost = match_items(banks, nit, choice, load);
                    int zb = 0;  // padding lanes share the zero slot of the least-loaded bank
                    if (hf.npad) {
                        for (int b = 1; b < 16; ++b)
                            if (load[b] < load[zb]) zb = b;
                        cost = std::max(cost, load[zb] + 1);
                    }
                    total += cost;
                    if (!vi) continue;
                    for (int q = 0; q < hf.n; ++q) {
                        const int t = w * 32 + hf.lanes[q], j = ls.rowof[t], i = j % s, c = j / s;
                        const int g = items[item_of[q]];
                        const int slot = base0 + g;
                        const int ent = (transposed ? tent[i] : aent[i])[e];
                        (*vi)[static_cast<size_t>(e) * T + t] = c * nnz + ent;
                        (*xo)[static_cast<size_t>(e) * T + t] = static_cast<uint16_t>(8 * slot);
                    }
                    for (int q = 0; q < hf.npad; ++q) {
                        const int t = w * 32 + hf.pad[q];
                        (*vi)[static_cast<size_t>(e) * T + t] = -1;
                        (*xo)[static_cast<size_t>(e) * T + t] = static_cast<uint16_t>(8 * (zero0 + zb));
                    }
                }
        }
        return total;
    };
    auto model = [&]() { return pass(false, nullptr, nullptr) + (bicg ? pass(true, nullptr, nullptr) : 0); };

    ls.model_wavefronts = model();

    ls.rvi.assign(static_cast<size_t>(ls.L) * T, -1);
    ls.rxo.assign(static_cast<size_t>(ls.L) * T, static_cast<uint16_t>(8 * zero0));
    pass(false, &ls.rvi, &ls.rxo);
    if (bicg) {
        ls.tvi.assign(static_cast<size_t>(ls.L) * T, -1);
        ls.txo.assign(static_cast<size_t>(ls.L) * T, static_cast<uint16_t>(8 * zero0));
        pass(true, &ls.tvi, &ls.txo);
    }
    ls.didx.assign(P, -1);  // by row (every warp holds every row's vector entries)
    for (int j = 0; j < n; ++j)
        if (pat.diag[j % s] >= 0) ls.didx[j] = (j / s) * nnz + pat.diag[j % s];
    return ls;
}

}  // namespace bc
