// bc_plan.hpp -- host-side geometry and SpMV schedules for the fused
// Block-cells kernel.  Built once per (pattern, group size, team width) and
// cached in the context; the device copies are shared by every group.
#pragma once

#include <cstdint>
#include <map>
#include <vector>

namespace bc {

// Schedule word: gather index | output row << 12 | end-of-row << 31.
constexpr uint32_t kColBits = 12;
constexpr uint32_t kColMask = (1u << kColBits) - 1;
constexpr uint32_t kEndBit = 1u << 31;
constexpr int kMaxGroupRows = 2048;  // 12-bit row/col fields

struct Pattern {
    int32_t species = 0;
    int32_t nnz = 0;
    std::vector<int32_t> row_ptr, col_idx;
    std::vector<int32_t> diag;  // CSR index of the diagonal entry per row, -1 if absent
};

// Reduction geometry of one group:
// rows i of the group live in warp w = (i/32) % W, lane i%32, register slot
// j = (i/32) / W.  P = padded length (reduction.cpp:34-36), Q = max(1, P/32),
// W * R = Q.  The per-lane tree over j, the cross-warp tree over w and the
// xor-butterfly over lanes reproduce tree_reduce_in_place's order exactly.
struct Geometry {
    int n = 0;    // rows in the group (k * species)
    int P = 1;    // padded reduction length
    int Q = 1;    // 32-row columns in the padded tree
    int W = 1;    // warps per group (team)
    int R = 1;    // register slots per lane in the tree
    int RV = 1;   // register slots that can hold real rows
};

Geometry choose_geometry(int n);

// SpMV schedule over the team's W*32 lanes: rows (or columns, for the
// transpose) assigned longest-first to the least-loaded lane; each lane
// walks its rows back to back, entries in CSR (resp. ascending row) order.
struct Schedule {
    int steps = 0;                  // S
    std::vector<uint32_t> words;    // S * LW
    std::vector<int32_t> vpos;      // group value index -> smem slot (t*LW + L)
    std::vector<int32_t> vidx;      // smem slot -> group value index (0 for padding)
    int xslots = 0;                 // shared-memory slots of the gathered vector
    std::vector<int32_t> xpos;      // group row -> slot of its gathered value
    int conflict_cost = 0;          // modelled gather wavefronts per pass
};

// Schedule of the TMEM kernel (bc_tmem.cuh), one warp per group:
//  * every row is padded to an even number of steps with value-0.0 entries
//    that gather a dedicated always-zero slot (acc + 0*0 == acc exactly, as a
//    CSR sum started at +0.0 is never -0.0), so row ends only fall on odd
//    steps and the end test runs every other step;
//  * with two streams, a lane runs two rows at a time, interleaved step by
//    step (even steps: stream 0, odd: stream 1), so that its two dependent
//    DADD chains overlap; stream 0 rows then end on steps 2 mod 4, stream 1
//    rows on steps 3 mod 4;
//  * lane L's k-th row of stream s lands in Y[s*ystream + k*32 + L]
//    (conflict-free stores, no output index in the word); yslot maps rows to
//    those slots for the owner lanes;
//  * words are 16 bits: gather byte offset (slot*8); bit 15 of step 4c+2's
//    word flags a row ending on step 4c+3, bit 15 of step 4c's a row ending
//    on step 4c+1 (one stream) or 4c+2 (two streams); odd steps' words have it
//    clear, so both halves of a TMEM word decode to an address in one op;
//  * the gather vector has `copies` independent placements (bc_tmem_plan.cpp).
struct TmemSchedule {
    int steps = 0;                  // S, a multiple of 4
    std::vector<uint16_t> words;    // S * 32W
    std::vector<int32_t> vidx;      // S * 32W: group value index, -1 for padding (value 0.0)
    int copies = 1;                 // independent copies of the gather vector
    int xslots = 0;                 // gather-vector slots, all copies, incl. zero slots
    int zero_slot = 0;
    std::vector<int32_t> xpos;      // [copy][group row] -> gather slot
    int model_total = 0;            // modelled wavefronts per SpMV (gathers+stores+reads)
    std::vector<int32_t> yslot;     // group row -> Y slot (stream*ystream + k*32 + lane)
    int yslots = 0;
    int streams = 1;                // interleaved row streams per lane (1 or 2)
    int pair = 0;                   // BiCG: A rows on stream 0, A^T rows on stream 1 (xpos: [copy][2n],
                                    // columns n + i gather p~; yslot: [2n], A^T output j at n + j)
    int ystream = 32;               // Y slots per stream
    int team = 1;                   // warps per group W: words/vidx are [S][32W], Y lane-major over 32W lanes
    int conflict_cost = 0;          // modelled gather wavefronts per pass
};

// Latency-mode schedule (bc_latency_plan.cpp, bc_latency.cuh): one SpMV row
// per thread, rows dealt to threads longest first, per-warp step counts,
// gather offsets into the warp's private copy of the vector.
struct LatencySchedule {
    int n = 0, P = 0, T = 0;        // rows, tree slots, threads (whole warps covering n)
    int lmax = 0, L = 0;            // longest row, padded step count (kernel template: 16, 24, 32)
    int xslots = 0;                 // doubles of one warp's gather region
    int model_wavefronts = 0;       // modelled gather wavefronts of one SpMV (A and A^T), all warps
    std::vector<int32_t> rowof;     // [T] group row of thread t, -1 none
    std::vector<int32_t> steps;     // [T] steps of thread t's warp
    std::vector<int32_t> rvi, tvi;  // [L][T] group value index, -1 padding (A, A^T)
    std::vector<uint16_t> rxo, txo; // [L][T] byte offsets of the gathers
    std::vector<int32_t> didx;      // [P] group value index of row j's diagonal, -1 none
};
// threads: the kernel instance's thread count (>= 32 * ceil(n / 32))
LatencySchedule build_latency_schedule(const Pattern& pat, int k, bool bicg, int threads);

struct GroupPlan {
    int k = 1;
    Geometry geo;
    Schedule a, at;              // A and A^T (at only built for BiCG)
    std::vector<int32_t> dpos;   // per group row: smem slot of the diagonal value, -1 if none
    std::vector<int32_t> didx;   // per group row: group value index of the diagonal, -1 if none
    // device copies
    uint32_t* d_words = nullptr;
    uint32_t* d_twords = nullptr;
    int32_t* d_vpos = nullptr;
    int32_t* d_tvpos = nullptr;
    int32_t* d_dpos = nullptr;
    int32_t* d_vidx = nullptr;
    int32_t* d_tvidx = nullptr;
    int32_t* d_didx = nullptr;
    int32_t* d_xpos = nullptr;
    int32_t* d_txpos = nullptr;
    // TMEM-kernel schedules, built on demand per team width (1, 2, 4 warps per group)
    std::map<int, struct TmemPlan> tmem;
};

struct TmemPlan {
    TmemSchedule tm;
    uint16_t* d_words = nullptr;
    int32_t* d_vidx = nullptr;
    int lane_rv = 0;                  // RV the lane tables below were built for
    uint32_t* d_xy = nullptr;
    uint32_t* d_x1 = nullptr;
    uint32_t* d_xyT = nullptr;        // pair schedules: p~ / A^T tables
    uint32_t* d_x1T = nullptr;
};

TmemSchedule build_tmem_schedule(const Pattern& pat, int k, bool pair = false, int team = 1,
                                  bool optimize = true, bool quick = false);

Schedule build_schedule(const Pattern& pat, int k, int lanes, bool transpose, bool optimize = true);
GroupPlan build_group_plan(const Pattern& pat, int k, bool with_transpose, bool optimize = true);
int gather_cost(int steps, int lanes, const std::vector<uint32_t>& words);

inline int64_t padded_len(int64_t n) {
    if (n <= 1) return 1;
    int64_t p = 1;
    while (p < n) p <<= 1;
    return p;
}

}  // namespace bc
