// spmm_blocked.cu -- column-blocked SpMM: C = A * B consumed one column
// block of B at a time (a rank's SpMM runs on each B row shard
// as it lands from the all-gather instead of after the whole gather).
//
// Exactness.  The reference accumulates C[i,f] over row i's entries in CSR
// order (src/kernels.cpp:217-226), HubSplit heavy rows over 2048-nnz pieces
// that are then summed in piece order (src/kernels.cpp:284-332).  Columns
// are sorted within a row, so a row's (or piece's) entries whose columns fall
// in blocks [c_0, c_1), [c_1, c_2), ... are consecutive runs in that same
// order.  Every row / piece is a "segment" with an f64 state slot: block b
// continues each segment's chain from its slot (spmm_seg_kernel CARRY mode)
// over the segment's run in block b, and the last block folds the slots per
// row in order (0.0 + s_0 + s_1 ...: the hub reduce; a single-segment row is
// 0.0 + s = s, the state itself never being -0.0).  Processing blocks in
// ascending order therefore yields the unblocked result bit for bit, for
// any cut positions.
//
// Cost: the state (segments x F doubles) is written by every block a segment
// has entries in but its last, and read by every such block but its first
// (slot flags, spmm_kernels.cuh); single-segment rows are rounded into C by
// their last block, so only hub rows and empty rows go through the fold --
// worth it when B's exchange is long against the SpMM (Products-shape
// shards), not for an L2-resident B.
#include "engine.hpp"
#include "spmm_kernels.cuh"

#include <algorithm>
#include <memory>
#include <numeric>
#include <vector>

namespace asb {

namespace {

__global__ void blocked_fold_kernel(const std::uint32_t* __restrict__ red_row,
                                    const std::uint32_t* __restrict__ red_first,
                                    const std::uint32_t* __restrict__ red_count, std::uint64_t n_red,
                                    const double* __restrict__ state, float* __restrict__ c, std::uint32_t f) {
    const std::uint64_t total = n_red * f;
    for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; i < total;
         i += std::uint64_t(gridDim.x) * blockDim.x) {
        const std::uint64_t r = i / f, t = i - r * f;
        const std::uint64_t first = red_first[r], cnt = red_count[r];
        double s = 0.0;
        for (std::uint64_t p = 0; p < cnt; ++p) s = __dadd_rn(s, state[(first + p) * f + t]);
        c[std::uint64_t(red_row[r]) * f + t] = float(s);
    }
}

template <int VEC, int LPR, int NCH>
void launch_carry(const SegArgs& a, bool has_val, cudaStream_t s) {
    constexpr int GPW = 32 / LPR;
    constexpr unsigned kWarps = 4;
    const std::uint64_t blocks = (a.n_items + kWarps * GPW - 1) / (kWarps * GPW);
    if (!blocks) return;
    const unsigned nt = kWarps * 32;
    constexpr int U = unroll_for(VEC, NCH), MR = maxreg_for(VEC, NCH);
    if (has_val)
        spmm_seg_kernel<VEC, LPR, NCH, true, true, U, MR, false, false, false, true>
            <<<unsigned(blocks), nt, seg_smem(nt), s>>>(a);
    else
        spmm_seg_kernel<VEC, LPR, NCH, false, true, U, MR, false, false, false, true>
            <<<unsigned(blocks), nt, seg_smem(nt), s>>>(a);
    check_launch("spmm_seg_kernel<carry>");
}

template <int VEC>
void launch_carry_vec(const SegArgs& a, bool has_val, std::uint32_t lanes, cudaStream_t s) {
    if (lanes <= 1) launch_carry<VEC, 1, 1>(a, has_val, s);
    else if (lanes <= 2) launch_carry<VEC, 2, 1>(a, has_val, s);
    else if (lanes <= 4) launch_carry<VEC, 4, 1>(a, has_val, s);
    else if (lanes <= 8) launch_carry<VEC, 8, 1>(a, has_val, s);
    else if (lanes <= 16) launch_carry<VEC, 16, 1>(a, has_val, s);
    else if (lanes <= 32) launch_carry<VEC, 32, 1>(a, has_val, s);
    else if (lanes <= 64) launch_carry<VEC, 32, 2>(a, has_val, s);
    else if (lanes <= 128) launch_carry<VEC, 32, 4>(a, has_val, s);
    else launch_carry<VEC, 32, 8>(a, has_val, s);
}

}  // namespace

struct BlockedPlan {
    Graph* g = nullptr;
    std::uint32_t n_blocks = 0;
    std::uint64_t f_tile = 64;
    std::uint64_t n_slots = 0;
    struct Block {
        std::uint64_t n = 0;
        DevBuf<std::uint32_t> row, len, slot;
        DevBuf<std::uint64_t> e0;
    };
    std::vector<Block> blocks;
    std::uint64_t n_red = 0;
    DevBuf<std::uint32_t> red_row, red_first, red_count;
    DevBuf<double> state;
    std::uint64_t state_f = 0;
};

// Segments: every row (Baseline / RowParallel: the row's chain) or, under
// HubSplit, the 2048-nnz pieces of rows of degree >= hub_threshold; slots
// numbered row by row.  Per block, the segments with entries in it.
BlockedPlan* blocked_plan_create(Graph& g, const as_variant* v, const std::uint64_t* cuts,
                                 std::uint32_t n_blocks) {
    if (n_blocks == 0) throw InvalidArgument("spmm_blocked: n_blocks must be > 0");
    if (cuts[0] != 0 || cuts[n_blocks] != g.n_cols)
        throw InvalidArgument("spmm_blocked: column cuts must run from 0 to n_cols");
    for (std::uint32_t b = 0; b < n_blocks; ++b)
        if (cuts[b + 1] < cuts[b]) throw InvalidArgument("spmm_blocked: column cuts must be non-decreasing");
    as_variant var = v ? *v : default_variant();
    if (!v) var.mapping = AS_MAP_BASELINE;
    if (var.op != AS_OP_SPMM) throw InvalidArgument("spmm_blocked: spmm variant required");
    check_variant(var);
    DeviceGuard dg(g.device);
    auto p = std::make_unique<BlockedPlan>();
    p->g = &g;
    p->n_blocks = n_blocks;
    p->f_tile = var.f_tile;
    std::vector<std::uint32_t> colind(g.nnz);
    if (g.nnz) {
        ASB_CUDA(cudaMemcpyAsync(colind.data(), g.colind.get(), g.nnz * 4, cudaMemcpyDeviceToHost, g.stream));
        ASB_CUDA(cudaStreamSynchronize(g.stream));
    }
    const bool hub = var.mapping == AS_MAP_HUBSPLIT;
    std::vector<std::vector<std::uint32_t>> brow(n_blocks), blen(n_blocks), bslot(n_blocks);
    std::vector<std::vector<std::uint64_t>> be0(n_blocks);
    std::vector<std::uint32_t> rrow, rfirst, rcount;
    std::uint64_t slots = 0;
    for (std::uint64_t i = 0; i < g.n_rows; ++i) {
        const std::uint64_t e0 = g.h_rowptr[i], e1 = g.h_rowptr[i + 1];
        const std::uint64_t step = hub && e1 - e0 >= var.hub_threshold ? kHubNnzChunk : std::max<std::uint64_t>(e1 - e0, 1);
        const std::uint64_t nseg = e1 > e0 ? (e1 - e0 + step - 1) / step : 0;
        // the fold sums multi-segment rows and zero-fills empty ones; a
        // single-segment row is rounded into C by its last block
        if (nseg != 1) {
            rrow.push_back(std::uint32_t(i));
            rfirst.push_back(std::uint32_t(slots));
            rcount.push_back(std::uint32_t(nseg));
        }
        for (std::uint64_t sg = 0; sg < nseg; ++sg, ++slots) {
            const std::uint64_t s0 = e0 + sg * step, s1 = std::min(e1, s0 + step);
            const std::uint32_t* c0 = colind.data() + s0;
            const std::uint32_t* c1 = colind.data() + s1;
            const std::uint32_t* lo = c0;
            std::uint32_t first = kCarryFirst;
            std::int64_t last_b = -1;
            for (std::uint32_t b = 0; b < n_blocks; ++b) {
                const std::uint32_t* hi = std::lower_bound(lo, c1, cuts[b + 1]);
                if (hi > lo) {
                    brow[b].push_back(std::uint32_t(i));
                    be0[b].push_back(std::uint64_t(lo - colind.data()));
                    blen[b].push_back(std::uint32_t(hi - lo));
                    bslot[b].push_back(std::uint32_t(slots) | first);
                    first = 0;
                    last_b = b;
                }
                lo = hi;
            }
            if (nseg == 1 && last_b >= 0) bslot[std::size_t(last_b)].back() |= kCarryFinal;
        }
    }
    if (slots > kCarrySlotMask) throw InvalidArgument("spmm_blocked: too many segments");
    p->n_slots = slots;
    auto up = [&](auto& d, const auto& h) {
        using T = typename std::decay_t<decltype(h)>::value_type;
        d.alloc(std::max<std::size_t>(h.size(), 1));
        if (!h.empty())
            ASB_CUDA(cudaMemcpyAsync(d.get(), h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, g.stream));
    };
    p->blocks.resize(n_blocks);
    for (std::uint32_t b = 0; b < n_blocks; ++b) {
        // longest runs first (LPT), as the hub plan orders its pieces
        std::vector<std::uint32_t> perm(brow[b].size());
        std::iota(perm.begin(), perm.end(), 0u);
        std::stable_sort(perm.begin(), perm.end(),
                         [&](std::uint32_t x, std::uint32_t y) { return blen[b][x] > blen[b][y]; });
        auto apply = [&](auto& vec) {
            auto tmp = vec;
            for (std::size_t k = 0; k < perm.size(); ++k) vec[k] = tmp[perm[k]];
        };
        apply(brow[b]);
        apply(be0[b]);
        apply(blen[b]);
        apply(bslot[b]);
        auto& B = p->blocks[b];
        B.n = brow[b].size();
        up(B.row, brow[b]);
        up(B.e0, be0[b]);
        up(B.len, blen[b]);
        up(B.slot, bslot[b]);
    }
    p->n_red = rrow.size();
    up(p->red_row, rrow);
    up(p->red_first, rfirst);
    up(p->red_count, rcount);
    ASB_CUDA(cudaStreamSynchronize(g.stream));
    return p.release();
}

void blocked_plan_run(BlockedPlan& p, std::uint32_t block, const float* vals, const float* b, std::uint64_t b_rows,
                      std::uint64_t f, float* c, cudaStream_t s) {
    Graph& g = *p.g;
    if (block >= p.n_blocks) throw InvalidArgument("spmm_blocked: block out of range");
    if (b_rows != g.n_cols) throw InvalidArgument("spmm: a.n_cols != b.n_rows");
    if (f == 0 || g.n_rows == 0) return;
    DeviceGuard dg(g.device);
    if (block == 0) {
        if (p.state_f != f || p.state.size() < std::max<std::uint64_t>(p.n_slots * f, 1)) {
            p.state.alloc(std::max<std::uint64_t>(p.n_slots * f, 1));
            p.state_f = f;
        }
        // no clearing: every slot's first block starts its chain from 0.0
    } else if (p.state_f != f) {
        throw InvalidArgument("spmm_blocked: blocks of one product need the same F, starting at block 0");
    }
    const auto& B = p.blocks[block];
    if (B.n) {
        const bool vec = f % 4 == 0 && (reinterpret_cast<std::uintptr_t>(b) & 15) == 0;
        const int v = vec ? 4 : 1;
        std::uint64_t tw = effective_tile(p.f_tile, f);
        if (vec) tw = (tw + 3) / 4 * 4;
        tw = std::min<std::uint64_t>(tw, std::uint64_t(32 * 8 * v));
        tw = std::max<std::uint64_t>(tw, 1);
        const std::uint32_t n_tiles = std::uint32_t((f + tw - 1) / tw);
        const std::uint32_t lanes = std::uint32_t((tw + v - 1) / v);
        SegArgs a{};
        a.rowptr = g.rowptr.get();
        a.colind = g.colind.get();
        a.val = vals;
        a.b = b;
        a.c = c;
        a.scratch = p.state.get();
        a.piece_row = B.row.get();
        a.piece_e0 = B.e0.get();
        a.piece_len = B.len.get();
        a.piece_slot = B.slot.get();
        a.finite = nullptr;  // all-F2F widening: no per-block operand scan
        a.n_items = B.n * n_tiles;
        a.n_tiles = n_tiles;
        a.f = std::uint32_t(f);
        a.tile_w = std::uint32_t(tw);
        a.off32 = std::uint64_t(g.n_cols) * f < (std::uint64_t(1) << 32);
        a.keep_b = std::uint64_t(g.n_cols) * f * 4 <= kKeepMaxBytes;
        a.n_rows = g.n_rows;
        a.n_cols = g.n_cols;
        a.nnz = g.nnz;
        if (vec) launch_carry_vec<4>(a, vals != nullptr, lanes, s);
        else launch_carry_vec<1>(a, vals != nullptr, lanes, s);
    }
    if (block + 1 == p.n_blocks && p.n_red) {
        const std::uint64_t total = p.n_red * f;
        const unsigned blocks = unsigned(std::min<std::uint64_t>((total + 255) / 256, std::uint64_t(g.sms) * 32));
        blocked_fold_kernel<<<blocks, 256, 0, s>>>(p.red_row.get(), p.red_first.get(), p.red_count.get(), p.n_red,
                                                   p.state.get(), c, std::uint32_t(f));
        check_launch("blocked_fold_kernel");
    }
}

void blocked_plan_destroy(BlockedPlan* p) { delete p; }

Graph& blocked_plan_graph(BlockedPlan& p) { return *p.g; }

}  // namespace asb
