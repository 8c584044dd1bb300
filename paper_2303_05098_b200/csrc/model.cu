// Decision-tree / random-forest inference on the device (model.cpp:202-228)
// and the fused ML tuner (tuners.cpp:92-114): features -> predict ->
// format_feasible -> CSR fallback, with no host round trip until the final
// 8-int outcome.
#include <atomic>
#include <string>
#include <vector>

#include "features.cuh"

#include "forest.cuh"

namespace sob {

namespace {

constexpr int kPB = 256;

struct ForestView {
    int kind, n_trees;
    const PackedNode* nodes;
    const int64_t* root;
    const PackedNode* bnodes;
    const int32_t* broot;
};

ForestView view(const so_forest& f) {
    return ForestView{f.f.kind, f.f.n_trees, f.f.nodes.get(), f.f.root.get(), f.f.bnodes.get(), f.f.broot.get()};
}

// features_to_row (features.cpp:155-166)
__device__ __forceinline__ void to_row(const so_feature_vector& f, double* row) {
    row[0] = double(f.nrows);
    row[1] = double(f.ncols);
    row[2] = double(f.nnz);
    row[3] = f.avg_nnz_per_row;
    row[4] = f.density;
    row[5] = double(f.max_nnz_per_row);
    row[6] = double(f.min_nnz_per_row);
    row[7] = f.nnz_row_spread;
    row[8] = double(f.ndiags);
    row[9] = double(f.ntrue_diags);
}

// Root-to-leaf walk: x[feature] <= threshold goes left (model.cpp:202-213).
__device__ __forceinline__ int walk(const ForestView& f, int t, const double* row) {
    PackedNode nd = f.nodes[f.root[t]];
    while (nd.feature != -1) nd = f.nodes[row[nd.feature] <= nd.threshold ? nd.left : nd.right];
    return nd.cls;
}

// One CTA per feature row: thread per tree, integer votes in shared memory,
// argmax with strict '>' so ties go to the lowest FormatId (model.cpp:215-228).
__device__ int predict_block(const ForestView& f, const double* row, int trees) {
    __shared__ int votes[8];
    if (threadIdx.x < 8) votes[threadIdx.x] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < trees; t += blockDim.x) atomicAdd(&votes[walk(f, t, row)], 1);
    __syncthreads();
    int best = 0;
    for (int c = 1; c < 6; ++c)
        if (votes[c] > votes[best]) best = c;
    __syncthreads();
    return best;
}

__global__ void __launch_bounds__(kPB) predict_rows_kernel(ForestView f, const double* __restrict__ rows, int64_t n,
                                                           int32_t* __restrict__ out) {
    __shared__ double row[10];
    for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
        if (threadIdx.x < 10) row[threadIdx.x] = rows[r * 10 + threadIdx.x];
        __syncthreads();
        const int best = predict_block(f, row, f.n_trees);  // predict_forest votes over every tree
        if (threadIdx.x == 0) out[r] = best;
        __syncthreads();
    }
}

// Warp-cooperative walk over the blocked layout (forest.cuh).  Lane j holds
// slot j of the current block and evaluates that node's own comparison
// (x[feature] <= threshold, model.cpp:206-209), so following the path through
// the block costs one shuffle per level; a leaf is encoded as -1 - class.
// Two trees are walked together so their block fetches overlap.
__device__ __forceinline__ int node_step(const PackedNode& nd, const double* row) {
    if (nd.feature == -1) return -1 - nd.cls;
    return row[nd.feature] <= nd.threshold ? nd.left : nd.right;
}

__device__ __forceinline__ void walk_warp2(const ForestView& f, int t0, int t1, const double* row, int& c0, int& c1) {
    const unsigned lane = threadIdx.x & 31u;
    int cur[2] = {f.broot[t0], t1 >= 0 ? f.broot[t1] : -1};
    int res[2] = {-1, t1 >= 0 ? -1 : 0};
    bool live[2] = {true, t1 >= 0};
    while (live[0] || live[1]) {
        int go[2] = {0, 0};
        int blk[2] = {0, 0};
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            if (live[k]) {
                blk[k] = cur[k] / kTreeBlock;
                const PackedNode nd = f.bnodes[int64_t(blk[k]) * kTreeBlock + lane];
                go[k] = node_step(nd, row);
            }
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            if (!live[k]) continue;
            while (true) {
                const int nxt = __shfl_sync(0xffffffffu, go[k], cur[k] - blk[k] * kTreeBlock);
                if (nxt < 0) {
                    res[k] = -1 - nxt;
                    live[k] = false;
                    break;
                }
                cur[k] = nxt;
                if (nxt / kTreeBlock != blk[k]) break;
            }
        }
    }
    c0 = res[0];
    c1 = res[1];
}

// One CTA of kTB threads for one feature row: a warp per pair of trees over
// the blocked layout, votes in shared memory, argmax with strict '>' so ties
// go to the lowest FormatId (model.cpp:215-228).
constexpr int kTB = 1024;
__device__ int predict_block_warps(const ForestView& f, const double* row, int trees) {
    __shared__ int votes[8];
    if (threadIdx.x < 8) votes[threadIdx.x] = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int t = 2 * warp; t < trees; t += 2 * nwarps) {
        int c0, c1;
        walk_warp2(f, t, t + 1 < trees ? t + 1 : -1, row, c0, c1);
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(&votes[c0], 1);
            if (t + 1 < trees) atomicAdd(&votes[c1], 1);
        }
    }
    __syncthreads();
    int best = 0;
    for (int c = 1; c < 6; ++c)
        if (votes[c] > votes[best]) best = c;
    __syncthreads();
    return best;
}

// The single-row latency path (tune_predict_kernel's blocked warp walk) over
// n host-given rows, one CTA of kTB threads per row: so_predict and the
// parity tests of the fused tuner's predict step run exactly this code.
__global__ void __launch_bounds__(kTB) predict_rows_blocked_kernel(ForestView f, const double* __restrict__ rows,
                                                                   int64_t n, int32_t* __restrict__ out) {
    __shared__ double row[10];
    for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
        if (threadIdx.x < 10) row[threadIdx.x] = rows[r * 10 + threadIdx.x];
        __syncthreads();
        const int best = predict_block_warps(f, row, f.kind == 0 ? 1 : f.n_trees);
        if (threadIdx.x == 0) out[r] = best;
        __syncthreads();
    }
}

struct CapCfg {
    int64_t kh_override;
    double max_padding_factor;
    int64_t max_padded_entries;
};

__device__ int64_t d_padded_entry_cap(const CapCfg& c, int64_t nnz) {  // formats.cpp:348-355
    if (c.max_padded_entries > 0) return c.max_padded_entries;
    const double cap = c.max_padding_factor * double(nnz);
    if (cap >= 9223372036854775807.0) return INT64_MAX;
    return int64_t(cap);
}

// tuners.cpp:26-45 (row_to_features already applied: integer fields)
__device__ bool d_feasible(int target, const so_feature_vector& f, const CapCfg& c) {
    const int64_t cap = d_padded_entry_cap(c, f.nnz);
    switch (target) {
        case SO_COO:
        case SO_CSR:
            return true;
        case SO_DIA:
            return f.ndiags * f.nrows <= cap;
        case SO_ELL:
            return f.max_nnz_per_row * f.nrows <= cap;
        case SO_HYB: {
            int64_t kh = c.kh_override > 0 ? c.kh_override
                         : (f.nrows <= 0 || f.nnz <= 0) ? 0
                                                         : (f.nnz + f.nrows - 1) / f.nrows;
            const int64_t w = kh < f.max_nnz_per_row ? kh : f.max_nnz_per_row;
            return w * f.nrows <= cap;
        }
        case SO_HDC:
            return f.ntrue_diags * f.nrows <= cap;
    }
    return false;
}

__global__ void __launch_bounds__(kTB) tune_predict_kernel(ForestView f, const FeatState* __restrict__ st, CapCfg cfg,
                                                           int active, so_tune_outcome* __restrict__ out) {
    pdl_enter();
    __shared__ double row[10];
    if (threadIdx.x == 0) to_row(st->out, row);
    __syncthreads();
    // kind tree evaluates trees.front() only (tuners.cpp:103-105)
    int chosen = predict_block_warps(f, row, f.kind == 0 ? 1 : f.n_trees);
    if (threadIdx.x == 0) {
        // the model saw row_to_features(features_to_row(f)); feasibility uses
        // the integer fields, identical for counts < 2^53
        const so_feature_vector& fv = st->out;
        int fallback = 0;
        if (!d_feasible(chosen, fv, cfg)) {
            chosen = SO_CSR;
            fallback = 1;
        }
        out->chosen = chosen;
        out->source = f.kind == 0 ? 1 : 2;
        out->switched = chosen != active;
        out->fallback_csr = fallback;
        out->features = fv;
        // T_FE: first feature kernel's start -> finalize; T_PRED: finalize ->
        // the vote (includes the launch gap between the two kernels)
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        out->feature_time_seconds = double(st->t_end - st->t_begin) * 1e-9;
        out->predict_time_seconds = double(t - st->t_end) * 1e-9;
    }
}

}  // namespace

so_forest* forest_upload(int32_t kind, int32_t n_trees, const int64_t* node_off, const int32_t* feature,
                         const double* threshold, const int32_t* left, const int32_t* right, const int32_t* cls,
                         cudaStream_t s) {
    if (n_trees < 1) fail(SO_INVALID_INPUT, "forest has no trees");
    const int64_t nn = node_off[n_trees];
    std::vector<int32_t> gl(nn), gr(nn), fe(nn), cl(nn);
    std::vector<int64_t> root(n_trees);
    for (int t = 0; t < n_trees; ++t) {
        const int64_t b = node_off[t], e = node_off[t + 1];
        if (e <= b) fail(SO_INVALID_INPUT, "tree with no nodes");
        root[t] = b;
        for (int64_t i = b; i < e; ++i) {
            fe[i] = feature[i];
            cl[i] = cls[i];
            if (feature[i] == -1) {
                gl[i] = gr[i] = -1;
                if (cls[i] < 0 || cls[i] > 5) fail(SO_MALFORMED_MODEL, "leaf class outside 0..5");
            } else {
                if (feature[i] < 0 || feature[i] > 9) fail(SO_MALFORMED_MODEL, "feature index outside 0..9");
                if (left[i] < 0 || left[i] >= e - b || right[i] < 0 || right[i] >= e - b)
                    fail(SO_MALFORMED_MODEL, "dangling child reference");
                gl[i] = int32_t(b + left[i]);
                gr[i] = int32_t(b + right[i]);
            }
        }
    }
    // every node reachable exactly once from the root (model.cpp:151-176):
    // rules out cycles before anything walks the tree on the device
    for (int t = 0; t < n_trees; ++t) {
        const int64_t b = node_off[t], e = node_off[t + 1];
        std::vector<char> seen(size_t(e - b), 0);
        std::vector<int64_t> stack{0};
        seen[0] = 1;
        int64_t visited = 0;
        while (!stack.empty()) {
            const int64_t id = stack.back();
            stack.pop_back();
            ++visited;
            if (feature[b + id] == -1) continue;
            for (int64_t ch : {int64_t(left[b + id]), int64_t(right[b + id])}) {
                if (seen[size_t(ch)]) fail(SO_MALFORMED_MODEL, "node " + std::to_string(ch) + " referenced more than once");
                seen[size_t(ch)] = 1;
                stack.push_back(ch);
            }
        }
        if (visited != e - b) fail(SO_MALFORMED_MODEL, "unreachable nodes in tree");
    }
    auto* f = new so_forest();
    static std::atomic<uint64_t> next_uid{1};
    f->uid = next_uid++;
    SOB_CUDA(cudaGetDevice(&f->device));
    ForestDev& d = f->f;
    d.kind = kind;
    d.n_trees = n_trees;
    d.n_nodes = nn;
    auto up = [&](auto& buf, const auto* src, int64_t n) {
        buf.alloc(n, s);
        SOB_CUDA(cudaMemcpyAsync(buf.get(), src, sizeof(*src) * size_t(n), cudaMemcpyHostToDevice, s));
    };
    up(d.feature, fe.data(), nn);
    up(d.left, gl.data(), nn);
    up(d.right, gr.data(), nn);
    up(d.cls, cl.data(), nn);
    up(d.threshold, threshold, nn);
    up(d.root, root.data(), n_trees);
    std::vector<PackedNode> packed(static_cast<size_t>(nn));
    for (int64_t i = 0; i < nn; ++i)
        packed[size_t(i)] = PackedNode{threshold[i], fe[size_t(i)], gl[size_t(i)], gr[size_t(i)], cl[size_t(i)], {0, 0}};
    up(d.nodes, packed.data(), nn);
    // blocked layout: depth-5 subtrees, BFS inside each 32-slot block
    std::vector<PackedNode> blk;
    std::vector<int32_t> broot(size_t(n_trees), 0);
    struct Pending {
        int64_t node;  // flat (global) node id
        int64_t parent_slot;
        bool left;
    };
    for (int t = 0; t < n_trees; ++t) {
        std::vector<Pending> q{{root[size_t(t)], -1, false}};
        for (size_t qi = 0; qi < q.size(); ++qi) {
            const Pending p = q[qi];
            const int64_t B = int64_t(blk.size()) / kTreeBlock;
            if (B * kTreeBlock + kTreeBlock > INT32_MAX) fail(SO_INVALID_INPUT, "forest too large");
            blk.resize(blk.size() + kTreeBlock, PackedNode{0.0, -1, -1, -1, 0, {0, 0}});
            const int32_t bslot = int32_t(B * kTreeBlock);
            if (p.parent_slot < 0)
                broot[size_t(t)] = bslot;
            else if (p.left)
                blk[size_t(p.parent_slot)].left = bslot;
            else
                blk[size_t(p.parent_slot)].right = bslot;
            int64_t local[kTreeBlock - 1];
            for (auto& v : local) v = -1;
            local[0] = p.node;
            for (int i = 0; i < kTreeBlock - 1; ++i) {
                const int64_t nd = local[i];
                if (nd < 0) continue;
                const int64_t slot = B * kTreeBlock + i;
                blk[size_t(slot)] = PackedNode{threshold[nd], fe[size_t(nd)], -1, -1, cl[size_t(nd)], {0, 0}};
                if (fe[size_t(nd)] == -1) continue;
                for (int side = 0; side < 2; ++side) {
                    const int64_t child = side == 0 ? gl[size_t(nd)] : gr[size_t(nd)];
                    const int ci = 2 * i + 1 + side;
                    if (ci < kTreeBlock - 1) {
                        local[ci] = child;
                        (side == 0 ? blk[size_t(slot)].left : blk[size_t(slot)].right) = int32_t(B * kTreeBlock + ci);
                    } else {
                        q.push_back(Pending{child, slot, side == 0});
                    }
                }
            }
        }
    }
    up(d.bnodes, blk.data(), int64_t(blk.size()));
    up(d.broot, broot.data(), n_trees);
    SOB_CUDA(cudaStreamSynchronize(s));  // host staging vectors go out of scope
    return f;
}

void predict_rows(const so_forest& f, const double* rows_dev, int64_t n, int32_t* out_dev, cudaStream_t s) {
    if (n <= 0) return;
    predict_rows_kernel<<<grid_for(n * kPB, kPB, 8), kPB, 0, s>>>(view(f), rows_dev, n, out_dev);
    SOB_LAUNCH("predict_rows_kernel");
}

void predict_rows_blocked(const so_forest& f, const double* rows_dev, int64_t n, int32_t* out_dev, cudaStream_t s) {
    if (n <= 0) return;
    predict_rows_blocked_kernel<<<grid_for(n * kTB, kTB, 2), kTB, 0, s>>>(view(f), rows_dev, n, out_dev);
    SOB_LAUNCH("predict_rows_blocked_kernel");
}

void enqueue_tune_predict(const so_forest& f, const FeatState* st, const so_conversion_config& cfg, int active,
                          so_tune_outcome* out_dev, cudaStream_t s) {
    CapCfg c{cfg.kh_override, cfg.max_padding_factor, cfg.max_padded_entries};
    launch_pdl(tune_predict_kernel, dim3(1), dim3(kTB), 0, s, view(f), st, c, active, out_dev);
    SOB_LAUNCH("tune_predict_kernel");
}

}  // namespace sob
