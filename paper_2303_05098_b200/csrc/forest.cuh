// Device-resident forest (SoA node arrays), shared by model.cu and capi.cu.
#pragma once

#include "common.cuh"

namespace sob {

// One node in one 32-byte record: a tree walk costs one dependent round trip
// per level instead of three.
struct alignas(16) PackedNode {
    double threshold;
    int32_t feature;  // -1: leaf
    int32_t left;     // global node ids
    int32_t right;
    int32_t cls;
    int32_t pad[2];
};

// Blocked layout for single-row (latency-bound) prediction: every tree is cut
// into depth-5 subtrees, each stored BFS-ordered in one 32-slot block (31
// nodes + pad) whose 32 records one warp fetches with a single coalesced 1 KB
// load; a child id (global slot = block*32 + local) inside the same block is
// followed through warp shuffles, so a depth-16 walk costs ~4 dependent loads
// instead of 16.
constexpr int kTreeBlock = 32;

struct ForestDev {
    DBuf<PackedNode> nodes;
    DBuf<PackedNode> bnodes;  // blocked layout (kTreeBlock slots per block)
    DBuf<int32_t> broot;      // root slot of each tree in bnodes
    int kind = 1;  // 0 tree, 1 forest
    int n_trees = 0;
    int64_t n_nodes = 0;
    DBuf<int32_t> feature, left, right, cls;  // left/right are GLOBAL node ids
    DBuf<double> threshold;
    DBuf<int64_t> root;
};

}  // namespace sob

struct so_forest {
    int device = 0;
    uint64_t uid = 0;  // unique per upload (tune plans are keyed by it)
    sob::ForestDev f;
};
