// Device-resident forest (SoA node arrays), shared by model.cu and capi.cu.
#pragma once

#include "common.cuh"

namespace sob {

struct ForestDev {
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
    sob::ForestDev f;
};
