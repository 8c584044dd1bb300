// Device-side feature state shared by features.cu (producer) and model.cu
// (tune_ml consumer: predict + feasibility read it without a host round trip).
#pragma once

#include "matrix.cuh"

namespace sob {

struct FeatState {
    unsigned long long visits;     // entry visits = NNZ (features.cpp:22-26)
    unsigned long long structure;  // structure reads (DIA holes, ELL sentinels)
    int max_row;
    int min_row;
    unsigned long long nd, ntd;    // N_D, N_TD
    double S;                      // exact sequential sum of squared deviations
    unsigned ticket;               // dynamic row-group counter of the CSR sweep
    so_feature_vector out;         // finalized vector
    // %globaltimer (ns, 32 ns ticks on B200) at the start of the first feature
    // kernel and after the finalize: the tuner's T_FE without event nodes
    unsigned long long t_begin, t_end;
};

// Scratch of the feature pipeline for one matrix (reusable across calls, e.g.
// by the cached tune graph, so the graph holds no allocation nodes).
struct FeatWorkspace {
    DBuf<int32_t> rc, bins;
    DBuf<unsigned long long> dcount;
    DBuf<double> csum, P;
    DBuf<unsigned char> rec;
    // optional second branch (enable_fork, before a stream capture): the
    // diagonal-bin reduction runs beside the spread chain instead of before it
    cudaStream_t aux = nullptr;
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    // CSR-part sweep: -1 = size heuristic, 0 = row-lockstep, 1 = entry-parallel,
    // 2 = row-lockstep with every key a global atomic (no hash); the tune
    // plan times them once and keeps the fastest (capi.cu)
    int sweep = -1;
    FeatWorkspace(const so_matrix& m, cudaStream_t s);
    ~FeatWorkspace();
    FeatWorkspace(const FeatWorkspace&) = delete;
    FeatWorkspace& operator=(const FeatWorkspace&) = delete;
    void enable_fork();
};

// Enqueue the whole feature pipeline on stream s; the finalized vector lands in
// st->out (device).  Without a workspace, scratch is stream-ordered and
// released on return.
void enqueue_features(const so_matrix& m, double ratio, FeatState* st, cudaStream_t s,
                      FeatWorkspace* ws = nullptr);

}  // namespace sob
