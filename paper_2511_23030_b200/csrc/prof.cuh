// Stage timing / launch counting hooks (see prof.cu).
#pragma once
#include <cuda_runtime.h>

#include <atomic>

namespace sm {

enum Stage {
    ST_PROJECT = 0,
    ST_DEPTH_SORT,
    ST_BIN,
    ST_TILE_SORT,
    ST_COMPOSITE_FWD,
    ST_LOSS,
    ST_COMPOSITE_BWD,
    ST_PROJECT_BWD,
    ST_ADAM,
    ST_CULL,
    ST_CODEC,
    ST_GRAD_GATHER,
    ST_COUNT
};

extern std::atomic<long long> g_launches;
void prof_begin(Stage s, cudaStream_t st);
void prof_end(Stage s, cudaStream_t st);

// count n kernel launches issued by this library (filed under the graph being
// captured, if any, so replays are counted too)
void count_launches(long long n);

}  // namespace sm
