// Per-stage CUDA-event timing and kernel-launch counting for bench.py.
//
// When enabled, every instrumented stage records a (start, stop) event pair
// on the stream it launches on; sm_profile_collect() synchronises on the
// recorded events and returns the summed milliseconds and launch counts per
// stage.  Disabled (the default) it costs one branch per stage.
#include <atomic>
#include <mutex>
#include <vector>

#include "prof.cuh"

namespace sm {

std::atomic<long long> g_launches{0};
static bool g_prof_on = false;
static std::mutex g_mu;
static std::vector<cudaEvent_t> g_pool;
struct Pending {
    int stage;
    cudaEvent_t a, b;
};
static std::vector<Pending> g_pending;
static cudaEvent_t g_open[ST_COUNT];
static bool g_is_open[ST_COUNT];
static double g_ms[ST_COUNT];
static long long g_calls[ST_COUNT];

static const char *kNames[ST_COUNT] = {"project_fwd", "depth_sort", "bin_emit", "tile_sort",
                                       "composite_fwd", "loss", "composite_bwd", "project_bwd",
                                       "adam", "cull", "codec", "grad_gather"};

// CUDA-graph support: while a graph is being captured, stage event pairs and
// kernel counts are filed under the graph id; every replay re-records the
// same events, so after a replay completes the host accumulates them again.
struct GraphProf {
    std::vector<Pending> pairs;
    long long launches = 0;
};
static std::vector<GraphProf> g_graphs;
static int g_capture_gid = -1;
static long long g_graph_timing_errors = 0;

static cudaEvent_t take_event() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// Inside stream capture a plain record becomes an internal graph edge that
// cannot be timed; an *external* event record node is re-recorded (and
// timeable) at every replay.
static void record(cudaEvent_t e, cudaStream_t st) {
    if (g_capture_gid >= 0)
        cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
    else
        cudaEventRecord(e, st);
}

void prof_begin(Stage s, cudaStream_t st) {
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_mu);
    cudaEvent_t e = take_event();
    record(e, st);
    g_open[s] = e;
    g_is_open[s] = true;
}

void prof_end(Stage s, cudaStream_t st) {
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_is_open[s]) return;
    cudaEvent_t e = take_event();
    record(e, st);
    if (g_capture_gid >= 0)
        g_graphs[g_capture_gid].pairs.push_back({(int)s, g_open[s], e});
    else
        g_pending.push_back({(int)s, g_open[s], e});
    g_is_open[s] = false;
}

void count_launches(long long n) {
    if (g_capture_gid >= 0)
        g_graphs[g_capture_gid].launches += n;   // executed (and counted) at each replay
    else
        g_launches.fetch_add(n, std::memory_order_relaxed);
}

}  // namespace sm

using namespace sm;

extern "C" {

void sm_profile_enable(int on) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_prof_on = on != 0;
}

long long sm_launch_count(void) { return g_launches.load(); }

// Begin filing stage events / launch counts under a new graph id (returned).
int sm_profile_capture_begin(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_graphs.emplace_back();
    g_capture_gid = (int)g_graphs.size() - 1;
    return g_capture_gid;
}

void sm_profile_capture_end(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_capture_gid = -1;
}

// Called after a replay of graph `gid` has completed (stream synchronised):
// adds its kernel count and, when profiling is on, its stage times.
void sm_profile_graph_replayed(int gid) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (gid < 0 || gid >= (int)g_graphs.size()) return;
    GraphProf &g = g_graphs[gid];
    g_launches.fetch_add(g.launches, std::memory_order_relaxed);
    if (!g_prof_on) return;
    for (const Pending &p : g.pairs) {
        float ms = 0.f;
        const cudaError_t e = cudaEventElapsedTime(&ms, p.a, p.b);
        if (e == cudaSuccess) {
            g_ms[p.stage] += ms;
            g_calls[p.stage] += 1;
        } else {
            g_graph_timing_errors++;
            cudaGetLastError();   // do not leave a sticky error for later launch checks
        }
    }
}

long long sm_profile_graph_timing_errors(void) { return g_graph_timing_errors; }

void sm_profile_graph_free(int gid) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (gid < 0 || gid >= (int)g_graphs.size()) return;
    for (const Pending &p : g_graphs[gid].pairs) {
        g_pool.push_back(p.a);
        g_pool.push_back(p.b);
    }
    g_graphs[gid].pairs.clear();
    g_graphs[gid].launches = 0;
}

int sm_profile_stage_count(void) { return ST_COUNT; }

const char *sm_profile_stage_name(int i) { return (i >= 0 && i < ST_COUNT) ? kNames[i] : ""; }

// Sums all completed (start, stop) pairs into the running totals, then copies
// the totals out and resets them.  Blocks until the recorded events complete.
int sm_profile_collect(double *ms_out, long long *calls_out) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (const Pending &p : g_pending) {
        cudaEventSynchronize(p.b);
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            g_ms[p.stage] += ms;
            g_calls[p.stage] += 1;
        } else {
            cudaGetLastError();
        }
        g_pool.push_back(p.a);
        g_pool.push_back(p.b);
    }
    g_pending.clear();
    for (int i = 0; i < ST_COUNT; i++) {
        if (ms_out) ms_out[i] = g_ms[i];
        if (calls_out) calls_out[i] = g_calls[i];
        g_ms[i] = 0.0;
        g_calls[i] = 0;
    }
    return ST_COUNT;
}

}  // extern "C"
