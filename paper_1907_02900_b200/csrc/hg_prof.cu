// hg_prof.cu -- in-library kernel timeline (the engine's tracing subsystem).
//
// The reference's only instrumentation is BuildStats op counters
// (core.hpp:40-56). On the device the useful evidence is per-kernel time, so
// when enabled every launch in the build/probe pipelines is bracketed by a
// pair of CUDA events recorded on the launching stream; hg_profiler_collect
// aggregates them per kernel name (launch count + total ms). Disabled
// (default), the hooks are a branch on a global flag.
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hg_b200.h"
#include "hg_internal.h"

namespace hg {

namespace {
struct Span {
    const char* name;
    cudaEvent_t a, b;
};
std::mutex g_mu;
std::vector<Span> g_spans;
std::vector<cudaEvent_t> g_pool;
bool g_enabled = false;

cudaEvent_t get_event() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

bool prof_enabled() { return g_enabled; }

int prof_begin(const char* name, cudaStream_t s) {
    if (!g_enabled) return -1;
    std::lock_guard<std::mutex> lk(g_mu);
    Span sp{name, get_event(), get_event()};
    cudaEventRecord(sp.a, s);
    g_spans.push_back(sp);
    return int(g_spans.size() - 1);
}

void prof_end(int token, cudaStream_t s) {
    if (token < 0) return;
    std::lock_guard<std::mutex> lk(g_mu);
    if (size_t(token) < g_spans.size()) cudaEventRecord(g_spans[token].b, s);
}

}  // namespace hg

extern "C" {

void hg_profiler_enable(int32_t on) {
    std::lock_guard<std::mutex> lk(hg::g_mu);
    hg::g_enabled = on != 0;
}

int32_t hg_profiler_collect(hg_kernel_time* out, int32_t max_out) {
    std::lock_guard<std::mutex> lk(hg::g_mu);
    std::vector<hg_kernel_time> agg;
    for (auto& sp : hg::g_spans) {
        cudaEventSynchronize(sp.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, sp.a, sp.b);
        size_t i = 0;
        for (; i < agg.size(); ++i)
            if (std::strncmp(agg[i].name, sp.name, sizeof agg[i].name) == 0) break;
        if (i == agg.size()) {
            hg_kernel_time k;
            std::memset(&k, 0, sizeof k);
            std::strncpy(k.name, sp.name, sizeof k.name - 1);
            agg.push_back(k);
        }
        agg[i].launches += 1;
        agg[i].total_ms += ms;
        hg::g_pool.push_back(sp.a);
        hg::g_pool.push_back(sp.b);
    }
    hg::g_spans.clear();
    const int32_t n = int32_t(agg.size());
    for (int32_t i = 0; i < n && i < max_out; ++i) out[i] = agg[i];
    return n;
}

}  // extern "C"
