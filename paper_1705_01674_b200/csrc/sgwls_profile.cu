// sgwls_profile.cu -- optional CUDA-event brackets around every kernel launch.
//
// When enabled (sgwls_b200_profile(1)), each launch is bracketed by a pair of
// events recorded on the launching stream; sgwls_b200_profile_read()
// synchronizes on the recorded events and returns per-kernel totals as JSON.
// Used by bench.py to measure kernel durations live inside the timed region.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "sgwls_profile.h"

namespace sgwls_b200 {

namespace {
std::atomic<int> g_enabled{0};
std::mutex g_mu;
struct Rec {
    const char* name;
    cudaEvent_t a, b;
};
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_free;

cudaEvent_t take_event() {
    if (!g_free.empty()) {
        cudaEvent_t e = g_free.back();
        g_free.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

int prof_begin(const char* name, cudaStream_t st) {
    if (!g_enabled.load(std::memory_order_relaxed)) return -1;
    std::lock_guard<std::mutex> lk(g_mu);
    Rec r{name, take_event(), take_event()};
    cudaEventRecord(r.a, st);
    g_recs.push_back(r);
    return (int)g_recs.size() - 1;
}

void prof_end(int idx, cudaStream_t st) {
    if (idx < 0) return;
    std::lock_guard<std::mutex> lk(g_mu);
    if (idx < (int)g_recs.size()) cudaEventRecord(g_recs[idx].b, st);
}

}  // namespace sgwls_b200

using namespace sgwls_b200;

extern "C" {

void sgwls_b200_profile(int enable) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_enabled.store(enable ? 1 : 0);
}

int sgwls_b200_profile_read(char* json, size_t len) {
    std::lock_guard<std::mutex> lk(g_mu);
    std::map<std::string, std::pair<long, double>> agg;
    for (auto& r : g_recs) {
        cudaEventSynchronize(r.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        auto& s = agg[r.name];
        s.first += 1;
        s.second += ms;
        g_free.push_back(r.a);
        g_free.push_back(r.b);
    }
    g_recs.clear();
    std::string out = "{";
    bool first = true;
    for (auto& kv : agg) {
        char buf[256];
        std::snprintf(buf, sizeof buf, "%s\"%s\": {\"launches\": %ld, \"ms\": %.6f}", first ? "" : ", ",
                      kv.first.c_str(), kv.second.first, kv.second.second);
        out += buf;
        first = false;
    }
    out += "}";
    if (json && len) {
        std::strncpy(json, out.c_str(), len - 1);
        json[len - 1] = '\0';
    }
    return (int)out.size();
}

}  // extern "C"
