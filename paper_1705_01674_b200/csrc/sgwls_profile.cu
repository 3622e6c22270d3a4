// sgwls_profile.cu -- optional CUDA-event brackets around every kernel launch.
//
// When enabled (sgwls_b200_profile(1)), each launch is bracketed by a pair of
// events recorded on the launching stream.  Launches made while a stream is
// being captured into a CUDA graph get "external" event-record nodes, so the
// events are re-recorded on every replay of that graph; such records are
// persistent and are counted once per replay that happened since the last
// collect.  sgwls_b200_profile_collect() folds the elapsed times into running
// totals; sgwls_b200_profile_read() collects and returns the totals as JSON.
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
    int* armed;  // graph records: non-null, points at the graph's "replayed" flag
};
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_free;
std::map<std::string, std::pair<long, double>> g_tot;
std::string g_timeline;  // last collected launch sequence: name@start-end (ms, relative to the first)
thread_local int* t_capture_armed = nullptr;

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

void record(cudaEvent_t e, cudaStream_t st, bool external) {
    if (external)
        cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
    else
        cudaEventRecord(e, st);
}

void collect_locked() {
    std::vector<Rec> keep;
    std::string tl;
    cudaEvent_t t0 = nullptr;
    for (auto& r : g_recs) {
        const bool count = r.armed == nullptr || *r.armed;
        if (count) {
            cudaEventSynchronize(r.b);
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
                auto& s = g_tot[r.name];
                s.first += 1;
                s.second += ms;
                if (!t0) t0 = r.a;
                float st = 0.f;
                cudaEventElapsedTime(&st, t0, r.a);
                char buf[128];
                std::snprintf(buf, sizeof buf, "%s%s@%.4f+%.4f", tl.empty() ? "" : " ", r.name, st, ms);
                tl += buf;
            }
        }
        if (r.armed) {
            keep.push_back(r);
        } else {
            g_free.push_back(r.a);
            g_free.push_back(r.b);
        }
    }
    for (auto& r : keep)
        if (r.armed) *r.armed = 0;
    if (!tl.empty()) g_timeline = tl;
    g_recs.swap(keep);
}
}  // namespace

bool prof_enabled() { return g_enabled.load(std::memory_order_relaxed) != 0; }

void prof_set_capture(int* armed) { t_capture_armed = armed; }

int prof_begin(const char* name, cudaStream_t st) {
    if (!g_enabled.load(std::memory_order_relaxed)) return -1;
    std::lock_guard<std::mutex> lk(g_mu);
    Rec r{name, take_event(), take_event(), t_capture_armed};
    record(r.a, st, r.armed != nullptr);
    g_recs.push_back(r);
    return (int)g_recs.size() - 1;
}

void prof_end(int idx, cudaStream_t st) {
    if (idx < 0) return;
    std::lock_guard<std::mutex> lk(g_mu);
    if (idx < (int)g_recs.size()) record(g_recs[idx].b, st, g_recs[idx].armed != nullptr);
}

}  // namespace sgwls_b200

using namespace sgwls_b200;

extern "C" {

void sgwls_b200_profile(int enable) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_enabled.store(enable ? 1 : 0);
}

void sgwls_b200_profile_collect(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    collect_locked();
}

int sgwls_b200_profile_read(char* json, size_t len) {
    std::lock_guard<std::mutex> lk(g_mu);
    collect_locked();
    std::string out = "{";
    bool first = true;
    for (auto& kv : g_tot) {
        char buf[256];
        std::snprintf(buf, sizeof buf, "%s\"%s\": {\"launches\": %ld, \"ms\": %.6f}", first ? "" : ", ",
                      kv.first.c_str(), kv.second.first, kv.second.second);
        out += buf;
        first = false;
    }
    out += first ? "" : ", ";
    out += "\"timeline\": \"" + g_timeline + "\"}";
    g_tot.clear();
    if (json && len) {
        std::strncpy(json, out.c_str(), len - 1);
        json[len - 1] = '\0';
    }
    return (int)out.size();
}

}  // extern "C"
