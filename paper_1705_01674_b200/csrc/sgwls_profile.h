// Optional per-launch CUDA-event profiling (sgwls_profile.cu).
#pragma once

#include <cuda_runtime.h>

namespace sgwls_b200 {

// Returns a record index (or -1 when profiling is off); pair with prof_end on the same stream.
int prof_begin(const char* name, cudaStream_t st);
bool prof_enabled();
// While a graph is being captured on this thread, records are tied to `armed`
// (set to 1 on every replay of that graph); nullptr ends the capture scope.
void prof_set_capture(int* armed);
void prof_end(int idx, cudaStream_t st);

struct ProfScope {
    int idx;
    cudaStream_t st;
    ProfScope(const char* name, cudaStream_t s) : idx(prof_begin(name, s)), st(s) {}
    ~ProfScope() { prof_end(idx, st); }
};

}  // namespace sgwls_b200
