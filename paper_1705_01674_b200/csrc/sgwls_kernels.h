// Host-visible launch interface of the SG-WLS kernels (sgwls_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "sgwls_device.cuh"

namespace sgwls_b200 {

struct PassLaunch {
    PassGeom geom;
    const float* src;   // pass input, layout geom (Hl x Wl x C per image)
    const float* guid;  // guidance in the same orientation (Hl x Wl x Cg per image)
    float* out;         // pass output (next orientation if transpose_out)
    int transpose_out;
    int kmax;           // max positions of a chunk (K3 shared-memory sizing)
    int bx;             // threads per block for K1/K3
    int fast;           // regular-geometry CTA-tiled path (sgwls_tile.cuh)
    int step;           // tiled: CTA band stride (32 - halo bands)
    int ncta;           // tiled: CTAs across the bands
    int nw;             // tiled: chunk warps per CTA (super-chunk size)
    int nph;            // tiled: averaging phases
    float* rec;         // K1 -> K2 records
    float* rs;          // K2 back-substitution scratch
    float* z;           // separator values
    float* U;           // band solutions
    unsigned long long* err;  // NaN-weight report (first pass only), or nullptr
    const WeightDev* w;
    float* maps = nullptr;    // tiled path: affine map of every inner chunk separator of a KA tile
                              // (KA -> KB), [chunk][field][line], map_floats(r, C) fields
    int nwa = 8;              // tiled path: chunks per KA tile (super-chunk)
    // tiled path, interpolate_sparse's last pass: out = C-1 channels num / den
    // (0 where den < ratio_floor), und = undefined mask (or nullptr)
    int ratio = 0;
    float ratio_floor = 0.f;
    float* und = nullptr;
    // tiled path, row-slab mode (geom.has_prev / has_next, sgwls_tile.cuh):
    // 1 = phase A (KA, then this slab's record -> slabrec), 2 = phase B (slabrec
    // = all nslab records; separators, KC, KB); z and sep then carry one slot in
    // front (the previous slab's separator)
    int slab_phase = 0;
    float* slabrec = nullptr;
    int nslab = 1, islab = 0;
    float* zg = nullptr;   // nslab-1 slab separators
    float* bsg = nullptr;  // their back-substitution rows
    float* grec = nullptr; // group records of the slab (phase A -> B), kSlabWarps x REC per band
    // any-radius path (r > kMaxR, sgwls_anyr.cu): line-interleaved workspace and the
    // lambda * spatial-factor table by squared distance (device)
    int anyr = 0;
    float* anyr_ws = nullptr;
    const float* anyr_lspat = nullptr;
};

cudaError_t launch_pass(const PassLaunch& pl, cudaStream_t st);
cudaError_t launch_pass_anyr(const PassLaunch& pl, cudaStream_t st);
size_t anyr_ws_floats(const PassGeom& g);
size_t anyr_lut_floats(int r);
// lut[d2] = lambda * spatial factor of squared distance d2 (proj/src/weights.cpp:55-71), in double then rounded
cudaError_t launch_anyr_lut(float* lut, size_t n, double lambda, bool exp_kind, double sigma_s, double alpha_s,
                            double eps, cudaStream_t st);
size_t rec_floats(int r, int C);
size_t rs_floats(int r, int C);
size_t map_floats(int r, int C);
cudaError_t launch_transpose(const float* in, float* out, int H, int W, int C, int batch, cudaStream_t st);
cudaError_t launch_pack_sparse(const float* values, const float* mask, float* packed, long long npx, int C,
                               cudaStream_t st);
cudaError_t launch_ratio(const float* packed, float* out, float* und, long long npx, int C, float floor_,
                         cudaStream_t st);
// batch pairs: status[b] = min violating pixel of pair b (~0 if none),
// status[batch + b] = nonzero if pair b has a mask pixel == 1
cudaError_t launch_validate_sparse(const float* values, const float* mask, long long npx, int C, int batch,
                                   unsigned long long* status, cudaStream_t st);

// application-pipeline stages (sgwls_apps.cu, proj/src/apps.cpp)
cudaError_t launch_detail(const float* img, const float* base, float boost, float* out, long long n, cudaStream_t st);
cudaError_t launch_luma(const float* img, int C, float* lum, long long n, cudaStream_t st);
cudaError_t launch_luma_log(const float* hdr, int C, float* lum, float* loglum, long long n, unsigned* bad,
                            cudaStream_t st);
cudaError_t launch_tone_out(const float* hdr, int C, const float* lum, const float* const lev[4], unsigned* red,
                            float target_range, const float dw[3], float* out, long long n, cudaStream_t st);
cudaError_t launch_scatter_depth(const float* low, int lw, int lh, int f, int W, float* values, float* mask,
                                 cudaStream_t st);
cudaError_t launch_colorize_pack(const float* scrib, const float* mask, float* uv, long long n, cudaStream_t st);
cudaError_t launch_colorize_out(const float* gray, const float* uv, float* out, long long n, cudaStream_t st);

}  // namespace sgwls_b200
