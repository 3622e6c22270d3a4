// sgwls_device.cuh -- device-side building blocks of the SG-WLS pass.
//
// Notation.  A pass works on a row-major layout of Hl rows x Wl
// columns x C channels in which the bands are vertical strips ("column pass";
// a row pass runs on the transposed layout).  Band b is centred on column
// center(b) (proj/src/snake.cpp:7-19), spans columns [lo, lo+m), and is walked
// serpentine row by row: position p = y*m + jj, column lo + (y odd ? m-1-jj : jj)
// (proj/src/snake.cpp:21-49).  Its 1-D WLS system (proj/src/banded.cpp:13-42)
// has unit row sums: diag = 1 + lambda*sum(w), off-diagonals -lambda*w.
//
// All eliminations below are written on MAGNITUDES of the (non-positive)
// off-diagonal entries and use the row-sum pivot
//     alpha_k = e_k + sum(remaining off-diagonal magnitudes of row k)
// where e is the forward-eliminated all-ones right-hand side.  Every term is
// non-negative, so fp32 loses nothing to cancellation; the
// recurrence is algebraically identical to the reference's r-band LU
// (proj/src/banded.cpp:44-118) with gamma = alpha*beta (symmetric A).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sgwls_b200 {

constexpr int kMaxR = 8;
constexpr int kMaxCg = 4;
constexpr int kLutMax = 2 * (2 * kMaxR + 1) * (2 * kMaxR + 1) + 1;

// Weight parameters, pre-folded on the host in double (proj/src/weights.cpp:14-22,63-71).
struct WeightDev {
    int kind;          // 0 = Frac, 1 = Exp
    float lam;         // lambda
    float exp_k;       // Exp: -gscale^2 * log2(e) / (2 sigma_r^2)
    float frac_half;   // Frac: alpha_r / 2
    float frac_lg2s;   // Frac: log2(gscale^2)
    float eps;         // Frac: epsilon
    float spat[kLutMax];  // spatial factor by squared 2-D distance d2
    // tiled path (r <= 4, d2 < kTileLut): lambda folded into the weight
    float lspat[32];      // lambda * spat[d2]                     (Frac)
    float lg2ls[32];      // log2(lambda * spat[d2]), -inf for 0   (Exp)
};

// Geometry of one pass in its own (possibly transposed) layout.
struct PassGeom {
    int Hl, Wl;        // rows (sweep) and columns (band-centre axis) of the layout
    int C, Cg;         // target / guidance channels
    int r, tau;
    int nb;            // bands per image
    int nreg;          // centres of the regular progression r, r+tau, ...
    int degenerate;    // extent < 2r+1: single clipped band
    int m;             // band width (2r+1, or the clipped width)
    int P;             // chunks per band
    int batch;         // images
    long long n;       // positions per band = m*Hl
    long long img_stride;   // floats per image of the target layout (Hl*Wl*C)
    long long gimg_stride;  // floats per image of the guidance layout
    unsigned tau_mul;       // ceil(2^32 / tau) (tau > 1): exact x / tau for 0 <= x < 2^28
    // Row-slab mode (tiled path, a Column pass over rows [row0, row0 + Hl) of a
    // taller image, sharded.py): the bands continue above (has_prev: the local
    // chunk 0 couples to the previous slab's last separator, whose guidance row
    // is readable at row -1) and/or below (has_next: the local last chunk ends
    // in a separator shared with the next slab).  0/0 for an ordinary pass.
    int has_prev, has_next;
    int row0;               // global row of local row 0 (error positions)
    // Split input (tiled path, interpolate_sparse's first pass): the pass input
    // is C-1 value channels at `src` plus the mask as channel C-1 at msk
    // (proj/src/smoother.cpp:146-147 smooths both) -- no packed copy.
    const float* msk;
};

__host__ __device__ __forceinline__ unsigned tau_multiplier(int tau) {
    return tau > 1 ? (unsigned)(0xffffffffu / (unsigned)tau) + 1u : 0u;
}

__device__ __forceinline__ int div_tau(const PassGeom& g, int x) {
    return g.tau == 1 ? x : (int)__umulhi((unsigned)x, g.tau_mul);
}

__host__ __device__ __forceinline__ int band_center(const PassGeom& g, int b) {
    if (g.degenerate) return (g.Wl - 1) / 2;
    return b < g.nreg ? g.r + g.tau * b : g.Wl - 1 - g.r;
}

__host__ __device__ __forceinline__ int band_lo(const PassGeom& g, int b) {
    const int c = band_center(g, b);
    return c - g.r > 0 ? c - g.r : 0;
}

__host__ __device__ __forceinline__ int chunk_row(const PassGeom& g, int j) {
    return (int)(((long long)j * g.Hl) / g.P);
}

// Rows per chunk of the CTA-tiled path: keeps a chunk's inputs and edge weights
// at ~64 registers (sgwls_tile.cuh).
#ifndef SGWLS_CHUNK_REGS
#define SGWLS_CHUNK_REGS 64
#endif
__host__ __device__ constexpr int tile_rows_per_chunk(int R, int C) {
    return (SGWLS_CHUNK_REGS / ((2 * R + 1) * (C + R))) < 1
               ? 1
               : ((SGWLS_CHUNK_REGS / ((2 * R + 1) * (C + R))) > 8 ? 8 : (SGWLS_CHUNK_REGS / ((2 * R + 1) * (C + R))));
}
constexpr int kTileMaxR = 4;
constexpr int kTileWarps = 8;
// warps per band group of the row-slab reduce / solve kernels (sgwls_tile.cuh)
constexpr int kSlabWarps = 16;

__device__ __forceinline__ float fast_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float fast_lg2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float fast_rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// (range*gscale)^alpha_r = exp2(alpha_r/2 * (log2(range2) + log2(gscale^2)))
// (proj/src/weights.cpp:67-71).  log2(0) = -inf is clamped to -FLT_MAX so that
// range = 0 gives 0 for alpha_r > 0 and exactly 1 for alpha_r = 0, like
// std::pow(0, alpha_r), instead of 0 * -inf = NaN.  A select, not fmaxf: a NaN
// guidance must still give a NaN weight (the reference's pivot failure).
__device__ __forceinline__ float frac_range_pow(const WeightDev& W, float range2) {
    const float l = fast_lg2(range2) + W.frac_lg2s;
    return fast_ex2(W.frac_half * (l < -3.402823466e38f ? -3.402823466e38f : l));
}

// Eq. 2 kernels on fp32 guidance (proj/src/weights.cpp:55-71).
__device__ __forceinline__ float guidance_weight(const WeightDev& W, float range2, int d2) {
    const float s = W.spat[d2];
    if (W.kind == 1) return s * fast_ex2(range2 * W.exp_k);
    return s / (frac_range_pow(W, range2) + W.eps);
}

// Same, with the kernel kind fixed at compile time (1 = Exp, 0 = Frac).
template <int WK>
__device__ __forceinline__ float guidance_weight_k(const WeightDev& W, float range2, int d2) {
    const float s = W.spat[d2];
    if constexpr (WK == 1) {
        return s * fast_ex2(range2 * W.exp_k);
    } else {
        return s / (frac_range_pow(W, range2) + W.eps);
    }
}

// lambda * weight for the tiled path (kind fixed at compile time).  Exp:
// lambda*s*exp2(k*range2) = exp2(k*range2 + log2(lambda*s)): one FFMA + one
// MUFU per edge instead of FMUL, MUFU and two more FMULs.
template <int WK>
__device__ __forceinline__ float guidance_lweight_k(const WeightDev& W, float range2, int d2) {
#ifdef SGWLS_EXPERIMENT_FREE_WEIGHTS
    // timing experiment only (factor reuse): every edge weight costs nothing,
    // the upper bound of what re-reading stored weights in passes 3/4 could save
    return W.lam;
#endif
    if constexpr (WK == 1) {
        return fast_ex2(fmaf(range2, W.exp_k, W.lg2ls[d2]));
    } else {
        // approximate reciprocal (MUFU.RCP, <= 1 ulp) instead of the IEEE division
        // and its slow path: pr + eps >= eps > 0, and rcp(inf) = 0
        return W.lspat[d2] * fast_rcp(frac_range_pow(W, range2) + W.eps);
    }
}

// Position walker: serpentine coordinate of position p = y*m + jj within a band.
__device__ __forceinline__ int serp_col(int lo, int m, int y, int jj) {
    return lo + ((y & 1) ? (m - 1 - jj) : jj);
}

}  // namespace sgwls_b200
