// sgwls_apps.cu -- elementwise stages of the reference's application pipelines
// (proj/src/apps.cpp), so the pipelines run on the device between smooth()
// calls instead of round-tripping every intermediate image through the host.
//
//   detail_enhance  proj/src/apps.cpp:58-64    k_detail
//   tone_map        proj/src/apps.cpp:66-109   k_luma_log, k_minmax, k_tone_out
//   depth_upsample  proj/src/apps.cpp:111-128  k_scatter_depth, k_luma
//   colorize        proj/src/apps.cpp:130-155  k_colorize_pack, k_colorize_out
//
// BT.601 constants of proj/src/image.cpp:255-256.  All stages are one pass over
// HBM (grid-stride, 148-SM multiple), fp32 like the filter.
#include <cuda_runtime.h>

#include "sgwls_kernels.h"

namespace sgwls_b200 {
namespace {

constexpr float kYR = 0.299f, kYG = 0.587f, kYB = 0.114f;
constexpr float kUDiv = 1.772f, kVDiv = 1.402f;

inline int grid_for(long long n) {
    long long b = (n + 255) / 256;
    const long long cap = 148LL * 16;
    return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

// order-preserving float <-> uint (for atomicMin / atomicMax reductions)
__device__ __forceinline__ unsigned f2ord(float f) {
    const unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// out = clamp(base + boost * (img - base), 0, 1)   (proj/src/apps.cpp:61-62)
__global__ void k_detail(const float* __restrict__ img, const float* __restrict__ base, float boost,
                         float* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float b = base[i];
        out[i] = fminf(fmaxf(fmaf(boost, img[i] - b, b), 0.f), 1.f);
    }
}

// luminance (proj/src/image.cpp:290-298) of a 1- or 3-channel image
__device__ __forceinline__ float luma_at(const float* __restrict__ p, int C, long long i) {
    if (C == 1) return p[i];
    const float* q = p + i * 3;
    return kYR * q[0] + kYG * q[1] + kYB * q[2];
}

__global__ void k_luma(const float* __restrict__ img, int C, float* __restrict__ lum, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        lum[i] = luma_at(img, C, i);
}

// lum, log10(lum); bad <- 1 if some lum is not > 0   (proj/src/apps.cpp:67-73)
__global__ void k_luma_log(const float* __restrict__ hdr, int C, float* __restrict__ lum,
                           float* __restrict__ loglum, long long n, unsigned* __restrict__ bad) {
    bool ok = true;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float l = luma_at(hdr, C, i);
        ok = ok && (l > 0.f);
        lum[i] = l;
        loglum[i] = log10f(l);
    }
    if (__syncthreads_or(!ok) && threadIdx.x == 0) atomicOr(bad, 1u);
}

// red[0] = ord(min log_lum), red[1] = ord(max log_lum), red[2] = ord(max level)
// (proj/src/apps.cpp:90-93); red must start as {~0, 0, 0}
__global__ void k_minmax(const float* __restrict__ loglum, const float* __restrict__ level, long long n,
                         unsigned* __restrict__ red) {
    unsigned mn = 0xffffffffu, mx = 0u, ma = 0u;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned a = f2ord(loglum[i]), b = f2ord(level[i]);
        mn = min(mn, a);
        mx = max(mx, a);
        ma = max(ma, b);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        ma = max(ma, __shfl_xor_sync(0xffffffffu, ma, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&red[0], mn);
        atomicMax(&red[1], mx);
        atomicMax(&red[2], ma);
    }
}

// Recombination and chroma reattachment (proj/src/apps.cpp:90-108).  lev[k] is
// level k (lev[0] = log luminance); detail_k = lev[k] - lev[k+1].
__global__ void k_tone_out(const float* __restrict__ hdr, int C, const float* __restrict__ lum,
                           const float* __restrict__ l0, const float* __restrict__ l1, const float* __restrict__ l2,
                           const float* __restrict__ l3, const unsigned* __restrict__ red, float target_range,
                           float dw0, float dw1, float dw2, float* __restrict__ out, long long n) {
    const float lo = ord2f(red[0]), hi = ord2f(red[1]), anchor = ord2f(red[2]);
    const float range = hi - lo;
    const float gain = range > 0.f ? target_range / range : 1.f;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float a = l0[i], b = l1[i], c = l2[i], d = l3[i];
        float v = anchor + (d - anchor) * gain;
        v += dw0 * (a - b);
        v += dw1 * (b - c);
        v += dw2 * (c - d);
        const float ratio = exp10f(v) / lum[i];
        for (int k = 0; k < C; ++k) out[i * C + k] = hdr[i * C + k] * ratio;
    }
}

// sparse field of depth_upsample: values/mask (pre-zeroed, W x H) get the
// low-resolution samples at (y*f, x*f)   (proj/src/apps.cpp:118-126)
__global__ void k_scatter_depth(const float* __restrict__ low, int lw, int lh, int f, int W,
                                float* __restrict__ values, float* __restrict__ mask) {
    const long long n = (long long)lw * lh;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long y = i / lw, x = i - y * lw;
        const long long o = (y * f) * W + x * f;
        values[o] = low[i];
        mask[o] = 1.f;
    }
}

// colorize: U, V of the scribbles where the mask is exactly 1, else 0, as one
// 2-channel sparse field   (proj/src/apps.cpp:136-149, rgb_to_yuv proj/src/image.cpp:259-272)
__global__ void k_colorize_pack(const float* __restrict__ scrib, const float* __restrict__ mask,
                                float* __restrict__ uv, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        float u = 0.f, v = 0.f;
        if (mask[i] == 1.f) {
            const float r = scrib[i * 3], g = scrib[i * 3 + 1], b = scrib[i * 3 + 2];
            const float luma = kYR * r + kYG * g + kYB * b;
            u = (b - luma) / kUDiv;
            v = (r - luma) / kVDiv;
        }
        uv[i * 2] = u;
        uv[i * 2 + 1] = v;
    }
}

// clamp01(yuv_to_rgb(merge_planes(gray, u, v)))   (proj/src/apps.cpp:154, proj/src/image.cpp:274-288)
__global__ void k_colorize_out(const float* __restrict__ gray, const float* __restrict__ uv,
                               float* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float luma = gray[i], u = uv[i * 2], v = uv[i * 2 + 1];
        const float r = luma + kVDiv * v;
        const float b = luma + kUDiv * u;
        const float g = (luma - kYR * r - kYB * b) / kYG;
        out[i * 3] = fminf(fmaxf(r, 0.f), 1.f);
        out[i * 3 + 1] = fminf(fmaxf(g, 0.f), 1.f);
        out[i * 3 + 2] = fminf(fmaxf(b, 0.f), 1.f);
    }
}

}  // namespace

cudaError_t launch_detail(const float* img, const float* base, float boost, float* out, long long n,
                          cudaStream_t st) {
    k_detail<<<grid_for(n), 256, 0, st>>>(img, base, boost, out, n);
    return cudaGetLastError();
}

cudaError_t launch_luma(const float* img, int C, float* lum, long long n, cudaStream_t st) {
    k_luma<<<grid_for(n), 256, 0, st>>>(img, C, lum, n);
    return cudaGetLastError();
}

cudaError_t launch_luma_log(const float* hdr, int C, float* lum, float* loglum, long long n, unsigned* bad,
                            cudaStream_t st) {
    k_luma_log<<<grid_for(n), 256, 0, st>>>(hdr, C, lum, loglum, n, bad);
    return cudaGetLastError();
}

cudaError_t launch_tone_out(const float* hdr, int C, const float* lum, const float* const lev[4], unsigned* red,
                            float target_range, const float dw[3], float* out, long long n, cudaStream_t st) {
    k_minmax<<<grid_for(n), 256, 0, st>>>(lev[0], lev[3], n, red);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_tone_out<<<grid_for(n), 256, 0, st>>>(hdr, C, lum, lev[0], lev[1], lev[2], lev[3], red, target_range, dw[0],
                                            dw[1], dw[2], out, n);
    return cudaGetLastError();
}

cudaError_t launch_scatter_depth(const float* low, int lw, int lh, int f, int W, float* values, float* mask,
                                 cudaStream_t st) {
    k_scatter_depth<<<grid_for((long long)lw * lh), 256, 0, st>>>(low, lw, lh, f, W, values, mask);
    return cudaGetLastError();
}

cudaError_t launch_colorize_pack(const float* scrib, const float* mask, float* uv, long long n, cudaStream_t st) {
    k_colorize_pack<<<grid_for(n), 256, 0, st>>>(scrib, mask, uv, n);
    return cudaGetLastError();
}

cudaError_t launch_colorize_out(const float* gray, const float* uv, float* out, long long n, cudaStream_t st) {
    k_colorize_out<<<grid_for(n), 256, 0, st>>>(gray, uv, out, n);
    return cudaGetLastError();
}

}  // namespace sgwls_b200
