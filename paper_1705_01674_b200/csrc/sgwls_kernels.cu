// sgwls_kernels.cu -- small helper kernels (layout transpose, sparse pack /
// ratio / validation) and the radius dispatch of the pass kernels, whose
// per-radius instantiations live in inst_r<R>.cu (compiled in parallel).
#include <cuda_runtime.h>

#include <cstdint>

#include "sgwls_device.cuh"
#include "sgwls_kernels.h"
#include "sgwls_profile.h"

namespace sgwls_b200 {

template <int R>
cudaError_t launch_pass_r(const PassLaunch& pl, cudaStream_t st);
namespace tile {
template <int R>
cudaError_t launch_tile_r(const PassLaunch& pl, cudaStream_t st);
}

// ============================================================ small kernels

// out[img][x][y][c] = in[img][y][x][c]  (H x W x C -> W x H x C), 32x32 pixel
// tiles through shared memory; both the read and the write are row-coalesced.
template <int C>
__global__ void __launch_bounds__(256) k_transpose(const float* __restrict__ in, float* __restrict__ out, int H, int W,
                                                   long long stride) {
    __shared__ float tile[32][32 * C + 1];
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32, img = blockIdx.z;
    const float* ii = in + img * stride;
    float* oo = out + img * stride;
    const int nx = min(32, W - x0), ny = min(32, H - y0);
    for (int yy = threadIdx.y; yy < ny; yy += blockDim.y) {
        const float* row = ii + ((long long)(y0 + yy) * W + x0) * C;
        for (int i = threadIdx.x; i < nx * C; i += 32) tile[yy][i] = __ldg(row + i);
    }
    __syncthreads();
    for (int xx = threadIdx.y; xx < nx; xx += blockDim.y) {
        float* row = oo + ((long long)(x0 + xx) * H + y0) * C;
        for (int i = threadIdx.x; i < ny * C; i += 32) {
            const int yy = i / C, c = i - yy * C;
            row[i] = tile[yy][xx * C + c];
        }
    }
}

// One-channel transpose (the guidance of every row pass): TS x TS tiles, 256
// threads, 16-byte loads and stores, all loads of a thread issued before the
// shared-memory stores (TS = 64: 4 x 16 B in flight per thread, for large
// images; TS = 32: one each, 4x the CTAs for small ones).  The pitch-(TS+1)
// tile keeps both phases at <= 2-way bank conflicts (TS = 32: none).  Needs
// W, H multiples of 4 and 16-byte aligned buffers; edge tiles go scalar.
template <int TS>
__global__ void __launch_bounds__(256) k_transpose1_v4(const float* __restrict__ in, float* __restrict__ out, int H,
                                                       int W, long long stride) {
    constexpr int TPR = TS / 4, RPP = 256 / TPR, IT = TS / RPP;  // float4 per row, rows per sweep, sweeps
    __shared__ float tile[TS][TS + 1];
    const int x0 = blockIdx.x * TS, y0 = blockIdx.y * TS, img = blockIdx.z;
    const float* ii = in + img * stride;
    float* oo = out + img * stride;
    const int t = threadIdx.x, rr = t / TPR, cc = t % TPR;
    if (x0 + TS <= W && y0 + TS <= H) {
        float4 v[IT];
#pragma unroll
        for (int i = 0; i < IT; ++i)
            v[i] = __ldg(reinterpret_cast<const float4*>(ii + (long long)(y0 + rr + RPP * i) * W + x0) + cc);
#pragma unroll
        for (int i = 0; i < IT; ++i) {
            float* d = &tile[rr + RPP * i][4 * cc];
            d[0] = v[i].x;
            d[1] = v[i].y;
            d[2] = v[i].z;
            d[3] = v[i].w;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < IT; ++i) {
            const int x = rr + RPP * i;
            const float4 o = make_float4(tile[4 * cc][x], tile[4 * cc + 1][x], tile[4 * cc + 2][x], tile[4 * cc + 3][x]);
            reinterpret_cast<float4*>(oo + (long long)(x0 + x) * H + y0)[cc] = o;
        }
    } else {
        const int nx = min(TS, W - x0), ny = min(TS, H - y0);
        for (int i = t; i < TS * TS; i += 256) {
            const int yy = i / TS, xx = i % TS;
            if (yy < ny && xx < nx) tile[yy][xx] = __ldg(ii + (long long)(y0 + yy) * W + x0 + xx);
        }
        __syncthreads();
        for (int i = t; i < TS * TS; i += 256) {
            const int xx = i / TS, yy = i % TS;
            if (yy < ny && xx < nx) oo[(long long)(x0 + xx) * H + y0 + yy] = tile[yy][xx];
        }
    }
}

// packed[px][0..C-1] = values[px][..], packed[px][C] = mask[px]
__global__ void k_pack_sparse(const float* __restrict__ values, const float* __restrict__ mask,
                              float* __restrict__ packed, long long npx, int C) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= npx) return;
    for (int c = 0; c < C; ++c) packed[i * (C + 1) + c] = values[i * C + c];
    packed[i * (C + 1) + C] = mask[i];
}

// Eq. 21 ratio with the reference floor (proj/src/smoother.cpp:149-161)
__global__ void k_ratio(const float* __restrict__ packed, float* __restrict__ out, float* __restrict__ und,
                        long long npx, int C, float floor_) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= npx) return;
    const float d = packed[i * (C + 1) + C];
    const bool undef = d < floor_;
    for (int c = 0; c < C; ++c) out[i * C + c] = undef ? 0.f : packed[i * (C + 1) + c] / d;
    if (und) und[i] = undef ? 1.f : 0.f;
}

// Sparse-field validation (proj/src/smoother.cpp:129-144).  status[0] = min
// violating pixel index (mask not 0/1, or value nonzero where mask is 0),
// status[1] = number of pixels with mask == 1 (saturating).
// One pixel's field checks (proj/src/smoother.cpp:133-141): mask in {0, 1}, values zero outside it
__device__ __forceinline__ void check_px(float mv, bool vnz, long long i, bool& any, long long& bad) {
    if ((mv != 0.f && mv != 1.f) || (mv == 0.f && vnz)) bad = bad < i ? bad : i;
    any = any || mv == 1.f;
}

// Streams mask and values once: VPT pixels per thread and step as 16-byte loads when the
// layout allows (all loads of a step issued before any test), one atomic per CTA at most.
// status[pair] = first offending pixel (row-major, min), status[batch + pair] = mask non-empty.
template <int C>
__global__ void __launch_bounds__(256) k_validate_sparse(const float* __restrict__ values,
                                                        const float* __restrict__ mask, long long npx, int Crt,
                                                        int batch, unsigned long long* status, int vec) {
    const int bi = blockIdx.y;  // pair
    const int Cn = C > 0 ? C : Crt;
    values += (long long)bi * npx * Cn;
    mask += (long long)bi * npx;
    unsigned long long* any_w = status + batch + bi;
    bool any = false;
    long long bad = 0x7fffffffffffffffLL;
    if (vec && C == 1) {
        const long long nq = npx >> 2;
        const float4* m4 = reinterpret_cast<const float4*>(mask);
        const float4* v4 = reinterpret_cast<const float4*>(values);
        constexpr int U = 4;
        for (long long q0 = (long long)blockIdx.x * blockDim.x * U + threadIdx.x; q0 < nq;
             q0 += (long long)gridDim.x * blockDim.x * U) {
            float4 m[U], v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long q = q0 + (long long)u * blockDim.x;
                m[u] = q < nq ? __ldcs(m4 + q) : make_float4(1.f, 1.f, 1.f, 1.f);
                v[u] = q < nq ? __ldcs(v4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long q = q0 + (long long)u * blockDim.x;
                if (q < nq) {
                    check_px(m[u].x, v[u].x != 0.f, 4 * q, any, bad);
                    check_px(m[u].y, v[u].y != 0.f, 4 * q + 1, any, bad);
                    check_px(m[u].z, v[u].z != 0.f, 4 * q + 2, any, bad);
                    check_px(m[u].w, v[u].w != 0.f, 4 * q + 3, any, bad);
                }
            }
        }
    } else {
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < npx;
             i += (long long)gridDim.x * blockDim.x) {
            const float mv = mask[i];
            bool vnz = false;
            for (int c = 0; c < Cn; ++c) vnz = vnz || values[i * Cn + c] != 0.f;
            check_px(mv, vnz, i, any, bad);
        }
    }
    if (bad != 0x7fffffffffffffffLL) atomicMin(&status[bi], (unsigned long long)bad);
    if (__syncthreads_or(any) && threadIdx.x == 0 && *reinterpret_cast<volatile unsigned long long*>(any_w) == 0ull)
        atomicOr(any_w, 1ull);
}

// =========================================================== dispatch

cudaError_t launch_pass(const PassLaunch& pl, cudaStream_t st) {
    ProfScope ps("pass", st);
    if (pl.anyr) return launch_pass_anyr(pl, st);
    if (pl.fast) {
        switch (pl.geom.r) {
            case 1: return tile::launch_tile_r<1>(pl, st);
            case 2: return tile::launch_tile_r<2>(pl, st);
            case 3: return tile::launch_tile_r<3>(pl, st);
            case 4: return tile::launch_tile_r<4>(pl, st);
            default: return cudaErrorInvalidValue;
        }
    }
    switch (pl.geom.r) {
        case 1: return launch_pass_r<1>(pl, st);
        case 2: return launch_pass_r<2>(pl, st);
        case 3: return launch_pass_r<3>(pl, st);
        case 4: return launch_pass_r<4>(pl, st);
        case 5: return launch_pass_r<5>(pl, st);
        case 6: return launch_pass_r<6>(pl, st);
        case 7: return launch_pass_r<7>(pl, st);
        case 8: return launch_pass_r<8>(pl, st);
        default: return cudaErrorInvalidValue;
    }
}

size_t rec_floats(int r, int C) { return (size_t)(r * (r - 1) + r * r + 2 * r + 2 * r * C); }
size_t rs_floats(int r, int C) { return (size_t)(2 * r - 1 + C); }
size_t map_floats(int r, int C) { return (size_t)((r * (C + 2 * r) + 3) & ~3); }  // padded (Rec::MAPP)

cudaError_t launch_transpose(const float* in, float* out, int H, int W, int C, int batch, cudaStream_t st) {
    dim3 grid((W + 31) / 32, (H + 31) / 32, batch);
    ProfScope ps("transpose", st);
    const long long stride = (long long)H * W * C;
    const bool v4 = C == 1 && W % 4 == 0 && H % 4 == 0 &&
                    ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    if (v4) {
        // 64x64 tiles when they fill the GPU (>= 8 per SM; c5 guidance 165 -> 89 us), else 32x32
        const long long tiles64 = (long long)((W + 63) / 64) * ((H + 63) / 64) * batch;
        if (tiles64 >= 148 * 8)
            k_transpose1_v4<64><<<dim3((W + 63) / 64, (H + 63) / 64, batch), 256, 0, st>>>(in, out, H, W, stride);
        else
            k_transpose1_v4<32><<<dim3((W + 31) / 32, (H + 31) / 32, batch), 256, 0, st>>>(in, out, H, W, stride);
        return cudaGetLastError();
    }
    switch (C) {
        case 1: k_transpose<1><<<grid, dim3(32, 8), 0, st>>>(in, out, H, W, stride); break;
        case 2: k_transpose<2><<<grid, dim3(32, 8), 0, st>>>(in, out, H, W, stride); break;
        case 3: k_transpose<3><<<grid, dim3(32, 8), 0, st>>>(in, out, H, W, stride); break;
        case 4: k_transpose<4><<<grid, dim3(32, 8), 0, st>>>(in, out, H, W, stride); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_pack_sparse(const float* values, const float* mask, float* packed, long long npx, int C,
                               cudaStream_t st) {
    ProfScope ps("pack_sparse", st);
    k_pack_sparse<<<(unsigned)((npx + 255) / 256), 256, 0, st>>>(values, mask, packed, npx, C);
    return cudaGetLastError();
}

cudaError_t launch_ratio(const float* packed, float* out, float* und, long long npx, int C, float floor_,
                         cudaStream_t st) {
    ProfScope ps("ratio", st);
    k_ratio<<<(unsigned)((npx + 255) / 256), 256, 0, st>>>(packed, out, und, npx, C, floor_);
    return cudaGetLastError();
}

cudaError_t launch_validate_sparse(const float* values, const float* mask, long long npx, int C, int batch,
                                   unsigned long long* status, cudaStream_t st) {
    ProfScope ps("validate_sparse", st);
    const bool vec = C == 1 && npx % 4 == 0 && ((reinterpret_cast<uintptr_t>(values) | reinterpret_cast<uintptr_t>(mask)) & 15) == 0;
    // 16 pixels per thread and step on the vector path; a few CTAs per SM over the whole batch
    const long long per_cta = vec ? 256LL * 16 : 256LL * 4;
    long long bx = (npx + per_cta - 1) / per_cta;
    const long long cap = (148LL * 16 + batch - 1) / batch;
    if (bx > cap) bx = cap;
    if (bx < 1) bx = 1;
    const dim3 grid((unsigned)bx, (unsigned)batch);
    if (C == 1)
        k_validate_sparse<1><<<grid, 256, 0, st>>>(values, mask, npx, C, batch, status, vec ? 1 : 0);
    else
        k_validate_sparse<0><<<grid, 256, 0, st>>>(values, mask, npx, C, batch, status, 0);
    return cudaGetLastError();
}

}  // namespace sgwls_b200
