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
__global__ void k_validate_sparse(const float* __restrict__ values, const float* __restrict__ mask, long long npx,
                                  int C, unsigned long long* status) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    bool any = false;
    if (i < npx) {
        const float mv = mask[i];
        bool bad = false;
        if (mv != 0.f && mv != 1.f) bad = true;
        if (mv == 1.f) any = true;
        if (mv == 0.f)
            for (int c = 0; c < C; ++c)
                if (values[i * C + c] != 0.f) bad = true;
        if (bad) atomicMin(&status[0], (unsigned long long)i);
    }
    if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(&status[1], 1ull);
}

// =========================================================== dispatch

cudaError_t launch_pass(const PassLaunch& pl, cudaStream_t st) {
    ProfScope ps("pass", st);
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

cudaError_t launch_transpose(const float* in, float* out, int H, int W, int C, int batch, cudaStream_t st) {
    dim3 grid((W + 31) / 32, (H + 31) / 32, batch);
    ProfScope ps("transpose", st);
    const long long stride = (long long)H * W * C;
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

cudaError_t launch_validate_sparse(const float* values, const float* mask, long long npx, int C,
                                   unsigned long long* status, cudaStream_t st) {
    k_validate_sparse<<<(unsigned)((npx + 255) / 256), 256, 0, st>>>(values, mask, npx, C, status);
    return cudaGetLastError();
}

}  // namespace sgwls_b200
