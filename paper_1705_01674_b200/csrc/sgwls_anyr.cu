// sgwls_anyr.cu -- one SG-WLS pass for ANY neighbourhood radius (r > kMaxR).
//
// The reference accepts every r >= 1 (proj/src/smoother.cpp:103-111); its
// presets stop at r = 4, which the tiled path (sgwls_tile.cuh, r <= 4) and the
// templated generic path (sgwls_pass.cuh, r <= 8) cover.  Beyond that this
// completeness path keeps the drop-in whole: one thread per band walks the
// band's n = m*Hl positions once (row-sum-pivot LDL^T on magnitudes, the same
// recurrence as every other kernel here, proj/src/banded.cpp:44-118) with its
// elimination window and factors in a line-interleaved global workspace, then
// back-substitutes into the band-solution array U that k4_average (sgwls_pass.cuh)
// merges.  Runtime r: no unrolling, no register window -- correct, not fast
// (a band is a serial chain of n dependent steps).
#include <cuda_runtime.h>

#include "sgwls_device.cuh"
#include "sgwls_kernels.h"
#include "sgwls_pass.cuh"
#include "sgwls_profile.h"

namespace sgwls_b200 {

namespace {

// Workspace of line L (element i at ws[i * NL + L], so a warp of lines reads rows):
//   cc  [n][r]        normalised couplings of every eliminated position
//   y   [n][C]        forward-eliminated right-hand side / pivot
//   A   [r+1][r+1]    window couplings, ring-indexed by position mod (r+1)
//   e   [r+1]         forward-eliminated all-ones right-hand side
//   gw  [r+1][C]      forward-eliminated right-hand side
//   gd  [r+1][CG]     guidance of the window positions
__host__ __device__ inline size_t anyr_ws_per_line(long long n, int r, int C, int Cg) {
    return (size_t)n * (r + C) + (size_t)(r + 1) * (r + 1) + (size_t)(r + 1) * (1 + C + Cg);
}

template <int C, int CG>
__global__ void __launch_bounds__(64) k_band_anyr(const PassGeom g, const float* __restrict__ src,
                                                 const float* __restrict__ guid, float* __restrict__ U,
                                                 float* __restrict__ ws, const float* __restrict__ lspat,
                                                 unsigned long long* __restrict__ err,
                                                 const __grid_constant__ WeightDev W) {
    const long long NL = (long long)g.nb * g.batch;
    const long long L = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (L >= NL) return;
    const int img = (int)(L / g.nb), b = (int)(L - (long long)img * g.nb);
    const int m = g.m, r = g.r, R1 = r + 1;
    const long long n = g.n;
    const int lo = band_lo(g, b);
    const float* F = src + (long long)img * g.img_stride;
    const float* G = guid + (long long)img * g.gimg_stride;
    float* cc = ws + L;
    float* yv = cc + (size_t)n * r * NL;
    float* A = yv + (size_t)n * C * NL;
    float* e = A + (size_t)R1 * R1 * NL;
    float* gw = e + (size_t)R1 * NL;
    float* gd = gw + (size_t)R1 * C * NL;
    auto a_at = [&](int i, int j) -> float& { return A[((size_t)i * R1 + j) * NL]; };
    for (int i = 0; i < R1 * R1; ++i) A[(size_t)i * NL] = 0.f;

    unsigned bad = 0xffffffffu;
    // forward: position k enters slot k % (r+1); position k - r is eliminated
    for (long long k = 0; k < n + r; ++k) {
        if (k < n) {
            const int y = (int)(k / m), jj = (int)(k - (long long)y * m);
            const int col = serp_col(lo, m, y, jj);
            const int s = (int)(k % R1);
            e[(size_t)s * NL] = 1.f;
            const float* fp = F + ((long long)y * g.Wl + col) * C;
            const float* gp = G + ((long long)y * g.Wl + col) * CG;
            float gk[CG];
#pragma unroll
            for (int c = 0; c < C; ++c) gw[((size_t)s * C + c) * NL] = fp[c];
#pragma unroll
            for (int c = 0; c < CG; ++c) {
                gk[c] = gp[c];
                gd[((size_t)s * CG + c) * NL] = gk[c];
            }
            for (int t = 1; t <= r && k - t >= 0; ++t) {
                const long long kp = k - t;
                const int yp = (int)(kp / m), jp = (int)(kp - (long long)yp * m);
                const int colp = serp_col(lo, m, yp, jp);
                const int sp = (int)(kp % R1);
                float r2 = 0.f;
#pragma unroll
                for (int c = 0; c < CG; ++c) {
                    const float d = gk[c] - gd[((size_t)sp * CG + c) * NL];
                    r2 = fmaf(d, d, r2);
                }
                const int dx = col - colp, dy = y - yp;
                // lambda * spatial factor by squared distance (host table), range factor as everywhere
                const float ls = lspat[dx * dx + dy * dy];
                const float lw = W.kind == 1 ? ls * fast_ex2(r2 * W.exp_k)
                                             : ls * fast_rcp(frac_range_pow(W, r2) + W.eps);
                if (!(lw >= 0.f) && (unsigned)kp < bad) bad = (unsigned)kp;  // NaN guidance: the reference's pivot failure
                a_at(sp, s) = lw;
            }
        }
        const long long pp = k - r;
        if (pp >= 0 && pp < n) {
            const int s0 = (int)(pp % R1);
            const float e0 = e[(size_t)s0 * NL];
            float piv = e0;
            const int nn = (int)((n - 1 - pp) < r ? (n - 1 - pp) : r);  // successors that exist
            for (int i = 1; i <= nn; ++i) piv += a_at(s0, (int)((pp + i) % R1));
            const float inv = 1.0f / piv;
            float g0[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                g0[c] = gw[((size_t)s0 * C + c) * NL];
                yv[((size_t)pp * C + c) * NL] = g0[c] * inv;
            }
            for (int i = 1; i <= r; ++i) {
                const int si = (int)((pp + i) % R1);
                const float a0i = i <= nn ? a_at(s0, si) : 0.f;
                const float ci = a0i * inv;
                cc[((size_t)pp * r + (i - 1)) * NL] = ci;
                if (i > nn) continue;
                e[(size_t)si * NL] = fmaf(ci, e0, e[(size_t)si * NL]);
#pragma unroll
                for (int c = 0; c < C; ++c) gw[((size_t)si * C + c) * NL] = fmaf(ci, g0[c], gw[((size_t)si * C + c) * NL]);
                for (int j = i + 1; j <= nn; ++j) {
                    const int sj = (int)((pp + j) % R1);
                    a_at(si, sj) = fmaf(a0i, a_at(s0, sj) * inv, a_at(si, sj));
                }
            }
            for (int j = 0; j < R1; ++j) a_at(s0, j) = 0.f;  // the slot is free for position pp + r + 1
        }
    }
    if (err != nullptr && bad != 0xffffffffu)
        atomicMin(err, ((unsigned long long)(unsigned)L << 32) | (unsigned long long)bad);

    // backward: u_p = y_p + sum_i cc[p][i] * u_{p+i}; the last r solutions ride in gw's ring
    // (free by now: slot p % (r+1), R1 slots >= r values)
    const long long rowstride = (long long)g.nb * m * C;
    float* Ui = U + (long long)img * g.Hl * rowstride;
    for (long long p = n - 1; p >= 0; --p) {
        float u[C];
#pragma unroll
        for (int c = 0; c < C; ++c) u[c] = yv[((size_t)p * C + c) * NL];
        for (int i = 1; i <= r && p + i < n; ++i) {
            const float ci = cc[((size_t)p * r + (i - 1)) * NL];
            const int si = (int)((p + i) % R1);
#pragma unroll
            for (int c = 0; c < C; ++c) u[c] = fmaf(ci, gw[((size_t)si * C + c) * NL], u[c]);
        }
        const int s = (int)(p % R1);
        const int y = (int)(p / m), jj = (int)(p - (long long)y * m);
        const int col = serp_col(lo, m, y, jj);
        float* up = Ui + (long long)y * rowstride + ((long long)b * m + (col - lo)) * C;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            gw[((size_t)s * C + c) * NL] = u[c];
            up[c] = u[c];
        }
    }
}

__global__ void k_anyr_lut(float* lut, size_t n, double lambda, int exp_kind, double sigma_s, double alpha_s,
                           double eps) {
    const size_t d2 = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (d2 >= n) return;
    const double sp = exp_kind ? exp(-(double)d2 / (2.0 * sigma_s * sigma_s))
                               : 1.0 / (pow(sqrt((double)d2), alpha_s) + eps);
    lut[d2] = (float)(lambda * sp);
}

template <int C>
cudaError_t launch_c(const PassLaunch& pl, cudaStream_t st) {
    const PassGeom& g = pl.geom;
    const long long NL = (long long)g.nb * g.batch;
    const dim3 grid((unsigned)((NL + 63) / 64));
    {
        ProfScope ps("k_band_anyr", st);
        switch (g.Cg) {
            case 1: k_band_anyr<C, 1><<<grid, 64, 0, st>>>(g, pl.src, pl.guid, pl.U, pl.anyr_ws, pl.anyr_lspat, pl.err, *pl.w); break;
            case 2: k_band_anyr<C, 2><<<grid, 64, 0, st>>>(g, pl.src, pl.guid, pl.U, pl.anyr_ws, pl.anyr_lspat, pl.err, *pl.w); break;
            case 3: k_band_anyr<C, 3><<<grid, 64, 0, st>>>(g, pl.src, pl.guid, pl.U, pl.anyr_ws, pl.anyr_lspat, pl.err, *pl.w); break;
            case 4: k_band_anyr<C, 4><<<grid, 64, 0, st>>>(g, pl.src, pl.guid, pl.U, pl.anyr_ws, pl.anyr_lspat, pl.err, *pl.w); break;
            default: return cudaErrorInvalidValue;
        }
    }
    {
        ProfScope ps("k4_average", st);
        const dim3 grid4((g.Wl + 31) / 32, (g.Hl + 31) / 32, g.batch);
        k4_average<C><<<grid4, dim3(32, 8), 0, st>>>(g, pl.U, pl.out, pl.transpose_out);
    }
    return cudaGetLastError();
}

}  // namespace

size_t anyr_ws_floats(const PassGeom& g) {
    return anyr_ws_per_line(g.n, g.r, g.C, g.Cg) * (size_t)g.nb * (size_t)g.batch;
}
// largest squared distance of an edge (k - t, k), t <= r: at most 2r columns and r rows apart
size_t anyr_lut_floats(int r) { return (size_t)5 * r * r + 2; }

cudaError_t launch_anyr_lut(float* lut, size_t n, double lambda, bool exp_kind, double sigma_s, double alpha_s,
                            double eps, cudaStream_t st) {
    k_anyr_lut<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(lut, n, lambda, exp_kind ? 1 : 0, sigma_s, alpha_s, eps);
    return cudaGetLastError();
}

// band solves into U, then the owner-computes averaging of the generic path
cudaError_t launch_pass_anyr(const PassLaunch& pl, cudaStream_t st) {
    switch (pl.geom.C) {
        case 1: return launch_c<1>(pl, st);
        case 2: return launch_c<2>(pl, st);
        case 3: return launch_c<3>(pl, st);
        case 4: return launch_c<4>(pl, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sgwls_b200
