// sgwls_fast.cuh -- K2: the sequential block-tridiagonal solve of the reduced
// system on the separators (r x r blocks), with the chunk records prefetched
// D separators ahead.  Used on the super-separators of the CTA-tiled path
// (sgwls_tile.cuh).  Row-sum pivots on magnitudes as everywhere else.
#pragma once

#include <cuda_runtime.h>

#include "sgwls_device.cuh"
#include "sgwls_kernels.h"

namespace sgwls_b200 {
namespace fast {

template <int R, int C>
struct Rec {
    static constexpr int NOFF = R * (R - 1) / 2;
    static constexpr int TOFF = 0;
    static constexpr int TCROSS = TOFF + NOFF;
    static constexpr int TE = TCROSS + R * R;
    static constexpr int TG = TE + R;
    static constexpr int HOFF = TG + R * C;
    static constexpr int HE = HOFF + NOFF;
    static constexpr int HG = HE + R;
    static constexpr int REC = HG + R * C;
    static constexpr int RS = (2 * R - 1) + C;
};

__device__ __forceinline__ int offi(int i, int j, int R) { return i * R - i * (i + 1) / 2 + (j - i - 1); }

// ===================================================================== K2

template <int R, int C>
struct SepRec {
    static constexpr int NO = R * (R - 1) / 2 > 0 ? R * (R - 1) / 2 : 1;
    float toff[NO], tcross[R][R], te[R], tg[R][C];
    float hoff[NO], he[R], hg[R][C];
};

template <int R, int C>
__device__ __forceinline__ void load_sep(SepRec<R, C>& s, const float* __restrict__ rec, int sep, int NS,
                                         long long NLl, int L) {
    using RL = Rec<R, C>;
    if (sep < NS) {
        const float* t = rec + (long long)sep * RL::REC * NLl + L;
        const float* h = rec + (long long)(sep + 1) * RL::REC * NLl + L;
#pragma unroll
        for (int i = 0; i < RL::NOFF; ++i) {
            s.toff[i] = t[(RL::TOFF + i) * NLl];
            s.hoff[i] = h[(RL::HOFF + i) * NLl];
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
#pragma unroll
            for (int k = 0; k < R; ++k) s.tcross[i][k] = sep > 0 ? t[(RL::TCROSS + i * R + k) * NLl] : 0.f;
            s.te[i] = t[(RL::TE + i) * NLl];
            s.he[i] = h[(RL::HE + i) * NLl];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                s.tg[i][c] = t[(RL::TG + i * C + c) * NLl];
                s.hg[i][c] = h[(RL::HG + i * C + c) * NLl];
            }
        }
    }
}

template <int R, int C, int D>
__global__ void __launch_bounds__(64) k2_fast(const PassGeom g, const float* __restrict__ rec,
                                              float* __restrict__ rs, float* __restrict__ z) {
    using RL = Rec<R, C>;
    constexpr int W2 = 2 * R;
    const int NL = g.nb * g.batch;
    const int L = blockIdx.x * blockDim.x + threadIdx.x;
    if (L >= NL) return;
    const long long NLl = NL;
    const int NS = g.P - 1;

    float e[W2], gg[W2][C], A[W2][W2];
#pragma unroll
    for (int i = 0; i < W2; ++i) {
        e[i] = 0.f;
#pragma unroll
        for (int c = 0; c < C; ++c) gg[i][c] = 0.f;
#pragma unroll
        for (int k = 0; k < W2; ++k) A[i][k] = 0.f;
    }
    SepRec<R, C> ring[D];
#pragma unroll
    for (int u = 0; u < D; ++u) load_sep<R, C>(ring[u], rec, u, NS, NLl, L);

    auto enter = [&](const SepRec<R, C>& s) {
#pragma unroll
        for (int mm = 0; mm < R; ++mm) {
            e[R + mm] = s.te[mm] + s.he[mm];
#pragma unroll
            for (int c = 0; c < C; ++c) gg[R + mm][c] = s.tg[mm][c] + s.hg[mm][c];
#pragma unroll
            for (int m2 = mm + 1; m2 < R; ++m2) A[R + mm][R + m2] = s.toff[offi(mm, m2, R)] + s.hoff[offi(mm, m2, R)];
#pragma unroll
            for (int mp = 0; mp < R; ++mp) A[mp][R + mm] = s.tcross[mm][mp];
        }
    };
    auto clear_hi = [&]() {
#pragma unroll
        for (int i = R; i < W2; ++i) {
            e[i] = 0.f;
#pragma unroll
            for (int c = 0; c < C; ++c) gg[i][c] = 0.f;
#pragma unroll
            for (int k = 0; k < W2; ++k) {
                A[i][k] = 0.f;
                A[k][i] = 0.f;
            }
        }
    };
    auto shift = [&]() {
#pragma unroll
        for (int i = 0; i < R; ++i) {
            e[i] = e[i + R];
#pragma unroll
            for (int c = 0; c < C; ++c) gg[i][c] = gg[i + R][c];
#pragma unroll
            for (int k = i + 1; k < R; ++k) A[i][k] = A[i + R][k + R];
        }
    };

    clear_hi();
    enter(ring[0]);
    load_sep<R, C>(ring[0], rec, D, NS, NLl, L);
    shift();
    for (int sb = 0; sb < NS; sb += D) {
#pragma unroll
        for (int u = 0; u < D; ++u) {
            const int s = sb + u;
            if (s < NS) {
                clear_hi();
                if (s + 1 < NS) {
                    enter(ring[(u + 1) % D]);
                    load_sep<R, C>(ring[(u + 1) % D], rec, s + 1 + D, NS, NLl, L);
                }
#pragma unroll
                for (int mm = 0; mm < R; ++mm) {
                    float piv = e[mm];
#pragma unroll
                    for (int i = mm + 1; i < W2; ++i) piv += A[mm][i];
                    const float inv = fast_rcp(piv);
                    float cc[W2];
#pragma unroll
                    for (int i = mm + 1; i < W2; ++i) cc[i] = A[mm][i] * inv;
#pragma unroll
                    for (int i = mm + 1; i < W2; ++i) {
                        e[i] = fmaf(cc[i], e[mm], e[i]);
#pragma unroll
                        for (int c = 0; c < C; ++c) gg[i][c] = fmaf(cc[i], gg[mm][c], gg[i][c]);
#pragma unroll
                        for (int k = i + 1; k < W2; ++k) A[i][k] = fmaf(A[mm][i], cc[k], A[i][k]);
                    }
                    float* o = rs + ((long long)(s * R + mm) * RL::RS) * NLl + L;
#pragma unroll
                    for (int i = mm + 1; i < W2; ++i) o[(i - mm - 1) * NLl] = cc[i];
#pragma unroll
                    for (int c = 0; c < C; ++c) o[(2 * R - 1 + c) * NLl] = gg[mm][c] * inv;
                }
                shift();
            }
        }
    }
    // back substitution with the per-separator coefficients prefetched D ahead
    constexpr int PER = R * RL::RS;
    float bring[D][PER];
    auto load_bs = [&](float (&dst)[PER], int s) {
        if (s >= 0) {
            const float* o = rs + ((long long)(s * R) * RL::RS) * NLl + L;
#pragma unroll
            for (int i = 0; i < PER; ++i) dst[i] = o[i * NLl];
        }
    };
#pragma unroll
    for (int u = 0; u < D; ++u) load_bs(bring[u], NS - 1 - u);
    float zn[R][C];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
        for (int c = 0; c < C; ++c) zn[i][c] = 0.f;
    for (int sb = NS - 1; sb >= 0; sb -= D) {
#pragma unroll
        for (int u = 0; u < D; ++u) {
            const int s = sb - u;
            if (s >= 0) {
                const float* o = bring[u];
                float zc[R][C];
#pragma unroll
                for (int mm = R - 1; mm >= 0; --mm) {
#pragma unroll
                    for (int c = 0; c < C; ++c) zc[mm][c] = o[mm * RL::RS + 2 * R - 1 + c];
#pragma unroll
                    for (int i = mm + 1; i < W2; ++i) {
                        const float ci = o[mm * RL::RS + (i - mm - 1)];
#pragma unroll
                        for (int c = 0; c < C; ++c)
                            zc[mm][c] = fmaf(ci, (i < R) ? zc[i < R ? i : 0][c] : zn[i >= R ? i - R : 0][c], zc[mm][c]);
                    }
                }
                float* zo = z + (long long)s * R * C * NLl + L;
#pragma unroll
                for (int mm = 0; mm < R; ++mm)
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        zo[(mm * C + c) * NLl] = zc[mm][c];
                        zn[mm][c] = zc[mm][c];
                    }
                load_bs(bring[u], s - D);
            }
        }
    }
}


// ---------------------------------------------------------------- K2 staged
//
// Same elimination as k2_fast, but the records of a window of WS separators
// for the warp's 32 lines are brought into shared memory cooperatively
// (coalesced 128-byte rows, cp.async, double-buffered), so the loop-carried
// elimination never waits on a dependent global load.

__device__ __forceinline__ void cp_async4(float* dst_smem, const float* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__host__ __device__ constexpr int k2_window(int R, int C) {
    return Rec<1, 1>::REC * 0 + ((R * (R - 1) + R * R + 2 * R + 2 * R * C) <= 12 ? 16
                                 : ((R * (R - 1) + R * R + 2 * R + 2 * R * C) <= 24 ? 8 : 4));
}

template <int R, int C>
__global__ void __launch_bounds__(32) k2_stage(const PassGeom g, const float* __restrict__ rec,
                                               float* __restrict__ rs, float* __restrict__ z) {
    using RL = Rec<R, C>;
    constexpr int NRF = RL::REC;
    constexpr int WS = k2_window(R, C);
    constexpr int W2 = 2 * R;
    extern __shared__ float sm[];
    const int lane = threadIdx.x;
    const int NL = g.nb * g.batch;
    const int L0 = blockIdx.x * 32;
    const int L = L0 + lane;
    const bool ok = L < NL;
    const long long NLl = NL;
    const int NS = g.P - 1;
    const int NREC = g.P;

    auto rbuf = [&](int b, int ri, int f) -> float* { return sm + (((b * (WS + 2) + ri) * NRF + f) << 5); };
    auto stage = [&](int b, int w0) {
        for (int ri = 0; ri <= WS + 1; ++ri) {  // window's records + the next block's two
            const int idx = w0 + ri;
            if (idx < NREC && ok) {
#pragma unroll
                for (int f = 0; f < NRF; ++f) cp_async4(rbuf(b, ri, f) + lane, rec + ((long long)idx * NRF + f) * NLl + L);
            }
        }
        cp_async_commit();
    };

    float e[W2], gg[W2][C], A[W2][W2];
#pragma unroll
    for (int i = 0; i < W2; ++i) {
        e[i] = 0.f;
#pragma unroll
        for (int c = 0; c < C; ++c) gg[i][c] = 0.f;
#pragma unroll
        for (int k = 0; k < W2; ++k) A[i][k] = 0.f;
    }
    auto clear_hi = [&]() {
#pragma unroll
        for (int i = R; i < W2; ++i) {
            e[i] = 0.f;
#pragma unroll
            for (int c = 0; c < C; ++c) gg[i][c] = 0.f;
#pragma unroll
            for (int k = 0; k < W2; ++k) {
                A[i][k] = 0.f;
                A[k][i] = 0.f;
            }
        }
    };
    auto enter = [&](int b, int ri, int sep) {  // tail of record ri + head of record ri+1
        const float* base = sm + lane;
        auto T = [&](int f) { return rbuf(b, ri, f)[lane]; };
        auto H = [&](int f) { return rbuf(b, ri + 1, f)[lane]; };
        (void)base;
#pragma unroll
        for (int mm = 0; mm < R; ++mm) {
            e[R + mm] = T(RL::TE + mm) + H(RL::HE + mm);
#pragma unroll
            for (int c = 0; c < C; ++c) gg[R + mm][c] = T(RL::TG + mm * C + c) + H(RL::HG + mm * C + c);
#pragma unroll
            for (int m2 = mm + 1; m2 < R; ++m2)
                A[R + mm][R + m2] = T(RL::TOFF + offi(mm, m2, R)) + H(RL::HOFF + offi(mm, m2, R));
#pragma unroll
            for (int mp = 0; mp < R; ++mp) A[mp][R + mm] = sep > 0 ? T(RL::TCROSS + mm * R + mp) : 0.f;
        }
    };
    auto shift = [&]() {
#pragma unroll
        for (int i = 0; i < R; ++i) {
            e[i] = e[i + R];
#pragma unroll
            for (int c = 0; c < C; ++c) gg[i][c] = gg[i + R][c];
#pragma unroll
            for (int k = i + 1; k < R; ++k) A[i][k] = A[i + R][k + R];
        }
    };

    // ---- forward over windows of WS separators
    const int nwin = (NS + WS - 1) / WS;
    stage(0, 0);
    for (int wdx = 0; wdx < nwin; ++wdx) {
        const int b = wdx & 1;
        if (wdx + 1 < nwin) {
            stage(b ^ 1, (wdx + 1) * WS);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        const int s0 = wdx * WS;
        const int s1 = min(NS, s0 + WS);
        for (int s = s0; s < s1; ++s) {
            const int ri = s - s0;
            if (s == 0) {
                clear_hi();
                enter(b, 0, 0);
                shift();
            }
            clear_hi();
            if (s + 1 < NS) enter(b, ri + 1, s + 1);  // records s+1 (tail), s+2 (head)
#pragma unroll
            for (int mm = 0; mm < R; ++mm) {
                float piv = e[mm];
#pragma unroll
                for (int i = mm + 1; i < W2; ++i) piv += A[mm][i];
                const float inv = fast_rcp(piv);
                float cc[W2];
#pragma unroll
                for (int i = mm + 1; i < W2; ++i) cc[i] = A[mm][i] * inv;
#pragma unroll
                for (int i = mm + 1; i < W2; ++i) {
                    e[i] = fmaf(cc[i], e[mm], e[i]);
#pragma unroll
                    for (int c = 0; c < C; ++c) gg[i][c] = fmaf(cc[i], gg[mm][c], gg[i][c]);
#pragma unroll
                    for (int k = i + 1; k < W2; ++k) A[i][k] = fmaf(A[mm][i], cc[k], A[i][k]);
                }
                if (ok) {
                    float* o = rs + ((long long)(s * R + mm) * RL::RS) * NLl + L;
#pragma unroll
                    for (int i = mm + 1; i < W2; ++i) o[(i - mm - 1) * NLl] = cc[i];
#pragma unroll
                    for (int c = 0; c < C; ++c) o[(2 * R - 1 + c) * NLl] = gg[mm][c] * inv;
                }
            }
            shift();
        }
        __syncwarp();
    }
    __syncwarp();
    // ---- back substitution over windows (reverse), coefficients staged the same way
    constexpr int PER = R * RL::RS;
    auto bbuf = [&](int b, int si, int f) -> float* { return sm + (((b * WS + si) * PER + f) << 5); };
    auto stage_bs = [&](int b, int shi) {  // separators shi-WS+1 .. shi
        for (int si = 0; si < WS; ++si) {
            const int s = shi - si;
            if (s >= 0 && ok) {
#pragma unroll
                for (int f = 0; f < PER; ++f)
                    cp_async4(bbuf(b, si, f) + lane, rs + ((long long)(s * R) * RL::RS + f) * NLl + L);
            }
        }
        cp_async_commit();
    };
    float zn[R][C];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
        for (int c = 0; c < C; ++c) zn[i][c] = 0.f;
    stage_bs(0, NS - 1);
    for (int wdx = 0; wdx < nwin; ++wdx) {
        const int b = wdx & 1;
        const int shi = NS - 1 - wdx * WS;
        if (wdx + 1 < nwin) {
            stage_bs(b ^ 1, shi - WS);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        for (int si = 0; si < WS && shi - si >= 0; ++si) {
            const int s = shi - si;
            float zc[R][C];
#pragma unroll
            for (int mm = R - 1; mm >= 0; --mm) {
#pragma unroll
                for (int c = 0; c < C; ++c) zc[mm][c] = bbuf(b, si, mm * RL::RS + 2 * R - 1 + c)[lane];
#pragma unroll
                for (int i = mm + 1; i < W2; ++i) {
                    const float ci = bbuf(b, si, mm * RL::RS + (i - mm - 1))[lane];
#pragma unroll
                    for (int c = 0; c < C; ++c)
                        zc[mm][c] = fmaf(ci, (i < R) ? zc[i < R ? i : 0][c] : zn[i >= R ? i - R : 0][c], zc[mm][c]);
                }
            }
            if (ok) {
                float* zo = z + (long long)s * R * C * NLl + L;
#pragma unroll
                for (int mm = 0; mm < R; ++mm)
#pragma unroll
                    for (int c = 0; c < C; ++c) zo[(mm * C + c) * NLl] = zc[mm][c];
            }
#pragma unroll
            for (int mm = 0; mm < R; ++mm)
#pragma unroll
                for (int c = 0; c < C; ++c) zn[mm][c] = zc[mm][c];
        }
        __syncwarp();
    }
}

template <int R, int C>
__host__ inline size_t k2_stage_smem() {
    using RL = Rec<R, C>;
    constexpr int WS = k2_window(R, C);
    const size_t fwd = (size_t)2 * (WS + 2) * RL::REC * 32;
    const size_t bwd = (size_t)2 * WS * R * RL::RS * 32;
    return (fwd > bwd ? fwd : bwd) * sizeof(float);
}

}  // namespace fast
}  // namespace sgwls_b200
