// sgwls_pass.cuh -- the SG-WLS pass as an exact partitioned band solver.
//
// One pass (proj/src/smoother.cpp:51-99) solves every band's 1-D WLS system and
// averages the overlapping band solutions.  A band of n = m*Hl positions is far
// too long and there are far too few bands (360..2730) to give one band to one
// thread, so each band is cut into P chunks of whole image
// rows and solved EXACTLY by a separator (partition) method:
//
//   chunk j = positions [a_j, a_{j+1}); its last r positions form the separator
//   sigma_j; the rest is the interior I_j.  Interiors of different chunks do not
//   couple once the separators are known.
//
//   K1 k1_spike_forward  (band x chunk)  eliminates I_j top-down while carrying
//        the couplings to sigma_{j-1} ("spike" columns).  Emits the chunk's
//        contribution to the reduced system on the separators: the Schur block
//        of sigma_j and its coupling to sigma_{j-1} (tail), and the update of
//        sigma_{j-1}'s own block (head).
//   K2 k2_reduced        (band)          solves the block-tridiagonal reduced
//        system (r x r blocks, P-1 of them) -> separator values z.
//   K3 k3_interior       (band x chunk)  re-walks the chunk, solves I_j with the
//        separator values as known boundary terms (forward elimination into
//        shared memory, back substitution), writes band solutions to U.
//   K4 k4_average        (pixel tile)    owner-computes averaging over the bands
//        covering each pixel in increasing centre order (deterministic), divides
//        by the analytic count and writes the next pass's layout (transposed).
//
// Every elimination uses magnitudes and the row-sum pivot (sgwls_device.cuh).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "sgwls_device.cuh"
#include "sgwls_kernels.h"
#include "sgwls_profile.h"

namespace sgwls_b200 {

// ------------------------------------------------------------ record layout

template <int R, int C>
struct RecLayout {
    static constexpr int NOFF = R * (R - 1) / 2;
    static constexpr int TOFF = 0;
    static constexpr int TCROSS = TOFF + NOFF;
    static constexpr int TE = TCROSS + R * R;
    static constexpr int TG = TE + R;
    static constexpr int HOFF = TG + R * C;
    static constexpr int HE = HOFF + NOFF;
    static constexpr int HG = HE + R;
    static constexpr int REC = HG + R * C;
    static constexpr int RS = (2 * R - 1) + C;  // per reduced scalar: couplings + y
};

template <int I, int J, int R>
struct OffIdx {  // index of pair (I<J) in a packed strictly-upper R x R
    static constexpr int v = I * R - I * (I + 1) / 2 + (J - I - 1);
};

__device__ __forceinline__ int off_idx(int i, int j, int R) { return i * R - i * (i + 1) / 2 + (j - i - 1); }

// Guidance ring entry: previous positions' guidance + 2-D coordinates.
template <int R>
struct Ring {
    float g[R > 0 ? R : 1][kMaxCg];
    int row[R > 0 ? R : 1];
    int col[R > 0 ? R : 1];
    int pos[R > 0 ? R : 1];
};

__device__ __forceinline__ void load_guid(const float* __restrict__ G, const PassGeom& g, int y, int col,
                                          float out[kMaxCg]) {
    const float* p = G + ((long long)y * g.Wl + col) * g.Cg;
#pragma unroll
    for (int c = 0; c < kMaxCg; ++c) out[c] = c < g.Cg ? __ldg(p + c) : 0.f;
}

// Prime the ring with positions a-R .. a-1 of the band (the previous chunk's separator).
template <int R>
__device__ __forceinline__ void ring_prime(Ring<R>& rg, const float* __restrict__ G, const PassGeom& g, int lo,
                                           int a) {
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int p = a - R + i;
        rg.pos[i] = p;
        rg.row[i] = 0;
        rg.col[i] = 0;
#pragma unroll
        for (int c = 0; c < kMaxCg; ++c) rg.g[i][c] = 0.f;
        if (p >= 0) {
            const int y = p / g.m;
            const int jj = p - y * g.m;
            const int col = serp_col(lo, g.m, y, jj);
            rg.row[i] = y;
            rg.col[i] = col;
            load_guid(G, g, y, col, rg.g[i]);
        }
    }
}

template <int R>
__device__ __forceinline__ void ring_push(Ring<R>& rg, int q, int y, int col, const float gq[kMaxCg]) {
#pragma unroll
    for (int i = 0; i + 1 < R; ++i) {
        rg.pos[i] = rg.pos[i + 1];
        rg.row[i] = rg.row[i + 1];
        rg.col[i] = rg.col[i + 1];
#pragma unroll
        for (int c = 0; c < kMaxCg; ++c) rg.g[i][c] = rg.g[i + 1][c];
    }
    rg.pos[R - 1] = q;
    rg.row[R - 1] = y;
    rg.col[R - 1] = col;
#pragma unroll
    for (int c = 0; c < kMaxCg; ++c) rg.g[R - 1][c] = gq[c];
}

// weight between ring entry i and the entering position (y, col, gq)
template <int R>
__device__ __forceinline__ float pair_weight(const WeightDev& W, const PassGeom& g, const Ring<R>& rg, int i, int y,
                                             int col, const float gq[kMaxCg]) {
    const int dr = y - rg.row[i], dc = col - rg.col[i];
    float range2 = 0.f;
#pragma unroll
    for (int c = 0; c < kMaxCg; ++c) {
        if (c < g.Cg) {
            const float d = gq[c] - rg.g[i][c];
            range2 = fmaf(d, d, range2);
        }
    }
    return guidance_weight(W, range2, dr * dr + dc * dc);
}

__device__ __forceinline__ void report_nan(unsigned long long* err, int line, int k0) {
    const unsigned long long key = ((unsigned long long)(unsigned)line << 32) | (unsigned)k0;
    atomicMin(err, key);
}

// ===================================================================== K1

template <int R, int C>
__global__ void __launch_bounds__(128) k1_spike_forward(const PassGeom g, const float* __restrict__ src,
                                                        const float* __restrict__ guid, float* __restrict__ rec,
                                                        const __grid_constant__ WeightDev W) {
    using RL = RecLayout<R, C>;
    const int NL = g.nb * g.batch;
    const int L = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (L >= NL) return;
    const int img = L / g.nb, b = L - img * g.nb;
    const float* __restrict__ F = src + img * g.img_stride;
    const float* __restrict__ G = guid + img * g.gimg_stride;
    const int m = g.m;
    const int lo = band_lo(g, b);
    const int y0 = chunk_row(g, j), y1 = chunk_row(g, j + 1);
    const int a = y0 * m, aend = y1 * m;
    const bool last = (j == g.P - 1);
    const int elim_end = last ? aend : aend - R;
    const float lam = W.lam;

    Ring<R> rg;
    ring_prime<R>(rg, G, g, lo, a);

    float e[R + 1], gg[R + 1][C], A[R + 1][R + 1], Q[R + 1][R];
    float he[R], hg[R][C], hoff[R][R];
#pragma unroll
    for (int i = 0; i <= R; ++i) {
        e[i] = 0.f;
#pragma unroll
        for (int c = 0; c < C; ++c) gg[i][c] = 0.f;
#pragma unroll
        for (int k = 0; k <= R; ++k) A[i][k] = 0.f;
#pragma unroll
        for (int k = 0; k < R; ++k) Q[i][k] = 0.f;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
        he[i] = 0.f;
#pragma unroll
        for (int c = 0; c < C; ++c) hg[i][c] = 0.f;
#pragma unroll
        for (int k = 0; k < R; ++k) hoff[i][k] = 0.f;
    }

    int y = y0, jj = 0;
    const int qend = aend + (last ? R : 0);
    for (int q = a; q < qend; ++q) {
        // ---- enter position q into slot R
        e[R] = 0.f;
#pragma unroll
        for (int c = 0; c < C; ++c) gg[R][c] = 0.f;
#pragma unroll
        for (int i = 0; i < R; ++i) {
            A[i][R] = 0.f;
            Q[R][i] = 0.f;
        }
        if (q < aend) {
            const int col = serp_col(lo, m, y, jj);
            const float* px = F + ((long long)y * g.Wl + col) * C;
#pragma unroll
            for (int c = 0; c < C; ++c) gg[R][c] = __ldg(px + c);
            e[R] = 1.f;
            float gq[kMaxCg];
            load_guid(G, g, y, col, gq);
#pragma unroll
            for (int t = 1; t <= R; ++t) {
                const int ri = R - t;
                const int p = rg.pos[ri];
                if (p >= 0) {
                    const float lw = lam * pair_weight<R>(W, g, rg, ri, y, col, gq);
                    if (p >= a) {
                        A[R - t][R] = lw;
                    } else {
                        const int sidx = p - (a - R);
#pragma unroll
                        for (int mm = 0; mm < R; ++mm)
                            if (sidx == mm) Q[R][mm] = lw;
                    }
                }
            }
            ring_push<R>(rg, q, y, col, gq);
            if (++jj == m) {
                jj = 0;
                ++y;
            }
        }
        // ---- eliminate slot 0 (position q - R)
        const int k = q - R;
        if (k >= a && k < elim_end) {
            float s = e[0];
#pragma unroll
            for (int i = 1; i <= R; ++i) s += A[0][i];
#pragma unroll
            for (int mm = 0; mm < R; ++mm) s += Q[0][mm];
            const float inv = fast_rcp(s);
            float cc[R + 1];
#pragma unroll
            for (int i = 1; i <= R; ++i) cc[i] = A[0][i] * inv;
#pragma unroll
            for (int i = 1; i <= R; ++i) {
                e[i] = fmaf(cc[i], e[0], e[i]);
#pragma unroll
                for (int c = 0; c < C; ++c) gg[i][c] = fmaf(cc[i], gg[0][c], gg[i][c]);
#pragma unroll
                for (int k2 = i + 1; k2 <= R; ++k2) A[i][k2] = fmaf(A[0][i], cc[k2], A[i][k2]);
#pragma unroll
                for (int mm = 0; mm < R; ++mm) Q[i][mm] = fmaf(cc[i], Q[0][mm], Q[i][mm]);
            }
            if (j > 0) {
#pragma unroll
                for (int mm = 0; mm < R; ++mm) {
                    const float d = Q[0][mm] * inv;
                    he[mm] = fmaf(d, e[0], he[mm]);
#pragma unroll
                    for (int c = 0; c < C; ++c) hg[mm][c] = fmaf(d, gg[0][c], hg[mm][c]);
#pragma unroll
                    for (int m2 = mm + 1; m2 < R; ++m2) hoff[mm][m2] = fmaf(d, Q[0][m2], hoff[mm][m2]);
                }
            }
        }
        // ---- shift the window
        if (q + 1 < qend || !last) {
#pragma unroll
            for (int i = 0; i < R; ++i) {
                e[i] = e[i + 1];
#pragma unroll
                for (int c = 0; c < C; ++c) gg[i][c] = gg[i + 1][c];
#pragma unroll
                for (int k2 = i + 1; k2 < R; ++k2) A[i][k2] = A[i + 1][k2 + 1];
#pragma unroll
                for (int mm = 0; mm < R; ++mm) Q[i][mm] = Q[i + 1][mm];
            }
        }
    }

    const long long NLl = NL;
    float* base = rec + (long long)j * RL::REC * NLl + L;
    if (!last) {
#pragma unroll
        for (int i = 0; i < R; ++i) {
#pragma unroll
            for (int k2 = i + 1; k2 < R; ++k2) base[(RL::TOFF + off_idx(i, k2, R)) * NLl] = A[i][k2];
#pragma unroll
            for (int mm = 0; mm < R; ++mm) base[(RL::TCROSS + i * R + mm) * NLl] = Q[i][mm];
            base[(RL::TE + i) * NLl] = e[i];
#pragma unroll
            for (int c = 0; c < C; ++c) base[(RL::TG + i * C + c) * NLl] = gg[i][c];
        }
    }
    if (j > 0) {
#pragma unroll
        for (int mm = 0; mm < R; ++mm) {
#pragma unroll
            for (int m2 = mm + 1; m2 < R; ++m2) base[(RL::HOFF + off_idx(mm, m2, R)) * NLl] = hoff[mm][m2];
            base[(RL::HE + mm) * NLl] = he[mm];
#pragma unroll
            for (int c = 0; c < C; ++c) base[(RL::HG + mm * C + c) * NLl] = hg[mm][c];
        }
    }
}

// ===================================================================== K2

template <int R, int C>
__global__ void __launch_bounds__(64) k2_reduced(const PassGeom g, const float* __restrict__ rec,
                                                 float* __restrict__ rs, float* __restrict__ z) {
    using RL = RecLayout<R, C>;
    constexpr int W2 = 2 * R;  // two blocks of slots
    const int NL = g.nb * g.batch;
    const int L = blockIdx.x * blockDim.x + threadIdx.x;
    if (L >= NL) return;
    const long long NLl = NL;
    const int NS = g.P - 1;  // separators

    float e[W2], gg[W2][C], A[W2][W2];
#pragma unroll
    for (int i = 0; i < W2; ++i) {
        e[i] = 0.f;
#pragma unroll
        for (int c = 0; c < C; ++c) gg[i][c] = 0.f;
#pragma unroll
        for (int k = 0; k < W2; ++k) A[i][k] = 0.f;
    }

    // enter separator block s into slots R..2R-1 (cross coupling to slots 0..R-1)
    auto enter = [&](int s) {
        const float* t = rec + (long long)s * RL::REC * NLl + L;       // tail of chunk s
        const float* h = rec + (long long)(s + 1) * RL::REC * NLl + L;  // head of chunk s+1
#pragma unroll
        for (int mm = 0; mm < R; ++mm) {
            e[R + mm] = t[(RL::TE + mm) * NLl] + h[(RL::HE + mm) * NLl];
#pragma unroll
            for (int c = 0; c < C; ++c) gg[R + mm][c] = t[(RL::TG + mm * C + c) * NLl] + h[(RL::HG + mm * C + c) * NLl];
#pragma unroll
            for (int m2 = mm + 1; m2 < R; ++m2)
                A[R + mm][R + m2] = t[(RL::TOFF + off_idx(mm, m2, R)) * NLl] + h[(RL::HOFF + off_idx(mm, m2, R)) * NLl];
#pragma unroll
            for (int mp = 0; mp < R; ++mp) A[mp][R + mm] = (s > 0) ? t[(RL::TCROSS + mm * R + mp) * NLl] : 0.f;
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
    enter(0);
    shift();
    for (int s = 0; s < NS; ++s) {
        clear_hi();
        if (s + 1 < NS) enter(s + 1);
#pragma unroll
        for (int mm = 0; mm < R; ++mm) {
            float piv = e[mm];
#pragma unroll
            for (int i = mm + 1; i < W2; ++i) piv += A[mm][i];
            const float inv = 1.0f / piv;
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
    // back substitution, block by block
    float zn[R][C];  // z of block s+1
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
        for (int c = 0; c < C; ++c) zn[i][c] = 0.f;
    for (int s = NS - 1; s >= 0; --s) {
        float zc[R][C];
#pragma unroll
        for (int mm = R - 1; mm >= 0; --mm) {
            const float* o = rs + ((long long)(s * R + mm) * RL::RS) * NLl + L;
#pragma unroll
            for (int c = 0; c < C; ++c) zc[mm][c] = o[(2 * R - 1 + c) * NLl];
#pragma unroll
            for (int i = mm + 1; i < W2; ++i) {
                const float ci = o[(i - mm - 1) * NLl];
#pragma unroll
                for (int c = 0; c < C; ++c) zc[mm][c] = fmaf(ci, (i < R) ? zc[i][c] : zn[i - R][c], zc[mm][c]);
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
    }
}

// ===================================================================== K3

template <int R, int C>
__global__ void __launch_bounds__(128) k3_interior(const PassGeom g, const float* __restrict__ src,
                                                   const float* __restrict__ guid, const float* __restrict__ z,
                                                   float* __restrict__ U, unsigned long long* __restrict__ err,
                                                   const __grid_constant__ WeightDev W) {
    extern __shared__ float sm[];
    constexpr int NF = R + C;
    const int NL = g.nb * g.batch;
    const int L = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (L >= NL) return;
    const int tid = threadIdx.x, bd = blockDim.x;
    const int img = L / g.nb, b = L - img * g.nb;
    const float* __restrict__ F = src + img * g.img_stride;
    const float* __restrict__ G = guid + img * g.gimg_stride;
    const int m = g.m;
    const int lo = band_lo(g, b);
    const int y0 = chunk_row(g, j), y1 = chunk_row(g, j + 1);
    const int a = y0 * m, aend = y1 * m;
    const bool last = (j == g.P - 1);
    const int end = last ? aend : aend - R;
    const float lam = W.lam;
    const long long NLl = NL;

    float zl[R][C], zr[R][C];
#pragma unroll
    for (int mm = 0; mm < R; ++mm)
#pragma unroll
        for (int c = 0; c < C; ++c) {
            zl[mm][c] = (j > 0) ? z[((long long)(j - 1) * R * C + mm * C + c) * NLl + L] : 0.f;
            zr[mm][c] = (!last) ? z[((long long)j * R * C + mm * C + c) * NLl + L] : 0.f;
        }

    Ring<R> rg;
    ring_prime<R>(rg, G, g, lo, a);

    float e[R + 1], gg[R + 1][C], A[R + 1][R + 1];
#pragma unroll
    for (int i = 0; i <= R; ++i) {
        e[i] = 0.f;
#pragma unroll
        for (int c = 0; c < C; ++c) gg[i][c] = 0.f;
#pragma unroll
        for (int k = 0; k <= R; ++k) A[i][k] = 0.f;
    }

    int y = y0, jj = 0;
    const int qend = aend + (last ? R : 0);
    for (int q = a; q < qend; ++q) {
        e[R] = 0.f;
#pragma unroll
        for (int c = 0; c < C; ++c) gg[R][c] = 0.f;
#pragma unroll
        for (int i = 0; i < R; ++i) A[i][R] = 0.f;
        if (q < aend) {
            const int col = serp_col(lo, m, y, jj);
            const bool kq = (q >= end);  // q is a known separator position of sigma_j
            if (!kq) {
                const float* px = F + ((long long)y * g.Wl + col) * C;
#pragma unroll
                for (int c = 0; c < C; ++c) gg[R][c] = __ldg(px + c);
                e[R] = 1.f;
            }
            float gq[kMaxCg];
            load_guid(G, g, y, col, gq);
#pragma unroll
            for (int t = 1; t <= R; ++t) {
                const int ri = R - t;
                const int p = rg.pos[ri];
                if (p >= 0) {
                    const float w = pair_weight<R>(W, g, rg, ri, y, col, gq);
                    if (err != nullptr && !(w >= 0.f)) report_nan(err, L, p);
                    const float lw = lam * w;
                    const bool kp = (p < a);  // partner is a known position of sigma_{j-1}
                    if (kq && p >= end) {
                        // both in sigma_j: known-known coupling, nothing to eliminate
                    } else if (!kq && !kp) {
                        A[R - t][R] = lw;
                    } else if (!kq && kp) {
                        const int sidx = p - (a - R);
                        e[R] += lw;
#pragma unroll
                        for (int mm = 0; mm < R; ++mm)
                            if (sidx == mm) {
#pragma unroll
                                for (int c = 0; c < C; ++c) gg[R][c] = fmaf(lw, zl[mm][c], gg[R][c]);
                            }
                    } else if (kq && !kp) {
                        const int sidx = q - end;
                        e[R - t] += lw;
#pragma unroll
                        for (int mm = 0; mm < R; ++mm)
                            if (sidx == mm) {
#pragma unroll
                                for (int c = 0; c < C; ++c) gg[R - t][c] = fmaf(lw, zr[mm][c], gg[R - t][c]);
                            }
                    }
                }
            }
            ring_push<R>(rg, q, y, col, gq);
            if (++jj == m) {
                jj = 0;
                ++y;
            }
        }
        const int k = q - R;
        if (k >= a && k < end) {
            float s = e[0];
#pragma unroll
            for (int i = 1; i <= R; ++i) s += A[0][i];
            const float inv = fast_rcp(s);
            float cc[R + 1];
#pragma unroll
            for (int i = 1; i <= R; ++i) cc[i] = A[0][i] * inv;
#pragma unroll
            for (int i = 1; i <= R; ++i) {
                e[i] = fmaf(cc[i], e[0], e[i]);
#pragma unroll
                for (int c = 0; c < C; ++c) gg[i][c] = fmaf(cc[i], gg[0][c], gg[i][c]);
#pragma unroll
                for (int k2 = i + 1; k2 <= R; ++k2) A[i][k2] = fmaf(A[0][i], cc[k2], A[i][k2]);
            }
            float* o = sm + (long long)(k - a) * NF * bd + tid;
#pragma unroll
            for (int i = 1; i <= R; ++i) o[(i - 1) * bd] = cc[i];
#pragma unroll
            for (int c = 0; c < C; ++c) o[(R + c) * bd] = gg[0][c] * inv;
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            e[i] = e[i + 1];
#pragma unroll
            for (int c = 0; c < C; ++c) gg[i][c] = gg[i + 1][c];
#pragma unroll
            for (int k2 = i + 1; k2 < R; ++k2) A[i][k2] = A[i + 1][k2 + 1];
        }
    }

    // ---- back substitution + store into U[img][y][b][col-lo][c]
    const long long rowstride = (long long)g.nb * m * C;
    float* Ub = U + ((long long)img * g.Hl * g.nb + b) * m * C;
    // known separator values sigma_j
    if (!last) {
        for (int p = end; p < aend; ++p) {
            const int yy = p / m, j2 = p - yy * m;
            const int cidx = (yy & 1) ? (m - 1 - j2) : j2;
            const int sidx = p - end;
#pragma unroll
            for (int mm = 0; mm < R; ++mm)
                if (sidx == mm) {
#pragma unroll
                    for (int c = 0; c < C; ++c) Ub[yy * rowstride + cidx * C + c] = zr[mm][c];
                }
        }
    }
    float ur[R][C];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
        for (int c = 0; c < C; ++c) ur[i][c] = 0.f;
    if (end > a) {
        int yy = (end - 1) / m;
        int j2 = (end - 1) - yy * m;
        for (int k = end - 1; k >= a; --k) {
            const float* o = sm + (long long)(k - a) * NF * bd + tid;
            float u[C];
#pragma unroll
            for (int c = 0; c < C; ++c) u[c] = o[(R + c) * bd];
#pragma unroll
            for (int i = 1; i <= R; ++i) {
                const float ci = o[(i - 1) * bd];
#pragma unroll
                for (int c = 0; c < C; ++c) u[c] = fmaf(ci, ur[i - 1][c], u[c]);
            }
#pragma unroll
            for (int i = R - 1; i > 0; --i)
#pragma unroll
                for (int c = 0; c < C; ++c) ur[i][c] = ur[i - 1][c];
#pragma unroll
            for (int c = 0; c < C; ++c) ur[0][c] = u[c];
            const int cidx = (yy & 1) ? (m - 1 - j2) : j2;
#pragma unroll
            for (int c = 0; c < C; ++c) Ub[yy * rowstride + cidx * C + c] = u[c];
            if (--j2 < 0) {
                j2 = m - 1;
                --yy;
            }
        }
    }
}

// ===================================================================== K4

// Owner-computes averaging (proj/src/smoother.cpp:78-97 + proj/src/snake.cpp:60-72):
// pixel (y, x) of the pass layout sums the solutions of the bands whose window
// covers column x in increasing centre order and divides by their number.
template <int C>
__global__ void __launch_bounds__(256) k4_average(const PassGeom g, const float* __restrict__ U,
                                                  float* __restrict__ out, int transpose_out) {
    __shared__ float tile[32][33 * C];
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32, img = blockIdx.z;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int m = g.m, r = g.r, tau = g.tau;
    const long long rowstride = (long long)g.nb * m * C;
    const float* Ui = U + (long long)img * g.Hl * rowstride;
    const int x = x0 + tx;
    // covering bands of column x
    int b0 = 0, b1 = -1, bf = -1;
    if (x < g.Wl) {
        if (g.degenerate) {
            b0 = 0;
            b1 = 0;
        } else {
            const int lo_b = x - 2 * r;
            b0 = lo_b <= 0 ? 0 : (lo_b + tau - 1) / tau;
            b1 = x / tau;
            if (b1 > g.nreg - 1) b1 = g.nreg - 1;
            if (g.nb > g.nreg && x >= g.Wl - 1 - 2 * r) bf = g.nreg;  // forced last centre
        }
    }
    const int cnt = (b1 >= b0 ? b1 - b0 + 1 : 0) + (bf >= 0 ? 1 : 0);
    const float invc = cnt > 0 ? 1.0f / (float)cnt : 0.f;
    for (int yy = ty; yy < 32; yy += blockDim.y) {
        const int y = y0 + yy;
        float acc[C];
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] = 0.f;
        if (x < g.Wl && y < g.Hl) {
            const float* Ur = Ui + (long long)y * rowstride;
            for (int b = b0; b <= b1; ++b) {
                const int lo = band_lo(g, b);
                const float* p = Ur + ((long long)b * m + (x - lo)) * C;
#pragma unroll
                for (int c = 0; c < C; ++c) acc[c] += p[c];
            }
            if (bf >= 0) {
                const int lo = band_lo(g, bf);
                const float* p = Ur + ((long long)bf * m + (x - lo)) * C;
#pragma unroll
                for (int c = 0; c < C; ++c) acc[c] += p[c];
            }
        }
#pragma unroll
        for (int c = 0; c < C; ++c) tile[yy][tx * C + c] = acc[c] / (float)(cnt > 0 ? cnt : 1);
    }
    (void)invc;
    __syncthreads();
    float* oi = out + (long long)img * g.img_stride;
    if (transpose_out) {
        // out layout: Wl rows x Hl cols; row x holds Hl*C floats
        for (int xx = ty; xx < 32; xx += blockDim.y) {
            const int xo = x0 + xx;
            if (xo >= g.Wl) continue;
            for (int idx = tx; idx < 32 * C; idx += 32) {
                const int yy = idx / C, c = idx - yy * C;
                const int yo = y0 + yy;
                if (yo < g.Hl) oi[((long long)xo * g.Hl + yo) * C + c] = tile[yy][xx * C + c];
            }
        }
    } else {
        for (int yy = ty; yy < 32; yy += blockDim.y) {
            const int yo = y0 + yy;
            if (yo >= g.Hl) continue;
            for (int idx = tx; idx < 32 * C; idx += 32) {
                const int xx = idx / C, c = idx - xx * C;
                const int xo = x0 + xx;
                if (xo < g.Wl) oi[((long long)yo * g.Wl + xo) * C + c] = tile[yy][xx * C + c];
            }
        }
    }
}

// =========================================================== launch helpers

template <int R, int C>
inline cudaError_t launch_pass_rc(const PassLaunch& pl, cudaStream_t st) {
    using RL = RecLayout<R, C>;
    const PassGeom& g = pl.geom;
    const int NL = g.nb * g.batch;
    const int bx = pl.bx;
    dim3 grid1((NL + bx - 1) / bx, g.P);
    if (g.P > 1) {
        {
            ProfScope ps("k1_spike_forward", st);
            k1_spike_forward<R, C><<<grid1, bx, 0, st>>>(g, pl.src, pl.guid, pl.rec, *pl.w);
        }
        {
            ProfScope ps("k2_reduced", st);
            k2_reduced<R, C><<<(NL + 63) / 64, 64, 0, st>>>(g, pl.rec, pl.rs, pl.z);
        }
    }
    const size_t smem = (size_t)bx * pl.kmax * (R + C) * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(k3_interior<R, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    {
        ProfScope ps("k3_interior", st);
        k3_interior<R, C><<<grid1, bx, smem, st>>>(g, pl.src, pl.guid, pl.z, pl.U, pl.err, *pl.w);
    }
    dim3 grid4((g.Wl + 31) / 32, (g.Hl + 31) / 32, g.batch);
    {
        ProfScope ps("k4_average", st);
        k4_average<C><<<grid4, dim3(32, 8), 0, st>>>(g, pl.U, pl.out, pl.transpose_out);
    }
    (void)sizeof(RL);
    return cudaGetLastError();
}

template <int R>
cudaError_t launch_pass_r(const PassLaunch& pl, cudaStream_t st) {
    switch (pl.geom.C) {
        case 1: return launch_pass_rc<R, 1>(pl, st);
        case 2: return launch_pass_rc<R, 2>(pl, st);
        case 3: return launch_pass_rc<R, 3>(pl, st);
        case 4: return launch_pass_rc<R, 4>(pl, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sgwls_b200
