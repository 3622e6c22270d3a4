// sgwls_tile.cuh -- CTA-tiled fast path of the SG-WLS pass (regular geometry).
//
// Same exact partitioned solver as sgwls_pass.cuh, reorganised around a CTA
// tile of 32 bands (lanes) x NW consecutive row chunks (warps):
//
//   chunk        = RW image rows of one band (K = RW*M positions, M = 2r+1),
//                  its inputs, edge weights and elimination window live in
//                  registers (all RW rows are loaded up front: full MLP);
//   super-chunk  = the NW chunks of a CTA tile.  The separators BETWEEN the
//                  chunks of a tile are reduced inside the CTA (shared memory,
//                  one lane per band), so only one record per super-chunk
//                  reaches global memory and the global reduced system (K2)
//                  is NW times shorter.
//
//   KA ka_tile   spike-forward of every chunk -> chunk records in smem ->
//                lane-per-band block elimination of the NW-1 inner separators
//                carrying the spike toward the previous super-separator ->
//                super-chunk record (same format as a chunk record), then the
//                symbolic back substitution of the inner separators: each one
//                as an affine map of the tile's two super-separators (HBM).
//   K2 k2_tree   block-tridiagonal solve over the super-separators of a line,
//                a tree over NG warps -> super-separator values.
//   KB kb_tile   every chunk takes its two separators from KA's affine maps
//                and the super-separators (a few FMAs), then solves its
//                interior (forward elimination + back substitution in
//                registers).  Overlapping bands are averaged in a fixed order
//                (warp shuffles or a shared output tile) and the result leaves
//                in the next pass's transposed layout.
//
// All eliminations: magnitudes + row-sum pivots (sgwls_device.cuh).
#pragma once

#include <cuda.h>  // CUtensorMap (types only; the encoder is fetched through the runtime)
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <utility>

#include "sgwls_device.cuh"
#include "sgwls_kernels.h"
#include "sgwls_profile.h"

namespace sgwls_b200 {
namespace tile {

// Programmatic dependent launch: a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor drains; griddepcontrol.wait blocks until the predecessor grid has
// completed and its memory is visible (a no-op for ordinary launches).
// launch_dependents lets the successor start launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Bulk (TMA) shared -> global copy; 16-byte aligned addresses, size % 16 == 0.
__device__ __forceinline__ void bulk_s2g(float* gdst, const float* ssrc, unsigned bytes) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(ssrc);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(sa), "r"(bytes)
                 : "memory");
}
// shared memory must stay valid until the bulk copies have read it
__device__ __forceinline__ void bulk_commit_and_wait_read() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// order this thread's generic-proxy shared-memory writes before async-proxy reads
__device__ __forceinline__ void fence_proxy_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Bulk (TMA) global -> shared copy completing on an mbarrier; 16-byte aligned
// addresses, size % 16 == 0.  One instruction moves a whole row segment: no
// per-lane loads, no L1 wavefronts.
__device__ __forceinline__ void bulk_g2s(float* sdst, const float* gsrc, unsigned bytes, unsigned long long* mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (unsigned)__cvta_generic_to_shared(sdst)),
        "l"(gsrc), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(mbar))
        : "memory");
}
// Tiled (tensor-map) TMA load of a 2-D box: element coordinates (x, y) of the box's
// first element, out-of-bounds elements arrive as zeros; 128-byte aligned destination.
__device__ __forceinline__ void tma_load_2d(float* sdst, const CUtensorMap* tm, int x, int y,
                                            unsigned long long* mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"((unsigned)__cvta_generic_to_shared(sdst)),
        "l"(tm), "r"(x), "r"(y), "r"((unsigned)__cvta_generic_to_shared(mbar))
        : "memory");
}

// Tensor map over `rows` rows of `row_elems` fp32 each (row pitch = row_elems), box
// box_w x box_h, no swizzle, zero fill.  False when the driver entry point is missing
// or the layout is outside TMA's rules (16-byte base and pitch, box sides <= 256).
inline bool encode_rows_map(CUtensorMap* tm, const float* base, long long row_elems, long long rows, int box_w,
                            int box_h) {
    typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return (EncodeFn)p;
    }();
    if (!fn || box_w > 256 || box_h > 256 || (box_w % 4) != 0 || (row_elems % 4) != 0 ||
        (reinterpret_cast<uintptr_t>(base) & 15) != 0)
        return false;
    const cuuint64_t gdim[2] = {(cuuint64_t)row_elems, (cuuint64_t)rows};
    const cuuint64_t gstr[1] = {(cuuint64_t)row_elems * sizeof(float)};
    const cuuint32_t box[2] = {(cuuint32_t)box_w, (cuuint32_t)box_h};
    const cuuint32_t estr[2] = {1, 1};
    return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim, gstr, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__device__ __forceinline__ void mbar_init(unsigned long long* mbar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(mbar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* mbar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(mbar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mbar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "MBAR_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@p bra MBAR_DONE;\n"
        "bra MBAR_WAIT;\n"
        "MBAR_DONE:\n"
        "}" ::"r"((unsigned)__cvta_generic_to_shared(mbar)),
        "r"(parity), "r"(0x989680u)  // suspend-time hint: the warp sleeps in the barrier instead of polling
        : "memory");
}

// 16-byte asynchronous global -> shared copy (LDGSTS: no registers held while in flight)
__device__ __forceinline__ void cp_async16(float* sdst, const float* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(sdst)),
                 "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("SGWLS_PDL");  // tuning knob: 0 = ordinary stream-ordered launches
        return v ? std::atoi(v) != 0 : true;
    }();
    return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

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
    // back-substitution row with the spike toward the left super-separator
    static constexpr int RSM = RS + R;
    // affine map of one inner separator of a KA tile: component q, basis b in
    // [value (C) | left super-separator zL (R) | right super-separator zR (R)]
    static constexpr int NB = C + 2 * R;
    static constexpr int MAPF = R * NB;
    // global layout of the maps: [chunk][line][MAPP] (MAPF padded to whole
    // 16-byte vectors: a lane's map is one run of MAPP/4 float4s)
    static constexpr int MAPP = (MAPF + 3) & ~3;
};

__host__ __device__ constexpr int rows_per_chunk(int R, int C) { return tile_rows_per_chunk(R, C); }

__device__ __forceinline__ constexpr int offi(int i, int j, int R) { return i * R - i * (i + 1) / 2 + (j - i - 1); }

// clamp a (compile-time) register-array index into [0, n): indices in branches
// that are dead for a given unrolled iteration must still be in bounds
__host__ __device__ constexpr int cl(int x, int n) { return x < 0 ? 0 : (x >= n ? n - 1 : x); }

// dst[k] = fma(s, src[k], dst[k]), k < N
template <int N>
__device__ __forceinline__ void row_fma(float* dst, float s, const float* src) {
#pragma unroll
    for (int k = 0; k < N; ++k) dst[k] = fmaf(s, src[k], dst[k]);
}
// dst[k] = src[k] * s, k < N
template <int N>
__device__ __forceinline__ void row_mul(float* dst, const float* src, float s) {
#pragma unroll
    for (int k = 0; k < N; ++k) dst[k] = src[k] * s;
}

// squared 2-D distance of the edge (q - t, q), q at in-row index jj (regular band)
__host__ __device__ constexpr int edge_d2(int jj, int t) {
    return jj >= t ? t * t : 1 + (t - 1 - 2 * jj) * (t - 1 - 2 * jj);
}

// ------------------------------------------------------------ chunk inputs

// Inputs of one chunk in POSITION order (serpentine resolved at load time).
template <int R, int C, int CG, int RW>
struct ChunkIn {
    static constexpr int M = 2 * R + 1, K = RW * M;
    float f[K][C];
    float w[K][R];  // w[k][t-1] = lambda * weight of edge (k - t, k)
};

template <int R, int C, int CG, int RW, int WK, bool FULLC>
__device__ __forceinline__ void load_chunk_k(ChunkIn<R, C, CG, RW>& in, const float* __restrict__ F,
                                             const float* __restrict__ Msk, const float* __restrict__ G,
                                             const PassGeom& g, const WeightDev& W, int lo, int y0, int nrows,
                                             unsigned long long* err, int line) {
    constexpr int M = 2 * R + 1, K = RW * M;
    float gp[K][CG];
    float gprev[R][CG];  // positions y0*M - R .. y0*M - 1 (last R of row y0-1)
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int jj = M - R + i;
        const int y = y0 - 1;
        if (y >= 0 || g.has_prev) {
            const int co = (y & 1) ? (M - 1 - jj) : jj;
            const float* p = G + ((long long)y * g.Wl + lo + co) * CG;
#pragma unroll
            for (int c = 0; c < CG; ++c) gprev[i][c] = __ldg(p + c);
        } else {
#pragma unroll
            for (int c = 0; c < CG; ++c) gprev[i][c] = 0.f;
        }
    }
    // Each row's M samples are loaded in memory order from one base address
    // (compile-time offsets, no per-sample address arithmetic) and the
    // serpentine reversal of odd rows (proj/src/snake.cpp:21-49) is applied to
    // the values.  With an even RW the row parity is compile-time (chunks start
    // on even rows).  FULLC: every row of the chunk exists (no predicates).
    // split input: F holds C-1 value channels, channel C-1 comes from the mask
    const bool split = C > 1 && g.msk != nullptr;
    constexpr int CV = C > 1 ? C - 1 : 1;
    const long long px0 = (long long)y0 * g.Wl + lo;
    const float* rowF = F + px0 * (split ? CV : C);
    const float* rowM = split ? Msk + px0 : nullptr;
    const float* rowG = G + px0 * CG;
    const long long stF = (long long)g.Wl * (split ? CV : C), stG = (long long)g.Wl * CG;
#pragma unroll
    for (int rr = 0; rr < RW; ++rr) {
        const bool valid = FULLC || rr < nrows;
        const bool odd = (RW % 2 == 0) ? ((rr & 1) != 0) : (((y0 + rr) & 1) != 0);
        float vf[M][C], vg[M][CG];
#pragma unroll
        for (int jj = 0; jj < M; ++jj) {
            if (valid) {
#pragma unroll
                for (int c = 0; c < C; ++c)
                    vf[jj][c] = !split ? __ldg(rowF + jj * C + c)
                                       : (c < C - 1 ? __ldg(rowF + jj * CV + c) : __ldg(rowM + jj));
#pragma unroll
                for (int c = 0; c < CG; ++c) vg[jj][c] = __ldg(rowG + jj * CG + c);
            } else {
#pragma unroll
                for (int c = 0; c < C; ++c) vf[jj][c] = 0.f;
#pragma unroll
                for (int c = 0; c < CG; ++c) vg[jj][c] = 0.f;
            }
        }
#pragma unroll
        for (int jj = 0; jj < M; ++jj) {
            const int k = rr * M + jj;
#pragma unroll
            for (int c = 0; c < C; ++c) in.f[k][c] = odd ? vf[M - 1 - jj][c] : vf[jj][c];
#pragma unroll
            for (int c = 0; c < CG; ++c) gp[k][c] = odd ? vg[M - 1 - jj][c] : vg[jj][c];
        }
        rowF += stF;
        rowG += stG;
        if (split) rowM += g.Wl;
    }
    // edge weights (proj/src/weights.cpp:48-71); spatial factor index is compile-time.
    // A NaN weight (NaN guidance) is the reference's "non-positive pivot" failure:
    // remember the first offending position and report it once.
    // Cheap detection: a weight can only be NaN where a guidance value it
    // reads is NaN or infinite, and x * 0 is NaN exactly for those; the exact
    // position is located from the weights only on that rare path.
    float acc = 0.f;
    if (err != nullptr) {
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int c = 0; c < CG; ++c) acc = fmaf(gp[k][c], 0.f, acc);
#pragma unroll
        for (int i = 0; i < R; ++i)
#pragma unroll
            for (int c = 0; c < CG; ++c) acc = fmaf(gprev[i][c], 0.f, acc);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
        for (int t = 1; t <= R; ++t) {
            float r2 = 0.f;
#pragma unroll
            for (int c = 0; c < CG; ++c) {
                const float other = (k - t >= 0) ? gp[cl(k - t, K)][c] : gprev[cl(k - t + R, R)][c];
                const float d = gp[k][c] - other;
                r2 = fmaf(d, d, r2);
            }
            in.w[k][t - 1] = guidance_lweight_k<WK>(W, r2, edge_d2(k % M, t));
        }
    }
    if (err != nullptr && !(acc >= 0.f)) {
        int bad = 0x7fffffff;
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int t = 1; t <= R; ++t) {
                const bool exists = (k / M < nrows) && (k - t >= 0 || y0 > 0 || g.has_prev);
                bad = (!(in.w[k][t - 1] >= 0.f) && exists) ? min(bad, (g.row0 + y0) * M + k - t) : bad;
            }
        if (bad != 0x7fffffff) atomicMin(err, ((unsigned long long)(unsigned)line << 32) | (unsigned)bad);
    }
}

// Lazy form (KA): the chunk's samples and guidance only; each edge weight is
// computed where the elimination consumes it (fewer live registers, MUFU work
// interleaved with the dependent elimination chain).
template <int R, int C, int CG, int RW>
struct ChunkInL {
    static constexpr int M = 2 * R + 1, K = RW * M;
    float f[K][C];
    float gp[K][CG];
    float gprev[R][CG];
};

template <int R, int C, int CG, int RW, bool FULLC>
__device__ __forceinline__ void load_chunk_lazy(ChunkInL<R, C, CG, RW>& in, const float* __restrict__ F,
                                                const float* __restrict__ Msk, const float* __restrict__ G,
                                                const PassGeom& g, int lo, int y0, int nrows) {
    constexpr int M = 2 * R + 1;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int jj = M - R + i;
        const int y = y0 - 1;
        if (y >= 0 || g.has_prev) {
            const int co = (y & 1) ? (M - 1 - jj) : jj;
            const float* p = G + ((long long)y * g.Wl + lo + co) * CG;
#pragma unroll
            for (int c = 0; c < CG; ++c) in.gprev[i][c] = __ldg(p + c);
        } else {
#pragma unroll
            for (int c = 0; c < CG; ++c) in.gprev[i][c] = 0.f;
        }
    }
    const bool split = C > 1 && Msk != nullptr;
    constexpr int CV = C > 1 ? C - 1 : 1;
    const long long px0 = (long long)y0 * g.Wl + lo;
    const float* rowF = F + px0 * (split ? CV : C);
    const float* rowM = split ? Msk + px0 : nullptr;
    const float* rowG = G + px0 * CG;
    const long long stF = (long long)g.Wl * (split ? CV : C), stG = (long long)g.Wl * CG;
#pragma unroll
    for (int rr = 0; rr < RW; ++rr) {
        const bool valid = FULLC || rr < nrows;
        const bool odd = (RW % 2 == 0) ? ((rr & 1) != 0) : (((y0 + rr) & 1) != 0);
        float vf[M][C], vg[M][CG];
#pragma unroll
        for (int jj = 0; jj < M; ++jj) {
#pragma unroll
            for (int c = 0; c < C; ++c)
                vf[jj][c] = !valid ? 0.f
                                   : (!split ? __ldg(rowF + jj * C + c)
                                             : (c < C - 1 ? __ldg(rowF + jj * CV + c) : __ldg(rowM + jj)));
#pragma unroll
            for (int c = 0; c < CG; ++c) vg[jj][c] = valid ? __ldg(rowG + jj * CG + c) : 0.f;
        }
#pragma unroll
        for (int jj = 0; jj < M; ++jj) {
            const int k = rr * M + jj;
#pragma unroll
            for (int c = 0; c < C; ++c) in.f[k][c] = odd ? vf[M - 1 - jj][c] : vf[jj][c];
#pragma unroll
            for (int c = 0; c < CG; ++c) in.gp[k][c] = odd ? vg[M - 1 - jj][c] : vg[jj][c];
        }
        rowF += stF;
        rowG += stG;
        if (split) rowM += g.Wl;
    }
}

// Same, from the CTA's staged rows in shared memory (kb_tile, bulk-copied row
// segments): sFr / sGr point at this lane's first sample of the chunk's first
// row (sGr: one row above it is the previous row), pf / pg are the row pitches.
template <int R, int C, int CG, int RW, bool FULLC>
__device__ __forceinline__ void load_chunk_lazy_staged(ChunkInL<R, C, CG, RW>& in, const float* sFr, int pf,
                                                       const float* sGr, int pg, const PassGeom& g, int y0,
                                                       int nrows) {
    constexpr int M = 2 * R + 1;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int jj = M - R + i;
        const int y = y0 - 1;
        if (y >= 0) {
            const int co = (y & 1) ? (M - 1 - jj) : jj;
#pragma unroll
            for (int c = 0; c < CG; ++c) in.gprev[i][c] = sGr[-pg + co * CG + c];
        } else {
#pragma unroll
            for (int c = 0; c < CG; ++c) in.gprev[i][c] = 0.f;
        }
    }
#pragma unroll
    for (int rr = 0; rr < RW; ++rr) {
        const bool valid = FULLC || rr < nrows;
        const bool odd = (RW % 2 == 0) ? ((rr & 1) != 0) : (((y0 + rr) & 1) != 0);
        float vf[M][C], vg[M][CG];
#pragma unroll
        for (int jj = 0; jj < M; ++jj) {
#pragma unroll
            for (int c = 0; c < C; ++c) vf[jj][c] = valid ? sFr[rr * pf + jj * C + c] : 0.f;
#pragma unroll
            for (int c = 0; c < CG; ++c) vg[jj][c] = valid ? sGr[rr * pg + jj * CG + c] : 0.f;
        }
#pragma unroll
        for (int jj = 0; jj < M; ++jj) {
            const int k = rr * M + jj;
#pragma unroll
            for (int c = 0; c < C; ++c) in.f[k][c] = odd ? vf[M - 1 - jj][c] : vf[jj][c];
#pragma unroll
            for (int c = 0; c < CG; ++c) in.gp[k][c] = odd ? vg[M - 1 - jj][c] : vg[jj][c];
        }
    }
}

// lambda * w of edge (k - t, k) of a lazily loaded chunk (k, t compile-time after unrolling)
template <int R, int C, int CG, int RW, int WK>
struct LazyWeights {
    const ChunkInL<R, C, CG, RW>& in;
    const WeightDev& W;
    __device__ __forceinline__ float operator()(int k, int t) const {
        constexpr int K = RW * (2 * R + 1);
        float r2 = 0.f;
#pragma unroll
        for (int c = 0; c < CG; ++c) {
            const float other = (k - t >= 0) ? in.gp[cl(k - t, K)][c] : in.gprev[cl(k - t + R, R)][c];
            const float d = in.gp[cl(k, K)][c] - other;
            r2 = fmaf(d, d, r2);
        }
        return guidance_lweight_k<WK>(W, r2, edge_d2(k % (2 * R + 1), t));
    }
};
template <int R, int C, int CG, int RW>
struct EagerWeights {
    const ChunkIn<R, C, CG, RW>& in;
    __device__ __forceinline__ float operator()(int k, int t) const {
        return in.w[cl(k, RW * (2 * R + 1))][t - 1];
    }
};

// One uniform branch per chunk on the weight kind instead of one per edge.
template <int R, int C, int CG, int RW>
__device__ __forceinline__ void load_chunk(ChunkIn<R, C, CG, RW>& in, const float* __restrict__ F,
                                           const float* __restrict__ G, const PassGeom& g, const WeightDev& W,
                                           int lo, int y0, int nrows, unsigned long long* err, int line, int img) {
    // image img of the pass input (split: C-1 value channels + the mask)
    const long long npx = (long long)g.Hl * g.Wl;
    const float* Msk = (C > 1 && g.msk != nullptr) ? g.msk + img * npx : nullptr;
    F += img * (Msk ? npx * (C > 1 ? C - 1 : 1) : g.img_stride);
#ifndef SGWLS_NO_FULL_LOAD
    if (W.kind == 1) {
        if (nrows == RW)
            load_chunk_k<R, C, CG, RW, 1, true>(in, F, Msk, G, g, W, lo, y0, nrows, err, line);
        else
            load_chunk_k<R, C, CG, RW, 1, false>(in, F, Msk, G, g, W, lo, y0, nrows, err, line);
    } else {
        load_chunk_k<R, C, CG, RW, 0, false>(in, F, Msk, G, g, W, lo, y0, nrows, err, line);
    }
#else
    if (W.kind == 1)
        load_chunk_k<R, C, CG, RW, 1, false>(in, F, G, g, W, lo, y0, nrows, err, line);
    else
        load_chunk_k<R, C, CG, RW, 0, false>(in, F, Msk, G, g, W, lo, y0, nrows, err, line);
#endif
}

// ------------------------------------------------- elimination window (scalar)

// Sliding window of R+1 scalar rows with spike columns toward the left separator.
template <int R, int C, bool SPIKE>
struct Win {
    float e[R + 1], g[R + 1][C], A[R + 1][R + 1], Q[R + 1][SPIKE ? R : 1];
    float he[R], hg[R][C], hoff[R][R];

    __device__ __forceinline__ void clear() {
#pragma unroll
        for (int i = 0; i <= R; ++i) {
            e[i] = 0.f;
#pragma unroll
            for (int c = 0; c < C; ++c) g[i][c] = 0.f;
#pragma unroll
            for (int k = 0; k <= R; ++k) A[i][k] = 0.f;
#pragma unroll
            for (int k = 0; k < (SPIKE ? R : 1); ++k) Q[i][k] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            he[i] = 0.f;
#pragma unroll
            for (int c = 0; c < C; ++c) hg[i][c] = 0.f;
#pragma unroll
            for (int k = 0; k < R; ++k) hoff[i][k] = 0.f;
        }
    }
    // eliminate slot 0; returns 1/pivot and the normalised couplings cc[1..R]
    __device__ __forceinline__ float elim(float (&cc)[R + 1], bool head) {
        float s = e[0];
#pragma unroll
        for (int i = 1; i <= R; ++i) s += A[0][i];
        if (SPIKE) {
#pragma unroll
            for (int mm = 0; mm < R; ++mm) s += Q[0][mm];
        }
        const float inv = fast_rcp(s);
#pragma unroll
        for (int i = 1; i <= R; ++i) cc[i] = A[0][i] * inv;
#pragma unroll
        for (int i = 1; i <= R; ++i) {
            e[i] = fmaf(cc[i], e[0], e[i]);
            row_fma<C>(g[i], cc[i], g[0]);
#pragma unroll
            for (int k2 = i + 1; k2 <= R; ++k2) A[i][k2] = fmaf(A[0][i], cc[k2], A[i][k2]);
            if (SPIKE) row_fma<R>(Q[i], cc[i], Q[0]);
        }
        if (SPIKE && head) {
            float d[R];
            row_mul<R>(d, Q[0], inv);
            row_fma<R>(he, e[0], d);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                float hgc[R];
#pragma unroll
                for (int mm = 0; mm < R; ++mm) hgc[mm] = hg[mm][c];
                row_fma<R>(hgc, g[0][c], d);
#pragma unroll
                for (int mm = 0; mm < R; ++mm) hg[mm][c] = hgc[mm];
            }
#pragma unroll
            for (int mm = 0; mm < R; ++mm)
#pragma unroll
                for (int m2 = mm + 1; m2 < R; ++m2) hoff[mm][m2] = fmaf(d[mm], Q[0][m2], hoff[mm][m2]);
        }
        return inv;
    }
    __device__ __forceinline__ void shift() {
#pragma unroll
        for (int i = 0; i < R; ++i) {
            e[i] = e[i + 1];
#pragma unroll
            for (int c = 0; c < C; ++c) g[i][c] = g[i + 1][c];
#pragma unroll
            for (int k2 = i + 1; k2 < R; ++k2) A[i][k2] = A[i + 1][k2 + 1];
            if (SPIKE) {
#pragma unroll
                for (int mm = 0; mm < R; ++mm) Q[i][mm] = Q[i + 1][mm];
            }
        }
        e[R] = 0.f;
#pragma unroll
        for (int c = 0; c < C; ++c) g[R][c] = 0.f;
#pragma unroll
        for (int i = 0; i < R; ++i) {
            A[i][R] = 0.f;
            if (SPIKE) Q[R][i] = 0.f;
        }
    }
};

// Spike-forward over one chunk: eliminates the interior, leaves sigma_j in
// slots 0..R-1 (non-last chunk) and the head update of sigma_{j-1}; writes the
// chunk record into `rec` (shared memory, stride `rs` floats between fields).
// FULL: the chunk has all RW rows (every chunk but possibly the band's last):
// the position loop is then free of runtime predicates, so the window shifts
// compile to register renames.
template <int R, int C, int CG, int RW, bool FULL, class IN, class WF>
__device__ __forceinline__ void chunk_spike_forward_impl(const IN& in, const WF& lwf, bool has_left, bool last, int kv,
                                                         float* rec, int rs) {
    using RL = Rec<R, C>;
    auto put = [&](int f, float v) { rec[f * rs] = v; };
    constexpr int K = RW * (2 * R + 1);
    Win<R, C, true> w;
    w.clear();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        if (FULL || k < kv) {
            w.e[R] = 1.f;
#pragma unroll
            for (int c = 0; c < C; ++c) w.g[R][c] = in.f[k][c];
#pragma unroll
            for (int t = 1; t <= R; ++t) {
                const float lw = lwf(k, t);
                if (k - t >= 0) {
                    w.A[R - t][R] = lw;
                } else if (has_left) {
                    w.Q[R][cl(R - t + k, R)] = lw;
                }
            }
            if (k >= R) {
                float cc[R + 1];
                w.elim(cc, has_left);
            }
            w.shift();
        }
    }
    if (last) {
#pragma unroll
        for (int d = 0; d < R; ++d) {
            float cc[R + 1];
            w.elim(cc, has_left);
            w.shift();
        }
    } else {
#pragma unroll
        for (int i = 0; i < R; ++i) {
#pragma unroll
            for (int k2 = i + 1; k2 < R; ++k2) put(RL::TOFF + offi(i, k2, R), w.A[i][k2]);
#pragma unroll
            for (int mm = 0; mm < R; ++mm) put(RL::TCROSS + i * R + mm, w.Q[i][mm]);
            put(RL::TE + i, w.e[i]);
#pragma unroll
            for (int c = 0; c < C; ++c) put(RL::TG + i * C + c, w.g[i][c]);
        }
    }
#pragma unroll
    for (int mm = 0; mm < R; ++mm) {
#pragma unroll
        for (int m2 = mm + 1; m2 < R; ++m2) put(RL::HOFF + offi(mm, m2, R), w.hoff[mm][m2]);
        put(RL::HE + mm, w.he[mm]);
#pragma unroll
        for (int c = 0; c < C; ++c) put(RL::HG + mm * C + c, w.hg[mm][c]);
    }
}

template <int R, int C, int CG, int RW, class IN, class WF>
__device__ __forceinline__ void chunk_spike_forward(const IN& in, const WF& lwf, bool has_left, bool last, int kv,
                                                    float* rec, int rs) {
    if (kv == RW * (2 * R + 1))
        chunk_spike_forward_impl<R, C, CG, RW, true>(in, lwf, has_left, last, kv, rec, rs);
    else
        chunk_spike_forward_impl<R, C, CG, RW, false>(in, lwf, has_left, last, kv, rec, rs);
}

// ---------------------------------------------- block window (separator level)

// Two blocks of R scalar slots (lo = 0..R-1, hi = R..2R-1) plus spike columns.
template <int R, int C, bool SPIKE>
struct BWin {
    static constexpr int W2 = 2 * R;
    float e[W2], g[W2][C], A[W2][W2], Q[W2][SPIKE ? R : 1];
    float he[R], hg[R][C], hoff[R][R];

    __device__ __forceinline__ void clear_all() {
#pragma unroll
        for (int i = 0; i < W2; ++i) {
            e[i] = 0.f;
#pragma unroll
            for (int c = 0; c < C; ++c) g[i][c] = 0.f;
#pragma unroll
            for (int k = 0; k < W2; ++k) A[i][k] = 0.f;
#pragma unroll
            for (int k = 0; k < (SPIKE ? R : 1); ++k) Q[i][k] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            he[i] = 0.f;
#pragma unroll
            for (int c = 0; c < C; ++c) hg[i][c] = 0.f;
#pragma unroll
            for (int k = 0; k < R; ++k) hoff[i][k] = 0.f;
        }
    }
    __device__ __forceinline__ void clear_hi() {
#pragma unroll
        for (int i = R; i < W2; ++i) {
            e[i] = 0.f;
#pragma unroll
            for (int c = 0; c < C; ++c) g[i][c] = 0.f;
#pragma unroll
            for (int k = 0; k < W2; ++k) {
                A[i][k] = 0.f;
                A[k][i] = 0.f;
            }
#pragma unroll
            for (int k = 0; k < (SPIKE ? R : 1); ++k) Q[i][k] = 0.f;
        }
    }
    // eliminate lo slot mm (scalar); stores the back-substitution row into bs (if non-null)
    __device__ __forceinline__ void elim(int mm_unused, const int mm, bool head, float* bs, int bstride) {
        (void)mm_unused;
        float piv = e[mm];
#pragma unroll
        for (int i = mm + 1; i < W2; ++i) piv += A[mm][i];
        if (SPIKE) {
#pragma unroll
            for (int q = 0; q < R; ++q) piv += Q[mm][q];
        }
        const float inv = fast_rcp(piv);
        float cc[W2];
#pragma unroll
        for (int i = mm + 1; i < W2; ++i) cc[i] = A[mm][i] * inv;
#pragma unroll
        for (int i = mm + 1; i < W2; ++i) {
            e[i] = fmaf(cc[i], e[mm], e[i]);
            row_fma<C>(g[i], cc[i], g[mm]);
#pragma unroll
            for (int k = i + 1; k < W2; ++k) A[i][k] = fmaf(A[mm][i], cc[k], A[i][k]);
            if (SPIKE) row_fma<R>(Q[i], cc[i], Q[mm]);
        }
        if (SPIKE && head) {
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const float d = Q[mm][q] * inv;
                he[q] = fmaf(d, e[mm], he[q]);
#pragma unroll
                for (int c = 0; c < C; ++c) hg[q][c] = fmaf(d, g[mm][c], hg[q][c]);
#pragma unroll
                for (int q2 = q + 1; q2 < R; ++q2) hoff[q][q2] = fmaf(d, Q[mm][q2], hoff[q][q2]);
            }
        }
        if (bs) {
#pragma unroll
            for (int i = mm + 1; i < W2; ++i) bs[(i - mm - 1) * bstride] = cc[i];
#pragma unroll
            for (int c = 0; c < C; ++c) bs[(W2 - 1 + c) * bstride] = g[mm][c] * inv;
            if (SPIKE) {  // x_mm also depends on the left super-separator: + (Q/pivot) . zL
#pragma unroll
                for (int q = 0; q < R; ++q) bs[(W2 - 1 + C + q) * bstride] = Q[mm][q] * inv;
            }
        }
    }
    __device__ __forceinline__ void shift() {
#pragma unroll
        for (int i = 0; i < R; ++i) {
            e[i] = e[i + R];
#pragma unroll
            for (int c = 0; c < C; ++c) g[i][c] = g[i + R][c];
#pragma unroll
            for (int k = i + 1; k < R; ++k) A[i][k] = A[i + R][k + R];
            if (SPIKE) {
#pragma unroll
                for (int q = 0; q < R; ++q) Q[i][q] = Q[i + R][q];
            }
        }
    }
};

// Enter separator block `s` (chunk s's tail + chunk s+1's head when `with_head`)
// into the hi slots; its coupling to the previous block goes to the window
// (prev_in_window) or to the spike columns.
template <int R, int C, bool SPIKE>
__device__ __forceinline__ void enter_block(BWin<R, C, SPIKE>& w, const float* tail, const float* head, int rs,
                                            bool with_head, bool prev_in_window, bool prev_exists) {
    using RL = Rec<R, C>;
    w.clear_hi();
#pragma unroll
    for (int mm = 0; mm < R; ++mm) {
        w.e[R + mm] = tail[(RL::TE + mm) * rs] + (with_head ? head[(RL::HE + mm) * rs] : 0.f);
#pragma unroll
        for (int c = 0; c < C; ++c)
            w.g[R + mm][c] = tail[(RL::TG + mm * C + c) * rs] + (with_head ? head[(RL::HG + mm * C + c) * rs] : 0.f);
#pragma unroll
        for (int m2 = mm + 1; m2 < R; ++m2)
            w.A[R + mm][R + m2] = tail[(RL::TOFF + offi(mm, m2, R)) * rs] +
                                  (with_head ? head[(RL::HOFF + offi(mm, m2, R)) * rs] : 0.f);
#pragma unroll
        for (int mp = 0; mp < R; ++mp) {
            const float x = prev_exists ? tail[(RL::TCROSS + mm * R + mp) * rs] : 0.f;
            if (prev_in_window) {
                w.A[mp][R + mm] = x;
            } else if (SPIKE) {
                w.Q[R + mm][mp] = x;
            }
        }
    }
}

// Reduce the NW chunk records of one band (lane) to its super-chunk record.
// L1 prefetch of record s of a GLOBAL record run (every field: one 128-byte
// line per warp when the lanes are consecutive lines).  The serial loops below
// otherwise wait a full L2/HBM round trip per record.
#ifndef SGWLS_REC_PF
#define SGWLS_REC_PF 2  // records ahead (0 = off); used for r >= 2 (vs none: c3 +4 %, c4 +1.4 %, c5 +2.3 %;
                        // 2 beats 4 and 8; the r = 1 K2 of c2 loses 3.6 % with it)
#endif
#ifndef SGWLS_REC_PF_MINR
#define SGWLS_REC_PF_MINR 2  // smallest radius that prefetches
#endif
template <int R, int C>
__device__ __forceinline__ void prefetch_record(const float* recs, long long rs, long long cs, int s) {
#pragma unroll
    for (int f = 0; f < Rec<R, C>::REC; ++f)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(recs + (long long)s * cs + (long long)f * rs));
}

template <int R, int C, bool GPF = false>
__device__ __forceinline__ void reduce_super(const float* recs, long long rs, long long cs, int nw, bool first_super,
                                             bool last_super, float* out, long long os) {
    // recs: chunk s's field f at recs[s * cs + f * rs]; GPF: recs is global, prefetch ahead
    using RL = Rec<R, C>;
    if (GPF && SGWLS_REC_PF > 0)
        for (int s = 0; s < min(nw, SGWLS_REC_PF); ++s) prefetch_record<R, C>(recs, rs, cs, s);
    BWin<R, C, true> w;
    w.clear_all();
    if (!first_super) {  // head of the tile's first chunk: update of the left super-separator
#pragma unroll
        for (int q = 0; q < R; ++q) {
            w.he[q] = recs[(RL::HE + q) * rs];
#pragma unroll
            for (int c = 0; c < C; ++c) w.hg[q][c] = recs[(RL::HG + q * C + c) * rs];
#pragma unroll
            for (int q2 = q + 1; q2 < R; ++q2) w.hoff[q][q2] = recs[(RL::HOFF + offi(q, q2, R)) * rs];
        }
    }
    const int nblk = last_super ? nw - 1 : nw;  // separators of this tile's chunks
    for (int s = 0; s < nblk; ++s) {
        if (GPF && SGWLS_REC_PF > 0 && s + SGWLS_REC_PF < nw) prefetch_record<R, C>(recs, rs, cs, s + SGWLS_REC_PF);
        const float* t = recs + (long long)s * cs;
        const float* h = recs + (long long)(s + 1) * cs;
        const bool inner = (s < nw - 1);  // sigma_s is internal (its next chunk is in the tile)
        enter_block<R, C, true>(w, t, h, (int)rs, inner, s > 0, s > 0 || !first_super);
        if (s > 0) {
#pragma unroll
            for (int mm = 0; mm < R; ++mm) w.elim(0, mm, !first_super, nullptr, 0);
        }
        w.shift();
    }
    if (last_super) {  // drain the final inner separator
        if (nblk > 0) {
            w.clear_hi();
#pragma unroll
            for (int mm = 0; mm < R; ++mm) w.elim(0, mm, !first_super, nullptr, 0);
        }
    } else {
#pragma unroll
        for (int i = 0; i < R; ++i) {
#pragma unroll
            for (int k2 = i + 1; k2 < R; ++k2) out[(RL::TOFF + offi(i, k2, R)) * os] = w.A[i][k2];
#pragma unroll
            for (int q = 0; q < R; ++q) out[(RL::TCROSS + i * R + q) * os] = w.Q[i][q];
            out[(RL::TE + i) * os] = w.e[i];
#pragma unroll
            for (int c = 0; c < C; ++c) out[(RL::TG + i * C + c) * os] = w.g[i][c];
        }
    }
    if (!first_super) {
#pragma unroll
        for (int q = 0; q < R; ++q) {
#pragma unroll
            for (int q2 = q + 1; q2 < R; ++q2) out[(RL::HOFF + offi(q, q2, R)) * os] = w.hoff[q][q2];
            out[(RL::HE + q) * os] = w.he[q];
#pragma unroll
            for (int c = 0; c < C; ++c) out[(RL::HG + q * C + c) * os] = w.hg[q][c];
        }
    }
}


// KA's in-tile reduction with affine separator maps.  The forward sweep is
// reduce_super's (the chunk records of one band in shared memory -> the
// super-record), keeping each elimination's back-substitution row, spike to
// the left super-separator included (bsm: row (s, mm) field f at
// bsm[((s*R + mm)*RSM + f)*32]).  The backward sweep then runs SYMBOLICALLY
// in the two unknown super-separators (maps_backward_column, one basis column
// per warp): every inner separator s of the tile (s < nw - 1) comes out as
// x_s = a_s + B_s zL + Cm_s zR, stored at maps[(s*MAPF + q*NB + b)*ms]
// (b: value | zL | zR basis).  Once K2 has solved the super-separators, any
// chunk separator is 2R^2 + R FMAs away -- no third solve over the chunk
// records (the former KC launch) and no record round trip through HBM.
template <int R, int C, bool GPF = false>
__device__ __forceinline__ void reduce_super_fwd(const float* recs, int rs, int nw, bool first_super,
                                                 bool last_super, float* out, long long os, float* bsm,
                                                 int cs = 32, int bst = 32) {
    // bst: stride of the back-substitution rows' fields (32 in shared memory,
    // the line count in global scratch); GPF: recs is global, L1-prefetch ahead
    using RL = Rec<R, C>;
    constexpr int RSM = RL::RSM;
    auto bsrow = [&](int s, int mm) { return bsm + (long long)(s * R + mm) * RSM * bst; };
    if (GPF && SGWLS_REC_PF > 0)
        for (int s = 0; s < min(nw, SGWLS_REC_PF); ++s) prefetch_record<R, C>(recs, rs, cs, s);
    BWin<R, C, true> w;
    w.clear_all();
    if (!first_super) {
#pragma unroll
        for (int q = 0; q < R; ++q) {
            w.he[q] = recs[(RL::HE + q) * rs];
#pragma unroll
            for (int c = 0; c < C; ++c) w.hg[q][c] = recs[(RL::HG + q * C + c) * rs];
#pragma unroll
            for (int q2 = q + 1; q2 < R; ++q2) w.hoff[q][q2] = recs[(RL::HOFF + offi(q, q2, R)) * rs];
        }
    }
    const int nblk = last_super ? nw - 1 : nw;
    for (int s = 0; s < nblk; ++s) {
        if (GPF && SGWLS_REC_PF > 0 && s + SGWLS_REC_PF < nw) prefetch_record<R, C>(recs, rs, cs, s + SGWLS_REC_PF);
        const float* t = recs + (long long)s * cs;
        const float* h = recs + (long long)(s + 1) * cs;
        enter_block<R, C, true>(w, t, h, rs, s < nw - 1, s > 0, s > 0 || !first_super);
        if (s > 0) {
#pragma unroll
            for (int mm = 0; mm < R; ++mm) w.elim(0, mm, !first_super, bsrow(s - 1, mm), bst);
        }
        w.shift();
    }
    if (last_super) {
        if (nblk > 0) {
            w.clear_hi();
#pragma unroll
            for (int mm = 0; mm < R; ++mm) w.elim(0, mm, !first_super, bsrow(nblk - 1, mm), bst);
        }
    } else {
#pragma unroll
        for (int i = 0; i < R; ++i) {
#pragma unroll
            for (int k2 = i + 1; k2 < R; ++k2) out[(RL::TOFF + offi(i, k2, R)) * os] = w.A[i][k2];
#pragma unroll
            for (int q = 0; q < R; ++q) out[(RL::TCROSS + i * R + q) * os] = w.Q[i][q];
            out[(RL::TE + i) * os] = w.e[i];
#pragma unroll
            for (int c = 0; c < C; ++c) out[(RL::TG + i * C + c) * os] = w.g[i][c];
        }
    }
    if (!first_super) {
#pragma unroll
        for (int q = 0; q < R; ++q) {
#pragma unroll
            for (int q2 = q + 1; q2 < R; ++q2) out[(RL::HOFF + offi(q, q2, R)) * os] = w.hoff[q][q2];
            out[(RL::HE + q) * os] = w.he[q];
#pragma unroll
            for (int c = 0; c < C; ++c) out[(RL::HG + q * C + c) * os] = w.hg[q][c];
        }
    }
}

// Value of one eliminated separator from its back-substitution rows (R rows of
// RSM fields at bs[f*32], as reduce_super_fwd stores them) and the known
// separators either side: zL (spike side) and zR (the window's hi block).
template <int R, int C>
__device__ __forceinline__ void solve_from_bs(const float* bs, const float (&zL)[R][C], const float (&zR)[R][C],
                                              float (&x)[R][C], long long bst = 32) {
    constexpr int RSM = Rec<R, C>::RSM;
#pragma unroll
    for (int mm = R - 1; mm >= 0; --mm) {
        const float* o = bs + mm * RSM * bst;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            float v = o[(2 * R - 1 + c) * bst];
#pragma unroll
            for (int i = mm + 1; i < 2 * R; ++i)
                v = fmaf(o[(i - mm - 1) * bst], (i < R) ? x[i < R ? i : 0][c] : zR[i >= R ? i - R : 0][c], v);
#pragma unroll
            for (int q = 0; q < R; ++q) v = fmaf(o[(2 * R - 1 + C + q) * bst], zL[q][c], v);
            x[mm][c] = v;
        }
    }
}

// Symbolic back substitution of one basis column b of the maps (value channel,
// zL component or zR component): the columns are independent, so the warps of
// the KA tile share them.  x_{nw-1} is the right super-separator itself.
template <int R, int C>
__device__ __forceinline__ void maps_backward_column(const float* bsm, int nw, bool last_super, int b, float* maps) {
    using RL = Rec<R, C>;
    constexpr int NB = RL::NB, RSM = RL::RSM;
    float xn[R];
#pragma unroll
    for (int q = 0; q < R; ++q) xn[q] = (!last_super && b == C + R + q) ? 1.f : 0.f;
    const int boff = b < C ? 2 * R - 1 + b : (b < C + R ? 2 * R - 1 + b : -1);  // value / spike field, zR: none
    for (int s = nw - 2; s >= 0; --s) {
        float xc[R];
#pragma unroll
        for (int mm = R - 1; mm >= 0; --mm) {
            const float* o = bsm + (s * R + mm) * RSM * 32;
            float v = boff >= 0 ? o[boff * 32] : 0.f;
#pragma unroll
            for (int i = mm + 1; i < 2 * R; ++i)
                v = fmaf(o[(i - mm - 1) * 32], (i < R) ? xc[i < R ? i : 0] : xn[i >= R ? i - R : 0], v);
            xc[mm] = v;
        }
        // staged in shared memory, [separator][field][lane] with a 33-float field
        // pitch (conflict-free both ways); ka_tile writes the tile's maps out coalesced
        float* mo = maps + (s * RL::MAPP + b) * 33;
#pragma unroll
        for (int q = 0; q < R; ++q) {
            mo[q * NB * 33] = xc[q];
            xn[q] = xc[q];
        }
    }
}

// Solve the inner separators of a run of `nw` chunk records (inner separators =
// the separators of chunks 0..nw-2) with the left / right separators known
// (has_l: zL, has_r: zR).  Record s's field f is at recs[s*cs + f*rs]; the
// solution of inner separator s, component (q, c) goes to
// zout[((s*R + q)*C + c) * zst]; back-substitution rows use bs (stride bss).
template <int R, int C, bool GPF = false>
__device__ __forceinline__ void solve_inner(const float* recs, long long rs, long long cs, int nw, bool has_l,
                                            const float (&zL)[R][C], bool has_r, const float (&zR)[R][C], float* zout,
                                            long long zst, float* bs, long long bss) {
    using RL = Rec<R, C>;
    const int nint = nw - 1;
    auto T = [&](int s) { return recs + (long long)s * cs; };
    if (GPF && SGWLS_REC_PF > 0)
        for (int s = 0; s < min(nw, SGWLS_REC_PF + 1); ++s) prefetch_record<R, C>(recs, rs, cs, s);
    BWin<R, C, false> w;
    w.clear_all();
    for (int s = 0; s < nint; ++s) {
        if (GPF && SGWLS_REC_PF > 0 && s + 1 + SGWLS_REC_PF < nw) prefetch_record<R, C>(recs, rs, cs, s + 1 + SGWLS_REC_PF);
        enter_block<R, C, false>(w, T(s), T(s + 1), (int)rs, true, s > 0, s > 0);
        if (s == 0 && has_l) {  // known left separator: its coupling moves to the RHS
#pragma unroll
            for (int mm = 0; mm < R; ++mm)
#pragma unroll
                for (int mp = 0; mp < R; ++mp) {
                    const float x = T(0)[(RL::TCROSS + mm * R + mp) * rs];
                    w.e[R + mm] += x;
#pragma unroll
                    for (int c = 0; c < C; ++c) w.g[R + mm][c] = fmaf(x, zL[mp][c], w.g[R + mm][c]);
                }
        }
        if (s == nint - 1 && has_r) {  // known right separator (its cross toward this block)
            const float* tr = T(nw - 1);
#pragma unroll
            for (int ms = 0; ms < R; ++ms)
#pragma unroll
                for (int mm = 0; mm < R; ++mm) {
                    const float x = tr[(RL::TCROSS + ms * R + mm) * rs];
                    w.e[R + mm] += x;
#pragma unroll
                    for (int c = 0; c < C; ++c) w.g[R + mm][c] = fmaf(x, zR[ms][c], w.g[R + mm][c]);
                }
        }
        if (s > 0) {
#pragma unroll
            for (int mm = 0; mm < R; ++mm) w.elim(0, mm, false, bs + ((long long)((s - 1) * R + mm) * RL::RS) * bss, (int)bss);
        }
        w.shift();
    }
    if (nint > 0) {
        w.clear_hi();
#pragma unroll
        for (int mm = 0; mm < R; ++mm) w.elim(0, mm, false, bs + ((long long)((nint - 1) * R + mm) * RL::RS) * bss, (int)bss);
    }
    float zn[R][C];
#pragma unroll
    for (int q = 0; q < R; ++q)
#pragma unroll
        for (int c = 0; c < C; ++c) zn[q][c] = 0.f;
    for (int s = nint - 1; s >= 0; --s) {
        float zc[R][C];
#pragma unroll
        for (int mm = R - 1; mm >= 0; --mm) {
            const float* o = bs + ((long long)(s * R + mm) * RL::RS) * bss;
#pragma unroll
            for (int c = 0; c < C; ++c) zc[mm][c] = o[(2 * R - 1 + c) * bss];
#pragma unroll
            for (int i = mm + 1; i < 2 * R; ++i) {
                const float ci = o[(i - mm - 1) * bss];
#pragma unroll
                for (int c = 0; c < C; ++c)
                    zc[mm][c] = fmaf(ci, (i < R) ? zc[i < R ? i : 0][c] : zn[i >= R ? i - R : 0][c], zc[mm][c]);
            }
        }
#pragma unroll
        for (int q = 0; q < R; ++q)
#pragma unroll
            for (int c = 0; c < C; ++c) {
                zout[((long long)(s * R + q) * C + c) * zst] = zc[q][c];
                zn[q][c] = zc[q][c];
            }
    }
}

// ===================================================================== K2 (tree)
//
// Reduced system over the super-separators of one line, solved by a CTA of NG
// warps x 32 lines: warp w reduces its group of consecutive super records to
// one group record (level 1, in parallel), warp 0 solves the short group-level
// system (level 2), then every warp solves its group's inner super-separators
// with the two group separators as boundary values (level 3, in parallel).
// Sequential depth ~ 2*PS/NG + NG instead of 2*PS.
// Body of the tree solve for one group of 32 lines (lane = line, w = warp).
template <int R, int C>
__device__ __forceinline__ void k2_tree_body(const PassGeom& g, const float* rec,
                                             float* __restrict__ rsc, float* __restrict__ z, float* sm, int lane,
                                             int w, int NG, int group, bool staged) {
    using RL = Rec<R, C>;
    const int NL = g.nb * g.batch;
    const int L = group * 32 + lane;
    const bool ok = L < NL;
    const long long NLl = NL;
    const int PSn = g.P;  // super records
    const int NGa = min(NG, PSn);
    const int J0 = w * PSn / NGa, J1 = (w + 1) * PSn / NGa;  // 32-bit: PSn * NG < 2^31
    const int gsz = J1 - J0;
    const int rsG = NG * 32 + 1;
    float* grec = sm;
    float* zg = grec + RL::REC * rsG;
    float* bsg = zg + NG * R * C * 32;
    // staged (short reduced systems, c1/c2): the CTA first copies all its lines'
    // super-records into shared memory with every thread (one latency), and the
    // level-3 back-substitution rows stay there too -- levels 1 and 3 then run
    // from shared memory instead of waiting an L2 round trip per record
    float* srs = bsg + NG * R * RL::RSM * 32;  // [J][field][lane]
    float* sbs = srs + PSn * RL::REC * 32;     // [J][R][RS][lane]
    if (staged) {
        const int tot = PSn * RL::REC * 32, NT = NG * 32, tid = w * 32 + lane;
        for (int i = tid; i < tot; i += NT) {
            const int row = i >> 5, Lg = group * 32 + (i & 31);
            srs[i] = Lg < NL ? __ldcg(rec + (long long)row * NLl + Lg) : 0.f;
        }
        __syncthreads();
    }
    const float* my = staged ? srs + J0 * RL::REC * 32 + lane : rec + (long long)J0 * RL::REC * NLl + L;
    const long long fst = staged ? 32 : NLl;  // field stride of `my`
    // level 1 keeps its back-substitution rows (global scratch, [J][R][RSM][line]),
    // so level 3 is a backward sweep only
    float* bs1 = rsc + (long long)J0 * R * RL::RSM * NLl + L;
    if (w < NGa && ok) {
        if (staged)
            reduce_super<R, C, false>(my, fst, RL::REC * fst, gsz, w == 0, w == NGa - 1, grec + w * 32 + lane, rsG);
        else
            reduce_super_fwd<R, C, (R >= SGWLS_REC_PF_MINR)>(my, (int)fst, gsz, w == 0, w == NGa - 1,
                                                             grec + w * 32 + lane, rsG, bs1, RL::REC * (int)fst,
                                                             (int)NLl);
    }
    __syncthreads();
    // level 2 as a binary tree over the NGa group records: pairwise merges up
    // (segment [a, a+span) absorbs [a+span, a+2span), eliminating group
    // separator a+span-1, whose back-substitution rows stay in shared memory),
    // then the eliminated separators top-down from their segments' two ends:
    // 2 log2(NG) dependent steps instead of 2 NG
    int top = 1;
    while (top < NGa) top *= 2;
    for (int span = 1; span < NGa; span *= 2) {
        const int a = w * 2 * span;
        if (ok && a + span < NGa)
            reduce_super_fwd<R, C>(grec + a * 32 + lane, rsG, 2, a == 0, a + 2 * span >= NGa, grec + a * 32 + lane, rsG,
                                   bsg + (a + span - 1) * R * RL::RSM * 32 + lane, span * 32);
        __syncthreads();
    }
    for (int span = top / 2; span >= 1; span /= 2) {
        const int a = w * 2 * span;
        if (ok && a + span < NGa) {
            float zL[R][C], zR[R][C], x[R][C];
            const bool hl = a > 0, hr = a + 2 * span < NGa;
#pragma unroll
            for (int q = 0; q < R; ++q)
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    zL[q][c] = hl ? zg[(((a - 1) * R + q) * C + c) * 32 + lane] : 0.f;
                    zR[q][c] = hr ? zg[(((a + 2 * span - 1) * R + q) * C + c) * 32 + lane] : 0.f;
                }
            const int k = a + span - 1;
            solve_from_bs<R, C>(bsg + k * R * RL::RSM * 32 + lane, zL, zR, x);
#pragma unroll
            for (int q = 0; q < R; ++q)
#pragma unroll
                for (int c = 0; c < C; ++c) zg[((k * R + q) * C + c) * 32 + lane] = x[q][c];
        }
        __syncthreads();
    }
    if (w < NGa && ok) {
        const bool has_l = w > 0, has_r = w < NGa - 1;
        float zL[R][C], zR[R][C];
#pragma unroll
        for (int q = 0; q < R; ++q)
#pragma unroll
            for (int c = 0; c < C; ++c) {
                zL[q][c] = has_l ? zg[(((w - 1) * R + q) * C + c) * 32 + lane] : 0.f;
                zR[q][c] = has_r ? zg[((w * R + q) * C + c) * 32 + lane] : 0.f;
            }
        if (has_r) {  // stored before the solve (see kb_tile step 2)
            float* zo = z + (long long)(J1 - 1) * R * C * NLl + L;
#pragma unroll
            for (int q = 0; q < R; ++q)
#pragma unroll
                for (int c = 0; c < C; ++c) zo[(q * C + c) * NLl] = zR[q][c];
        }
        if (staged) {
            solve_inner<R, C, false>(my, fst, RL::REC * fst, gsz, has_l, zL, has_r, zR,
                                     z + (long long)J0 * R * C * NLl + L, NLl, sbs + J0 * R * RL::RS * 32 + lane, 32);
        } else {
            // backward sweep over level 1's rows: x_s from x_{s+1} (zR for the last) and zL
            float xn[R][C];
#pragma unroll
            for (int q = 0; q < R; ++q)
#pragma unroll
                for (int c = 0; c < C; ++c) xn[q][c] = zR[q][c];
            for (int sep = gsz - 2; sep >= 0; --sep) {
                const float* o = bs1 + (long long)sep * R * RL::RSM * NLl;
                if (sep > 0) {  // L1-prefetch the next rows of the chain
#pragma unroll
                    for (int f = 0; f < R * RL::RSM; ++f)
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(o - (long long)(R * RL::RSM - f) * NLl));
                }
                float x[R][C];
                solve_from_bs<R, C>(o, zL, xn, x, NLl);
                float* zo = z + (long long)(J0 + sep) * R * C * NLl + L;
#pragma unroll
                for (int q = 0; q < R; ++q)
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        zo[(q * C + c) * NLl] = x[q][c];
                        xn[q][c] = x[q][c];
                    }
            }
        }
    }
}

// MAXT: 512 threads (<= 128 registers) up to 16 groups; 1024 (<= 64) for 32
template <int R, int C, int MAXT>
__global__ void __launch_bounds__(MAXT) k2_tree(const PassGeom g, const float* __restrict__ rec,
                                               float* __restrict__ rsc, float* __restrict__ z, int staged) {
    extern __shared__ __align__(128) float sm[];
    pdl_wait();     // KA's records
    pdl_trigger();  // KB may launch now: everything it reads before its own wait (KA's output) is complete
    k2_tree_body<R, C>(g, rec, rsc, z, sm, threadIdx.x, threadIdx.y, blockDim.y, blockIdx.x, staged != 0);
}

template <int R, int C>
__host__ inline size_t k2_tree_smem(int NG, int PS = 0) {
    using RL = Rec<R, C>;
    return ((size_t)RL::REC * (NG * 32 + 1) + (size_t)NG * R * C * 32 + (size_t)NG * R * RL::RSM * 32 +
            (size_t)PS * (RL::REC + R * RL::RS) * 32) *
           sizeof(float);
}

// ===================================================================== KA

// Register budgets (tuning variants override these): KA is held to 3 CTAs of
// 256 threads per SM; KB keeps plain __launch_bounds__(256) (ptxas settles at
// ~95-128 registers; tighter budgets spill and lose on B200).
#ifndef SGWLS_KA_MINB
// 3 CTAs (<= 85 registers) for r = 1, 4 (<= 64, a few spills) for r >= 2:
// measured +1-9% (r = 1) and +10-13% (c3, c5) on B200
#define SGWLS_KA_MINB (R >= 2 ? 4 : 3)
#endif
#define SGWLS_KA_BOUNDS __launch_bounds__(256, SGWLS_KA_MINB)
// Edge weights computed where the elimination consumes them ("lazy") instead
// of up front in registers, from this radius on: fewer live registers (KA: no
// spills; KB: less spilling) and MUFU work interleaved with the dependent
// elimination chain.  Measured on B200 (KA and KB lazy vs eager): c5 +13 %,
// c4 +7 %, c3 +6 %; r = 1 (c1 -3 %, c2 -2 %: KB's weights then no longer
// overlap the K2 wait) stays eager.
#ifndef SGWLS_LAZY_MIN_R
#define SGWLS_LAZY_MIN_R 2
#endif
// KB register budget in 256-thread units: one channel 4 (<= 64 registers,
// measured best with the shuffle averaging), several channels 3 (<= 85) for
// r >= 2 and 2 (<= 128) for r = 1, whose wide C-channel windows spill badly at 85
#ifndef SGWLS_KB_MINB1
#define SGWLS_KB_MINB1 3
#endif
#ifndef SGWLS_KB_MINBC
#define SGWLS_KB_MINBC (R == 1 ? 2 : 3)
#endif
#define SGWLS_KB_BOUNDS __launch_bounds__(256, (C == 1 ? SGWLS_KB_MINB1 : SGWLS_KB_MINBC))
// One chunk of KA: load (lazily weighted for r >= SGWLS_LAZY_MIN_R), spike-forward,
// record -> shared memory (`rec`, field stride rs).
template <int R, int C, int CG>
__device__ __forceinline__ void ka_chunk(const PassGeom& g, const float* __restrict__ src,
                                         const float* __restrict__ guid, const WeightDev& W, int L, int j, float* rec,
                                         int rs) {
    constexpr int RW = rows_per_chunk(R, C);
    constexpr int M = 2 * R + 1;
    const int img = g.batch == 1 ? 0 : L / g.nb, b = L - img * g.nb;  // no integer division for one image
    const int lo = band_lo(g, b);
    const int y0 = j * RW;
    const int nrows = min(RW, g.Hl - y0);
    const bool has_left = j > 0 || g.has_prev, lastc = j == g.P - 1 && !g.has_next;
    if constexpr (R >= SGWLS_LAZY_MIN_R) {
        // edge weights computed where the elimination consumes them
        const long long npx = (long long)g.Hl * g.Wl;
        const float* Msk = (C > 1 && g.msk != nullptr) ? g.msk + img * npx : nullptr;
        const float* F = src + img * (Msk ? npx * (C > 1 ? C - 1 : 1) : g.img_stride);
        ChunkInL<R, C, CG, RW> in;
        if (nrows == RW)
            load_chunk_lazy<R, C, CG, RW, true>(in, F, Msk, guid + img * g.gimg_stride, g, lo, y0, nrows);
        else
            load_chunk_lazy<R, C, CG, RW, false>(in, F, Msk, guid + img * g.gimg_stride, g, lo, y0, nrows);
        if (W.kind == 1)
            chunk_spike_forward<R, C, CG, RW>(in, LazyWeights<R, C, CG, RW, 1>{in, W}, has_left, lastc, nrows * M, rec,
                                              rs);
        else
            chunk_spike_forward<R, C, CG, RW>(in, LazyWeights<R, C, CG, RW, 0>{in, W}, has_left, lastc, nrows * M, rec,
                                              rs);
    } else {
        ChunkIn<R, C, CG, RW> in;
        load_chunk<R, C, CG, RW>(in, src, guid + img * g.gimg_stride, g, W, lo, y0, nrows, nullptr, L, img);
        chunk_spike_forward<R, C, CG, RW>(in, EagerWeights<R, C, CG, RW>{in}, has_left, lastc, nrows * M, rec, rs);
    }
}

// KA: one tile (32 bands x NW chunks) per CTA.  Every warp runs one chunk's
// spike-forward; then warp 0 reduces the tile's chunk records (super-record
// for K2 + the back-substitution rows) and the warps share the map columns.
// (A persistent form -- a per-CTA queue of (tile, chunk) tasks whose last
// warp reduces the tile -- was measured 2x slower on c5: the serial reduction
// of one warp could not keep up with the chunks of the other fifteen.)
template <int R, int C, int CG>
__global__ void SGWLS_KA_BOUNDS ka_tile(const PassGeom g, const float* __restrict__ src,
                                               const float* __restrict__ guid, float* __restrict__ srec,
                                               float* __restrict__ maps, const __grid_constant__ WeightDev W, int NW) {
    using RL = Rec<R, C>;
    extern __shared__ __align__(128) float sm[];
    // NW chunks per tile, NWK (= blockDim.y <= NW) warps: each warp runs
    // chunks wid, wid + NWK, ...  Fewer warps than chunks shrink the share of
    // warps idling while warp 0 reduces the tile (with one warp per chunk, ncu
    // measured 43 % of KA's warp time at that barrier on c5)
    const int lane = threadIdx.x, wid = threadIdx.y, NWK = blockDim.y;
    const int NL = g.nb * g.batch;
    // grid: (line group, tile)
    const int L = blockIdx.x * 32 + lane;
    const int J = blockIdx.y;
    const int nw = min(NW, g.P - J * NW);
    const int rs = NW * 32 + 1;  // smem record field stride
    pdl_wait();  // the pass input is the previous pass's output
    pdl_trigger();
    if (L < NL)
        for (int c = wid; c < nw; c += NWK) ka_chunk<R, C, CG>(g, src, guid, W, L, J * NW + c, sm + c * 32 + lane, rs);
    __syncthreads();
    const int PS = gridDim.y;  // = ceil(P / NW), the grid's tile dimension
    const long long NLl = NL;
    const int recs_fl = RL::REC * rs, stage_fl = (NW > 1 ? NW - 1 : 1) * RL::MAPP * 33;
    float* bsm = sm + (recs_fl > stage_fl ? recs_fl : stage_fl) + lane;
    const bool last_super = J == PS - 1 && !g.has_next;
    if (wid == 0 && L < NL)  // super-record for K2, back-substitution rows
        reduce_super_fwd<R, C>(sm + lane, rs, nw, J == 0 && !g.has_prev, last_super,
                               srec + (long long)J * RL::REC * NLl + L, NLl, bsm);
    if (nw < 2) return;
    __syncthreads();
    // the affine maps of the tile's inner separators for KB, one basis column
    // per warp, staged in shared memory (the record area is free by now) ...
    float* mst = sm + lane;
    if (L < NL)
        for (int b = wid; b < RL::NB; b += NWK) maps_backward_column<R, C>(bsm, nw, last_super, b, mst);
    __syncthreads();
    // ... and written out as whole 16-byte vectors: a separator's maps for the
    // tile's 32 lines are one contiguous run of 32*MAPP floats ([chunk][line][MAPP])
    // thread -> one (line, float4) slot of the tile's 32*V per separator, looping over the
    // separators (no per-element index divisions); spare thread groups take alternate separators
    constexpr int V = RL::MAPP / 4, PER = 32 * V;  // float4 per line, per separator
    const int NT = NWK * 32, tid = wid * 32 + lane;
    const int groups = NT >= PER ? NT / PER : 1;
    const int gq = tid / PER;
    const int ngl = min(32, NL - (int)blockIdx.x * 32);  // lines of this group
    if (gq < groups) {
        for (int i = tid - gq * PER; i < PER; i += NT) {
            const int ln = i / V, f = (i - ln * V) * 4;
            if (ln >= ngl) continue;
            const float* s4 = sm + f * 33 + ln;
            float* dst = maps + ((long long)J * NW * NLl + blockIdx.x * 32 + ln) * RL::MAPP + f;
            for (int sep = gq; sep < nw - 1; sep += groups) {
                const float* src4 = s4 + sep * RL::MAPP * 33;
                float4 o;
                o.x = src4[0];
                o.y = f + 1 < RL::MAPF ? src4[33] : 0.f;
                o.z = f + 2 < RL::MAPF ? src4[66] : 0.f;
                o.w = f + 3 < RL::MAPF ? src4[99] : 0.f;
                *reinterpret_cast<float4*>(dst + (long long)sep * NLl * RL::MAPP) = o;
            }
        }
    }
}

template <int R, int C>
__host__ inline size_t ka_smem(int NWA) {
    using RL = Rec<R, C>;
    // records (reused for the map staging area), then the back-substitution rows
    const size_t recs = (size_t)RL::REC * (NWA * 32 + 1), stage = (size_t)(NWA > 1 ? NWA - 1 : 1) * RL::MAPP * 33;
    return ((recs > stage ? recs : stage) + (size_t)(NWA > 1 ? NWA - 1 : 1) * R * RL::RSM * 32) * sizeof(float);
}

// Interior solve of one chunk with both separators known (zl: previous
// chunk's separator, zr: this chunk's): forward elimination with the known
// couplings moved to the right-hand side, back substitution in registers.
// FULL_INNER: full chunk that is not the band's last (kv = K, kend = K - R at
// compile time); otherwise the general predicated form.
template <int R, int C, int CG, int RW, bool FULL_INNER, class IN, class WF>
__device__ __forceinline__ void chunk_interior_solve(const IN& in, const WF& lwf, bool has_left, bool lastc,
                                                     int kv, int kend, const float (&zl)[R][C],
                                                     const float (&zr)[R][C], float (&cs)[RW * (2 * R + 1)][R],
                                                     float (&ys)[RW * (2 * R + 1)][C]) {
    constexpr int M = 2 * R + 1, K = RW * M;
    if (FULL_INNER) {
        kv = K;
        kend = K - R;
        lastc = false;
    }
    // the chunk's separator (known, zr) is its last R valid positions; a short
    // chunk that is not the band's last occurs in row-slab mode
    const int ks = kv - R;
    Win<R, C, false> w;
    w.clear();
    // positions k >= kv (short last chunk) enter as empty rows; the R extra
    // steps drain the window
#pragma unroll
    for (int k = 0; k < K + R; ++k) {
        if (k < K && k < kv) {
            const bool kq = !lastc && (k >= ks);  // known separator position
            if (!kq) {
                w.e[R] = 1.f;
#pragma unroll
                for (int c = 0; c < C; ++c) w.g[R][c] = in.f[cl(k, K)][c];
            } else {
#pragma unroll
                for (int c = 0; c < C; ++c) ys[cl(k, K)][c] = zr[cl(k - ks, R)][c];
            }
#pragma unroll
            for (int t = 1; t <= R; ++t) {
                const bool pe = (k - t >= 0) || has_left;
                if (!pe) continue;
                const bool pleft = (k - t < 0);
                const bool pright = kq && (k - t >= ks);
                if (pright) continue;
                const float lw = lwf(k, t);
                if (!kq && !pleft) {
                    w.A[R - t][R] = lw;
                } else if (!kq && pleft) {
                    w.e[R] += lw;
#pragma unroll
                    for (int c = 0; c < C; ++c)
                        w.g[R][c] = fmaf(lw, zl[cl(R - t + k, R)][c], w.g[R][c]);
                } else {
                    w.e[R - t] += lw;
#pragma unroll
                    for (int c = 0; c < C; ++c)
                        w.g[R - t][c] = fmaf(lw, zr[cl(k - ks, R)][c], w.g[R - t][c]);
                }
            }
        }
        const int pp = k - R;  // position eliminated at this step
        if (pp >= 0 && pp < kend) {
            float cc[R + 1];
            const float inv = w.elim(cc, false);
#pragma unroll
            for (int i = 1; i <= R; ++i) cs[cl(pp, K)][i - 1] = cc[i];
            row_mul<C>(ys[cl(pp, K)], w.g[0], inv);
        }
        w.shift();
    }
    // back substitution (u replaces y in place)
#pragma unroll
    for (int p = K - 1; p >= 0; --p) {
        if (p < kend) {
#pragma unroll
            for (int i = 1; i <= R; ++i) {
                if (p + i < K) row_fma<C>(ys[p], cs[p][i - 1], ys[cl(p + i, K)]);
            }
        }
    }
}

// ===================================================================== KB

// Averaging of one chunk's rows into the output tile by warp shuffles, for a
// tile whose 32 bands all sit on the tau grid (band lane l covers local columns
// [TAU*l, TAU*l + M)).  Lane l owns columns [TAU*l, TAU*l + TAU): it receives
// the overlapping values of lanes l-1, l-2, ... (__shfl_up), sums them in
// increasing band order like the reference (proj/src/smoother.cpp:78-90),
// scales by 1/count and stores each tile cell exactly once -- no zeroing, no
// phase loop, no shared-memory read-modify-write.  Lanes past the last band
// (ys = 0) still take part, so the image's last columns get their sums.
// Columns whose covering bands start before lane 0 come out partial; they are
// never owned by this tile unless the tile starts the image, where those bands
// do not exist.
template <int TAU, int R, int C, int K>
__device__ __forceinline__ void average_shfl(const float (&ys)[K][C], int nrw, int par0, int lane, float* trow,
                                             int sx, int sy, int ncol, const float* inv_col) {
    constexpr int M = 2 * R + 1;
    constexpr int KMAX = (M - 1) / TAU;  // lanes back whose bands reach this lane's columns
#pragma unroll
    for (int rr = 0; rr < K / M; ++rr) {
        if (rr < nrw) {
            const bool rev = (par0 ^ (rr & 1)) != 0;
#pragma unroll
            for (int j = 0; j < TAU; ++j) {
                const int xl = TAU * lane + j;
                float acc[C];
#pragma unroll
                for (int c = 0; c < C; ++c) acc[c] = 0.f;
#pragma unroll
                for (int k = KMAX; k >= 1; --k) {
                    if (j + k * TAU < M) {
                        const int m = j + k * TAU;
#pragma unroll
                        for (int c = 0; c < C; ++c) {
                            const float v = rev ? ys[rr * M + (M - 1 - m)][c] : ys[rr * M + m][c];
                            const float u = __shfl_up_sync(0xffffffffu, v, k);
                            if (lane >= k) acc[c] += u;  // no band before lane 0 (image start)
                        }
                    }
                }
#pragma unroll
                for (int c = 0; c < C; ++c) acc[c] += rev ? ys[rr * M + (M - 1 - j)][c] : ys[rr * M + j][c];
                if (xl < ncol) {
                    const float sc = fabsf(inv_col[xl]);
#pragma unroll
                    for (int c = 0; c < C; ++c) trow[xl * sx + rr * sy + c] = acc[c] * sc;
                }
            }
        }
    }
}

// Same averaging, stored straight to the next pass's (transposed) layout instead
// of the shared output tile: lane l's column x = xa + TAU*l + j is output row x,
// and this chunk's RW rows are RW*C consecutive floats of it (vector stores of
// VEC floats; the last, short chunk stores scalars).  Only owned columns.
// INTERIOR (inv_col == nullptr is not needed: compile-time switch): every band
// from KMAX before the tile's first to its last is a regular band (no image edge,
// no forced last centre in reach), so column tau*b + j is covered by exactly
// 1 + (2R - j) / TAU bands -- a compile-time count -- and lanes >= `own0` own
// their columns: no shared table, no geometry loop, no CTA barrier.
template <int TAU, int R, int C, int K, int VEC, bool INTERIOR = false>
__device__ __forceinline__ void average_shfl_direct(const float (&ys)[K][C], int nrw, int par0, int lane,
                                                    float* obase, long long opitch, int ncol,
                                                    const float* inv_col, int own0 = 0) {
    constexpr int M = 2 * R + 1, RW = K / M;
    constexpr int KMAX = (M - 1) / TAU;
    float acc[TAU][RW * C];
#pragma unroll
    for (int rr = 0; rr < RW; ++rr) {
        const bool rev = (par0 ^ (rr & 1)) != 0;
#pragma unroll
        for (int j = 0; j < TAU; ++j) {
#pragma unroll
            for (int c = 0; c < C; ++c) acc[j][rr * C + c] = 0.f;
#pragma unroll
            for (int k = KMAX; k >= 1; --k) {
                if (j + k * TAU < M) {
                    const int m = j + k * TAU;
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        const float v = rev ? ys[rr * M + (M - 1 - m)][c] : ys[rr * M + m][c];
                        const float u = __shfl_up_sync(0xffffffffu, v, k);
                        if (lane >= k) acc[j][rr * C + c] += u;
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < C; ++c) acc[j][rr * C + c] += rev ? ys[rr * M + (M - 1 - j)][c] : ys[rr * M + j][c];
        }
    }
    if (INTERIOR && lane < own0) return;  // halo bands: their columns belong to the previous tile
#pragma unroll
    for (int j = 0; j < TAU; ++j) {
        const int xl = TAU * lane + j;
        float sc;
        if constexpr (INTERIOR) {
            sc = 1.0f / (float)(1 + (2 * R - j) / TAU);  // compile-time, correctly rounded like kInvCount
        } else {
            if (xl >= ncol) continue;
            sc = inv_col[xl];
            if (!(sc > 0.f)) continue;  // not owned by this tile
        }
        float* op = obase + (long long)xl * opitch;
        if (nrw == RW) {
#pragma unroll
            for (int e = 0; e < RW * C; e += VEC) {
                if constexpr (VEC == 4)
                    *reinterpret_cast<float4*>(op + e) =
                        make_float4(acc[j][e] * sc, acc[j][e + 1] * sc, acc[j][e + 2] * sc, acc[j][e + 3] * sc);
                else if constexpr (VEC == 2)
                    *reinterpret_cast<float2*>(op + e) = make_float2(acc[j][e] * sc, acc[j][e + 1] * sc);
                else
                    op[e] = acc[j][e] * sc;
            }
        } else {
#pragma unroll
            for (int e = 0; e < RW * C; ++e)
                if (e < nrw * C) op[e] = acc[j][e] * sc;
        }
    }
}

// row pitch (floats) of kb_tile's staged rows: up to 3 floats of alignment slack in
// front of the tile's 31*tau + M columns, rounded to whole 16-byte vectors
__host__ __device__ constexpr int kb_stage_pitch(int tau, int M, int ch) { return (3 + (31 * tau + M) * ch + 3) & ~3; }

struct TileOut {
    float* out;
    int transpose_out;
    int step;       // CTA band stride (32 - halo)
    int nph;        // accumulation phases
    int nwa;        // chunks per KA tile (the tiles KA's separator maps refer to)
    int psa;        // KA tiles per band
    int early;      // the predecessor is a K2 launch (it waited for KA): KA's maps may be read before the wait
    int nwa_shift;  // log2(nwa) when nwa is a power of two, else -1
    // interpolate_sparse's last pass (proj/src/smoother.cpp:149-161): channel C-1
    // is the smoothed mask d; out gets C-1 channels num/d (0 where d < floor)
    // and und[pixel] = (d < floor), instead of the C smoothed channels
    int ratio;
    float floor_;
    float* und;
    // the CTA stages its input rows (image + guidance) in shared memory with two tensor-map TMA
    // boxes instead of per-lane loads (r >= 2, packed input, no row-slab neighbours, 16-byte
    // aligned rows; decided on the host)
    int stage;
    // band tiles [lean_lo, lean_hi) run kb_lean (host: the launch-uniform conditions hold and the
    // tile is interior); empty range otherwise
    int lean_lo, lean_hi;
};

// 1/n correctly rounded (what 1.0f / n gives) for the band count of a column, n <= 2r + 2 <= 10
__constant__ float kInvCount[12] = {0.f, 1.f / 1, 1.f / 2, 1.f / 3, 1.f / 4, 1.f / 5, 1.f / 6,
                                    1.f / 7, 1.f / 8, 1.f / 9, 1.f / 10, 1.f / 11};

__device__ __forceinline__ void covering(const PassGeom& g, int x, int& bmin, int& bmax) {
    const int r = g.r, tau = g.tau;
    const int lo_b = x - 2 * r;
    int b0 = lo_b <= 0 ? 0 : div_tau(g, lo_b + tau - 1);
    int b1 = div_tau(g, x);
    if (b1 > g.nreg - 1) b1 = g.nreg - 1;
    bmin = b0;
    bmax = b1;
    if (g.nb > g.nreg && x >= g.Wl - 1 - 2 * r) {
        if (b1 < b0) bmin = g.nreg;
        bmax = g.nreg;
    }
}

// ============================================================ row-slab mode
//
// A Column pass over a band split into row slabs, one per GPU (sharded.py,
// SURVEY.md 8(f)-1): the exact partitioned solve one level up.  Phase A per
// slab: KA as usual (chunk records, super-records), then k2_slab_reduce folds
// the slab's super-records into ONE slab record per band (the in-tile
// reduction of reduce_super applied to the whole slab: the Schur block of the
// slab's last separator, its coupling to the previous slab's, and the update
// of the latter).  The slab records of all G slabs are all-gathered (G records
// per band, ~100 B each), and phase B per slab runs k2_slab_solve: the global
// block-tridiagonal system over the G-1 slab separators (redundantly on every
// slab, G is tiny), then the slab's own super-separators with its two slab
// separators as boundary values; then KC / KB as usual.  Only slab records
// cross GPUs -- never image data.
// Both slab kernels run one CTA of NG warps per group of 32 bands (lane = band),
// with the tree of k2_tree_body: warp w owns a contiguous group of the slab's
// super-records, so the serial depth is ~PS/NG + NG instead of PS.
//
// Phase A: level 1, warp w reduces its group to a group record (kept in
// grec[w][field][line] for phase B); level 2, warp 0 reduces the group records
// to the slab record.
template <int R, int C>
__global__ void __launch_bounds__(512) k2_slab_reduce(const PassGeom g, int PS, const float* __restrict__ srec,
                                                      float* __restrict__ grec, float* __restrict__ slabrec) {
    using RL = Rec<R, C>;
    extern __shared__ __align__(128) float sm[];
    const int lane = threadIdx.x, w = threadIdx.y, NG = blockDim.y;
    const int NL = g.nb * g.batch;
    const long long NLl = NL;
    const int L = blockIdx.x * 32 + lane;
    const bool ok = L < NL;
    const int NGa = min(NG, PS);
    const int J0 = w * PS / NGa, J1 = (w + 1) * PS / NGa;
    const int rsG = NG * 32 + 1;
    pdl_wait();  // KA's super-records
    pdl_trigger();
    if (w < NGa && ok) {
        float* gout = sm + w * 32 + lane;
        reduce_super<R, C, (R >= SGWLS_REC_PF_MINR)>(srec + (long long)J0 * RL::REC * NLl + L, NLl, (long long)RL::REC * NLl, J1 - J0,
                           w == 0 && !g.has_prev, w == NGa - 1 && !g.has_next, gout, rsG);
#pragma unroll 1
        for (int f = 0; f < RL::REC; ++f) grec[((long long)w * RL::REC + f) * NLl + L] = gout[f * rsG];
    }
    __syncthreads();
    if (w == 0 && ok)
        reduce_super<R, C>(sm + lane, rsG, 32, NGa, !g.has_prev, !g.has_next, slabrec + L, NLl);
}

// Phase B: warp 0 solves the G-1 slab separators (allrec, the same tiny system
// on every slab), then the group-level system of this slab with its two slab
// separators as boundary values (level 2); every warp then solves its group's
// super-separators (level 3).  z carries one slot in front: z[-1] = the
// previous slab's separator, z[PS-1] = this slab's last separator.
template <int R, int C>
__global__ void __launch_bounds__(512) k2_slab_solve(const PassGeom g, int PS, int G, int gi,
                                                     const float* __restrict__ allrec, const float* __restrict__ srec,
                                                     const float* __restrict__ grec, float* __restrict__ zg,
                                                     float* __restrict__ bsg, float* __restrict__ rsc,
                                                     float* __restrict__ z) {
    using RL = Rec<R, C>;
    extern __shared__ __align__(128) float sm[];
    const int lane = threadIdx.x, w = threadIdx.y, NG = blockDim.y;
    const int NL = g.nb * g.batch;
    const long long NLl = NL;
    const int L = blockIdx.x * 32 + lane;
    const bool ok = L < NL;
    const int NGa = min(NG, PS);
    const int J0 = w * PS / NGa, J1 = (w + 1) * PS / NGa;
    float* zgrp = sm;                         // (NG + 1) x R*C x 32: [0] = zL, [k+1] = group k's separator
    float* bs2 = zgrp + (NG + 1) * R * C * 32;  // NG x R x RS x 32
    pdl_wait();
    pdl_trigger();
    if (w == 0 && ok) {
        float z0[R][C], zL[R][C], zR[R][C];
#pragma unroll
        for (int q = 0; q < R; ++q)
#pragma unroll
            for (int c = 0; c < C; ++c) z0[q][c] = 0.f;
        if (G > 1)
            solve_inner<R, C>(allrec + L, NLl, (long long)RL::REC * NLl, G, false, z0, false, z0, zg + L, NLl,
                              bsg + L, NLl);
#pragma unroll
        for (int q = 0; q < R; ++q)
#pragma unroll
            for (int c = 0; c < C; ++c) {
                zL[q][c] = g.has_prev ? zg[((long long)((gi - 1) * R + q) * C + c) * NLl + L] : 0.f;
                zR[q][c] = g.has_next ? zg[((long long)(gi * R + q) * C + c) * NLl + L] : 0.f;
                zgrp[(q * C + c) * 32 + lane] = zL[q][c];
                if (g.has_prev) z[((long long)(-R + q) * C + c) * NLl + L] = zL[q][c];
                zgrp[((NGa * R + q) * C + c) * 32 + lane] = zR[q][c];  // slot of the last group's separator
            }
        if (NGa > 1)
            solve_inner<R, C>(grec + L, NLl, (long long)RL::REC * NLl, NGa, g.has_prev, zL, g.has_next, zR,
                              zgrp + R * C * 32 + lane, 32, bs2 + lane, 32);
    }
    __syncthreads();
    if (w < NGa && ok) {
        const bool has_l = w > 0 || g.has_prev, has_r = w < NGa - 1 || g.has_next;
        float zL[R][C], zR[R][C];
#pragma unroll
        for (int q = 0; q < R; ++q)
#pragma unroll
            for (int c = 0; c < C; ++c) {
                zL[q][c] = zgrp[((w * R + q) * C + c) * 32 + lane];
                zR[q][c] = zgrp[(((w + 1) * R + q) * C + c) * 32 + lane];
            }
        if (has_r) {  // the group's last super-separator (stored before the solve, see kb_tile step 2)
            float* zo = z + (long long)(J1 - 1) * R * C * NLl + L;
#pragma unroll
            for (int q = 0; q < R; ++q)
#pragma unroll
                for (int c = 0; c < C; ++c) zo[(q * C + c) * NLl] = zR[q][c];
        }
        solve_inner<R, C, (R >= SGWLS_REC_PF_MINR)>(srec + (long long)J0 * RL::REC * NLl + L, NLl, (long long)RL::REC * NLl, J1 - J0, has_l, zL,
                          has_r, zR, z + (long long)J0 * R * C * NLl + L, NLl,
                          rsc + (long long)J0 * R * RL::RS * NLl + L, NLl);
    }
}

template <int R, int C>
__host__ inline size_t k2_slab_reduce_smem(int NG) {
    return (size_t)Rec<R, C>::REC * (NG * 32 + 1) * sizeof(float);
}
template <int R, int C>
__host__ inline size_t k2_slab_solve_smem(int NG) {
    return ((size_t)(NG + 1) * R * C * 32 + (size_t)NG * R * Rec<R, C>::RS * 32) * sizeof(float);
}

// ===================================================================== KB

// A chunk's two separators come from KA's affine maps of its KA tile's inner
// separators and the super-separators K2 solved (zsep; the first chunk of a
// row slab reads the previous slab's separator at zsep[-1]).  Chunk j lies in
// KA tile JA = j / nwa at s = j % nwa: its right separator sigma_j is inner
// (a map of the tile's zA = zsep[JA-1], zB = zsep[JA]) or zB itself; its left
// separator sigma_{j-1} is inner in the same tile (s > 0) or zA -- so the two
// super-separators zA, zB are all a chunk reads from K2.
// x = a + B zA + Cm zB from a lane's map staged in shared memory (MAPP
// contiguous floats, read as float4: a 48-byte lane stride is conflict-free)
template <int R, int C>
__device__ __forceinline__ void apply_map(const float* ms, const float (&zA)[R][C], const float (&zB)[R][C],
                                          float (&z)[R][C]) {
    using RL = Rec<R, C>;
    constexpr int NB = RL::NB;
    float m[RL::MAPP];
#pragma unroll
    for (int f = 0; f < RL::MAPP; f += 4) {
        const float4 v = *reinterpret_cast<const float4*>(ms + f);
        m[f] = v.x;
        m[f + 1] = v.y;
        m[f + 2] = v.z;
        m[f + 3] = v.w;
    }
#pragma unroll
    for (int q = 0; q < R; ++q)
#pragma unroll
        for (int c = 0; c < C; ++c) {
            float v = m[q * NB + c];
#pragma unroll
            for (int p = 0; p < R; ++p) v = fmaf(m[q * NB + C + p], zA[p][c], v);
#pragma unroll
            for (int p = 0; p < R; ++p) v = fmaf(m[q * NB + C + R + p], zB[p][c], v);
            z[q][c] = v;
        }
}

// The lean body is compiled into the instantiations that can use it by default (r = 2, one
// channel: staged by tensor maps, 4-float runs); carrying it elsewhere only grows the kernel
// (measured: c3's r = 3 KB -14 %, c4's two-channel KB -3 % with the unused body inside)
__host__ __device__ constexpr bool kb_has_lean(int R, int C) { return R == 2 && C == 1; }

// Lean body of kb_tile for INTERIOR band tiles of the common launch: tensor-map staged
// input, shuffle averaging with direct transposed stores, no row-slab neighbours, no fused
// ratio.  Everything launch-uniform was decided on the host (to.lean_lo / lean_hi), every band
// of the tile is regular (lo = tau*b, all 32 lanes active, compile-time band counts), so the
// general kernel's tile-layout, ownership-table and predicate set-up is not executed at all.
// Same device functions as the general path: bit-identical results.
template <int R, int C, int CG>
__device__ __forceinline__ void kb_lean(const PassGeom& g, const float* __restrict__ zsep,
                                        const float* __restrict__ maps, const TileOut& to,
                                        unsigned long long* __restrict__ err, const WeightDev& W,
                                        const CUtensorMap* tmF, const CUtensorMap* tmG, float* sm) {
    constexpr int RW = rows_per_chunk(R, C);
    constexpr int M = 2 * R + 1, K = RW * M;
    constexpr int DVEC = (RW * C) % 4 == 0 ? 4 : ((RW * C) % 2 == 0 ? 2 : 1);
    using RL = Rec<R, C>;
    const int lane = threadIdx.x, wid = threadIdx.y, NW = blockDim.y;
    const int tid = wid * 32 + lane;
    const int tau = g.tau;
    const int B0 = blockIdx.x * to.step, J = blockIdx.y, img = blockIdx.z;
    const int j = J * NW + wid, y0 = j * RW, Y0 = J * NW * RW;
    const int nw = min(NW, g.P - J * NW);
    const int xa = tau * B0;
    const long long NLl = (long long)g.nb * g.batch;
    const long long L0 = (long long)img * g.nb + B0;
    // shared memory: [maps: warp x slot x lane x MAPP][mbarriers, 128 B][image rows][guidance rows]
    const int PF = kb_stage_pitch(tau, M, C), PG = kb_stage_pitch(tau, M, CG);
    float* mapw = sm + wid * 2 * 32 * RL::MAPP;
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(sm + NW * 2 * 32 * RL::MAPP);
    unsigned long long* mbar_w = mbar + 1 + wid;
    float* sF = sm + NW * 2 * 32 * RL::MAPP + 32;
    float* sG = sF + ((NW * RW * PF + 31) & ~31);
    const int xoF = (xa * C) & 3, xoG = (xa * CG) & 3;
    if (tid <= NW) mbar_init(mbar + tid, 1);
    __syncthreads();
    if (tid == 0) {
        mbar_arrive_expect_tx(mbar, (unsigned)((NW * RW * PF + (NW * RW + 1) * PG) * sizeof(float)));
        tma_load_2d(sF, tmF, xa * C - xoF, img * g.Hl + Y0, mbar);
        tma_load_2d(sG, tmG, xa * CG - xoG, img * g.Hl + Y0 - 1, mbar);
    }
    if (wid >= nw) return;  // chunk rows past the image: nothing else synchronises the CTA
    const int JA = to.nwa_shift >= 0 ? j >> to.nwa_shift : j / to.nwa, sj = j - JA * to.nwa;
    const bool lastc = j == g.P - 1, has_left = j > 0;
    const bool r_inner = !lastc && sj < to.nwa - 1, l_inner = sj > 0;
    auto fetch_maps = [&]() {
        if (lane == 0 && (l_inner || r_inner)) {
            const unsigned by = (unsigned)(32 * RL::MAPP * sizeof(float));
            const float* gp0 = maps + ((long long)j * NLl + L0) * RL::MAPP;
            mbar_arrive_expect_tx(mbar_w, by * ((l_inner ? 1 : 0) + (r_inner ? 1 : 0)));
            if (l_inner) bulk_g2s(mapw, gp0 - NLl * RL::MAPP, by, mbar_w);
            if (r_inner) bulk_g2s(mapw + 32 * RL::MAPP, gp0, by, mbar_w);
        }
    };
    if (to.early) fetch_maps();
    const int nrows = min(RW, g.Hl - y0);
    ChunkInL<R, C, CG, RW> in;
    mbar_wait(mbar, 0);
    {
        const float* sFr = sF + (y0 - Y0) * PF + xoF + tau * lane * C;
        const float* sGr = sG + (y0 - Y0 + 1) * PG + xoG + tau * lane * CG;
        if (nrows == RW)
            load_chunk_lazy_staged<R, C, CG, RW, true>(in, sFr, PF, sGr, PG, g, y0, nrows);
        else
            load_chunk_lazy_staged<R, C, CG, RW, false>(in, sFr, PF, sGr, PG, g, y0, nrows);
    }
    const long long L = L0 + lane;
    if (err != nullptr) {  // NaN guidance: the reference's pivot failure (rare path locates it)
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int c = 0; c < CG; ++c) acc = fmaf(in.gp[k][c], 0.f, acc);
#pragma unroll
        for (int i = 0; i < R; ++i)
#pragma unroll
            for (int c = 0; c < CG; ++c) acc = fmaf(in.gprev[i][c], 0.f, acc);
        if (!(acc >= 0.f)) {
            const LazyWeights<R, C, CG, RW, 1> we{in, W};
            const LazyWeights<R, C, CG, RW, 0> wf{in, W};
            int bad = 0x7fffffff;
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int t = 1; t <= R; ++t) {
                    const float lw = W.kind == 1 ? we(k, t) : wf(k, t);
                    const bool exists = (k / M < nrows) && (k - t >= 0 || y0 > 0);
                    bad = (!(lw >= 0.f) && exists) ? min(bad, (g.row0 + y0) * M + k - t) : bad;
                }
            if (bad != 0x7fffffff) atomicMin(err, ((unsigned long long)(unsigned)L << 32) | (unsigned)bad);
        }
    }
    pdl_wait();  // super-separators (K2), maps (KA)
    pdl_trigger();
    if (!to.early) fetch_maps();
    float zl[R][C], zr[R][C];
    {
        const bool hA = JA > 0, hB = JA < to.psa - 1;
        const float* zb = zsep + (long long)JA * R * C * NLl + L;
        float zA[R][C], zB[R][C];
#pragma unroll
        for (int q = 0; q < R; ++q)
#pragma unroll
            for (int c = 0; c < C; ++c) {
                zA[q][c] = hA ? zb[((long long)(q - R) * C + c) * NLl] : 0.f;
                zB[q][c] = hB ? zb[(q * C + c) * NLl] : 0.f;
                zl[q][c] = has_left ? zA[q][c] : 0.f;
                zr[q][c] = lastc ? 0.f : zB[q][c];
            }
        if (l_inner || r_inner) mbar_wait(mbar_w, 0);
        if (r_inner) apply_map<R, C>(mapw + (32 + lane) * RL::MAPP, zA, zB, zr);
        if (l_inner) apply_map<R, C>(mapw + lane * RL::MAPP, zA, zB, zl);
    }
    const int kv = nrows * M;
    const int kend = lastc ? kv : kv - R;
    float cs[K][R], ys[K][C];
#pragma unroll
    for (int p = 0; p < K; ++p) {
#pragma unroll
        for (int i = 0; i < R; ++i) cs[p][i] = 0.f;
#pragma unroll
        for (int c = 0; c < C; ++c) ys[p][c] = 0.f;
    }
    auto solve = [&](const auto& lwf) {
        if (!lastc && kv == K)
            chunk_interior_solve<R, C, CG, RW, true>(in, lwf, has_left, lastc, kv, kend, zl, zr, cs, ys);
        else
            chunk_interior_solve<R, C, CG, RW, false>(in, lwf, has_left, lastc, kv, kend, zl, zr, cs, ys);
    };
    if (W.kind == 1)
        solve(LazyWeights<R, C, CG, RW, 1>{in, W});
    else
        solve(LazyWeights<R, C, CG, RW, 0>{in, W});
    float* obase = to.out + img * g.img_stride + ((long long)xa * g.Hl + y0) * C;
    const long long opitch = (long long)g.Hl * C;
    const int own0 = 32 - to.step, par0 = y0 & 1;
    switch (tau) {
        case 1: average_shfl_direct<1, R, C, K, DVEC, true>(ys, nrows, par0, lane, obase, opitch, 0, nullptr, own0); break;
        case 2: average_shfl_direct<2, R, C, K, DVEC, true>(ys, nrows, par0, lane, obase, opitch, 0, nullptr, own0); break;
        default: average_shfl_direct<3, R, C, K, DVEC, true>(ys, nrows, par0, lane, obase, opitch, 0, nullptr, own0); break;
    }
}

template <int R, int C, int CG>
__global__ void SGWLS_KB_BOUNDS kb_tile(const PassGeom g, const float* __restrict__ src,
                                               const float* __restrict__ guid, const float* __restrict__ zsep,
                                               const float* __restrict__ maps, const TileOut to,
                                               unsigned long long* __restrict__ err,
                                               const __grid_constant__ WeightDev W,
                                               const __grid_constant__ CUtensorMap tmF,
                                               const __grid_constant__ CUtensorMap tmG) {
    constexpr int RW = rows_per_chunk(R, C);
    constexpr int M = 2 * R + 1, K = RW * M;
    extern __shared__ __align__(128) float sm[];
    if constexpr (kb_has_lean(R, C)) {
        if ((int)blockIdx.x >= to.lean_lo && (int)blockIdx.x < to.lean_hi) {  // interior band tiles of a lean launch
            kb_lean<R, C, CG>(g, zsep, maps, to, err, W, &tmF, &tmG, sm);
            return;
        }
    }
    const int lane = threadIdx.x, wid = threadIdx.y, NW = blockDim.y;
    const int tid = wid * 32 + lane, NT = NW * 32;
    // grid: (band tile, chunk tile, image)
    const int bxi = blockIdx.x;
    const int B0 = bxi * to.step;
    const int b = B0 + lane;
    const int J = blockIdx.y;
    const int img = blockIdx.z;
    const int j = J * NW + wid;
    const int nw = min(NW, g.P - J * NW);
    const bool active = (b < g.nb) && (wid < nw);
    const int L = img * g.nb + b;
    const long long NLl = (long long)g.nb * g.batch;
    const float lam = W.lam;
    const int Y0 = J * NW * RW;
    const int TR = min(NW * RW, g.Hl - Y0);  // tile rows

    using RL = Rec<R, C>;
    // shared memory: [separator-map staging: warp x slot x lane x MAPP][output tile][1/count per column]
    float* mapsm = sm + (wid * 2 * 32 + lane) * RL::MAPP;
    // staged input rows: [mbarrier, 16 B][image rows NW*RW x PF][guidance rows (1 + NW*RW) x PG]
    const bool stage = (R >= SGWLS_LAZY_MIN_R) && to.stage != 0;
    const int PF = stage ? kb_stage_pitch(g.tau, M, C) : 0, PG = stage ? kb_stage_pitch(g.tau, M, CG) : 0;
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(sm + NW * 2 * 32 * RL::MAPP);
    float* sF = sm + NW * 2 * 32 * RL::MAPP + 32;
    float* sG = sF + ((NW * RW * PF + 31) & ~31);
    float* tl = stage ? sG + (((NW * RW + 1) * PG + 31) & ~31)
                      : sm + NW * 2 * 32 * RL::MAPP;  // output tile [x][y*C + c] or [y][x*C + c]
    const int bl = min(B0 + 32, g.nb) - 1;
    // interior tile: bands B0 - KMAX .. B0 + 31 are all regular (centres r + tau*b), neither
    // image edge nor the forced last centre reaches its columns
    const bool interior = bxi > 0 && B0 + 32 < g.nb && B0 + 32 <= g.nreg &&
                          (B0 + 32) * g.tau <= g.Wl - 1 - 2 * g.r;
    const int xa = interior ? g.tau * B0 : band_lo(g, B0);
    const int xb = (interior ? g.tau * bl : band_lo(g, bl)) + M - 1;
    const int ncol = xb - xa + 1;
    // Output tile layout.  Column-major [x][y*C + c] (pitch TP, 16-byte rows)
    // when every owned column leaves as one bulk copy; otherwise row-major
    // [y][x*C + c] with an odd pitch XP, so that the 32 bands of a warp
    // (columns tau apart) hit distinct banks when they accumulate.
    float* oi = to.out + img * g.img_stride;
    const int n = TR * C;
    const bool vec = ((g.Hl * C) % 4 == 0) && ((Y0 * C) % 4 == 0) && (n % 4 == 0) &&
                     ((reinterpret_cast<uintptr_t>(oi) & 15) == 0);
    // Column-major accumulation is 4-way bank-conflicted for odd tau (pitch = 4
    // mod 8) and 8-way for even tau; row-major with an odd pitch is conflict-free
    // (odd tau) or 2-way (even tau) for one channel, and its columns still leave
    // as float4 stores (4 gathered rows).  Bulk copies need column-major.
    const bool colmaj = to.transpose_out && vec && (n >= 64 || C > 1);
    const int TP = ((n + 3) & ~3) + ((((n + 3) & ~3) % 8 == 0) ? 4 : 8);
    const int XP = (ncol * C) | 1;
    const int sx = colmaj ? TP : C, sy = colmaj ? C : XP;  // tile strides of x and y
    const int tsize = colmaj ? ncol * TP : TR * XP;

    // ---- 0b. staged input: two tensor-map boxes per CTA, the tile's image rows and its guidance
    //          rows from Y0 - 1 (the rows of the pass input are complete before KA began, so this
    //          precedes the dependent-launch wait).  A box's first element must sit on a 16-byte
    //          boundary: it starts up to 3 floats before column xa (the pitch has that slack) and
    //          xoF / xoG skip them; the offset is the same for every row ((Wl*C) % 4 == 0).
    int xoF = 0, xoG = 0;
    if (stage) {
        xoF = (xa * C) & 3;
        xoG = (xa * CG) & 3;
        if (tid <= NW) mbar_init(mbar + tid, 1);  // [0]: the tile's rows; [1 + w]: warp w's separator maps
        __syncthreads();
        if (tid == 0) {
            mbar_arrive_expect_tx(mbar, (unsigned)((NW * RW * PF + (NW * RW + 1) * PG) * sizeof(float)));
            tma_load_2d(sF, &tmF, xa * C - xoF, img * g.Hl + Y0, mbar);
            tma_load_2d(sG, &tmG, xa * CG - xoG, img * g.Hl + Y0 - 1, mbar);
        }
    }
    // ---- 1. chunk inputs and edge weights before the dependent-launch wait:
    //         the pass input was complete before KA began
    std::conditional_t<(R >= SGWLS_LAZY_MIN_R), ChunkInL<R, C, CG, RW>, ChunkIn<R, C, CG, RW>> in;
    const int y0 = j * RW;
    const int nrows = active ? min(RW, g.Hl - y0) : 0;
    const int lo = active ? (interior ? g.tau * b : band_lo(g, b)) : 0;
    const bool multi = g.P > 1 || g.has_prev || g.has_next;  // separators exist
    // ---- 0. tile geometry (column ownership, 1/count, zeroing): independent of the
    //         predecessor, so it runs before the dependent-launch wait
    // Shuffle averaging (average_shfl) when the bands overlap, all bands of the
    // tile are on the tau grid, tau <= 3, and the last owned column has a writer lane
    const bool last_cta = B0 + 32 >= g.nb;
    const bool shfl_avg = to.nph > 1 && g.tau <= 3 && bl < g.nreg &&
                          (!last_cta || (bl - B0) + div_tau(g, M - 1) <= 31);
    // direct stores to the transposed output (no tile round trip) when the
    // vector width divides the output rows
    constexpr int DVEC = (RW * C) % 4 == 0 ? 4 : ((RW * C) % 2 == 0 ? 2 : 1);
#ifndef SGWLS_NO_DIRECT
    // measured on B200: c1 +8.5 %, c3 +1.8 %, c5 +0.6 %; c4 (2 channels, float2 runs) -4.7 % (+0.5 %
    // once its rows were TMA-staged: still not worth a second code path), so only for one channel
    // or full float4 runs
    const bool direct = shfl_avg && !to.ratio && to.transpose_out && (C == 1 || DVEC == 4) &&
                        ((long long)g.Hl * C) % DVEC == 0 &&
                        (reinterpret_cast<uintptr_t>(oi) & (DVEC * 4 - 1)) == 0;
#else
    const bool direct = false;
#endif
    // interior tiles that store directly need no column table (compile-time counts, lane ownership)
    const bool lean = direct && interior;
    // per-column averaging scale 1/count, positive if this CTA owns the column
    // (writes it out), negative otherwise
    float* inv_col = tl + ((tsize + 3) & ~3);
    for (int xl = tid; xl < (lean ? 0 : ncol); xl += NT) {
        int bmin, bmax;
        covering(g, xa + xl, bmin, bmax);
        // owner CTA = ceil((bmax - 31) / step) (0 if bmax <= 31), tested without a division
        const int bx = bxi, q = bmax - 31;
        const bool owned = bx == 0 ? q <= 0 : (q > (bx - 1) * to.step && q <= bx * to.step);
        const float inv = kInvCount[bmax - bmin + 1];  // == 1.0f / count, without the IEEE-division slow path
        inv_col[xl] = owned ? inv : -inv;
        if (to.nph == 2 && !shfl_avg) {
            // phase 0 STORES (step 4), so only the columns no phase-0 band of this
            // tile covers start from zero (measured: c5 +1.2 %, c4 +0.7 %; with
            // more phases the sparse phase-0 coverage makes it a loss, c3 -6 %)
            bool cov0 = false;
            for (int bb = bmin; bb <= bmax; ++bb) {
                const int l = bb - B0;
                cov0 = cov0 || (l >= 0 && l < 32 && bb < g.nb && (l % to.nph) == 0);
            }
            if (!cov0)
                for (int y = 0; y < TR; ++y)
#pragma unroll
                    for (int c = 0; c < C; ++c) tl[xl * sx + y * sy + c] = 0.f;
        }
    }
    const bool store_first = to.nph == 2;
    if (to.nph > 1 && !store_first && !shfl_avg) {
        for (int i = tid; i < (tsize + 3) / 4; i += NT) reinterpret_cast<float4*>(tl)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // this chunk's separator maps -> shared memory (per warp: slot 0 = sigma_{j-1},
    // slot 1 = sigma_j; [slot][lane][MAPP], 16-byte aligned), asynchronously; before
    // the wait when KA is not the predecessor
    const int JA = to.nwa_shift >= 0 ? j >> to.nwa_shift : j / to.nwa, sj = j - JA * to.nwa;
    const bool lastc = (j == g.P - 1) && !g.has_next;
    const bool has_left = j > 0 || g.has_prev;
    const bool r_inner = !lastc && sj < to.nwa - 1 && j < g.P - 1;  // sigma_j inner in KA tile JA
    const bool l_inner = sj > 0;  // sigma_{j-1} inner in the same KA tile
    // staged mode: the warp's 32 maps of a separator are one contiguous run
    // ([chunk][line][MAPP]), moved by ONE bulk copy per slot onto the warp's own mbarrier
    unsigned long long* mbar_w = mbar + 1 + wid;
    auto fetch_maps = [&]() {
        if (stage) {
            if (lane == 0 && wid < nw && multi && (l_inner || r_inner)) {
                const long long L0 = (long long)img * g.nb + B0;
                const int nl = (int)min((long long)32, NLl - L0);
                const unsigned by = (unsigned)(nl * RL::MAPP * sizeof(float));
                const float* gp0 = maps + ((long long)j * NLl + L0) * RL::MAPP;
                float* dst = sm + wid * 2 * 32 * RL::MAPP;
                mbar_arrive_expect_tx(mbar_w, by * ((l_inner ? 1 : 0) + (r_inner ? 1 : 0)));
                if (l_inner) bulk_g2s(dst, gp0 - NLl * RL::MAPP, by, mbar_w);
                if (r_inner) bulk_g2s(dst + 32 * RL::MAPP, gp0, by, mbar_w);
            }
            return;
        }
        if (!(active && multi)) return;
        const float* gp = maps + ((long long)j * NLl + L) * RL::MAPP;
        if (l_inner) {
            const float* gl = gp - NLl * RL::MAPP;
#pragma unroll
            for (int f = 0; f < RL::MAPP; f += 4) cp_async16(mapsm + f, gl + f);
        }
        if (r_inner) {
#pragma unroll
            for (int f = 0; f < RL::MAPP; f += 4) cp_async16(mapsm + 32 * RL::MAPP + f, gp + f);
        }
        cp_async_commit();
    };
    if (to.early) fetch_maps();
    if constexpr (R >= SGWLS_LAZY_MIN_R) {
    if (stage) mbar_wait(mbar, 0);  // every thread: the staged rows have landed
    if (active) {
        if (stage) {
            const float* sFr = sF + (y0 - Y0) * PF + xoF + (lo - xa) * C;
            const float* sGr = sG + (y0 - Y0 + 1) * PG + xoG + (lo - xa) * CG;
            if (nrows == RW)
                load_chunk_lazy_staged<R, C, CG, RW, true>(in, sFr, PF, sGr, PG, g, y0, nrows);
            else
                load_chunk_lazy_staged<R, C, CG, RW, false>(in, sFr, PF, sGr, PG, g, y0, nrows);
        } else {
        const long long npx = (long long)g.Hl * g.Wl;
        const float* Msk = (C > 1 && g.msk != nullptr) ? g.msk + img * npx : nullptr;
        const float* F = src + img * (Msk ? npx * (C > 1 ? C - 1 : 1) : g.img_stride);
        if (nrows == RW)
            load_chunk_lazy<R, C, CG, RW, true>(in, F, Msk, guid + img * g.gimg_stride, g, lo, y0, nrows);
        else
            load_chunk_lazy<R, C, CG, RW, false>(in, F, Msk, guid + img * g.gimg_stride, g, lo, y0, nrows);
        }
        if (err != nullptr) {  // NaN guidance: the reference's pivot failure (rare path locates it)
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int c = 0; c < CG; ++c) acc = fmaf(in.gp[k][c], 0.f, acc);
#pragma unroll
            for (int i = 0; i < R; ++i)
#pragma unroll
                for (int c = 0; c < CG; ++c) acc = fmaf(in.gprev[i][c], 0.f, acc);
            if (!(acc >= 0.f)) {
                const LazyWeights<R, C, CG, RW, 1> we{in, W};
                const LazyWeights<R, C, CG, RW, 0> wf{in, W};
                int bad = 0x7fffffff;
#pragma unroll
                for (int k = 0; k < K; ++k)
#pragma unroll
                    for (int t = 1; t <= R; ++t) {
                        const float lw = W.kind == 1 ? we(k, t) : wf(k, t);
                        const bool exists = (k / M < nrows) && (k - t >= 0 || y0 > 0 || g.has_prev);
                        bad = (!(lw >= 0.f) && exists) ? min(bad, (g.row0 + y0) * M + k - t) : bad;
                    }
                if (bad != 0x7fffffff) atomicMin(err, ((unsigned long long)(unsigned)L << 32) | (unsigned)bad);
            }
        }
    }
    } else {
    if (active)
        load_chunk<R, C, CG, RW>(in, src, guid + img * g.gimg_stride, g, W, lo, y0, nrows, err, L, img);
    }
    pdl_wait();  // super-separators (K2), maps (KA)
    pdl_trigger();
    if (!to.early) fetch_maps();

    // ---- 2. this chunk's two separators: the KA tile's super-separators zA
    //         (left, zsep[JA-1]) and zB (right, zsep[JA]) from K2, the maps
    float zl[R][C], zr[R][C];
#pragma unroll
    for (int q = 0; q < R; ++q)
#pragma unroll
        for (int c = 0; c < C; ++c) {
            zl[q][c] = 0.f;
            zr[q][c] = 0.f;
        }
    if (active && multi) {
        const bool hA = JA > 0 || g.has_prev, hB = JA < to.psa - 1 || g.has_next;
        const float* zb = zsep + (long long)JA * R * C * NLl + L;
        float zA[R][C], zB[R][C];
#pragma unroll
        for (int q = 0; q < R; ++q)
#pragma unroll
            for (int c = 0; c < C; ++c) {
                zA[q][c] = hA ? zb[((long long)(q - R) * C + c) * NLl] : 0.f;
                zB[q][c] = hB ? zb[(q * C + c) * NLl] : 0.f;
            }
        if (stage) {
            if (l_inner || r_inner) mbar_wait(mbar_w, 0);
        } else {
            cp_async_wait_all();  // this lane's own map columns (no cross-lane reads: no warp barrier)
        }
        if (r_inner) {
            apply_map<R, C>(mapsm + 32 * RL::MAPP, zA, zB, zr);
        } else if (!lastc) {
#pragma unroll
            for (int q = 0; q < R; ++q)
#pragma unroll
                for (int c = 0; c < C; ++c) zr[q][c] = zB[q][c];
        }
        if (l_inner) {
            apply_map<R, C>(mapsm, zA, zB, zl);
        } else if (has_left) {
#pragma unroll
            for (int q = 0; q < R; ++q)
#pragma unroll
                for (int c = 0; c < C; ++c) zl[q][c] = zA[q][c];
        }
    }
    const int kv = nrows * M;
    const int kend = lastc ? kv : kv - R;  // interior positions [0, kend)

    // chunk factor state in registers: couplings cs[p][i] and y / u values ys[p][c]
    float cs[K][R], ys[K][C];
#pragma unroll
    for (int p = 0; p < K; ++p) {
#pragma unroll
        for (int i = 0; i < R; ++i) cs[p][i] = 0.f;
#pragma unroll
        for (int c = 0; c < C; ++c) ys[p][c] = 0.f;
    }
    if (active) {
        if constexpr (R >= SGWLS_LAZY_MIN_R) {
        auto solve = [&](const auto& lwf) {
            if (!lastc && kv == K)
                chunk_interior_solve<R, C, CG, RW, true>(in, lwf, has_left, lastc, kv, kend, zl, zr, cs, ys);
            else
                chunk_interior_solve<R, C, CG, RW, false>(in, lwf, has_left, lastc, kv, kend, zl, zr, cs, ys);
        };
        if (W.kind == 1)
            solve(LazyWeights<R, C, CG, RW, 1>{in, W});
        else
            solve(LazyWeights<R, C, CG, RW, 0>{in, W});
        } else {
        const EagerWeights<R, C, CG, RW> lwf{in};
        if (!lastc && kv == K)
            chunk_interior_solve<R, C, CG, RW, true>(in, lwf, has_left, lastc, kv, kend, zl, zr, cs, ys);
        else
            chunk_interior_solve<R, C, CG, RW, false>(in, lwf, has_left, lastc, kv, kend, zl, zr, cs, ys);
        }
    }
    const int par0 = y0 & 1;
    if (lean) {  // no shared table, no barrier: counts are compile-time, lanes >= 32 - step own their columns
        const int nrw = wid < nw ? min(RW, g.Hl - y0) : 0;
        float* obase = oi + ((long long)xa * g.Hl + y0) * C;
        const long long opitch = (long long)g.Hl * C;
        const int own0 = 32 - to.step;
        if (nrw > 0) {
            switch (g.tau) {
                case 1: average_shfl_direct<1, R, C, K, DVEC, true>(ys, nrw, par0, lane, obase, opitch, ncol, nullptr, own0); break;
                case 2: average_shfl_direct<2, R, C, K, DVEC, true>(ys, nrw, par0, lane, obase, opitch, ncol, nullptr, own0); break;
                default: average_shfl_direct<3, R, C, K, DVEC, true>(ys, nrw, par0, lane, obase, opitch, ncol, nullptr, own0); break;
            }
        }
        return;
    }
    __syncthreads();
    // ---- 4. averaging into the shared output tile, fixed phase order
    //         (nph == 1: no two bands overlap, every tile cell has one writer)
    //         Values enter the tile already divided by their column's count.
    float* tbase = tl + (lo - xa) * sx + (y0 - Y0) * sy;
    if (direct) {
        const int nrw = wid < nw ? min(RW, g.Hl - y0) : 0;
        float* obase = oi + ((long long)xa * g.Hl + y0) * C;
        const long long opitch = (long long)g.Hl * C;
        if (nrw > 0) {
            switch (g.tau) {
                case 1: average_shfl_direct<1, R, C, K, DVEC>(ys, nrw, par0, lane, obase, opitch, ncol, inv_col); break;
                case 2: average_shfl_direct<2, R, C, K, DVEC>(ys, nrw, par0, lane, obase, opitch, ncol, inv_col); break;
                default: average_shfl_direct<3, R, C, K, DVEC>(ys, nrw, par0, lane, obase, opitch, ncol, inv_col); break;
            }
        }
        return;
    }
    if (shfl_avg) {
        const int nrw = wid < nw ? min(RW, g.Hl - y0) : 0;  // rows of this warp's chunk (all lanes)
        float* trow = tl + (y0 - Y0) * sy;
        switch (g.tau) {
            case 1: average_shfl<1, R, C, K>(ys, nrw, par0, lane, trow, sx, sy, ncol, inv_col); break;
            case 2: average_shfl<2, R, C, K>(ys, nrw, par0, lane, trow, sx, sy, ncol, inv_col); break;
            default: average_shfl<3, R, C, K>(ys, nrw, par0, lane, trow, sx, sy, ncol, inv_col); break;
        }
        fence_proxy_async_shared();
        __syncthreads();
    }
    float csc[M];
#pragma unroll
    for (int jj = 0; jj < M; ++jj) csc[jj] = (active && !shfl_avg) ? fabsf(inv_col[lo - xa + jj]) : 0.f;
    for (int ph = 0; ph < (shfl_avg ? 0 : to.nph); ++ph) {
        if (active && (lane % to.nph) == ph) {
            const bool first = to.nph == 1 || (store_first && ph == 0);  // first writer of every cell it touches
            // column m of the band at tile column (lo - xa) + m: per-row stores at
            // compile-time offsets from M column bases; the serpentine reversal of
            // a row is applied to the values, not to the addresses
            float* tcol[M];
#pragma unroll
            for (int m = 0; m < M; ++m) tcol[m] = tbase + m * sx;
#pragma unroll
            for (int rr = 0; rr < RW; ++rr) {
                if (rr * M < kv) {
                    const bool rev = (par0 ^ (rr & 1)) != 0;
                    const int ro = rr * sy;
#pragma unroll
                    for (int m = 0; m < M; ++m) {
                        float* tp = tcol[m] + ro;
#pragma unroll
                        for (int c = 0; c < C; ++c) {
                            const float v = rev ? ys[rr * M + (M - 1 - m)][c] : ys[rr * M + m][c];
                            tp[c] = first ? v * csc[m] : fmaf(v, csc[m], tp[c]);
                        }
                    }
                }
            }
        }
        fence_proxy_async_shared();  // the tile is read by bulk copies (async proxy) below
        __syncthreads();
    }
    // ---- 5. owned columns -> global.  Transposed layout: each owned column is
    //         TR*C contiguous floats of the output.
    if (to.ratio) {  // fused Eq. 21 ratio with the reference floor, one thread per (column, row)
        constexpr int CV = C > 1 ? C - 1 : 1;
        const long long npx = (long long)g.Hl * g.Wl;
        float* ov = to.out + img * npx * CV;
        float* ou = to.und ? to.und + img * npx : nullptr;
        for (int idx = tid; idx < ncol * TR; idx += NT) {
            const int xl = idx / TR, y = idx - xl * TR;
            if (inv_col[xl] <= 0.f) continue;
            const float* tp = tl + xl * sx + y * sy;
            const float d = tp[C - 1];
            const bool undef = d < to.floor_;
            const long long px = to.transpose_out ? (long long)(xa + xl) * g.Hl + Y0 + y
                                                  : (long long)(Y0 + y) * g.Wl + xa + xl;
#pragma unroll
            for (int c = 0; c < CV; ++c) ov[px * CV + c] = undef ? 0.f : tp[c] / d;
            if (ou) ou[px] = undef ? 1.f : 0.f;
        }
    } else if (colmaj && n >= 64) {  // >= 256-byte runs: one bulk (TMA) shared->global copy per owned column
        bool issued = false;
        for (int xl = tid; xl < ncol; xl += NT) {
            if (inv_col[xl] > 0.f) {
                bulk_s2g(oi + ((long long)(xa + xl) * g.Hl + Y0) * C, tl + xl * TP, (unsigned)(n * 4));
                issued = true;
            }
        }
        if (issued) bulk_commit_and_wait_read();
    } else if (colmaj) {  // short runs, column-major tile: float4 slot e4 of columns c0, c0 + cps, ...
        const int nv = n >> 2;
        const int cps = nv <= NT ? NT / nv : 1;
        const int c0 = nv <= NT ? tid / nv : 0;
        const int e = tid - c0 * nv;
        if (c0 < cps && e < nv) {
            const long long ostep = (long long)cps * g.Hl * C;
            float* op = oi + ((long long)(xa + c0) * g.Hl + Y0) * C;
            const float* tp = tl + c0 * TP;
            for (int xl = c0; xl < ncol; xl += cps, op += ostep, tp += cps * TP) {
                if (inv_col[xl] <= 0.f) continue;
                for (int e4 = e; e4 < nv; e4 += NT)
                    reinterpret_cast<float4*>(op)[e4] = reinterpret_cast<const float4*>(tp)[e4];
            }
        }
    } else if (to.transpose_out && vec && C == 1) {
        // row-major tile, one channel: thread tid gathers 4 rows (slot e4) of
        // columns c0, c0 + cps, ... into one float4 store
        const int nv = n >> 2;
        const int cps = nv <= NT ? NT / nv : 1;
        const int c0 = nv <= NT ? tid / nv : 0;
        const int e4 = tid - c0 * nv;
        if (c0 < cps && e4 < nv) {
            const long long ostep = (long long)cps * g.Hl;
            float* op = oi + (long long)(xa + c0) * g.Hl + Y0;
            const float* tq = tl + 4 * e4 * XP;
            for (int xl = c0; xl < ncol; xl += cps, op += ostep) {
                if (inv_col[xl] <= 0.f) continue;
                reinterpret_cast<float4*>(op)[e4] =
                    make_float4(tq[xl], tq[XP + xl], tq[2 * XP + xl], tq[3 * XP + xl]);
            }
        }
    } else if (to.transpose_out) {
        // thread tid owns element e of columns c0, c0 + cps, ... (row-major tile)
        const int cps = n <= NT ? NT / n : 1;
        const int c0 = n <= NT ? tid / n : 0;
        const int e = tid - c0 * n;
        if (c0 < cps && e < n) {
            const long long ostep = (long long)cps * g.Hl * C;
            float* op = oi + ((long long)(xa + c0) * g.Hl + Y0) * C;
            for (int xl = c0; xl < ncol; xl += cps, op += ostep) {
                if (inv_col[xl] <= 0.f) continue;
                for (int e2 = e; e2 < n; e2 += NT) op[e2] = tl[(e2 / C) * XP + xl * C + e2 % C];
            }
        }
    } else {
        for (int yl = wid; yl < TR; yl += NW) {
            float* orow = oi + ((long long)(Y0 + yl) * g.Wl + xa) * C;
            for (int e2 = lane; e2 < ncol * C; e2 += 32) {
                const int xl = e2 / C;
                if (inv_col[xl] > 0.f) orow[e2] = tl[yl * XP + e2];
            }
        }
    }
}

// =========================================================== host helpers

template <int R, int C>
__host__ inline size_t kb_smem_bytes(int NW, int TR, int ncol, int stage_floats = 0) {
    const int n4 = (TR * C + 3) & ~3;
    const size_t tile = (size_t)ncol * (n4 + (n4 % 8 == 0 ? 4 : 8));
    return (((tile + 3) & ~(size_t)3) + ((ncol + 3) & ~3) + (size_t)NW * 2 * Rec<R, C>::MAPP * 32 + stage_floats) *
           sizeof(float);
}


// =========================================================== launchers

template <int R, int C, int CG>
inline cudaError_t launch_tile_rcg(const PassLaunch& pl, cudaStream_t st) {
    using RL = Rec<R, C>;
    const PassGeom& g = pl.geom;
    const int NL = g.nb * g.batch;
    const int NWA = pl.nwa;  // KA super-chunk (chunks per KA tile)
    const int NW = pl.nw;    // KB tile height (chunks)
    const int PSA = (g.P + NWA - 1) / NWA;
    const int PB = (g.P + NW - 1) / NW;
    cudaError_t e;
    const bool slab = pl.slab_phase != 0;
    const bool multi = g.P > 1 || slab;
    if (pl.slab_phase != 2 && multi) {  // KA (ordinary pass, or row-slab phase A)
        ProfScope ps("ka_tile", st);
        const size_t smem = ka_smem<R, C>(NWA);
        e = cudaFuncSetAttribute(ka_tile<R, C, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        // warps per KA CTA: NWA (one chunk each), or NWA/2 (two chunks each)
        // when that keeps as many warps resident per SM and the grid is several
        // waves deep -- fewer warps idle while warp 0 reduces the tile (c5: 4
        // warps x 2 chunks, KA -15 %; c4 / c3 / r = 1 keep one chunk per warp)
        static const int kaw_env = [] {
            const char* v = std::getenv("SGWLS_KA_CTA_WARPS");  // schedule knob: warps per KA CTA
            return v ? std::atoi(v) : 0;
        }();
        int kaw = NWA;
        if (kaw_env > 0) {
            kaw = kaw_env < NWA ? kaw_env : NWA;
        } else if (NWA % 2 == 0) {
            static int nsm = 0;
            if (!nsm) {
                int dev = 0;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            }
            int occ_full = 0, occ_half = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_full, ka_tile<R, C, CG>, 32 * NWA, smem);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_half, ka_tile<R, C, CG>, 16 * NWA, smem);
            const long long warps = (long long)((NL + 31) / 32) * PSA * NWA;
            if (occ_half * (NWA / 2) >= occ_full * NWA && warps >= 4LL * nsm * occ_full * NWA) kaw = NWA / 2;
        }
        e = launch_pdl(ka_tile<R, C, CG>, dim3((NL + 31) / 32, PSA), dim3(32, kaw), smem, st, g, pl.src, pl.guid,
                       pl.rec, pl.maps, *pl.w, NWA);
        if (e != cudaSuccess) return e;
    }
    if (pl.slab_phase == 1) {  // row-slab phase A: this slab's record
        ProfScope ps("k2_slab_reduce", st);
        const size_t sm2 = k2_slab_reduce_smem<R, C>(kSlabWarps);
        e = cudaFuncSetAttribute(k2_slab_reduce<R, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
        if (e != cudaSuccess) return e;
        e = launch_pdl(k2_slab_reduce<R, C>, dim3((NL + 31) / 32), dim3(32, kSlabWarps), sm2, st, g, PSA,
                       (const float*)pl.rec, pl.grec, pl.slabrec);
        if (e != cudaSuccess) return e;
        return cudaGetLastError();
    }
    if (pl.slab_phase == 2) {  // row-slab phase B: super-separators, then KB below
        ProfScope ps("k2_slab_solve", st);
        const size_t sm2 = k2_slab_solve_smem<R, C>(kSlabWarps);
        e = cudaFuncSetAttribute(k2_slab_solve<R, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
        if (e != cudaSuccess) return e;
        e = launch_pdl(k2_slab_solve<R, C>, dim3((NL + 31) / 32), dim3(32, kSlabWarps), sm2, st, g, PSA, pl.nslab,
                       pl.islab, (const float*)pl.slabrec, (const float*)pl.rec, (const float*)pl.grec, pl.zg, pl.bsg,
                       pl.rs, pl.z);
        if (e != cudaSuccess) return e;
    } else if (g.P > 1 && PSA > 1) {  // K2: the reduced system over the super-separators
        ProfScope ps("k2_tree", st);
        PassGeom gs = g;
        gs.P = PSA;
        static const int ng_env = [] {
            const char* v = std::getenv("SGWLS_K2_NG");  // schedule knob: warps (groups) of the K2 tree
            const int n = v ? std::atoi(v) : 0;
            return n == 4 || n == 8 || n == 16 || n == 32 ? n : 0;
        }();
        // measured on B200 (level 2 as a merge tree): 32 warps for the long
        // reduced systems of r <= 2 (c5, 256 super records: +4 %; c4, 86: K2 -8 %), 16 from 16 super
        // records on, 8 below (c1 +3 %)
        int NG = ng_env ? ng_env : (PSA >= 64 && R <= 2 ? 32 : (PSA >= 20 ? 16 : 8));
        if (R > 2 && NG > 16) NG = 16;  // 1024 threads hold only 64 registers
        while (NG > 4 && k2_tree_smem<R, C>(NG) > 200 * 1024) NG /= 2;
        // staging all the CTA's super-records in shared memory first (one latency)
        // was measured slower on the short systems of c1 / c2 (their groups hold
        // only 2-3 records): off; kept as an option of the kernel
        const bool staged = false;
        const size_t sm2 = k2_tree_smem<R, C>(NG, staged ? PSA : 0);
        auto kern = NG > 16 ? k2_tree<R, C, 1024> : k2_tree<R, C, 512>;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
        if (e != cudaSuccess) return e;
        e = launch_pdl(kern, dim3((NL + 31) / 32), dim3(32, NG), sm2, st, gs, (const float*)pl.rec, pl.rs, pl.z,
                       staged ? 1 : 0);
        if (e != cudaSuccess) return e;
    }
    {
        ProfScope ps("kb_tile", st);
        constexpr int RW = rows_per_chunk(R, C);
        const int ncol = 31 * g.tau + 2 * g.r + 1;
        // staged input rows (bulk copies): lazy-weight radii, packed input, no slab neighbours,
        // rows and bases on 16-byte bounds
        static const int stage_env = [] {
            const char* v = std::getenv("SGWLS_KB_STAGE");  // schedule knob: 0 = per-lane loads, 1 = tensor-map staging
            return v ? std::atoi(v) : -1;
        }();
        // default: tensor-map staging for r = 2 -- measured c5 +6.5 %, c4 +3.5 %; c3 (r = 3, 8-row
        // tiles) -1.9 %, so r >= 3 keeps the per-lane loads.  (One bulk copy per row segment instead
        // of two tensor-map boxes per CTA was 15 % SLOWER than no staging on c5: removed.)
        const int stage_sel = stage_env >= 0 ? stage_env : (R == 2 ? 1 : 0);
        const bool stage = stage_sel && R >= SGWLS_LAZY_MIN_R && !slab && g.msk == nullptr &&
                           ((long long)g.Wl * C) % 4 == 0 && ((long long)g.Wl * CG) % 4 == 0 &&
                           (reinterpret_cast<uintptr_t>(pl.src) & 15) == 0 &&
                           (reinterpret_cast<uintptr_t>(pl.guid) & 15) == 0;
        const int M = 2 * R + 1;
        const int PFh = kb_stage_pitch(g.tau, M, C), PGh = kb_stage_pitch(g.tau, M, CG);
        const int stage_floats = stage ? 32 + ((NW * RW * PFh + 31) & ~31) + (((NW * RW + 1) * PGh + 31) & ~31) : 0;
        const size_t smem = kb_smem_bytes<R, C>(NW, NW * RW, ncol, stage_floats);
        // mode 2: one tensor-map box per array and CTA instead of one bulk copy per row
        CUtensorMap tmF, tmG;
        std::memset(&tmF, 0, sizeof tmF);
        std::memset(&tmG, 0, sizeof tmG);
        // no tensor map (box side > 256, no driver entry point): per-lane loads
        const int stage_mode =
            (stage && encode_rows_map(&tmF, pl.src, (long long)g.Wl * C, (long long)g.batch * g.Hl, PFh, NW * RW) &&
             encode_rows_map(&tmG, pl.guid, (long long)g.Wl * CG, (long long)g.batch * g.Hl, PGh, NW * RW + 1))
                ? 1
                : 0;
        // KB's predecessor: k2_tree / k2_slab_solve (they wait for KA before
        // triggering) or, with a single KA tile per band, KA itself
        const bool early = slab || PSA > 1;
        const int nwa_shift = (NWA & (NWA - 1)) == 0 ? __builtin_ctz((unsigned)NWA) : -1;
        TileOut to{pl.out, pl.transpose_out, pl.step, pl.nph, NWA, PSA, early ? 1 : 0, nwa_shift, pl.ratio,
                   pl.ratio_floor, pl.und, stage_mode, 0, 0};
        {
            // lean launch: staged by tensor maps, overlapping bands averaged by shuffles and stored
            // directly (the conditions of kb_tile's `direct`, all launch-uniform here), several chunks
            static const int lean_env = [] {
                const char* v = std::getenv("SGWLS_KB_LEAN");  // schedule knob: 0 = general body everywhere
                return v ? std::atoi(v) : 1;
            }();
            constexpr int DV = (RW * C) % 4 == 0 ? 4 : ((RW * C) % 2 == 0 ? 2 : 1);
            const bool lean_ok = kb_has_lean(R, C) && lean_env && stage_mode != 0 && g.P > 1 && pl.nph > 1 && g.tau <= 3 &&
                                 !pl.ratio && pl.transpose_out && (C == 1 || DV == 4) &&
                                 ((long long)g.Hl * C) % DV == 0 && (g.img_stride % DV) == 0 &&
                                 (reinterpret_cast<uintptr_t>(pl.out) & (DV * 4 - 1)) == 0;
            if (lean_ok) {
                int lo_bx = -1, hi_bx = -1;
                for (int bx = 0; bx < pl.ncta; ++bx) {
                    const int B0 = bx * pl.step;
                    const bool interior = bx > 0 && B0 + 32 < g.nb && B0 + 32 <= g.nreg &&
                                          (long long)(B0 + 32) * g.tau <= g.Wl - 1 - 2 * g.r;
                    if (interior) {
                        if (lo_bx < 0) lo_bx = bx;
                        hi_bx = bx + 1;
                    } else if (lo_bx >= 0) {
                        break;
                    }
                }
                if (lo_bx >= 0) {
                    to.lean_lo = lo_bx;
                    to.lean_hi = hi_bx;
                }
            }
        }
        const dim3 kgrid(pl.ncta, PB, g.batch);
        e = cudaFuncSetAttribute(kb_tile<R, C, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = launch_pdl(kb_tile<R, C, CG>, kgrid, dim3(32, NW), smem, st, g, pl.src, pl.guid, (const float*)pl.z,
                       (const float*)pl.maps, to, pl.err, *pl.w, tmF, tmG);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

template <int R, int C>
inline cudaError_t launch_tile_rc(const PassLaunch& pl, cudaStream_t st) {
    return pl.geom.Cg == 1 ? launch_tile_rcg<R, C, 1>(pl, st) : launch_tile_rcg<R, C, 3>(pl, st);
}

template <int R>
cudaError_t launch_tile_r(const PassLaunch& pl, cudaStream_t st) {
    switch (pl.geom.C) {
        case 1: return launch_tile_rc<R, 1>(pl, st);
        case 2: return launch_tile_rc<R, 2>(pl, st);
        case 3: return launch_tile_rc<R, 3>(pl, st);
        case 4: return launch_tile_rc<R, 4>(pl, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace tile
}  // namespace sgwls_b200
