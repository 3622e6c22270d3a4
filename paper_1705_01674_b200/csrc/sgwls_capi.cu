// sgwls_capi.cu -- host runtime and C ABI (include/sgwls_b200.h).
//
// Mirrors the reference pipeline (proj/src/smoother.cpp:103-163): validate the
// configuration with the reference's error texts, then run T directional
// passes alternating from first_axis, each pass = K1..K4 of sgwls_kernels.cu.
// A column pass runs on the current layout; its output is written transposed
// so the next (row) pass is again a column pass on its own layout, and the
// last pass writes the caller's orientation.  All device memory is
// stream-ordered (cudaMallocAsync) so concurrent host callers on different
// streams are independent; results are deterministic (fixed summation order,
// no float atomics).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sgwls_b200.h"
#include "sgwls_kernels.h"
#include "sgwls_profile.h"

using namespace sgwls_b200;

namespace {

constexpr double kMaskFloor = 1e-8;   // proj/src/smoother.cpp:15
constexpr int kTargetChunkPositions = 48;

void put_err(char* err, size_t errlen, const std::string& msg) {
    if (err && errlen) {
        std::strncpy(err, msg.c_str(), errlen - 1);
        err[errlen - 1] = '\0';
    }
}

struct Fail {
    int code;
    std::string msg;
};

#define CK(call)                                                                             \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            throw Fail{SGWLS_B200_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                             " at " #call};                                  \
    } while (0)

// SmoothConfig::validate + WeightParams::validate, same order and texts
// (proj/src/smoother.cpp:103-111, proj/src/weights.cpp:7-12).
int validate_cfg(const sgwls_b200_config* c, std::string& msg) {
    if (!c) {
        msg = "sgwls_b200: null config";
        return SGWLS_B200_EINVAL;
    }
    if (!(c->lambda >= 0.0) || !std::isfinite(c->lambda)) {
        msg = "smooth: lambda must be finite and >= 0";
        return SGWLS_B200_EINVAL;
    }
    if (c->r < 1) {
        msg = "smooth: r must be >= 1";
        return SGWLS_B200_EINVAL;
    }
    if (c->tau < 1 || c->tau > 2 * c->r + 1) {
        msg = "smooth: tau must be in [1, 2r+1], got " + std::to_string(c->tau);
        return SGWLS_B200_EINVAL;
    }
    if (c->iterations < 1) {
        msg = "smooth: iterations must be >= 1";
        return SGWLS_B200_EINVAL;
    }
    if (c->threads < 1) {
        msg = "smooth: threads must be >= 1";
        return SGWLS_B200_EINVAL;
    }
    if (!(c->epsilon > 0.0)) {
        msg = "weights: epsilon must be > 0";
        return SGWLS_B200_EINVAL;
    }
    if (c->weight_kind == SGWLS_B200_WEIGHT_EXP && (!(c->sigma_s > 0.0) || !(c->sigma_r > 0.0))) {
        msg = "weights: sigma_s and sigma_r must be > 0 for exponential weights";
        return SGWLS_B200_EINVAL;
    }
    if (!(c->guidance_scale > 0.0)) {
        msg = "weights: guidance_scale must be > 0";
        return SGWLS_B200_EINVAL;
    }
    if (c->weight_kind != SGWLS_B200_WEIGHT_EXP && c->weight_kind != SGWLS_B200_WEIGHT_FRAC) {
        msg = "sgwls_b200: unknown weight kind";
        return SGWLS_B200_EINVAL;
    }
    if (c->first_axis != 0 && c->first_axis != 1) {
        msg = "sgwls_b200: unknown axis";
        return SGWLS_B200_EINVAL;
    }
    return SGWLS_B200_OK;
}

int check_shape(int batch, int width, int height, int channels, int gch, std::string& msg) {
    if (batch < 1 || width <= 0 || height <= 0 || channels <= 0) {
        msg = "smooth: empty target";
        return SGWLS_B200_EINVAL;
    }
    if (channels > 4 || gch < 1 || gch > kMaxCg) {
        msg = "sgwls_b200: channels must be in [1, 4]";
        return SGWLS_B200_EUNSUPPORTED;
    }
    return SGWLS_B200_OK;
}

// Spatial LUT and folded range constants, in double then rounded once
// (proj/src/weights.cpp:14-22, 40-71).
void build_weights(const sgwls_b200_config* c, WeightDev& w) {
    std::memset(&w, 0, sizeof w);
    w.kind = c->weight_kind;
    w.lam = (float)c->lambda;
    const double log2e = 1.4426950408889634;
    // clamped to the finite range: an exponent that overflows float must not
    // turn range = 0 (a flat guidance region) into 0 * -inf = NaN
    const double ek = -(c->guidance_scale * c->guidance_scale) * log2e / (2.0 * c->sigma_r * c->sigma_r);
    w.exp_k = ek < -3.4e38 ? -3.4e38f : (float)ek;
    w.frac_half = (float)(c->alpha_r * 0.5);
    w.frac_lg2s = (float)std::log2(c->guidance_scale * c->guidance_scale);
    w.eps = (float)c->epsilon;
    for (int d2 = 0; d2 < kLutMax; ++d2) {
        double s;
        if (c->weight_kind == SGWLS_B200_WEIGHT_EXP)
            s = std::exp(-d2 / (2.0 * c->sigma_s * c->sigma_s));
        else
            s = 1.0 / (std::pow(std::sqrt((double)d2), c->alpha_s) + c->epsilon);
        w.spat[d2] = (float)s;
        if (d2 < 32) {
            const double ls = c->lambda * s;
            w.lspat[d2] = (float)ls;
            w.lg2ls[d2] = ls > 0.0 ? (float)std::log2(ls) : -INFINITY;
        }
    }
}

struct AxisPlan {
    PassGeom g;
    int kmax;
    int bx;
    int fast, step, ncta, nw, nph, nwa = 8;
    size_t rec_n, rs_n, z_n, u_n, map_n = 0;
    int anyr = 0;      // r > kMaxR: the any-radius path (sgwls_anyr.cu)
    size_t anyr_n = 0; // its workspace
};



// Band geometry (proj/src/snake.cpp:7-19, 21-49) and chunking of one pass layout.
AxisPlan plan_axis(int Hl, int Wl, int C, int Cg, int r, int tau, int batch) {
    AxisPlan ap;
    PassGeom& g = ap.g;
    std::memset(&g, 0, sizeof g);
    g.Hl = Hl;
    g.Wl = Wl;
    g.C = C;
    g.Cg = Cg;
    g.r = r;
    g.tau = tau;
    g.tau_mul = tau_multiplier(tau);
    g.batch = batch;
    if (Wl < 2 * r + 1) {
        g.degenerate = 1;
        g.nb = 1;
        g.nreg = 0;
        g.m = Wl;  // clipped window [0, Wl-1]
    } else {
        const int last = Wl - 1 - r;
        g.nreg = (last - r) / tau + 1;
        const int lastreg = r + tau * (g.nreg - 1);
        g.nb = g.nreg + (lastreg != last ? 1 : 0);
        g.m = 2 * r + 1;
    }
    g.n = (long long)g.m * Hl;
    g.img_stride = (long long)Hl * Wl * C;
    g.gimg_stride = (long long)Hl * Wl * Cg;
    const long long NL = (long long)g.nb * batch;
    static const int force_generic = [] {
        const char* v = std::getenv("SGWLS_FORCE_GENERIC");  // debugging knob: bypass the tiled path
        return v ? std::atoi(v) : 0;
    }();
    static const int tile_warps_env = [] {
        const char* v = std::getenv("SGWLS_TILE_WARPS");  // tuning knob: chunks per CTA tile
        const int n = v ? std::atoi(v) : 0;
        return n < 0 ? 0 : (n > 8 ? 8 : n);
    }();
    // measured on B200: 8-chunk KB tiles for r = 1 with several channels, 4-chunk tiles otherwise
    const int tile_warps = tile_warps_env ? tile_warps_env : ((r == 1 && C >= 2) ? kTileWarps : kTileWarps / 2);
    ap.fast = (!force_generic && !g.degenerate && r <= kTileMaxR && (Cg == 1 || Cg == 3)) ? 1 : 0;
    ap.step = 32;
    ap.ncta = 1;
    ap.nw = tile_warps;
    ap.nph = 1;
    ap.bx = 128;
    if (ap.fast) {
        // CTA-tiled path (sgwls_tile.cuh): chunks of RW rows, tiles of nw chunks x 32 bands
        const int RW = tile_rows_per_chunk(r, C);
        const int P = (Hl + RW - 1) / RW;
        g.P = P;
        ap.kmax = RW * g.m;
        static const int ka_warps_env = [] {
            const char* v = std::getenv("SGWLS_KA_WARPS");  // tuning knob: chunks per KA tile
            const int n = v ? std::atoi(v) : 0;
            return n < 0 ? 0 : (n > 8 ? 8 : n);
        }();
        // KA tiles (separator maps) and KB tiles are independent; measured
        // schedule of round 1 kept: r >= 2: 8-chunk KA tiles for one channel,
        // 4 with several right-hand sides; r = 1: as the KB tiles
        ap.nwa = ka_warps_env ? ka_warps_env : (r == 1 ? ap.nw : (C >= 2 ? kTileWarps / 2 : kTileWarps));
        const int PS = (P + ap.nwa - 1) / ap.nwa;
        // halo: widest span of bands covering one column (incl. the forced last centre)
        int hspan = 0;
        for (int x = 0; x < Wl; ++x) {
            int b0 = x - 2 * r <= 0 ? 0 : (x - 2 * r + tau - 1) / tau;
            int b1 = x / tau;
            if (b1 > g.nreg - 1) b1 = g.nreg - 1;
            int bmin = b0, bmax = b1;
            if (g.nb > g.nreg && x >= Wl - 1 - 2 * r) {
                if (b1 < b0) bmin = g.nreg;
                bmax = g.nreg;
            }
            if (bmax - bmin > hspan) hspan = bmax - bmin;
        }
        ap.step = 32 - hspan;
        ap.ncta = g.nb > 32 ? 1 + (g.nb - 32 + ap.step - 1) / ap.step : 1;
        // phases: bands of one phase must have disjoint windows
        int nph = 1;
        for (;; ++nph) {
            bool ok = true;
            for (int b = 0; b + nph < g.nb && ok; ++b)
                if (band_center(g, b + nph) - band_center(g, b) < g.m) ok = false;
            if (ok) break;
        }
        ap.nph = nph;
        ap.rec_n = P > 1 ? (size_t)PS * rec_floats(r, C) * NL : 0;
        ap.map_n = P > 1 ? (size_t)P * map_floats(r, C) * NL : 0;
        // K2 back-substitution rows with their spike column (level 1 keeps them for level 3)
        ap.rs_n = PS > 1 ? (size_t)PS * r * (rs_floats(r, C) + r) * NL : 0;
        ap.z_n = PS > 1 ? (size_t)(PS - 1) * r * C * NL : 0;
        ap.u_n = 0;
        return ap;
    }
    if (r > kMaxR) {  // beyond the templated kernels: one thread per band, whole band, runtime r
        ap.anyr = 1;
        g.P = 1;
        ap.kmax = 0;
        ap.rec_n = ap.rs_n = ap.z_n = 0;
        ap.u_n = (size_t)batch * Hl * g.nb * g.m * C;
        ap.anyr_n = anyr_ws_floats(g);
        return ap;
    }
    static const int target_pos = [] {
        const char* v = std::getenv("SGWLS_CHUNK_POS");  // tuning knob (positions per chunk)
        return v ? std::atoi(v) : kTargetChunkPositions;
    }();
    int rows = target_pos / g.m;
    if (rows < 1) rows = 1;
    const int need = (2 * r + 1 + g.m - 1) / g.m;  // chunk must hold >= 2r+1 positions
    if (rows < need) rows = need;
    int P = (Hl + rows - 1) / rows;
    while (P > 1 && (long long)(Hl / P) * g.m < 2 * r + 1) --P;
    if (P < 1) P = 1;
    g.P = P;
    ap.kmax = ((Hl + P - 1) / P) * g.m;
    while (ap.bx > 32 && (size_t)ap.bx * ap.kmax * (r + C) * 4 > 200 * 1024) ap.bx /= 2;
    ap.rec_n = P > 1 ? (size_t)P * rec_floats(r, C) * NL : 0;
    ap.rs_n = P > 1 ? (size_t)(P - 1) * r * rs_floats(r, C) * NL : 0;
    ap.z_n = P > 1 ? (size_t)(P - 1) * r * C * NL : 0;
    ap.u_n = (size_t)batch * Hl * g.nb * g.m * C;
    return ap;
}

int kernels_per_pass(const AxisPlan& ap) {
    if (ap.fast) {
        const int PS = (ap.g.P + ap.nwa - 1) / ap.nwa;
        // ka_tile [+ k2_tree] when the lines have several chunks; kb_tile
        return (ap.g.P > 1 ? (1 + (PS > 1 ? 1 : 0)) : 0) + 1;
    }
    if (ap.anyr) return 2;  // k_band_anyr + k4_average
    return (ap.g.P > 1 ? 2 : 0) + 2;
}

struct DevBuf {
    float* p = nullptr;
    cudaStream_t st = nullptr;
    void alloc(size_t nfloats, cudaStream_t s) {
        st = s;
        if (nfloats) CK(cudaMallocAsync((void**)&p, nfloats * sizeof(float), s));
    }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
};

void init_pool_once() {
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return;
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            unsigned long long thr = ULLONG_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
}

void require_device() {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw Fail{SGWLS_B200_ECUDA, "sgwls_b200: no CUDA device available (there is no CPU fallback)"};
    init_pool_once();
}

// The T-pass pipeline on device buffers (proj/src/smoother.cpp:113-125).
// Returns after enqueueing; *d_err receives the first-pass NaN-weight report.
// pass_only: exactly one Column-axis pass (proj/src/smoother.cpp:51-99) whose
// output is written in the transposed layout (the building block of the
// line-slab sharded filter, sharded.py).
// Sparse hooks (interpolate_sparse, proj/src/smoother.cpp:146-161): d_mask !=
// nullptr -> d_t holds C-1 value channels and the mask is channel C-1 (read
// split by the first pass); ratio -> d_out gets C-1 channels num/den and d_und
// the undefined mask, computed in the last pass's epilogue.  Both only where
// run_smooth_sparse_fusable() says the tiled path runs those passes.
struct SparseHooks {
    const float* d_mask = nullptr;
    bool ratio = false;
    float floor_ = 0.f;
    float* d_und = nullptr;
};

void run_smooth(const float* d_t, const float* d_g, int batch, int W, int H, int C, int Cg,
                const sgwls_b200_config* cfg, float* d_out, unsigned long long* d_err, cudaStream_t st,
                bool pass_only = false, const SparseHooks* sh = nullptr) {
    WeightDev wd;
    build_weights(cfg, wd);
    const int T = pass_only ? 1 : cfg->iterations;
    const int fa = pass_only ? 0 : cfg->first_axis;
    const bool need0 = (fa == 0) || T >= 2;
    const bool need1 = (fa == 1) || T >= 2;
    AxisPlan ap0 = plan_axis(H, W, C, Cg, cfg->r, cfg->tau, batch);  // column passes
    AxisPlan ap1 = plan_axis(W, H, C, Cg, cfg->r, cfg->tau, batch);  // row passes (transposed layout)
    auto mx = [](size_t a, size_t b) { return a > b ? a : b; };
    size_t rec_n = 0, rs_n = 0, z_n = 0, u_n = 0, map_n = 0;
    if (need0) {
        rec_n = mx(rec_n, ap0.rec_n);
        map_n = mx(map_n, ap0.map_n);
        rs_n = mx(rs_n, ap0.rs_n);
        z_n = mx(z_n, ap0.z_n);
        u_n = mx(u_n, ap0.u_n);
    }
    if (need1) {
        rec_n = mx(rec_n, ap1.rec_n);
        map_n = mx(map_n, ap1.map_n);
        rs_n = mx(rs_n, ap1.rs_n);
        z_n = mx(z_n, ap1.z_n);
        u_n = mx(u_n, ap1.u_n);
    }
    const size_t img_n = (size_t)batch * W * H * C;
    DevBuf rec, rs, z, U, bufA, bufB, gt, maps, anyws, anylut;
    if (ap0.anyr || ap1.anyr) {
        // any-radius path: workspace of the larger axis, lambda * spatial factor by squared distance
        anyws.alloc(mx(need0 ? ap0.anyr_n : 0, need1 ? ap1.anyr_n : 0), st);
        // (filled on the device: stream-ordered and safe inside a graph capture)
        anylut.alloc(anyr_lut_floats(cfg->r), st);
        CK(launch_anyr_lut(anylut.p, anyr_lut_floats(cfg->r), cfg->lambda, cfg->weight_kind == SGWLS_B200_WEIGHT_EXP,
                           cfg->sigma_s, cfg->alpha_s, cfg->epsilon, st));
    }
    maps.alloc(map_n, st);
    rec.alloc(rec_n, st);
    rs.alloc(rs_n, st);
    z.alloc(z_n, st);
    U.alloc(u_n, st);
    const int ninter = (T > 1 ? 1 : 0) + (T > 2 ? 1 : 0) + (fa == 1 ? 1 : 0);
    if (ninter >= 1) bufA.alloc(img_n, st);
    if (ninter >= 2) bufB.alloc(img_n, st);
    if (need1) {
        gt.alloc((size_t)batch * W * H * Cg, st);
        CK(launch_transpose(d_g, gt.p, H, W, Cg, batch, st));
    }
    const float* src = d_t;
    float* pingpong[2] = {bufA.p, bufB.p};
    int src_idx = -1;  // -1: caller's buffer, else pingpong index
    if (fa == 1) {
        CK(launch_transpose(d_t, pingpong[0], H, W, C, batch, st));
        src = pingpong[0];
        src_idx = 0;
    }
    for (int p = 0; p < T; ++p) {
        const int o = (fa + p) & 1;
        const AxisPlan& ap = o == 0 ? ap0 : ap1;
        PassLaunch pl;
        pl.geom = ap.g;
        pl.bx = ap.bx;
        pl.fast = ap.fast;
        pl.step = ap.step;
        pl.ncta = ap.ncta;
        pl.nw = ap.nw;
        pl.nwa = ap.nwa;

        pl.nph = ap.nph;
        pl.maps = maps.p;
        pl.src = src;
        pl.guid = o == 0 ? d_g : gt.p;
        const bool lastp = (p == T - 1);
        pl.transpose_out = (lastp && !pass_only) ? (o == 1) : 1;
        float* out = d_out;
        if (!lastp) {  // never overwrite the pass input
            const int out_idx = (src_idx == 0) ? 1 : 0;
            out = pingpong[out_idx];
            src_idx = out_idx;
        }
        pl.out = out;
        pl.kmax = ap.kmax;
        pl.rec = rec.p;
        pl.rs = rs.p;
        pl.z = z.p;
        pl.U = U.p;
        pl.err = (p == 0) ? d_err : nullptr;
        pl.w = &wd;
        pl.anyr = ap.anyr;
        pl.anyr_ws = anyws.p;
        pl.anyr_lspat = anylut.p;
        if (sh && p == 0 && sh->d_mask) pl.geom.msk = sh->d_mask;
        if (sh && lastp && sh->ratio) {
            pl.ratio = 1;
            pl.ratio_floor = sh->floor_;
            pl.und = sh->d_und;
        }
        CK(launch_pass(pl, st));
        src = out;
    }
}

// Can interpolate_sparse read values + mask unpacked in its first pass and
// fuse the ratio into its last (both passes on the tiled path, first pass on
// the caller's layout)?
void sparse_fusable(int batch, int W, int H, int C, int Cg, const sgwls_b200_config* cfg, bool& split, bool& ratio) {
    const int T = cfg->iterations, fa = cfg->first_axis;
    const AxisPlan ap0 = plan_axis(H, W, C, Cg, cfg->r, cfg->tau, batch);
    const AxisPlan ap1 = plan_axis(W, H, C, Cg, cfg->r, cfg->tau, batch);
    split = fa == 0 && ap0.fast;
    ratio = (((fa + T - 1) & 1) == 0 ? ap0 : ap1).fast;
}

// interpolate_sparse of a host batch through the host pipeline.  Field validation of every
// sub-batch is enqueued with it (no host synchronisation in flight); the statuses are read once
// at the end and the first failing pair in batch order decides the error, as the reference's
// per-call checks would (proj/src/smoother.cpp:129-144), before any pivot failure of that pair's
// sub-batch.  On an error the output buffers hold unspecified values.
void sparse_host_pipelined(const float* v, const float* m, const float* g, int batch, int sub, int width, int height,
                           int channels, int gch, const sgwls_b200_config* cfg, float* out, float* und);

std::string pivot_message(unsigned long long key) {
    const unsigned k0 = (unsigned)(key & 0xffffffffu);
    return "rband_lu_factorize: non-positive pivot at row " + std::to_string(k0) + " (input not SPD)";
}

struct ErrWord {
    unsigned long long* d = nullptr;
    cudaStream_t st;
    explicit ErrWord(cudaStream_t s) : st(s) {
        CK(cudaMallocAsync((void**)&d, 2 * sizeof(unsigned long long), s));
        CK(cudaMemsetAsync(d, 0xff, sizeof(unsigned long long), s));
        CK(cudaMemsetAsync(d + 1, 0, sizeof(unsigned long long), s));
    }
    ~ErrWord() {
        if (d) cudaFreeAsync(d, st);
    }
};

// Sparse validation in the reference's order (proj/src/smoother.cpp:129-144),
// every pair in one launch and one host synchronisation; the first failing
// pair (in batch order) decides the error, as the reference's per-call checks.
void validate_sparse(const float* d_v, const float* d_m, int batch, long long npx, int C, cudaStream_t st) {
    unsigned long long* status = nullptr;
    CK(cudaMallocAsync((void**)&status, 2 * (size_t)batch * sizeof(unsigned long long), st));
    std::vector<unsigned long long> h(2 * (size_t)batch);
    try {
        CK(cudaMemsetAsync(status, 0xff, (size_t)batch * sizeof(unsigned long long), st));
        CK(cudaMemsetAsync(status + batch, 0, (size_t)batch * sizeof(unsigned long long), st));
        CK(launch_validate_sparse(d_v, d_m, npx, C, batch, status, st));
        CK(cudaMemcpyAsync(h.data(), status, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int b = 0; b < batch; ++b) {
            if (h[b] != ULLONG_MAX) {
                // which violation? read that pixel's mask
                float mv = 0.f;
                CK(cudaMemcpy(&mv, d_m + (size_t)b * npx + h[b], sizeof(float), cudaMemcpyDeviceToHost));
                if (mv != 0.f && mv != 1.f) throw Fail{SGWLS_B200_EINVAL, "interpolate_sparse: mask must be 0/1"};
                throw Fail{SGWLS_B200_EINVAL, "interpolate_sparse: values nonzero outside mask"};
            }
            if (h[batch + b] == 0) throw Fail{SGWLS_B200_EINVAL, "interpolate_sparse: empty mask"};
        }
    } catch (...) {
        cudaFreeAsync(status, st);
        throw;
    }
    cudaFreeAsync(status, st);
}

void run_sparse(const float* d_v, const float* d_m, const float* d_g, int batch, int W, int H, int C, int Cg,
                const sgwls_b200_config* cfg, float* d_out, float* d_und, unsigned long long* d_err,
                cudaStream_t st) {
    const long long npx = (long long)batch * W * H;
    // num = smooth(values), den = smooth(mask) share every factorization: one
    // (C+1)-channel smooth (proj/src/smoother.cpp:146-147); on the tiled path the
    // first pass reads values and mask where they lie and the last pass writes
    // the ratio (proj/src/smoother.cpp:149-161) -- no pack / ratio kernels
    bool split = false, ratio = false;
    sparse_fusable(batch, W, H, C + 1, Cg, cfg, split, ratio);
    DevBuf packed, res;
    SparseHooks sh;
    if (split) {
        sh.d_mask = d_m;
    } else {
        packed.alloc((size_t)npx * (C + 1), st);
        CK(launch_pack_sparse(d_v, d_m, packed.p, npx, C, st));
    }
    if (ratio) {
        sh.ratio = true;
        sh.floor_ = (float)kMaskFloor;
        sh.d_und = d_und;
    } else {
        res.alloc((size_t)npx * (C + 1), st);
    }
    run_smooth(split ? d_v : packed.p, d_g, batch, W, H, C + 1, Cg, cfg, ratio ? d_out : res.p, d_err, st, false,
               &sh);
    if (!ratio) CK(launch_ratio(res.p, d_out, d_und, npx, C, (float)kMaskFloor, st));
}

void finish_sync(unsigned long long* d_err, cudaStream_t st) {
    unsigned long long h = ULLONG_MAX;
    CK(cudaMemcpyAsync(&h, d_err, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h != ULLONG_MAX) throw Fail{SGWLS_B200_EINVAL, pivot_message(h)};
}


// host buffers -> device -> T passes -> host, on the calling thread's stream
// Host-buffer batches run as a three-stage pipeline over sub-batches: the upload of
// sub-batch i+1, the filter of sub-batch i and the download of sub-batch i-1 proceed on
// three streams (PCIe is full duplex; from pinned buffers the copies are truly
// asynchronous), two buffer slots.  `upload(i0, n, slot, st)`, `compute(i0, n, slot, st)`,
// `download(i0, n, slot, st)` enqueue the stage of images [i0, i0 + n) on the given stream.
struct HostPipeline {
    cudaStream_t s_in = nullptr, s_cmp = nullptr, s_out = nullptr;
    std::vector<cudaEvent_t> ev;
    HostPipeline() {
        CK(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&s_cmp, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
    }
    ~HostPipeline() {
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
        if (s_in) cudaStreamDestroy(s_in);
        if (s_cmp) cudaStreamDestroy(s_cmp);
        if (s_out) cudaStreamDestroy(s_out);
    }
    cudaEvent_t event() {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ev.push_back(e);
        return e;
    }
    template <class U, class F, class D>
    void run(int batch, int sub, U&& upload, F&& compute, D&& download) {
        const int nsub = (batch + sub - 1) / sub;
        std::vector<cudaEvent_t> in_done(nsub), cmp_done(nsub), out_done(nsub);
        for (int i = 0; i < nsub; ++i) {
            const int i0 = i * sub, n = std::min(sub, batch - i0), slot = i & 1;
            in_done[i] = event();
            cmp_done[i] = event();
            out_done[i] = event();
            if (i >= 2) CK(cudaStreamWaitEvent(s_in, cmp_done[i - 2], 0));  // the slot's inputs were consumed
            upload(i0, n, slot, s_in);
            CK(cudaEventRecord(in_done[i], s_in));
            CK(cudaStreamWaitEvent(s_cmp, in_done[i], 0));
            if (i >= 2) CK(cudaStreamWaitEvent(s_cmp, out_done[i - 2], 0));  // the slot's outputs were read
            compute(i0, n, slot, s_cmp);
            CK(cudaEventRecord(cmp_done[i], s_cmp));
            CK(cudaStreamWaitEvent(s_out, cmp_done[i], 0));
            download(i0, n, slot, s_out);
            CK(cudaEventRecord(out_done[i], s_out));
        }
        CK(cudaStreamSynchronize(s_in));
        CK(cudaStreamSynchronize(s_cmp));
        CK(cudaStreamSynchronize(s_out));
    }
};

// images per sub-batch of the host pipeline: up to ~32 stages of at least ~1 MPix each, one stage
// for small batches (measured on c4, 64 pairs of 1 MPix, pinned buffers: 8 stages 18.9 ms, 16
// stages 18.9 ms, 32 stages 17.8 ms, 64 stages 21.7 ms per batch)
int pipeline_sub(int batch, long long px_per_image) {
    if (batch < 4) return batch;
    long long sub = (batch + 31) / 32;
    const long long min_imgs = (1LL << 20) / (px_per_image > 0 ? px_per_image : 1) + 1;
    if (sub < min_imgs) sub = min_imgs;
    return sub >= batch ? batch : (int)sub;
}

void smooth_host(const float* t, const float* g, int batch, int width, int height, int channels, int gch,
                 const sgwls_b200_config* cfg, float* out) {
    const size_t it = (size_t)width * height * channels, ig = (size_t)width * height * gch;
    // self-guided call (sgwls::smooth(img, img, cfg), e.g. proj/src/apps.cpp:59): one upload serves both
    const bool same = (g == t) && gch == channels;
    const int sub = pipeline_sub(batch, (long long)width * height);
    if (sub >= batch) {
        cudaStream_t st = cudaStreamPerThread;
        DevBuf dt, dg, dout;
        dt.alloc(it * batch, st);
        if (!same) dg.alloc(ig * batch, st);
        dout.alloc(it * batch, st);
        CK(cudaMemcpyAsync(dt.p, t, it * batch * 4, cudaMemcpyHostToDevice, st));
        if (!same) CK(cudaMemcpyAsync(dg.p, g, ig * batch * 4, cudaMemcpyHostToDevice, st));
        ErrWord ew(st);
        run_smooth(dt.p, same ? dt.p : dg.p, batch, width, height, channels, gch, cfg, dout.p, ew.d, st);
        CK(cudaMemcpyAsync(out, dout.p, it * batch * 4, cudaMemcpyDeviceToHost, st));
        finish_sync(ew.d, st);
        return;
    }
    HostPipeline hp;
    const int nsub = (batch + sub - 1) / sub;
    DevBuf dt[2], dg[2], dout[2];
    for (int k = 0; k < 2; ++k) {
        dt[k].alloc(it * sub, hp.s_in);
        if (!same) dg[k].alloc(ig * sub, hp.s_in);
        dout[k].alloc(it * sub, hp.s_in);
    }
    // one pivot-error word per sub-batch: the first failing sub-batch (batch order) reports
    unsigned long long* d_errs = nullptr;
    CK(cudaMallocAsync((void**)&d_errs, (size_t)nsub * sizeof(unsigned long long), hp.s_in));
    CK(cudaMemsetAsync(d_errs, 0xff, (size_t)nsub * sizeof(unsigned long long), hp.s_in));
    std::vector<unsigned long long> h_errs(nsub, ULLONG_MAX);
    try {
        hp.run(
            batch, sub,
            [&](int i0, int n, int k, cudaStream_t st) {
                CK(cudaMemcpyAsync(dt[k].p, t + it * i0, it * n * 4, cudaMemcpyHostToDevice, st));
                if (!same) CK(cudaMemcpyAsync(dg[k].p, g + ig * i0, ig * n * 4, cudaMemcpyHostToDevice, st));
            },
            [&](int i0, int n, int k, cudaStream_t st) {
                run_smooth(dt[k].p, same ? dt[k].p : dg[k].p, n, width, height, channels, gch, cfg, dout[k].p,
                           d_errs + i0 / sub, st);
            },
            [&](int i0, int n, int k, cudaStream_t st) {
                CK(cudaMemcpyAsync(out + it * i0, dout[k].p, it * n * 4, cudaMemcpyDeviceToHost, st));
            });
        CK(cudaMemcpyAsync(h_errs.data(), d_errs, (size_t)nsub * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           hp.s_cmp));
        CK(cudaStreamSynchronize(hp.s_cmp));
    } catch (...) {
        cudaDeviceSynchronize();
        cudaFreeAsync(d_errs, hp.s_in);
        cudaStreamSynchronize(hp.s_in);
        throw;
    }
    cudaFreeAsync(d_errs, hp.s_in);
    // (the slots are released by their DevBufs on s_in, before hp's streams go: reverse declaration order)
    for (unsigned long long h : h_errs)
        if (h != ULLONG_MAX) throw Fail{SGWLS_B200_EINVAL, pivot_message(h)};
}

void sparse_host_pipelined(const float* v, const float* m, const float* g, int batch, int sub, int width, int height,
                           int channels, int gch, const sgwls_b200_config* cfg, float* out, float* und) {
    const size_t ipx = (size_t)width * height;
    const int nsub = (batch + sub - 1) / sub;
    HostPipeline hp;
    DevBuf dv[2], dm[2], dg[2], dout[2], dund[2];
    for (int k = 0; k < 2; ++k) {
        dv[k].alloc(ipx * channels * sub, hp.s_in);
        dm[k].alloc(ipx * sub, hp.s_in);
        dg[k].alloc(ipx * gch * sub, hp.s_in);
        dout[k].alloc(ipx * channels * sub, hp.s_in);
        if (und) dund[k].alloc(ipx * sub, hp.s_in);
    }
    // per pair: [first offending pixel | mask non-empty]; per sub-batch: the pivot word
    unsigned long long* d_stat = nullptr;
    const size_t nstat = 2 * (size_t)batch + nsub;
    CK(cudaMallocAsync((void**)&d_stat, nstat * sizeof(unsigned long long), hp.s_in));
    CK(cudaMemsetAsync(d_stat, 0xff, nstat * sizeof(unsigned long long), hp.s_in));
    std::vector<unsigned long long> h(nstat);
    try {
        hp.run(
            batch, sub,
            [&](int i0, int n, int k, cudaStream_t st) {
                CK(cudaMemcpyAsync(dv[k].p, v + ipx * channels * i0, ipx * channels * n * 4, cudaMemcpyHostToDevice, st));
                CK(cudaMemcpyAsync(dm[k].p, m + ipx * i0, ipx * n * 4, cudaMemcpyHostToDevice, st));
                CK(cudaMemcpyAsync(dg[k].p, g + ipx * gch * i0, ipx * gch * n * 4, cudaMemcpyHostToDevice, st));
            },
            [&](int i0, int n, int k, cudaStream_t st) {
                // status layout of launch_validate_sparse for this sub-batch: [n minima][n non-empty flags]
                unsigned long long* stat = d_stat + 2 * (size_t)i0;
                CK(cudaMemsetAsync(stat + n, 0, (size_t)n * sizeof(unsigned long long), st));
                CK(launch_validate_sparse(dv[k].p, dm[k].p, (long long)ipx, channels, n, stat, st));
                run_sparse(dv[k].p, dm[k].p, dg[k].p, n, width, height, channels, gch, cfg, dout[k].p, dund[k].p,
                           d_stat + 2 * (size_t)batch + i0 / sub, st);
            },
            [&](int i0, int n, int k, cudaStream_t st) {
                CK(cudaMemcpyAsync(out + ipx * channels * i0, dout[k].p, ipx * channels * n * 4, cudaMemcpyDeviceToHost, st));
                if (und) CK(cudaMemcpyAsync(und + ipx * i0, dund[k].p, ipx * n * 4, cudaMemcpyDeviceToHost, st));
            });
        CK(cudaMemcpyAsync(h.data(), d_stat, nstat * sizeof(unsigned long long), cudaMemcpyDeviceToHost, hp.s_cmp));
        CK(cudaStreamSynchronize(hp.s_cmp));
    } catch (...) {
        cudaDeviceSynchronize();
        cudaFreeAsync(d_stat, hp.s_in);
        throw;
    }
    cudaFreeAsync(d_stat, hp.s_in);
    for (int i = 0; i < nsub; ++i) {
        const int i0 = i * sub, n = std::min(sub, batch - i0);
        for (int b = 0; b < n; ++b) {
            const unsigned long long bad = h[2 * (size_t)i0 + b], any = h[2 * (size_t)i0 + n + b];
            if (bad != ULLONG_MAX) {
                const float mv = m[ipx * (i0 + b) + bad];  // which violation: the host mask tells
                if (mv != 0.f && mv != 1.f) throw Fail{SGWLS_B200_EINVAL, "interpolate_sparse: mask must be 0/1"};
                throw Fail{SGWLS_B200_EINVAL, "interpolate_sparse: values nonzero outside mask"};
            }
            if (any == 0) throw Fail{SGWLS_B200_EINVAL, "interpolate_sparse: empty mask"};
        }
        const unsigned long long piv = h[2 * (size_t)batch + i];
        if (piv != ULLONG_MAX) throw Fail{SGWLS_B200_EINVAL, pivot_message(piv)};
    }
}

// ------------------------------------------------------ CUDA-graph replay
//
// With SGWLS_B200_GRAPH the whole call (every pass, every kernel, the
// stream-ordered scratch allocations) is captured once into a CUDA graph keyed
// by (pointers, shape, configuration) and replayed on later calls with the
// same key: one launch per call instead of ~4 per pass, no host gaps.  The
// graph runs on a private stream joined to the caller's stream with events.
// The cache is a small LRU (kGraphCacheMax entries): an evicted entry waits for
// its last replay and releases its exec, stream, events and error word.
struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    cudaStream_t st = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    unsigned long long* d_err = nullptr;
    int armed = 0;
    unsigned long long used = 0;  // LRU stamp
    int dev = 0;
    ~GraphEntry() {
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != dev) cudaSetDevice(dev);
        if (st) cudaStreamSynchronize(st);
        if (exec) cudaGraphExecDestroy(exec);
        if (ev_in) cudaEventDestroy(ev_in);
        if (ev_out) cudaEventDestroy(ev_out);
        if (d_err) cudaFree(d_err);
        if (st) cudaStreamDestroy(st);
        if (cur != dev) cudaSetDevice(cur);
    }
};
constexpr size_t kGraphCacheMax = 64;
std::mutex g_graph_mu;
std::map<std::string, std::unique_ptr<GraphEntry>> g_graphs;
unsigned long long g_graph_clock = 0;

void graph_evict_lru_locked() {
    while (g_graphs.size() >= kGraphCacheMax) {
        auto victim = g_graphs.begin();
        for (auto it = g_graphs.begin(); it != g_graphs.end(); ++it)
            if (it->second->used < victim->second->used) victim = it;
        g_graphs.erase(victim);
    }
}

std::string graph_key(const void* const* ptrs, int nptr, const int* dims, int ndims, const sgwls_b200_config* cfg,
                      int kind) {
    std::string k;
    k.append((const char*)ptrs, sizeof(void*) * nptr);
    k.append((const char*)dims, sizeof(int) * ndims);
    k.append((const char*)cfg, sizeof(*cfg));
    k.append((const char*)&kind, sizeof kind);
    const int prof = prof_enabled() ? 1 : 0;
    k.append((const char*)&prof, sizeof prof);
    int dev = 0;
    cudaGetDevice(&dev);
    k.append((const char*)&dev, sizeof dev);
    return k;
}

template <class F>
void run_graphed(const std::string& key, cudaStream_t user, bool sync, F&& body) {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    if (g_graphs.find(key) == g_graphs.end()) graph_evict_lru_locked();
    std::unique_ptr<GraphEntry>& slot = g_graphs[key];
    if (!slot) {
        auto ge = std::make_unique<GraphEntry>();
        CK(cudaGetDevice(&ge->dev));
        CK(cudaStreamCreateWithFlags(&ge->st, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ge->ev_in, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ge->ev_out, cudaEventDisableTiming));
        CK(cudaMalloc((void**)&ge->d_err, 2 * sizeof(unsigned long long)));
        cudaGraph_t graph = nullptr;
        CK(cudaStreamBeginCapture(ge->st, cudaStreamCaptureModeRelaxed));
        prof_set_capture(&ge->armed);
        try {
            CK(cudaMemsetAsync(ge->d_err, 0xff, sizeof(unsigned long long), ge->st));
            body(ge->st, ge->d_err);
        } catch (...) {
            prof_set_capture(nullptr);
            cudaStreamEndCapture(ge->st, &graph);
            if (graph) cudaGraphDestroy(graph);
            g_graphs.erase(key);
            throw;
        }
        prof_set_capture(nullptr);
        CK(cudaStreamEndCapture(ge->st, &graph));
        cudaError_t ie = cudaGraphInstantiate(&ge->exec, graph, 0);
        cudaGraphDestroy(graph);
        CK(ie);
        slot = std::move(ge);
    }
    GraphEntry& ge = *slot;
    ge.used = ++g_graph_clock;
    CK(cudaEventRecord(ge.ev_in, user));
    CK(cudaStreamWaitEvent(ge.st, ge.ev_in, 0));
    CK(cudaGraphLaunch(ge.exec, ge.st));
    ge.armed = 1;
    CK(cudaEventRecord(ge.ev_out, ge.st));
    CK(cudaStreamWaitEvent(user, ge.ev_out, 0));
    if (sync) {
        unsigned long long h = ULLONG_MAX;
        CK(cudaMemcpyAsync(&h, ge.d_err, sizeof h, cudaMemcpyDeviceToHost, user));
        CK(cudaStreamSynchronize(user));
        if (h != ULLONG_MAX) throw Fail{SGWLS_B200_EINVAL, pivot_message(h)};
    }
}

template <class F>
int guarded(char* err, size_t errlen, F&& f) {
    try {
        f();
        return SGWLS_B200_OK;
    } catch (const Fail& e) {
        put_err(err, errlen, e.msg);
        return e.code;
    } catch (const std::exception& e) {
        put_err(err, errlen, std::string("sgwls_b200: ") + e.what());
        return SGWLS_B200_ECUDA;
    }
}

// ---------------------------------------------------------- row-slab mode
// One Column pass of an image split into row slabs (one per GPU): layout of
// the caller-provided workspace and the launch description of both phases
// (sgwls_tile.cuh "row-slab mode", sharded.py).
struct SlabLayout {
    AxisPlan ap;
    size_t maps = 0, srec = 0, rsc = 0, zext = 0, zg = 0, bsg = 0, grec = 0, total = 0, record = 0;
};

SlabLayout slab_layout(int width, int rows, int C, int Cg, const sgwls_b200_config* cfg, int nslabs) {
    SlabLayout L;
    L.ap = plan_axis(rows, width, C, Cg, cfg->r, cfg->tau, 1);
    if (!L.ap.fast)
        throw Fail{SGWLS_B200_EUNSUPPORTED, "sgwls_b200: row-slab mode needs the tiled path (r <= 4, 1 or 3 guidance "
                                            "channels, width >= 2r+1)"};
    const size_t NL = L.ap.g.nb, r = cfg->r, REC = rec_floats(cfg->r, C), RS = rs_floats(cfg->r, C);
    const size_t P = L.ap.g.P, NWA = L.ap.nwa, PS = (P + NWA - 1) / NWA;
    const size_t G = nslabs > 1 ? nslabs - 1 : 1;
    size_t off = 0;
    auto take = [&](size_t n) {
        const size_t o = off;
        off += (n + 31) & ~(size_t)31;
        return o;
    };
    L.maps = take(P * map_floats(cfg->r, C) * NL);
    L.srec = take(PS * REC * NL);
    L.rsc = take((PS > 1 ? PS : 1) * r * (RS + r) * NL);
    L.zext = take((PS + 1) * r * C * NL);
    L.zg = take(G * r * C * NL);
    L.bsg = take(G * r * RS * NL);
    L.grec = take((size_t)kSlabWarps * REC * NL);
    L.total = off;
    L.record = REC * NL;
    return L;
}

void slab_check(int width, int rows, int C, int Cg, int row0, int nslabs, int islab, const sgwls_b200_config* cfg) {
    std::string msg;
    int rc = validate_cfg(cfg, msg);
    if (rc) throw Fail{rc, msg};
    rc = check_shape(1, width, rows, C, Cg, msg);
    if (rc) throw Fail{rc, msg};
    if (nslabs < 1 || islab < 0 || islab >= nslabs)
        throw Fail{SGWLS_B200_EINVAL, "sgwls_b200: slab index out of range"};
    if (row0 & 1) throw Fail{SGWLS_B200_EINVAL, "sgwls_b200: slab row offset must be even (serpentine parity)"};
}

PassLaunch slab_launch(const SlabLayout& L, const float* src, const float* guid, int row0, int nslabs, int islab,
                       float* work, const WeightDev* wd, int C) {
    const AxisPlan& ap = L.ap;
    PassLaunch pl;
    pl.geom = ap.g;
    pl.geom.has_prev = islab > 0;
    pl.geom.has_next = islab < nslabs - 1;
    pl.geom.row0 = row0;
    pl.bx = ap.bx;
    pl.fast = 1;
    pl.step = ap.step;
    pl.ncta = ap.ncta;
    pl.nw = ap.nw;
    pl.nwa = ap.nwa;
    pl.nph = ap.nph;
    pl.kmax = ap.kmax;
    pl.src = src;
    pl.guid = guid;
    pl.w = wd;
    pl.err = nullptr;
    pl.U = nullptr;
    const size_t NL = ap.g.nb, rC = (size_t)ap.g.r * C;
    pl.maps = work + L.maps;
    pl.rec = work + L.srec;
    pl.rs = work + L.rsc;
    pl.z = work + L.zext + rC * NL;      // one slot in front: z[-1]
    pl.zg = work + L.zg;
    pl.bsg = work + L.bsg;
    pl.grec = work + L.grec;
    pl.nslab = nslabs;
    pl.islab = islab;
    pl.transpose_out = 0;
    pl.out = nullptr;
    return pl;
}

}  // namespace

extern "C" {

void sgwls_b200_config_default(sgwls_b200_config* c) {
    c->lambda = 900.0;
    c->r = 1;
    c->tau = 1;
    c->iterations = 4;
    c->first_axis = SGWLS_B200_AXIS_COLUMN;
    c->threads = 1;
    c->weight_kind = SGWLS_B200_WEIGHT_FRAC;
    c->alpha_s = 1.2;
    c->alpha_r = 1.2;
    c->sigma_s = 4.0;
    c->sigma_r = 3.0;
    c->epsilon = 1e-4;
    c->guidance_scale = 1.0;
}

int sgwls_b200_validate(const sgwls_b200_config* cfg, char* err, size_t errlen) {
    std::string msg;
    const int rc = validate_cfg(cfg, msg);
    if (rc) put_err(err, errlen, msg);
    return rc;
}

int sgwls_b200_smooth_device(const float* d_t, const float* d_g, int batch, int width, int height, int channels,
                             int gch, const sgwls_b200_config* cfg, float* d_out, void* stream, int flags,
                             char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::string msg;
        int rc = validate_cfg(cfg, msg);
        if (rc) throw Fail{rc, msg};
        rc = check_shape(batch, width, height, channels, gch, msg);
        if (rc) throw Fail{rc, msg};
        require_device();
        cudaStream_t st = (cudaStream_t)stream;
        if (flags & SGWLS_B200_GRAPH) {
            const void* ptrs[3] = {d_t, d_g, d_out};
            const int dims[5] = {batch, width, height, channels, gch};
            run_graphed(graph_key(ptrs, 3, dims, 5, cfg, 0), st, flags & SGWLS_B200_SYNC,
                        [&](cudaStream_t gs, unsigned long long* de) {
                            run_smooth(d_t, d_g, batch, width, height, channels, gch, cfg, d_out, de, gs);
                        });
            return;
        }
        ErrWord ew(st);
        run_smooth(d_t, d_g, batch, width, height, channels, gch, cfg, d_out, ew.d, st);
        if (flags & SGWLS_B200_SYNC) finish_sync(ew.d, st);
    });
}

int sgwls_b200_pass_device(const float* d_src, const float* d_g, int batch, int width, int height, int channels,
                           int gch, const sgwls_b200_config* cfg, float* d_out_t, void* stream, int flags,
                           char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::string msg;
        int rc = validate_cfg(cfg, msg);
        if (rc) throw Fail{rc, msg};
        rc = check_shape(batch, width, height, channels, gch, msg);
        if (rc) throw Fail{rc, msg};
        require_device();
        cudaStream_t st = (cudaStream_t)stream;
        if (flags & SGWLS_B200_GRAPH) {
            const void* ptrs[3] = {d_src, d_g, d_out_t};
            const int dims[5] = {batch, width, height, channels, gch};
            run_graphed(graph_key(ptrs, 3, dims, 5, cfg, 2), st, flags & SGWLS_B200_SYNC,
                        [&](cudaStream_t gs, unsigned long long* de) {
                            run_smooth(d_src, d_g, batch, width, height, channels, gch, cfg, d_out_t, de, gs, true);
                        });
            return;
        }
        ErrWord ew(st);
        run_smooth(d_src, d_g, batch, width, height, channels, gch, cfg, d_out_t, ew.d, st, true);
        if (flags & SGWLS_B200_SYNC) finish_sync(ew.d, st);
    });
}

int sgwls_b200_smooth_batch(const float* t, const float* g, int batch, int width, int height, int channels,
                            int gch, const sgwls_b200_config* cfg, float* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::string msg;
        int rc = validate_cfg(cfg, msg);
        if (rc) throw Fail{rc, msg};
        rc = check_shape(batch, width, height, channels, gch, msg);
        if (rc) throw Fail{rc, msg};
        require_device();
        smooth_host(t, g, batch, width, height, channels, gch, cfg, out);
    });
}

int sgwls_b200_smooth(const float* t, int width, int height, int channels, const float* g, int gch,
                      const sgwls_b200_config* cfg, float* out, char* err, size_t errlen) {
    return sgwls_b200_smooth_batch(t, g, 1, width, height, channels, gch, cfg, out, err, errlen);
}

int sgwls_b200_interpolate_sparse_device(const float* d_v, const float* d_m, const float* d_g, int batch,
                                         int width, int height, int channels, int gch,
                                         const sgwls_b200_config* cfg, float* d_out, float* d_und, void* stream,
                                         int flags, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::string msg;
        int rc = check_shape(batch, width, height, channels + 1, gch, msg);
        if (rc) throw Fail{rc, msg};
        rc = validate_cfg(cfg, msg);
        require_device();
        cudaStream_t st = (cudaStream_t)stream;
        if (flags & SGWLS_B200_VALIDATE) validate_sparse(d_v, d_m, batch, (long long)width * height, channels, st);
        if (rc) throw Fail{rc, msg};
        if (flags & SGWLS_B200_GRAPH) {
            const void* ptrs[5] = {d_v, d_m, d_g, d_out, d_und};
            const int dims[5] = {batch, width, height, channels, gch};
            run_graphed(graph_key(ptrs, 5, dims, 5, cfg, 1), st, flags & SGWLS_B200_SYNC,
                        [&](cudaStream_t gs, unsigned long long* de) {
                            run_sparse(d_v, d_m, d_g, batch, width, height, channels, gch, cfg, d_out, d_und, de, gs);
                        });
            return;
        }
        ErrWord ew(st);
        run_sparse(d_v, d_m, d_g, batch, width, height, channels, gch, cfg, d_out, d_und, ew.d, st);
        if (flags & SGWLS_B200_SYNC) finish_sync(ew.d, st);
    });
}

int sgwls_b200_interpolate_sparse_batch(const float* v, const float* m, const float* g, int batch, int width,
                                        int height, int channels, int gch, const sgwls_b200_config* cfg,
                                        float* out, float* und, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::string msg;
        // a field without pixels fails the reference's mask scan first
        // (proj/src/smoother.cpp:131-144): "empty mask", before smooth()'s checks
        if (batch >= 1 && channels >= 1 && (width <= 0 || height <= 0))
            throw Fail{SGWLS_B200_EINVAL, "interpolate_sparse: empty mask"};
        int rc = check_shape(batch, width, height, channels + 1, gch, msg);
        if (rc) throw Fail{rc, msg};
        require_device();
        const int sub = pipeline_sub(batch, (long long)width * height);
        rc = validate_cfg(cfg, msg);
        if (sub < batch && rc == 0) {  // three-stage pipeline over sub-batches (valid configuration)
            sparse_host_pipelined(v, m, g, batch, sub, width, height, channels, gch, cfg, out, und);
            return;
        }
        cudaStream_t st = cudaStreamPerThread;
        const size_t npx = (size_t)batch * width * height;
        DevBuf dv, dm, dg, dout, dund;
        dv.alloc(npx * channels, st);
        dm.alloc(npx, st);
        dg.alloc(npx * gch, st);
        dout.alloc(npx * channels, st);
        if (und) dund.alloc(npx, st);
        CK(cudaMemcpyAsync(dv.p, v, npx * channels * 4, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(dm.p, m, npx * 4, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(dg.p, g, npx * gch * 4, cudaMemcpyHostToDevice, st));
        // the reference validates the field before the configuration (smooth() validates cfg)
        validate_sparse(dv.p, dm.p, batch, (long long)width * height, channels, st);
        if (rc) throw Fail{rc, msg};
        ErrWord ew(st);
        run_sparse(dv.p, dm.p, dg.p, batch, width, height, channels, gch, cfg, dout.p, dund.p, ew.d, st);
        CK(cudaMemcpyAsync(out, dout.p, npx * channels * 4, cudaMemcpyDeviceToHost, st));
        if (und) CK(cudaMemcpyAsync(und, dund.p, npx * 4, cudaMemcpyDeviceToHost, st));
        finish_sync(ew.d, st);
    });
}

int sgwls_b200_interpolate_sparse(const float* v, const float* m, int width, int height, int channels,
                                  const float* g, int gch, const sgwls_b200_config* cfg, float* out, float* und,
                                  char* err, size_t errlen) {
    return sgwls_b200_interpolate_sparse_batch(v, m, g, 1, width, height, channels, gch, cfg, out, und, err,
                                               errlen);
}

int sgwls_b200_kernel_launches(int width, int height, int channels, int gch, int batch, int sparse,
                               const sgwls_b200_config* cfg) {
    std::string msg;
    const int C = channels + (sparse ? 1 : 0);
    if (validate_cfg(cfg, msg) || check_shape(batch, width, height, C, gch, msg)) return -1;
    const AxisPlan ap0 = plan_axis(height, width, C, gch, cfg->r, cfg->tau, batch);
    const AxisPlan ap1 = plan_axis(width, height, C, gch, cfg->r, cfg->tau, batch);
    const int T = cfg->iterations, fa = cfg->first_axis;
    int n = 0;
    if (fa == 1 || T >= 2) n += 1;  // guidance transpose
    if (fa == 1) n += 1;            // input transpose
    for (int p = 0; p < T; ++p) n += kernels_per_pass(((fa + p) & 1) == 0 ? ap0 : ap1);
    if (sparse) {  // pack / ratio kernels unless the tiled passes read the field unpacked and fuse the ratio
        bool split = false, ratio = false;
        sparse_fusable(batch, width, height, C, gch, cfg, split, ratio);
        n += (split ? 0 : 1) + (ratio ? 0 : 1);
    }
    return n;
}

int sgwls_b200_describe_pass(int extent, int sweep, int r, int tau, int* info, int* centers, int cap) {
    if (extent < 1 || sweep < 1 || r < 1 || tau < 1) return -1;
    const AxisPlan ap = plan_axis(sweep, extent, 1, 1, r, tau, 1);
    if (info) {
        info[0] = ap.g.nb;
        info[1] = ap.g.m;
        info[2] = ap.g.P;
        info[3] = ap.kmax;
        info[4] = ap.g.nreg;
        info[5] = ap.g.degenerate;
    }
    for (int b = 0; b < ap.g.nb && b < cap; ++b) centers[b] = band_center(ap.g, b);
    if (info && cap > 0) {
        // chunk row boundaries follow the centres when room is left
        const int rw = ap.kmax / ap.g.m;  // tiled path: uniform chunks of rw rows
        for (int j = 0; j <= ap.g.P && ap.g.nb + j < cap; ++j)
            centers[ap.g.nb + j] = ap.fast ? (j * rw < sweep ? j * rw : sweep) : chunk_row(ap.g, j);
    }
    return ap.g.nb;
}

const char* sgwls_b200_version(void) { return "sgwls_b200 0.2.0 (sm_100a)"; }

int sgwls_b200_graph_clear(void) {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    const int n = (int)g_graphs.size();
    g_graphs.clear();
    return n;
}

int sgwls_b200_graph_count(void) {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    return (int)g_graphs.size();
}

// ------------------------------------------------------------ row-slab mode

int sgwls_b200_transpose_device(const float* d_in, float* d_out, int batch, int width, int height, int channels,
                                void* stream, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (batch < 1 || width < 1 || height < 1 || channels < 1 || channels > 4)
            throw Fail{SGWLS_B200_EINVAL, "sgwls_b200: transpose needs a non-empty image of 1-4 channels"};
        require_device();
        CK(launch_transpose(d_in, d_out, height, width, channels, batch, (cudaStream_t)stream));
    });
}

int sgwls_b200_slab_sizes(int width, int rows, int channels, int gch, int nslabs, const sgwls_b200_config* cfg,
                          size_t* work_floats, size_t* record_floats, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        slab_check(width, rows, channels, gch, 0, nslabs, 0, cfg);
        const SlabLayout L = slab_layout(width, rows, channels, gch, cfg, nslabs);
        if (work_floats) *work_floats = L.total;
        if (record_floats) *record_floats = L.record;
    });
}

int sgwls_b200_slab_pass_a(const float* d_src, const float* d_guid, int width, int rows, int channels, int gch,
                           int row0, int nslabs, int islab, const sgwls_b200_config* cfg, float* d_work,
                           float* d_record, void* stream, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        slab_check(width, rows, channels, gch, row0, nslabs, islab, cfg);
        require_device();
        const SlabLayout L = slab_layout(width, rows, channels, gch, cfg, nslabs);
        WeightDev wd;
        build_weights(cfg, wd);
        PassLaunch pl = slab_launch(L, d_src, d_guid, row0, nslabs, islab, d_work, &wd, channels);
        pl.slab_phase = 1;
        pl.slabrec = d_record;
        CK(launch_pass(pl, (cudaStream_t)stream));
    });
}

int sgwls_b200_slab_pass_b(const float* d_src, const float* d_guid, int width, int rows, int channels, int gch,
                           int row0, int nslabs, int islab, const sgwls_b200_config* cfg, float* d_work,
                           const float* d_records, float* d_out, unsigned long long* d_pivot_err, void* stream,
                           char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        slab_check(width, rows, channels, gch, row0, nslabs, islab, cfg);
        require_device();
        const SlabLayout L = slab_layout(width, rows, channels, gch, cfg, nslabs);
        WeightDev wd;
        build_weights(cfg, wd);
        PassLaunch pl = slab_launch(L, d_src, d_guid, row0, nslabs, islab, d_work, &wd, channels);
        pl.slab_phase = 2;
        pl.slabrec = const_cast<float*>(d_records);
        pl.out = d_out;
        pl.err = d_pivot_err;
        CK(launch_pass(pl, (cudaStream_t)stream));
    });
}

// ------------------------------------------------ application pipelines
// proj/src/apps.cpp, every stage on the device (sgwls_apps.cu).

void sgwls_b200_enhance_preset(sgwls_b200_config* c) {  // proj/src/apps.cpp:8-20
    sgwls_b200_config_default(c);
    c->lambda = 900.0;
    c->r = 1;
    c->tau = 1;
    c->iterations = 4;
    c->weight_kind = SGWLS_B200_WEIGHT_FRAC;
    c->alpha_s = 1.2;
    c->alpha_r = 1.2;
    c->guidance_scale = 1.0;
}

void sgwls_b200_tonemap_layer_preset(double lambda, sgwls_b200_config* c) {  // proj/src/apps.cpp:22-26
    sgwls_b200_enhance_preset(c);
    c->lambda = lambda;
}

int sgwls_b200_upsample_preset(int factor, sgwls_b200_config* c, char* err, size_t errlen) {  // :28-44
    sgwls_b200_config_default(c);
    c->r = 4;
    c->tau = 4;
    c->iterations = 4;
    c->weight_kind = SGWLS_B200_WEIGHT_EXP;
    c->sigma_s = 4.0;
    c->sigma_r = 3.0;
    c->guidance_scale = 255.0;
    switch (factor) {
        case 2: c->lambda = 100.0; return SGWLS_B200_OK;
        case 4: c->lambda = 200.0; return SGWLS_B200_OK;
        case 8: c->lambda = 400.0; return SGWLS_B200_OK;
        default:
            put_err(err, errlen, "upsample_preset: published lambdas cover factors 2, 4 and 8");
            return SGWLS_B200_EINVAL;
    }
}

void sgwls_b200_colorize_preset(sgwls_b200_config* c) {  // proj/src/apps.cpp:46-56
    sgwls_b200_config_default(c);
    c->lambda = 900.0;
    c->r = 4;
    c->tau = 2;
    c->iterations = 4;
    c->weight_kind = SGWLS_B200_WEIGHT_EXP;
    c->sigma_s = 4.0;
    c->sigma_r = 2.0;
    c->guidance_scale = 255.0;
}

void sgwls_b200_tonemap_params_default(sgwls_b200_tonemap_params* p) {  // proj/include/sgwls/apps.hpp:21-30
    p->lambdas[0] = 5.0;
    p->lambdas[1] = 40.0;
    p->lambdas[2] = 320.0;
    p->detail_weights[0] = p->detail_weights[1] = p->detail_weights[2] = 1.0;
    p->target_log_range = 2.0;
    sgwls_b200_tonemap_layer_preset(5.0, &p->smoothing);
}

int sgwls_b200_detail_enhance(const float* img, int width, int height, int channels, double boost,
                              const sgwls_b200_config* cfg, float* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        // base = smooth(img, img, cfg): the configuration is validated first
        std::string msg;
        int rc = validate_cfg(cfg, msg);
        if (rc) throw Fail{rc, msg};
        rc = check_shape(1, width, height, channels, channels, msg);
        if (rc) throw Fail{rc, msg};
        require_device();
        cudaStream_t st = cudaStreamPerThread;
        const size_t n = (size_t)width * height * channels;
        DevBuf dimg, dbase, dout;
        dimg.alloc(n, st);
        dbase.alloc(n, st);
        dout.alloc(n, st);
        CK(cudaMemcpyAsync(dimg.p, img, n * 4, cudaMemcpyHostToDevice, st));
        ErrWord ew(st);
        run_smooth(dimg.p, dimg.p, 1, width, height, channels, channels, cfg, dbase.p, ew.d, st);
        CK(launch_detail(dimg.p, dbase.p, (float)boost, dout.p, (long long)n, st));
        CK(cudaMemcpyAsync(out, dout.p, n * 4, cudaMemcpyDeviceToHost, st));
        finish_sync(ew.d, st);
    });
}

int sgwls_b200_tone_map(const float* hdr, int width, int height, int channels, const sgwls_b200_tonemap_params* p,
                        float* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (channels != 1 && channels != 3) throw Fail{SGWLS_B200_EINVAL, "luminance needs 1 or 3 channels"};
        require_device();
        cudaStream_t st = cudaStreamPerThread;
        const long long npx = (long long)(width > 0 ? width : 0) * (height > 0 ? height : 0);
        const size_t n = (size_t)npx * channels;
        DevBuf dhdr, dlum, dout, dlev[4];
        DevBuf flags;  // [bad | min | max | anchor]
        dhdr.alloc(n, st);
        dout.alloc(n, st);
        dlum.alloc(npx, st);
        for (auto& b : dlev) b.alloc(npx, st);
        flags.alloc(4, st);
        unsigned* dflags = reinterpret_cast<unsigned*>(flags.p);
        const unsigned init[4] = {0u, 0xffffffffu, 0u, 0u};
        CK(cudaMemcpyAsync(dflags, init, sizeof init, cudaMemcpyHostToDevice, st));
        if (npx > 0) {
            CK(cudaMemcpyAsync(dhdr.p, hdr, n * 4, cudaMemcpyHostToDevice, st));
            CK(launch_luma_log(dhdr.p, channels, dlum.p, dlev[0].p, npx, dflags, st));
            unsigned bad = 0;
            CK(cudaMemcpyAsync(&bad, dflags, sizeof bad, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (bad) throw Fail{SGWLS_B200_EINVAL, "tone_map: luminance must be strictly positive"};
        }
        // level_{i+1} = smooth(level_i, log_lum, smoothing with lambda_i)   (proj/src/apps.cpp:78-88)
        ErrWord ew(st);
        for (int i = 0; i < 3; ++i) {
            sgwls_b200_config c = p->smoothing;
            c.lambda = p->lambdas[i];
            std::string msg;
            int rc = validate_cfg(&c, msg);
            if (rc) throw Fail{rc, msg};
            rc = check_shape(1, width, height, 1, 1, msg);
            if (rc) throw Fail{rc, msg};
            run_smooth(dlev[i].p, dlev[0].p, 1, width, height, 1, 1, &c, dlev[i + 1].p, ew.d, st);
        }
        const float* lev[4] = {dlev[0].p, dlev[1].p, dlev[2].p, dlev[3].p};
        const float dw[3] = {(float)p->detail_weights[0], (float)p->detail_weights[1], (float)p->detail_weights[2]};
        CK(launch_tone_out(dhdr.p, channels, dlum.p, lev, dflags + 1, (float)p->target_log_range, dw, dout.p, npx,
                           st));
        CK(cudaMemcpyAsync(out, dout.p, n * 4, cudaMemcpyDeviceToHost, st));
        finish_sync(ew.d, st);
    });
}

int sgwls_b200_depth_upsample(const float* lowres, int low_width, int low_height, int low_channels,
                              const float* guidance, int width, int height, int guidance_channels, int factor,
                              const sgwls_b200_config* cfg, float* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        // checks in the reference's order (proj/src/apps.cpp:113-116, then luminance(guidance))
        if (low_channels != 1) throw Fail{SGWLS_B200_EINVAL, "depth_upsample: depth must be single-channel"};
        if (factor < 1) throw Fail{SGWLS_B200_EINVAL, "depth_upsample: factor must be >= 1"};
        if (width != low_width * factor || height != low_height * factor)
            throw Fail{SGWLS_B200_EINVAL, "depth_upsample: guidance must be exactly factor times the depth size"};
        if (guidance_channels != 1 && guidance_channels != 3)
            throw Fail{SGWLS_B200_EINVAL, "luminance needs 1 or 3 channels"};
        // the projected field is 0/1 by construction; an empty one is the reference's error
        if ((long long)low_width * low_height <= 0) throw Fail{SGWLS_B200_EINVAL, "interpolate_sparse: empty mask"};
        std::string msg;
        int rc = validate_cfg(cfg, msg);
        if (rc) throw Fail{rc, msg};
        rc = check_shape(1, width, height, 2, 1, msg);
        if (rc) throw Fail{rc, msg};
        require_device();
        cudaStream_t st = cudaStreamPerThread;
        const long long npx = (long long)width * height, nlow = (long long)low_width * low_height;
        DevBuf dlow, dguid, dlum, dval, dmask, dout;
        dlow.alloc(nlow, st);
        dguid.alloc(npx * guidance_channels, st);
        dval.alloc(npx, st);
        dmask.alloc(npx, st);
        dout.alloc(npx, st);
        CK(cudaMemcpyAsync(dlow.p, lowres, nlow * 4, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(dguid.p, guidance, npx * guidance_channels * 4, cudaMemcpyHostToDevice, st));
        const float* g = dguid.p;
        if (guidance_channels == 3) {
            dlum.alloc(npx, st);
            CK(launch_luma(dguid.p, 3, dlum.p, npx, st));
            g = dlum.p;
        }
        CK(cudaMemsetAsync(dval.p, 0, npx * 4, st));
        CK(cudaMemsetAsync(dmask.p, 0, npx * 4, st));
        CK(launch_scatter_depth(dlow.p, low_width, low_height, factor, width, dval.p, dmask.p, st));
        ErrWord ew(st);
        run_sparse(dval.p, dmask.p, g, 1, width, height, 1, 1, cfg, dout.p, nullptr, ew.d, st);
        CK(cudaMemcpyAsync(out, dout.p, npx * 4, cudaMemcpyDeviceToHost, st));
        finish_sync(ew.d, st);
    });
}

int sgwls_b200_colorize(const float* gray, int gray_channels, const float* scribbles, int scribble_channels,
                        const float* scribble_mask, int width, int height, const sgwls_b200_config* cfg, float* out,
                        char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (gray_channels != 1) throw Fail{SGWLS_B200_EINVAL, "colorize: gray image must be single-channel"};
        if (scribble_channels != 3) throw Fail{SGWLS_B200_EINVAL, "colorize: scribbles must be 3-channel"};
        require_device();
        cudaStream_t st = cudaStreamPerThread;
        const long long npx = (long long)(width > 0 ? width : 0) * (height > 0 ? height : 0);
        DevBuf dgray, dscrib, dmask, duv, dres, dout;
        dgray.alloc(npx, st);
        dscrib.alloc(npx * 3, st);
        dmask.alloc(npx, st);
        duv.alloc(npx * 2, st);
        dres.alloc(npx * 2, st);
        dout.alloc(npx * 3, st);
        CK(cudaMemcpyAsync(dgray.p, gray, npx * 4, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(dscrib.p, scribbles, npx * 3 * 4, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(dmask.p, scribble_mask, npx * 4, cudaMemcpyHostToDevice, st));
        // U and V share the mask and the guidance: one 2-channel interpolate_sparse
        // (the reference's two calls, proj/src/apps.cpp:151-152, factor identically)
        CK(launch_colorize_pack(dscrib.p, dmask.p, duv.p, npx, st));
        if (npx <= 0) throw Fail{SGWLS_B200_EINVAL, "interpolate_sparse: empty mask"};
        validate_sparse(duv.p, dmask.p, 1, npx, 2, st);
        std::string msg;
        int rc = validate_cfg(cfg, msg);
        if (rc) throw Fail{rc, msg};
        rc = check_shape(1, width, height, 3, 1, msg);
        if (rc) throw Fail{rc, msg};
        ErrWord ew(st);
        run_sparse(duv.p, dmask.p, dgray.p, 1, width, height, 2, 1, cfg, dres.p, nullptr, ew.d, st);
        CK(launch_colorize_out(dgray.p, dres.p, dout.p, npx, st));
        CK(cudaMemcpyAsync(out, dout.p, npx * 3 * 4, cudaMemcpyDeviceToHost, st));
        finish_sync(ew.d, st);
    });
}

}  // extern "C"

// ====================================================== multi-GPU (row slabs)
//
// sgwls::smooth of ONE image over several GPUs driven from this process: the
// row-slab mode of sgwls_tile.cuh (paper_1705_01674_b200/slabs.py is the same
// schedule over torch.distributed ranks).  Device i keeps image rows
// [a_i, a_{i+1}) for the whole filter.  A Column pass is the exact partitioned
// solve: phase A (KA + one slab record per band) on every device, an
// all-gather of the slab records (cudaMemcpyPeerAsync: NVLink P2P when the
// devices can reach each other, staged by the driver otherwise), phase B
// (slab separators, KB) -- only ~G*bands*REC floats cross GPUs.  A Row pass
// runs each device's row window [s_i, e_i) (its slab plus a halo of <= 2r+1
// rows, exchanged peer to peer) as an ordinary pass on the transposed window.
// Every device works on its own stream; pass boundaries are cross-device event
// barriers.  The same device may appear several times (slabs on one GPU).
namespace {

struct SlabDev {
    int dev = 0, a = 0, b = 0, s = 0, e = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t ev = nullptr;
    float* buf[2] = {nullptr, nullptr};  // row window [s, e) x W x C, ping-pong
    float* gwin = nullptr;               // guidance rows [s, e)
    float* gwinT = nullptr;              // transposed guidance window (W x (e-s))
    float* tmpT = nullptr;               // transposed image window
    float* work = nullptr;               // slab-pass workspace
    float* allrec = nullptr;             // G slab records
    unsigned long long* err = nullptr;   // first-pass pivot report
};

struct DevGuard {
    int saved = 0;
    DevGuard() { cudaGetDevice(&saved); }
    ~DevGuard() { cudaSetDevice(saved); }
};

class MultiSlab {
   public:
    MultiSlab(const int* devices, int ndev, int W, int H, int C, int Cg, const sgwls_b200_config* cfg)
        : W_(W), H_(H), C_(C), Cg_(Cg), cfg_(*cfg), G_(ndev) {
        pcfg_ = cfg_;
        pcfg_.iterations = 1;
        pcfg_.first_axis = SGWLS_B200_AXIS_COLUMN;
        build_weights(&pcfg_, wd_);
        const int r = cfg->r, tau = cfg->tau;
        sl_.resize(G_);
        for (int g = 0; g < G_; ++g) {  // slabs with even starts (serpentine parity), as slabs.slab_rows
            sl_[g].dev = devices[g];
            sl_[g].a = 2 * (int)(((long long)g * H) / (2LL * G_));
        }
        for (int g = 0; g < G_; ++g) {
            SlabDev& d = sl_[g];
            d.b = g + 1 < G_ ? sl_[g + 1].a : H;
            if (d.b <= d.a) throw Fail{SGWLS_B200_EINVAL, "sgwls_b200: image too short for " + std::to_string(G_) + " row slabs"};
            d.s = d.a == 0 ? 0 : ((d.a - 2 * r > 0 ? d.a - 2 * r : 0) / tau) * tau;
            d.e = d.b == H ? H : (d.b + 2 * r + 1 < H ? d.b + 2 * r + 1 : H);
        }
    }
    // allocation separate from construction: a failure part-way is cleaned up by the destructor
    void init() {
        const int W = W_, C = C_, Cg = Cg_;
        for (int g = 0; g < G_; ++g) {
            SlabDev& d = sl_[g];
            CK(cudaSetDevice(d.dev));
            init_pool_once_dev(d.dev);
            CK(cudaStreamCreateWithFlags(&d.st, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&d.ev, cudaEventDisableTiming));
            const size_t ws = (size_t)(d.e - d.s) * W;
            CK(cudaMalloc((void**)&d.buf[0], ws * C * 4));
            CK(cudaMalloc((void**)&d.buf[1], ws * C * 4));
            CK(cudaMalloc((void**)&d.gwin, ws * Cg * 4));
            CK(cudaMalloc((void**)&d.gwinT, ws * Cg * 4));
            CK(cudaMalloc((void**)&d.tmpT, ws * C * 4));
            const SlabLayout L = slab_layout(W, d.b - d.a, C, Cg, &pcfg_, G_);
            recn_ = L.record;
            CK(cudaMalloc((void**)&d.work, (L.total ? L.total : 1) * 4));
            CK(cudaMalloc((void**)&d.allrec, (size_t)G_ * L.record * 4));
            CK(cudaMalloc((void**)&d.err, sizeof(unsigned long long)));
            for (int h = 0; h < G_; ++h)  // P2P where the topology allows it (errors: already on / unsupported)
                if (sl_[h].dev != d.dev && cudaDeviceEnablePeerAccess(sl_[h].dev, 0) != cudaSuccess)
                    cudaGetLastError();
        }
    }
    ~MultiSlab() {
        for (SlabDev& d : sl_) {
            cudaSetDevice(d.dev);
            if (d.st) cudaStreamSynchronize(d.st);
            for (float* p : {d.buf[0], d.buf[1], d.gwin, d.gwinT, d.tmpT, d.work, d.allrec}) cudaFree(p);
            cudaFree(d.err);
            if (d.ev) cudaEventDestroy(d.ev);
            if (d.st) cudaStreamDestroy(d.st);
        }
    }

    void run(const float* target, const float* guidance, float* out) {
        const size_t rowC = (size_t)W_ * C_, rowG = (size_t)W_ * Cg_;
        for (SlabDev& d : sl_) {  // upload: own rows + guidance window
            CK(cudaSetDevice(d.dev));
            CK(cudaMemsetAsync(d.err, 0xff, sizeof(unsigned long long), d.st));
            CK(cudaMemcpyAsync(d.buf[0] + (size_t)(d.a - d.s) * rowC, target + (size_t)d.a * rowC,
                               (size_t)(d.b - d.a) * rowC * 4, cudaMemcpyHostToDevice, d.st));
            CK(cudaMemcpyAsync(d.gwin, guidance + (size_t)d.s * rowG, (size_t)(d.e - d.s) * rowG * 4,
                               cudaMemcpyHostToDevice, d.st));
            CK(launch_transpose(d.gwin, d.gwinT, d.e - d.s, W_, Cg_, 1, d.st));
        }
        int cur = 0;
        for (int p = 0; p < cfg_.iterations; ++p) {
            const bool column = ((cfg_.first_axis + p) & 1) == 0;
            if (column)
                column_pass(cur, p == 0);
            else
                row_pass(cur, p == 0);
            cur ^= 1;
        }
        for (SlabDev& d : sl_) {  // download own rows
            CK(cudaSetDevice(d.dev));
            CK(cudaMemcpyAsync(out + (size_t)d.a * rowC, d.buf[cur] + (size_t)(d.a - d.s) * rowC,
                               (size_t)(d.b - d.a) * rowC * 4, cudaMemcpyDeviceToHost, d.st));
        }
        unsigned long long key = ULLONG_MAX;
        for (SlabDev& d : sl_) {
            CK(cudaSetDevice(d.dev));
            unsigned long long h = ULLONG_MAX;
            CK(cudaMemcpyAsync(&h, d.err, sizeof h, cudaMemcpyDeviceToHost, d.st));
            CK(cudaStreamSynchronize(d.st));
            if (h < key) key = h;
        }
        if (key != ULLONG_MAX) throw Fail{SGWLS_B200_EINVAL, pivot_message(key)};
    }

   private:
    // every stream waits for every other stream's work so far
    void barrier() {
        for (SlabDev& d : sl_) {
            CK(cudaSetDevice(d.dev));
            CK(cudaEventRecord(d.ev, d.st));
        }
        for (SlabDev& d : sl_) {
            CK(cudaSetDevice(d.dev));
            for (SlabDev& o : sl_)
                if (&o != &d) CK(cudaStreamWaitEvent(d.st, o.ev, 0));
        }
    }

    void column_pass(int cur, bool first) {
        const size_t rowC = (size_t)W_ * C_, rowG = (size_t)W_ * Cg_;
        for (int g = 0; g < G_; ++g) {  // phase A: chunk records + this slab's record
            SlabDev& d = sl_[g];
            CK(cudaSetDevice(d.dev));
            const SlabLayout L = slab_layout(W_, d.b - d.a, C_, Cg_, &pcfg_, G_);
            PassLaunch pl = slab_launch(L, d.buf[cur] + (size_t)(d.a - d.s) * rowC, d.gwin + (size_t)(d.a - d.s) * rowG,
                                        d.a, G_, g, d.work, &wd_, C_);
            pl.slab_phase = 1;
            pl.slabrec = d.allrec + (size_t)g * recn_;
            CK(launch_pass(pl, d.st));
        }
        barrier();
        for (int h = 0; h < G_; ++h) {  // all-gather of the slab records, pulled by each device
            SlabDev& d = sl_[h];
            CK(cudaSetDevice(d.dev));
            for (int g = 0; g < G_; ++g)
                if (g != h)
                    CK(cudaMemcpyPeerAsync(d.allrec + (size_t)g * recn_, d.dev, sl_[g].allrec + (size_t)g * recn_,
                                           sl_[g].dev, recn_ * 4, d.st));
        }
        barrier();
        for (int g = 0; g < G_; ++g) {  // phase B: slab separators, chunk interiors, own rows
            SlabDev& d = sl_[g];
            CK(cudaSetDevice(d.dev));
            const SlabLayout L = slab_layout(W_, d.b - d.a, C_, Cg_, &pcfg_, G_);
            PassLaunch pl = slab_launch(L, d.buf[cur] + (size_t)(d.a - d.s) * rowC, d.gwin + (size_t)(d.a - d.s) * rowG,
                                        d.a, G_, g, d.work, &wd_, C_);
            pl.slab_phase = 2;
            pl.slabrec = d.allrec;
            pl.out = d.buf[cur ^ 1] + (size_t)(d.a - d.s) * rowC;
            pl.err = first ? d.err : nullptr;
            CK(launch_pass(pl, d.st));
        }
    }

    void row_pass(int cur, bool first) {
        const size_t rowC = (size_t)W_ * C_;
        barrier();
        for (int h = 0; h < G_; ++h) {  // halo rows: window rows of h owned by other slabs
            SlabDev& d = sl_[h];
            CK(cudaSetDevice(d.dev));
            for (int g = 0; g < G_; ++g) {
                if (g == h) continue;
                const SlabDev& o = sl_[g];
                const int lo = o.a > d.s ? o.a : d.s, hi = o.b < d.e ? o.b : d.e;
                if (lo >= hi) continue;
                CK(cudaMemcpyPeerAsync(d.buf[cur] + (size_t)(lo - d.s) * rowC, d.dev, o.buf[cur] + (size_t)(lo - o.s) * rowC,
                                       o.dev, (size_t)(hi - lo) * rowC * 4, d.st));
            }
        }
        barrier();
        for (SlabDev& d : sl_) {  // the window as an ordinary Column pass on its transpose
            CK(cudaSetDevice(d.dev));
            const int ws = d.e - d.s;
            CK(launch_transpose(d.buf[cur], d.tmpT, ws, W_, C_, 1, d.st));
            run_smooth(d.tmpT, d.gwinT, 1, ws, W_, C_, Cg_, &pcfg_, d.buf[cur ^ 1], first ? d.err : nullptr, d.st, true);
        }
    }

    static void init_pool_once_dev(int dev) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            unsigned long long thr = ULLONG_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }

    int W_, H_, C_, Cg_;
    sgwls_b200_config cfg_, pcfg_;
    WeightDev wd_;
    int G_;
    size_t recn_ = 0;
    std::vector<SlabDev> sl_;
};

// devices / ndev -> the device list; ndev <= 0: SGWLS_B200_DEVICES ("0,1,...") or device 0
std::vector<int> device_list(const int* devices, int ndev) {
    std::vector<int> v;
    if (ndev > 0) {
        if (!devices) throw Fail{SGWLS_B200_EINVAL, "sgwls_b200: null device list"};
        v.assign(devices, devices + ndev);
    } else if (const char* e = std::getenv("SGWLS_B200_DEVICES")) {
        std::string s(e);
        size_t i = 0;
        while (i < s.size()) {
            size_t j = s.find(',', i);
            if (j == std::string::npos) j = s.size();
            if (j > i) v.push_back(std::atoi(s.substr(i, j - i).c_str()));
            i = j + 1;
        }
    }
    if (v.empty()) v.push_back(0);
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    for (int d : v)
        if (d < 0 || d >= n) throw Fail{SGWLS_B200_EINVAL, "sgwls_b200: device " + std::to_string(d) + " does not exist"};
    return v;
}

}  // namespace

extern "C" {

int sgwls_b200_smooth_multi(const float* target, int width, int height, int channels, const float* guidance,
                            int gch, const sgwls_b200_config* cfg, const int* devices, int ndev, float* out,
                            char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::string msg;
        int rc = validate_cfg(cfg, msg);
        if (rc) throw Fail{rc, msg};
        rc = check_shape(1, width, height, channels, gch, msg);
        if (rc) throw Fail{rc, msg};
        require_device();
        DevGuard keep;
        const std::vector<int> devs = device_list(devices, ndev);
        // one device, or a geometry the slab mode does not cover (clipped bands,
        // r > 4, 2/4 guidance channels, too few rows per slab): the whole image on
        // the first device
        const AxisPlan ap = plan_axis(height, width, channels, gch, cfg->r, cfg->tau, 1);
        const int G = (int)devs.size();
        bool slabs_ok = G > 1 && ap.fast && width >= 2 * cfg->r + 1;
        auto slab_start = [&](int g) { return g >= G ? height : 2 * (int)(((long long)g * height) / (2LL * G)); };
        for (int g = 0; g < G && slabs_ok; ++g) slabs_ok = slab_start(g + 1) > slab_start(g);  // non-empty slabs
        if (!slabs_ok) {
            CK(cudaSetDevice(devs[0]));
            smooth_host(target, guidance, 1, width, height, channels, gch, cfg, out);
            return;
        }
        MultiSlab ms(devs.data(), G, width, height, channels, gch, cfg);
        ms.init();
        ms.run(target, guidance, out);
    });
}

// `batch` independent interpolate_sparse pairs split over the devices (each
// device runs a contiguous share of the pairs on its own host thread).
int sgwls_b200_interpolate_sparse_batch_multi(const float* values, const float* masks, const float* guidances,
                                              int batch, int width, int height, int channels, int gch,
                                              const sgwls_b200_config* cfg, const int* devices, int ndev, float* out,
                                              float* undefined_mask, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        DevGuard keep;
        std::vector<int> devs = device_list(devices, ndev);
        if (batch < 1) throw Fail{SGWLS_B200_EINVAL, "smooth: empty target"};
        if ((int)devs.size() > batch) devs.resize(batch);
        const int G = (int)devs.size();
        const size_t npx = (size_t)width * height;
        std::vector<int> rcs(G, 0);
        std::vector<std::string> msgs(G);
        std::vector<std::thread> th;
        for (int g = 0; g < G; ++g) {
            th.emplace_back([&, g] {
                const int b0 = (int)((long long)g * batch / G), b1 = (int)((long long)(g + 1) * batch / G);
                char e2[512] = {0};
                if (cudaSetDevice(devs[g]) != cudaSuccess) {
                    rcs[g] = SGWLS_B200_ECUDA;
                    msgs[g] = "sgwls_b200: cannot select device " + std::to_string(devs[g]);
                    return;
                }
                rcs[g] = sgwls_b200_interpolate_sparse_batch(
                    values + b0 * npx * channels, masks + b0 * npx, guidances + b0 * npx * gch, b1 - b0, width, height,
                    channels, gch, cfg, out + b0 * npx * channels, undefined_mask ? undefined_mask + b0 * npx : nullptr,
                    e2, sizeof e2);
                msgs[g] = e2;
            });
        }
        for (auto& t : th) t.join();
        for (int g = 0; g < G; ++g)  // the first failing share in batch order, like the serial loop
            if (rcs[g]) throw Fail{rcs[g], msgs[g]};
    });
}

}  // extern "C"
