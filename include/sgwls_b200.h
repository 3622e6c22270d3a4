/*
 * sgwls_b200.h -- C ABI of the B200-native SG-WLS filter (arXiv 1705.01674).
 *
 * Drop-in boundary for the reference's filter entry points.  The reference is
 * a plain C++ static library with no plugin/FFI layer; the
 * two functions a caller binds are
 *
 *   sgwls::smooth              proj/include/sgwls/smoother.hpp:30
 *                              (definition proj/src/smoother.cpp:113-125)
 *   sgwls::interpolate_sparse  proj/include/sgwls/smoother.hpp:41-42
 *                              (definition proj/src/smoother.cpp:127-163)
 *
 * and this header exposes them as extern "C" calls on plain pointers.  The C++
 * shim csrc/shim/smoother_gpu.cpp re-creates the exact reference signatures on
 * top of these calls (link-substitution for proj/src/smoother.cpp); the
 * ctypes / cffi bindings in INTEGRATION.md bind them directly.
 *
 * Buffers are row-major and channel-interleaved exactly like sgwls::Image
 * (proj/include/sgwls/image.hpp:13-27): sample (y, x, c) lives at
 * ((y*width + x)*channels + c).  Samples are fp32 (the reference holds
 * doubles; the shim converts).  Batched calls take `batch` images back to back.
 *
 * Errors: every entry returns a status; on SGWLS_B200_EINVAL the message
 * written to `err` is the reference's sgwls::Error text verbatim (config
 * validation proj/src/smoother.cpp:103-111, proj/src/weights.cpp:7-12; input
 * checks proj/src/smoother.cpp:115-116,129-144; pivot failure
 * proj/src/banded.cpp:66-68).  There is no CPU fallback: without a CUDA device
 * every compute call returns SGWLS_B200_ECUDA.
 */
#ifndef SGWLS_B200_H
#define SGWLS_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGWLS_B200_OK 0
#define SGWLS_B200_EINVAL 1       /* sgwls::Error equivalent; reference text in err */
#define SGWLS_B200_ECUDA 2        /* CUDA runtime failure or no device */
#define SGWLS_B200_EUNSUPPORTED 3 /* valid for the reference, outside this build's limits (more than 4 channels) */

/* device-call flags */
#define SGWLS_B200_SYNC 1     /* synchronize the stream and report pivot failures */
#define SGWLS_B200_VALIDATE 2 /* interpolate_sparse: validate mask/values (synchronizes) */
#define SGWLS_B200_GRAPH 4    /* capture the call into a CUDA graph once per (pointers, shape, config)
                                 and replay it on later identical calls */

#define SGWLS_B200_AXIS_COLUMN 0
#define SGWLS_B200_AXIS_ROW 1
#define SGWLS_B200_WEIGHT_FRAC 0
#define SGWLS_B200_WEIGHT_EXP 1

/* Field-for-field mirror of sgwls::SmoothConfig (proj/include/sgwls/smoother.hpp:12-24)
 * with sgwls::WeightParams (proj/include/sgwls/weights.hpp:14-27) flattened in. */
typedef struct sgwls_b200_config {
    double lambda;      /* default 900 */
    int r;              /* default 1 */
    int tau;            /* default 1 */
    int iterations;     /* default 4 */
    int first_axis;     /* SGWLS_B200_AXIS_*, default Column */
    int threads;        /* validated like the reference (>= 1); unused on the GPU */
    int weight_kind;    /* SGWLS_B200_WEIGHT_*, default Frac */
    double alpha_s;     /* 1.2 */
    double alpha_r;     /* 1.2 */
    double sigma_s;     /* 4.0 */
    double sigma_r;     /* 3.0 */
    double epsilon;     /* 1e-4 */
    double guidance_scale; /* 1.0 */
} sgwls_b200_config;

/* Reference defaults (proj/include/sgwls/smoother.hpp:12-24, weights.hpp:14-27). */
void sgwls_b200_config_default(sgwls_b200_config* cfg);

/* SmoothConfig::validate (proj/src/smoother.cpp:103-111) incl. WeightParams::validate. */
int sgwls_b200_validate(const sgwls_b200_config* cfg, char* err, size_t errlen);

/* sgwls::smooth on host buffers (synchronous).  out: width*height*channels floats.  A self-guided
 * call (guidance == target, same channel count; proj/src/apps.cpp:59) uploads the buffer once. */
int sgwls_b200_smooth(const float* target, int width, int height, int channels, const float* guidance,
                      int guidance_channels, const sgwls_b200_config* cfg, float* out, char* err, size_t errlen);

/* `batch` independent smooth calls (target i with guidance i).  Larger batches run as an
 * upload / filter / download pipeline over sub-batches on three streams (fastest from pinned
 * host buffers); results and errors as `batch` serial calls (the first failing image decides). */
int sgwls_b200_smooth_batch(const float* targets, const float* guidances, int batch, int width, int height,
                            int channels, int guidance_channels, const sgwls_b200_config* cfg, float* out,
                            char* err, size_t errlen);

/* Device-pointer form, ordered on `stream` (cudaStream_t; NULL = legacy default).
 * Asynchronous unless flags & SGWLS_B200_SYNC. */
int sgwls_b200_smooth_device(const float* d_targets, const float* d_guidances, int batch, int width, int height,
                             int channels, int guidance_channels, const sgwls_b200_config* cfg, float* d_out,
                             void* stream, int flags, char* err, size_t errlen);

/* ONE Column-axis pass (proj/src/smoother.cpp:51-99, run_pass with Axis::Column;
 * cfg->iterations and cfg->first_axis are ignored) on device buffers.  The output
 * is written TRANSPOSED: d_out_t[b][x][y][c] = pass(d_src)[b][y][x][c], i.e. a
 * height-wide, width-tall image ready to be the next (Row-axis) pass's input.
 * Building block of the line-slab sharded filter (paper_1705_01674_b200/sharded.py,
 * BASELINE c5 "lines sharded across GPUs"); same flags as smooth_device. */
int sgwls_b200_pass_device(const float* d_src, const float* d_guidances, int batch, int width, int height,
                           int channels, int guidance_channels, const sgwls_b200_config* cfg, float* d_out_t,
                           void* stream, int flags, char* err, size_t errlen);

/* sgwls::interpolate_sparse on host buffers (synchronous).  values: width*height*channels,
 * mask: width*height (0/1), out: like values, undefined_mask: width*height or NULL. */
int sgwls_b200_interpolate_sparse(const float* values, const float* mask, int width, int height, int channels,
                                  const float* guidance, int guidance_channels, const sgwls_b200_config* cfg,
                                  float* out, float* undefined_mask, char* err, size_t errlen);

int sgwls_b200_interpolate_sparse_batch(const float* values, const float* masks, const float* guidances,
                                        int batch, int width, int height, int channels, int guidance_channels,
                                        const sgwls_b200_config* cfg, float* out, float* undefined_mask,
                                        char* err, size_t errlen);

int sgwls_b200_interpolate_sparse_device(const float* d_values, const float* d_masks, const float* d_guidances,
                                         int batch, int width, int height, int channels, int guidance_channels,
                                         const sgwls_b200_config* cfg, float* d_out, float* d_undefined_mask,
                                         void* stream, int flags, char* err, size_t errlen);

/* Number of kernel launches one smooth / interpolate_sparse call of this shape issues
 * (used by the benchmark's gpu_launches accounting).  Returns -1 on invalid input. */
int sgwls_b200_kernel_launches(int width, int height, int channels, int guidance_channels, int batch, int sparse,
                               const sgwls_b200_config* cfg);

/* Host-side pass geometry (test/diagnostic hook): bands along an axis of `extent`
 * columns swept over `sweep` rows.  info[6] = {bands, band width m, chunks P,
 * max chunk positions, regular centres, degenerate}; centers[0..bands) = band
 * centres (proj/src/snake.cpp:7-19), followed by the P+1 chunk row boundaries
 * while `cap` allows.  Returns the band count or -1. */
int sgwls_b200_describe_pass(int extent, int sweep, int r, int tau, int* info, int* centers, int cap);

/* Profiling hook: when enabled, every kernel launch is bracketed by CUDA events
 * recorded on its own stream.  profile_read synchronizes on them, writes
 * {"<kernel>": {"launches": n, "ms": total}, ...} (plus "pass" = whole passes)
 * into json and clears the log.  Returns the JSON length. */
void sgwls_b200_profile(int enable);
int sgwls_b200_profile_read(char* json, size_t len);
/* Fold the recorded launch times into the running totals (synchronizes on them);
 * call after every replay when profiling graph-replayed calls. */
void sgwls_b200_profile_collect(void);

/* out[b][x][y][c] = in[b][y][x][c] on device buffers (width x height -> height x width), stream-ordered */
int sgwls_b200_transpose_device(const float* d_in, float* d_out, int batch, int width, int height, int channels,
                                void* stream, char* err, size_t errlen);

/* ---- row-slab mode: one Column pass of an image split into row slabs ----
 * (one slab per GPU; paper_1705_01674_b200/sharded.py).  The
 * band solves are partitioned exactly across slabs: phase A computes each
 * slab's chunk records and ONE slab record per band (record_floats floats,
 * layout [field][band]); the caller all-gathers the records of the nslabs
 * slabs back to back ([slab][field][band]); phase B solves the slab separators
 * and finishes the pass.  Only the slab records cross GPUs, never image data.
 * d_src: the slab's rows x width x channels; d_guid: the slab's guidance rows,
 * with row -1 (the previous slab's last row) readable when islab > 0; d_work:
 * work_floats floats kept between the phases; d_out: rows x width x channels
 * (caller layout, not transposed).  row0 (global row of the slab's first row)
 * must be even.  NaN guidance: see d_pivot_err of phase B below. */
int sgwls_b200_slab_sizes(int width, int rows, int channels, int guidance_channels, int nslabs,
                          const sgwls_b200_config* cfg, size_t* work_floats, size_t* record_floats, char* err,
                          size_t errlen);
int sgwls_b200_slab_pass_a(const float* d_src, const float* d_guidance, int width, int rows, int channels,
                           int guidance_channels, int row0, int nslabs, int islab, const sgwls_b200_config* cfg,
                           float* d_work, float* d_record, void* stream, char* err, size_t errlen);
/* d_pivot_err (device, may be NULL): a 64-bit word the caller sets to ~0 before the
 * filter's FIRST pass; that pass's phase B lowers it (atomicMin) to (line << 32 | k)
 * for the first position k of the reference's "non-positive pivot at row k"
 * failure (proj/src/banded.cpp:66-68), k counted from the image's first row.
 * The caller min-reduces the words of all slabs. */
int sgwls_b200_slab_pass_b(const float* d_src, const float* d_guidance, int width, int rows, int channels,
                           int guidance_channels, int row0, int nslabs, int islab, const sgwls_b200_config* cfg,
                           float* d_work, const float* d_records, float* d_out, unsigned long long* d_pivot_err,
                           void* stream, char* err, size_t errlen);

/* ---- multi-GPU (one process driving several devices) ----
 * sgwls::smooth of ONE image over `ndev` devices (devices[i] = CUDA ordinal of row
 * slab i; repeats allowed): the row-slab partitioned solve of the slab API above,
 * with the slab records all-gathered and the row-pass halos exchanged peer to peer
 * (cudaMemcpyPeerAsync over NVLink).  Same result as sgwls_b200_smooth (exact).
 * ndev <= 0: the devices listed in SGWLS_B200_DEVICES ("0,1,2,3"), else device 0.
 * Geometry outside the slab mode (r > 4, clipped bands, 2/4 guidance channels, fewer
 * rows than slabs) runs on the first device.  Host buffers, synchronous. */
int sgwls_b200_smooth_multi(const float* target, int width, int height, int channels, const float* guidance,
                            int guidance_channels, const sgwls_b200_config* cfg, const int* devices, int ndev,
                            float* out, char* err, size_t errlen);
/* `batch` independent interpolate_sparse pairs split over the devices (contiguous
 * shares, one host thread per device); errors as the serial batch call. */
int sgwls_b200_interpolate_sparse_batch_multi(const float* values, const float* masks, const float* guidances,
                                              int batch, int width, int height, int channels, int guidance_channels,
                                              const sgwls_b200_config* cfg, const int* devices, int ndev,
                                              float* out, float* undefined_mask, char* err, size_t errlen);

/* ---- application pipelines (proj/include/sgwls/apps.hpp, proj/src/apps.cpp) ----
 * The reference's four callers of the filter, with every stage on the device:
 * one upload, the smooth() / interpolate_sparse() passes and the elementwise
 * stages (sgwls_apps.cu) on device buffers, one download.  Same parameters,
 * presets and error texts as the reference; fp32 samples. */

/* ToneMapParams (proj/include/sgwls/apps.hpp:21-30) */
typedef struct sgwls_b200_tonemap_params {
    double lambdas[3];           /* {5, 40, 320} */
    double detail_weights[3];    /* {1, 1, 1} */
    double target_log_range;     /* 2 */
    sgwls_b200_config smoothing; /* tonemap_layer_preset(5); lambda set per stage */
} sgwls_b200_tonemap_params;

/* presets (proj/src/apps.cpp:8-56) */
void sgwls_b200_enhance_preset(sgwls_b200_config* cfg);
void sgwls_b200_tonemap_layer_preset(double lambda, sgwls_b200_config* cfg);
int sgwls_b200_upsample_preset(int factor, sgwls_b200_config* cfg, char* err, size_t errlen);
void sgwls_b200_colorize_preset(sgwls_b200_config* cfg);
void sgwls_b200_tonemap_params_default(sgwls_b200_tonemap_params* p);

/* detail_enhance (proj/src/apps.cpp:58-64): clamp(base + boost*(img - base)), base = smooth(img, img) */
int sgwls_b200_detail_enhance(const float* img, int width, int height, int channels, double boost,
                              const sgwls_b200_config* cfg, float* out, char* err, size_t errlen);
/* tone_map (proj/src/apps.cpp:66-109); channels 1 or 3, out like hdr */
int sgwls_b200_tone_map(const float* hdr, int width, int height, int channels, const sgwls_b200_tonemap_params* p,
                        float* out, char* err, size_t errlen);
/* depth_upsample (proj/src/apps.cpp:111-128): lowres low_width x low_height x low_channels (must be 1),
 * guidance width x height x guidance_channels (1 or 3), out width x height x 1 */
int sgwls_b200_depth_upsample(const float* lowres, int low_width, int low_height, int low_channels,
                              const float* guidance, int width, int height, int guidance_channels, int factor,
                              const sgwls_b200_config* cfg, float* out, char* err, size_t errlen);
/* colorize (proj/src/apps.cpp:130-155): gray (1 channel), scribbles (3), mask (1), out width x height x 3 */
int sgwls_b200_colorize(const float* gray, int gray_channels, const float* scribbles, int scribble_channels,
                        const float* scribble_mask, int width, int height, const sgwls_b200_config* cfg, float* out,
                        char* err, size_t errlen);

/* Library version string. */
const char* sgwls_b200_version(void);

/* ---- image files (proj/include/sgwls/image.hpp:38-46, proj/src/image.cpp:111-250) ----
 * read_image: PGM (P2/P5), PPM (P3/P6) scaled to [0,1] (maxval <= 255 -> /255, else /65535,
 * 16-bit samples big-endian) and PFM (Pf/PF, raw floats, bottom-up rows, the scale's sign
 * is the byte order).  *data is malloc'ed (release with sgwls_b200_image_free), row-major
 * channel-interleaved.  write_image: by extension .pgm (P5, 1 channel), .ppm (P6, 3
 * channels), .pfm; LDR writers clamp to [0,1] and quantise round-half-up to 255.
 * Failures return SGWLS_B200_EINVAL with the reference's text ("<path>: byte N: ..."). */
int sgwls_b200_image_read(const char* path, float** data, int* width, int* height, int* channels, char* err,
                          size_t errlen);
void sgwls_b200_image_free(float* data);
int sgwls_b200_image_write(const char* path, const float* data, int width, int height, int channels, char* err,
                           size_t errlen);

/* CUDA-graph cache of SGWLS_B200_GRAPH calls: an LRU of at most 64 entries per
 * process.  _clear waits for and releases every cached graph (returns how many
 * there were); _count reports the cache size. */
int sgwls_b200_graph_clear(void);
int sgwls_b200_graph_count(void);

#ifdef __cplusplus
}
#endif

#endif /* SGWLS_B200_H */
