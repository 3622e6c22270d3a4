/* TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference SG-WLS path.
 * See sgwls_oracle.c for the parity contract.  Not linked by the product. */
#pragma once
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Field-for-field mirror of sgwls::SmoothConfig + sgwls::WeightParams
 * (proj/include/sgwls/smoother.hpp:12-24, proj/include/sgwls/weights.hpp:14-27). */
typedef struct oracle_config {
    double lambda;
    int r;
    int tau;
    int iterations;
    int first_axis; /* 0 = Column, 1 = Row */
    int threads;
    int kind;       /* 0 = Frac, 1 = Exp */
    double alpha_s, alpha_r, sigma_s, sigma_r, epsilon, guidance_scale;
} oracle_config;

void oracle_config_default(oracle_config* c);
int oracle_validate(const oracle_config* c, char* err, size_t errlen);
int oracle_band_centers(int extent, int r, int tau, int* out, int cap);
int oracle_band_layout(int height, int width, int center, int r, int axis, int* rows, int* cols);
int oracle_edge_weights(const double* guidance, int width, int height, int gch, int center, int r, int axis,
                        const oracle_config* cfg, double* w);
int oracle_solve_band(int n, int r, const double* w, double lambda, const double* rhs, double* u,
                      double* alpha_out, double* beta_out, double* gamma_out);
int oracle_solve_system(int n, int r, const double* diag, const double* off, const double* rhs, double* u,
                        double* alpha_out, double* beta_out, double* gamma_out);
int oracle_smooth_f64(const double* target, int width, int height, int channels, const double* guidance,
                      int guidance_channels, const oracle_config* cfg, double* out, char* err, size_t errlen);
int oracle_smooth_f32(const float* target, int width, int height, int channels, const float* guidance,
                      int guidance_channels, const oracle_config* cfg, double* out, char* err, size_t errlen);
int oracle_interpolate_sparse_f32(const float* values, int width, int height, int channels, const float* mask,
                                  const float* guidance, int guidance_channels, const oracle_config* cfg,
                                  double* out, double* undefined_mask, char* err, size_t errlen);

#ifdef __cplusplus
}
#endif
