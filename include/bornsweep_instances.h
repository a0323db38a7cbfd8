/*
 * bornsweep_instances.h -- seeded synthetic Helmholtz instances (host-only C ABI,
 * libbornsweep_host.so).
 *
 * BASELINE.json's configs are synthetic: media are Gaussian-smoothed seeded white noise,
 * sources are Gaussian bumps.  Every arm (CUDA path, plain-C oracle, the reference's own
 * code in oracle/_ref) consumes the SAME arrays produced here, so "same seeded inputs"
 * holds by construction.  Randomness uses the reference's RngState
 * (proj/include/bp/rng.hpp:10-62: mt19937_64 seeded through splitmix64, split(index),
 * Box-Muller normals); the sponge and the bump follow proj/src/samplers.cpp:86-105,130-150
 * and make_helmholtz's damping fold (proj/src/helmholtz.cpp:62-87).  tests/ pin all three
 * against the reference build.
 *
 * Layout of every field: DirichletInterior, N = n-1 points per side, h = 1/n,
 * row-major x slow (data[ix*N + iy]), complex interleaved re/im.
 */
#ifndef BORNSWEEP_INSTANCES_H
#define BORNSWEEP_INSTANCES_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t n;              /* cells per side; N = n-1 interior points, h = 1/n            */
    double ppw;             /* points per wavelength at c = 1: omega = 2 pi / (ppw h)       */
    double contrast;        /* c = 1 + contrast * g, g in [-1, 1]                           */
    double sigma_cells;     /* Gaussian smoothing of the white noise, in cells (trunc 4 sigma) */
    double src_sigma_cells; /* source bump width, in cells                                 */
    int32_t n_sources;      /* 0: one unit bump at the centre; >0: seeded uniform positions */
    uint64_t seed;          /* member b uses RngState(seed).split(b)                        */
    int32_t sponge_points;  /* -1: reference default N/8 (proj/src/helmholtz.cpp:67)        */
    double sponge_strength; /* reference default 1.0                                        */
    double eta_factor;      /* eta = eta_factor * max|k2_damped - k0^2|                     */
    int32_t dim;            /* 2 (default when 0) or 3: N^3 cube, 3-D smoothing / sponge / bump */
} bp_instance_spec;

/* Members first..first+count-1 into k2/f (count x N^dim complex) and k0/eta (count). */
int bp_make_instances(const bp_instance_spec* spec, int64_t first, int32_t count, double* k2,
                      double* f, double* k0, double* eta, int32_t nthreads);

/* Config c4: convection-diffusion-reaction media on the Neumann cell-centred n x n grid
 * (h = 1/n).  Four seeded white-noise fields (sigma, bx, by, f, in that order) are Gaussian-
 * smoothed with reflective padding (truncated at 3 sigma) and normalised to unit max-abs:
 * sigma = smax/2 (1 + g_s) in [0, smax], b = bmax/sqrt(2) (g_x, g_y) (|b| <= bmax), f = g_f;
 * sigma0 = mean sigma (the reference's CDR default, proj/src/cdr.cpp:215). */
typedef struct {
    int32_t n;             /* points per side (cell-centred) */
    double b_max;          /* 20 */
    double sigma_max;      /* 50 */
    double smooth_cells;   /* medium smoothing sigma in cells (<= 0: n/16) */
    double src_smooth_cells; /* source smoothing sigma in cells (<= 0: n/32) */
    uint64_t seed;
} bp_cdr_spec;

int bp_make_cdr_instances(const bp_cdr_spec* spec, int64_t first, int32_t count, double* bx,
                          double* by, double* sigma, double* sigma0, double* f, int32_t nthreads);

/* The building blocks, exported for the pins in tests/. */
void bp_rng_normals(uint64_t seed, int64_t index, int32_t count, double* out);
void bp_rng_uniforms(uint64_t seed, int64_t index, int32_t count, double* out);
void bp_sponge_profile(int32_t nx, int32_t ny, int32_t layer, double strength, double* out);
void bp_gaussian_bump(int32_t nx, int32_t ny, double lx, double ly, double cx, double cy,
                      double width, double amplitude, double* out);
void bp_gaussian_smooth(int32_t nx, int32_t ny, double sigma_cells, const double* in, double* out);

#ifdef __cplusplus
}
#endif

#endif
