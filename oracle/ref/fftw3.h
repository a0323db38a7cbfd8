/*
 * fftw3.h -- project-owned FFTW-API shim header (ORACLE infrastructure only).
 *
 * FFTW3 is not available in this image (no headers, no library, no network), so the
 * reference's own transform layer (proj/src/transforms.cpp) is compiled against this
 * declaration set and linked with oracle/ref/fftw_shim.c, which implements exactly the
 * five entry points the reference calls (proj/src/transforms.cpp:50-60,70,84-85,160)
 * with FFTW's documented transform definitions:
 *   FFTW_FORWARD  DFT   Y_k = sum x_j exp(-2 pi i jk/n)          (unnormalized)
 *   FFTW_BACKWARD DFT   Y_k = sum x_j exp(+2 pi i jk/n)
 *   FFTW_RODFT00  DST-I Y_k = 2 sum x_j sin(pi (j+1)(k+1)/(n+1))
 *   FFTW_REDFT10  DCT-II Y_k = 2 sum x_j cos(pi (j+1/2) k / n)
 *   FFTW_REDFT01  DCT-III Y_k = x_0 + 2 sum_{j>=1} x_j cos(pi j (k+1/2) / n)
 * The shim is NOT FFTW: any CPU timing taken through it says so.
 */
#ifndef BP_FFTW3_SHIM_H
#define BP_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct bp_fftw_plan_s* fftw_plan;

typedef enum {
    FFTW_R2HC = 0,
    FFTW_HC2R = 1,
    FFTW_DHT = 2,
    FFTW_REDFT00 = 3,
    FFTW_REDFT01 = 4,
    FFTW_REDFT10 = 5,
    FFTW_REDFT11 = 6,
    FFTW_RODFT00 = 7,
    FFTW_RODFT01 = 8,
    FFTW_RODFT10 = 9,
    FFTW_RODFT11 = 10
} fftw_r2r_kind;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_DESTROY_INPUT (1U << 0)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
fftw_plan fftw_plan_r2r_2d(int n0, int n1, double* in, double* out, fftw_r2r_kind kind0,
                           fftw_r2r_kind kind1, unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_execute_r2r(const fftw_plan p, double* in, double* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
