/*
 * bp_oracle.c -- CPU ORACLE (test infrastructure only; see bp_oracle.h).
 *
 * A plain-C restatement of the reference's hot path.  Every function names the
 * reference file:line it follows.  The DST-I here is computed through the classic
 * odd extension (one complex FFT of length 2(n+1)) or, for lengths whose 2(n+1) is not a
 * power of two, by the direct O(n^2) sine sum -- deliberately a different algorithm
 * from the CUDA path (half-length FFT + prefix sum), so agreement is evidence.
 */
#include "bp_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static const double kPi = 3.14159265358979323846;
/* proj/src/iterate.cpp:14-16 */
static const double kDivergenceThreshold = 1e8;
static const double kStagnationTol = 1e-14;
static const int kStagnationWindow = 20;
/* proj/include/bp/symbol.hpp:24 */
static const double kSymbolDivGuard = 1e-14;

static char g_err[256] = "";
const char* bpo_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

void bpo_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ------------------------------------------------------------------ 1-D DST-I */

typedef struct {
    int n;       /* DST length */
    int L;       /* 2(n+1) */
    int pow2;    /* L is a power of two */
    bpo_c* tw;   /* L/2 twiddles e^{-2 pi i k / L} (pow2) */
    int* rev;    /* bit reversal (pow2) */
    double* sn;  /* sin(2 pi m / L), m < L (direct path) */
} dst_plan;

static int is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

static void plan_init(dst_plan* pl, int n) {
    memset(pl, 0, sizeof *pl);
    pl->n = n;
    pl->L = 2 * (n + 1);
    pl->pow2 = is_pow2(pl->L);
    if (pl->pow2) {
        const int L = pl->L;
        pl->tw = (bpo_c*)malloc(sizeof(bpo_c) * (size_t)(L / 2));
        for (int k = 0; k < L / 2; ++k) {
            const double a = -2.0 * kPi * k / L;
            pl->tw[k] = cos(a) + I * sin(a);
        }
        pl->rev = (int*)malloc(sizeof(int) * (size_t)L);
        int bits = 0;
        while ((1 << bits) < L) ++bits;
        for (int i = 0; i < L; ++i) {
            int r = 0;
            for (int b = 0; b < bits; ++b)
                if (i & (1 << b)) r |= 1 << (bits - 1 - b);
            pl->rev[i] = r;
        }
    } else {
        pl->sn = (double*)malloc(sizeof(double) * (size_t)pl->L);
        for (int m = 0; m < pl->L; ++m) pl->sn[m] = sin(2.0 * kPi * m / pl->L);
    }
}

static void plan_free(dst_plan* pl) {
    free(pl->tw);
    free(pl->rev);
    free(pl->sn);
}

/* In-place iterative radix-2 DIT FFT, forward sign. */
static void fft_pow2(const dst_plan* pl, bpo_c* z) {
    const int L = pl->L;
    for (int i = 0; i < L; ++i) {
        const int r = pl->rev[i];
        if (r > i) {
            bpo_c t = z[i];
            z[i] = z[r];
            z[r] = t;
        }
    }
    for (int len = 2; len <= L; len <<= 1) {
        const int half = len >> 1, step = L / len;
        for (int s = 0; s < L; s += len) {
            for (int k = 0; k < half; ++k) {
                const bpo_c w = pl->tw[k * step];
                const bpo_c a = z[s + k], b = z[s + k + half] * w;
                z[s + k] = a + b;
                z[s + k + half] = a - b;
            }
        }
    }
}

/* Plain sine sum Y_k = sum_j x_j sin(pi (j+1)(k+1)/(n+1)), strided in/out.
 * Equals FFTW RODFT00 / 2 (proj/src/transforms.cpp:55, scale 0.25 per 2-D at :117). */
static void dst1_strided(const dst_plan* pl, const bpo_c* in, long istride, bpo_c* out,
                         long ostride, bpo_c* work) {
    const int n = pl->n;
    if (pl->pow2) {
        const int L = pl->L;
        work[0] = 0;
        work[n + 1] = 0;
        for (int j = 0; j < n; ++j) {
            work[j + 1] = in[j * istride];
            work[L - 1 - j] = -in[j * istride];
        }
        fft_pow2(pl, work);
        /* Z_k = -2i Y_k  =>  Y_k = (i/2) Z_k */
        for (int k = 0; k < n; ++k) out[k * ostride] = 0.5 * I * work[k + 1];
    } else {
        for (int k = 0; k < n; ++k) {
            bpo_c s = 0;
            for (int j = 0; j < n; ++j) {
                const long m = ((long)(j + 1) * (k + 1)) % pl->L;
                s += in[j * istride] * pl->sn[m];
            }
            work[k] = s;
        }
        for (int k = 0; k < n; ++k) out[k * ostride] = work[k];
    }
}

void bpo_dst1_1d(int n, const double* in_c, double* out_c) {
    dst_plan pl;
    plan_init(&pl, n);
    bpo_c* work = (bpo_c*)malloc(sizeof(bpo_c) * (size_t)(pl.L + n));
    dst1_strided(&pl, (const bpo_c*)in_c, 1, (bpo_c*)out_c, 1, work);
    free(work);
    plan_free(&pl);
}

/* 2-D plain sine transform (rows then columns). */
static void dst2(int nx, int ny, const bpo_c* in, bpo_c* out) {
    dst_plan px, py;
    plan_init(&px, nx);
    plan_init(&py, ny);
    if (out != in) memcpy(out, in, sizeof(bpo_c) * (size_t)nx * ny);
#pragma omp parallel
    {
        bpo_c* work = (bpo_c*)malloc(sizeof(bpo_c) * (size_t)(py.L + ny + px.L + nx));
#pragma omp for schedule(static)
        for (int i = 0; i < nx; ++i)
            dst1_strided(&py, out + (long)i * ny, 1, out + (long)i * ny, 1, work);
#pragma omp for schedule(static)
        for (int j = 0; j < ny; ++j) dst1_strided(&px, out + j, ny, out + j, ny, work);
        free(work);
    }
    plan_free(&px);
    plan_free(&py);
}

/* 3-D plain sine transform, layout [x][y][z] (z contiguous) */
static void dst3(int nx, int ny, int nz, const bpo_c* in, bpo_c* out) {
    dst_plan px, py, pz;
    plan_init(&px, nx);
    plan_init(&py, ny);
    plan_init(&pz, nz);
    const long plane = (long)ny * nz;
    if (out != in) memcpy(out, in, sizeof(bpo_c) * (size_t)nx * plane);
#pragma omp parallel
    {
        bpo_c* work = (bpo_c*)malloc(sizeof(bpo_c) * (size_t)(px.L + nx + py.L + ny + pz.L + nz));
#pragma omp for schedule(static)
        for (long l = 0; l < (long)nx * ny; ++l)
            dst1_strided(&pz, out + l * nz, 1, out + l * nz, 1, work);
#pragma omp for schedule(static)
        for (long l = 0; l < (long)nx * nz; ++l) {
            const long x = l / nz, z = l % nz;
            dst1_strided(&py, out + x * plane + z, nz, out + x * plane + z, nz, work);
        }
#pragma omp for schedule(static)
        for (long l = 0; l < plane; ++l) dst1_strided(&px, out + l, plane, out + l, plane, work);
        free(work);
    }
    plan_free(&px);
    plan_free(&py);
    plan_free(&pz);
}

void bpo_forward_dst3(int nx, int ny, int nz, const double* in_c, double* out_c) {
    dst3(nx, ny, nz, (const bpo_c*)in_c, (bpo_c*)out_c);
}

void bpo_inverse_dst3(int nx, int ny, int nz, const double* in_c, double* out_c) {
    bpo_c* o = (bpo_c*)out_c;
    dst3(nx, ny, nz, (const bpo_c*)in_c, o);
    const double s = 8.0 / ((double)(nx + 1) * (ny + 1) * (nz + 1));
    const long n = (long)nx * ny * nz;
    for (long i = 0; i < n; ++i) o[i] = s * o[i];
}

/* ------------------------------------------------------------------ periodic FFT */
/* length-n complex DFT, sign -1 forward / +1 backward, unnormalized; radix-2 for powers of two,
 * direct sum otherwise */
static void dft1_strided(int n, int sign, const bpo_c* twf, const int* rev, bpo_c* z, long stride,
                         bpo_c* work) {
    for (int i = 0; i < n; ++i) work[i] = z[i * stride];
    if (rev) {
        for (int i = 0; i < n; ++i) {
            const int r = rev[i];
            if (r > i) {
                bpo_c t = work[i];
                work[i] = work[r];
                work[r] = t;
            }
        }
        for (int len = 2; len <= n; len <<= 1) {
            const int half = len >> 1, step = n / len;
            for (int s0 = 0; s0 < n; s0 += len)
                for (int k = 0; k < half; ++k) {
                    bpo_c w = twf[k * step];
                    if (sign > 0) w = conj(w);
                    const bpo_c a = work[s0 + k], b = work[s0 + k + half] * w;
                    work[s0 + k] = a + b;
                    work[s0 + k + half] = a - b;
                }
        }
        for (int i = 0; i < n; ++i) z[i * stride] = work[i];
    } else {
        for (int k = 0; k < n; ++k) {
            bpo_c acc = 0;
            for (int j = 0; j < n; ++j) {
                bpo_c w = twf[(long)j * k % n];
                if (sign > 0) w = conj(w);
                acc += work[j] * w;
            }
            z[k * stride] = acc;
        }
    }
}

static void fft_tables(int n, bpo_c** twf, int** rev) {
    *twf = (bpo_c*)malloc(sizeof(bpo_c) * (size_t)n);
    for (int k = 0; k < n; ++k) (*twf)[k] = cos(-2.0 * kPi * k / n) + I * sin(-2.0 * kPi * k / n);
    *rev = NULL;
    if (is_pow2(n)) {
        int bits = 0;
        while ((1 << bits) < n) ++bits;
        *rev = (int*)malloc(sizeof(int) * (size_t)n);
        for (int i = 0; i < n; ++i) {
            int r = 0;
            for (int b = 0; b < bits; ++b)
                if (i & (1 << b)) r |= 1 << (bits - 1 - b);
            (*rev)[i] = r;
        }
    }
}

/* 2-D DFT: forward (sign -1) unnormalized, backward (sign +1) unnormalized */
static void fft2(int nx, int ny, int sign, const bpo_c* in, bpo_c* out) {
    bpo_c *twx, *twy;
    int *rvx, *rvy;
    fft_tables(nx, &twx, &rvx);
    fft_tables(ny, &twy, &rvy);
    if (out != in) memcpy(out, in, sizeof(bpo_c) * (size_t)nx * ny);
#pragma omp parallel
    {
        bpo_c* work = (bpo_c*)malloc(sizeof(bpo_c) * (size_t)(nx > ny ? nx : ny));
#pragma omp for schedule(static)
        for (int i = 0; i < nx; ++i) dft1_strided(ny, sign, twy, rvy, out + (long)i * ny, 1, work);
#pragma omp for schedule(static)
        for (int j = 0; j < ny; ++j) dft1_strided(nx, sign, twx, rvx, out + j, ny, work);
        free(work);
    }
    free(twx);
    free(twy);
    free(rvx);
    free(rvy);
}

void bpo_fft2(int nx, int ny, int sign, const double* in_c, double* out_c) {
    fft2(nx, ny, sign, (const bpo_c*)in_c, (bpo_c*)out_c);
}

/* ------------------------------------------------------------------ DCT-II / DCT-III */
/* REDFT10 Y_k = 2 sum x_j cos(pi (j+1/2) k / n) and REDFT01 Y_k = x_0 + 2 sum_{j>=1} x_j
 * cos(pi j (k+1/2)/n) via the even/odd extension to a length-4n DFT (real-linear, so complex
 * inputs transform component-wise). */
static void dct1_strided(int n, int inverse, const bpo_c* tw4, const int* rev4, bpo_c* x, long stride,
                         bpo_c* z, bpo_c* work) {
    const int L = 4 * n;
    for (int i = 0; i < L; ++i) z[i] = 0;
    if (!inverse) {
        for (int j = 0; j < n; ++j) {
            z[2 * j + 1] = x[j * stride];
            z[L - 2 * j - 1] = x[j * stride];
        }
    } else {
        for (int j = 0; j < n; ++j) {
            z[j] = x[j * stride];
            if (j > 0) z[L - j] = x[j * stride];
        }
    }
    dft1_strided(L, -1, tw4, rev4, z, 1, work);
    for (int k = 0; k < n; ++k) x[k * stride] = inverse ? z[2 * k + 1] : z[k];
}

void bpo_dct2(int nx, int ny, int inverse, const double* in_c, double* out_c) {
    bpo_c* out = (bpo_c*)out_c;
    if ((const double*)out_c != in_c) memcpy(out, in_c, sizeof(bpo_c) * (size_t)nx * ny);
    bpo_c *twx, *twy;
    int *rvx, *rvy;
    fft_tables(4 * nx, &twx, &rvx);
    fft_tables(4 * ny, &twy, &rvy);
    const int L = 4 * (nx > ny ? nx : ny);
#pragma omp parallel
    {
        bpo_c* z = (bpo_c*)malloc(sizeof(bpo_c) * (size_t)L * 2);
#pragma omp for schedule(static)
        for (int i = 0; i < nx; ++i) dct1_strided(ny, inverse, twy, rvy, out + (long)i * ny, 1, z, z + L);
#pragma omp for schedule(static)
        for (int j = 0; j < ny; ++j) dct1_strided(nx, inverse, twx, rvx, out + j, ny, z, z + L);
        free(z);
    }
    free(twx);
    free(twy);
    free(rvx);
    free(rvy);
}

/* forward_transform(DST1): RODFT00 then x0.25 == plain sine sum (proj/src/transforms.cpp:111-118) */
void bpo_forward_dst(int nx, int ny, const double* in_c, double* out_c) {
    dst2(nx, ny, (const bpo_c*)in_c, (bpo_c*)out_c);
}

/* inverse_transform(DST1): RODFT00 x0.25 then x 4/((nx+1)(ny+1)) (proj/src/transforms.cpp:127-148) */
void bpo_inverse_dst(int nx, int ny, const double* in_c, double* out_c) {
    bpo_c* o = (bpo_c*)out_c;
    dst2(nx, ny, (const bpo_c*)in_c, o);
    const double s = 4.0 / ((double)(nx + 1) * (ny + 1));
    const long n = (long)nx * ny;
    for (long i = 0; i < n; ++i) o[i] = s * o[i];
}

/* ------------------------------------------------------------------ problem */

static long npts(const bpo_problem* p) { return (long)p->nx * p->ny * p->nz; }

/* forward_transform / inverse_transform in the problem's basis (transforms.cpp:105-148) */
static void dstn(const bpo_problem* p, const bpo_c* in, bpo_c* out) {
    if (p->cdr) bpo_dct2(p->nx, p->ny, 0, (const double*)in, (double*)out);
    else if (p->periodic) fft2(p->nx, p->ny, -1, in, out);
    else if (p->nz > 1) dst3(p->nx, p->ny, p->nz, in, out);
    else dst2(p->nx, p->ny, in, out);
}

static void inverse_n(const bpo_problem* p, const bpo_c* in, bpo_c* out) {
    if (p->cdr) {
        bpo_dct2(p->nx, p->ny, 1, (const double*)in, (double*)out);
        const double s = 1.0 / (4.0 * (double)p->nx * p->ny);  /* transforms.cpp:100 */
        const long n = (long)p->nx * p->ny;
        for (long i = 0; i < n; ++i) out[i] = s * out[i];
    } else if (p->periodic) {
        fft2(p->nx, p->ny, +1, in, out);
        const double s = 1.0 / ((double)p->nx * p->ny);
        const long n = (long)p->nx * p->ny;
        for (long i = 0; i < n; ++i) out[i] = s * out[i];
    } else if (p->nz > 1) {
        bpo_inverse_dst3(p->nx, p->ny, p->nz, (const double*)in, (double*)out);
    } else {
        bpo_inverse_dst(p->nx, p->ny, (const double*)in, (double*)out);
    }
}

double bpo_norm2(int n, const double* x) {
    /* serial kernels::norm2sq (proj/src/kernels.cpp:38-42) */
    double s = 0.0;
    for (long i = 0; i < 2L * n; i += 2) s += x[i] * x[i] + x[i + 1] * x[i + 1];
    return sqrt(s);
}

static double norm2sq_c(long n, const bpo_c* a) {
    double s = 0.0;
    for (long i = 0; i < n; ++i) s += creal(a[i]) * creal(a[i]) + cimag(a[i]) * cimag(a[i]);
    return s;
}

static bpo_c dotc_c(long n, const bpo_c* a, const bpo_c* b) {
    /* kernels::dotc: sum conj(a) b (proj/src/kernels.cpp:44-48) */
    bpo_c s = 0;
    for (long i = 0; i < n; ++i) s += conj(a[i]) * b[i];
    return s;
}

int bpo_problem_create(int nx, int ny, double lx, double ly, const double* k2_c, double k0,
                       double eta, bpo_problem** out) {
    *out = NULL;
    /* validate(GridSpec) proj/include/bp/grid.hpp:45-50 */
    if (nx < 2 || ny < 2) return fail(BPO_EINVAL, "GridSpec: nx,ny must be >= 2");
    if (!(lx > 0.0) || !(ly > 0.0)) return fail(BPO_EINVAL, "GridSpec: lx,ly must be > 0");
    /* proj/src/helmholtz.cpp:18 */
    if (!(eta > 0.0)) return fail(BPO_EINVAL, "HelmholtzProblem: eta must be > 0");
    const long n = (long)nx * ny;
    const bpo_c* k2 = (const bpo_c*)k2_c;
    for (long i = 0; i < n; ++i)
        if (!isfinite(creal(k2[i])) || !isfinite(cimag(k2[i])))
            return fail(BPO_EINVAL, "HelmholtzProblem: k2 not finite");
    bpo_problem* p = (bpo_problem*)calloc(1, sizeof *p);
    p->nx = nx;
    p->ny = ny;
    p->nz = 1;
    p->lx = lx;
    p->ly = ly;
    p->k0 = k0;
    p->eta = eta;
    p->k2 = (bpo_c*)malloc(sizeof(bpo_c) * n);
    p->v = (bpo_c*)malloc(sizeof(bpo_c) * n);
    p->lambda = (bpo_c*)malloc(sizeof(bpo_c) * n);
    memcpy(p->k2, k2, sizeof(bpo_c) * n);
    /* v_coeff = k2 - (k0^2 + i eta)   proj/src/helmholtz.cpp:22-24 */
    const bpo_c shift = k0 * k0 + I * eta;
    for (long i = 0; i < n; ++i) p->v[i] = p->k2[i] - shift;
    /* laplacian_symbol DirichletInterior (proj/src/symbol.cpp:69-80), then
     * shift_symbol(-cplx(k0^2, eta)) (proj/src/symbol.cpp:97-100, helmholtz.cpp:12) */
    const double hx = lx / (nx + 1), hy = ly / (ny + 1);
    const double ax = 4.0 / (hx * hx), ay = 4.0 / (hy * hy);
    const bpo_c c = -(k0 * k0 + I * eta);
    double mn = INFINITY, mx = 0.0;
    for (int pp = 0; pp < nx; ++pp) {
        const double sx = sin((pp + 1) * kPi / (2.0 * (nx + 1)));
        for (int q = 0; q < ny; ++q) {
            const double sy = sin((q + 1) * kPi / (2.0 * (ny + 1)));
            const bpo_c v = (ax * sx * sx + ay * sy * sy) + c;
            p->lambda[(long)pp * ny + q] = v;
            const double a = cabs(v);
            if (a < mn) mn = a;
            if (a > mx) mx = a;
        }
    }
    /* check_invertible (proj/src/symbol.cpp:102-111) */
    if (mn < kSymbolDivGuard * mx) {
        bpo_problem_destroy(p);
        return fail(BPO_ERUNTIME, "symbol has a (near-)zero entry; reference operator not invertible");
    }
    *out = p;
    return BPO_OK;
}

int bpo_problem_create_periodic(int nx, int ny, double lx, double ly, const double* k2_c,
                                double k0, double eta, bpo_problem** out) {
    int rc = bpo_problem_create(nx, ny, lx, ly, k2_c, k0, eta, out);
    if (rc) return rc;
    bpo_problem* p = *out;
    p->periodic = 1;
    /* laplacian_symbol Periodic: |xi|^2 with xi = 2 pi m / L, m in FFT order
     * (symbol.cpp:58-67, grid.hpp:67-85), shifted by -(k0^2 + i eta) */
    const bpo_c c = -(k0 * k0 + I * eta);
    double mn = INFINITY, mx = 0.0;
    for (int i = 0; i < nx; ++i) {
        const int mi = (i < (nx + 1) / 2) ? i : i - nx;
        const double xi = 2.0 * kPi * mi / lx;
        for (int j = 0; j < ny; ++j) {
            const int mj = (j < (ny + 1) / 2) ? j : j - ny;
            const double yj = 2.0 * kPi * mj / ly;
            const bpo_c v = (xi * xi + yj * yj) + c;
            p->lambda[(long)i * ny + j] = v;
            const double a = cabs(v);
            if (a < mn) mn = a;
            if (a > mx) mx = a;
        }
    }
    if (mn < kSymbolDivGuard * mx) {
        bpo_problem_destroy(p);
        *out = NULL;
        return fail(BPO_ERUNTIME, "symbol has a (near-)zero entry; reference operator not invertible");
    }
    return BPO_OK;
}

int bpo_problem_create_cdr(int nx, int ny, double lx, double ly, const double* bx,
                           const double* by, const double* sigma, double sigma0,
                           bpo_problem** out) {
    *out = NULL;
    if (nx < 2 || ny < 2) return fail(BPO_EINVAL, "GridSpec: nx,ny must be >= 2");
    if (!(lx > 0.0) || !(ly > 0.0)) return fail(BPO_EINVAL, "GridSpec: lx,ly must be > 0");
    const long n = (long)nx * ny;
    bpo_problem* p = (bpo_problem*)calloc(1, sizeof *p);
    p->nx = nx;
    p->ny = ny;
    p->nz = 1;
    p->cdr = 1;
    p->lx = lx;
    p->ly = ly;
    p->sigma0 = sigma0;
    p->eta = 1.0;
    p->bx = (double*)malloc(sizeof(double) * n);
    p->by = (double*)malloc(sizeof(double) * n);
    p->sigma = (double*)malloc(sizeof(double) * n);
    memcpy(p->bx, bx, sizeof(double) * n);
    memcpy(p->by, by, sizeof(double) * n);
    memcpy(p->sigma, sigma, sizeof(double) * n);
    p->k2 = (bpo_c*)calloc(n, sizeof(bpo_c));
    p->v = (bpo_c*)calloc(n, sizeof(bpo_c));
    p->lambda = (bpo_c*)malloc(sizeof(bpo_c) * n);
    /* Neumann five-point symbol (symbol.cpp:81-92) + sigma0 */
    const double hx = lx / nx, hy = ly / ny;
    const double ax = 4.0 / (hx * hx), ay = 4.0 / (hy * hy);
    double mn = INFINITY, mx = 0.0;
    for (int q = 0; q < nx; ++q) {
        const double sx = sin(q * kPi / (2.0 * nx));
        for (int r = 0; r < ny; ++r) {
            const double sy = sin(r * kPi / (2.0 * ny));
            const double v = (ax * sx * sx + ay * sy * sy) + sigma0;
            p->lambda[(long)q * ny + r] = v;
            if (fabs(v) < mn) mn = fabs(v);
            if (fabs(v) > mx) mx = fabs(v);
        }
    }
    if (mn < kSymbolDivGuard * mx) {
        bpo_problem_destroy(p);
        return fail(BPO_ERUNTIME, "symbol has a (near-)zero entry; reference operator not invertible");
    }
    *out = p;
    return BPO_OK;
}

/* c4 operators on complex arrays with zero imaginary part.
 *   Lap_N u: (sum of reflective-ghost neighbours - 4u)/h^2
 *   conv u : bx * (upwind x difference) + by * (upwind y difference)   (first-order upwind) */
static void cdr_parts(const bpo_problem* p, const bpo_c* u, bpo_c* lap, bpo_c* conv) {
    const int nx = p->nx, ny = p->ny;
    const double h = p->lx / nx, ih = 1.0 / h, ih2 = 1.0 / (h * h);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j) {
            const long k = (long)i * ny + j;
            const bpo_c c = u[k];
            const bpo_c w = i > 0 ? u[k - ny] : c, e = i < nx - 1 ? u[k + ny] : c;
            const bpo_c s = j > 0 ? u[k - 1] : c, nn = j < ny - 1 ? u[k + 1] : c;
            lap[k] = (4.0 * c - w - e - s - nn) * ih2; /* -Lap */
            const double vx = p->bx[k], vy = p->by[k];
            const bpo_c dx = vx >= 0.0 ? (c - w) * ih : (e - c) * ih;
            const bpo_c dy = vy >= 0.0 ? (c - s) * ih : (nn - c) * ih;
            conv[k] = vx * dx + vy * dy;
        }
}

int bpo_problem_create3(int nx, int ny, int nz, double l, const double* k2_c, double k0, double eta,
                        bpo_problem** out) {
    *out = NULL;
    if (nx < 2 || ny < 2 || nz < 2) return fail(BPO_EINVAL, "GridSpec: nx,ny,nz must be >= 2");
    if (!(l > 0.0)) return fail(BPO_EINVAL, "GridSpec: l must be > 0");
    if (!(eta > 0.0)) return fail(BPO_EINVAL, "HelmholtzProblem: eta must be > 0");
    if (nx != ny || ny != nz) return fail(BPO_EINVAL, "3-D grid must be cubic (hx == hy == hz)");
    const long n = (long)nx * ny * nz;
    const bpo_c* k2 = (const bpo_c*)k2_c;
    for (long i = 0; i < n; ++i)
        if (!isfinite(creal(k2[i])) || !isfinite(cimag(k2[i])))
            return fail(BPO_EINVAL, "HelmholtzProblem: k2 not finite");
    bpo_problem* p = (bpo_problem*)calloc(1, sizeof *p);
    p->nx = nx;
    p->ny = ny;
    p->nz = nz;
    p->lx = l;
    p->ly = l;
    p->k0 = k0;
    p->eta = eta;
    p->k2 = (bpo_c*)malloc(sizeof(bpo_c) * n);
    p->v = (bpo_c*)malloc(sizeof(bpo_c) * n);
    p->lambda = (bpo_c*)malloc(sizeof(bpo_c) * n);
    memcpy(p->k2, k2, sizeof(bpo_c) * n);
    const bpo_c shift = k0 * k0 + I * eta;
    for (long i = 0; i < n; ++i) p->v[i] = p->k2[i] - shift;
    const double h = l / (nx + 1), a = 4.0 / (h * h);
    const bpo_c c = -(k0 * k0 + I * eta);
    double* f1 = (double*)malloc(sizeof(double) * nx);
    for (int q = 0; q < nx; ++q) {
        const double sq = sin((q + 1) * kPi / (2.0 * (nx + 1)));
        f1[q] = a * sq * sq;
    }
    double mn = INFINITY, mx = 0.0;
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j)
            for (int k = 0; k < nz; ++k) {
                const bpo_c v = ((f1[i] + f1[j]) + f1[k]) + c;
                p->lambda[((long)i * ny + j) * nz + k] = v;
                const double av = cabs(v);
                if (av < mn) mn = av;
                if (av > mx) mx = av;
            }
    free(f1);
    if (mn < kSymbolDivGuard * mx) {
        bpo_problem_destroy(p);
        return fail(BPO_ERUNTIME, "symbol has a (near-)zero entry; reference operator not invertible");
    }
    *out = p;
    return BPO_OK;
}

void bpo_problem_destroy(bpo_problem* p) {
    if (!p) return;
    free(p->bx);
    free(p->by);
    free(p->sigma);
    free(p->k2);
    free(p->v);
    free(p->lambda);
    free(p);
}

void bpo_problem_symbol(const bpo_problem* p, double* lambda_c) {
    memcpy(lambda_c, p->lambda, sizeof(bpo_c) * (size_t)npts(p));
}

/* seven-point analogue of kernels::five_point: (6u - six neighbours)/h^2, zero halo */
static void seven_point(const bpo_c* u, int nx, int ny, int nz, double h2, bpo_c* out) {
    const double inv = 1.0 / h2;
    const long plane = (long)ny * nz;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j)
            for (int k = 0; k < nz; ++k) {
                const long c = (long)i * plane + (long)j * nz + k;
                bpo_c s = 6.0 * u[c];
                if (i > 0) s -= u[c - plane];
                if (i < nx - 1) s -= u[c + plane];
                if (j > 0) s -= u[c - nz];
                if (j < ny - 1) s -= u[c + nz];
                if (k > 0) s -= u[c - 1];
                if (k < nz - 1) s -= u[c + 1];
                out[c] = s * inv;
            }
}

/* kernels::five_point serial (proj/src/kernels.cpp:56-69), zero halo, h2 = hx^2 */
static void five_point(const bpo_c* u, int nx, int ny, double h2, bpo_c* out) {
    const double inv = 1.0 / h2;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < nx; ++i) {
        for (int j = 0; j < ny; ++j) {
            const long k = (long)i * ny + j;
            bpo_c s = 4.0 * u[k];
            if (i > 0) s -= u[k - ny];
            if (i < nx - 1) s -= u[k + ny];
            if (j > 0) s -= u[k - 1];
            if (j < ny - 1) s -= u[k + 1];
            out[k] = s * inv;
        }
    }
}

/* A u = five_point(u) - k2 u  (NewtonJacobianProblem::apply_A pattern, newton_problem.cpp:38-44) */
void bpo_apply_A(const bpo_problem* p, const double* u_c, double* out_c) {
    const bpo_c* u = (const bpo_c*)u_c;
    bpo_c* out = (bpo_c*)out_c;
    const long n = npts(p);
    if (p->cdr) {  /* A u = -Lap_N u + b . grad_up u + sigma u */
        bpo_c* conv = (bpo_c*)malloc(sizeof(bpo_c) * n);
        cdr_parts(p, u, out, conv);
        for (long i = 0; i < n; ++i) out[i] = (out[i] + conv[i]) + p->sigma[i] * u[i];
        free(conv);
        return;
    }
    if (p->periodic) {
        /* HelmholtzProblem::apply_A: F^-1(|xi|^2 F u) - k2 u (helmholtz.cpp:27-32) */
        bpo_c* modes = (bpo_c*)malloc(sizeof(bpo_c) * n);
        fft2(p->nx, p->ny, -1, u, modes);
        for (int i = 0; i < p->nx; ++i) {
            const int mi = (i < (p->nx + 1) / 2) ? i : i - p->nx;
            const double xi = 2.0 * kPi * mi / p->lx;
            for (int j = 0; j < p->ny; ++j) {
                const int mj = (j < (p->ny + 1) / 2) ? j : j - p->ny;
                const double yj = 2.0 * kPi * mj / p->ly;
                modes[(long)i * p->ny + j] *= (xi * xi + yj * yj);  /* |xi|^2 */
            }
        }
        inverse_n(p, modes, out);
        free(modes);
        for (long i = 0; i < n; ++i) out[i] -= p->k2[i] * u[i];
        return;
    }
    const double hx = p->lx / (p->nx + 1);
    if (p->nz > 1) seven_point(u, p->nx, p->ny, p->nz, hx * hx, out);
    else five_point(u, p->nx, p->ny, hx * hx, out);
    for (long i = 0; i < n; ++i) out[i] -= p->k2[i] * u[i];
}

/* HelmholtzProblem::apply_V = kernels::mul(u, v_coeff) (proj/src/helmholtz.cpp:34-39) */
void bpo_apply_V(const bpo_problem* p, const double* u_c, double* out_c) {
    const bpo_c* u = (const bpo_c*)u_c;
    bpo_c* out = (bpo_c*)out_c;
    const long n = npts(p);
    if (p->cdr) {  /* V u = (sigma0 - sigma) u - b . grad_up u */
        bpo_c* lap = (bpo_c*)malloc(sizeof(bpo_c) * n);
        cdr_parts(p, u, lap, out);
        for (long i = 0; i < n; ++i) out[i] = (p->sigma0 - p->sigma[i]) * u[i] - out[i];
        free(lap);
        return;
    }
    for (long i = 0; i < n; ++i) out[i] = u[i] * p->v[i];
}

/* Transpose of cdr_parts' upwind convection (a real operator: its adjoint is its transpose).
 * Row k of conv reads u_k and one upwind neighbour per direction; column m therefore collects
 * its own diagonal entries and the rows of the neighbours whose upwind side is m.  Boundary
 * rows whose upwind neighbour is the reflective ghost contribute nothing (c - c = 0). */
static void cdr_conv_transpose(const bpo_problem* p, const bpo_c* y, bpo_c* out) {
    const int nx = p->nx, ny = p->ny;
    const double ih = (double)nx / p->lx;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j) {
            const long k = (long)i * ny + j;
            const double vx = p->bx[k], vy = p->by[k];
            bpo_c t = 0.0;
            if (vx >= 0.0 && i > 0) t += vx * ih * y[k];
            if (vx < 0.0 && i < nx - 1) t -= vx * ih * y[k];
            if (i < nx - 1 && p->bx[k + ny] >= 0.0) t -= p->bx[k + ny] * ih * y[k + ny];
            if (i > 0 && p->bx[k - ny] < 0.0) t += p->bx[k - ny] * ih * y[k - ny];
            if (vy >= 0.0 && j > 0) t += vy * ih * y[k];
            if (vy < 0.0 && j < ny - 1) t -= vy * ih * y[k];
            if (j < ny - 1 && p->by[k + 1] >= 0.0) t -= p->by[k + 1] * ih * y[k + 1];
            if (j > 0 && p->by[k - 1] < 0.0) t += p->by[k - 1] * ih * y[k - 1];
            out[k] = t;
        }
}

/* proj/src/helmholtz.cpp:41-46; CDR (c4): V^H = V^T = (sigma0 - sigma) - conv^T, the role of
 * CdrProblem::apply_V_adjoint (proj/src/cdr.cpp:139-176) for the upwind family */
void bpo_apply_V_adjoint(const bpo_problem* p, const double* u_c, double* out_c) {
    const bpo_c* u = (const bpo_c*)u_c;
    bpo_c* out = (bpo_c*)out_c;
    const long n = npts(p);
    if (p->cdr) {
        cdr_conv_transpose(p, u, out);
        for (long i = 0; i < n; ++i) out[i] = (p->sigma0 - p->sigma[i]) * u[i] - out[i];
        return;
    }
    for (long i = 0; i < n; ++i) out[i] = conj(p->v[i]) * u[i];
}

/* apply_symbol Multiply (proj/src/symbol.cpp:19-39 with op=Multiply) */
void bpo_apply_Lref(const bpo_problem* p, const double* u_c, double* out_c) {
    const long n = npts(p);
    bpo_c* modes = (bpo_c*)malloc(sizeof(bpo_c) * n);
    dstn(p, (const bpo_c*)u_c, modes);
    for (long i = 0; i < n; ++i) modes[i] *= p->lambda[i];
    inverse_n(p, modes, (bpo_c*)out_c);
    free(modes);
}

/* apply_symbol Divide (proj/src/symbol.cpp:19-39): forward, guard scan, divide, inverse */
int bpo_apply_G(const bpo_problem* p, const double* q_c, double* out_c) {
    const long n = npts(p);
    bpo_c* modes = (bpo_c*)malloc(sizeof(bpo_c) * n);
    dstn(p, (const bpo_c*)q_c, modes);
    double mn = cabs(p->lambda[0]), mx = mn;
    for (long i = 0; i < n; ++i) {
        const double a = cabs(p->lambda[i]);
        if (a < mn) mn = a;
        if (a > mx) mx = a;
    }
    if (mn < kSymbolDivGuard * mx) {
        free(modes);
        return fail(BPO_ERUNTIME, "apply_symbol: near-zero symbol entry under division");
    }
    for (long i = 0; i < n; ++i) modes[i] /= p->lambda[i];
    inverse_n(p, modes, (bpo_c*)out_c);
    free(modes);
    return BPO_OK;
}

/* Problem::born_residual = G(V u + f) - u (proj/src/problem.cpp:41-49) */
int bpo_born_residual(const bpo_problem* p, const double* u_c, const double* f_c, double* out_c) {
    const long n = npts(p);
    bpo_c* vu = (bpo_c*)malloc(sizeof(bpo_c) * n);
    bpo_apply_V(p, u_c, (double*)vu);
    const bpo_c* f = (const bpo_c*)f_c;
    for (long i = 0; i < n; ++i) vu[i] = vu[i] + f[i];
    int rc = bpo_apply_G(p, (const double*)vu, out_c);
    bpo_c* out = (bpo_c*)out_c;
    const bpo_c* u = (const bpo_c*)u_c;
    for (long i = 0; i < n; ++i) out[i] = out[i] - u[i];
    free(vu);
    return rc;
}

/* residual = f - A u (proj/src/iterate.cpp:45-50) */
void bpo_residual(const bpo_problem* p, const double* u_c, const double* f_c, double* out_c) {
    const long n = npts(p);
    bpo_c* au = (bpo_c*)malloc(sizeof(bpo_c) * n);
    bpo_apply_A(p, u_c, (double*)au);
    const bpo_c* f = (const bpo_c*)f_c;
    bpo_c* out = (bpo_c*)out_c;
    for (long i = 0; i < n; ++i) out[i] = f[i] - au[i];
    free(au);
}

/* ------------------------------------------------------------------ correction maps */

/* apply_correction (proj/src/correction.cpp:52-76) + optimal scalar (:10-48).
 * BPO_MAP_POINTWISE is the diagonal relaxation gamma(x) = (i/eta) V(x) (PAPER.md:207,
 * Osnabrugge-style CBS); it is linear in x like every reference map. */
static int apply_correction(const bpo_problem* p, const bpo_map* map, const bpo_c* x,
                            const bpo_c* euclid_r, bpo_c* out) {
    const long n = npts(p);
    switch (map->kind) {
        case BPO_MAP_SCALAR: {
            const bpo_c g = map->gamma_re + I * map->gamma_im;
            for (long i = 0; i < n; ++i) out[i] = g * x[i];
            return BPO_OK;
        }
        case BPO_MAP_OPTIMAL_SCALAR: {
            bpo_c* w = (bpo_c*)malloc(sizeof(bpo_c) * n);
            bpo_c gamma = 0;
            double denom;
            if (map->metric == BPO_METRIC_EUCLIDEAN) {
                bpo_apply_A(p, (const double*)x, (double*)w);
                denom = norm2sq_c(n, w);
                if (denom <= 0.0 || !isfinite(denom)) gamma = 0;
                else gamma = dotc_c(n, w, euclid_r) / denom;
            } else {
                bpo_c* vx = (bpo_c*)malloc(sizeof(bpo_c) * n);
                bpo_apply_V(p, (const double*)x, (double*)vx);
                int rc = bpo_apply_G(p, (const double*)vx, (double*)w);
                free(vx);
                if (rc) {
                    free(w);
                    return rc;
                }
                for (long i = 0; i < n; ++i) w[i] = x[i] - w[i];
                denom = norm2sq_c(n, w);
                if (denom <= 0.0 || !isfinite(denom)) gamma = 0;
                else gamma = dotc_c(n, w, x) / denom;
            }
            free(w);
            for (long i = 0; i < n; ++i) out[i] = gamma * x[i];
            return BPO_OK;
        }
        case BPO_MAP_FOURIER_DIAG: {
            if (!map->m) return fail(BPO_EINVAL, "FourierDiag correction: shape mismatch");
            const bpo_c* m = (const bpo_c*)map->m;
            bpo_c* modes = (bpo_c*)malloc(sizeof(bpo_c) * n);
            dstn(p, x, modes);
            for (long i = 0; i < n; ++i) modes[i] = modes[i] * m[i];
            inverse_n(p, modes, out);
            free(modes);
            return BPO_OK;
        }
        case BPO_MAP_POINTWISE: {
            for (long i = 0; i < n; ++i) out[i] = ((I / p->eta) * p->v[i]) * x[i];
            return BPO_OK;
        }
        default: return fail(BPO_EINVAL, "unknown correction map");
    }
}

/* ------------------------------------------------------------------ driver */

/* bp::run (proj/src/iterate.cpp:88-153) */
int bpo_run(const bpo_problem* p, const bpo_map* map, const double* f_c, int format, double rtol,
            int max_iters, const double* u0_c, double* u_out_c, double* res_l2, double* res_reta,
            bpo_trace* info, double* snapshots, int n_snap) {
    if (!(rtol > 0.0 && rtol < 1.0)) return fail(BPO_EINVAL, "run: rtol must lie in (0,1)");
    if (max_iters < 1) return fail(BPO_EINVAL, "run: max_iters must be >= 1");
    const long n = npts(p);
    const bpo_c* f = (const bpo_c*)f_c;
    const double fnorm = sqrt(norm2sq_c(n, f));
    if (fnorm <= 0.0) return fail(BPO_EINVAL, "run: zero source");

    bpo_c* u = (bpo_c*)u_out_c;
    if (u0_c) memcpy(u, u0_c, sizeof(bpo_c) * n);
    else memset(u, 0, sizeof(bpo_c) * n);
    if (snapshots && n_snap > 0) memcpy(snapshots, u, sizeof(bpo_c) * n);

    bpo_c* r = (bpo_c*)malloc(sizeof(bpo_c) * n);
    bpo_c* gr = (bpo_c*)malloc(sizeof(bpo_c) * n);
    bpo_c* dir = (bpo_c*)malloc(sizeof(bpo_c) * n);
    bpo_c* du = (bpo_c*)malloc(sizeof(bpo_c) * n);
    int rc = BPO_OK;

    info->fnorm_l2 = fnorm;
    rc = bpo_apply_G(p, f_c, (double*)gr);
    if (rc) goto done;
    info->fnorm_reta = sqrt(norm2sq_c(n, gr));
    info->terminated = BPO_TERM_MAXITERS;
    info->iters = 0;

    int count = 0;
    bpo_residual(p, (const double*)u, f_c, (double*)r);
    rc = bpo_apply_G(p, (const double*)r, (double*)gr);
    if (rc) goto done;
    res_l2[count] = sqrt(norm2sq_c(n, r)) / info->fnorm_l2;
    res_reta[count] = sqrt(norm2sq_c(n, gr)) / info->fnorm_reta;
    ++count;
    if (res_l2[0] <= rtol) {
        info->terminated = BPO_TERM_CONVERGED;
        goto done;
    }

    for (int it = 0; it < max_iters; ++it) {
        switch (format) {
            case BPO_FMT_DIRECT: memcpy(dir, r, sizeof(bpo_c) * n); break;
            case BPO_FMT_CBS: memcpy(dir, gr, sizeof(bpo_c) * n); break;
            case BPO_FMT_NPBS:
                rc = bpo_born_residual(p, (const double*)u, f_c, (double*)dir);
                if (rc) goto done;
                break;
            default: rc = fail(BPO_EINVAL, "unknown iteration format"); goto done;
        }
        rc = apply_correction(p, map, dir, r, du);
        if (rc) goto done;
        for (long i = 0; i < n; ++i) u[i] = u[i] + du[i];
        info->iters = it + 1;
        if (snapshots && it + 1 < n_snap) memcpy(snapshots + 2 * n * (it + 1), u, sizeof(bpo_c) * n);

        bpo_residual(p, (const double*)u, f_c, (double*)r);
        rc = bpo_apply_G(p, (const double*)r, (double*)gr);
        if (rc) goto done;
        res_l2[count] = sqrt(norm2sq_c(n, r)) / info->fnorm_l2;
        res_reta[count] = sqrt(norm2sq_c(n, gr)) / info->fnorm_reta;
        ++count;

        const double rel = res_l2[count - 1];
        if (!isfinite(rel) || rel > kDivergenceThreshold) {
            info->terminated = BPO_TERM_DIVERGED;
            goto done;
        }
        if (rel <= rtol) {
            info->terminated = BPO_TERM_CONVERGED;
            goto done;
        }
        if (count > kStagnationWindow) {
            const double past = res_l2[count - 1 - kStagnationWindow];
            if (fabs(past - rel) < kStagnationTol * fmax(1.0, past)) {
                info->terminated = BPO_TERM_STAGNATED;
                goto done;
            }
        }
    }
done:
    free(r);
    free(gr);
    free(dir);
    free(du);
    return rc;
}
