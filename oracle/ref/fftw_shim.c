/*
 * fftw_shim.c -- project-owned implementation of the five FFTW entry points the
 * reference's transform layer uses (ORACLE infrastructure; see fftw3.h).
 *
 * Power-of-two embedding lengths go through an iterative radix-2 complex FFT; two real
 * rows share one complex FFT (their embeddings are real-even or real-odd, so the real and
 * imaginary parts of the packed transform separate exactly).  Other lengths evaluate the
 * defining sums directly (O(n^2)).  Plans are immutable after creation and execution is
 * reentrant, matching how proj/src/transforms.cpp:25-65 uses FFTW (planning under a mutex,
 * execution from many OpenMP threads, proj/src/bench.cpp:143-151).
 */
#include "fftw3.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef double _Complex cpx;
static const double kPi = 3.14159265358979323846;

/* ---- 1-D complex FFT tables -------------------------------------------------------- */
typedef struct {
    int L;      /* transform length */
    int pow2;
    cpx* tw;    /* e^{-2 pi i k/L}, k < L (full table; also serves the direct path) */
    int* rev;
} fft1;

static int is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

static void fft1_init(fft1* t, int L) {
    t->L = L;
    t->pow2 = is_pow2(L);
    t->tw = (cpx*)malloc(sizeof(cpx) * (size_t)L);
    for (int k = 0; k < L; ++k) {
        const double a = -2.0 * kPi * (double)k / (double)L;
        t->tw[k] = cos(a) + I * sin(a);
    }
    t->rev = NULL;
    if (t->pow2) {
        t->rev = (int*)malloc(sizeof(int) * (size_t)L);
        int bits = 0;
        while ((1 << bits) < L) ++bits;
        for (int i = 0; i < L; ++i) {
            int r = 0;
            for (int b = 0; b < bits; ++b)
                if (i & (1 << b)) r |= 1 << (bits - 1 - b);
            t->rev[i] = r;
        }
    }
}

static void fft1_free(fft1* t) {
    free(t->tw);
    free(t->rev);
}

/* forward (sign -1) or backward (sign +1) unnormalized DFT in place; work: L entries */
static void fft1_exec(const fft1* t, cpx* z, int sign, cpx* work) {
    const int L = t->L;
    if (t->pow2) {
        for (int i = 0; i < L; ++i) {
            const int r = t->rev[i];
            if (r > i) {
                cpx s = z[i];
                z[i] = z[r];
                z[r] = s;
            }
        }
        for (int len = 2; len <= L; len <<= 1) {
            const int half = len >> 1, step = L / len;
            for (int s = 0; s < L; s += len) {
                cpx* a = z + s;
                cpx* b = z + s + half;
                for (int k = 0; k < half; ++k) {
                    cpx w = t->tw[k * step];
                    if (sign > 0) w = conj(w);
                    const cpx x = a[k], y = b[k] * w;
                    a[k] = x + y;
                    b[k] = x - y;
                }
            }
        }
    } else {
        for (int k = 0; k < L; ++k) {
            cpx s = 0;
            for (int j = 0; j < L; ++j) {
                cpx w = t->tw[(int)(((long)j * k) % L)];
                if (sign > 0) w = conj(w);
                s += z[j] * w;
            }
            work[k] = s;
        }
        memcpy(z, work, sizeof(cpx) * (size_t)L);
    }
}

/* ---- 1-D real-to-real kinds via complex embeddings ---------------------------------- */
typedef struct {
    int kind; /* fftw_r2r_kind or -1 for c2c */
    int n;
    fft1 f;   /* embedding FFT: RODFT00 2(n+1), REDFT10/01 4n, c2c n */
} dim_plan;

static void dim_init(dim_plan* d, int kind, int n) {
    d->kind = kind;
    d->n = n;
    int L = n;
    if (kind == FFTW_RODFT00) L = 2 * (n + 1);
    else if (kind == FFTW_REDFT10 || kind == FFTW_REDFT01) L = 4 * n;
    fft1_init(&d->f, L);
}

/* Apply a real kind to two real rows a, b (b may be NULL) of length n, in place. */
static void r2r_pair(const dim_plan* d, double* a, long sa, double* b, long sb, cpx* z,
                     cpx* work) {
    const int n = d->n, L = d->f.L;
    memset(z, 0, sizeof(cpx) * (size_t)L);
#define VAL(j) (a[(long)(j) * sa] + I * (b ? b[(long)(j) * sb] : 0.0))
    switch (d->kind) {
        case FFTW_RODFT00:
            for (int j = 0; j < n; ++j) {
                const cpx v = VAL(j);
                z[j + 1] = v;
                z[L - 1 - j] = -v;
            }
            fft1_exec(&d->f, z, -1, work);
            /* Z = -2i S_a + 2 S_b, RODFT00 = 2 S */
            for (int k = 0; k < n; ++k) {
                a[(long)k * sa] = -cimag(z[k + 1]);
                if (b) b[(long)k * sb] = creal(z[k + 1]);
            }
            break;
        case FFTW_REDFT10:
            for (int j = 0; j < n; ++j) {
                const cpx v = VAL(j);
                z[2 * j + 1] = v;
                z[L - 2 * j - 1] = v;
            }
            fft1_exec(&d->f, z, -1, work);
            for (int k = 0; k < n; ++k) {
                a[(long)k * sa] = creal(z[k]);
                if (b) b[(long)k * sb] = cimag(z[k]);
            }
            break;
        case FFTW_REDFT01:
            for (int j = 0; j < n; ++j) {
                const cpx v = VAL(j);
                z[j] = v;
                if (j > 0) z[L - j] = v;
            }
            fft1_exec(&d->f, z, -1, work);
            for (int k = 0; k < n; ++k) {
                a[(long)k * sa] = creal(z[2 * k + 1]);
                if (b) b[(long)k * sb] = cimag(z[2 * k + 1]);
            }
            break;
        default:
            break;
    }
#undef VAL
}

/* ---- plans -------------------------------------------------------------------------- */
struct bp_fftw_plan_s {
    int n0, n1;
    int sign; /* c2c only */
    int c2c;
    dim_plan d0, d1;
};

static int supported_kind(int k) {
    return k == FFTW_RODFT00 || k == FFTW_REDFT10 || k == FFTW_REDFT01;
}

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags) {
    (void)in;
    (void)out;
    (void)flags;
    if (n0 < 1 || n1 < 1) return NULL;
    fftw_plan p = (fftw_plan)calloc(1, sizeof *p);
    p->n0 = n0;
    p->n1 = n1;
    p->sign = sign;
    p->c2c = 1;
    dim_init(&p->d0, -1, n0);
    dim_init(&p->d1, -1, n1);
    return p;
}

fftw_plan fftw_plan_r2r_2d(int n0, int n1, double* in, double* out, fftw_r2r_kind kind0,
                           fftw_r2r_kind kind1, unsigned flags) {
    (void)in;
    (void)out;
    (void)flags;
    if (n0 < 1 || n1 < 1 || !supported_kind(kind0) || !supported_kind(kind1)) return NULL;
    fftw_plan p = (fftw_plan)calloc(1, sizeof *p);
    p->n0 = n0;
    p->n1 = n1;
    p->c2c = 0;
    dim_init(&p->d0, kind0, n0);
    dim_init(&p->d1, kind1, n1);
    return p;
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    const int n0 = p->n0, n1 = p->n1;
    cpx* o = (cpx*)out;
    if ((void*)in != (void*)out) memcpy(o, in, sizeof(cpx) * (size_t)n0 * n1);
    const int Lmax = p->d0.f.L > p->d1.f.L ? p->d0.f.L : p->d1.f.L;
    cpx* z = (cpx*)malloc(sizeof(cpx) * (size_t)Lmax * 2);
    cpx* work = z + Lmax;
    for (int i = 0; i < n0; ++i) fft1_exec(&p->d1.f, o + (long)i * n1, p->sign, work);
    for (int j = 0; j < n1; ++j) {
        for (int i = 0; i < n0; ++i) z[i] = o[(long)i * n1 + j];
        fft1_exec(&p->d0.f, z, p->sign, work);
        for (int i = 0; i < n0; ++i) o[(long)i * n1 + j] = z[i];
    }
    free(z);
}

void fftw_execute_r2r(const fftw_plan p, double* in, double* out) {
    const int n0 = p->n0, n1 = p->n1;
    if (in != out) memcpy(out, in, sizeof(double) * (size_t)n0 * n1);
    const int Lmax = p->d0.f.L > p->d1.f.L ? p->d0.f.L : p->d1.f.L;
    cpx* z = (cpx*)malloc(sizeof(cpx) * (size_t)Lmax * 2);
    cpx* work = z + Lmax;
    /* dimension 1 (contiguous rows), two rows per complex FFT */
    for (int i = 0; i < n0; i += 2) {
        double* a = out + (long)i * n1;
        double* b = (i + 1 < n0) ? out + (long)(i + 1) * n1 : NULL;
        r2r_pair(&p->d1, a, 1, b, 1, z, work);
    }
    /* dimension 0 (strided columns), two columns per complex FFT */
    for (int j = 0; j < n1; j += 2) {
        double* a = out + j;
        double* b = (j + 1 < n1) ? out + j + 1 : NULL;
        r2r_pair(&p->d0, a, n1, b, n1, z, work);
    }
    free(z);
}

void fftw_destroy_plan(fftw_plan p) {
    if (!p) return;
    fft1_free(&p->d0.f);
    fft1_free(&p->d1.f);
    free(p);
}
