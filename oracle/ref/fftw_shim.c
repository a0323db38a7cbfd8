/*
 * fftw_shim.c -- project-owned implementation of the five FFTW entry points the
 * reference's transform layer uses (ORACLE infrastructure; see fftw3.h).
 *
 * Power-of-two embedding lengths go through radix-4 Stockham complex FFTs; two real
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

/* ---- 1-D complex FFT ------------------------------------------------------------------
 * Power-of-two lengths: radix-4 Stockham autosort passes (DIF, ping-pong between the line and
 * a work buffer, no bit reversal) with a final radix-2 pass when log2 L is odd; every pass
 * reads its twiddles w^p, w^2p, w^3p from a per-pass table built at plan time (forward and
 * backward tables, so the inner loops carry no sign branch).  Other lengths evaluate the
 * defining sums directly (O(L^2)).  This is NOT FFTW: it is the project's shim for the five
 * FFTW entry points the reference's transform layer calls (FFTW is absent from the image). */
typedef struct {
    int L;      /* transform length */
    int pow2;
    int npass;  /* Stockham passes */
    int radix[32];
    int off[32];  /* start of each pass's twiddles in tw_f / tw_b (3 per p, radix 4) */
    cpx* tw_f;  /* per-pass twiddles, forward sign   */
    cpx* tw_b;  /*                    backward sign  */
    cpx* dtw;   /* e^{-2 pi i k/L}, direct path only */
} fft1;

static int is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

static cpx expi(double a) { return cos(a) + I * sin(a); }

/* plain complex product: C99 `a * b` calls the Annex-G __muldc3 (inf/nan recovery), which is
 * several times slower than the four multiplications the transforms need */
static inline cpx cmulx(cpx a, cpx b) {
    const double ar = creal(a), ai = cimag(a), br = creal(b), bi = cimag(b);
    return (ar * br - ai * bi) + I * (ar * bi + ai * br);
}

static void fft1_init(fft1* t, int L) {
    memset(t, 0, sizeof *t);
    t->L = L;
    t->pow2 = is_pow2(L);
    if (!t->pow2) {
        t->dtw = (cpx*)malloc(sizeof(cpx) * (size_t)L);
        for (int k = 0; k < L; ++k) t->dtw[k] = expi(-2.0 * kPi * (double)k / (double)L);
        return;
    }
    int n = L, tot = 0;
    while (n > 1) {
        const int r = (n % 4 == 0) ? 4 : 2;
        t->radix[t->npass] = r;
        t->off[t->npass] = tot;
        tot += (r - 1) * (n / r);
        ++t->npass;
        n /= r;
    }
    t->tw_f = (cpx*)malloc(sizeof(cpx) * (size_t)(tot > 0 ? tot : 1));
    t->tw_b = (cpx*)malloc(sizeof(cpx) * (size_t)(tot > 0 ? tot : 1));
    n = L;
    for (int ps = 0; ps < t->npass; ++ps) {
        const int r = t->radix[ps], m = n / r;
        for (int p = 0; p < m; ++p)
            for (int e = 1; e < r; ++e) {
                const double a = -2.0 * kPi * (double)(e * p) / (double)n;
                t->tw_f[t->off[ps] + (r - 1) * p + e - 1] = expi(a);
                t->tw_b[t->off[ps] + (r - 1) * p + e - 1] = expi(-a);
            }
        n = m;
    }
}

static void fft1_free(fft1* t) {
    free(t->tw_f);
    free(t->tw_b);
    free(t->dtw);
}

/* one radix-4 Stockham pass: n = current length, s = stride (product of earlier radices) */
static void pass4(int n, int s, const cpx* tw, int inv, const cpx* x, cpx* y) {
    const int m = n / 4;
    for (int p = 0; p < m; ++p) {
        const cpx w1 = tw[3 * p], w2 = tw[3 * p + 1], w3 = tw[3 * p + 2];
        const cpx* xa = x + (size_t)s * p;
        const cpx* xb = x + (size_t)s * (p + m);
        const cpx* xc = x + (size_t)s * (p + 2 * m);
        const cpx* xd = x + (size_t)s * (p + 3 * m);
        cpx* y0 = y + (size_t)s * (4 * p);
        for (int q = 0; q < s; ++q) {
            const cpx a = xa[q], b = xb[q], c = xc[q], d = xd[q];
            const cpx apc = a + c, amc = a - c, bpd = b + d, bmd = b - d;
            /* forward: -i (b - d); backward: +i (b - d) */
            const cpx jb = inv ? (-cimag(bmd) + I * creal(bmd)) : (cimag(bmd) - I * creal(bmd));
            y0[q] = apc + bpd;
            y0[q + s] = cmulx(amc + jb, w1);
            y0[q + 2 * s] = cmulx(apc - bpd, w2);
            y0[q + 3 * s] = cmulx(amc - jb, w3);
        }
    }
}

static void pass2(int n, int s, const cpx* tw, const cpx* x, cpx* y) {
    const int m = n / 2;
    for (int p = 0; p < m; ++p) {
        const cpx w = tw[p];
        const cpx* xa = x + (size_t)s * p;
        const cpx* xb = x + (size_t)s * (p + m);
        cpx* y0 = y + (size_t)s * (2 * p);
        for (int q = 0; q < s; ++q) {
            const cpx a = xa[q], b = xb[q];
            y0[q] = a + b;
            y0[q + s] = cmulx(a - b, w);
        }
    }
}

/* forward (sign -1) or backward (sign +1) unnormalized DFT in place; work: L entries */
static void fft1_exec(const fft1* t, cpx* z, int sign, cpx* work) {
    const int L = t->L;
    if (t->pow2) {
        const int inv = sign > 0;
        const cpx* tw = inv ? t->tw_b : t->tw_f;
        cpx *x = z, *y = work;
        int n = L, s = 1;
        for (int ps = 0; ps < t->npass; ++ps) {
            if (t->radix[ps] == 4) pass4(n, s, tw + t->off[ps], inv, x, y);
            else pass2(n, s, tw + t->off[ps], x, y);
            n /= t->radix[ps];
            s *= t->radix[ps];
            cpx* tmp = x;
            x = y;
            y = tmp;
        }
        if (x != z) memcpy(z, x, sizeof(cpx) * (size_t)L);
    } else {
        for (int k = 0; k < L; ++k) {
            cpx s = 0;
            for (int j = 0; j < L; ++j) {
                cpx w = t->dtw[(int)(((long)j * k) % L)];
                if (sign > 0) w = conj(w);
                s += cmulx(z[j], w);
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

/* Column passes go through a cache-blocked scratch: CB adjacent columns (one 64-byte line of
 * doubles / four complex) are gathered row by row into contiguous lines, transformed, and
 * scattered back, so every row's cache line is read and written once per block. */
enum { CB_R = 8, CB_C = 4 };

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    const int n0 = p->n0, n1 = p->n1;
    cpx* o = (cpx*)out;
    if ((void*)in != (void*)out) memcpy(o, in, sizeof(cpx) * (size_t)n0 * n1);
    const int Lmax = p->d0.f.L > p->d1.f.L ? p->d0.f.L : p->d1.f.L;
    cpx* z = (cpx*)malloc(sizeof(cpx) * ((size_t)Lmax * 2 + (size_t)CB_C * n0));
    cpx* work = z + Lmax;
    cpx* blk = work + Lmax;
    for (int i = 0; i < n0; ++i) fft1_exec(&p->d1.f, o + (long)i * n1, p->sign, work);
    for (int j0 = 0; j0 < n1; j0 += CB_C) {
        const int w = (n1 - j0) < CB_C ? (n1 - j0) : CB_C;
        for (int i = 0; i < n0; ++i)
            for (int c = 0; c < w; ++c) blk[(long)c * n0 + i] = o[(long)i * n1 + j0 + c];
        for (int c = 0; c < w; ++c) fft1_exec(&p->d0.f, blk + (long)c * n0, p->sign, work);
        for (int i = 0; i < n0; ++i)
            for (int c = 0; c < w; ++c) o[(long)i * n1 + j0 + c] = blk[(long)c * n0 + i];
    }
    free(z);
}

void fftw_execute_r2r(const fftw_plan p, double* in, double* out) {
    const int n0 = p->n0, n1 = p->n1;
    if (in != out) memcpy(out, in, sizeof(double) * (size_t)n0 * n1);
    const int Lmax = p->d0.f.L > p->d1.f.L ? p->d0.f.L : p->d1.f.L;
    cpx* z = (cpx*)malloc(sizeof(cpx) * (size_t)Lmax * 2);
    double* blk = (double*)malloc(sizeof(double) * (size_t)CB_R * n0);
    cpx* work = z + Lmax;
    /* dimension 1 (contiguous rows), two rows per complex FFT */
    for (int i = 0; i < n0; i += 2) {
        double* a = out + (long)i * n1;
        double* b = (i + 1 < n0) ? out + (long)(i + 1) * n1 : NULL;
        r2r_pair(&p->d1, a, 1, b, 1, z, work);
    }
    /* dimension 0 (strided columns): blocks of CB_R columns, two columns per complex FFT */
    for (int j0 = 0; j0 < n1; j0 += CB_R) {
        const int w = (n1 - j0) < CB_R ? (n1 - j0) : CB_R;
        for (int i = 0; i < n0; ++i)
            for (int c = 0; c < w; ++c) blk[(long)c * n0 + i] = out[(long)i * n1 + j0 + c];
        for (int c = 0; c < w; c += 2)
            r2r_pair(&p->d0, blk + (long)c * n0, 1, (c + 1 < w) ? blk + (long)(c + 1) * n0 : NULL, 1,
                     z, work);
        for (int i = 0; i < n0; ++i)
            for (int c = 0; c < w; ++c) out[(long)i * n1 + j0 + c] = blk[(long)c * n0 + i];
    }
    free(blk);
    free(z);
}

void fftw_destroy_plan(fftw_plan p) {
    if (!p) return;
    fft1_free(&p->d0.f);
    fft1_free(&p->d1.f);
    free(p);
}
