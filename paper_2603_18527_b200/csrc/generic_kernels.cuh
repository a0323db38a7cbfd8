// generic_kernels.cuh -- any-shape path (sm_100a): grids whose sides are not 2^k - 1, and
// rectangular grids (proj/src/transforms.cpp:39-65 plans any nx x ny through FFTW; the
// reference's own verify suite round-trips a 16 x 12 grid, verify.cpp:90-100).
//
// Transforms: one CTA per line, the line's length-n DFT in shared memory --
//   * n = 2^k: in-place radix-2 on the bit-reversed line;
//   * otherwise Bluestein: X_k = c_k sum_j (x_j c_j) b_{k-j}, c_j = exp(-i pi j^2 / n),
//     b_m = conj(c_m), the linear convolution done as a cyclic one of length L = 2^k >= 2n - 1
//     (FFT of the chirped line, x FFT(b) precomputed per plan, inverse FFT by conjugation).
// DST-I of length N uses the DFT of length n = N + 1 with the fused engine's pre-/post-
// processing (dst_engine.cuh): y_j = sin(pi j/n)(x_j + x_{n-j}) + (x_j - x_{n-j})/2, W = DFT_n y,
// Y_2k = (i/2)(W_k - W_{n-k}), Y_2k+1 = W_0/2 + sum_{m=1..k} (W_m + W_{n-m})/2 -- exact for any n
// (checked against scipy's dst type 1 for odd and even n).  Periodic FFT lines are the plain DFT.
// Lines are addressed as base(l) = (l / lpm) mstride + (l mod lpm) lstride, element j at
// base + j estride: y-lines (estride 1) and x-lines (estride ny) of a dense batch.
#pragma once

#include "sweep_kernels.cuh"

namespace bs {

enum GLineMode { GL_DST = 0, GL_DFT = 1, GL_IDFT = 2 };

struct GLineArgs {
    const double2* in;
    double2* out;
    int n;           // DFT length (DST: N + 1)
    int L;           // FFT length (power of two; L == n: direct)
    int lgL;
    long lines, lpm, mstride, lstride, estride;
    const double2* chirp;  // [n] exp(-i pi j^2 / n)          (Bluestein)
    const double2* filt;   // [L] FFT_L of the wrapped conj chirp (Bluestein)
    const double2* tw;     // [L / 2] exp(-2 pi i k / L)
    double scale;
    const int* status;     // nullable: lines of members that are no longer ACTIVE are skipped
};

// In-place radix-2 DIT FFT (forward, exp(-)) of F[0..L) holding the line in bit-reversed order.
__device__ __forceinline__ void gl_fft(double2* F, int L, const double2* __restrict__ tw) {
    for (int half = 1; half < L; half <<= 1) {
        const int tstride = L / (2 * half);
        for (int b = threadIdx.x; b < L / 2; b += blockDim.x) {
            const int pos = b & (half - 1);
            const int i = ((b - pos) << 1) + pos;
            const int j = i + half;
            const double2 t = cmul(F[j], __ldg(&tw[pos * tstride]));
            const double2 u = F[i];
            F[i] = cadd(u, t);
            F[j] = csub(u, t);
        }
        __syncthreads();
    }
}

__device__ __forceinline__ int gl_brev(int i, int lg) { return lg ? (int)(__brev((unsigned)i) >> (32 - lg)) : 0; }

// Block-wide inclusive prefix sum of S[0..K) in place (fixed order: per-thread contiguous chunks,
// then the chunk totals sequentially) -- the DST post-processing's odd outputs.
__device__ __forceinline__ void gl_scan(double2* S, int K, double2* tot) {
    const int T = blockDim.x, t = threadIdx.x;
    const int c = (K + T - 1) / T, lo = t * c, hi = min(K, lo + c);
    double2 acc = make_double2(0.0, 0.0);
    for (int k = lo; k < hi; ++k) {
        acc = cadd(acc, S[k]);
        S[k] = acc;
    }
    tot[t] = acc;
    __syncthreads();
    if (t == 0) {
        double2 run = make_double2(0.0, 0.0);
        for (int k = 0; k < T; ++k) {
            const double2 v = tot[k];
            tot[k] = run;  // exclusive
            run = cadd(run, v);
        }
    }
    __syncthreads();
    const double2 off = tot[t];
    for (int k = lo; k < hi; ++k) S[k] = cadd(S[k], off);
    __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(256) gline_kernel(const GLineArgs a) {
    extern __shared__ double2 gsm[];
    const long l = blockIdx.x;
    if (l >= a.lines) return;
    if (a.status && __ldcg(&a.status[l / a.lpm]) != ST_ACTIVE) return;  // uniform per CTA
    const int n = a.n, L = a.L, lg = a.lgL, T = blockDim.x, t = threadIdx.x;
    const bool blue = L != n;
    const long base = (l / a.lpm) * a.mstride + (l % a.lpm) * a.lstride;
    double2* X = gsm;      // [n] the line (DST: x_0 = 0, x_1..x_N) / the DFT result
    double2* F = gsm + n;  // [L] FFT workspace (+ scan scratch)
    const double2 zero = make_double2(0.0, 0.0);
    if constexpr (MODE == GL_DST) {
        for (int j = t; j < n; j += T) X[j] = j == 0 ? zero : a.in[base + (long)(j - 1) * a.estride];
        __syncthreads();
    }
    for (int j = t; j < L; j += T) {
        double2 v = zero;
        if (j < n) {
            if constexpr (MODE == GL_DST) {
                if (j > 0) {
                    const double2 x = X[j], xm = X[n - j];
                    const double s = sinpi((double)j / n);
                    const double2 sm = cadd(x, xm), df = csub(x, xm);
                    v = make_double2(fma(s, sm.x, 0.5 * df.x), fma(s, sm.y, 0.5 * df.y));
                }
            } else {
                v = a.in[base + (long)j * a.estride];
                if constexpr (MODE == GL_IDFT) v = cconj(v);
            }
            if (blue) v = cmul(v, __ldg(&a.chirp[j]));
        }
        F[gl_brev(j, lg)] = v;
    }
    __syncthreads();
    gl_fft(F, L, a.tw);
    if (blue) {
        // cyclic convolution with b: inverse FFT of F * FFT(b) as conj(FFT(conj(.))) / L
        for (int k = t; k < L; k += T) F[k] = cconj(cmul(F[k], __ldg(&a.filt[k])));
        __syncthreads();
        for (int k = t; k < L; k += T) {
            const int r = gl_brev(k, lg);
            if (k < r) {
                const double2 tmp = F[k];
                F[k] = F[r];
                F[r] = tmp;
            }
        }
        __syncthreads();
        gl_fft(F, L, a.tw);
    }
    const double invL = 1.0 / L;
    for (int k = t; k < n; k += T) {
        double2 w = F[k];
        if (blue) w = cmul(__ldg(&a.chirp[k]), cscale(cconj(w), invL));
        if constexpr (MODE == GL_DST) {
            X[k] = w;
        } else {
            if constexpr (MODE == GL_IDFT) w = cconj(w);
            a.out[base + (long)k * a.estride] = cscale(w, a.scale);
        }
    }
    if constexpr (MODE == GL_DST) {
        __syncthreads();
        const int N = n - 1;
        const int K = n / 2;                // odd outputs Y_1, Y_3, ..., Y_{2K-1}
        double2* S = F;                     // prefix terms (F is free now)
        double2* tot = F + K;
        for (int k = t; k < K; k += T) {
            const double2 w = k == 0 ? cscale(X[0], 0.5) : cscale(cadd(X[k], X[n - k]), 0.5);
            S[k] = w;
        }
        __syncthreads();
        gl_scan(S, K, tot);
        for (int j = t + 1; j <= N; j += T) {
            double2 y;
            if (j & 1) {
                y = S[j >> 1];
            } else {
                const int k = j >> 1;
                const double2 d = csub(X[k], X[n - k]);
                y = make_double2(-0.5 * d.y, 0.5 * d.x);  // (i/2)(W_k - W_{n-k})
            }
            a.out[base + (long)(j - 1) * a.estride] = cscale(y, a.scale);
        }
    }
}

// ------------------------------------------------------------------ element-wise (dense batch)
struct GenArgs {
    int batch, nx, ny;
    double inv_h2;           // 1 / hx^2 (the reference's five_point takes one h2, kernels.cpp:56-69)
    const double2* k2;
    const double* k0sq;
    const double* eta;
    const double* ax;        // (4/hx^2) sin^2((p+1) pi / (2(nx+1))), p < nx  (symbol.cpp:69-80)
    const double* ay;        // same for y
    double gscale;           // 4 / ((nx+1)(ny+1)): the two inverse DSTs' normalisation
};

__device__ __forceinline__ double2 gen_stencil(const double2* __restrict__ u, long idx, int i, int j, int nx, int ny) {
    double2 s = cscale(u[idx], 4.0);
    if (i > 0) s = csub(s, u[idx - ny]);
    if (i < nx - 1) s = csub(s, u[idx + ny]);
    if (j > 0) s = csub(s, u[idx - 1]);
    if (j < ny - 1) s = csub(s, u[idx + 1]);
    return s;
}

// op: 0 A u, 1 V u, 2 V^H u, 3 f - A u, 4 V u + f, 5 k2 u
__global__ void gen_pointwise_kernel(GenArgs g, int op, const double2* __restrict__ u,
                                     const double2* __restrict__ f, double2* __restrict__ out) {
    const long per = (long)g.nx * g.ny, total = per * g.batch;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
        const int b = (int)(idx / per);
        const long r = idx % per;
        const int i = (int)(r / g.ny), j = (int)(r % g.ny);
        const double2 uu = u[idx], kk = g.k2[idx];
        const double2 V = csub(kk, make_double2(g.k0sq[b], g.eta[b]));
        double2 o;
        if (op == 1) o = cmul(uu, V);
        else if (op == 2) o = cmul(cconj(V), uu);
        else if (op == 4) o = cadd(cmul(V, uu), f[idx]);
        else if (op == 5) o = cmul(kk, uu);
        else {
            o = csub(cscale(gen_stencil(u, idx, i, j, g.nx, g.ny), g.inv_h2), cmul(kk, uu));
            if (op == 3) o = csub(f[idx], o);
        }
        out[idx] = o;
    }
}

// spectral multiply in the DST basis: x scale / lambda_pq (Green) or x scale lambda_pq (L_ref),
// lambda = (a_p + a_q) - (k0^2 + i eta)  (symbol.cpp:69-80 + shift_symbol :97-100)
__global__ void gen_symbol_kernel(GenArgs g, int divide, double scale, double2* __restrict__ x) {
    const long per = (long)g.nx * g.ny, total = per * g.batch;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
        const int b = (int)(idx / per);
        const long r = idx % per;
        const int p = (int)(r / g.ny), q = (int)(r % g.ny);
        const double lr = (g.ax[p] + g.ay[q]) - g.k0sq[b], li = -g.eta[b];
        double2 w;
        if (divide == 2) {
            w = make_double2((g.ax[p] + g.ay[q]) * scale, 0.0);  // |xi|^2 (periodic A's symbol part)
        } else if (divide) {
            const double s = scale / fma(lr, lr, li * li);
            w = make_double2(lr * s, -li * s);
        } else {
            w = make_double2(lr * scale, li * scale);
        }
        x[idx] = cmul(x[idx], w);
    }
}

// q^m = V u^m + f for the members still ACTIVE (u^m in buffer sweep & 1), 0 otherwise
__global__ void gen_source_kernel(GenArgs g, Control c, const double2* __restrict__ u0,
                                  const double2* __restrict__ u1, const double2* __restrict__ f,
                                  double2* __restrict__ q) {
    const long per = (long)g.nx * g.ny, total = per * g.batch;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
        const int b = (int)(idx / per);
        double2 o = make_double2(0.0, 0.0);
        if (__ldcg(&c.status[b]) == ST_ACTIVE) {
            const double2* u = (__ldcg(&c.sweep[b]) & 1) ? u1 : u0;
            o = cadd(cmul(csub(g.k2[idx], make_double2(g.k0sq[b], g.eta[b])), u[idx]), f[idx]);
        }
        q[idx] = o;
    }
}

// One sweep's element-wise tail for the generic run (members still ACTIVE): r_bs = z - u^m,
// res = f - A u^m; per-chunk partial sums of |res|^2 and |r_bs|^2 (the R_eta norm by the key
// identity, as the fused row kernel); u^{m+1} = u^m + gamma d, d = r_bs (NPBS / CBS) or res
// (Direct), gamma scalar or (i/eta) V (pointwise map).  grid = (chunks, batch).
__global__ void __launch_bounds__(256) gen_sweep_kernel(GenArgs g, Control c, const double2* __restrict__ z,
                                                        const double2* __restrict__ f, const double2* __restrict__ u0,
                                                        const double2* __restrict__ u1, double2* __restrict__ w0,
                                                        double2* __restrict__ w1, int map_kind, double2 gamma,
                                                        int direct, double* __restrict__ part, int nchunk,
                                                        double2* __restrict__ rout) {
    const int b = blockIdx.y, ch = blockIdx.x;
    __shared__ double red[2][256];
    const bool active = __ldcg(&c.status[b]) == ST_ACTIVE;
    const int m = __ldcg(&c.sweep[b]);
    const long per = (long)g.nx * g.ny;
    const long chunk = (per + nchunk - 1) / nchunk, lo = ch * chunk, hi = min(per, lo + chunk);
    const double2* u = (m & 1) ? u1 : u0;  // u^m
    double2* un = (m & 1) ? w0 : w1;       // u^{m+1}
    double s0 = 0.0, s1 = 0.0;
    if (active) {
        const double2 shift = make_double2(g.k0sq[b], g.eta[b]);
        for (long r = lo + threadIdx.x; r < hi; r += blockDim.x) {
            const long idx = b * per + r;
            const int i = (int)(r / g.ny), j = (int)(r % g.ny);
            const double2 uu = u[idx], kk = g.k2[idx];
            const double2 rbs = csub(z[idx], uu);
            const double2 res = csub(f[idx], csub(cscale(gen_stencil(u, idx, i, j, g.nx, g.ny), g.inv_h2), cmul(kk, uu)));
            s0 += cnorm(res);
            s1 += cnorm(rbs);
            if (rout) rout[idx] = res;  // hx != hy: the R_eta norm needs G r explicitly
            double2 gm = gamma;
            if (map_kind == MK_POINTWISE) gm = cscale(mul_pi(csub(kk, shift)), 1.0 / g.eta[b]);
            un[idx] = cadd(uu, cmul(gm, direct ? res : rbs));
        }
    }
    red[0][threadIdx.x] = s0;
    red[1][threadIdx.x] = s1;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
        if (threadIdx.x < h) {
            red[0][threadIdx.x] += red[0][threadIdx.x + h];
            red[1][threadIdx.x] += red[1][threadIdx.x + h];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[((long)b * nchunk + ch) * 2] = red[0][0];
        part[((long)b * nchunk + ch) * 2 + 1] = red[1][0];
    }
}

// per-chunk |x|^2 of the active members into part[..][1] (replaces the key-identity sum)
__global__ void __launch_bounds__(256) gen_part_kernel(GenArgs g, Control c, const double2* __restrict__ x,
                                                       double* __restrict__ part, int nchunk) {
    const int b = blockIdx.y, ch = blockIdx.x;
    __shared__ double red[256];
    const long per = (long)g.nx * g.ny;
    const long chunk = (per + nchunk - 1) / nchunk, lo = ch * chunk, hi = min(per, lo + chunk);
    double s = 0.0;
    if (__ldcg(&c.status[b]) == ST_ACTIVE)
        for (long r = lo + threadIdx.x; r < hi; r += blockDim.x) s += cnorm(x[b * per + r]);
    red[threadIdx.x] = s;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
        if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[((long)b * nchunk + ch) * 2 + 1] = red[0];
}

// Periodic any-shape sweep in Fourier space (U = DFT(u^m), Q = DFT(V u^m + f)): R = Q/lambda - U
// is the transform of r_bs and lambda R that of the residual f - A u^m = q - L_ref u^m, so both
// trace norms follow by Parseval (sum |x|^2 = sum |X|^2 / (nx ny)) without another transform;
// U^{m+1} = U + gamma R (Direct: + gamma lambda R).  Inactive members are left untouched.
__global__ void __launch_bounds__(256) gen_psweep_kernel(GenArgs g, Control c, const double2* __restrict__ Q,
                                                         double2* __restrict__ U, double2 gamma, int direct,
                                                         double* __restrict__ part, int nchunk) {
    const int b = blockIdx.y, ch = blockIdx.x;
    __shared__ double red[2][256];
    const bool active = __ldcg(&c.status[b]) == ST_ACTIVE;
    const long per = (long)g.nx * g.ny;
    const long chunk = (per + nchunk - 1) / nchunk, lo = ch * chunk, hi = min(per, lo + chunk);
    double s0 = 0.0, s1 = 0.0;
    if (active) {
        for (long r = lo + threadIdx.x; r < hi; r += blockDim.x) {
            const long idx = b * per + r;
            const int p = (int)(r / g.ny), q = (int)(r % g.ny);
            const double lr = (g.ax[p] + g.ay[q]) - g.k0sq[b], li = -g.eta[b];
            const double inv = 1.0 / fma(lr, lr, li * li);
            const double2 qq = Q[idx], uu = U[idx];
            const double2 z = make_double2((qq.x * lr + qq.y * li) * inv, (qq.y * lr - qq.x * li) * inv);
            const double2 R = csub(z, uu);
            const double2 lR = cmul(make_double2(lr, li), R);
            s0 += cnorm(lR);
            s1 += cnorm(R);
            U[idx] = cadd(uu, cmul(gamma, direct ? lR : R));
        }
    }
    red[0][threadIdx.x] = s0;
    red[1][threadIdx.x] = s1;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
        if (threadIdx.x < h) {
            red[0][threadIdx.x] += red[0][threadIdx.x + h];
            red[1][threadIdx.x] += red[1][threadIdx.x + h];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double invn = 1.0 / (double)per;
        part[((long)b * nchunk + ch) * 2] = red[0][0] * invn;
        part[((long)b * nchunk + ch) * 2 + 1] = red[1][0] * invn;
    }
}

// entry m of every active member from the chunk partials (fixed order) + termination test
__global__ void gen_finalize_kernel(Control c, int batch, const double* __restrict__ part, int nchunk) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch || c.status[b] != ST_ACTIVE) return;
    double s0 = 0.0, s1 = 0.0;
    for (int k = 0; k < nchunk; ++k) {
        s0 += part[((long)b * nchunk + k) * 2];
        s1 += part[((long)b * nchunk + k) * 2 + 1];
    }
    finalize_entry(c, b, c.sweep[b], s0, s1);
}

// ---- OptimalScalar / FourierDiag maps on any-shape handles (staged sweep, run_core_generic_maps)
// per-chunk partials of sum conj(a) b (re, im) and sum |a|^2 over the ACTIVE members
__global__ void __launch_bounds__(256) gen_dot_kernel(GenArgs g, Control c, const double2* __restrict__ a,
                                                      const double2* __restrict__ bb, double* __restrict__ part,
                                                      int nchunk) {
    const int b = blockIdx.y, ch = blockIdx.x;
    __shared__ double red[3][256];
    const long per = (long)g.nx * g.ny;
    const long chunk = (per + nchunk - 1) / nchunk, lo = ch * chunk, hi = min(per, lo + chunk);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    if (__ldcg(&c.status[b]) == ST_ACTIVE)
        for (long r = lo + threadIdx.x; r < hi; r += blockDim.x) {
            const double2 w = a[b * per + r], x = bb[b * per + r];
            s0 += w.x * x.x + w.y * x.y;
            s1 += w.x * x.y - w.y * x.x;
            s2 += cnorm(w);
        }
    red[0][threadIdx.x] = s0;
    red[1][threadIdx.x] = s1;
    red[2][threadIdx.x] = s2;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
        if (threadIdx.x < h)
            for (int k = 0; k < 3; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x < 3) part[((long)b * nchunk + ch) * 4 + threadIdx.x] = red[threadIdx.x][0];
}

// gamma_b = <w, r> / <w, w> (correction.cpp:10-18) from the chunk partials, fixed order
// (real_only: real fields read as pairs -- the CDR family -- have a real inner product, s0)
__global__ void gen_gamma_kernel(Control c, int batch, const double* __restrict__ part, int nchunk,
                                 int real_only = 0) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch || c.status[b] != ST_ACTIVE) return;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int k = 0; k < nchunk; ++k) {
        s0 += part[((long)b * nchunk + k) * 4];
        s1 += part[((long)b * nchunk + k) * 4 + 1];
        s2 += part[((long)b * nchunk + k) * 4 + 2];
    }
    finalize_gamma(c, b, s0, real_only ? 0.0 : s1, s2);
}

// per-chunk |a|^2 -> part[..][0], |b|^2 -> part[..][1] of the ACTIVE members (the trace entry)
__global__ void __launch_bounds__(256) gen_norms_kernel(GenArgs g, Control c, const double2* __restrict__ a,
                                                        const double2* __restrict__ bb, double* __restrict__ part,
                                                        int nchunk) {
    const int b = blockIdx.y, ch = blockIdx.x;
    __shared__ double red[2][256];
    const long per = (long)g.nx * g.ny;
    const long chunk = (per + nchunk - 1) / nchunk, lo = ch * chunk, hi = min(per, lo + chunk);
    double s0 = 0.0, s1 = 0.0;
    if (__ldcg(&c.status[b]) == ST_ACTIVE)
        for (long r = lo + threadIdx.x; r < hi; r += blockDim.x) {
            s0 += cnorm(a[b * per + r]);
            s1 += cnorm(bb[b * per + r]);
        }
    red[0][threadIdx.x] = s0;
    red[1][threadIdx.x] = s1;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
        if (threadIdx.x < h) {
            red[0][threadIdx.x] += red[0][threadIdx.x + h];
            red[1][threadIdx.x] += red[1][threadIdx.x + h];
        }
        __syncthreads();
    }
    if (threadIdx.x < 2) part[((long)b * nchunk + ch) * 2 + threadIdx.x] = red[threadIdx.x][0];
}

// u^{m+1} = u^m + gamma_b x (use_gamma) or u^m + x, for the members still ACTIVE after entry m
// was recorded (m = sweep - 1); u^m in buffer m & 1, u^{m+1} into the other one
__global__ void gen_update_kernel(GenArgs g, Control c, double2* __restrict__ u0, double2* __restrict__ u1,
                                  const double2* __restrict__ x, int use_gamma) {
    const long per = (long)g.nx * g.ny, total = per * g.batch;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
        const int b = (int)(idx / per);
        if (__ldcg(&c.status[b]) != ST_ACTIVE) continue;
        const int m = __ldcg(&c.sweep[b]) - 1;
        const double2* u = (m & 1) ? u1 : u0;
        double2* un = (m & 1) ? u0 : u1;
        const double2 d = use_gamma ? cmul(c.gamma[b], x[idx]) : x[idx];
        un[idx] = cadd(u[idx], d);
    }
}

// u^m of every member (buffer sweep & 1) gathered into one dense array (operator inputs)
__global__ void gen_gather_kernel(GenArgs g, Control c, const double2* __restrict__ u0,
                                  const double2* __restrict__ u1, double2* __restrict__ out) {
    const long per = (long)g.nx * g.ny, total = per * g.batch;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
        const int b = (int)(idx / per);
        out[idx] = ((__ldcg(&c.sweep[b]) & 1) ? u1 : u0)[idx];
    }
}

// x <- x * m (FourierDiag multiplier, one nx x ny mode array shared by the batch), or a - b
__global__ void gen_modemul_kernel(GenArgs g, double2* __restrict__ x, const double2* __restrict__ m) {
    const long per = (long)g.nx * g.ny, total = per * g.batch;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x)
        x[idx] = cmul(x[idx], m[idx % per]);
}
__global__ void gen_sub_kernel(double2* __restrict__ out, const double2* __restrict__ a,
                               const double2* __restrict__ b, long total) {
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x)
        out[idx] = csub(a[idx], b[idx]);
}

// dense result copy: member b from buffer p1 when select[b] (its result_buf) else p0
__global__ void gen_select_kernel(const double2* __restrict__ p0, const double2* __restrict__ p1,
                                  const int* __restrict__ select, double2* __restrict__ out, long per, int batch) {
    const long total = per * batch;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
        const int b = (int)(idx / per);
        out[idx] = (select && select[b]) ? p1[idx] : p0[idx];
    }
}

}  // namespace bs
