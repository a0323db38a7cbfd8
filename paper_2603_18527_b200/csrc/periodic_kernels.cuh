// periodic_kernels.cuh -- the reference's own family on sm_100a: periodic pseudospectral
// Helmholtz (bp::HelmholtzProblem, proj/src/helmholtz.cpp:11-53), FFT basis.
//
// The state is carried in Fourier space.  With A = L_ref - V (helmholtz.cpp:22-32) and the
// key identity, for q^m = V u^m + f:
//     r_bs^m = G q^m - u^m        ->  x^ = Q^/lambda - U^          (spectral, diagonal)
//     r^m    = f - A u^m = q^m - L_ref u^m  ->  r^ = Q^ - lambda U^
// so both trace norms come from Parseval (||x||^2 = sum |x^|^2 / (nx ny)) and a diagonal map
// (ScalarMap gamma, FourierDiagMap m) updates U^{m+1} = U^m + M x^ in place.  Per sweep:
//   col kernel  (64 B/pt)  T -> forward x-FFT = Q^; U^m in; x^, r^ partials; U^{m+1} out;
//                          inverse x-FFT of U^{m+1} / (nx ny) -> T; entry m + termination
//   row kernel  (64 B/pt)  T -> inverse y-FFT = u^{m+1}; q = V u^{m+1} + f -> forward y-FFT -> T
// OptimalScalar (correction.cpp:22-48) needs its gamma from a global reduction before the update,
// so a sweep becomes (Euclidean metric, w = A d):
//   CP_OPT_A (col)  Q^; x^, r^; entry m; D^ = direction (x^ or, Direct format, r^) stored;
//                   T = F_x^-1 D^, T2 = F_x^-1 (r^ or lambda D^) (both / (nx ny))
//   RP_OPT_B (row)  d = F_y^-1 T, s = F_y^-1 T2 (= r, or L_ref d); w = s - V d (key identity
//                   A x = r - V x, or A r = L_ref r - V r); <w, r>, |w|^2 -> gamma (last CTA)
//   CP_OPT_C (col)  U^{m+1} = U^m + gamma D^; T = F_x^-1 U^{m+1} / (nx ny)
//   RP_SWEEP (row)  as the scalar sweep
// and for the R_eta metric (w = d - G V d, gamma = <w, d> / |w|^2, correction.cpp:38-44):
//   CP_OPT_A (T only), RP_RETA_B (row: d = F_y^-1 T; F_y (V d) -> T),
//   CP_RETA_C (col: (V d)^ = F_x T; w^ = D^ - (V d)^ / lambda; <w, d>, |w|^2 by Parseval ->
//   gamma), CP_OPT_C, RP_SWEEP.
// Transforms follow proj/include/bp/transforms.hpp:16-17: unnormalised forward DFT, inverse
// with 1/(nx ny).  Grids are n x n, n = 2^k, no padding (every node is a degree of freedom).
#pragma once

#include "sweep_kernels.cuh"

namespace bs {

// Stockham passes for a full length-N complex FFT: radices P, then <= P, product N.
template <int LOG2N, int PP = 16>
struct FftPasses {
    using G = Geom<LOG2N, PP>;
    static constexpr int RMAX = G::P;
    static constexpr int REM = G::N / G::P;
    static constexpr int R2 = REM >= RMAX ? RMAX : REM;
    static constexpr int REM2 = REM / R2;
    static constexpr int R3 = REM2 >= RMAX ? RMAX : REM2;
    static constexpr int REM3 = REM2 / R3;
    static constexpr int R4 = REM3 >= RMAX ? RMAX : REM3;
    static constexpr int REM4 = REM3 / R4;
    static constexpr int R5 = REM4;
    static_assert(R5 <= RMAX, "line too long");
};

template <int LOG2N, int PP = 16>
struct FftEngine {
    using G = Geom<LOG2N, PP>;
    using PS = FftPasses<LOG2N, PP>;
    static constexpr int N = G::N, P = G::P, T = G::T;

    // In: x[m] = x_{t + T m} (stride layout).  Out: y[m] = X_{t + T m}, X = forward DFT
    // (INVERSE: unnormalised backward DFT via conj(DFT(conj x))).
    template <bool INVERSE, class Pol>
    __device__ __forceinline__ static void run(const double2 (&x)[P], double2 (&y)[P], int t,
                                               double2* buf, const double2* __restrict__ tw,
                                               const Pol& pol) {
        double2 v[P];
#pragma unroll
        for (int m = 0; m < P; ++m) v[m] = INVERSE ? cconj(x[m]) : x[m];
        Dft<P>::template run<1>(v);
#pragma unroll
        for (int r = 0; r < P; ++r) buf[G::pidx(t * P + r)] = v[r];
        pol.sync();
        DstEngine<LOG2N, PP>::template pass<PS::R2, P>(buf, t, tw, pol);
        DstEngine<LOG2N, PP>::template pass<PS::R3, P * PS::R2>(buf, t, tw, pol);
        DstEngine<LOG2N, PP>::template pass<PS::R4, P * PS::R2 * PS::R3>(buf, t, tw, pol);
        DstEngine<LOG2N, PP>::template pass<PS::R5, P * PS::R2 * PS::R3 * PS::R4>(buf, t, tw, pol);
#pragma unroll
        for (int m = 0; m < P; ++m) {
            const double2 o = buf[G::pidx(t + T * m)];
            y[m] = INVERSE ? cconj(o) : o;
        }
        pol.sync();
    }
};

enum PRowMode { RP_FWD = 0, RP_FWD_BORN = 1, RP_INV = 2, RP_SWEEP = 3, RP_OPT_B = 4, RP_RETA_B = 5 };
enum PColMode { CP_ONE = 0, CP_GREEN = 1, CP_LREF = 2, CP_SWEEP = 3, CP_INV = 4, CP_OPT_A = 5,
                CP_OPT_C = 6, CP_RETA_C = 7 };

struct PerArgs {
    int batch;
    const double* k0sq;
    const double* eta;
    const double* xi2;         // xi_j^2 = (2 pi m_j / L)^2, m_j in FFT order (grid.hpp:67-85)
    const double2* k2;
    const double2* f;
    const double2* in;         // RP_FWD / RP_FWD_BORN source
    double2* out;              // RP_INV output
    const double2* sub;        // RP_INV: optional field subtracted
    double2* T;                // intermediate
    double2* U0;               // spectral iterate ping
    double2* U1;               // spectral iterate pong
    const double2* fd;         // FourierDiag multiplier (mode layout, shared by the batch)
    const double2* tw;
    double scale;              // CP_ONE / CP_GREEN / CP_LREF / CP_INV output scale
    double inv_npts;           // 1 / (nx ny)
    int map_kind;              // MK_SCALAR / MK_FOURIER_DIAG
    double2 gamma;
    int direct;                // IterFormat::Direct: direction = r (iterate.cpp:122), else r_bs
    int metric_reta;           // OptimalScalar metric R_eta (CP_OPT_A writes T only)
    double2* D;                // OptimalScalar: spectral direction D^ (CP_OPT_A -> CP_OPT_C / CP_RETA_C)
    double2* T2;               // OptimalScalar (Euclidean): second intermediate (r, or L_ref d)
    Control ctl;
};

// Fixed-order CTA sum of NP per-thread values, then the member's CTAs are combined by its
// last-arriving CTA (atomic counter; partial slots [b][slot]): `fin(sums)` runs on one thread
// of that CTA.  Deterministic: the per-CTA partials are summed in slot order.
template <int NP, int NTHR, class Fin>
__device__ __forceinline__ void member_reduce(const Control& c, int b, int slot, int nslots, int slot_stride,
                                              const double (&v)[NP], Fin fin) {
    __shared__ double red[NP][NTHR];
#pragma unroll
    for (int k = 0; k < NP; ++k) red[k][threadIdx.x] = v[k];
    __syncthreads();
    if (threadIdx.x == 0) {
        double* pr = c.partial + ((size_t)b * slot_stride + slot) * kPartStride;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            double s = 0.0;
            for (int i = 0; i < NTHR; ++i) s += red[k][i];
            pr[k] = s;
        }
        __threadfence();
        const unsigned old = atomicAdd(&c.counter[b], 1u);
        if (old == (unsigned)(nslots - 1)) {
            __threadfence();
            double s[NP];
#pragma unroll
            for (int k = 0; k < NP; ++k) s[k] = 0.0;
            for (int i = 0; i < nslots; ++i) {
                const double* pk = c.partial + ((size_t)b * slot_stride + i) * kPartStride;
#pragma unroll
                for (int k = 0; k < NP; ++k) s[k] += __ldcg(pk + k);
            }
            c.counter[b] = 0u;
            fin(s);
        }
    }
}

// ------------------------------------------------------------------ row kernel (y lines)
template <int LOG2N, int MODE, int NW, int PP>
__global__ void __launch_bounds__(NW * 32, (MinBlocks<NW * 32, PP >= 16 ? 128 : 80>::value))
prow_kernel(const PerArgs a) {
    using G = Geom<LOG2N, PP>;
    using RG = RowGeom<LOG2N, PP, NW>;
    using Pol = typename PolicyFor<G::T>::type;
    using Engine = FftEngine<LOG2N, PP>;
    constexpr int N = G::N, P = G::P, T = G::T;
    constexpr int EPB = RG::EPB;
    extern __shared__ double2 smem[];

    const int t = threadIdx.x % T;
    const int e = threadIdx.x / T;
    const long grow = (long)blockIdx.x * EPB + e;
    const int b = (int)(grow >> LOG2N);
    bool valid = b < a.batch;
    constexpr bool ITER = MODE == RP_SWEEP || MODE == RP_OPT_B || MODE == RP_RETA_B;
    if (ITER && valid) valid = __ldcg(&a.ctl.status[b]) == ST_ACTIVE;
    // (RP_OPT_B reduces over the member's rows: a CTA exits only when none of its rows is
    // active, so every row of an active member reaches the counter)
    if (!__syncthreads_or(valid)) return;
    double2* buf = smem + e * G::PAD_N;
    const Pol pol = make_policy((Pol*)nullptr, smem + EPB * G::PAD_N, e);
    const size_t row = (size_t)(valid ? grow : 0) * N;
    const double2 zero = make_double2(0.0, 0.0);
    const double2 shift = make_double2(valid ? a.k0sq[b] : 0.0, valid ? a.eta[b] : 1.0);

    double2 q[P];
    if constexpr (MODE == RP_OPT_B) {
        // d = F_y^-1 T, s = F_y^-1 T2 (physical; the column pass applied 1/(nx ny)); w = s - V d
        double2 x[P], d[P], sv[P];
#pragma unroll
        for (int m = 0; m < P; ++m) x[m] = a.T[row + t + T * m];
        Engine::template run<true>(x, d, t, buf, a.tw, pol);
#pragma unroll
        for (int m = 0; m < P; ++m) x[m] = a.T2[row + t + T * m];
        Engine::template run<true>(x, sv, t, buf, a.tw, pol);
        double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int m = 0; m < P; ++m) {
            const int j = t + T * m;
            const double2 V = csub(a.k2[row + j], shift);
            const double2 w = csub(sv[m], cmul(V, d[m]));
            const double2 r = a.direct ? d[m] : sv[m];   // the Euclidean residual r
            acc[0] += w.x * r.x + w.y * r.y;              // Re conj(w) r   (kernels::dotc)
            acc[1] += w.x * r.y - w.y * r.x;              // Im conj(w) r
            acc[2] += cnorm(w);                           // |w|^2          (kernels::norm2sq)
        }
        // per-row partials (engine-wide fixed-order sums); the member's last row sums its n
        // row partials in row order (lanes strided, fixed tree) and finalises gamma.  A CTA may
        // hold rows of several members (small n), so the reduction is per row, not per CTA.
        const int i = (int)(grow & (N - 1));
#pragma unroll
        for (int k = 0; k < 3; ++k) acc[k] = pol.sum(acc[k], t);
        int last = 0;
        if (valid && t == 0) {
            double* pr = a.ctl.partial + ((size_t)b * N + i) * kPartStride;
#pragma unroll
            for (int k = 0; k < 3; ++k) pr[k] = acc[k];
            __threadfence();
            last = atomicAdd(&a.ctl.counter[b], 1u) == (unsigned)(N - 1);
        }
        last = pol.bcast0(last, t);
        if (last) {
            __threadfence();
            double sm[3] = {0.0, 0.0, 0.0};
            for (int r = t; r < N; r += T) {
                const double* pr = a.ctl.partial + ((size_t)b * N + r) * kPartStride;
#pragma unroll
                for (int k = 0; k < 3; ++k) sm[k] += __ldcg(pr + k);
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) sm[k] = pol.sum(sm[k], t);
            if (t == 0) {
                a.ctl.counter[b] = 0u;
                finalize_gamma(a.ctl, b, sm[0], sm[1], sm[2]);
            }
        }
        return;
    } else if constexpr (MODE == RP_RETA_B) {
        // d = F_y^-1 T (physical); V d -> forward y-FFT -> T (for G V d)
        double2 x[P], d[P];
#pragma unroll
        for (int m = 0; m < P; ++m) x[m] = a.T[row + t + T * m];
        Engine::template run<true>(x, d, t, buf, a.tw, pol);
#pragma unroll
        for (int m = 0; m < P; ++m) {
            const int j = t + T * m;
            q[m] = cmul(d[m], csub(a.k2[row + j], shift));  // apply_V(d)
        }
    } else if constexpr (MODE == RP_INV || MODE == RP_SWEEP) {
        double2 x[P], z[P];
#pragma unroll
        for (int m = 0; m < P; ++m) x[m] = valid ? a.T[row + t + T * m] : zero;
        Engine::template run<true>(x, z, t, buf, a.tw, pol);
#pragma unroll
        for (int m = 0; m < P; ++m) {
            const int j = t + T * m;
            if constexpr (MODE == RP_INV) {
                double2 o = z[m];
                if (a.sub) o = csub(o, valid ? a.sub[row + j] : zero);
                if (valid) a.out[row + j] = o;
            } else {
                // u^{m+1} (already scaled by 1/(nx ny)); q^{m+1} = V u^{m+1} + f
                const double2 V = csub(valid ? a.k2[row + j] : zero, shift);
                q[m] = cadd(cmul(z[m], V), valid ? a.f[row + j] : zero);
            }
        }
        if constexpr (MODE == RP_INV) return;
    } else {
#pragma unroll
        for (int m = 0; m < P; ++m) {
            const int j = t + T * m;
            double2 v = valid ? a.in[row + j] : zero;
            if constexpr (MODE == RP_FWD_BORN) {
                const double2 V = csub(valid ? a.k2[row + j] : zero, shift);
                v = cadd(cmul(v, V), valid ? a.f[row + j] : zero);  // kernels::mul(u, v) + f
            }
            q[m] = v;
        }
    }
    double2 y[P];
    Engine::template run<false>(q, y, t, buf, a.tw, pol);
#pragma unroll
    for (int m = 0; m < P; ++m)
        if (valid) a.T[row + t + T * m] = y[m];
}

// ------------------------------------------------------------------ column kernel (x lines)
template <int LOG2N, int MODE, int C, int PP>
__global__ void __launch_bounds__(C * Geom<LOG2N, PP>::T, (MinBlocks<C * Geom<LOG2N, PP>::T, PP >= 16 ? 128 : 64>::value))
pcol_kernel(const PerArgs a) {
    using G = Geom<LOG2N, PP>;
    using Engine = FftEngine<LOG2N, PP>;
    constexpr int N = G::N, P = G::P, T = G::T;
    extern __shared__ double2 smem[];
    int c, t;
    col_thread_map<G::T, C>(t, c);
    constexpr int GROUPS = N / C;
    const int bid = BS_COL_REVERSE && a.batch > 1 ? gridDim.x - 1 - blockIdx.x : blockIdx.x;  // (col_kernel)
    const int b = bid / GROUPS;
    const int q = (bid % GROUPS) * C + c;
    int mstep = 0;
    constexpr bool ITER = MODE == CP_SWEEP || MODE == CP_OPT_A || MODE == CP_OPT_C || MODE == CP_RETA_C;
    if constexpr (ITER) {
        if (__ldcg(&a.ctl.status[b]) != ST_ACTIVE) return;  // uniform per CTA
        // entry m of this sweep; CP_OPT_C / CP_RETA_C run after CP_OPT_A recorded it
        mstep = __ldcg(&a.ctl.sweep[b]) - ((MODE == CP_OPT_C || MODE == CP_RETA_C) ? 1 : 0);
    }
    double2* buf = smem + c * G::PAD_N;
    const BlockSeg<T, C> pol{smem + C * G::PAD_N, c};
    const size_t mem = (size_t)b * N * N;

    double2 x[P], y[P];
    if constexpr (MODE != CP_OPT_C) {
#pragma unroll
        for (int m = 0; m < P; ++m) x[m] = a.T[mem + (size_t)(t + T * m) * N + q];
    }
    if constexpr (MODE == CP_INV) {
        Engine::template run<true>(x, y, t, buf, a.tw, pol);
#pragma unroll
        for (int m = 0; m < P; ++m) a.T[mem + (size_t)(t + T * m) * N + q] = cscale(y[m], a.scale);
        return;
    } else if constexpr (MODE != CP_OPT_C) {
        Engine::template run<false>(x, y, t, buf, a.tw, pol);
    }
    if constexpr (MODE == CP_ONE) {
#pragma unroll
        for (int m = 0; m < P; ++m) a.T[mem + (size_t)(t + T * m) * N + q] = cscale(y[m], a.scale);
        return;
    } else if constexpr (MODE == CP_OPT_C) {
        // U^{m+1} = U^m + gamma D^ (kernels::scale + add); T = F_x^-1 U^{m+1} / (nx ny)
        const double2* Ucur = (mstep & 1) ? a.U1 : a.U0;
        double2* Unext = (mstep & 1) ? a.U0 : a.U1;
        const double2 g = a.ctl.gamma[b];
#pragma unroll
        for (int m = 0; m < P; ++m) {
            const size_t idx = mem + (size_t)(t + T * m) * N + q;
            const double2 Un = cadd(Ucur[idx], cmul(g, a.D[idx]));
            Unext[idx] = Un;
            x[m] = Un;
        }
        Engine::template run<true>(x, y, t, buf, a.tw, pol);
#pragma unroll
        for (int m = 0; m < P; ++m) a.T[mem + (size_t)(t + T * m) * N + q] = cscale(y[m], a.inv_npts);
        return;
    } else if constexpr (MODE == CP_RETA_C) {
        // y = (V d)^; w^ = D^ - (V d)^ / lambda (= F(d - G V d)); Parseval: <w, d>, |w|^2 carry
        // the same 1/(nx ny) factor, which cancels in gamma = <w, d> / |w|^2
        const double k0sq = a.k0sq[b], eta = a.eta[b];
        const double xq = a.xi2[q];
        double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int m = 0; m < P; ++m) {
            const int p = t + T * m;
            const double lr = (a.xi2[p] + xq) - k0sq, li = -eta;
            const double inv = rcp_green(fma(lr, lr, li * li));
            const double2 D = a.D[mem + (size_t)p * N + q];
            const double2 w = csub(D, cmul(y[m], make_double2(lr * inv, -li * inv)));
            acc[0] += w.x * D.x + w.y * D.y;
            acc[1] += w.x * D.y - w.y * D.x;
            acc[2] += cnorm(w);
        }
        member_reduce<3, C * T>(a.ctl, b, bid % GROUPS, GROUPS, N, acc, [&](const double (&s)[3]) {
            finalize_gamma(a.ctl, b, s[0], s[1], s[2]);
        });
        return;
    } else {
        const double k0sq = a.k0sq[b], eta = a.eta[b];
        const double xq = a.xi2[q];
        double s_r = 0.0, s_x = 0.0;
        const double2* Ucur = (mstep & 1) ? a.U1 : a.U0;
        double2* Unext = (mstep & 1) ? a.U0 : a.U1;
#pragma unroll
        for (int m = 0; m < P; ++m) {
            const int p = t + T * m;
            // lambda = |xi|^2 - (k0^2 + i eta)  (symbol.cpp:58-67 + shift_symbol :97-100)
            const double lr = (a.xi2[p] + xq) - k0sq;
            const double li = -eta;
            if constexpr (MODE == CP_GREEN) {
                const double s = a.scale * rcp_green(fma(lr, lr, li * li));
                x[m] = cmul(y[m], make_double2(lr * s, -li * s));
            } else if constexpr (MODE == CP_LREF) {
                x[m] = cmul(y[m], make_double2(lr * a.scale, li * a.scale));
            } else {  // CP_SWEEP, CP_OPT_A
                const size_t idx = mem + (size_t)p * N + q;
                const double2 U = Ucur[idx];
                const double inv = rcp_green(fma(lr, lr, li * li));
                const double2 ginv = make_double2(lr * inv, -li * inv);      // 1/lambda
                const double2 xs = csub(cmul(y[m], ginv), U);                // r_bs^
                const double2 rs = csub(y[m], cmul(make_double2(lr, li), U)); // r^
                s_x += cnorm(xs);
                s_r += cnorm(rs);
                const double2 dir = a.direct ? rs : xs;  // iterate.cpp:118-123 direction
                if constexpr (MODE == CP_OPT_A) {
                    a.D[idx] = dir;
                    x[m] = dir;
                    // second line: r^ (Euclidean, NPBS) or L_ref d^ = lambda r^ (Direct)
                    y[m] = a.direct ? cmul(make_double2(lr, li), rs) : rs;
                } else {
                    double2 g = a.gamma;
                    if (a.map_kind == MK_FOURIER_DIAG) g = a.fd[(size_t)p * N + q];
                    const double2 Un = cadd(U, cmul(g, dir));
                    Unext[idx] = Un;
                    x[m] = Un;
                }
            }
        }
        if constexpr (MODE == CP_OPT_A) {
            if (!a.metric_reta) {  // T2 = F_x^-1 (second line) / (nx ny)
                double2 y2[P];
                Engine::template run<true>(y, y2, t, buf, a.tw, pol);
#pragma unroll
                for (int m = 0; m < P; ++m) a.T2[mem + (size_t)(t + T * m) * N + q] = cscale(y2[m], a.inv_npts);
            }
        }
        // inverse x-FFT -> T (scaled so the row kernel's inverse y-FFT is the physical field)
        Engine::template run<true>(x, y, t, buf, a.tw, pol);
        const double osc = (MODE == CP_SWEEP || MODE == CP_OPT_A) ? a.inv_npts : 1.0;
#pragma unroll
        for (int m = 0; m < P; ++m) a.T[mem + (size_t)(t + T * m) * N + q] = cscale(y[m], osc);

        if constexpr (MODE == CP_SWEEP || MODE == CP_OPT_A) {
            // CTA partial sums (fixed order), last CTA of the member finalises entry mstep
            __shared__ double red[2][C * T];
            red[0][threadIdx.x] = s_r;
            red[1][threadIdx.x] = s_x;
            __syncthreads();
            if (threadIdx.x == 0) {
                double r = 0.0, xx = 0.0;
                for (int k = 0; k < C * T; ++k) {
                    r += red[0][k];
                    xx += red[1][k];
                }
                const int g = bid % GROUPS;
                double* pr = a.ctl.partial + ((size_t)b * N + g) * kPartStride;
                pr[0] = r;
                pr[1] = xx;
                __threadfence();
                const unsigned old = atomicAdd(&a.ctl.counter[b], 1u);
                if (old == (unsigned)(GROUPS - 1)) {
                    __threadfence();
                    double sr = 0.0, sx = 0.0;
                    for (int k = 0; k < GROUPS; ++k) {
                        const double* pk = a.ctl.partial + ((size_t)b * N + k) * kPartStride;
                        sr += __ldcg(pk);
                        sx += __ldcg(pk + 1);
                    }
                    a.ctl.counter[b] = 0u;
                    // Parseval: ||v||^2 = sum |v^|^2 / (nx ny)
                    finalize_entry(a.ctl, b, mstep, sr * a.inv_npts, sx * a.inv_npts);
                }
            }
        }
    }
}

}  // namespace bs
