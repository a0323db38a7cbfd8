// cdr_kernels.cuh -- config c4 on sm_100a: convection-diffusion-reaction Born series, real fp64,
// Neumann cell-centred n x n grids, reference operator L0 = -Lap_N + sigma0 diagonalised by the
// DCT-II (proj/src/symbol.cpp:81-92, transforms.cpp:120-121,142-143), upwind first-order
// convection in V (no reference counterpart).
//
// Real data, packed: every complex engine line carries two real lines (rows 2e, 2e+1 in the row
// kernels; columns 2c, 2c+1 -- one 16-byte load -- in the column kernel).  DCT-II (REDFT10) and
// DCT-III (REDFT01) of a packed pair via ONE length-n complex FFT (Makhoul):
//   DCT-II : v_j = z_2j, v_{n-1-j} = z_{2j+1};  V = DFT(v);  Y_k = w_k V_k + conj(w_k) V_{n-k}
//   DCT-III: V_k = conj(w_k) (Y_k - i Y_{n-k});  v = DFT^-1(V) (unnormalised);
//            z_2j = v_j, z_{2j+1} = v_{n-1-j}            with w_k = exp(-i pi k / (2n)).
// V = L0 - A = (sigma0 - sigma) - b . grad_upwind is a stencil, so the source q = V u + f of the
// next sweep needs the neighbours of u^{m+1}: one sweep is three launches --
//   RC_A  T -> DCT-III rows = G q^m; x^m = G q^m - u^m (||x||^2 = R_eta norm); entry m and the
//         termination test; u^{m+1} = u^m + gamma x^m                       (48 B/pt real)
//   RC_B  u^{m+1} (+halo), b, sigma, f -> r^{m+1} = f - A u^{m+1} (||r||^2), q^{m+1} = V u + f,
//         DCT-II rows -> T                                                   (48 B/pt)
//   CC    T -> DCT-II columns, x 1/(4 n^2 lambda), DCT-III columns -> T       (16 B/pt)
#pragma once

#include "periodic_kernels.cuh"

#ifndef BS_CDR_PD
#define BS_CDR_PD 1  // RC_B operand prefetch distance (measured c4 RC_A+RC_B: 0 -> 620, 1 -> 570, 2 -> 657 us)
#endif

namespace bs {

template <int LOG2N, int PP = 16>
struct DctEngine {
    using G = Geom<LOG2N, PP>;
    using PS = FftPasses<LOG2N, PP>;
    static constexpr int N = G::N, P = G::P, T = G::T;

    // Stockham FFT of v (stride layout in registers); result W in buf (natural order)
    template <bool INVERSE, class Pol>
    __device__ __forceinline__ static void fft_to_smem(double2 (&v)[P], int t, double2* buf,
                                                       const double2* __restrict__ tw, const Pol& pol) {
        if (INVERSE) {
#pragma unroll
            for (int m = 0; m < P; ++m) v[m] = cconj(v[m]);
        }
        Dft<P>::template run<1>(v);
#pragma unroll
        for (int r = 0; r < P; ++r) buf[G::pidx(t * P + r)] = v[r];
        pol.sync();
        DstEngine<LOG2N, PP>::template pass<PS::R2, P>(buf, t, tw, pol);
        DstEngine<LOG2N, PP>::template pass<PS::R3, P * PS::R2>(buf, t, tw, pol);
        DstEngine<LOG2N, PP>::template pass<PS::R4, P * PS::R2 * PS::R3>(buf, t, tw, pol);
        DstEngine<LOG2N, PP>::template pass<PS::R5, P * PS::R2 * PS::R3 * PS::R4>(buf, t, tw, pol);
    }

    // REDFT10 of a packed pair: x, y in stride layout (x_{t+Tm})
    template <class Pol>
    __device__ __forceinline__ static void dct2(const double2 (&x)[P], double2 (&y)[P], int t,
                                                double2* buf, const double2* __restrict__ tw,
                                                const double2* __restrict__ w4, const Pol& pol) {
        double2 v[P];
#pragma unroll
        for (int m = 0; m < P; ++m) buf[G::pidx(t + T * m)] = x[m];
        pol.sync();
#pragma unroll
        for (int m = 0; m < P; ++m) {  // Makhoul permutation
            const int j = t + T * m;
            v[m] = buf[G::pidx(j < N / 2 ? 2 * j : 2 * (N - 1 - j) + 1)];
        }
        pol.sync();
        fft_to_smem<false>(v, t, buf, tw, pol);
#pragma unroll
        for (int m = 0; m < P; ++m) {
            const int k = t + T * m;
            const double2 w = __ldg(&w4[k]);
            const double2 a = buf[G::pidx(k)];
            const double2 b = buf[G::pidx((N - k) & (N - 1))];
            y[m] = cadd(cmul(w, a), cmul(cconj(w), b));
        }
        pol.sync();
    }

    // REDFT01 of a packed pair: y (stride layout) and its mirror ym[m] = y_{N - (t+Tm)} (0 at N)
    template <class Pol>
    __device__ __forceinline__ static void dct3(const double2 (&y)[P], const double2 (&ym)[P],
                                                double2 (&x)[P], int t, double2* buf,
                                                const double2* __restrict__ tw,
                                                const double2* __restrict__ w4, const Pol& pol) {
        double2 v[P];
#pragma unroll
        for (int m = 0; m < P; ++m) {
            const int k = t + T * m;
            const double2 w = cconj(__ldg(&w4[k]));
            v[m] = cmul(w, csub(y[m], mul_pi(ym[m])));  // conj(w) (Y_k - i Y_{N-k})
        }
        fft_to_smem<true>(v, t, buf, tw, pol);
#pragma unroll
        for (int m = 0; m < P; ++m) {  // inverse permutation; conj of the conj-trick FFT
            const int j = t + T * m;
            x[m] = cconj(buf[G::pidx((j & 1) ? N - 1 - (j >> 1) : (j >> 1))]);
        }
        pol.sync();
    }

    // REDFT01 of a packed pair whose spectrum Y already sits in buf (natural order)
    template <class Pol>
    __device__ __forceinline__ static void dct3_smem(double2 (&x)[P], int t, double2* buf,
                                                     const double2* __restrict__ tw,
                                                     const double2* __restrict__ w4, const Pol& pol) {
        double2 v[P];
#pragma unroll
        for (int m = 0; m < P; ++m) {
            const int k = t + T * m;
            const double2 w = cconj(__ldg(&w4[k]));
            const double2 ym = k ? buf[G::pidx(N - k)] : make_double2(0.0, 0.0);
            v[m] = cmul(w, csub(buf[G::pidx(k)], mul_pi(ym)));
        }
        pol.sync();
        fft_to_smem<true>(v, t, buf, tw, pol);
#pragma unroll
        for (int m = 0; m < P; ++m) {
            const int j = t + T * m;
            x[m] = cconj(buf[G::pidx((j & 1) ? N - 1 - (j >> 1) : (j >> 1))]);
        }
        pol.sync();
    }
};

enum CRowMode { RC_FWD = 0, RC_INV = 1, RC_A = 2, RC_B = 3 };
enum CColMode { CC_ONE = 0, CC_GREEN = 1, CC_INV = 2, CC_LREF = 3 };

struct CdrArgs {
    int batch;
    double h;                  // grid spacing (lx / n)
    const double* sigma0;      // [batch]
    const double* bx;          // real [batch][n][n]
    const double* by;
    const double* sigma;
    const double* f;
    const double* in;          // RC_FWD source (real)
    double* out;               // RC_INV output (real)
    const double* sub;         // RC_INV: optional field subtracted
    double* T;                 // real intermediate
    double* u0;                // iterate ping
    double* u1;                // iterate pong
    double* rnorm2;            // [batch] ||r^m||^2 handed from RC_B to RC_A
    const double* lapn;        // (4/h^2) sin^2(k pi / (2n)), k < n (Neumann symbol factor)
    const double2* tw;         // exp(-2 pi i k / n)
    const double2* w4;         // exp(-i pi k / (2n))
    double scale;
    double gamma;
    Control ctl;
};

// ------------------------------------------------------------------ row kernels (row pairs)
template <int LOG2N, int MODE, int NW, int PP>
__global__ void __launch_bounds__(NW * 32, (MinBlocks<NW * 32, PP >= 16 ? 128 : 80>::value))
crow_kernel(const CdrArgs a) {
    using G = Geom<LOG2N, PP>;
    using RG = RowGeom<LOG2N, PP, NW>;
    using Pol = typename PolicyFor<G::T>::type;
    using Eng = DctEngine<LOG2N, PP>;
    constexpr int N = G::N, P = G::P, T = G::T;
    constexpr int EPB = RG::EPB;
    constexpr int PAIRS = N / 2;
    extern __shared__ double2 smem[];

    const int t = threadIdx.x % T;
    const int e = threadIdx.x / T;
    const long gp = (long)blockIdx.x * EPB + e;          // global row pair
    const int b = (int)(gp / PAIRS);
    const int pr = (int)(gp % PAIRS);
    bool valid = b < a.batch;
    int m = 0;
    if ((MODE == RC_A || MODE == RC_B) && valid) {
        valid = __ldcg(&a.ctl.status[b]) == ST_ACTIVE;
        m = __ldcg(&a.ctl.sweep[b]);
    }
    if (!__syncthreads_or(valid)) return;
    double2* buf = smem + e * G::PAD_N;
    const Pol pol = make_policy((Pol*)nullptr, smem + EPB * G::PAD_N, e);
    const size_t rowA = ((size_t)(valid ? b : 0) * N + 2 * pr) * N;
    const size_t rowB = rowA + N;
    const double2 zero = make_double2(0.0, 0.0);
    double acc = 0.0;

    // Everything an engine reads sits in two adjacent rows (+ a halo row each side for the
    // RC_B stencil): one bulk L2 prefetch per array puts all of it in flight at once; the loads
    // below (RC_B stencil, RC_A u after the transform) then hit L2.
    const double* ucur = (m & 1) ? a.u1 : a.u0;
    const bool firstA = (2 * pr == 0), lastB = (2 * pr + 1 == N - 1);
    if ((MODE == RC_A || MODE == RC_B) && valid && t == 0) {
        constexpr unsigned R2 = 2 * N * sizeof(double);
        prefetch_l2(ucur + rowA, R2);
        if constexpr (MODE == RC_A) {
            prefetch_l2(a.T + rowA, R2);
        } else {
            prefetch_l2(a.bx + rowA, R2);
            prefetch_l2(a.by + rowA, R2);
            prefetch_l2(a.sigma + rowA, R2);
            prefetch_l2(a.f + rowA, R2);
            if (!firstA) prefetch_l2(ucur + rowA - N, R2 / 2);
            if (!lastB) prefetch_l2(ucur + rowB + N, R2 / 2);
        }
    }

    double2 q[P];
    if constexpr (MODE == RC_INV || MODE == RC_A) {
        double2 y[P], ym[P], z[P];
#pragma unroll
        for (int mm = 0; mm < P; ++mm) {
            const int k = t + T * mm;
            y[mm] = valid ? make_double2(a.T[rowA + k], a.T[rowB + k]) : zero;
            ym[mm] = (valid && k != 0) ? make_double2(a.T[rowA + N - k], a.T[rowB + N - k]) : zero;
        }
        Eng::dct3(y, ym, z, t, buf, a.tw, a.w4, pol);
#pragma unroll
        for (int mm = 0; mm < P; ++mm) {
            const int j = t + T * mm;
            if constexpr (MODE == RC_INV) {
                double2 o = cscale(z[mm], a.scale);
                if (a.sub && valid) o = csub(o, make_double2(a.sub[rowA + j], a.sub[rowB + j]));
                if (valid) {
                    a.out[rowA + j] = o.x;
                    a.out[rowB + j] = o.y;
                }
            } else {
                // RC_A: z = G q^m (scaled in CC); x = z - u^m; u^{m+1} = u^m + gamma x
                double* unext = (m & 1) ? a.u0 : a.u1;
                const double2 u = valid ? make_double2(ucur[rowA + j], ucur[rowB + j]) : zero;
                const double2 x = csub(z[mm], u);
                acc += cnorm(x);
                if (valid) {
                    unext[rowA + j] = u.x + a.gamma * x.x;
                    unext[rowB + j] = u.y + a.gamma * x.y;
                }
            }
        }
        if constexpr (MODE == RC_INV) return;
    } else {
        if constexpr (MODE == RC_FWD) {
#pragma unroll
            for (int mm = 0; mm < P; ++mm) {
                const int j = t + T * mm;
                q[mm] = valid ? make_double2(a.in[rowA + j], a.in[rowB + j]) : zero;
            }
        } else {
            // RC_B on u^m (m = sweep[b]): r = f - A u, q = V u + f, A = -Lap_N + conv + sigma,
            // V = (sigma0 - sigma) - conv; reflective ghosts (cell-centred Neumann).  The pair's
            // own values go through shared memory for the y-neighbours (j -+ 1); rows A and B
            // are each other's x-neighbour, so only the halo rows come from global memory.
#pragma unroll
            for (int mm = 0; mm < P; ++mm) {
                const int j = t + T * mm;
                q[mm] = valid ? make_double2(ucur[rowA + j], ucur[rowB + j]) : zero;
                buf[G::pidx(j)] = q[mm];
            }
            pol.sync();
            const double ih = 1.0 / a.h, ih2 = ih * ih;
            const double s0 = valid ? a.sigma0[b] : 0.0;
            // global operands of element mm, issued CDR_PD elements ahead of their use (like the
            // Dirichlet row kernel's element-wise pipeline); halo rows of the boundary pairs
            // are replaced by the reflective ghosts at use
            struct Op {
                double w, e, vx[2], vy[2], sg[2], ff[2];
            };
            auto load_op = [&](int mm) {
                Op o{};
                if (valid) {
                    const int j = t + T * mm;
                    o.w = firstA ? 0.0 : ucur[rowA - N + j];
                    o.e = lastB ? 0.0 : ucur[rowB + N + j];
#pragma unroll
                    for (int s = 0; s < 2; ++s) {
                        const size_t ix = (s ? rowB : rowA) + j;
                        o.vx[s] = a.bx[ix];
                        o.vy[s] = a.by[ix];
                        o.sg[s] = a.sigma[ix];
                        o.ff[s] = a.f[ix];
                    }
                }
                return o;
            };
            constexpr int PD = BS_CDR_PD < P ? BS_CDR_PD : P;
            Op ops[P];
#pragma unroll
            for (int mm = 0; mm < PD; ++mm) ops[mm] = load_op(mm);
#pragma unroll
            for (int mm = 0; mm < P; ++mm) {
                if (mm + PD < P) ops[mm + PD] = load_op(mm + PD);
                const int j = t + T * mm;
                const double2 c = q[mm];
                const double2 so = j > 0 ? buf[G::pidx(j - 1)] : c;
                const double2 no = j + 1 < N ? buf[G::pidx(j + 1)] : c;
                const Op& op = ops[mm];
                const double wA = (valid && !firstA) ? op.w : c.x, eB = (valid && !lastB) ? op.e : c.y;
                const double* vx = op.vx;
                const double* vy = op.vy;
                const double* sg = op.sg;
                const double* ff = op.ff;
                double res[2], qq[2];
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const double cv = s ? c.y : c.x;
                    const double w = s ? c.x : wA, e2 = s ? eB : c.y;
                    const double sv = s ? so.y : so.x, nv = s ? no.y : no.x;
                    const double lap = (4.0 * cv - w - e2 - sv - nv) * ih2;  // -Lap_N u
                    const double dx = vx[s] >= 0.0 ? (cv - w) * ih : (e2 - cv) * ih;
                    const double dy = vy[s] >= 0.0 ? (cv - sv) * ih : (nv - cv) * ih;
                    const double conv = vx[s] * dx + vy[s] * dy;
                    res[s] = ff[s] - ((lap + conv) + sg[s] * cv);
                    qq[s] = ((s0 - sg[s]) * cv - conv) + ff[s];
                }
                acc += res[0] * res[0] + res[1] * res[1];
                q[mm] = make_double2(qq[0], qq[1]);
            }
            pol.sync();  // buf is the transform's workspace next
        }
    }

    // forward DCT-II along the rows -> T (RC_FWD, RC_B)
    if constexpr (MODE == RC_FWD || MODE == RC_B) {
        double2 y[P];
        Eng::dct2(q, y, t, buf, a.tw, a.w4, pol);
#pragma unroll
        for (int mm = 0; mm < P; ++mm) {
            const int k = t + T * mm;
            if (valid) {
                a.T[rowA + k] = y[mm].x * a.scale;
                a.T[rowB + k] = y[mm].y * a.scale;
            }
        }
    }

    // per-pair partials -> member sums (deterministic), RC_B hands ||r||^2 to RC_A, RC_A records
    if constexpr (MODE == RC_A || MODE == RC_B) {
        acc = pol.sum(acc, t);
        int last = 0;
        if (valid && t == 0) {
            a.ctl.partial[((size_t)b * PAIRS + pr) * kPartStride] = acc;
            __threadfence();
            const unsigned old = atomicAdd(&a.ctl.counter[b], 1u);
            last = (old == (unsigned)(PAIRS - 1));
        }
        last = pol.bcast0(last, t);
        if (last) {
            __threadfence();
            double s = 0.0;
            for (int r = t; r < PAIRS; r += T) s += __ldcg(&a.ctl.partial[((size_t)b * PAIRS + r) * kPartStride]);
            s = pol.sum(s, t);
            if (t == 0) {
                a.ctl.counter[b] = 0u;
                if constexpr (MODE == RC_B) a.rnorm2[b] = s;
                else finalize_entry(a.ctl, b, m, __ldcg(&a.rnorm2[b]), s);
            }
        }
    }
}

// ------------------------------------------------------------------ column kernel (column pairs)
template <int LOG2N, int MODE, int C, int PP>
__global__ void __launch_bounds__(C * Geom<LOG2N, PP>::T, (MinBlocks<C * Geom<LOG2N, PP>::T, PP >= 16 ? 128 : 64>::value))
ccol_kernel(const CdrArgs a) {
    using G = Geom<LOG2N, PP>;
    using Eng = DctEngine<LOG2N, PP>;
    constexpr int N = G::N, P = G::P, T = G::T;
    extern __shared__ double2 smem[];
    int c, t;
    col_thread_map<G::T, C>(t, c);
    constexpr int GROUPS = N / (2 * C);  // C packed column pairs per CTA
    const int bid = BS_COL_REVERSE && a.batch > 1 ? gridDim.x - 1 - blockIdx.x : blockIdx.x;  // (col_kernel)
    const int b = bid / GROUPS;
    const int q0 = (bid % GROUPS) * 2 * C + 2 * c;  // real columns q0, q0 + 1
    if (a.ctl.status && __ldcg(&a.ctl.status[b]) != ST_ACTIVE) return;
    double2* buf = smem + c * G::PAD_N;
    const BlockSeg<T, C> pol{smem + C * G::PAD_N, c};
    const size_t mem = (size_t)b * N * N;
    double2* Tp = reinterpret_cast<double2*>(a.T);
    const size_t col = (mem + q0) / 2;  // double2 index of (row 0, columns q0..q0+1)
    constexpr size_t LS = N / 2;         // row stride in double2

    double2 x[P], y[P];
    if constexpr (MODE == CC_INV) {
        double2 ym[P];
#pragma unroll
        for (int mm = 0; mm < P; ++mm) {
            const int k = t + T * mm;
            x[mm] = Tp[col + (size_t)k * LS];
            ym[mm] = k ? Tp[col + (size_t)(N - k) * LS] : make_double2(0.0, 0.0);
        }
        Eng::dct3(x, ym, y, t, buf, a.tw, a.w4, pol);
#pragma unroll
        for (int mm = 0; mm < P; ++mm) Tp[col + (size_t)(t + T * mm) * LS] = cscale(y[mm], a.scale);
        return;
    } else {
#pragma unroll
        for (int mm = 0; mm < P; ++mm) x[mm] = Tp[col + (size_t)(t + T * mm) * LS];
        Eng::dct2(x, y, t, buf, a.tw, a.w4, pol);
        if constexpr (MODE == CC_ONE) {
#pragma unroll
            for (int mm = 0; mm < P; ++mm) Tp[col + (size_t)(t + T * mm) * LS] = cscale(y[mm], a.scale);
            return;
        } else {
            // lambda_pq = (a_p + a_q) + sigma0, real; the pair carries columns q0 (re), q0+1 (im)
            const double s0 = a.sigma0[b];
            const double la = a.lapn[q0], lb = a.lapn[q0 + 1];
#pragma unroll
            for (int mm = 0; mm < P; ++mm) {
                const int p = t + T * mm;
                const double lre = (a.lapn[p] + la) + s0, lim = (a.lapn[p] + lb) + s0;
                if constexpr (MODE == CC_GREEN)  // lambda >= sigma0 > 0: reciprocal + Newton
                    y[mm] = make_double2(y[mm].x * (a.scale * rcp_green(lre)), y[mm].y * (a.scale * rcp_green(lim)));
                else
                    y[mm] = make_double2(y[mm].x * (a.scale * lre), y[mm].y * (a.scale * lim));
                buf[G::pidx(p)] = y[mm];
            }
            pol.sync();
            Eng::dct3_smem(x, t, buf, a.tw, a.w4, pol);
#pragma unroll
            for (int mm = 0; mm < P; ++mm) Tp[col + (size_t)(t + T * mm) * LS] = x[mm];
        }
    }
}

}  // namespace bs
