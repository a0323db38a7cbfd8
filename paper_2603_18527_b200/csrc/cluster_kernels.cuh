// cluster_kernels.cuh -- whole-solve persistent kernel for small grids (config c0: 127^2).
//
// A 128^2 (or 64^2) padded grid fits in the distributed shared memory of ONE thread-block
// cluster: CL = n / 8 CTAs (16 for n = 128, the non-portable maximum; 8 for n = 64), CTA r owns
// rows 8r .. 8r+7 of u (ping-pong), k^2, f and the transform intermediate T in its shared
// memory.  The kernel runs bp::run's whole sweep loop (iterate.cpp:88-153) on the device, one
// cluster per member, with two cluster barriers per sweep and no launch in between -- the c0
// solve was latency-bound at two launches (~30 us) per 127^2 sweep.
//
// Per sweep m (same arithmetic as row_kernel<R_SWEEP> + tri_kernel):
//   rows   (one 16-lane engine per row, DstEngine<L, 8>): T -> inverse y-DST = G q^m; r_bs =
//          G q^m - u^m; r^m = f - A u^m (five-point; the rows next to a CTA boundary read the
//          neighbour's u^m row through DSMEM); u^{m+1} = u^m + gamma d; q^{m+1} = V u^{m+1} + f;
//          forward y-DST -> T; per-CTA partial sums of |r|^2 and |r_bs|^2
//   cluster barrier A; every CTA sums the CL partials in rank order (identical in every CTA),
//          rank 0 records trace entry m and the termination test (finalize_entry); every CTA
//          takes the same decision from its own copy (a ring of the last 21 entries)
//   columns (one thread per column, the tridiagonal x-solve of tri_kernels.cuh with 8-row
//          segments = one segment per CTA): zero-boundary eliminations of the CTA's 7 interior
//          rows; cluster barrier B; the 16-unknown reduced system read from every CTA's shared
//          memory and solved by plain Thomas (pivots from the CTA's table); back substitution.
#pragma once

#include <cooperative_groups.h>

#include "tri_kernels.cuh"

namespace bs {

constexpr int kClRows = 8;  // rows per CTA = tridiagonal segment length

template <int LOG2N>
struct ClGeom {
    static constexpr int N = 1 << LOG2N;
    static constexpr int CL = N / kClRows;     // CTAs per cluster (= segments per column)
    using G = Geom<LOG2N, 8>;                  // P = 8 points per engine thread
    static constexpr int T = G::T;             // engine threads
    static constexpr int THREADS = kClRows * T;  // == N: one thread per column in the column pass
    static constexpr int TSC = kClRows + CL;   // table: p_1..p_7, gamma, pr_0..pr_{CL-1}
    static constexpr int TSCP = TSC + 1;
    static constexpr int RN = kClRows * N;     // one field block
    // U[2], K2, F, TT (RN each), engine lines, table, red/zl, partials + entry ring
    static constexpr size_t SMEM = sizeof(double2) * ((size_t)5 * RN + (size_t)kClRows * G::PAD_N +
                                                      (size_t)N * TSCP + 2 * (size_t)CL * N + 4 * (size_t)N + 32);
    static_assert(THREADS == N, "one column per thread");
};

struct ClArgs {
    ColArgs col;   // tri_scale, k0sq, eta, lap
    RowArgs row;   // u0/u1, k2, f, T, tw, sinp, inv_h2, map, gamma, ctl
    double h2;     // h^2 (tridiagonal pivots)
    int direct;    // IterFormat::Direct: the update direction is r
};

template <int LOG2N>
__global__ void __launch_bounds__(ClGeom<LOG2N>::THREADS, 1) cluster_solve_kernel(const ClArgs ca) {
    namespace cg = cooperative_groups;
    using CGm = ClGeom<LOG2N>;
    using G = typename CGm::G;
    using Engine = DstEngine<LOG2N, 8>;
    constexpr int N = CGm::N, CL = CGm::CL, T = CGm::T, P = G::P, R = kClRows, RN = CGm::RN;
    constexpr int TSCP = CGm::TSCP;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int b = blockIdx.x / CL;
    const RowArgs& a = ca.row;
    const Control& c = a.ctl;

    extern __shared__ double2 csm[];
    double2* U = csm;                    // [2][R][N]
    double2* K2 = U + 2 * RN;            // [R][N]
    double2* F = K2 + RN;                // [R][N]
    double2* TT = F + RN;                // [R][N]
    double2* LB = TT + RN;               // [R][PAD_N] engine lines
    double2* TAB = LB + R * G::PAD_N;    // [N][TSCP]
    // [2][CL][N]: every segment's b_sep + zp_1 and zp_7, pushed by its CTA into every CTA of the
    // cluster (DSMEM stores need no round trip; the reduced solve then reads locally)
    double2* RED = TAB + N * TSCP;
    // [0..1] this CTA's entry sums (read by every CTA between barriers A and B), [4..24] ring of
    // the last 21 entries (local), [32..47] the row engines' partials (local: RED may still be
    // read by a slower CTA's reduced solve while this CTA runs the next row pass)
    // [2 parity][2][N]: u rows of the neighbours (above, below), pushed by them when written
    double2* HALO = RED + 2 * CL * N;
    double* PS = reinterpret_cast<double*>(HALO + 4 * N);

    const int tid = threadIdx.x;
    const size_t mem = (size_t)b * N * N;
    const int row0 = rank * R;
    const double2 zero = make_double2(0.0, 0.0);

    // ---- load the member's rows; pivot table (thread = column)
    for (int k = tid; k < N; k += CGm::THREADS) {  // u^0 halo rows (global rows 8r - 1, 8r + 8)
        HALO[k] = row0 > 0 ? a.u0[mem + (size_t)(row0 - 1) * N + k] : zero;
        HALO[N + k] = row0 + R < N ? a.u0[mem + (size_t)(row0 + R) * N + k] : zero;
        HALO[2 * N + k] = zero;  // parity 1: pushed by the neighbours (zero at the grid edges)
        HALO[3 * N + k] = zero;
    }
    for (int k = tid; k < RN; k += CGm::THREADS) {
        const size_t g = mem + (size_t)row0 * N + k;
        U[k] = a.u0[g];
        U[RN + k] = zero;
        K2[k] = a.k2[g];
        F[k] = a.f[g];
        TT[k] = a.T[g];
    }
    const double k0sq = ca.col.k0sq[b], eta = ca.col.eta[b];
    {
        const int q = tid;
        double2* t = TAB + q * TSCP;
        if (q == 0) {
            for (int k = 0; k < CGm::TSC; ++k) t[k] = zero;
        } else {
            const double dr = 2.0 + ca.h2 * (ca.col.lap[q] - k0sq), di = -ca.h2 * eta;
            auto rcp = [](double x, double y) {
                const double den = x * x + y * y;
                return make_double2(x / den, -y / den);
            };
            double2 p = rcp(dr, di), gm = p;
            t[0] = p;
            for (int k = 1; k < R - 1; ++k) {
                p = rcp(dr - p.x, di - p.y);
                gm = cmul(gm, p);
                t[k] = p;
            }
            t[R - 1] = gm;
            const double2 D = make_double2(dr - 2.0 * p.x, di - 2.0 * p.y), g2 = cmul(gm, gm);
            double2 pr = zero;
            t[R] = zero;  // pr_0 = 0: X_0 = z_0 = 0
            for (int s = 1; s < CL; ++s) {
                const double2 gp = cmul(g2, pr);
                pr = rcp(D.x - gp.x, D.y - gp.y);
                t[R + s] = pr;
            }
        }
    }
    cluster.sync();

    const int e = tid / T, t = tid % T;        // row engine
    const int gi = row0 + e;                   // global row
    const bool vrow = gi > 0;                  // row 0 is the Dirichlet padding
    double2* buf = LB + e * G::PAD_N;
    const WarpSeg<T> pol{};
    const double sc = ca.col.tri_scale;
    const double2 shift = make_double2(k0sq, eta);
    int m = 0;
    for (;; ++m) {
        double2* uc = U + (m & 1) * RN;
        double2* un = U + ((m + 1) & 1) * RN;
        // neighbour rows of the stencil (u^m), pushed by the previous / next CTA
        const double2* up = HALO + (m & 1) * 2 * N;
        const double2* dn = up + N;

        // ---- inverse y-DST of the row (T -> G q^m), natural order back in buf
        double2 y[P];
#pragma unroll
        for (int mm = 0; mm < P; ++mm) buf[t + T * mm] = TT[e * N + t + T * mm];
        pol.sync();
        {
            double2 v[P];
            Engine::template run_smem<true>(v, y, t, buf, a.tw, a.sinp, pol);
        }
#pragma unroll
        for (int l = 0; l < P; ++l) buf[G::at_block(t, G::pidx(t * P), l)] = y[l];
        pol.sync();
        double s0 = 0.0, s1 = 0.0;
        double2 q[P];
#pragma unroll
        for (int mm = 0; mm < P; ++mm) {
            const int j = t + T * mm;
            const double2 zz = buf[G::at_stride(t, G::pidx(t), mm)];
            const double2 u = uc[e * N + j], k2 = K2[e * N + j], f = F[e * N + j];
            const double2 V = csub(k2, shift);
            const double2 un_ = e > 0 ? uc[(e - 1) * N + j] : up[j];
            const double2 us_ = e < R - 1 ? uc[(e + 1) * N + j] : dn[j];
            const double2 uw = j > 0 ? uc[e * N + j - 1] : zero;
            const double2 ue = j + 1 < N ? uc[e * N + j + 1] : zero;
            double2 s = cscale(u, 4.0);
            s = csub(s, un_);
            s = csub(s, us_);
            s = csub(s, uw);
            s = csub(s, ue);
            const double2 r = csub(f, csub(cscale(s, a.inv_h2), cmul(k2, u)));
            const double2 x = csub(zz, u);
            if (j != 0 && vrow) {
                s0 += cnorm(r);
                s1 += cnorm(x);
            }
            double2 g = a.gamma;
            if (a.map_kind == MK_POINTWISE) g = cscale(mul_pi(V), 1.0 / eta);
            double2 unew = cadd(u, cmul(g, ca.direct ? r : x));
            if (j == 0 || !vrow) unew = zero;
            un[e * N + j] = unew;
            // edge rows of u^{m+1} -> the neighbours' halo (parity m+1), read next sweep
            if (e == 0 && rank > 0) cluster.map_shared_rank(HALO, rank - 1)[((m + 1) & 1) * 2 * N + N + j] = unew;
            if (e == R - 1 && rank < CL - 1) cluster.map_shared_rank(HALO, rank + 1)[((m + 1) & 1) * 2 * N + j] = unew;
            q[mm] = (j == 0 || !vrow) ? zero : cadd(cmul(V, unew), f);
        }
        s0 = pol.sum(s0, t);
        s1 = pol.sum(s1, t);
        pol.sync();
#pragma unroll
        for (int mm = 0; mm < P; ++mm) buf[t + T * mm] = q[mm];
        pol.sync();
        {
            double2 v[P], y2[P];
            Engine::template run_smem<true>(v, y2, t, buf, a.tw, a.sinp, pol);
#pragma unroll
            for (int l = 0; l < P; ++l) TT[e * N + t * P + l] = vrow ? y2[l] : zero;
        }
        // per-CTA partials in engine (row) order
        if (t == 0) {
            PS[32 + 2 * e] = s0;
            PS[33 + 2 * e] = s1;
        }
        __syncthreads();
        if (tid == 0) {
            double a0 = 0.0, a1 = 0.0;
            for (int k = 0; k < R; ++k) {
                a0 += PS[32 + 2 * k];
                a1 += PS[33 + 2 * k];
            }
            PS[0] = a0;
            PS[1] = a1;
        }
        cluster.sync();  // A: partials + u^{m+1} visible cluster-wide

        // ---- trace entry m (identical decision in every CTA; rank 0 records it)
        // warp 0 gathers the CL partials (lane k <- rank k, one DSMEM round trip) and reduces
        // them by a fixed xor tree: the same order, hence the same bits, in every CTA
        if (tid < 32) {
            double v0 = 0.0, v1 = 0.0;
            if (tid < CL) {
                const double* ps = cluster.map_shared_rank(PS, tid);
                v0 = ps[0];
                v1 = ps[1];
            }
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) {
                v0 += __shfl_xor_sync(0xffffffffu, v0, d);
                v1 += __shfl_xor_sync(0xffffffffu, v1, d);
            }
            if (tid == 0) {
                PS[2] = v0;
                PS[3] = v1;
            }
        }
        __syncthreads();
        const double sl2 = PS[2], sre = PS[3];
        const double rel = sqrt(sl2) / c.fnorm_l2[b];
        double* ring = PS + 4;  // rel of entries m - 20 .. m (ring of 21)
        int term = -1;
        if (m == 0) {
            if (rel <= c.rtol) term = 0;
        } else {
            if (!isfinite(rel) || rel > 1e8) term = 2;
            else if (rel <= c.rtol) term = 0;
            else if (m + 1 > 20) {
                const double past = ring[(m - 20) % 21];
                if (fabs(past - rel) < 1e-14 * fmax(1.0, past)) term = 3;
            }
        }
        if (term < 0 && m >= c.max_iters) term = 1;
        __syncthreads();  // every thread read the ring before thread 0 updates it
        if (tid == 0) {
            ring[m % 21] = rel;
            if (rank == 0) finalize_entry(c, b, m, sl2, sre);
        }
        if (term >= 0) break;

        // ---- column pass on T (thread = column, this CTA = segment `rank`)
        {
            const int qc = tid;
            const double2* pt = TAB + qc * TSCP;
            double2 v[R];
#pragma unroll
            for (int i = 0; i < R; ++i) v[i] = TT[i * N + qc];
            double2 yd = v[1], yu = v[R - 1];
#pragma unroll
            for (int k = 1; k < R - 1; ++k) {
                yd = cfma(pt[k - 1], yd, v[1 + k]);
                yu = cfma(pt[k - 1], yu, v[R - 1 - k]);
            }
            const double2 pl = pt[R - 2];
            const double2 rsep = cfma(pl, yu, v[0]);  // b_sep + zp_1
            const double2 rz7 = cmul(pl, yd);         // zp_7
#pragma unroll 4
            for (int k = 0; k < CL; ++k) {
                double2* dst = cluster.map_shared_rank(RED, k);
                dst[rank * N + qc] = rsep;
                dst[(CL + rank) * N + qc] = rz7;
            }
            cluster.sync();                // B: every segment's boundary data visible
            // reduced system over the CL separators (X_0 = 0 = X_CL): Thomas with the pivots
            const double2 gam = pt[R - 1];
            double2 yv[CL];
            yv[0] = zero;
#pragma unroll
            for (int s = 1; s < CL; ++s) yv[s] = cadd(RED[s * N + qc], RED[(CL + s - 1) * N + qc]);
#pragma unroll
            for (int s = 1; s < CL; ++s) yv[s] = cfma(cmul(gam, pt[R + s - 1]), yv[s - 1], yv[s]);
            double2 Xn = zero, X = zero, Xr = zero;  // X_{s+1} while walking down
#pragma unroll
            for (int s = CL - 1; s >= 1; --s) {
                const double2 prs = pt[R + s];
                const double2 Xs = cfma(cmul(gam, prs), Xn, cmul(prs, yv[s]));
                if (s == rank) X = Xs;
                if (s == rank + 1) Xr = Xs;
                Xn = Xs;
            }
            // back substitution of this segment with the separators as boundary values
            v[1] = cadd(v[1], X);
#pragma unroll
            for (int i = 2; i < R; ++i) v[i] = cfma(pt[i - 2], v[i - 1], v[i]);
            v[R - 1] = cmul(pl, cadd(v[R - 1], Xr));
#pragma unroll
            for (int i = R - 2; i >= 1; --i) v[i] = cmul(pt[i - 1], cadd(v[i], v[i + 1]));
            v[0] = X;
#pragma unroll
            for (int i = 0; i < R; ++i) TT[i * N + qc] = qc == 0 ? zero : cscale(v[i], sc);
        }
        __syncthreads();
    }
    // result u^m (buffer m & 1, finalize_entry's result_buf) -> the handle's ping / pong field
    double2* dst = (m & 1) ? a.u1 : a.u0;
    const double2* src = U + (m & 1) * RN;
    for (int k = tid; k < RN; k += CGm::THREADS) dst[mem + (size_t)row0 * N + k] = src[k];
    cluster.sync();  // no CTA exits while its shared memory may still be read
}

}  // namespace bs
