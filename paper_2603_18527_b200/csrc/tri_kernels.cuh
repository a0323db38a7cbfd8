// tri_kernels.cuh -- the Green column pass as a batched Toeplitz tridiagonal solve (sm_100a).
//
// The Dirichlet symbol is separable and its x factor a_p = (4/h^2) sin^2(p pi / 2n)
// (proj/src/symbol.cpp:69-80) is exactly the spectrum of the three-point second difference
// with zero ends.  After the row pass has taken y into the DST basis, the column pass
//     forward x-DST -> x 1/lambda_pq -> inverse x-DST           (symbol.cpp:19-39, Divide)
// is therefore, column q by column q, the solve
//     (-D_xx + a_q - k0^2 - i eta) z = r,   z_0 = z_n = 0,
// i.e. h^2-scaled: d z_i - z_{i-1} - z_{i+1} = h^2 r_i with d = 2 + h^2 (a_q - k0^2 - i eta).
// Same operator, O(n) work per column instead of two length-n transforms: ~20 FP64
// instructions per point instead of ~80, and the column never leaves registers except for a
// handful of boundary values.  d lies off the real segment [-2, 2] (eta > 0), so the
// elimination needs no pivoting and is backward stable.
//
// Parallel algorithm (one thread = one segment of P = 16 consecutive rows of one column):
//   row 16s of each segment is a separator X_s (X_0 = z_0 = 0, X_S = z_n = 0); rows
//   16s+1 .. 16s+15 are the segment interior, a 15 x 15 Toeplitz system with the separators
//   as boundary values.  With p_k the LU pivots 1/u_k of that system (u_1 = d,
//   u_k = d - p_{k-1}), delta = p_15 and gamma = prod p_k (the corner entries of its inverse):
//     1. each thread eliminates its interior downwards and upwards (zero boundaries) ->
//        zp_15, zp_1;
//     2. the separators satisfy the reduced Toeplitz system
//          (d - 2 delta) X_s - gamma (X_{s-1} + X_{s+1}) = h^2 r_{16s} + zp^{s-1}_15 + zp^s_1,
//        solved by its own LU pivots pr_s as two first-order linear recurrences, each an
//        affine-map scan across the segments (warp shuffles; chunk carries through shared
//        memory for n >= 1024);
//     3. each thread re-runs its elimination with the separators added and back-substitutes.
// The pivot tables (p_1..p_15, gamma, pr_1..pr_{S-1} per column and member) depend on the
// medium only through (k0, eta): tri_setup_kernel builds them when the medium is set.
// Deterministic: fixed operation order, batch members independent (bit-identical to single
// runs).
#pragma once

#include "sweep_kernels.cuh"

namespace bs {

constexpr int kTriP = 16;  // rows per segment
#ifndef TRI_THREADS
#define TRI_THREADS 256  // threads per CTA (n < 4096)
#endif
#ifndef TRI_REV
#define TRI_REV 1
#endif

template <int LOG2N>
struct TriGeom {
    static constexpr int N = 1 << LOG2N;
    static constexpr int S = N / kTriP;                  // segments per column
    static constexpr int C = S >= TRI_THREADS ? 2 : TRI_THREADS / S;  // columns per CTA
    static constexpr int THREADS = C * S;
    static constexpr int CW = C < 8 ? C : 8;             // columns side by side in a warp (16*CW-B rows)
    static constexpr int SPW = 32 / CW;                  // segments per warp (load phase)
    static constexpr int WPG = S / SPW;                  // warps per column group
    static constexpr int TS = 16 + S;                    // table entries per column (double2)
    // shared-memory row pitches, odd in 16-B units: the CW columns a warp reads at one index
    // land on distinct bank groups (pitch TS = 48 put all 8 on one group: 8-way conflicts)
    static constexpr int TSP = TS + 1;
    // Neumann (CDR) lines: + p'_15 and the 15 upward pivots of the last segment's system
    static constexpr int TSN = TS + 16;
    static constexpr int SP = S + 1;
    static constexpr int LPC = S < 32 ? S : 32;          // lanes per column (reduced phase)
    static constexpr int CH = S / LPC;                   // warps per column (reduced phase)
    static_assert(S >= SPW, "tridiagonal column pass needs n >= 64");
};

__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {  // a*b + c
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

// Pivot tables, one thread per (member, line).  Lines: 2-D columns q (a_t = a_q); 3-D x-lines
// (y, z) (a_t = a_y + a_z).  Entry layout per line: [0..14] p_1..p_15, [15] gamma,
// [16 + s] pr_s (pr_0 = 0).  Dirichlet zero lines (q = 0; y = 0 or z = 0) get zeros.
static __global__ void tri_setup_kernel(const double* __restrict__ lap, const double* __restrict__ k0sq,
                                 const double* __restrict__ eta, double h2, int batch, int log2n,
                                 int dim, double2* __restrict__ tab) {
    const int n = 1 << log2n, S = n / kTriP, TS = 16 + S;
    const long lines = (long)batch << ((dim - 1) * log2n);
    const long idx = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (idx >= lines) return;
    const int b = (int)(idx >> ((dim - 1) * log2n));
    const long l = idx & ((1L << ((dim - 1) * log2n)) - 1);
    double2* t = tab + idx * TS;
    bool zero;
    double at;
    if (dim == 2) {
        zero = l == 0;
        at = lap[l];
    } else {
        const int y = (int)(l >> log2n), z = (int)(l & (n - 1));
        zero = y == 0 || z == 0;
        at = lap[y] + lap[z];
    }
    if (zero) {
        for (int k = 0; k < TS; ++k) t[k] = make_double2(0.0, 0.0);
        return;
    }
    const double dr = 2.0 + h2 * (at - k0sq[b]), di = -h2 * eta[b];
    auto rcp = [](double x, double y) {
        const double den = x * x + y * y;
        return make_double2(x / den, -y / den);
    };
    double2 p = rcp(dr, di), g = p;
    t[0] = p;
    for (int k = 1; k < kTriP - 1; ++k) {
        p = rcp(dr - p.x, di - p.y);
        g = cmul(g, p);
        t[k] = p;
    }
    t[15] = g;
    // reduced system: D X_s - gamma (X_{s-1} + X_{s+1}); u_1 = D, u_s = D - gamma^2 pr_{s-1}
    const double2 D = make_double2(dr - 2.0 * p.x, di - 2.0 * p.y);
    const double2 g2 = cmul(g, g);
    t[16] = make_double2(0.0, 0.0);
    double2 pr = make_double2(0.0, 0.0);
    for (int s = 1; s < S; ++s) {
        const double2 gp = cmul(g2, pr);
        pr = rcp(D.x - gp.x, D.y - gp.y);
        t[16 + s] = pr;
    }
}

// Neumann pivot tables (CL_CDR), one thread per (member, real column q), written into the
// .x (q even) / .y (q odd) component of the pair's entries.  Layout per pair: [0..14] p_1..p_15,
// [15] gamma, [16 + s] pr_s (s = 0..S-1, modified first / last diagonals), [16 + S] p'_15,
// [17 + S + k] q'_{k+1} (k = 0..14).
static __global__ void tri_setup_neumann_kernel(const double* __restrict__ lapn, const double* __restrict__ sigma0,
                                                double h2, int batch, int log2n, double2* __restrict__ tab) {
    const int n = 1 << log2n, S = n / kTriP, TS = 32 + S;
    const long idx = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (idx >= ((long)batch << log2n)) return;
    const int b = (int)(idx >> log2n), q = (int)(idx & (n - 1));
    double* t = reinterpret_cast<double*>(tab + ((size_t)b * (n / 2) + q / 2) * TS) + (q & 1);
    auto at = [&](int k) -> double& { return t[2 * k]; };
    const double d = 2.0 + h2 * (lapn[q] + sigma0[b]);
    double p = 1.0 / d, g = p, p14 = 0.0;
    at(0) = p;
    for (int k = 1; k < kTriP - 1; ++k) {
        if (k == kTriP - 2) p14 = p;
        p = 1.0 / (d - p);
        g *= p;
        at(k) = p;
    }
    at(15) = g;
    const double delta = p;
    double qk = 1.0 / (d - 1.0);
    at(17 + S) = qk;
    for (int k = 1; k < kTriP - 1; ++k) {
        qk = 1.0 / (d - qk);
        at(17 + S + k) = qk;
    }
    const double deltap = qk;
    at(16 + S) = 1.0 / (d - 1.0 - p14);
    double pr = 0.0;
    for (int s = 0; s < S; ++s) {
        const double D = s == 0 ? d - 1.0 - delta : (s == S - 1 ? d - delta - deltap : d - 2.0 * delta);
        pr = 1.0 / (D - g * g * pr);
        at(16 + s) = pr;
    }
}

// cp.async (16 B, L2 only) global -> shared
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
// same with an L2 eviction-priority policy (sweep_kernels.cuh l2_policy_*); bit 4 of BS_L2_HINTS
__device__ __forceinline__ void cp_async16_hint(void* smem, const void* gmem, unsigned long long pol) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Tile = C adjacent lines (columns) of one plane, all n rows.  Shared-memory tile layout:
// element (row r, column c) at e + e / (16 C), e = r C + c -- one pad slot per 16 rows, so the
// 16-row segments a warp reads (SPW segments x CW columns per load) fall on distinct bank
// groups for every C.
template <int LOG2N, bool NEU = false>
struct TriTile {
    using G = TriGeom<LOG2N>;
    static constexpr int TB = G::C * G::N + G::N / kTriP;   // tile buffer (double2)
    static constexpr int TSX = NEU ? G::TSN : G::TS;        // table entries per line
    static constexpr int TSXP = TSX + 1;                    // shared pitch (odd)
    static constexpr size_t SMEM =
        sizeof(double2) * ((size_t)TB + 2 * (size_t)G::C * TSXP + 3 * (size_t)G::C * G::SP + 2 * (size_t)G::C * G::CH);
    __device__ __forceinline__ static int sidx(int r, int c) {
        const int e = r * G::C + c;
        return e + e / (kTriP * G::C);
    }
};

// Line-tile addressing per layout.  CL_PLANE (2-D): tile (b, q0): lines = columns q0..q0+C-1
// of member b, row stride n, table lines b n + q.  CL_X3 (3-D x-lines): tile (b, y, z0): lines
// (y, z0..z0+C-1), row (= x) stride n^2, table lines (b n + y) n + z; the padding y-plane is
// skipped (its lines are the Dirichlet zero).  CL_SLAB (a rank's n x slab_cols column block
// after the forward all-to-all, batch 1): tile qa0: block columns qa0..qa0+C-1, row stride
// slab_cols; global lines col0 + qa (2-D) or, with slab3, the (y, z) pairs col0 n + qa (3-D).
// CL_CDR (config c4, real n x n fields): a line is a pair of adjacent real columns (one 16-B
// double2 per row, the DCT route's packing), n / 2 pairs per member, row stride n / 2.
template <int LOG2N, int LAYOUT>
struct TriLines {
    static constexpr int N = 1 << LOG2N, C = TriGeom<LOG2N>::C, GROUPS = N / C;
    int b, q0, yl;
    size_t base, tline, ls;
    bool skip;
    __device__ __forceinline__ static long count(const ColArgs& a) {
        if constexpr (LAYOUT == CL_SLAB) return a.slab_cols / C;
        if constexpr (LAYOUT == CL_CDR) return (long)a.batch * (N / 2 >= C ? N / 2 / C : 1);
        return LAYOUT == CL_X3 ? (long)a.batch * N * GROUPS : (long)a.batch * GROUPS;
    }
    __device__ __forceinline__ TriLines(long t, const ColArgs& a) {
        q0 = (int)(t % GROUPS) * C;
        ls = LAYOUT == CL_X3 ? (size_t)N * N : (size_t)N;
        if constexpr (LAYOUT == CL_CDR) {
            constexpr int PG = N / 2 >= C ? N / 2 / C : 1;  // pair groups per member (launch needs n/2 >= C)
            b = (int)(t / PG);
            q0 = (int)(t % PG) * C;  // pair index
            yl = 0;
            ls = N / 2;
            base = ((size_t)b << (2 * LOG2N - 1)) + q0;
            tline = (size_t)b * (N / 2) + q0;
            skip = false;
        } else if constexpr (LAYOUT == CL_SLAB) {
            q0 = (int)t * C;  // block column
            b = 0;
            yl = 0;
            ls = (size_t)a.slab_cols;
            base = q0;
            tline = (a.slab3 ? (size_t)a.col0 * N : (size_t)a.col0) + q0;
            skip = false;
        } else if constexpr (LAYOUT == CL_X3) {
            const long g = t / GROUPS;  // (b, y)
            b = (int)(g >> LOG2N);
            yl = (int)(g & (N - 1));
            base = ((size_t)b << (3 * LOG2N)) + (size_t)yl * N + q0;
            tline = (size_t)g * N + q0;
            skip = yl == 0;
        } else {
            b = (int)(t / GROUPS);
            yl = 0;
            base = ((size_t)b << (2 * LOG2N)) + q0;
            tline = (size_t)b * N + q0;
            skip = false;
        }
    }
};

// Persistent CTAs over the line tiles (grid = resident CTAs).  Per tile: its n x C values and
// pivot table were prefetched by cp.async while the previous tile was solved; the CTA copies
// them into registers, immediately prefetches the next tile into the same buffer, solves, and
// stores straight from registers.  Load phase mapping: warp w, lane l -> column
// (w / WPG) CW + l mod CW, segment (w mod WPG) SPW + l / CW.  Reduced phase: thread t ->
// column t / S, segment t mod S (a column's segments on consecutive lanes).
//
// NEU (config c4, CL_CDR): the real Neumann system of the cell-centred grid, d = 2 + h^2 (a_q +
// sigma0) with d - 1 in the first and last rows (reflective ghosts; the DCT-II spectrum of
// symbol.cpp:81-92).  Each line carries two real columns, so every operation is component-wise.
// X_0 = z_0 is an unknown separator (reduced diagonal d - 1 - delta), and the last segment's
// interior ends in the modified row (its own last pivot p'_15, upward pivots q'_k, corner
// delta'; reduced diagonal d - delta - delta').  The reduced pivots of tri_setup_neumann_kernel
// carry the modified diagonals, so the scans are the Dirichlet ones.
template <bool NEU>
__device__ __forceinline__ double2 tmul(double2 a, double2 b) {
    if constexpr (NEU) return make_double2(a.x * b.x, a.y * b.y);
    else return cmul(a, b);
}
template <bool NEU>
__device__ __forceinline__ double2 tfma(double2 a, double2 b, double2 c) {
    if constexpr (NEU) return make_double2(fma(a.x, b.x, c.x), fma(a.y, b.y, c.y));
    else return cfma(a, b, c);
}

template <int LOG2N, int LAYOUT, bool NEU = false>
__global__ void __launch_bounds__(TriGeom<LOG2N>::THREADS, TriGeom<LOG2N>::THREADS >= 512 ? 1 : 2)
tri_kernel(const ColArgs a) {
    using G = TriGeom<LOG2N>;
    using TT = TriTile<LOG2N, NEU>;
    using TL = TriLines<LOG2N, LAYOUT>;
    constexpr int N = G::N, S = G::S, C = G::C, TS = TT::TSX, TSP = TT::TSXP, SP = G::SP, LPC = G::LPC,
                  CH = G::CH;
    static_assert(LAYOUT == CL_PLANE || LAYOUT == CL_X3 || LAYOUT == CL_SLAB || LAYOUT == CL_CDR, "layout");
    static_assert(NEU == (LAYOUT == CL_CDR), "Neumann lines are CDR column pairs");
    extern __shared__ double2 sm[];
    double2* tbuf = sm;                    // [TB] tile
    double2* tabs = tbuf + TT::TB;         // [2][C][TSP] pivot tables (double-buffered)
    double2* red = tabs + 2 * C * TSP;     // [C][SP] h^2 r_sep + zp_1
    double2* zl = red + C * SP;            // [C][SP] zp_15
    double2* xs = zl + C * SP;             // [C][SP] separators (X_S = 0 at [S])
    double2* tot = xs + C * SP;            // [C][CH] chunk maps (A, B)

    [[maybe_unused]] const unsigned long long keep_pol =
        BS_L2_KEEP_T ? ((a.l2_hints & 4) ? l2_policy_last() : l2_policy_normal()) : 0ull;
    const long ntiles = TL::count(a);
    // reversed order on multi-plane launches: start on the row pass's L2-resident tail
    const bool rev = TRI_REV && (LAYOUT == CL_CDR ? a.batch > 1 : col_reversed<LAYOUT == CL_X3 ? CL_PLANE : LAYOUT>(a));
    auto tile_at = [&](long k) { return rev ? ntiles - 1 - k : k; };
    auto issue = [&](long k, int tb) {
        const TL ln(tile_at(k), a);
        const double2* src = a.T + ln.base;
#pragma unroll 4
        for (int e = threadIdx.x; e < C * N; e += G::THREADS) {
#if BS_L2_KEEP_T
            if (LAYOUT == CL_PLANE)
                cp_async16_hint(tbuf + e + e / (kTriP * C), src + (size_t)(e / C) * ln.ls + (e % C), keep_pol);
            else
#endif
            cp_async16(tbuf + e + e / (kTriP * C), src + (size_t)(e / C) * ln.ls + (e % C));
        }
        const double2* ts = a.tri + ln.tline * TS;
        double2* td = tabs + tb * C * TSP;
        for (int k2 = threadIdx.x; k2 < C * TS; k2 += G::THREADS) cp_async16(td + (k2 / TS) * TSP + k2 % TS, ts + k2);
    };


    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int c = (w / G::WPG) * G::CW + lane % G::CW;
    const int s = (w % G::WPG) * G::SPW + lane / G::CW;
    const int cr = threadIdx.x / S, sr = threadIdx.x % S, ls = sr % LPC, ch = sr / LPC;
    const double2 zero = make_double2(0.0, 0.0);
    const double sc = a.tri_scale;

    long k = blockIdx.x;
    if (k < ntiles) issue(k, 0);
    cp_async_commit();
    for (int it = 0; k < ntiles; k += gridDim.x, ++it) {
        // member status: issued before the tile wait so its round trip overlaps it
        const int stv = a.status ? __ldcg(&a.status[TL(tile_at(k), a).b]) : (int)ST_ACTIVE;
        cp_async_wait_all();
        // ONE decision per CTA: another CTA may finalise this member's entry (status -> DONE)
        // while this CTA's warps read the status, and warps that disagreed took different paths
        // around the barriers below -- in a persistent CTA that corrupted the tiles it solved
        // next, i.e. other members (found by the waves determinism stress, r02j: members next to
        // an early-terminating one converged sweeps late or never).  A member seen DONE by any
        // thread is done: skipping its tile is always safe.
        const bool tile_active = __syncthreads_and(stv == (int)ST_ACTIVE) != 0;
        double2 v[kTriP];
#pragma unroll
        for (int i = 0; i < kTriP; ++i) v[i] = tbuf[TT::sidx(kTriP * s + i, c)];
        __syncthreads();  // tile buffer free: prefetch the next tile under this one's solve
        if (k + gridDim.x < ntiles) issue(k + gridDim.x, (it + 1) & 1);
        cp_async_commit();

        const long t = tile_at(k);
        const TL ln(t, a);
        if (ln.skip) continue;
        if (a.status) {
            const bool active = tile_active;  // read before finalising, uniform over the CTA
            if constexpr (LAYOUT == CL_PLANE)
                if (a.finalize && active && ln.q0 == 0 && threadIdx.x < 32) finalize_member(a, ln.b, 1 << a.fin_lsh);
            if (!active) continue;  // uniform per CTA
        }
        const double2* tab = tabs + (it & 1) * C * TSP;

        // 1. zero-boundary eliminations of the interior, downwards and upwards (shared pivots)
        const double2* pt = tab + c * TSP;
        // Neumann: the last segment eliminates upwards with its own pivots and ends on p'_15
        const bool lastseg = NEU && s == S - 1;
        const double2* pu = lastseg ? pt + 17 + S : pt;
        const double2 plast = lastseg ? pt[16 + S] : pt[kTriP - 2];
        {
            double2 yd = v[1], yu = v[kTriP - 1];
#pragma unroll
            for (int j = 1; j < kTriP - 1; ++j) {
                yd = tfma<NEU>(pt[j - 1], yd, v[1 + j]);
                yu = tfma<NEU>(NEU ? pu[j - 1] : pt[j - 1], yu, v[kTriP - 1 - j]);
            }
            zl[c * SP + s] = tmul<NEU>(plast, yd);
            red[c * SP + s] = tfma<NEU>(NEU ? pu[kTriP - 2] : plast, yu, v[0]);
        }
        __syncthreads();

        // 2. reduced system: forward recurrence y_s = gamma pr_{s-1} y_{s-1} + rr_s, then
        //    X_s = gamma pr_s X_{s+1} + pr_s y_s, each as an inclusive affine-map scan
        {
            const double2* tr = tab + cr * TSP;
            const double2 gam = tr[15];
            const double2 prs = tr[16 + sr];
            const double2 prm = sr > 0 ? tr[16 + sr - 1] : zero;
            double2 A = tmul<NEU>(gam, prm);
            double2 B = sr > 0 ? cadd(red[cr * SP + sr], zl[cr * SP + sr - 1]) : (NEU ? red[cr * SP] : zero);
#pragma unroll
            for (int d = 1; d < LPC; d <<= 1) {
                const double ax = __shfl_up_sync(0xffffffffu, A.x, d, LPC), ay = __shfl_up_sync(0xffffffffu, A.y, d, LPC);
                const double bx = __shfl_up_sync(0xffffffffu, B.x, d, LPC), by = __shfl_up_sync(0xffffffffu, B.y, d, LPC);
                if (ls >= d) {
                    B = tfma<NEU>(A, make_double2(bx, by), B);
                    A = tmul<NEU>(A, make_double2(ax, ay));
                }
            }
            double2 y = B;
            if constexpr (CH > 1) {
                if (ls == LPC - 1) {
                    tot[(cr * CH + ch) * 2] = A;
                    tot[(cr * CH + ch) * 2 + 1] = B;
                }
                __syncthreads();
                double2 yc = zero;  // y at the end of the previous chunk
                for (int j = 0; j < ch; ++j) yc = tfma<NEU>(tot[(cr * CH + j) * 2], yc, tot[(cr * CH + j) * 2 + 1]);
                y = tfma<NEU>(A, yc, B);
                __syncthreads();  // tot reused below
            }
            A = tmul<NEU>(gam, prs);
            B = tmul<NEU>(prs, y);
#pragma unroll
            for (int d = 1; d < LPC; d <<= 1) {
                const double ax = __shfl_down_sync(0xffffffffu, A.x, d, LPC), ay = __shfl_down_sync(0xffffffffu, A.y, d, LPC);
                const double bx = __shfl_down_sync(0xffffffffu, B.x, d, LPC), by = __shfl_down_sync(0xffffffffu, B.y, d, LPC);
                if (ls + d < LPC) {
                    B = tfma<NEU>(A, make_double2(bx, by), B);
                    A = tmul<NEU>(A, make_double2(ax, ay));
                }
            }
            double2 X = B;
            if constexpr (CH > 1) {
                if (ls == 0) {
                    tot[(cr * CH + ch) * 2] = A;
                    tot[(cr * CH + ch) * 2 + 1] = B;
                }
                __syncthreads();
                double2 xc = zero;  // X at the start of the next chunk
                for (int j = CH - 1; j > ch; --j) xc = tfma<NEU>(tot[(cr * CH + j) * 2], xc, tot[(cr * CH + j) * 2 + 1]);
                X = tfma<NEU>(A, xc, B);
            }
            xs[cr * SP + sr] = X;
            if (sr == S - 1) xs[cr * SP + S] = zero;
        }
        __syncthreads();

        // 3. elimination with the separators as boundary values, back substitution, store
        const double2 xl = xs[c * SP + s], xr = xs[c * SP + s + 1];
        v[1] = cadd(v[1], xl);
#pragma unroll
        for (int i = 2; i < kTriP; ++i) v[i] = tfma<NEU>(pt[i - 2], v[i - 1], v[i]);
        v[kTriP - 1] = tmul<NEU>(plast, cadd(v[kTriP - 1], xr));  // (Neumann last segment: xr = X_S = 0)
#pragma unroll
        for (int i = kTriP - 2; i >= 1; --i) v[i] = tmul<NEU>(pt[i - 1], cadd(v[i], v[i + 1]));
        v[0] = xl;
        // Dirichlet zero line (2-D: q = 0; 3-D: z = 0): its table is zero, store zeros explicitly
        // (on a slab the zero lines' all-zero tables already give zeros)
        const bool zc = LAYOUT != CL_SLAB && LAYOUT != CL_CDR && ln.q0 + c == 0;
        if constexpr (LAYOUT == CL_SLAB) {
            if (a.xchg_on) {
                // fused inverse exchange: row j belongs to source rank j >> xchg_log2r; stored into
                // that rank's t_rows at block xchg_rank (same element map as col_group's st_out)
                const int rr = a.xchg_log2r;
#pragma unroll
                for (int i = 0; i < kTriP; ++i) {
                    const int j = kTriP * s + i;
                    a.xchg[j >> rr][(((size_t)a.xchg_rank << rr) + (size_t)(j & ((1 << rr) - 1))) * ln.ls + ln.q0 + c] =
                        cscale(v[i], sc);
                }
                continue;
            }
        }
        double2* col = a.T + ln.base + (size_t)(kTriP * s) * ln.ls + c;
#pragma unroll
        for (int i = 0; i < kTriP; ++i) {
            if (LAYOUT == CL_PLANE) st_keep<(BS_L2_KEEP_T != 0)>(&col[(size_t)i * ln.ls], zc ? zero : cscale(v[i], sc), keep_pol);
            else col[(size_t)i * ln.ls] = zc ? zero : cscale(v[i], sc);
        }
    }
    cp_async_wait_all();
}

}  // namespace bs
