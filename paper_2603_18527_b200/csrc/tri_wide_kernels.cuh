// tri_wide_kernels.cuh -- the tridiagonal Green column pass (tri_kernels.cuh) for long lines
// (n >= 2048): one WIDE tile of 8 columns per 4-CTA thread-block cluster (sm_100a).
//
// Why: with n >= 2048 a CTA's shared memory holds two columns (n x 2 x 16 B = 128 KB at n = 4096),
// so tri_kernel's tile rows are 32 B: every warp-level cp.async / store touches 16 distinct
// sectors, and the source-level ncu of the c2 pass put 51 % of its stall samples on issuing them
// (LSU address divergence; profiles/r02h/c2_tri_hot.txt) -- 0.41 of HBM peak against 0.65-0.77 for
// the 8-column tiles of n = 512.
//
// Here the cluster's four CTAs (four SMs) share an n x 8 tile BY ROWS: CTA r holds rows
// [r n/4, (r+1) n/4) of all 8 columns -- whole 128-B lines, 4 rows per warp instruction, loaded
// by cp.async and stored straight from registers -- i.e. n/64 of the 16-row segments of every
// column.  The segment eliminations (phases 1 and 3 of tri_kernel) are local to a segment, so
// only the reduced system crosses CTAs: each CTA scans its own segments and publishes the affine
// maps of its 32-segment chunks (2 per column at n = 4096) into every CTA's shared memory
// (DSMEM, 16 B x 2 per chunk), one cluster barrier per scan direction.  zp_15 of the segment
// above a CTA's first one is recomputed locally from 16 halo rows (no barrier); the separator
// below its last one is the backward scan's carry.  The next tile is prefetched under the solve
// as in tri_kernel.  Arithmetic and operation order are tri_kernel's: results are bit-identical.
// A first version that split the tile by COLUMNS (each CTA gathering its two columns' segments
// from the owners' shared memory) moved the whole tile through DSMEM in 32-B pieces and was
// slower than tri_kernel (c2: 396 vs 234 us).  2-D whole members (CL_PLANE), Dirichlet lines.
#pragma once

#include <cooperative_groups.h>

#include "tri_kernels.cuh"

namespace bs {

#ifndef BS_TRIW_CLW
#define BS_TRIW_CLW 4  // CTAs per cluster (8: half the rows per CTA, two CTAs per SM)
#endif

template <int LOG2N>
struct TriWide {
    static constexpr int N = 1 << LOG2N;
    static constexpr int S = N / kTriP;            // segments per column
    static constexpr int CLW = BS_TRIW_CLW;        // CTAs per cluster
    static constexpr int WC = 8;                   // columns per wide tile (128-B rows)
    static constexpr int ROWS = N / CLW;           // rows held per CTA
    static constexpr int SL = ROWS / kTriP;        // segments per CTA and column
    static constexpr int THREADS = WC * SL;        // one thread per (column, local segment)
    static constexpr int LPC = SL < 32 ? SL : 32;  // lanes per chunk (reduced phase)
    static constexpr int CHL = SL / LPC;           // chunks per CTA and column
    static constexpr int CH = CHL * CLW;           // chunks per column
    static constexpr int TROWS = ROWS + kTriP;     // + the halo segment above the CTA's rows
    static constexpr int TB = TROWS * WC + TROWS / kTriP;  // padded tile (double2): one slot per 16 rows
    static constexpr int TSL = 16 + SL + 1;        // table entries held per column: p_1..15, gamma, pr_{s0-1 .. s0+SL-1}
    static constexpr int TSP = TSL | 1;            // odd pitch
    static constexpr int SP = SL + 2;              // [zl of the halo segment | SL local | X below the last]
    static constexpr size_t SMEM =
        sizeof(double2) * ((size_t)TB + 2 * (size_t)WC * TSP + 3 * (size_t)WC * SP + 2 * 2 * (size_t)WC * CH);
    static_assert(SL >= 4 && THREADS <= 1024 && LPC == 32, "wide tiles need n >= 2048");
    // tile row tr (0 .. TROWS-1; the halo segment first), column col -> padded slot
    __device__ __forceinline__ static int sidx(int tr, int col) {
        const int e = tr * WC + col;
        return e + e / (kTriP * WC);
    }
};

template <int LOG2N>
__global__ void __launch_bounds__(TriWide<LOG2N>::THREADS, TriWide<LOG2N>::THREADS <= 256 ? 2 : 1)
tri_wide_kernel(const ColArgs a) {
    namespace cg = cooperative_groups;
    using TW = TriWide<LOG2N>;
    constexpr int N = TW::N, S = TW::S, WC = TW::WC, ROWS = TW::ROWS, SL = TW::SL, CLW = TW::CLW;
    constexpr int LPC = TW::LPC, CHL = TW::CHL, CH = TW::CH, TSP = TW::TSP, SP = TW::SP;
    constexpr int TS = 16 + S;  // table entries per column in global memory (tri_setup_kernel)
    extern __shared__ double2 sm[];
    double2* tbuf = sm;                     // [TB] halo segment + this CTA's rows of the wide tile
    double2* tabs = tbuf + TW::TB;          // [2][WC][TSP] pivot tables (double-buffered)
    double2* red = tabs + 2 * WC * TSP;     // [WC][SP]
    double2* zl = red + WC * SP;            // [WC][SP]   ([0] = the halo segment's zp_15)
    double2* xs = zl + WC * SP;             // [WC][SP]   ([SL] = the separator below the last segment)
    double2* totf = xs + WC * SP;           // [WC][CH][2] forward chunk maps of the whole column
    double2* totb = totf + 2 * WC * CH;     // [WC][CH][2] backward chunk maps
    __shared__ int flag[2];                 // member status of this / the next tile, read by rank 0

    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const long ncl = gridDim.x / CLW, cid = blockIdx.x / CLW;
    const long ntiles = (long)a.batch * (N / WC);
    const bool rev = TRI_REV && col_reversed<CL_PLANE>(a);
    auto tile_at = [&](long k) { return rev ? ntiles - 1 - k : k; };
    auto member_of = [&](long k) { return (int)(tile_at(k) / (N / WC)); };
    const int s0 = rank * SL;  // first global segment of this CTA

    // next tile -> shared memory (tile rows incl. the halo segment, the table slices)
    auto issue = [&](long k, int tb) {
        const long t = tile_at(k);
        const int b = (int)(t / (N / WC)), q0w = (int)(t % (N / WC)) * WC;
        const double2* src = a.T + ((size_t)b << (2 * LOG2N)) + q0w;
        const int r0 = rank * ROWS - kTriP;  // global row of tile row 0 (rank 0: its halo is skipped)
#pragma unroll 4
        for (int e = threadIdx.x + (rank == 0 ? kTriP * WC : 0); e < TW::TROWS * WC; e += TW::THREADS)
            cp_async16(tbuf + e + e / (kTriP * WC), src + (size_t)(r0 + e / WC) * N + (e % WC));
        const double2* ts = a.tri + ((size_t)b * N + q0w) * TS;
        double2* td = tabs + tb * WC * TSP;
        for (int k2 = threadIdx.x; k2 < WC * TW::TSL; k2 += TW::THREADS) {
            const int col = k2 / TW::TSL, j = k2 % TW::TSL;
            // j < 16: p_1..15, gamma; j >= 16: pr_{s0 - 1 + (j - 16)} (rank 0: pr_{-1} unused)
            const int g = j < 16 ? j : 16 + s0 - 1 + (j - 16);
            if (g >= 16 || j < 16) cp_async16(td + col * TSP + j, ts + (size_t)col * TS + (g < 0 ? 0 : g));
        }
    };

    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int c = lane % WC;                       // load / solve mapping: 8 columns side by side
    const int sl = w * (32 / WC) + lane / WC;      //   x 4 segments per warp
    const int cr = threadIdx.x / SL, srl = threadIdx.x % SL;  // reduced mapping: a column's segments on
    const int ls = srl % LPC, chl = srl / LPC;                //   consecutive lanes
    const int sr = s0 + srl, ch = rank * CHL + chl;           // global segment / chunk
    const double2 zero = make_double2(0.0, 0.0);
    const double sc = a.tri_scale;

    long k = cid;
    if (k < ntiles) issue(k, 0);
    cp_async_commit();
    if (rank == 0 && threadIdx.x < CLW && k < ntiles)
        *cluster.map_shared_rank(&flag[0], threadIdx.x) = a.status ? __ldcg(&a.status[member_of(k)]) : (int)ST_ACTIVE;
    cluster.sync();
    for (int it = 0; k < ntiles; k += ncl, ++it) {
        const long t = tile_at(k);
        const int b = (int)(t / (N / WC)), q0w = (int)(t % (N / WC)) * WC;
        // One status decision per cluster (rank 0 read it; flag[it & 1] arrived with the previous
        // tile's barrier): another cluster finalising the member may flip it at any time, and the
        // four CTAs must take the same branch around the cluster barriers.
        const bool active = flag[it & 1] == ST_ACTIVE;
        const bool more = k + ncl < ntiles;
        if (rank == 0 && threadIdx.x < CLW && more)  // the next tile's status, delivered by this tile's barrier
            *cluster.map_shared_rank(&flag[(it + 1) & 1], threadIdx.x) =
                a.status ? __ldcg(&a.status[member_of(k + ncl)]) : (int)ST_ACTIVE;
        if (a.status && a.finalize && active && rank == 0 && q0w == 0 && threadIdx.x < 32)
            finalize_member(a, b, 1 << a.fin_lsh);
        cp_async_wait_all();
        __syncthreads();
        double2 v[kTriP], hv = zero;
        if (active) {
#pragma unroll
            for (int i = 0; i < kTriP; ++i) v[i] = tbuf[TW::sidx(kTriP * (sl + 1) + i, c)];
        }
        const double2* tab = tabs + (it & 1) * WC * TSP;
        const double2* pt = tab + c * TSP;
        const double2 plast = pt[kTriP - 2];
        if (active && sl == 0 && rank > 0) {
            // zp_15 of the segment above this CTA's first one, from the halo rows (the same
            // downward elimination its owner runs)
            double2 yd = tbuf[TW::sidx(1, c)];
#pragma unroll
            for (int j = 1; j < kTriP - 1; ++j) yd = cfma(pt[j - 1], yd, tbuf[TW::sidx(1 + j, c)]);
            hv = cmul(plast, yd);
        }
        __syncthreads();  // tile buffer free: prefetch the next tile under this one's solve
        if (more) issue(k + ncl, (it + 1) & 1);
        cp_async_commit();
        if (!active) {
            cluster.sync();  // delivers the next tile's status
            continue;
        }

        // 1. zero-boundary eliminations of the interior, downwards and upwards
        {
            double2 yd = v[1], yu = v[kTriP - 1];
#pragma unroll
            for (int j = 1; j < kTriP - 1; ++j) {
                yd = cfma(pt[j - 1], yd, v[1 + j]);
                yu = cfma(pt[j - 1], yu, v[kTriP - 1 - j]);
            }
            zl[c * SP + sl + 1] = cmul(plast, yd);
            red[c * SP + sl + 1] = cfma(plast, yu, v[0]);
            if (sl == 0) zl[c * SP] = hv;
        }
        __syncthreads();

        // 2. reduced system: y_s = gamma pr_{s-1} y_{s-1} + rr_s forwards, X_s = gamma pr_s X_{s+1} +
        //    pr_s y_s backwards, each a warp scan of affine maps per chunk + the fold of the
        //    column's chunk maps (this CTA's and its peers') in tri_kernel's order
        {
            const double2* tr = tab + cr * TSP;
            const double2 gam = tr[15];
            const double2 prs = tr[16 + 1 + srl];           // pr_{sr}
            const double2 prm = sr > 0 ? tr[16 + srl] : zero;  // pr_{sr-1}
            double2 A = cmul(gam, prm);
            double2 B = sr > 0 ? cadd(red[cr * SP + srl + 1], zl[cr * SP + srl]) : zero;
#pragma unroll
            for (int d = 1; d < LPC; d <<= 1) {
                const double ax = __shfl_up_sync(0xffffffffu, A.x, d, LPC), ay = __shfl_up_sync(0xffffffffu, A.y, d, LPC);
                const double bx = __shfl_up_sync(0xffffffffu, B.x, d, LPC), by = __shfl_up_sync(0xffffffffu, B.y, d, LPC);
                if (ls >= d) {
                    B = cfma(A, make_double2(bx, by), B);
                    A = cmul(A, make_double2(ax, ay));
                }
            }
            if (ls == LPC - 1) {
#pragma unroll
                for (int r = 0; r < CLW; ++r) {
                    double2* dst = cluster.map_shared_rank(totf, r) + (cr * CH + ch) * 2;
                    dst[0] = A;
                    dst[1] = B;
                }
            }
            cluster.sync();  // forward chunk maps of the whole column (+ the next tile's status)
            double2 yc = zero;  // y at the end of the previous chunk
            for (int j = 0; j < ch; ++j) yc = cfma(totf[(cr * CH + j) * 2], yc, totf[(cr * CH + j) * 2 + 1]);
            const double2 y = cfma(A, yc, B);
            A = cmul(gam, prs);
            B = cmul(prs, y);
#pragma unroll
            for (int d = 1; d < LPC; d <<= 1) {
                const double ax = __shfl_down_sync(0xffffffffu, A.x, d, LPC), ay = __shfl_down_sync(0xffffffffu, A.y, d, LPC);
                const double bx = __shfl_down_sync(0xffffffffu, B.x, d, LPC), by = __shfl_down_sync(0xffffffffu, B.y, d, LPC);
                if (ls + d < LPC) {
                    B = cfma(A, make_double2(bx, by), B);
                    A = cmul(A, make_double2(ax, ay));
                }
            }
            if (ls == 0) {
#pragma unroll
                for (int r = 0; r < CLW; ++r) {
                    double2* dst = cluster.map_shared_rank(totb, r) + (cr * CH + ch) * 2;
                    dst[0] = A;
                    dst[1] = B;
                }
            }
            cluster.sync();  // backward chunk maps of the whole column
            double2 xc = zero;  // X at the start of the next chunk (X_S = 0 after the last one)
            for (int j = CH - 1; j > ch; --j) xc = cfma(totb[(cr * CH + j) * 2], xc, totb[(cr * CH + j) * 2 + 1]);
            xs[cr * SP + srl] = cfma(A, xc, B);
            if (srl == SL - 1) xs[cr * SP + SL] = xc;  // the separator below this CTA's last segment
        }
        __syncthreads();

        // 3. elimination with the separators as boundary values, back substitution, store
        const double2 xl = xs[c * SP + sl], xr = xs[c * SP + sl + 1];
        v[1] = cadd(v[1], xl);
#pragma unroll
        for (int i = 2; i < kTriP; ++i) v[i] = cfma(pt[i - 2], v[i - 1], v[i]);
        v[kTriP - 1] = cmul(plast, cadd(v[kTriP - 1], xr));
#pragma unroll
        for (int i = kTriP - 2; i >= 1; --i) v[i] = cmul(pt[i - 1], cadd(v[i], v[i + 1]));
        v[0] = xl;
        const bool zc = q0w + c == 0;  // the Dirichlet zero column: its table is zero, store zeros
        double2* col = a.T + ((size_t)b << (2 * LOG2N)) + (size_t)(kTriP * (s0 + sl)) * N + q0w + c;
#pragma unroll
        for (int i = 0; i < kTriP; ++i) col[(size_t)i * N] = zc ? zero : cscale(v[i], sc);
        __syncthreads();  // red / zl / xs are free for the next tile
    }
    cp_async_wait_all();
    // no CTA may exit while a peer can still address its shared memory
    cluster.sync();
}

}  // namespace bs
