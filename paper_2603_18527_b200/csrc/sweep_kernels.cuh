// sweep_kernels.cuh -- fused Born-sweep kernels for sm_100a (fp64 complex).
//
// HBM layout (per member b of the batch, "padded" n x n with n = nx+1 = 2^LOG2N):
//   element (ix, iy) of the reference's dense nx*ny field lives at [(ix+1)*n + (iy+1)];
//   row 0 and column 0 are the Dirichlet zero nodes.  Every field buffer has one extra
//   zero row at its end so the five-point stencil of the last member reads zeros.
//   Rows are 16*n bytes (128-B aligned); the DST-I engine's x_0 slot is column 0.
//
// Per sweep (two launches, 128 algorithmic bytes per grid point):
//   row kernel   (96 B/pt)  T -> inverse y-DST -> G q^m;  r_bs = G q^m - u^m;
//                           ||r_bs||^2 (= ||G r^m||^2, the R_eta norm, by the key identity
//                           PAPER.md:149-156); ||f - A u^m||^2 (five-point stencil);
//                           u^{m+1} = u^m + gamma r_bs;  q^{m+1} = V u^{m+1} + f;
//                           forward y-DST -> T;  last row of a member finalises the
//                           trace entry m and the termination test of proj/src/iterate.cpp:134-150.
//   column kernel (32 B/pt) T -> forward x-DST -> x 4/(n^2 lambda) -> inverse x-DST -> T.
#pragma once

#include "dst_engine.cuh"

#ifndef BS_SHFL_MIRROR
#define BS_SHFL_MIRROR 1
#endif
#ifndef BS_COL_SMEM_MIRROR
#define BS_COL_SMEM_MIRROR 1
#endif
#ifndef BS_ROW_SMEM
#define BS_ROW_SMEM 1
#endif
// element-wise phase of the row kernel: operands (u, k2, f, stencil neighbours) are loaded
// BS_EW_PD elements ahead of their use, so a warp keeps several row segments in flight
// instead of waiting one L2 round trip per element (r01 ncu: 65 % of the long-scoreboard
// stalls were the stencil operands consumed right after their loads)
#ifndef BS_EW_PD
#define BS_EW_PD 2
#endif
// shared-memory staging of G q / the next source also for single-warp 2-D rows (frees the
// 64 registers of z[] / q[] for the prefetched operands)
// register budget of the row kernel (128: 2 CTAs of 8 warps per SM; 85: 3 CTAs)
#ifndef BS_ROW_REGS
#define BS_ROW_REGS 128
#endif
#ifndef BS_COL_LD256
#define BS_COL_LD256 1  // 256-bit paired-column loads in the 2-column (n >= 2048) column kernel
#endif
#ifndef BS_ROW_FWD_DENSE
#define BS_ROW_FWD_DENSE 1
#endif
#ifndef BS_COL_WIDE
#define BS_COL_WIDE 1  // warp-contiguous engines + named barriers for 2-column CTAs (n >= 2048)
#endif
#ifndef BS_RSM_ALL
#define BS_RSM_ALL 1
#endif

namespace bs {

// Row-kernel modes.  Per sweep the driver launches (SC = scalar / pointwise map,
// L2 / RE = OptimalScalar Euclidean / R_eta, FD = FourierDiag):
//   SC: R_SWEEP, C_GREEN
//   L2: R_OPT_A, R_OPT_B, C_GREEN
//   RE: R_RETA_A, C_GREEN, R_RETA_C, R_OPT_B, C_GREEN
//   FD: R_FD_A, C_FD, R_FD_B, C_GREEN
enum RowMode {
    R_FWD = 0,       // in -> forward y-DST -> T
    R_FWD_BORN = 1,  // V in + f -> forward -> T
    R_INV = 2,       // T -> inverse -> out (- sub)
    R_SWEEP = 3,     // fused scalar/pointwise sweep (entry m, update, next source)
    R_OPT_A = 4,     // entry m; x = r_bs -> X; <w,r>, |w|^2 with w = A x = r - V x -> gamma
    R_OPT_B = 5,     // u' = u + gamma X; q = V u' + f -> forward -> T
    R_RETA_A = 6,    // entry m; x = r_bs -> X; V x -> forward -> T (for G V x)
    R_RETA_C = 7,    // T -> inverse = G V x; w = x - G V x; <w,x>, |w|^2 -> gamma
    R_FD_A = 8,      // entry m; x = r_bs -> forward -> T (for the FourierDiag multiply)
    R_FD_B = 9,      // T -> inverse = du; u' = u + du; q = V u' + f -> forward -> T
    R_SWEEP_D = 10,  // R_SWEEP with IterFormat::Direct: the update direction is r^m itself
};
enum ColMode { C_ONE = 0, C_GREEN = 1, C_LREF = 2, C_FD = 3 };
enum Status { ST_ACTIVE = 0, ST_DONE = 1 };
enum MapKind { MK_SCALAR = 0, MK_OPTIMAL = 1, MK_FOURIER_DIAG = 2, MK_POINTWISE = 3 };
constexpr int kPartStride = 8;  // doubles of per-row partial sums

template <int MODE>
struct RowSpec {
    static constexpr bool SWEEP = MODE == R_SWEEP || MODE == R_SWEEP_D;
    static constexpr bool INV = MODE == R_INV || SWEEP || MODE == R_OPT_A ||
                                MODE == R_RETA_A || MODE == R_RETA_C || MODE == R_FD_A || MODE == R_FD_B;
    static constexpr bool FWD = MODE == R_FWD || MODE == R_FWD_BORN || SWEEP ||
                                MODE == R_OPT_B || MODE == R_RETA_A || MODE == R_FD_A || MODE == R_FD_B;
    // records trace entry m = sweep[b] (and the termination test)
    static constexpr bool ENTRY = SWEEP || MODE == R_OPT_A || MODE == R_RETA_A || MODE == R_FD_A;
    // runs after the entry of this sweep was recorded: m = sweep[b] - 1
    static constexpr bool POST = MODE == R_OPT_B || MODE == R_RETA_C || MODE == R_FD_B;
    static constexpr bool ITER = ENTRY || POST;
    static constexpr bool GAMMA = MODE == R_OPT_A || MODE == R_RETA_C;  // reduces a gamma
    static constexpr int NPART = MODE == R_OPT_A ? 5 : MODE == R_RETA_C ? 3 : ENTRY ? 2 : 0;
    static constexpr bool UPDATE = SWEEP || MODE == R_OPT_B || MODE == R_FD_B;
};

constexpr int kMaxXchg = 8;  // ranks of a fused-exchange slab group

struct Control {
    int* status;          // [batch]
    int* sweep;           // [batch] next trace entry to record
    unsigned* counter;    // [batch] rows finished in the current launch
    int* iters;           // [batch]
    int* term;            // [batch]
    int* result_buf;      // [batch] ping-pong index holding the result
    int* n_active;        // [1]
    double* partial;      // [batch][n][kPartStride] per-row partial sums
    double2* gamma;       // [batch] optimal-scalar gamma of the current sweep
    const double* fnorm_l2;
    const double* fnorm_reta;
    double* trace_l2;     // [batch][max_iters+1]
    double* trace_reta;
    int trace_stride;     // allocated entries per member (>= max_iters+1)
    int max_iters;
    double rtol;
};

struct RowArgs {
    int batch;
    double inv_h2;             // 1/h^2
    const double* k0sq;        // [batch]
    const double* eta;         // [batch]
    const double2* k2;         // padded
    const double2* f;          // padded (R_FWD_BORN, R_SWEEP)
    const double2* in;         // R_FWD: field to transform; R_FWD_BORN: u
    double2* out;              // R_INV output (padded)
    const double2* sub;        // R_INV: optional field subtracted from the output
    double2* T;                // intermediate (padded)
    double2* u0;               // iterate ping
    double2* u1;               // iterate pong
    double2* X;                // direction x^m (optimal-scalar / FourierDiag modes)
    const double2* tw;         // exp(-2 pi i k/n), k < n
    const double* sinp;        // sin(pi j/n), j < n
    int map_kind;
    double2 gamma;
    // IterFormat::Direct (iterate.cpp:118-123): the direction is the residual r^m itself
    // instead of r_bs^m = G r^m (CBS / NPBS)
    int direct;
    // Direct format + OptimalScalar (Euclidean): w = A r = L_ref r - V r.  R_FD_A also stores
    // the direction into X and R_RETA_C forms w = (L_ref r) - V r from its inverse transform
    // of the C_LREF column pass instead of w = x - G V x
    int lw;
    Control ctl;
    // x-slab of a grid distributed over ranks (2-D, batch 1; 0 = whole members): the launch
    // covers 2^slab_log2 rows starting at global row row0; u / k2 / f hold those rows (u with
    // one halo row on each side), T is blocked [dest rank][row][col within the dest's block]
    // for the all-to-all, and the reducing modes write their per-slab sums (RowSpec::NPART of
    // them: entry sums, then the optimal-scalar numerator / denominator) to slab_sums instead
    // of finalising (the driver all-reduces them and launches slab_finalize_kernel)
    int slab_log2;
    int row0;
    double* slab_sums;
    // R_SWEEP (2-D whole members): store the per-row partials only; the NEXT launch (the
    // column pass, ColArgs::finalize) sums them and records entry m -- no fence / atomic /
    // last-row wait at the end of every row (r01 ncu: ~13 % of the long-scoreboard stalls)
    int defer_final;
    // Fused exchange on a slab (xchg_on): the forward transform's blocks are stored straight
    // into the destination ranks' receive buffers (xchg[d] = rank d's t_cols, mapped on this
    // device: same-device parts or NVLink peer memory) at block `xchg_rank` -- the forward
    // all-to-all becomes part of the row kernel's epilogue.
    int xchg_on;
    int xchg_rank;
    double2* xchg[kMaxXchg];
    // L2 eviction-priority hints of this launch (BS_L2_HINTS bits; 0 = normal priority)
    int l2_hints;
};

struct ColArgs {
    int batch;
    const double* k0sq;
    const double* eta;
    const double* lap;         // (4/h^2) sin^2(j pi / (2n)), j < n
    double scale;              // C_ONE scale / Green normalisation 4/n^2 (/ engine gain)
    const double2* fd;         // C_FD: FourierDiag multiplier, padded n x n (shared by the batch)
    double2* T;
    const double2* tw;
    const double* sinp;
    const int* status;         // nullable: skip inactive members
    int planes_per_member;     // CL_PLANE: 1 (2-D) or n (3-D y-lines)
    int slab_cols;             // CL_SLAB: columns held by this rank (n x slab_cols block, row stride slab_cols)
    int col0;                  // CL_SLAB: global index of the first of them
    // finalize != 0 (2-D CL_PLANE): the first CTA of each member sums the per-row partials of
    // the preceding R_SWEEP launch (RowArgs::defer_final) and records its trace entry +
    // termination test (finalize_entry); ctl as in RowArgs, log2 rows per member = fin_lsh
    int finalize;
    int fin_lsh;
    int fin_step;  // 3-D: lines per row CTA (one partial per row CTA, finalize_member3)
    Control ctl;
    // 3-D slabs: CL_YBLK y-lines of the rank's R = 2^slab_log2 x-planes in the blocked layout
    // of t_index<DIM = 3, SLAB>; CL_SLAB with slab3 != 0: the received block's columns are
    // (y, z) pairs (slab_cols = R n), symbol a_y + a_z
    int slab_log2;
    int slab3;
    // fused inverse exchange (CL_SLAB): line element j belongs to source rank j >> xchg_log2r;
    // it is stored into that rank's t_rows (xchg[src]) at block xchg_rank
    int xchg_on;
    int xchg_rank;
    int xchg_log2r;
    double2* xchg[kMaxXchg];
    // C_GREEN as a tridiagonal x-solve (tri_kernels.cuh): pivot tables per (member, line) and
    // the scale that makes it equal the transform route (8 n h^2 x scale)
    const double2* tri;
    double tri_scale;
    int l2_hints;  // as RowArgs::l2_hints (the tridiagonal pass keeps T: bit 4)
};

// 1/eta of the pointwise map hoisted out of the row kernel's element loop: measured slower on
// c1 (r02: 337.5 vs 329.5 us per row launch) -- the hoisted reciprocal stays live through the
// unrolled loop and pushes the 128-register kernel into spills, which cost more than the
// per-element divide; so did re-reading it from shared memory per element (335.5 vs 331 us)
#ifndef BS_INV_ETA_HOIST
#define BS_INV_ETA_HOIST 0
#endif

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ double2 ldcg2(const double2* p) { return __ldcg(p); }

// 1/x for the Green weights (x = |lambda|^2 > 0): hardware approximation + two Newton steps
// (quadratic: ~2^-22 -> 2^-88), branch-free; __drcp_rn adds a correctly-rounded fix-up path.
#ifndef BS_FAST_RCP
#define BS_FAST_RCP 1
#endif
__device__ __forceinline__ double rcp_green(double x) {
#if BS_FAST_RCP
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
#else
    return __drcp_rn(x);
#endif
}

// L2 eviction-priority hints (experiment knob BS_L2_HINTS): with the batch swept in waves of 8
// members (bornsweep.cu group_members) a wave's fields are re-read every sweep, but its 160 MB do
// not fit the L2.  Bit 1: the medium k2 and the source f (read once per sweep, never written) are
// loaded evict_first -- measured on c1: 37.4 -> 38.6 Gpts/s (38.1 -> 39.2 on a less power-capped
// board); bit 4: the intermediate T (written by one launch, read by the next) loaded and stored
// evict_last, row kernel and tridiagonal pass -- 39.17 -> 39.53; bit 2: the iterate likewise --
// all three together measured lower (38.3 vs 38.6).  Default 5 = bits 1 + 4.
#ifndef BS_L2_HINTS
#define BS_L2_HINTS 5
#endif
#define BS_L2_STREAM (BS_L2_HINTS & 1)  // k2, f loads evict_first
#define BS_L2_KEEP_U (BS_L2_HINTS & 2)  // iterate loads / stores evict_last
#define BS_L2_KEEP_T (BS_L2_HINTS & 4)  // intermediate T loads / stores evict_last
// (sm_100a: the plain .L2::evict_* qualifiers need 256-bit accesses; 128-bit ones take a policy)
__device__ __forceinline__ unsigned long long l2_policy_first() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ unsigned long long l2_policy_normal() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ unsigned long long l2_policy_last() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double2 ld_stream(const double2* p, [[maybe_unused]] unsigned long long pol) {
#if BS_L2_STREAM
    double2 v;
    asm("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
#else
    return *p;
#endif
}
template <bool ON>
__device__ __forceinline__ double2 ld_keep(const double2* p, [[maybe_unused]] unsigned long long pol) {
    if constexpr (ON) {
        double2 v;
        asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol) : "memory");
        return v;
    } else {
        return *p;
    }
}
template <bool ON>
__device__ __forceinline__ void st_keep(double2* p, double2 v, [[maybe_unused]] unsigned long long pol) {
    if constexpr (ON) {
        asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
    } else {
        *p = v;
    }
}

// TMA bulk prefetch of a contiguous range into L2 (sm_90+: cp.async.bulk.prefetch.L2).
// bytes: multiple of 16, address 16-B aligned.  Fire-and-forget, no registers held.
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}


// Trace entry m for member b + termination test, restating proj/src/iterate.cpp:105-150.
static __device__ void finalize_entry(const Control& c, int b, int m, double sum_l2, double sum_reta) {
    const int stride = c.trace_stride;
    const double rel = sqrt(sum_l2) / c.fnorm_l2[b];
    const double rel_reta = sqrt(sum_reta) / c.fnorm_reta[b];
    c.trace_l2[(size_t)b * stride + m] = rel;
    c.trace_reta[(size_t)b * stride + m] = rel_reta;
    int term = -1;
    if (m == 0) {
        if (rel <= c.rtol) term = 0;  // converged before any update (iterate.cpp:112-115)
    } else {
        if (!isfinite(rel) || rel > 1e8) term = 2;  // diverged
        else if (rel <= c.rtol) term = 0;           // converged
        else if (m + 1 > 20) {                      // stagnated over a 20-step window
            const double past = c.trace_l2[(size_t)b * stride + (m - 20)];
            if (fabs(past - rel) < 1e-14 * fmax(1.0, past)) term = 3;
        }
    }
    if (term < 0 && m >= c.max_iters) term = 1;  // max_iters
    if (term >= 0) {
        c.iters[b] = m;
        c.term[b] = term;
        c.result_buf[b] = m & 1;
        c.status[b] = ST_DONE;
        atomicSub(c.n_active, 1);
    }
    c.sweep[b] = m + 1;
}

// optimal_scalar (proj/src/correction.cpp:10-18): <w, r> / <w, w>, 0 on a zero / non-finite
// denominator.  num = sum conj(w) r.
static __device__ void finalize_gamma(const Control& c, int b, double num_re, double num_im, double den) {
    double2 g = make_double2(0.0, 0.0);
    if (den > 0.0 && isfinite(den)) g = make_double2(num_re / den, num_im / den);
    c.gamma[b] = g;
}

// ------------------------------------------------------------------ row kernel
// NW warps per CTA; engine = one global row of T = n/P threads (several engines per warp when
// T < 32, several warps per engine -- named barriers -- when T > 32).
template <int THREADS, int REGS>
struct MinBlocks {
    static constexpr int V = 65536 / (THREADS * REGS);
    static constexpr int value = V > 32 ? 32 : (V < 1 ? 1 : V);
};

template <int T>
struct PolicyFor {
    using type = WarpSeg<T>;
};
template <>
struct PolicyFor<64> {
    using type = BarSeg<64>;
};
template <>
struct PolicyFor<128> {
    using type = BarSeg<128>;
};
template <>
struct PolicyFor<256> {
    using type = BarSeg<256>;
};

template <int T>
__device__ __forceinline__ WarpSeg<T> make_policy(WarpSeg<T>*, double2*, int) { return WarpSeg<T>{}; }
template <int T>
__device__ __forceinline__ BarSeg<T> make_policy(BarSeg<T>*, double2* scratch, int e) {
    return BarSeg<T>{scratch + e * (T / 32), 1 + e};
}

template <int LOG2N, int PP, int NW>
struct RowGeom {
    using G = Geom<LOG2N, PP>;
    static constexpr int T = G::T;
    static constexpr int EPB = NW * 32 / T;  // engines (rows) per CTA
    static_assert(T <= 32 || (T % 32 == 0 && EPB <= 15), "row engine layout");
    static constexpr int SCRATCH = T > 32 ? EPB * (T / 32) : 0;
    static constexpr size_t SMEM = sizeof(double2) * ((size_t)EPB * G::PAD_N + SCRATCH);
};

// DIM = 2: lines are the rows of each member (x index i, y contiguous), five-point stencil.
// DIM = 3: lines are the z-lines (x, y) of each member ([x][y][z], z contiguous), seven-point
//          stencil (the 3-D extension of config c3; no reference counterpart).
// SLAB: the launch covers one rank's x-slab (RowArgs::slab_log2 / row0 / slab_sums); a separate
// instantiation so the whole-member path keeps its compile-time indexing.
// One group of EPB lines (the work of one CTA).  `staged`: the group's operands are already
// in L2 (skip the per-line prefetch).
// Element j of line i (of the member starting at `mem`) in the intermediate T: row-major for
// whole members; on a slab (batch 1) blocked by the destination rank of the all-to-all --
// 2-D: [dest = j >> sl][row i][j mod R]; 3-D (line i = (xl, y), xl the local x-plane):
// [dest = y >> sl][xl][y mod R][z = j], i.e. the rank owning y-block `dest` receives its
// x-lines contiguous (slab.py / bp_slab_*).
template <int LOG2N, int DIM, bool SLAB>
__device__ __forceinline__ size_t t_index(int sl, size_t mem, int i, int j) {
    constexpr int N = 1 << LOG2N;
    if constexpr (!SLAB) {
        return mem + (size_t)i * N + j;
    } else if constexpr (DIM == 2) {
        return mem + ((size_t)(j >> sl) << (2 * sl)) + ((size_t)i << sl) + (j & ((1 << sl) - 1));
    } else {
        const int xl = i >> LOG2N, y = i & (N - 1);
        const size_t blk = ((size_t)(y >> sl) << sl) + xl;
        return mem + (((blk << sl) + (size_t)(y & ((1 << sl) - 1))) << LOG2N) + j;
    }
}

template <int LOG2N, int MODE, int NW, int PP, int DIM, bool SLAB>
__device__ __forceinline__ void row_group(const RowArgs& a, const long grp, const bool staged) {
    using G = Geom<LOG2N, PP>;
    using RG = RowGeom<LOG2N, PP, NW>;
    using Pol = typename PolicyFor<G::T>::type;
    using Engine = DstEngine<LOG2N, PP>;
    using S = RowSpec<MODE>;
    constexpr int N = G::N, P = G::P, T = G::T;
    constexpr int EPB = RG::EPB;
    constexpr int LLINES = (DIM - 1) * LOG2N;          // log2(lines per member)
    constexpr size_t PLANE = (size_t)N * N;            // x-stride in 3-D
    constexpr unsigned VALID_LINES = DIM == 3 ? (unsigned)((N - 1) * (N - 1)) : (unsigned)(N - 1);
    extern __shared__ double2 smem[];

    // the launch decides (RowArgs::l2_hints): the priorities pay off where a launch's fields are
    // re-read out of L2 by the next launches (the waves' single-member launches, single-member
    // handles); a launch over a whole multi-member batch measured slower with them (row kernel
    // 0.351 -> 0.360 ms on c1) and keeps the normal priority
    [[maybe_unused]] const unsigned long long pol_s =
        BS_L2_STREAM ? ((a.l2_hints & 1) ? l2_policy_first() : l2_policy_normal()) : 0ull;
    [[maybe_unused]] const unsigned long long pol_k =
        (BS_L2_KEEP_U || BS_L2_KEEP_T) ? ((a.l2_hints & 4) ? l2_policy_last() : l2_policy_normal()) : 0ull;
    const int t = threadIdx.x % T;
    const int e = threadIdx.x / T;
    const long grow = grp * EPB + e;
    // log2(lines per member or slab): a slab holds 2^slab_log2 rows (2-D) / x-planes (3-D)
    const int lsh = SLAB ? a.slab_log2 + (DIM - 2) * LOG2N : LLINES;
    const int b = (int)(grow >> lsh);
    const int i = (int)(grow & ((1L << lsh) - 1));      // line index within the member (slab)
    // global x index of the line (2-D: the row; 3-D: the plane) and its Dirichlet padding
    const int xg = (SLAB ? a.row0 : 0) + (DIM == 2 ? i : (i >> LOG2N));
    bool valid = (b < a.batch) && (xg & (N - 1)) != 0 && (DIM == 2 || (i & (N - 1)) != 0);
    // shared-memory staging of the inverse transform's input (see RSM below)
    constexpr bool RSM = BS_ROW_SMEM && (T > 32 || DIM == 3 || (BS_RSM_ALL && S::ITER));
    // forward transform's staged line unpadded too (warp-private engines only, see below)
    constexpr bool FWD_DENSE = BS_ROW_FWD_DENSE && RSM && T <= 32;
    // The T line is loaded before the member's status / sweep counter are known (they are
    // an L2 round trip of their own): the two latencies overlap instead of adding up.  A
    // terminated member's line is loaded and dropped (16 B/pt, its CTA then exits).
    double2 xT[(S::INV && RSM) ? P : 1];
    if constexpr (S::INV && RSM) {
        const int sl0 = SLAB ? a.slab_log2 : 0;
        const size_t mem0 = (size_t)(valid ? b : 0) << (lsh + LOG2N);
        const int i0 = valid ? i : 0;
#pragma unroll
        for (int mm = 0; mm < P; ++mm)  // in bounds for every thread (member / line clamped)
            xT[mm] = ld_keep<(BS_L2_KEEP_T != 0)>(&a.T[t_index<LOG2N, DIM, SLAB>(sl0, mem0, i0, t + T * mm)], pol_k);
    }
    int m = 0;  // trace entry this launch belongs to
    if (S::ITER && valid) {
        valid = __ldcg(&a.ctl.status[b]) == ST_ACTIVE;
        m = __ldcg(&a.ctl.sweep[b]) - (S::POST ? 1 : 0);
    }
    if (!__syncthreads_or(valid)) return;

    double2* buf = smem + e * G::PAD_N;
    const Pol pol = make_policy((Pol*)nullptr, smem + EPB * G::PAD_N, e);
    // invalid lines (padding, inactive, past the batch) are clamped to a line whose stencil
    // neighbours are in bounds, so the element-wise loads need no predicates or zero fills;
    // their results are never stored or summed
    constexpr int ISAFE = SLAB ? 0 : (DIM == 3 ? N + 1 : 1);
    const size_t mem = (size_t)(valid ? b : 0) << (lsh + LOG2N);
    const size_t row = mem + (size_t)(valid ? i : ISAFE) * N;
    // T element (this line, column j): row-major, or blocked by destination rank on a slab
    const int sl = SLAB ? a.slab_log2 : 0;
    auto tix = [&](int j) -> size_t {
        if constexpr (!SLAB) return row + j;
        return t_index<LOG2N, DIM, SLAB>(sl, mem, valid ? i : 0, j);
    };
    const double2 zero = make_double2(0.0, 0.0);
    const double2* ucur = (m & 1) ? a.u1 : a.u0;  // u^m
    double2* unext = (m & 1) ? a.u0 : a.u1;       // u^{m+1}
    const double k0sq = valid ? a.k0sq[b] : 0.0;
    const double eta = valid ? a.eta[b] : 1.0;
    const double2 shift = make_double2(k0sq, eta);
    // pointwise map gamma(x) = (i/eta) V(x): one division per line, not one per element (the
    // unrolled element loop otherwise carried an FP64 divide + slow-path call per element)
    [[maybe_unused]] const double inv_eta = BS_INV_ETA_HOIST ? 1.0 / eta : 0.0;


    // Stage the element-wise operands of this row (and the stencil halo rows at the CTA's
    // edges) into L2 while the transform runs: the loads after the engine then hit L2.
    // Issued after the T row's own loads so those do not queue behind the prefetches.
    auto prefetch_row = [&]() {
    if constexpr (S::ITER && MODE != R_RETA_C) {
        if (valid && t == 0 && !staged) {
            constexpr unsigned RB = N * sizeof(double2);
            prefetch_l2(ucur + row, RB);
            prefetch_l2(a.k2 + row, RB);
            prefetch_l2(a.f + row, RB);
            if constexpr (S::ENTRY) {
                if (e == 0) prefetch_l2(ucur + row - N, RB);
                if (e == EPB - 1) prefetch_l2(ucur + row + N, RB);
                if constexpr (DIM == 3) {
                    prefetch_l2(ucur + row - PLANE, RB);
                    prefetch_l2(ucur + row + PLANE, RB);
                }
            }
            if constexpr (MODE == R_OPT_B) prefetch_l2(a.X + row, RB);
        }
    }
    };
    if constexpr (!S::INV) prefetch_row();

    double acc[S::NPART > 0 ? S::NPART : 1] = {};
    // shared-memory staging pays off for multi-warp lines (n >= 1024) and the 3-D stencil;
    // single-warp 2-D lines keep the register path (measured, r01)
    double2 q[P];                    // register path: source of the forward transform
    double2 z[P];                    // register path: G q

    // ---- inverse y-DST of the column-pass output, staged to the stride layout.  BS_ROW_SMEM:
    // the T row goes through shared memory (pre-processing reads x_j and x_{N-j} there) and
    // G q stays there in natural order for the element-wise phase, which writes the next
    // source into the same slots (same thread, same j): neither the line, its mirror, G q nor
    // the next source occupies registers, so the element-wise loads can be kept in flight.
    if constexpr (S::INV) {
        double2 y[P];
        if constexpr (RSM) {
            prefetch_row();
#pragma unroll
            for (int mm = 0; mm < P; ++mm) buf[t + T * mm] = xT[mm];  // unpadded (run_smem<true>); invalid lines: discarded
            pol.sync();
            {
                double2 v[P];
                Engine::template run_smem<true>(v, y, t, buf, a.tw, a.sinp, pol);
            }
#pragma unroll
            for (int l = 0; l < P; ++l) buf[G::at_block(t, G::pidx(t * P), l)] = y[l];
            pol.sync();
        } else {
        double2 x[P], xm[P];
#pragma unroll
        for (int mm = 0; mm < P; ++mm) {
            const int j = t + T * mm;
            x[mm] = valid ? a.T[tix(j)] : zero;
            xm[mm] = (valid && j != 0) ? a.T[tix(N - j)] : zero;  // mirror: L1 hit
        }
        prefetch_row();
        Engine::run(x, xm, y, t, buf, a.tw, a.sinp, pol);
#pragma unroll
        for (int l = 0; l < P; ++l) buf[G::at_block(t, G::pidx(t * P), l)] = y[l];
        pol.sync();
#pragma unroll
        for (int mm = 0; mm < P; ++mm) z[mm] = buf[G::at_stride(t, G::pidx(t), mm)];
        pol.sync();
        }
    }

    // ---- element-wise phase
    // operands of element mm, issued BS_EW_PD elements ahead (iterate modes)
    struct Opnd {
        double2 u, k2, f, un, us, uw, ue, ua, ub, x;
    };
    constexpr bool PIPE = S::ITER && MODE != R_RETA_C;
    auto load_op = [&](int mm) {
        // unpredicated: `row` is clamped for invalid lines; uw at j = 0 reads the previous
        // line's last element (its result is discarded: j = 0 is the Dirichlet node) and ue at
        // j = n-1 reads the next line's zero node (the five-point zero halo, as before)
        Opnd o;
        o.un = o.us = o.uw = o.ue = o.ua = o.ub = o.x = zero;
        const int j = t + T * mm;
        o.u = ld_keep<(BS_L2_KEEP_U != 0)>(&ucur[row + j], pol_k);
        o.k2 = ld_stream(&a.k2[row + j], pol_s);
        o.f = ld_stream(&a.f[row + j], pol_s);
        if constexpr (S::ENTRY) {
            o.un = ld_keep<(BS_L2_KEEP_U != 0)>(&ucur[row - N + j], pol_k);
            o.us = ld_keep<(BS_L2_KEEP_U != 0)>(&ucur[row + N + j], pol_k);
            o.uw = ld_keep<(BS_L2_KEEP_U != 0)>(&ucur[row + j - 1], pol_k);
            o.ue = ld_keep<(BS_L2_KEEP_U != 0)>(&ucur[row + j + 1], pol_k);
            if constexpr (DIM == 3) {
                o.ua = ucur[row - PLANE + j];
                o.ub = ucur[row + PLANE + j];
            }
        }
        if constexpr (MODE == R_OPT_B) o.x = a.X[row + j];
        return o;
    };
    constexpr int PD = PIPE ? (BS_EW_PD < P ? BS_EW_PD : P) : 0;
    Opnd ops[P];
    if constexpr (PIPE) {
#pragma unroll
        for (int mm = 0; mm < PD; ++mm) ops[mm] = load_op(mm);
    }
#pragma unroll
    for (int mm = 0; mm < P; ++mm) {
        const int j = t + T * mm;
        if constexpr (PIPE) {
            if (mm + PD < P) ops[mm + PD] = load_op(mm + PD);
        }
        const double2 zz = !S::INV ? zero : RSM ? buf[G::at_stride(t, G::pidx(t), mm)] : z[mm];
        double2 qv = zero;
        if constexpr (MODE == R_INV) {
            double2 o = zz;
            if (a.sub) o = csub(o, valid ? a.sub[row + j] : zero);
            if (valid) a.out[row + j] = (j == 0) ? zero : o;
        } else if constexpr (MODE == R_FWD) {
            const double2 v = valid ? a.in[row + j] : zero;
            qv = (j == 0) ? zero : v;
        } else if constexpr (MODE == R_FWD_BORN) {
            const double2 v = valid ? a.in[row + j] : zero;
            const double2 V = csub(valid ? a.k2[row + j] : zero, shift);
            const double2 o = cadd(cmul(v, V), valid ? a.f[row + j] : zero);  // mul(u, v) + f
            qv = (j == 0) ? zero : o;
        } else if constexpr (MODE == R_RETA_C) {
            // z = G V x: w = x - G V x (correction.cpp:38-44); gamma = <w, x> / <w, w>
            const double2 x = valid ? a.X[row + j] : zero;
            // R_eta metric: w = x - G V x; Direct + Euclidean: w = L_ref x - V x (= A x)
            const double2 w = a.lw ? csub(zz, cmul(csub(valid ? a.k2[row + j] : zero, shift), x))
                                   : csub(x, zz);
            if (j != 0) {
                acc[0] += w.x * x.x + w.y * x.y;  // Re conj(w) x
                acc[1] += w.x * x.y - w.y * x.x;  // Im conj(w) x
                acc[2] += cnorm(w);
            }
        } else {
            const Opnd& op = ops[mm];
            const double2 u = op.u, k2 = op.k2, f = op.f;
            const double2 V = csub(k2, shift);
            if constexpr (S::ENTRY) {
                // r^m = f - A u^m (five-point in proj/src/kernels.cpp:56-69 order);
                // x^m = G q^m - u^m = born_residual (problem.cpp:41-49) = G r^m (key identity)
                const double2 un = op.un, us = op.us, uw = op.uw, ue = op.ue, ua = op.ua, ub = op.ub;
                const double2 x = csub(zz, u);
                double2 s;
                if constexpr (DIM == 3) {
                    // seven-point: (6u - x-1 - x+1 - y-1 - y+1 - z-1 - z+1) / h^2
                    s = cscale(u, 6.0);
                    s = csub(s, ua);
                    s = csub(s, ub);
                } else {
                    s = cscale(u, 4.0);
                }
                s = csub(s, un);
                s = csub(s, us);
                s = csub(s, uw);
                s = csub(s, ue);
                const double2 r = csub(f, csub(cscale(s, a.inv_h2), cmul(k2, u)));
                if (j != 0) {
                    acc[0] += cnorm(r);
                    acc[1] += cnorm(x);
                }
                // direction of the update (iterate.cpp:118-123): r (Direct) or r_bs = G r
                // (a compile-time choice: a runtime select kept r and x live together and made
                // the c1 row kernel spill, 328 -> 368 us)
                const double2 d = MODE == R_SWEEP_D ? r : (MODE == R_SWEEP ? x : (a.direct ? r : x));
                if constexpr (RowSpec<MODE>::SWEEP) {
                    double2 g = a.gamma;
#if BS_INV_ETA_HOIST
                    if (a.map_kind == MK_POINTWISE) g = cscale(mul_pi(V), inv_eta);  // (i/eta) V
#else
                    if (a.map_kind == MK_POINTWISE) g = cscale(mul_pi(V), 1.0 / eta);
#endif
                    double2 unew = cadd(u, cmul(g, d));
                    if (j == 0) unew = zero;
                    if (valid) st_keep<(BS_L2_KEEP_U != 0)>(&unext[row + j], unew, pol_k);
                    qv = cadd(cmul(V, unew), f);
                } else if constexpr (MODE == R_OPT_A) {
                    // w = A x = (L_ref - V) G r = r - V x (key identity; the reference applies
                    // A by stencil, correction.cpp:33-36 -- equal to roundoff)
                    // (NPBS / CBS only: Direct + Euclidean takes the R_FD_A / C_LREF plan)
                    const double2 w = csub(r, cmul(V, x));
                    if (j != 0) {
                        acc[2] += w.x * r.x + w.y * r.y;
                        acc[3] += w.x * r.y - w.y * r.x;
                        acc[4] += cnorm(w);
                    }
                    if (valid) a.X[row + j] = (j == 0) ? zero : x;
                } else if constexpr (MODE == R_RETA_A) {
                    if (valid) a.X[row + j] = (j == 0) ? zero : d;
                    qv = (j == 0) ? zero : cmul(d, V);  // apply_V(d)
                } else {  // R_FD_A: forward transform of the direction itself
                    if (a.lw && valid) a.X[row + j] = (j == 0) ? zero : d;
                    qv = (j == 0) ? zero : d;
                }
            } else {
                // R_OPT_B: u' = u + gamma x ; R_FD_B: u' = u + du (du = z)
                double2 du;
                if constexpr (MODE == R_OPT_B) {
                    const double2 x = op.x;
                    const double2 g = valid ? a.ctl.gamma[b] : zero;
                    du = cmul(g, x);  // kernels::scale(x, gamma)
                } else {
                    du = zz;
                }
                double2 unew = cadd(u, du);
                if (j == 0) unew = zero;
                if (valid) st_keep<(BS_L2_KEEP_U != 0)>(&unext[row + j], unew, pol_k);
                qv = cadd(cmul(V, unew), f);
            }
        }
        if constexpr (S::FWD) {
            if constexpr (RSM) {
                if constexpr (FWD_DENSE) {
                    // unpadded next source (run_smem<true>: conflict-free mirror reads).  Slot j
                    // can only alias the padded G q slot of an element j' <= j, i.e. of this
                    // iteration or an earlier one: the warp sync orders every lane's G q read of
                    // this iteration before any lane's write (one engine never spans warps here)
                    __syncwarp();
                    buf[t + T * mm] = qv;
                } else {
                    buf[G::at_stride(t, G::pidx(t), mm)] = qv;  // the slot this thread read G q from
                }
            }
            else q[mm] = qv;
        }
    }
    if constexpr (MODE == R_INV) return;

    // ---- forward y-DST of q (mirror by warp shuffles, or shared memory for multi-warp rows)
    if constexpr (S::FWD) {
        double2 y2[P];
        if constexpr (RSM) {
        pol.sync();
        {
            double2 v[P];
            Engine::template run_smem<FWD_DENSE>(v, y2, t, buf, a.tw, a.sinp, pol);
        }
        } else {
        double2 qm[P];
#if BS_SHFL_MIRROR
        pol.mirror(q, qm, t, buf, typename G::Pidx{});
#else
#pragma unroll
        for (int mm = 0; mm < P; ++mm) buf[G::at_stride(t, G::pidx(t), mm)] = q[mm];
        pol.sync();
#pragma unroll
        for (int mm = 0; mm < P; ++mm) {
            const int j = t + T * mm;
            qm[mm] = (j == 0) ? zero : buf[G::pidx(N - j)];
        }
        pol.sync();
#endif
        Engine::run(q, qm, y2, t, buf, a.tw, a.sinp, pol);
        }
#pragma unroll
        for (int l = 0; l < P; ++l) buf[G::at_block(t, G::pidx(t * P), l)] = y2[l];
        pol.sync();
#pragma unroll
        for (int mm = 0; mm < P; ++mm) {
            const int j = t + T * mm;
            if (valid) {
                const double2 v = buf[G::at_stride(t, G::pidx(t), mm)];
                size_t ix = tix(j);
                if constexpr (SLAB) {
                    if (a.xchg_on) {  // block d -> rank d's receive buffer, at block xchg_rank
                        const int lb = 2 * sl + (DIM - 2) * LOG2N;  // log2 elements per block
                        const size_t d = ix >> lb;
                        a.xchg[d][((size_t)a.xchg_rank << lb) + (ix & ((1ull << lb) - 1))] = v;
                        continue;
                    }
                }
                st_keep<(BS_L2_KEEP_T != 0)>(&a.T[ix], v, pol_k);
            }
        }
    }

    // ---- per-row partials; the last row of the member finalises (deterministic order)
    if constexpr (S::NPART > 0) {
#pragma unroll
        for (int k = 0; k < S::NPART; ++k) acc[k] = pol.sum(acc[k], t);
        if constexpr (RowSpec<MODE>::SWEEP && !SLAB) {
            if (a.defer_final) {  // finalised by the next launch (col_group, ColArgs::finalize)
                if constexpr (DIM == 3) {
                    // one partial per CTA (its EPB lines summed in engine order), stored in the
                    // slot of the CTA's first line: n^2 / EPB values for the finalising CTA
                    __shared__ double cpart[EPB][2];
                    if (t == 0) {
                        cpart[e][0] = valid ? acc[0] : 0.0;
                        cpart[e][1] = valid ? acc[1] : 0.0;
                    }
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        double s0 = 0.0, s1 = 0.0;
                        for (int k = 0; k < EPB; ++k) {
                            s0 += cpart[k][0];
                            s1 += cpart[k][1];
                        }
                        const long g0 = grp * EPB;  // first line of the CTA (members hold whole CTAs)
                        double* pr = a.ctl.partial + (size_t)g0 * kPartStride;
                        pr[0] = s0;
                        pr[1] = s1;
                    }
                } else if (valid && t == 0) {
                    double* pr = a.ctl.partial + (((size_t)b << lsh) + i) * kPartStride;
#pragma unroll
                    for (int k = 0; k < S::NPART; ++k) pr[k] = acc[k];
                }
                return;
            }
        }
        int last = 0;
        if (valid && t == 0) {
            double* pr = a.ctl.partial + (((size_t)b << lsh) + i) * kPartStride;
#pragma unroll
            for (int k = 0; k < S::NPART; ++k) pr[k] = acc[k];
            __threadfence();
            const unsigned old = atomicAdd(&a.ctl.counter[b], 1u);
            const unsigned nvalid = SLAB ? ((1u << sl) - (a.row0 == 0 ? 1u : 0u)) * (DIM == 3 ? N - 1u : 1u)
                                         : VALID_LINES;
            last = (old == nvalid - 1u);
        }
        if constexpr (DIM == 3) {
            // 3-D: the member's n^2 line partials are summed by the whole last CTA (a CTA holds
            // lines of one member once 2^lsh >= EPB) -- one engine of 16 lanes took ~600 us
            // at n = 256 (single-SM tail, r01c); strided per thread, fixed-order tree
            if ((1L << lsh) >= EPB) {
                if (!__syncthreads_or(last)) return;
                __threadfence();
                __shared__ double red[S::NPART][32];
                double s[S::NPART];
#pragma unroll
                for (int k = 0; k < S::NPART; ++k) s[k] = 0.0;
                for (int r = threadIdx.x; r < (1 << lsh); r += blockDim.x) {
                    if ((r & (N - 1)) == 0 || (((SLAB ? a.row0 : 0) + (r >> LOG2N)) & (N - 1)) == 0)
                        continue;  // padding lines
                    const double* pr = a.ctl.partial + (((size_t)b << lsh) + r) * kPartStride;
#pragma unroll
                    for (int k = 0; k < S::NPART; ++k) s[k] += __ldcg(pr + k);
                }
#pragma unroll
                for (int k = 0; k < S::NPART; ++k) {
#pragma unroll
                    for (int d = 16; d >= 1; d >>= 1) s[k] += __shfl_xor_sync(0xffffffffu, s[k], d);
                }
                if ((threadIdx.x & 31) == 0) {
#pragma unroll
                    for (int k = 0; k < S::NPART; ++k) red[k][threadIdx.x >> 5] = s[k];
                }
                __syncthreads();
                if (threadIdx.x == 0) {
#pragma unroll
                    for (int k = 0; k < S::NPART; ++k) {
                        s[k] = 0.0;
                        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s[k] += red[k][w];
                    }
                    a.ctl.counter[b] = 0u;
                    if constexpr (SLAB) {  // this rank's sums; finalised after the all-reduce
#pragma unroll
                        for (int k = 0; k < S::NPART; ++k) a.slab_sums[k] = s[k];
                    } else {
                        if constexpr (MODE == R_OPT_A) finalize_gamma(a.ctl, b, s[2], s[3], s[4]);
                        if constexpr (MODE == R_RETA_C) finalize_gamma(a.ctl, b, s[0], s[1], s[2]);
                        if constexpr (S::ENTRY) {
                            // m of this member (thread 0's own line may be a padding line, for
                            // which m was not read); the counter is advanced only here
                            const int mb = __ldcg(&a.ctl.sweep[b]) - (S::POST ? 1 : 0);
                            finalize_entry(a.ctl, b, mb, s[0], s[1]);
                        }
                    }
                }
                return;
            }
        }
        last = pol.bcast0(last, t);
        if (last) {
            __threadfence();
            double s[S::NPART];
#pragma unroll
            for (int k = 0; k < S::NPART; ++k) s[k] = 0.0;
            for (int r = t; r < (1 << lsh); r += T) {
                const int rg = SLAB ? a.row0 + r : r;
                if (DIM == 2 ? (rg & (N - 1)) == 0
                             : ((r & (N - 1)) == 0 || (((SLAB ? a.row0 : 0) + (r >> LOG2N)) & (N - 1)) == 0))
                    continue;  // padding lines
                const double* pr = a.ctl.partial + (((size_t)b << lsh) + r) * kPartStride;
#pragma unroll
                for (int k = 0; k < S::NPART; ++k) s[k] += __ldcg(pr + k);
            }
#pragma unroll
            for (int k = 0; k < S::NPART; ++k) s[k] = pol.sum(s[k], t);
            if (t == 0) {
                a.ctl.counter[b] = 0u;
                if constexpr (SLAB) {  // this rank's sums (batch 1), finalised after the all-reduce
#pragma unroll
                    for (int k = 0; k < S::NPART; ++k) a.slab_sums[k] = s[k];
                } else {
                    if constexpr (MODE == R_OPT_A) finalize_gamma(a.ctl, b, s[2], s[3], s[4]);
                    if constexpr (MODE == R_RETA_C) finalize_gamma(a.ctl, b, s[0], s[1], s[2]);
                    if constexpr (S::ENTRY) finalize_entry(a.ctl, b, m, s[0], s[1]);
                }
            }
        }
    }
}

template <int LOG2N, int MODE, int NW, int PP, int DIM = 2, bool SLAB = false>
__global__ void __launch_bounds__(NW * 32, (MinBlocks<NW * 32, PP >= 16 ? BS_ROW_REGS : 80>::value))
row_kernel(const RowArgs a) {
    // (a persistent variant looping over groups with next-group L2 prefetch measured 23-48 %
    // slower on c1, r01: the hardware's CTA scheduling is kept)
    row_group<LOG2N, MODE, NW, PP, DIM, SLAB>(a, blockIdx.x, false);
}

// ------------------------------------------------------------------ column kernel
// C columns per CTA, T threads per column (thread = c + C*t): row segments of C*16 bytes.
template <int LOG2N, int PP, int C>
struct ColGeom {
    using G = Geom<LOG2N, PP>;
    static constexpr int THREADS = C * G::T;
    static constexpr size_t SMEM = sizeof(double2) * (C * G::PAD_N + BlockSeg<G::T, C>::SCRATCH);
};

// LAYOUT 0: lines along the slow axis of n x n planes (2-D x-lines; 3-D y-lines of every
//           x-plane, planes_per_member = n).  LAYOUT 2: 3-D x-lines (stride n^2).
//           CL_SLAB: 2-D x-lines of the n x slab_cols column block a rank holds after the
//           all-to-all of a slab-decomposed grid (row stride slab_cols, global column col0 + q).
//           CL_YBLK: 3-D slab y-lines on the dest-blocked layout (t_index<3, true>).
//           CL_CDR: config c4 real column pairs (the tridiagonal pass only, tri_kernels.cuh).
enum ColLayout { CL_PLANE = 0, CL_X3 = 2, CL_SLAB = 3, CL_YBLK = 4, CL_CDR = 5 };

#ifndef BS_COL_REVERSE
#define BS_COL_REVERSE 1
#endif
// One plane (a single 2-D grid, c2) has no member/plane order to exploit: kept forward
// (measured: c2 column 490 us forward vs 512 reversed; c1 -1 %, c3 -1 %, c4 -7 % reversed).
template <int LAYOUT>
__device__ __forceinline__ bool col_reversed(const ColArgs& a) {
    const bool one_plane = (LAYOUT == CL_PLANE && (long)a.batch * a.planes_per_member == 1) ||
                           (LAYOUT == CL_SLAB && a.batch == 1);
    return BS_COL_REVERSE && !one_plane;
}

// Deferred finalisation of trace entry m for member b (ColArgs::finalize): one warp sums the
// per-row partials of the preceding R_SWEEP launch in the row kernel's own order (lane r over
// rows r, r+32, ...; xor-shuffle tree) and runs finalize_entry.  Visibility of the partials
// is given by the launch boundary.
__device__ __forceinline__ void finalize_member(const ColArgs& a, int b, int nlines) {
    const int lane = threadIdx.x & 31;
    const int m = __ldcg(&a.ctl.sweep[b]);
    double s0 = 0.0, s1 = 0.0;
    const double* base = a.ctl.partial + ((size_t)b << a.fin_lsh) * kPartStride;
    for (int r = lane; r < nlines; r += 32) {
        if (r == 0) continue;  // Dirichlet padding line
        s0 += __ldcg(base + (size_t)r * kPartStride);
        s1 += __ldcg(base + (size_t)r * kPartStride + 1);
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, d);
        s1 += __shfl_xor_sync(0xffffffffu, s1, d);
    }
    if (lane == 0) finalize_entry(a.ctl, b, m, s0, s1);
}

// 3-D variant (ColArgs::finalize on the first y-line launch of the column stage): the whole CTA
// sums the member's per-row-CTA partials -- lane-strided, then a fixed-order warp and CTA
// tree -- and thread 0 runs finalize_entry.  Previously the 3-D row
// kernel's last engine did this alone (16 lanes over 65536 lines at n = 256): a ~600 us
// single-SM tail on a ~340 us launch (ncu sm__cycles_active min 650 K vs max 1.81 M, r01c).
// The row kernel leaves one partial per row CTA (a.fin_step lines, padding lines contributing 0)
// in the slot of the CTA's first line; CTAs of the padding x-plane 0 exit without one.
template <int LOG2N>
__device__ __forceinline__ void finalize_member3(const ColArgs& a, int b) {
    constexpr int N = 1 << LOG2N;
    __shared__ double red[2][32];
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, w = tid >> 5;
    const int m = __ldcg(&a.ctl.sweep[b]);
    double s0 = 0.0, s1 = 0.0;
    const double* base = a.ctl.partial + ((size_t)b << (2 * LOG2N)) * kPartStride;
    const int step = a.fin_step;
    for (int r = N + tid * step; r < N * N; r += nthr * step) {  // from x-plane 1
        s0 += __ldcg(base + (size_t)r * kPartStride);
        s1 += __ldcg(base + (size_t)r * kPartStride + 1);
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, d);
        s1 += __shfl_xor_sync(0xffffffffu, s1, d);
    }
    if (lane == 0) {
        red[0][w] = s0;
        red[1][w] = s1;
    }
    __syncthreads();
    if (tid == 0) {
        double t0 = 0.0, t1 = 0.0;
        for (int k = 0; k < (nthr + 31) / 32; ++k) {
            t0 += red[0][k];
            t1 += red[1][k];
        }
        finalize_entry(a.ctl, b, m, t0, t1);
    }
}

// One CTA's column group (bid = the CTA index of the column launch).
template <int LOG2N, int MODE, int C, int PP, int LAYOUT>
__device__ __forceinline__ void col_group(const ColArgs& a, const int bid) {
    using G = Geom<LOG2N, PP>;
    using Engine = DstEngine<LOG2N, PP>;
    constexpr int N = G::N, P = G::P, T = G::T;
    extern __shared__ double2 smem[];
    // WIDE (two 2048/4096-point columns per CTA): warp-contiguous engines synchronised by their
    // own named barriers (the engines no longer wait for each other at every pass), the CTA
    // loading and storing both columns of a row with 256-bit accesses through shared memory
    constexpr bool WIDE = BS_COL_WIDE && BS_COL_LD256 && LAYOUT == CL_PLANE && C == 2 && T > 32 && (T % 32) == 0;
    int c, t;
    if constexpr (WIDE) {
        c = threadIdx.x / T;
        t = threadIdx.x % T;
    } else {
        col_thread_map<G::T, C>(t, c);
    }
    constexpr int GROUPS = N / C;
    // line group -> member b, base offset `mem`, line stride LS, and (3-D x-lines) the y index
    int b, yl = 0, qa;
    size_t mem;
    size_t LS = LAYOUT == CL_X3 ? (size_t)N * N : (size_t)N;
    int xl = 0;  // CL_YBLK: local x-plane
    if constexpr (LAYOUT == CL_YBLK) {
        b = 0;
        xl = bid / GROUPS;
        qa = (bid % GROUPS) * C + c;  // z
        mem = 0;
    } else if constexpr (LAYOUT == CL_SLAB) {
        const int groups = a.slab_cols / C;
        b = bid / groups;
        qa = (bid % groups) * C + c;  // column within the block (address)
        LS = (size_t)a.slab_cols;
        mem = (size_t)b * N * a.slab_cols;
    } else if constexpr (LAYOUT == CL_X3) {
        const int grp = bid / GROUPS;  // (member, y)
        b = grp >> LOG2N;
        yl = grp & (N - 1);
        if (yl == 0) return;                   // padding y-plane
        mem = ((size_t)b << (3 * LOG2N)) + (size_t)yl * N;
    } else {
        const int plane = bid / GROUPS;
        b = plane / a.planes_per_member;
        if (a.planes_per_member > 1 && (plane & (N - 1)) == 0) return;  // padding x-plane (3-D)
        mem = (size_t)plane * N * N;
    }
    int q;  // global column index (symbol, Dirichlet zero column)
    double lq3 = 0.0;  // 3-D slab columns: a_y + a_z
    if constexpr (LAYOUT == CL_SLAB) {
        q = a.col0 + qa;
        if (a.slab3) {
            const int yq = a.col0 + (qa >> LOG2N), zq = qa & (N - 1);
            q = (yq == 0 || zq == 0) ? 0 : 1;  // only the Dirichlet test uses q below
            lq3 = a.lap[yq] + a.lap[zq];
        }
    } else if constexpr (LAYOUT == CL_YBLK) {
        q = qa;
    } else {
        q = (bid % GROUPS) * C + c;
        qa = q;
    }
    // element j of this thread's line
    const int sly = LAYOUT == CL_YBLK ? a.slab_log2 : 0;
    auto gidx = [&](int j) -> size_t {
        if constexpr (LAYOUT == CL_YBLK) {
            const size_t blk = ((size_t)(j >> sly) << sly) + xl;
            return (((blk << sly) + (size_t)(j & ((1 << sly) - 1))) << LOG2N) + qa;
        } else {
            return mem + (size_t)j * LS + qa;
        }
    };
    // output element j: in place, or (fused inverse exchange, CL_SLAB) into the source rank's
    // t_rows at block xchg_rank -- row j & (R-1) of that block, same column
    // (CL_YBLK forward y-lines of a 3-D slab: the dest-blocked element goes to rank d's t_cols,
    // like the 2-D row kernel's fused store)
    auto st_out = [&](int j, double2 v) {
        if constexpr (LAYOUT == CL_SLAB) {
            if (a.xchg_on) {
                const int rr = a.xchg_log2r;
                a.xchg[j >> rr][((size_t)a.xchg_rank << rr) * LS + (size_t)(j & ((1 << rr) - 1)) * LS + qa] = v;
                return;
            }
        } else if constexpr (LAYOUT == CL_YBLK) {
            if (a.xchg_on) {
                const size_t ix = gidx(j);
                const int lb = 2 * sly + LOG2N;  // log2 elements per destination block
                a.xchg[ix >> lb][((size_t)a.xchg_rank << lb) + (ix & ((1ull << lb) - 1))] = v;
                return;
            }
        }
        a.T[gidx(j)] = v;
    };
    if (a.status) {
        const bool active = __ldcg(&a.status[b]) == ST_ACTIVE;  // read before finalising
        if constexpr (LAYOUT == CL_PLANE) {
            if (a.finalize && active && a.planes_per_member == 1 && (bid % GROUPS) == 0 && threadIdx.x < 32)
                finalize_member(a, b, 1 << a.fin_lsh);
            if (a.finalize && active && a.planes_per_member > 1) {
                // 3-D: the member's first-dispatched CTA (reversed order: its last valid plane
                // and group; forward: plane 1, group 0) finalises -- CTA-uniform condition
                const int pim = (bid / GROUPS) & (N - 1), g = bid % GROUPS;
                if (col_reversed<LAYOUT>(a) ? (pim == N - 1 && g == GROUPS - 1) : (pim == 1 && g == 0))
                    finalize_member3<LOG2N>(a, b);
            }
        }
        if (!active) return;  // uniform per CTA
    }

    double2* buf = smem + c * G::PAD_N;
    auto make_pol = [&]() {
        if constexpr (WIDE) return BarSeg<T>{smem + C * G::PAD_N + c * (T / 32), 1 + c};
        else return BlockSeg<T, C>{smem + C * G::PAD_N, c};
    };
    const auto pol = make_pol();
    const double2 zero = make_double2(0.0, 0.0);
    const size_t pair0 = mem + (size_t)((bid % GROUPS) * C);  // (row 0, first column) of the CTA
    // WIDE: y (block layout, this thread's P outputs) -> both lines -> 256-bit row-pair stores
    auto store_wide = [&](const double2 (&v)[P]) {
#pragma unroll
        for (int l = 0; l < P; ++l) buf[G::at_block(t, G::pidx(t * P), l)] = v[l];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < N / (C * T); ++k) {
            const int r = threadIdx.x + C * T * k;
            const double2 v0 = smem[G::pidx(r)], v1 = smem[G::PAD_N + G::pidx(r)];
            double* dst = reinterpret_cast<double*>(a.T + pair0 + (size_t)r * N);
            asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(dst), "d"(v0.x), "d"(v0.y),
                         "d"(v1.x), "d"(v1.y) : "memory");
        }
    };

    double2 x[P], y[P];
    // n >= 512: the column goes through shared memory and the pre-processing reads x_j and
    // x_{N-j} there (no mirror registers); shorter lines keep the register path (measured, r01)
    constexpr bool CSM = BS_COL_SMEM_MIRROR && LOG2N >= 9;
    if constexpr (CSM) {
    if constexpr (LAYOUT == CL_PLANE && C == 2 && BS_COL_LD256) {
        // two columns per CTA (n >= 2048): each thread loads BOTH columns of a row with one
        // 256-bit load (LDG.E.ENL2.256; the pair is 32-B aligned, q0 even) and splits them into
        // the two engines' lines -- half the load instructions of the per-engine map, whose warp
        // requests touch 16 rows x 32 B each (lg_throttle-bound on c2, r01c)
        double2* buf0 = smem;
        double2* buf1 = smem + G::PAD_N;
#pragma unroll
        for (int k = 0; k < N / (C * T); ++k) {
            const int r = threadIdx.x + C * T * k;
            const double* src = reinterpret_cast<const double*>(a.T + pair0 + (size_t)r * N);
            double v0, v1, v2, v3;
            asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                         : "=d"(v0), "=d"(v1), "=d"(v2), "=d"(v3) : "l"(src));
            buf0[r] = make_double2(v0, v1);
            buf1[r] = make_double2(v2, v3);
        }
        __syncthreads();  // both lines were filled by the whole CTA
    } else {
#pragma unroll
    for (int mm = 0; mm < P; ++mm) {
        const int j = t + T * mm;
        buf[j] = a.T[gidx(j)];  // unpadded: conflict-free mirror reads in run_smem<true>
    }
    pol.sync();
    }
    Engine::template run_smem<true>(x, y, t, buf, a.tw, a.sinp, pol);
    } else {
        double2 xm[P];
#pragma unroll
        for (int mm = 0; mm < P; ++mm) {
            const int j = t + T * mm;
            x[mm] = a.T[gidx(j)];
            xm[mm] = (j == 0) ? zero : a.T[gidx(N - j)];
        }
        Engine::run(x, xm, y, t, buf, a.tw, a.sinp, pol);
    }

    if constexpr (MODE == C_ONE) {
        if constexpr (WIDE) {
#pragma unroll
            for (int l = 0; l < P; ++l) y[l] = cscale(y[l], a.scale);
            store_wide(y);
        } else {
#pragma unroll
            for (int l = 0; l < P; ++l) st_out(t * P + l, cscale(y[l], a.scale));
        }
    } else {
        const double k0sq = a.k0sq[b], eta = a.eta[b];
        // transverse symbol part: a_q (2-D) or a_y + a_z (3-D x-lines)
        const double lq = LAYOUT == CL_X3 ? a.lap[yl] + a.lap[q] : (LAYOUT == CL_SLAB && a.slab3) ? lq3 : a.lap[q];
#pragma unroll
        for (int l = 0; l < P; ++l) {
            const int p = t * P + l;
            // lambda = (a_p + a_q) - (k0^2 + i eta)   (symbol.cpp:69-80 + shift_symbol :97-100)
            const double lr = (a.lap[p] + lq) - k0sq;
            const double li = -eta;
            double2 w;
            if constexpr (MODE == C_FD) {
                // FourierDiag m (correction.cpp:63-68), padded mode layout shared by the batch
                // (CL_SLAB: the rank's own n x slab_cols block of m, in the t_cols layout)
                const size_t fi = LAYOUT == CL_X3     ? ((size_t)p * N + yl) * N + q
                                  : LAYOUT == CL_SLAB ? (size_t)p * LS + qa
                                                      : (size_t)p * N + q;
                w = cscale(a.fd[fi], a.scale);
            } else if constexpr (MODE == C_GREEN) {
                const double s = a.scale * rcp_green(fma(lr, lr, li * li));
                w = make_double2(lr * s, -li * s);  // scale / lambda
            } else {
                w = make_double2(lr * a.scale, li * a.scale);  // scale * lambda
            }
            const double2 v = (p == 0 || q == 0) ? zero : cmul(y[l], w);
            buf[G::at_block(t, G::pidx(t * P), l)] = v;
        }
        pol.sync();
        if constexpr (CSM) {
            Engine::run_smem(x, y, t, buf, a.tw, a.sinp, pol);
        } else {
            double2 xm[P];
#pragma unroll
            for (int mm = 0; mm < P; ++mm) {
                const int j = t + T * mm;
                x[mm] = buf[G::pidx(j)];
                xm[mm] = (j == 0) ? zero : buf[G::pidx(N - j)];
            }
            pol.sync();
            Engine::run(x, xm, y, t, buf, a.tw, a.sinp, pol);
        }
        if constexpr (WIDE) {
            store_wide(y);
        } else {
#pragma unroll
            for (int l = 0; l < P; ++l) st_out(t * P + l, y[l]);
        }
    }
}

#ifndef BS_COL_REGS
#define BS_COL_REGS 128  // register budget the column kernel's launch bounds are sized for (P = 16)
#endif
template <int LOG2N, int MODE, int C, int PP, int LAYOUT = CL_PLANE>
__global__ void __launch_bounds__(C * Geom<LOG2N, PP>::T, (MinBlocks<C * Geom<LOG2N, PP>::T, PP >= 16 ? BS_COL_REGS : 64>::value))
col_kernel(const ColArgs a) {
    // BS_COL_REVERSE: CTAs take the column groups in reverse order.  The hardware dispatches
    // CTAs by increasing index, so the column pass starts on the last members the row pass
    // wrote (their T still in L2) and ends on the first ones, which the next row pass then
    // reads first, again from L2: each handoff reuses the L2-resident tail of the other pass.
    col_group<LOG2N, MODE, C, PP, LAYOUT>(a, col_reversed<LAYOUT>(a) ? gridDim.x - 1 - blockIdx.x : blockIdx.x);
}

}  // namespace bs
