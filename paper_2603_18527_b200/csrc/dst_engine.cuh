// dst_engine.cuh -- register/shared-memory DST-I engine for sm_100a (fp64 complex).
//
// One "engine" transforms one line of n = 2^LOG2N complex samples x_0..x_{n-1}
// (x_0 == 0 is the Dirichlet padding slot; the DST-I length is n-1) into
//     Y_k = sum_{j=1}^{n-1} x_j sin(pi j k / n),     k = 0..n-1 (Y_0 = 0),
// i.e. the reference's forward DST-I convention (plain sine sum; FFTW RODFT00 / 2,
// proj/include/bp/transforms.hpp:15-24), TIMES kEngineGain = 4: the factors 1/2 of the pre-
// and post-processing below are dropped and callers fold 4^k into one scale (exact).
//
// Algorithm (one length-n complex FFT per complex line, not the 2(n+1) odd extension):
//   y_j = sin(pi j/n)(x_j + x_{n-j}) + (x_j - x_{n-j})/2          (pre-processing)
//   W   = DFT_n(y)                                                (Stockham passes)
//   Y_2k   = (i/2)(W_k - W_{n-k})                                 (post-processing)
//   Y_2k+1 = W_0/2 + sum_{m=1}^{k} (W_m + W_{n-m})/2              (prefix sum)
// The real and imaginary parts of x are two real DST-I problems; packing them as one
// complex y makes W_k and W_{n-k} separate them with no extra work.  The last radix-2
// Stockham pass is fused into the post-processing.
//
// Thread layout: T = n/P threads per engine, P points per thread.
//   input   thread t holds x_{t + T m} and the mirror x_{n - t - T m}, m < P
//           (stride-T: consecutive threads read consecutive addresses -> coalesced)
//   output  thread t holds Y_{t P + l}, l < P (contiguous block)
// Passes exchange data through one padded shared-memory line per engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

// Twiddles and pre-processing sines are built by in-register complex multiplications from one
// table load each (device tables for every power measured slower, r01: c1 row 463 vs 365 us,
// c4 +13 % -- L1 latency on the butterfly critical path).

namespace bs {

constexpr double kEngineGain = 4.0;  // each engine pass returns 4 x the plain sine sum

// ------------------------------------------------------------------ complex helpers
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double cnorm(double2 a) { return a.x * a.x + a.y * a.y; }
// multiply by -i / +i
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }
__device__ __forceinline__ double2 mul_pi(double2 a) { return make_double2(-a.y, a.x); }

// a * exp(-2 pi i K / R), R <= 16, compile-time K
template <int K, int R>
__device__ __forceinline__ double2 mul_w(double2 a) {
    constexpr int k16 = (K * 16 / R) % 16;  // angle in units of 2pi/16
    constexpr double C1 = 0.92387953251128673848;  // cos(pi/8)
    constexpr double S1 = 0.38268343236508978178;  // sin(pi/8)
    constexpr double R2 = 0.70710678118654752440;  // 1/sqrt(2)
    if constexpr (k16 == 0) return a;
    else if constexpr (k16 == 4) return mul_mi(a);
    else if constexpr (k16 == 8) return make_double2(-a.x, -a.y);
    else if constexpr (k16 == 12) return mul_pi(a);
    else if constexpr (k16 == 2) return make_double2((a.x + a.y) * R2, (a.y - a.x) * R2);
    else if constexpr (k16 == 6) return make_double2((a.y - a.x) * R2, -(a.x + a.y) * R2);
    else {
        // exp(-i pi k16/8) = c - i s
        constexpr double c = k16 == 1 ? C1 : k16 == 3 ? S1 : k16 == 5 ? -S1 : k16 == 7 ? -C1
                           : k16 == 9 ? -C1 : k16 == 11 ? -S1 : k16 == 13 ? S1 : C1;
        constexpr double s = k16 == 1 ? S1 : k16 == 3 ? C1 : k16 == 5 ? C1 : k16 == 7 ? S1
                           : k16 == 9 ? -S1 : k16 == 11 ? -C1 : k16 == 13 ? -C1 : -S1;
        return make_double2(a.x * c + a.y * s, a.y * c - a.x * s);
    }
}

// In-register forward DFT of size R (natural order in and out), radix-2 DIT recursion.
template <int R>
struct Dft {
    template <int STRIDE = 1>
    __device__ __forceinline__ static void run(double2* v) {
        double2 e[R / 2], o[R / 2];
#pragma unroll
        for (int k = 0; k < R / 2; ++k) {
            e[k] = v[(2 * k) * STRIDE];
            o[k] = v[(2 * k + 1) * STRIDE];
        }
        Dft<R / 2>::template run<1>(e);
        Dft<R / 2>::template run<1>(o);
        combine<0, STRIDE>(e, o, v);
    }
    template <int K, int STRIDE = 1>
    __device__ __forceinline__ static void combine(const double2* e, const double2* o, double2* v) {
        if constexpr (K < R / 2) {
            const double2 t = mul_w<K, R>(o[K]);
            v[K * STRIDE] = cadd(e[K], t);
            v[(K + R / 2) * STRIDE] = csub(e[K], t);
            combine<K + 1, STRIDE>(e, o, v);
        }
    }
};
template <>
struct Dft<1> {
    template <int STRIDE = 1>
    __device__ __forceinline__ static void run(double2*) {}
};
template <>
struct Dft<2> {
    template <int STRIDE = 1>
    __device__ __forceinline__ static void run(double2* v) {
        const double2 a = v[0], b = v[STRIDE];
        v[0] = cadd(a, b);
        v[STRIDE] = csub(a, b);
    }
};

// (cos, sin)(pi m / 16), m < 16: the pre-processing factor sin(pi (t + T m)/N) with
// T m / N = m / P is sin(pi t/N) cos(pi m/P) + cos(pi t/N) sin(pi m/P).
struct CS {
    double c, s;
};
__device__ constexpr CS kCS16[16] = {
    {1.0, 0.0},
    {0.9807852804032304, 0.19509032201612825},
    {0.9238795325112867, 0.3826834323650898},
    {0.8314696123025452, 0.5555702330196022},
    {0.7071067811865476, 0.7071067811865475},
    {0.5555702330196023, 0.8314696123025452},
    {0.38268343236508984, 0.9238795325112867},
    {0.19509032201612833, 0.9807852804032304},
    {0.0, 1.0},
    {-0.1950903220161282, 0.9807852804032304},
    {-0.3826834323650897, 0.9238795325112867},
    {-0.555570233019602, 0.8314696123025455},
    {-0.7071067811865475, 0.7071067811865476},
    {-0.8314696123025453, 0.5555702330196022},
    {-0.9238795325112867, 0.3826834323650899},
    {-0.9807852804032304, 0.1950903220161286},
};

// powers pw[r] = w^r, r < R, by squaring (depth <= log2 R + 1 multiplications)
template <int R>
__device__ __forceinline__ void twiddle_powers(double2 w, double2 (&pw)[R]) {
    pw[0] = make_double2(1.0, 0.0);
    if constexpr (R > 1) pw[1] = w;
#pragma unroll
    for (int r = 2; r < R; ++r) pw[r] = (r & 1) ? cmul(pw[r - 1], w) : cmul(pw[r / 2], pw[r / 2]);
}

// ------------------------------------------------------------------ engine geometry
// PP: requested points per thread (16 or 8); capped at N/2 for tiny lines.
template <int LOG2N, int PP = 16>
struct Geom {
    static constexpr int N = 1 << LOG2N;
    static constexpr int P = (N / 2) < PP ? (N / 2) : PP;  // points per thread
    static constexpr int T = N / P;                        // threads per engine
    static constexpr int H = N / 2;
    static constexpr int PAD_N = N + N / 8 + N / 64 + 1;   // padded smem line (double2)
    // i + i/8 + i/64: every access pattern of the engine (stride 1, 4, 8, 16, 32 over the 8
    // lanes of a 128-bit shared-memory phase) lands on 8 distinct 16-byte bank groups.
    __host__ __device__ static constexpr int pidx(int i) { return i + (i >> 3) + (i >> 6); }
    struct Pidx {
        __device__ __forceinline__ int operator()(int i) const { return pidx(i); }
    };
    // Split addressing: pidx(x + k) = pidx(x) + pidx(k) whenever 8 | k and (x mod 64) +
    // (k mod 64) < 64.  With the per-thread base px = pidx(x) computed once and k a constant
    // of an unrolled loop, every access becomes [base + immediate] (the compiler cannot prove
    // the split itself and otherwise recomputes i + i/8 + i/64 per access: ~10 % of all
    // instructions, r01 ncu).  x64max: an upper bound of x mod 64 over the threads; both
    // branches compute the same index, the condition folds at compile time.
    __device__ __forceinline__ static int padd(int x, int px, int x64max, int k) {
        return ((k & 7) == 0 && (k & 63) + x64max < 64) ? px + pidx(k) : pidx(x + k);
    }
    // pidx(x + r) for x = 0 mod 8, (x mod 64) + r < 64 (block layout t*P + r, P in {8, 16})
    __device__ __forceinline__ static int psmall(int px, int r) { return px + r + (r >> 3); }
    static constexpr int TM64 = (T < 64 ? T : 64) - 1;  // bound of t mod 64, t < T
    // element t + T m of the stride layout (bt = pidx(t))
    __device__ __forceinline__ static int at_stride(int t, int bt, int m) {
        return T >= 8 ? padd(t, bt, TM64, T * m) : pidx(t + T * m);
    }
    // element t P + l of the block layout (bp = pidx(t P))
    __device__ __forceinline__ static int at_block(int t, int bp, int l) {
        return (P == 8 || P == 16) ? psmall(bp, l) : pidx(t * P + l);
    }
};

// Stockham pass list: product of radices == N/2; first radix == P; radices <= P.
template <int LOG2N, int PP = 16>
struct Passes {
    using G = Geom<LOG2N, PP>;
    static constexpr int RMAX = G::P;
    static constexpr int REM = G::H / G::P;  // remaining product after the first pass
    static constexpr int R2 = REM >= RMAX ? RMAX : REM;  // second pass radix (1 = none)
    static constexpr int REM2 = REM / R2;
    static constexpr int R3 = REM2 >= RMAX ? RMAX : REM2;
    static constexpr int REM3 = REM2 / R3;
    static constexpr int R4 = REM3 >= RMAX ? RMAX : REM3;
    static constexpr int REM4 = REM3 / R4;
    static constexpr int R5 = REM4;
    static_assert(R5 <= RMAX, "line too long for this engine");
};

// ------------------------------------------------------------------ sync/scan policies
// Engine threads are T contiguous lanes of one warp (T <= 32).
template <int T>
struct WarpSeg {
    static_assert(T <= 32, "WarpSeg spans one warp");
    __device__ __forceinline__ void sync() const { __syncwarp(); }
    // exclusive prefix over the T lanes of this engine (lane segment aligned to T)
    __device__ __forceinline__ double2 exclusive_scan(double2 v, int t) const {
        double2 incl = v;
#pragma unroll
        for (int d = 1; d < T; d <<= 1) {
            const double ux = __shfl_up_sync(0xffffffffu, incl.x, d, T);
            const double uy = __shfl_up_sync(0xffffffffu, incl.y, d, T);
            if (t >= d) {
                incl.x += ux;
                incl.y += uy;
            }
        }
        return csub(incl, v);
    }
    // deterministic sum over the T lanes of the engine (result valid in every lane)
    __device__ __forceinline__ double sum(double v, int) const {
#pragma unroll
        for (int d = T / 2; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d, T);
        return v;
    }
    __device__ __forceinline__ int bcast0(int v, int) const {
        return __shfl_sync(0xffffffffu, v, ((threadIdx.x & 31) / T) * T);
    }
    // xm[m] = x_{N - t - T m} for data in the stride layout x[m] = x_{t + T m} (N = T P):
    // lane T - t holds it in register P-1-m; lane 0 holds its own mirror in register P-m.
    template <int P, class Idx>
    __device__ __forceinline__ void mirror(const double2 (&x)[P], double2 (&xm)[P], int t, double2*,
                                           Idx) const {
        const int src = ((threadIdx.x & 31) / T) * T + ((T - t) & (T - 1));
#pragma unroll
        for (int m = 0; m < P; ++m) {
            const double2 v = make_double2(__shfl_sync(0xffffffffu, x[P - 1 - m].x, src),
                                           __shfl_sync(0xffffffffu, x[P - 1 - m].y, src));
            xm[m] = (t != 0) ? v : (m == 0 ? make_double2(0.0, 0.0) : x[P - m]);
        }
    }
};

// Engine = T/32 consecutive whole warps synchronised by named barrier `id` (1..15).
// scratch: >= T/32 double2 of shared memory private to the engine.
template <int T>
struct BarSeg {
    static_assert(T % 32 == 0 && T > 32, "BarSeg spans several whole warps");
    static constexpr int W = T / 32;
    double2* scratch;
    int id;
    __device__ __forceinline__ void sync() const {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(T) : "memory");
    }
    __device__ __forceinline__ double2 exclusive_scan(double2 v, int t) const {
        const int lane = t & 31, w = t >> 5;
        double2 incl = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const double ux = __shfl_up_sync(0xffffffffu, incl.x, d);
            const double uy = __shfl_up_sync(0xffffffffu, incl.y, d);
            if (lane >= d) {
                incl.x += ux;
                incl.y += uy;
            }
        }
        if (lane == 31) scratch[w] = incl;
        sync();
        double2 off = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < W; ++k)
            if (k < w) off = cadd(off, scratch[k]);
        sync();
        return cadd(off, csub(incl, v));
    }
    __device__ __forceinline__ double sum(double v, int t) const {
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
        if ((t & 31) == 0) scratch[t >> 5].x = v;
        sync();
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < W; ++k) s += scratch[k].x;
        sync();
        return s;
    }
    __device__ __forceinline__ int bcast0(int v, int t) const {
        if (t == 0) scratch[0].y = __longlong_as_double((long long)v);
        sync();
        const int r = (int)__double_as_longlong(scratch[0].y);
        sync();
        return r;
    }
    // mirror exchange through the engine's shared-memory line (idx = padding function)
    template <int P, class Idx>
    __device__ __forceinline__ void mirror(const double2 (&x)[P], double2 (&xm)[P], int t, double2* buf,
                                           Idx idx) const {
        constexpr int N = T * P;
#pragma unroll
        for (int m = 0; m < P; ++m) buf[idx(t + T * m)] = x[m];
        sync();
#pragma unroll
        for (int m = 0; m < P; ++m) {
            const int j = t + T * m;
            xm[m] = (j == 0) ? make_double2(0.0, 0.0) : buf[idx(N - j)];
        }
        sync();
    }
};

// Engines spread over the CTA (column kernel): E engines x T threads; scan scratch in smem,
// laid out [t][e] with row pitch E+1 so both the write (lanes = engines) and the per-engine
// scan read (lanes = t) are bank-conflict free.
template <int T, int E>
struct BlockSeg {
    static constexpr int CH = (T + 31) / 32;  // 32-wide chunks per engine
    // scan scratch + the chunk totals of the parallel scan (T >= 64: one warp per chunk)
    static constexpr int SCRATCH = T * (E + 1) + (CH > 1 ? E * CH : 0);  // double2
    double2* scratch;
    int e;
    __device__ __forceinline__ static int sidx(int ee, int tt) { return tt * (E + 1) + ee; }
    __device__ __forceinline__ void sync() const { __syncthreads(); }
    __device__ __forceinline__ double2 exclusive_scan(double2 v, int t) const {
        scratch[sidx(e, t)] = v;
        __syncthreads();
        if constexpr (CH > 1 && (T % 32) == 0) {
            // long lines: the CTA has exactly E * CH warps (C * T threads), one per 32-value
            // chunk; each scans its chunk, the chunk totals are combined afterwards in the same
            // order as the sequential carry (bit-identical; the serial version kept 14 of 16
            // warps waiting at the barrier on c2's 4096-point columns)
            double2* tot = scratch + T * (E + 1);
            const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
            const int ee = warp / CH, c = warp % CH, tt = c * 32 + lane;
            const double2 x = scratch[sidx(ee, tt)];
            double2 incl = x;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const double ux = __shfl_up_sync(0xffffffffu, incl.x, d);
                const double uy = __shfl_up_sync(0xffffffffu, incl.y, d);
                if (lane >= d) {
                    incl.x += ux;
                    incl.y += uy;
                }
            }
            scratch[sidx(ee, tt)] = csub(incl, x);
            if (lane == 31) tot[ee * CH + c] = incl;
            __syncthreads();
            double2 carry = make_double2(0.0, 0.0);
            const int cm = t >> 5;
            for (int k = 0; k < cm; ++k) carry = cadd(carry, tot[e * CH + k]);
            return cadd(carry, scratch[sidx(e, t)]);
        }
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int nwarps = (blockDim.x + 31) >> 5;
        constexpr int CH = (T + 31) / 32;  // 32-wide chunks per engine
        for (int ee = warp; ee < E; ee += nwarps) {
            double2 carry = make_double2(0.0, 0.0);
            for (int c = 0; c < CH; ++c) {
                const int tt = c * 32 + lane;
                double2 x = tt < T ? scratch[sidx(ee, tt)] : make_double2(0.0, 0.0);
                double2 incl = x;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const double ux = __shfl_up_sync(0xffffffffu, incl.x, d);
                    const double uy = __shfl_up_sync(0xffffffffu, incl.y, d);
                    if (lane >= d) {
                        incl.x += ux;
                        incl.y += uy;
                    }
                }
                if (tt < T) scratch[sidx(ee, tt)] = cadd(carry, csub(incl, x));
                const double tx = __shfl_sync(0xffffffffu, incl.x, 31);
                const double ty = __shfl_sync(0xffffffffu, incl.y, 31);
                carry = cadd(carry, make_double2(tx, ty));
            }
        }
        __syncthreads();
        return scratch[sidx(e, t)];
    }
};

// Thread -> (engine c, engine thread t) for the column kernels (C engines per CTA, T threads
// each).  Global coalescing wants the C engines (adjacent columns) side by side in a warp; the
// shared-memory side wants each 8-lane phase of a 16-B access inside ONE engine, where the pidx
// padding makes the accesses conflict-free.  With C in {2, 4}: lane = (t mod 32/C) + (32/C) c,
// so a warp still covers C adjacent columns x 32/C rows.  C = 8 keeps c fastest (a phase is 8
// engines at one t; the odd engine stride PAD_N keeps those conflict-free).
template <int T, int C>
__device__ __forceinline__ void col_thread_map(int& t, int& c) {
    constexpr int LPE = 32 / C;
    // (t masked to [0, T) in the C in {2, 4} map: a no-op for the launched block size that lets
    // the compiler split pidx(t + T m) into a base + immediates; c4 column pass 398 -> 385 us)
    if constexpr ((C == 2 || C == 4) && T >= LPE) {
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        c = lane / LPE;
        t = (lane % LPE + LPE * w) & (T - 1);
    } else {
        c = threadIdx.x % C;
        t = threadIdx.x / C;  // (masking here measured slower on c1: 247 vs 234 us)
    }
}

// ------------------------------------------------------------------ the engine
template <int LOG2N, int PP = 16>
struct DstEngine {
    using G = Geom<LOG2N, PP>;
    using PS = Passes<LOG2N, PP>;
    static constexpr int N = G::N, P = G::P, T = G::T, H = G::H;

    // One Stockham pass of radix R over the line in `buf` (read all, sync, write all, sync).
    // Ns = product of previous radices.  Twiddles from tw[k] = exp(-2 pi i k / N).
    template <int R, int NS, class Pol>
    __device__ __forceinline__ static void pass(double2* buf, int t, const double2* __restrict__ tw,
                                                const Pol& pol) {
        if constexpr (R > 1) {
            constexpr int V = P / R;  // butterflies per thread
            constexpr int STRIDE_IN = N / R;
            double2 v[P];
            const int bt = G::pidx(t);
#pragma unroll
            for (int b = 0; b < V; ++b) {
                const int jj = t + T * b;
                const int jm = jj % NS;
                // exp(-2 pi i jm r / (NS R)) = w^r with w = tw[jm N/(NS R)]: one load per butterfly
                double2 pw[R];
                twiddle_powers<R>(__ldg(&tw[jm * (N / (NS * R))]), pw);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    // jj + r STRIDE_IN = t + (T b + r STRIDE_IN), a multiple of T added
                    double2 x = buf[G::at_stride(t, bt, b + r * (STRIDE_IN / T))];
                    if (r > 0) x = cmul(x, pw[r]);
                    v[b * R + r] = x;
                }
                Dft<R>::template run<1>(&v[b * R]);
            }
            pol.sync();
            // write index base(b) + r NS with base(b) = (jj/NS) NS R + jj%NS, jj = t + T b:
            // = wt + K(b) for the per-thread wt below (t < T, T and NS powers of 2)
            constexpr int Q = NS > T ? NS / T : 1;
            const int wt = NS <= T ? (t / NS) * NS * R + t % NS : t;
            const int pwt = G::pidx(wt);
            // bound of wt mod 64 over t < T
            constexpr int W64 = NS <= T ? ((NS * R) % 64 == 0 ? (NS < 64 ? NS : 64) - 1 : 63)
                                        : G::TM64;
#pragma unroll
            for (int b = 0; b < V; ++b) {
                const int kb = NS <= T ? T * R * b : (b / Q) * NS * R + T * (b % Q);
#pragma unroll
                for (int r = 0; r < R; ++r) buf[G::padd(wt, pwt, W64, kb + r * NS)] = v[b * R + r];
            }
            pol.sync();
        }
    }

    // x[m] = x_{t+Tm}, xm[m] = x_{N-t-Tm} (mirror; must be 0 where the index is N).
    // On return y[l] = Y_{tP+l}.  buf: this engine's padded smem line (G::PAD_N double2).
    // DST-I pre-processing of one element: y_j = 2 sin(pi j/N)(x_j + x_{N-j}) + (x_j - x_{N-j})
    // with 2 sin(pi j/N) = st cos(2 pi m/P') + ct sin(...) for j = t + T m (kCS16 table)
    __device__ __forceinline__ static double2 pre(double2 x, double2 xm, int m, double st, double ct) {
        constexpr int STEP = 16 / P;
        const double s = fma(st, kCS16[m * STEP].c, ct * kCS16[m * STEP].s);
        const double2 a = cadd(x, xm);
        const double2 d = csub(x, xm);
        return make_double2(fma(s, a.x, d.x), fma(s, a.y, d.y));
    }
    // same with s = 2 sin(pi j/N) given
    __device__ __forceinline__ static double2 pre_s(double2 x, double2 xm, double s) {
        const double2 a = cadd(x, xm);
        const double2 d = csub(x, xm);
        return make_double2(fma(s, a.x, d.x), fma(s, a.y, d.y));
    }
    // 2 sin(pi j/N) for j = t + T m (sinp holds 2 sin(pi j/N), j < N)
    __device__ __forceinline__ static double sin2(const double* __restrict__ sinp, int t, int m, double st,
                                                  double ct) {
        constexpr int STEP = 16 / P;
        return fma(st, kCS16[m * STEP].c, ct * kCS16[m * STEP].s);
    }

    template <class Pol>
    __device__ __forceinline__ static void run(const double2 (&x)[P], const double2 (&xm)[P], double2 (&y)[P],
                                               int t, double2* buf, const double2* __restrict__ tw,
                                               const double* __restrict__ sinp, const Pol& pol) {
        // --- pre-processing + first Stockham pass (radix P, Ns = 1, data already in registers)
        double2 v[P];
        // 2 sin(pi t/N), 2 cos(pi t/N): the engine computes 4x the sine sum (the 1/2 factors
        // of pre- and post-processing are folded into the caller's scale, exact powers of 2)
        const double st = 2.0 * __ldg(&sinp[t]), ct = 2.0 * __ldg(&sinp[t + H]);
#pragma unroll
        for (int m = 0; m < P; ++m) {
            const int j = t + T * m;
            v[m] = (j == 0) ? make_double2(0.0, 0.0) : pre_s(x[m], xm[m], sin2(sinp, t, m, st, ct));
        }
        transform(v, y, t, buf, tw, pol);
    }

    // Same transform with the line already in buf (natural order at pidx(j)): the mirror
    // x_{N-j} is read from shared memory as each element is pre-processed, so neither the
    // line nor its mirror has to be held in registers.  v: scratch of P registers.
    // DENSE: the line sits UNPADDED in buf (x_j at buf[j]).  The mirror reads of one 8-lane
    // phase, x_{N-t-Tm} for 8 consecutive t, are 8 consecutive elements that straddle an 8-block
    // boundary; under the pidx padding every such phase is a 2-way bank conflict (91 % of the
    // row kernel's excess wavefronts, r01c), unpadded any 8 consecutive elements hit 8 distinct
    // 16-byte bank groups.  The passes after the pre-processing use the padded layout as before.
    template <bool DENSE = false, class Pol>
    __device__ __forceinline__ static void run_smem(double2 (&v)[P], double2 (&y)[P], int t, double2* buf,
                                                    const double2* __restrict__ tw,
                                                    const double* __restrict__ sinp, const Pol& pol) {
        const double st = 2.0 * __ldg(&sinp[t]), ct = 2.0 * __ldg(&sinp[t + H]);
        // x_{N-j}, j = t + T m: (T - t) + T (P-1-m) for t > 0; T (P-m) (its own slot P-m)
        // for t = 0 (the split needs T - t < T, so lane 0 takes a direct constant index)
        const int bt = G::pidx(t), tm = (T - t) & (T - 1), btm = G::pidx(tm);
#pragma unroll
        for (int m = 0; m < P; ++m) {
            const int j = t + T * m;
            const double2 x = DENSE ? buf[j] : buf[G::at_stride(t, bt, m)];
            const int mi = DENSE ? ((N - j) & (N - 1))
                                 : t == 0 ? G::pidx((N - T * m) & (N - 1)) : G::at_stride(tm, btm, P - 1 - m);
            const double2 xm = buf[mi];
            v[m] = (j == 0) ? make_double2(0.0, 0.0) : pre_s(x, xm, sin2(sinp, t, m, st, ct));
        }
        pol.sync();
        transform(v, y, t, buf, tw, pol);
    }

    // first Stockham pass (radix P in registers), the remaining passes, fused post-processing
    template <class Pol>
    __device__ __forceinline__ static void transform(double2 (&v)[P], double2 (&y)[P], int t, double2* buf,
                                                     const double2* __restrict__ tw, const Pol& pol) {
        Dft<P>::template run<1>(v);
        const int bp = G::pidx(t * P);
#pragma unroll
        for (int r = 0; r < P; ++r) buf[G::at_block(t, bp, r)] = v[r];
        pol.sync();
        // --- remaining passes up to length N/2 (radix-2 last pass fused below)
        pass<PS::R2, P>(buf, t, tw, pol);
        pass<PS::R3, P * PS::R2>(buf, t, tw, pol);
        pass<PS::R4, P * PS::R2 * PS::R3>(buf, t, tw, pol);
        pass<PS::R5, P * PS::R2 * PS::R3 * PS::R4>(buf, t, tw, pol);
        // --- fused final radix-2 pass + DST-I post-processing + prefix sum
        constexpr int K = P / 2;  // k values per thread: k = t*K + i
        double2 ev[K], od[K];     // Y_2k and S_k
        // split bases (K = 8): k = 8t + i -> pidx(8t) + i; H - k, N - k -> pidx(H - 8t) for
        // i = 0, pidx(H - 8t - 8) + 8 - i otherwise (same for N); H a multiple of 64 (N >= 128)
        constexpr bool KS = K == 8 && H % 64 == 0;
        const int pk = G::pidx(t * K), ph0 = G::pidx(H - t * K), ph1 = G::pidx(H - t * K - K);
        const int pn0 = G::pidx((N - t * K) & (N - 1)), pn1 = G::pidx(N - t * K - K);
        const double2 w0 = __ldg(&tw[t * K]), w1 = __ldg(&tw[1]);
        double2 w = w0;           // exp(-2 pi i k/N), stepped by exp(-2 pi i/N)
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const int k = t * K + i;
            if (i > 0) w = cmul(w, w1);
            const double2 a = buf[KS ? pk + i : G::pidx(k)];
            const double2 b = cmul(buf[KS ? pk + i + G::pidx(H) : G::pidx(k + H)], w);
            const double2 Wk = cadd(a, b);
            if (k == 0) {
                ev[i] = make_double2(0.0, 0.0);
                od[i] = Wk;
            } else {
                // W_{N-k} = a_{H-k} - w^{H-k} b_{H-k},  w^{H-k} = -conj(w^k)
                const double2 a2 = buf[KS ? (i == 0 ? ph0 : ph1 + K - i) : G::pidx(H - k)];
                const double2 b2 = buf[KS ? (i == 0 ? pn0 : pn1 + K - i) : G::pidx(N - k)];
                const double2 Wnk = cadd(a2, cmul(b2, cconj(w)));
                const double2 dif = csub(Wk, Wnk);
                ev[i] = make_double2(-dif.y, dif.x);  // i (Wk - Wnk)
                od[i] = cadd(Wk, Wnk);
            }
        }
        // local inclusive prefix of S
#pragma unroll
        for (int i = 1; i < K; ++i) od[i] = cadd(od[i], od[i - 1]);
        const double2 off = pol.exclusive_scan(od[K - 1], t);
#pragma unroll
        for (int i = 0; i < K; ++i) {
            y[2 * i] = ev[i];
            y[2 * i + 1] = cadd(od[i], off);
        }
        pol.sync();  // buffer free for reuse
    }
};

}  // namespace bs
