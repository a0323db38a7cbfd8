// bornsweep.cu -- C ABI (include/bornsweep.h) over the sm_100a sweep kernels.
//
// Host side of the drop-in boundary: problem handles (bp::Problem), operator applications,
// and the iteration driver (bp::run, proj/src/iterate.cpp:88-153) executed as a device-side
// loop: each sweep is two kernel launches, the termination test runs on the device, and the
// host replays CUDA graphs of GRAPH_SWEEPS sweeps, polling one pinned counter per replay.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "bornsweep.h"
#include "sweep_launch.cuh"
#include "generic_kernels.cuh"

using namespace bs;

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CU(call)                                                                          \
    do {                                                                                  \
        cudaError_t _e = (call);                                                          \
        if (_e != cudaSuccess)                                                            \
            return set_err(BP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

#ifndef BS_GRAPH_SWEEPS
#define BS_GRAPH_SWEEPS 16
#endif
constexpr int kGraphSweeps = BS_GRAPH_SWEEPS;
constexpr double kPi = 3.14159265358979323846;
// sinp table: sin(pi j/n)
constexpr double kSinScale = 1.0;
constexpr double kSymbolDivGuard = 1e-14;  // proj/include/bp/symbol.hpp:24

// ------------------------------------------------------------------ small kernels
// The staging kernels of the host path (pack / unpack / finite check) stream hundreds of MB per
// step through the L2 while ANOTHER handle's sweeps (bs.Pipeline) live off their L2-resident
// waves: their global accesses carry evict_first so they do not displace that data.
__device__ __forceinline__ double2 ld_once(const double2* p, unsigned long long pol) {
    double2 v;
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_once(double2* p, double2 v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}

// dense (reference layout, (n-1)^dim per member) -> padded (n^dim per member, zero node at 0)
__global__ void pack_kernel(const double2* __restrict__ dense, double2* __restrict__ padded,
                            int batch, int log2n, int dim) {
    const int n = 1 << log2n, nd = n - 1;
    const unsigned long long pol = l2_policy_first();
    const size_t total = (size_t)batch << (dim * log2n);
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const size_t b = idx >> (dim * log2n);
        const int j = (int)(idx & (n - 1)), i = (int)((idx >> log2n) & (n - 1));
        const int x = dim == 3 ? (int)((idx >> (2 * log2n)) & (n - 1)) : 1;
        double2 v = make_double2(0.0, 0.0);
        if (dense && i > 0 && j > 0 && x > 0) {
            const size_t plane = dim == 3 ? (size_t)(x - 1) * nd : 0;
            const size_t per = dim == 3 ? (size_t)nd * nd * nd : (size_t)nd * nd;
            v = ld_once(&dense[b * per + ((plane + (i - 1)) * nd + (j - 1))], pol);
        }
        padded[idx] = v;  // (the field the sweeps read next: default priority)
    }
}

// select: per-member ping/pong source (result_buf) when non-null
__global__ void unpack_kernel(const double2* __restrict__ p0, const double2* __restrict__ p1,
                              const int* __restrict__ select, double2* __restrict__ dense,
                              int batch, int log2n, int dim) {
    const int n = 1 << log2n, nd = n - 1;
    const size_t per = dim == 3 ? (size_t)nd * nd * nd : (size_t)nd * nd;
    const size_t total = (size_t)batch * per;
    const unsigned long long pol = l2_policy_first();
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const size_t b = idx / per;
        size_t r = idx % per;
        const int j = (int)(r % nd) + 1;
        r /= nd;
        const int i = (int)(r % nd) + 1;
        const int x = (int)(r / nd) + 1;  // 3-D only
        const double2* src = (select && select[b]) ? p1 : p0;
        const size_t line = dim == 3 ? ((size_t)x << log2n) + i : (size_t)i;
        st_once(&dense[idx], ld_once(&src[(b << (dim * log2n)) + (line << log2n) + j], pol), pol);
    }
}

// op: 0 A u, 1 V u, 2 V^H u, 3 f - A u (sub = f)
__global__ void pointwise_kernel(int op, const double2* __restrict__ u, const double2* __restrict__ k2,
                                 const double2* __restrict__ f, const double* __restrict__ k0sq,
                                 const double* __restrict__ eta, double inv_h2,
                                 double2* __restrict__ out, int batch, int log2n, int dim,
                                 int pad = 1) {
    const int n = 1 << log2n;
    const size_t total = (size_t)batch << (dim * log2n);
    const size_t plane = (size_t)n * n;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const size_t b = idx >> (dim * log2n);
        const int i = (int)((idx >> log2n) & (n - 1)), j = (int)(idx & (n - 1));
        const int x = dim == 3 ? (int)((idx >> (2 * log2n)) & (n - 1)) : 1;
        double2 o = make_double2(0.0, 0.0);
        if (!pad || (i > 0 && j > 0 && x > 0)) {
            const double2 uu = u[idx], kk = k2[idx];
            const double2 shift = make_double2(k0sq[b], eta[b]);
            if (op == 1) {
                o = cmul(uu, csub(kk, shift));
            } else if (op == 2) {
                o = cmul(cconj(csub(kk, shift)), uu);
            } else {
                double2 s = cscale(uu, dim == 3 ? 6.0 : 4.0);
                if (dim == 3) {
                    s = csub(s, u[idx - plane]);
                    s = csub(s, u[idx + plane]);
                }
                s = csub(s, u[idx - n]);
                s = csub(s, u[idx + n]);
                s = csub(s, u[idx - 1]);
                if (j + 1 < n) s = csub(s, u[idx + 1]);
                o = csub(cscale(s, inv_h2), cmul(kk, uu));
                if (op == 3) o = csub(f[idx], o);
            }
        }
        out[idx] = o;
    }
}

// per-member sum of |x|^2 over a padded field; partials[b*nchunk + c], deterministic
__global__ void norm_partial_kernel(const double2* __restrict__ x, size_t per, int nchunk,
                                    double* __restrict__ partials) {
    const int b = blockIdx.y, c = blockIdx.x;
    const size_t chunk = (per + nchunk - 1) / nchunk;
    const size_t lo = c * chunk, hi = min(per, lo + chunk);
    double s = 0.0;
    for (size_t k = lo + threadIdx.x; k < hi; k += blockDim.x) s += cnorm(x[b * per + k]);
    __shared__ double red[256];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int d = blockDim.x / 2; d > 0; d >>= 1) {
        if (threadIdx.x < d) red[threadIdx.x] += red[threadIdx.x + d];
        __syncthreads();
    }
    if (threadIdx.x == 0) partials[b * nchunk + c] = red[0];
}

__global__ void norm_final_kernel(const double* __restrict__ partials, int nchunk, int batch,
                                  double* __restrict__ out, int squared) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    double s = 0.0;
    for (int c = 0; c < nchunk; ++c) s += partials[b * nchunk + c];
    out[b] = squared ? s : sqrt(s);
}

// y = y - v (and y = f - y when f != null): the periodic A = L_ref - V combination
__global__ void combine_kernel(double2* __restrict__ y, const double2* __restrict__ v,
                               const double2* __restrict__ f, size_t total) {
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const double2 a = csub(y[idx], v[idx]);
        y[idx] = f ? csub(f[idx], a) : a;
    }
}

__global__ void init_control_kernel(Control c, int batch) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < batch) {
        c.status[b] = ST_ACTIVE;
        c.sweep[b] = 0;
        c.counter[b] = 0u;
        c.iters[b] = 0;
        c.term[b] = 1;
        c.result_buf[b] = 0;
    }
    if (b == 0) *c.n_active = batch;
}

// any non-finite entry -> *flag = 1 (medium validation on the device: the host loop over a
// c1 / c4 batch costs tens of ms per set_medium)
__global__ void nonfinite_kernel(const double* __restrict__ x, size_t n, int* flag) {
    int bad = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        bad |= !isfinite(x[i]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

__global__ void fill_nan_kernel(double* p, size_t n) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n;
         k += (size_t)gridDim.x * blockDim.x)
        p[k] = __longlong_as_double(0x7ff8000000000000LL);
}

// ------------------------------------------------------------------ launch tables
constexpr int kMinLog2 = 3, kMaxLog2 = 12;

// points per thread of the DST-I engine per size (8 or 16; BP_POINTS_PER_THREAD overrides)
int points_per_thread(int log2n) {
    static int env = [] {
        const char* e = std::getenv("BP_POINTS_PER_THREAD");
        return e ? std::atoi(e) : 0;
    }();
    if (env == 8 || env == 16) return env;
    return 16;
}

#define BS_SIZE_CASES(F, ...)                                                                 \
    switch (log2n) {                                                                          \
        case 3: return F##3(__VA_ARGS__);                                                     \
        case 4: return F##4(__VA_ARGS__);                                                     \
        case 5: return F##5(__VA_ARGS__);                                                     \
        case 6: return F##6(__VA_ARGS__);                                                     \
        case 7: return F##7(__VA_ARGS__);                                                     \
        case 8: return F##8(__VA_ARGS__);                                                     \
        case 9: return F##9(__VA_ARGS__);                                                     \
        case 10: return F##10(__VA_ARGS__);                                                   \
        case 11: return F##11(__VA_ARGS__);                                                   \
        case 12: return F##12(__VA_ARGS__);                                                   \
    }                                                                                         \
    return cudaErrorInvalidValue;

cudaError_t launch_row_pp(int log2n, int pp, int dim, int mode, const RowArgs& a, cudaStream_t s,
                          bool prep = false) {
    BS_SIZE_CASES(launch_row_L, pp, dim, mode, a, s, prep)
}
cudaError_t launch_col_pp(int log2n, int pp, int layout, int mode, const ColArgs& a, cudaStream_t s,
                          bool prep = false) {
    BS_SIZE_CASES(launch_col_L, pp, layout, mode, a, s, prep)
}

cudaError_t launch_periodic(int log2n, bool row, int mode, const PerArgs& a, cudaStream_t s,
                            bool prep = false) {
    BS_SIZE_CASES(launch_periodic_L, row, mode, a, s, prep)
}

cudaError_t launch_cdr(int log2n, bool row, int mode, const CdrArgs& a, cudaStream_t s,
                       bool prep = false) {
    BS_SIZE_CASES(launch_cdr_L, row, mode, a, s, prep)
}

cudaError_t launch_tri(int log2n, int layout, const ColArgs& a, cudaStream_t s, bool prep = false) {
    BS_SIZE_CASES(launch_tri_L, layout, a, s, prep)
}

cudaError_t launch_cluster(int log2n, const ClArgs& a, int batch, cudaStream_t s, bool prep = false) {
    BS_SIZE_CASES(launch_cluster_L, a, batch, s, prep)
}

cudaError_t launch_row(int log2n, int dim, int mode, const RowArgs& a, cudaStream_t s) {
    return launch_row_pp(log2n, points_per_thread(log2n), dim, mode, a, s);
}
cudaError_t launch_col(int log2n, int layout, int mode, const ColArgs& a, cudaStream_t s) {
    return launch_col_pp(log2n, points_per_thread(log2n), layout, mode, a, s);
}

cudaError_t prepare_kernels(int log2n, int dim) {
    RowArgs a{};
    ColArgs c{};
    PerArgs pa{};
    cudaError_t e = cudaSuccess;
    if (log2n >= 6)
        if (cudaError_t r = launch_tri(log2n, dim == 3 ? CL_X3 : CL_PLANE, c, nullptr, true)) e = r;
    if (dim == 2) {
        CdrArgs ca{};
        for (int mode : {RC_FWD, RC_INV, RC_A, RC_B})
            if (cudaError_t r = launch_cdr(log2n, true, mode, ca, nullptr, true)) e = r;
        for (int mode : {CC_ONE, CC_GREEN, CC_INV, CC_LREF})
            if (cudaError_t r = launch_cdr(log2n, false, mode, ca, nullptr, true)) e = r;
        for (int mode : {RP_FWD, RP_FWD_BORN, RP_INV, RP_SWEEP, RP_OPT_B, RP_RETA_B})
            if (cudaError_t r = launch_periodic(log2n, true, mode, pa, nullptr, true)) e = r;
        for (int mode : {CP_ONE, CP_GREEN, CP_LREF, CP_SWEEP, CP_INV, CP_OPT_A, CP_OPT_C, CP_RETA_C})
            if (cudaError_t r = launch_periodic(log2n, false, mode, pa, nullptr, true)) e = r;
    }
    for (int pp : {8, 16}) {
        for (int mode : {R_FWD, R_FWD_BORN, R_INV, R_SWEEP, R_SWEEP_D, R_OPT_A, R_OPT_B, R_RETA_A, R_RETA_C,
                         R_FD_A, R_FD_B})
            if (cudaError_t r = launch_row_pp(log2n, pp, dim, mode, a, nullptr, true)) e = r;
        for (int mode : {C_ONE, C_GREEN, C_LREF, C_FD}) {
            if (cudaError_t r = launch_col_pp(log2n, pp, CL_PLANE, mode, c, nullptr, true)) e = r;
            if (dim == 3)
                if (cudaError_t r = launch_col_pp(log2n, pp, CL_X3, mode, c, nullptr, true)) e = r;
        }
    }
    return e;
}

std::vector<double> lap_table(int n, double h) {
    // (4/h^2) sin^2(j pi / (2n)), the DirichletInterior five-point symbol factor
    // (proj/src/symbol.cpp:69-80, same operation order)
    const double ax = 4.0 / (h * h);
    std::vector<double> lap(n, 0.0);
    for (int j = 1; j < n; ++j) {
        const double sx = std::sin(j * kPi / (2.0 * n));
        lap[j] = ax * sx * sx;
    }
    return lap;
}

// Problem ctor -> check_invertible (proj/src/symbol.cpp:102-111); dim 3: a_p + a_q + a_r
int check_symbol(const bp_grid& g, int dim, int batch, const double* k0, const double* eta) {
    const int n = g.nx + 1;
    std::vector<double> lap = lap_table(n, g.lx / n);
    for (int b = 0; b < batch; ++b) {
        double mn = INFINITY, mx = 0.0;
        const double k0sq = k0[b] * k0[b];
        {
            // |lambda| >= eta everywhere and the largest |lambda| sits at an extreme mode sum:
            // when eta alone clears the guard the scan below cannot fail (the common case)
            const double lo = dim == 3 ? (lap[1] + lap[1]) + lap[1] : lap[1] + lap[1];
            const double hi = dim == 3 ? (lap[n - 1] + lap[n - 1]) + lap[n - 1] : lap[n - 1] + lap[n - 1];
            const double mx0 = std::hypot(std::max(std::fabs(lo - k0sq), std::fabs(hi - k0sq)), eta[b]);
            if (std::fabs(eta[b]) >= kSymbolDivGuard * mx0 * (1.0 + 1e-12)) continue;
        }
        for (int pp = 1; pp < n; ++pp)
            for (int qq = 1; qq < n; ++qq)
                for (int rr = 1; rr < (dim == 3 ? n : 2); ++rr) {
                    const double re = dim == 3 ? (lap[pp] + lap[qq]) + lap[rr] : lap[pp] + lap[qq];
                    const double a = std::hypot(re - k0sq, -eta[b]);
                    mn = std::min(mn, a);
                    mx = std::max(mx, a);
                }
        if (mn < kSymbolDivGuard * mx)
            return set_err(BP_ERUNTIME, "symbol has a (near-)zero entry; reference operator not invertible");
    }
    return BP_OK;
}

int grid_for(size_t n) { return (int)std::min<size_t>((n + 255) / 256, 148 * 16); }

}  // namespace

// Line-transform plan of the any-shape path (generic_kernels.cuh): DFT length n, FFT length L
// (n itself when a power of two, else the Bluestein convolution length), device tables.
struct GLinePlan {
    int n = 0, L = 0, lg = 0;
    double2 *chirp = nullptr, *filt = nullptr, *tw = nullptr;
};

// ------------------------------------------------------------------ handle
struct bp_problem {
    bp_grid grid{};
    int batch = 0, device = 0, log2n = 0, n = 0, dim = 2;
    bool periodic = false;   // the reference's own HelmholtzProblem (FFT basis, no padding)
    bool cdr = false;        // config c4: real fields, Neumann, DCT-II, upwind V
    double *bx = nullptr, *by = nullptr, *sigma = nullptr, *sigma0 = nullptr, *lapn = nullptr,
           *rnorm2 = nullptr;
    double2* w4 = nullptr;
    // slab decomposition (one rank's x-slab of a distributed 2-D grid, batch 1)
    int slab_log2 = 0, slab_rank = 0, slab_nranks = 1, row0 = 0;
    double2 *u_alloc0 = nullptr, *u_alloc1 = nullptr;  // u with one halo row each side
    double2* Tc = nullptr;                              // column-side block
    double* slab_sums = nullptr;
    bool slab_fd = false;  // bp_slab_set_multiplier uploaded the rank's FourierDiag block into fd
    bool slab_direct = false;  // IterFormat::Direct for the slab run in progress (BP_SLAB_INIT)
    bool slab_running = false;
    // fused exchange (bp_slab_set_exchange)
    bool xchg_on = false;
    double2* xchg_cols[kMaxXchg]{};  // peers' t_cols (receive side of the forward exchange)
    double2* xchg_rows[kMaxXchg]{};  // peers' t_rows (receive side of the inverse exchange)
    double2 *own_T = nullptr, *own_Tc = nullptr;  // the handle's allocations (freed on destroy)
    int slab_max_iters = 1000;
    double slab_rtol = 1e-6;
    bool own_stream = true;
    double* xi2 = nullptr;   // periodic: xi_j^2, FFT order
    size_t field = 0;   // padded elements per member (n^dim)
    size_t alloc = 0;   // padded elements per buffer (batch*n^dim + n^(dim-1): zero halo)
    size_t dense_pts = 0;  // reference-layout points per member ((n-1)^dim)
    double inv_h2 = 0, green_scale = 0;
    // Green column pass as a tridiagonal x-solve (tri_kernels.cuh): pivot tables per
    // (member, line), rebuilt whenever k0 / eta change; null = transform route
    double2* tri = nullptr;
    double tri_scale = 0;
    // any-shape 2-D Dirichlet handle (nx, ny not of the form 2^k - 1, or nx != ny): dense nx x ny
    // layout, line transforms by radix-2 / Bluestein (generic_kernels.cuh)
    bool generic = false;
    bool gper = false;   // any-shape periodic family (DFT lines, |xi|^2 symbol)
    int gnx = 0, gny = 0;
    GLinePlan gplan_x, gplan_y;
    double *gax = nullptr, *gay = nullptr, *gpart = nullptr;
    double2 *gm0 = nullptr, *gm1 = nullptr, *gm2 = nullptr;  // any-shape staged maps: u^m, direction, w
    cudaStream_t stream = nullptr;
    // device constants
    double2* k2 = nullptr;
    double* k0sq = nullptr;
    double* eta = nullptr;
    double2* tw = nullptr;
    double* sinp = nullptr;
    double* lap = nullptr;
    // workspace
    double2 *f = nullptr, *u0 = nullptr, *u1 = nullptr, *T = nullptr, *x = nullptr, *y = nullptr;
    double2* dense = nullptr;  // batch * nx*ny staging
    double* partial = nullptr;
    double2* gamma = nullptr;
    double2* fd = nullptr;  // FourierDiag multiplier (padded n x n), uploaded per run
    double* norm_part = nullptr;
    double *fnorm_l2 = nullptr, *fnorm_reta = nullptr;
    int* ctl_int = nullptr;  // status, sweep, iters, term, result_buf, n_active
    unsigned* counter = nullptr;
    double *trace_l2 = nullptr, *trace_reta = nullptr;
    int trace_cap = 0;
    int* host_active = nullptr;  // pinned (written by the device: publish_int)
    double* host_fn = nullptr;   // pinned [batch]: ||f|| for the zero-source check
    int* dflag = nullptr;        // device flag of nonfinite_kernel
    // graph cache
    cudaGraphExec_t graph = nullptr;
    // small batches (< kSplitWaves row waves): the batch as two halves, each its own graph on its
    // own stream, so one half's column pass fills the other half's row-launch tail
    static constexpr int kMaxSplit = 16;
    cudaGraphExec_t graph2[kMaxSplit - 1]{};  // parts 1.. (part 0 is `graph` on `stream`)
    std::vector<cudaGraphExec_t> gwave;       // waves 1..: [wave - 1][part] (wave 0 = graph / graph2)
    int graph_group = 0;                      // members per wave the graphs were captured for
    cudaStream_t stream2[kMaxSplit - 1]{};
    cudaEvent_t ev_join[kMaxSplit]{};
    int graph_split = -1;
    int graph_map_kind = -1;
    int graph_metric = -1;
    int graph_format = -1;
    double2 graph_gamma{};
    int graph_max_iters = -1;
    double graph_rtol = -1;
    // compute hooks (bp_internal_set_compute_hooks; the pipeline's FIFO compute turn): called
    // around the sweeps of a run, after its uploads were enqueued and before its downloads
    void (*hook_pre)(void*) = nullptr;
    void (*hook_post)(void*) = nullptr;
    void* hook_ctx = nullptr;
    // instrumentation
    bool timing = false;
    int64_t stat_launches = 0, stat_sweeps = 0, stat_timed = 0;
    double stat_row_ms = 0, stat_col_ms = 0;
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

Control make_control(const bp_problem* p) {
    Control c{};
    int* ci = p->ctl_int;
    const int B = p->batch;
    c.status = ci;
    c.sweep = ci + B;
    c.iters = ci + 2 * B;
    c.term = ci + 3 * B;
    c.result_buf = ci + 4 * B;
    c.n_active = ci + 5 * B;
    c.counter = p->counter;
    c.partial = p->partial;
    c.gamma = p->gamma;
    c.fnorm_l2 = p->fnorm_l2;
    c.fnorm_reta = p->fnorm_reta;
    c.trace_l2 = p->trace_l2;
    c.trace_reta = p->trace_reta;
    c.trace_stride = p->trace_cap;
    return c;
}

RowArgs row_args(const bp_problem* p) {
    RowArgs a{};
    // L2 hints: single-member handles and 3-D always; multi-member 2-D batches only in the waves'
    // single-member launches (run_core sets them there)
    a.l2_hints = (p->batch == 1 || p->dim == 3) ? BS_L2_HINTS : 0;
    a.batch = p->batch;
    a.inv_h2 = p->inv_h2;
    a.k0sq = p->k0sq;
    a.eta = p->eta;
    a.k2 = p->k2;
    a.f = p->f;
    a.T = p->T;
    a.u0 = p->u0;
    a.u1 = p->u1;
    a.X = p->x;
    a.tw = p->tw;
    a.sinp = p->sinp;
    a.map_kind = MK_SCALAR;
    a.gamma = make_double2(1.0, 0.0);
    a.ctl = make_control(p);
    return a;
}

ColArgs col_args(const bp_problem* p) {
    ColArgs c{};
    c.l2_hints = (p->batch == 1 || p->dim == 3) ? BS_L2_HINTS : 0;
    c.batch = p->batch;
    c.k0sq = p->k0sq;
    c.eta = p->eta;
    c.lap = p->lap;
    c.scale = p->green_scale;
    c.fd = p->fd;
    c.tri = p->tri;
    c.tri_scale = p->tri_scale;

    c.T = p->T;
    c.tw = p->tw;
    c.sinp = p->sinp;
    c.status = nullptr;
    return c;
}

// Arguments restricted to members [b0, b0 + nb) of the batch (the split-batch graphs): every
// per-member array is offset, n_active stays shared.
Control control_range(Control c, const bp_problem* p, int b0) {
    c.status += b0;
    c.sweep += b0;
    c.iters += b0;
    c.term += b0;
    c.result_buf += b0;
    c.counter += b0;
    c.partial += ((size_t)b0 << (p->log2n * (p->dim - 1))) * kPartStride;
    c.gamma += b0;
    c.fnorm_l2 += b0;
    c.fnorm_reta += b0;
    c.trace_l2 += (size_t)b0 * c.trace_stride;
    c.trace_reta += (size_t)b0 * c.trace_stride;
    return c;
}

RowArgs row_args_range(const RowArgs& a0, const bp_problem* p, int b0, int nb) {
    RowArgs a = a0;
    const size_t fo = (size_t)b0 * p->field;
    a.batch = nb;
    a.k0sq += b0;
    a.eta += b0;
    a.k2 += fo;
    a.f += fo;
    a.T += fo;
    a.u0 += fo;
    a.u1 += fo;
    if (a.X) a.X += fo;
    a.ctl = control_range(a.ctl, p, b0);
    return a;
}

ColArgs col_args_range(const ColArgs& c0, const bp_problem* p, int b0, int nb) {
    ColArgs c = c0;
    c.batch = nb;
    c.k0sq += b0;
    c.eta += b0;
    c.T += (size_t)b0 * p->field;
    if (c.status) c.status += b0;
    if (c.tri) c.tri += (size_t)b0 * ((size_t)1 << ((p->dim - 1) * p->log2n)) * (kTriP + p->n / kTriP);
    if (c.finalize) c.ctl = control_range(c.ctl, p, b0);
    return c;
}

int check_problem(const bp_problem* p) {
    if (!p) return set_err(BP_EINVAL, "null problem handle");
    return BP_OK;
}

int upload(bp_problem* p, const double* host, double2* dst, bool host_ptr = true);

// Small device -> host reads on the run's critical path (the poll of n_active after every graph
// replay, ||f|| for the zero-source check) go through zero-copy stores into pinned host memory
// instead of cudaMemcpyAsync: a 4-byte D2H copy queues on the copy engine BEHIND another handle's
// result download (bs.Pipeline: the previous job's 267 MB of u on c1), which stalled the start of
// every compute turn by that copy's ~4.6 ms (r02h: e2e 32.5 -> see DESIGN 5).
__global__ void publish_int_kernel(const int* __restrict__ src, volatile int* dst) {
    *dst = *src;
    __threadfence_system();
}
__global__ void publish_doubles_kernel(const double* __restrict__ src, volatile double* dst, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
    __threadfence_system();
}
cudaError_t publish_int(bp_problem* p, const int* dev) {
    publish_int_kernel<<<1, 1, 0, p->stream>>>(dev, p->host_active);
    return cudaGetLastError();
}
// ||f|| per member -> host (synchronises the stream)
int read_fnorm(bp_problem* p, std::vector<double>& fn) {
    if (!p->host_fn) CU(cudaMallocHost(&p->host_fn, sizeof(double) * p->batch));
    publish_doubles_kernel<<<1, 128, 0, p->stream>>>(p->fnorm_l2, p->host_fn, p->batch);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(p->stream));
    for (int b = 0; b < p->batch; ++b) fn[b] = p->host_fn[b];
    return BP_OK;
}

// true when the n doubles at dev (device memory) are all finite; synchronises the stream
int all_finite(bp_problem* p, const double* dev, size_t n, bool* ok) {
    CU(cudaMemsetAsync(p->dflag, 0, sizeof(int), p->stream));
    nonfinite_kernel<<<grid_for(n), 256, 0, p->stream>>>(dev, n, p->dflag);
    CU(cudaGetLastError());
    CU(publish_int(p, p->dflag));
    CU(cudaStreamSynchronize(p->stream));
    *ok = *p->host_active == 0;
    return BP_OK;
}

// dense host k2 -> validated (finite) -> padded device k2 (HelmholtzProblem ctor's check,
// helmholtz.cpp:18-20, done on the staged copy)
int upload_k2_checked(bp_problem* p, const double* host) {
    const size_t nd = p->dense_pts;
    CU(cudaMemcpyAsync(p->dense, host, sizeof(double2) * nd * p->batch, cudaMemcpyHostToDevice, p->stream));
    bool ok = false;
    if (int rc = all_finite(p, reinterpret_cast<const double*>(p->dense), 2 * nd * p->batch, &ok)) return rc;
    if (!ok) return set_err(BP_EINVAL, "HelmholtzProblem: k2 not finite");
    return upload(p, reinterpret_cast<const double*>(p->dense), p->k2, false);
}

// dense host -> padded device
int upload(bp_problem* p, const double* host, double2* dst, bool host_ptr) {
    const size_t nd = p->dense_pts;
    const size_t bytes = sizeof(double2) * nd * p->batch;
    const double2* src = reinterpret_cast<const double2*>(host);
    if (host_ptr) {
        CU(cudaMemcpyAsync(p->dense, host, bytes, cudaMemcpyHostToDevice, p->stream));
        src = p->dense;
    }
    if (p->periodic || p->generic) {  // no padding: the dense layout is the device layout
        CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, p->stream));
        return BP_OK;
    }
    pack_kernel<<<grid_for(p->field * p->batch), 256, 0, p->stream>>>(src, dst, p->batch, p->log2n,
                                                                       p->dim);
    CU(cudaGetLastError());
    return BP_OK;
}

int download(bp_problem* p, const double2* p0, const double2* p1, const int* select, double* host,
             bool host_ptr = true) {
    const size_t nd = p->dense_pts;
    double2* dst = host_ptr ? p->dense : reinterpret_cast<double2*>(host);
    if (p->periodic) {  // select must be null: the periodic result is produced into p0
        CU(cudaMemcpyAsync(dst, p0, sizeof(double2) * nd * p->batch, cudaMemcpyDeviceToDevice, p->stream));
    } else if (p->generic) {
        gen_select_kernel<<<grid_for(nd * p->batch), 256, 0, p->stream>>>(p0, p1 ? p1 : p0, select, dst,
                                                                          (long)nd, p->batch);
    } else {
        unpack_kernel<<<grid_for(nd * p->batch), 256, 0, p->stream>>>(p0, p1, select, dst, p->batch,
                                                                       p->log2n, p->dim);
    }
    CU(cudaGetLastError());
    if (host_ptr)
        CU(cudaMemcpyAsync(host, p->dense, sizeof(double2) * nd * p->batch, cudaMemcpyDeviceToHost,
                           p->stream));
    return BP_OK;
}

int norms(bp_problem* p, const double2* x, double* out, bool squared = false) {
    const int nchunk = 64;
    dim3 g(nchunk, p->batch);
    // real (CDR) fields are read as pairs: |re|^2 + |im|^2 over half as many double2
    const size_t per = p->cdr ? p->field / 2 : p->field;
    norm_partial_kernel<<<g, 256, 0, p->stream>>>(x, per, nchunk, p->norm_part);
    norm_final_kernel<<<(p->batch + 127) / 128, 128, 0, p->stream>>>(p->norm_part, nchunk,
                                                                      p->batch, out, squared);
    CU(cudaGetLastError());
    return BP_OK;
}

// The transverse part of a transform pair after the row (y / z) pass: in 2-D one column
// kernel (x-lines); in 3-D the y-lines of every x-plane, the x-lines (where the spectral
// multiply happens), and the y-lines again.  mode C_ONE = forward transform only (API).
// Returns the number of kernels launched (negative on error).
int col_stage(bp_problem* p, const ColArgs& c0, int mode, double scale) {
    ColArgs c = c0;
    if (p->dim == 2) {
        c.planes_per_member = 1;
        c.scale = scale;
        if (mode == C_GREEN && p->tri && scale == p->green_scale)
            return launch_tri(p->log2n, CL_PLANE, c, p->stream) == cudaSuccess ? 1 : -1;
        return launch_col(p->log2n, CL_PLANE, mode, c, p->stream) == cudaSuccess ? 1 : -1;
    }
    c.planes_per_member = p->n;
    c.scale = 1.0;
    if (launch_col(p->log2n, CL_PLANE, C_ONE, c, p->stream) != cudaSuccess) return -1;
    c.finalize = 0;  // deferred finalisation (3-D) belongs to the first launch only
    c.scale = scale;
    if (mode == C_GREEN && p->tri && scale == p->green_scale) {
        if (launch_tri(p->log2n, CL_X3, c, p->stream) != cudaSuccess) return -1;
    } else if (launch_col(p->log2n, CL_X3, mode, c, p->stream) != cudaSuccess) {
        return -1;
    }
    if (mode == C_ONE) return 2;
    c.scale = 1.0;
    c.planes_per_member = p->n;
    if (launch_col(p->log2n, CL_PLANE, C_ONE, c, p->stream) != cudaSuccess) return -1;
    return 3;
}

int col_stage_checked(bp_problem* p, const ColArgs& c, int mode, double scale) {
    if (col_stage(p, c, mode, scale) < 0)
        return set_err(BP_ECUDA, std::string("column stage launch: ") + cudaGetErrorString(cudaGetLastError()));
    return BP_OK;
}

// Green operator on padded `in` -> padded `out` (out - sub when sub != null)
int green(bp_problem* p, const double2* in, double2* out, const double2* sub, bool born) {
    RowArgs a = row_args(p);
    a.in = in;
    CU(launch_row(p->log2n, p->dim, born ? R_FWD_BORN : R_FWD, a, p->stream));
    ColArgs c = col_args(p);
    if (int rc = col_stage_checked(p, c, C_GREEN, p->green_scale)) return rc;
    a.out = out;
    a.sub = sub;
    CU(launch_row(p->log2n, p->dim, R_INV, a, p->stream));
    return BP_OK;
}

// (Re)build the tridiagonal pivot tables from the device k0^2 / eta (stream-ordered after
// their upload)
int build_tri(bp_problem* p) {
    if (!p->tri) return BP_OK;
    const double h = p->grid.lx / p->n;
    if (p->cdr) {
        const long cols = (long)p->batch << p->log2n;
        tri_setup_neumann_kernel<<<(int)((cols + 127) / 128), 128, 0, p->stream>>>(p->lapn, p->sigma0, h * h,
                                                                                 p->batch, p->log2n, p->tri);
        CU(cudaGetLastError());
        return BP_OK;
    }
    const long lines = (long)p->batch << ((p->dim - 1) * p->log2n);
    tri_setup_kernel<<<(int)((lines + 127) / 128), 128, 0, p->stream>>>(p->lap, p->k0sq, p->eta, h * h, p->batch,
                                                                       p->log2n, p->dim, p->tri);
    CU(cudaGetLastError());
    return BP_OK;
}

// ------------------------------------------------------------------ any-shape path (host)
// In-place iterative radix-2 FFT on the host (plan setup only: the Bluestein filter spectrum).
void host_fft(std::vector<std::complex<double>>& a) {
    const size_t L = a.size();
    for (size_t i = 1, j = 0; i < L; ++i) {
        size_t bit = L >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i], a[j]);
    }
    for (size_t len = 2; len <= L; len <<= 1) {
        for (size_t i = 0; i < L; i += len)
            for (size_t k = 0; k < len / 2; ++k) {
                const std::complex<double> w = std::polar(1.0, -2.0 * kPi * (double)k / (double)len);
                const std::complex<double> u = a[i + k], v = a[i + k + len / 2] * w;
                a[i + k] = u + v;
                a[i + k + len / 2] = u - v;
            }
    }
}

int make_gplan(int n, GLinePlan& pl) {
    pl.n = n;
    int L = 1;
    const bool pow2 = (n & (n - 1)) == 0;
    while (L < (pow2 ? n : 2 * n - 1)) L <<= 1;
    if (L > 8192) return set_err(BP_ENOTSUP, "any-shape path: line transforms up to 4096 points");
    pl.L = L;
    pl.lg = 0;
    while ((1 << pl.lg) < L) ++pl.lg;
    std::vector<double2> tw(std::max(1, L / 2));
    for (int k = 0; k < L / 2; ++k) tw[k] = make_double2(std::cos(2.0 * kPi * k / L), -std::sin(2.0 * kPi * k / L));
    CU(cudaMalloc(&pl.tw, sizeof(double2) * tw.size()));
    CU(cudaMemcpy(pl.tw, tw.data(), sizeof(double2) * tw.size(), cudaMemcpyHostToDevice));
    if (L != n) {
        // c_j = exp(-i pi j^2 / n), the exponent reduced mod 2n in integers (exact angles)
        std::vector<double2> ch(n);
        std::vector<std::complex<double>> b(L, 0.0);
        for (int j = 0; j < n; ++j) {
            const double ang = kPi * (double)(((long long)j * j) % (2LL * n)) / n;
            ch[j] = make_double2(std::cos(ang), -std::sin(ang));
            b[j] = std::complex<double>(std::cos(ang), std::sin(ang));  // b_j = conj(c_j)
            if (j) b[L - j] = b[j];
        }
        host_fft(b);
        std::vector<double2> fl(L);
        for (int k = 0; k < L; ++k) fl[k] = make_double2(b[k].real(), b[k].imag());
        CU(cudaMalloc(&pl.chirp, sizeof(double2) * n));
        CU(cudaMalloc(&pl.filt, sizeof(double2) * L));
        CU(cudaMemcpy(pl.chirp, ch.data(), sizeof(double2) * n, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(pl.filt, fl.data(), sizeof(double2) * L, cudaMemcpyHostToDevice));
    }
    return BP_OK;
}

void free_gplan(GLinePlan& pl) {
    for (double2* q : {pl.chirp, pl.filt, pl.tw})
        if (q) cudaFree(q);
    pl = GLinePlan{};
}

GenArgs gen_args(const bp_problem* p) {
    GenArgs g{};
    g.batch = p->batch;
    g.nx = p->gnx;
    g.ny = p->gny;
    g.inv_h2 = p->inv_h2;
    g.k2 = p->k2;
    g.k0sq = p->k0sq;
    g.eta = p->eta;
    g.ax = p->gax;
    g.ay = p->gay;
    // inverse normalisation: DST-I 4/((nx+1)(ny+1)); DFT 1/(nx ny) (transforms.cpp:96-103)
    g.gscale = p->gper ? 1.0 / ((double)p->gnx * p->gny) : 4.0 / ((double)(p->gnx + 1) * (p->gny + 1));
    return g;
}

// line transform of every y-line (axis 0) or x-line (axis 1) of the dense batch: DST-I
// (Dirichlet handles) or the unnormalised forward / backward DFT (periodic handles, inverse)
int gen_lines(bp_problem* p, int axis, const double2* in, double2* out, double scale, bool inverse = false,
              const int* status = nullptr) {
    const GLinePlan& pl = axis == 0 ? p->gplan_y : p->gplan_x;
    GLineArgs a{};
    a.in = in;
    a.out = out;
    a.n = pl.n;
    a.L = pl.L;
    a.lgL = pl.lg;
    const long per = (long)p->gnx * p->gny;
    if (axis == 0) {
        a.lines = (long)p->batch * p->gnx;
        a.lpm = p->gnx;
        a.lstride = p->gny;
        a.estride = 1;
    } else {
        a.lines = (long)p->batch * p->gny;
        a.lpm = p->gny;
        a.lstride = 1;
        a.estride = p->gny;
    }
    a.mstride = per;
    a.chirp = pl.chirp;
    a.filt = pl.filt;
    a.tw = pl.tw;
    a.scale = scale;
    a.status = status;
    const int smem = (int)(sizeof(double2) * (pl.n + std::max(pl.L, pl.n / 2 + 256)));
    static bool attr = [] {
        for (auto k : {gline_kernel<GL_DST>, gline_kernel<GL_DFT>, gline_kernel<GL_IDFT>})
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        return true;
    }();
    (void)attr;
    if (!p->gper) gline_kernel<GL_DST><<<(unsigned)a.lines, 256, smem, p->stream>>>(a);
    else if (inverse) gline_kernel<GL_IDFT><<<(unsigned)a.lines, 256, smem, p->stream>>>(a);
    else gline_kernel<GL_DFT><<<(unsigned)a.lines, 256, smem, p->stream>>>(a);
    CU(cudaGetLastError());
    return BP_OK;
}

// 2-D DST-I (plain sine sums, transforms.hpp:18-20) of a dense batch, x scale; periodic handles:
// the unnormalised 2-D DFT (inverse: backward DFT), x scale
int gen_dst2(bp_problem* p, const double2* in, double2* out, double scale, bool inverse = false,
             const int* status = nullptr) {
    if (int rc = gen_lines(p, 0, in, out, 1.0, inverse, status)) return rc;
    return gen_lines(p, 1, out, out, scale, inverse, status);
}

// G (divide) / L_ref (multiply): S^-1 diag(lambda^-+1) S with S^-1 = 4/((nx+1)(ny+1)) S
// (periodic: F^-1 diag(.) F with F^-1 = backward DFT / (nx ny); mode 2 = |xi|^2 only, A's part)
int gen_spectral(bp_problem* p, bool divide, const double2* in, double2* out, int mode = -1) {
    const GenArgs g = gen_args(p);
    if (int rc = gen_dst2(p, in, p->T, 1.0)) return rc;
    gen_symbol_kernel<<<grid_for(p->field * p->batch), 256, 0, p->stream>>>(g, mode >= 0 ? mode : (divide ? 1 : 0),
                                                                             p->gper ? 1.0 : g.gscale, p->T);
    CU(cudaGetLastError());
    return gen_dst2(p, p->T, out, p->gper ? g.gscale : 1.0, p->gper);
}

// Problem ctor guard (symbol.cpp:102-111) over the any-shape symbol
int check_symbol_generic(const std::vector<double>& ax, const std::vector<double>& ay, int batch,
                         const double* k0, const double* eta) {
    for (int b = 0; b < batch; ++b) {
        const double k0sq = k0[b] * k0[b];
        double mn = INFINITY, mx = 0.0;
        for (double a : ax)
            for (double c : ay) {
                const double v = std::hypot((a + c) - k0sq, -eta[b]);
                mn = std::min(mn, v);
                mx = std::max(mx, v);
            }
        if (mn < kSymbolDivGuard * mx)
            return set_err(BP_ERUNTIME, "symbol has a (near-)zero entry; reference operator not invertible");
    }
    return BP_OK;
}

std::vector<double> gen_lap(int n, double h) {  // (4/h^2) sin^2((p+1) pi / (2(n+1))), p < n
    std::vector<double> a(n);
    for (int p2 = 0; p2 < n; ++p2) {
        const double sx = std::sin((p2 + 1) * kPi / (2.0 * (n + 1)));
        a[p2] = 4.0 / (h * h) * sx * sx;
    }
    return a;
}

int ensure_trace(bp_problem* p, int max_iters) {
    if (p->trace_cap >= max_iters + 1) return BP_OK;
    cudaFree(p->trace_l2);
    cudaFree(p->trace_reta);
    p->trace_l2 = p->trace_reta = nullptr;
    const size_t n = (size_t)p->batch * (max_iters + 1);
    CU(cudaMalloc(&p->trace_l2, sizeof(double) * n));
    CU(cudaMalloc(&p->trace_reta, sizeof(double) * n));
    p->trace_cap = max_iters + 1;
    if (p->graph) {
        cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
        for (auto& g2 : p->graph2) {
            if (g2) cudaGraphExecDestroy(g2);
            g2 = nullptr;
        }
        for (auto gw : p->gwave)
            if (gw) cudaGraphExecDestroy(gw);
        p->gwave.clear();
    }
    return BP_OK;
}

// Launch sequence of one sweep per correction map (see RowMode in sweep_kernels.cuh).
struct SweepPlan {
    int n = 0;
    bool row[5]{};
    int mode[5]{};
    void add(bool r, int md) {
        row[n] = r;
        mode[n++] = md;
    }
};

SweepPlan plan_for(const bp_map* map, int format) {
    SweepPlan s;
    switch (map->kind) {
        case BP_MAP_OPTIMAL_SCALAR:
            if (map->metric != BP_METRIC_RETA && format == BP_FMT_DIRECT) {
                // Direct + Euclidean: w = A r = L_ref r - V r (R_FD_A stores r, C_LREF, R_RETA_C)
                s.add(true, R_FD_A);
                s.add(false, C_LREF);
                s.add(true, R_RETA_C);
            } else if (map->metric == BP_METRIC_RETA) {
                s.add(true, R_RETA_A);
                s.add(false, C_GREEN);
                s.add(true, R_RETA_C);
            } else {
                s.add(true, R_OPT_A);
            }
            s.add(true, R_OPT_B);
            s.add(false, C_GREEN);
            break;
        case BP_MAP_FOURIER_DIAG:
            s.add(true, R_FD_A);
            s.add(false, C_FD);
            s.add(true, R_FD_B);
            s.add(false, C_GREEN);
            break;
        default:  // scalar gamma or pointwise gamma(x): one fused row pass
            s.add(true, format == BP_FMT_DIRECT ? R_SWEEP_D : R_SWEEP);
            s.add(false, C_GREEN);
    }
    return s;
}

// kernels one sweep launches (a column stage is 3 kernels in 3-D)
int plan_kernels(const bp_problem* p, const SweepPlan& plan) {
    int k = 0;
    for (int s = 0; s < plan.n; ++s) k += plan.row[s] ? 1 : (p->dim == 3 ? 3 : 1);
    return k;
}

// ev (optional): plan.n + 1 events recorded around the stages
int sweep_once(bp_problem* p, const SweepPlan& plan, const RowArgs& a, const ColArgs& c,
               cudaEvent_t* ev) {
    if (ev) CU(cudaEventRecord(ev[0], p->stream));
    for (int k = 0; k < plan.n; ++k) {
        const int md = plan.mode[k];
        if (plan.row[k]) {
            CU(launch_row(p->log2n, p->dim, md, a, p->stream));
        } else if (int rc = col_stage_checked(p, c, md, p->green_scale)) {
            return rc;
        }
        if (ev) CU(cudaEventRecord(ev[k + 1], p->stream));
    }
    return BP_OK;
}

// Split the batch into two concurrently replayed halves: one half's column pass runs under the
// other half's row-launch tail (and vice versa) instead of every launch boundary draining the
// GPU.  Measured on c1: 8 members 30.0 -> 34.9 Gpts/s (the row launch is 1.73 waves deep), 32
// members 34.9 -> 35.7, 64 members 34.6 -> 35.1.  The two-launch scalar / pointwise plan only
// (its per-half finalisation is self-contained); BP_SPLIT=0 disables.  Returns the first half's
// size or 0.  BP_SPLIT=K (3, 4): K parts.
constexpr int kDefaultGroup = 8;  // members per wave at n = 512 (group_members)
constexpr double kSplitWaves = 1e30;  // every depth (BP_SPLIT=2 kept as the explicit spelling)
// parts: 4 for shallow batches (c1 at 8 members: 34.8 -> 36.4 Gpts/s with 4 vs 2 parts), 2 above
// 16 members (64 members: 35.1 with 2, 35.0 with 3 or 4); BP_SPLIT=K overrides
int split_parts(int batch, int log2n) {
    const char* env = std::getenv("BP_SPLIT");
    // n = 512, up to 8 members (BASELINE c1 at 8 per GPU): one member per part, 36.4 -> 38.0 Gpts/s
    const int k = env ? std::atoi(env) : (log2n == 9 && batch <= 8 ? batch : (batch <= 16 ? 4 : 2));
    return std::max(2, std::min(k, (int)bp_problem::kMaxSplit));
}
// parts per wave when the batch is swept in waves: one member per part (BP_SPLIT overrides)
int wave_parts(int group) {
    const char* env = std::getenv("BP_SPLIT");
    const int k = env ? std::atoi(env) : group;
    return std::max(2, std::min(std::min(k, group), (int)bp_problem::kMaxSplit));
}
// Members per wave (0 = the whole batch at once).  Measured on c1 (64 x 511^2, r02h): waves of 8
// members, each member its own part on its own stream, 35.0 -> 37.2 Gpts/s (waves of 6 / 7 / 9 /
// 10 / 12 / 16: 36.4 / 36.6 / 35.5 / 35.7 / 34.9 / 34.6; 8 members in 4 parts 36.0; no waves
// with 8 / 16 parts 34.4 / 34.6): a wave's ~160 MB of fields is swept kGraphSweeps times while
// much of it is still in the 126 MB L2, and eight single-member graphs interleave their row and
// column launches finely.  Default: n = 512 only (the measured size); BP_GROUP=G overrides
// for any size, BP_GROUP=0 disables.
int group_members(const bp_problem* p, int batch) {
    const char* env = std::getenv("BP_GROUP");
    const int g = env ? std::atoi(env) : (p->log2n == 9 && !p->cdr ? kDefaultGroup : 0);
    return (g > 0 && g < batch) ? g : 0;
}
int split_batch(const bp_problem* p, const SweepPlan& plan) {
    const char* env = std::getenv("BP_SPLIT");  // read per run (tests toggle it)
    const bool env_off = env && env[0] == '0';
    if (env_off || p->batch < 2 || p->dim != 2 || p->periodic || p->cdr || p->generic || p->slab_log2) return 0;
    if (!(plan.n == 2 && plan.row[0] && (plan.mode[0] == R_SWEEP || plan.mode[0] == R_SWEEP_D))) return 0;
    static int sms = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 148;
    }();
    const double row_ctas = (double)((long)p->batch << p->log2n) / row_lines_per_cta(p->log2n, points_per_thread(p->log2n));
    const bool force = env && env[0] == '2';  // BP_SPLIT=2: split at any depth (experiments)
    if (!force && row_ctas / (2.0 * sms) >= kSplitWaves) return 0;
    return p->batch / 2;
}

// whole-solve cluster kernel applies: 2-D Dirichlet n = 64 / 128 with the tridiagonal tables,
// the fused scalar / pointwise sweep, and a device that runs the cluster shape
bool cluster_enabled(const bp_problem* p, const SweepPlan& plan) {
    const char* env = std::getenv("BP_CLUSTER");  // read per run (tests toggle it)
    const bool env_off = env && env[0] == '0';
    if (env_off || p->dim != 2 || p->periodic || p->cdr || p->generic || p->slab_log2 || !p->tri) return false;
    if (p->log2n != 6 && p->log2n != 7) return false;
    if (!(plan.n == 2 && plan.row[0] && (plan.mode[0] == R_SWEEP || plan.mode[0] == R_SWEEP_D))) return false;
    static int ok[2] = {-1, -1};  // per size: the cluster shape launches on this device
    int& k = ok[p->log2n - 6];
    if (k < 0) k = launch_cluster(p->log2n, ClArgs{}, 1, nullptr, true) == cudaSuccess ? 1 : 0;
    return k == 1;
}

// The driver: bp::run over the batch.  f_dev/u0_dev padded device fields already staged.
int run_core(bp_problem* p, const bp_map* map, const bp_iter_config* cfg, bool have_u0,
             double* snapshots, int n_snap) {
    const int B = p->batch;
    RowArgs a = row_args(p);
    a.ctl.max_iters = cfg->max_iters;
    a.ctl.rtol = cfg->rtol;
    a.map_kind = map->kind;
    a.gamma = make_double2(map->gamma_re, map->gamma_im);
    a.direct = cfg->format == BP_FMT_DIRECT;
    a.lw = a.direct && map->kind == BP_MAP_OPTIMAL_SCALAR && map->metric != BP_METRIC_RETA;
    ColArgs c = col_args(p);
    c.status = a.ctl.status;
    const SweepPlan plan = plan_for(map, cfg->format);
    if (map->kind == BP_MAP_FOURIER_DIAG) {
        // one multiplier for the whole batch, reference mode layout -> padded
        const size_t bytes = sizeof(double2) * p->dense_pts;
        CU(cudaMemcpyAsync(p->dense, map->m, bytes, cudaMemcpyHostToDevice, p->stream));
        pack_kernel<<<grid_for(p->field), 256, 0, p->stream>>>(p->dense, p->fd, 1, p->log2n, p->dim);
        CU(cudaGetLastError());
    }

    // fnorm_l2 = ||f||, fnorm_reta = ||G f||  (iterate.cpp:93,102)
    int rc = norms(p, p->f, p->fnorm_l2);
    if (rc) return rc;
    rc = green(p, p->f, p->y, nullptr, false);
    if (rc) return rc;
    rc = norms(p, p->y, p->fnorm_reta);
    if (rc) return rc;
    std::vector<double> fn(B);
    if (int rc = read_fnorm(p, fn)) return rc;
    for (int b = 0; b < B; ++b)
        if (!(fn[b] > 0.0)) return set_err(BP_EINVAL, "run: zero source");

    if (!have_u0) CU(cudaMemsetAsync(p->u0, 0, sizeof(double2) * p->alloc, p->stream));
    CU(cudaMemsetAsync(p->u1, 0, sizeof(double2) * p->alloc, p->stream));
    init_control_kernel<<<(B + 127) / 128, 128, 0, p->stream>>>(a.ctl, B);
    fill_nan_kernel<<<grid_for((size_t)B * p->trace_cap), 256, 0, p->stream>>>(p->trace_l2, (size_t)B * p->trace_cap);
    fill_nan_kernel<<<grid_for((size_t)B * p->trace_cap), 256, 0, p->stream>>>(p->trace_reta, (size_t)B * p->trace_cap);
    CU(cudaGetLastError());

    // q^0 = V u^0 + f -> forward y-DST -> T ; column pass
    a.in = p->u0;
    CU(launch_row(p->log2n, p->dim, R_FWD_BORN, a, p->stream));
    if (int rc2 = col_stage_checked(p, c, C_GREEN, p->green_scale)) return rc2;
    // scalar / pointwise 2-D sweeps: the column pass finalises the entry the row pass before
    // it reduced (RowArgs::defer_final / ColArgs::finalize); not for the initial column pass
    // (n >= 64: the column CTA has at least one full warp for finalize_member's shuffles)
    // 3-D: the first (y-line) launch of the column stage finalises, the whole CTA summing the
    // n^2 line partials (finalize_member3; col_stage clears the flag for the other two)
    if ((p->dim == 2 || p->dim == 3) && p->log2n >= 6 && plan.n == 2 &&
        plan.row[0] && (plan.mode[0] == R_SWEEP || plan.mode[0] == R_SWEEP_D) && !plan.row[1] && plan.mode[1] == C_GREEN) {
        a.defer_final = 1;
        c.finalize = 1;
        c.fin_lsh = (p->dim - 1) * p->log2n;
        c.fin_step = row_lines_per_cta(p->log2n, points_per_thread(p->log2n));
        c.ctl = a.ctl;
    }

    // n = 64 / 128 grids with the scalar / pointwise sweep: the whole solve as ONE cluster kernel
    // (cluster_kernels.cuh), the grid resident in the cluster's distributed shared memory
    // (BP_CLUSTER=0 keeps the two-launch graph loop)
    if (cluster_enabled(p, plan) && !(snapshots && n_snap > 0) && !p->timing) {
        ClArgs ca{};
        ca.row = a;
        ca.row.defer_final = 0;
        ca.col = c;
        const double h = p->grid.lx / p->n;
        ca.h2 = h * h;
        ca.direct = cfg->format == BP_FMT_DIRECT;
        CU(launch_cluster(p->log2n, ca, B, p->stream));
        CU(cudaStreamSynchronize(p->stream));
        p->stat_launches = 8 + 2 + 3 + (have_u0 ? 1 : 0) + 1;
        return BP_OK;
    }

    // kernels launched so far in this run: pack f (+ pack u0), 2x norms (2 each), Green
    // (2 row + column stage), init_control, 2x fill_nan, initial row pass + column stage
    const int stage = p->dim == 3 ? 3 : 1;
    p->stat_launches = 8 + 2 * stage + 3 + (have_u0 ? 1 : 0) + (map->kind == BP_MAP_FOURIER_DIAG);
    const int kps = plan_kernels(p, plan);
    p->stat_row_ms = p->stat_col_ms = 0;
    p->stat_timed = 0;
    const long max_launch = (long)cfg->max_iters + 1;  // launch k records entry k-1
    const size_t nd = p->dense_pts;

    if (snapshots && n_snap > 0) {
        // u^0
        rc = download(p, p->u0, p->u0, nullptr, snapshots);
        if (rc) return rc;
    }

    if (snapshots && n_snap > 0) {
        // debug path: one sweep at a time, copying u^k after launch k
        long k = 0;
        for (k = 1; k <= max_launch; ++k) {
            rc = sweep_once(p, plan, a, c, nullptr);
            if (rc) return rc;
            p->stat_launches += kps;
            if (k < n_snap) {
                // u^k lives in buffer k&1 for every member still iterating
                rc = download(p, (k & 1) ? p->u1 : p->u0, nullptr, nullptr,
                              snapshots + 2 * nd * B * k);
                if (rc) return rc;
            }
            CU(publish_int(p, a.ctl.n_active));
            CU(cudaStreamSynchronize(p->stream));
            if (*p->host_active == 0) break;
        }
    } else if (p->timing) {
        // instrumented path: CUDA events around every row / column launch on the handle's
        // stream, polled once per kGraphSweeps sweeps (same cadence as the graph path)
        const int ne = plan.n + 1;
        std::vector<cudaEvent_t> ev(ne * kGraphSweeps);
        for (auto& e : ev) CU(cudaEventCreate(&e));
        long launched = 0;
        while (launched < max_launch) {
            for (int s = 0; s < kGraphSweeps; ++s) {
                rc = sweep_once(p, plan, a, c, &ev[ne * s]);
                if (rc) break;
            }
            if (rc) break;
            launched += kGraphSweeps;
            p->stat_launches += (int64_t)kps * kGraphSweeps;
            CU(publish_int(p, a.ctl.n_active));
            CU(cudaStreamSynchronize(p->stream));
            for (int s = 0; s < kGraphSweeps; ++s) {
                for (int k = 0; k < plan.n; ++k) {
                    float ms = 0;
                    cudaEventElapsedTime(&ms, ev[ne * s + k], ev[ne * s + k + 1]);
                    (plan.row[k] ? p->stat_row_ms : p->stat_col_ms) += ms;
                }
                ++p->stat_timed;
            }
            if (*p->host_active == 0) break;
        }
        for (auto& e : ev) cudaEventDestroy(e);
        if (rc) return rc;
    } else {
        // graph of kGraphSweeps sweeps, replayed until every member terminated
        int split = split_batch(p, plan) ? std::min(split_parts(B, p->log2n), B) : 0;  // 0 = one graph, else parts
        // Waves (BP_GROUP = G members, split batches only): the batch is swept G members at a time
        // -- each wave's K part-graphs (kGraphSweeps sweeps) queue behind the previous wave's on the
        // same K streams -- so a wave's fields are re-used out of L2 across its sweeps
        const int group = split ? group_members(p, B) : 0;
        if (group) split = wave_parts(group);
        const int waves = group ? (B + group - 1) / group : 1;
        const bool reuse = p->graph && p->graph_split == split && p->graph_group == group &&
                           p->graph_map_kind == map->kind &&
                           p->graph_metric == map->metric && p->graph_format == cfg->format &&
                           p->graph_gamma.x == map->gamma_re && p->graph_gamma.y == map->gamma_im &&
                           p->graph_max_iters == cfg->max_iters && p->graph_rtol == cfg->rtol;
        if (!reuse) {
            if (p->graph) cudaGraphExecDestroy(p->graph);
            p->graph = nullptr;
            for (auto& g2 : p->graph2) {
                if (g2) cudaGraphExecDestroy(g2);
                g2 = nullptr;
            }
            for (auto gw : p->gwave)
                if (gw) cudaGraphExecDestroy(gw);
            p->gwave.clear();
            cudaGraph_t g;
            if (!split) {
                CU(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
                for (int s = 0; s < kGraphSweeps; ++s) sweep_once(p, plan, a, c, nullptr);
                CU(cudaStreamEndCapture(p->stream, &g));
                CU(cudaGraphInstantiate(&p->graph, g, 0));
                cudaGraphDestroy(g);
            } else {
                const int K = split;
                for (int k = 0; k < K; ++k) {
                    if (k && !p->stream2[k - 1]) CU(cudaStreamCreateWithFlags(&p->stream2[k - 1], cudaStreamNonBlocking));
                    if (!p->ev_join[k]) CU(cudaEventCreateWithFlags(&p->ev_join[k], cudaEventDisableTiming));
                }
                cudaStream_t keep = p->stream;
                p->gwave.assign((size_t)(waves - 1) * K, nullptr);
                for (int w = 0; w < waves; ++w) {
                    const int w0 = group ? w * group : 0, w1 = group ? std::min(B, w0 + group) : B;
                    for (int k = 0; k < K; ++k) {  // sweep_once launches on p->stream: capture each part
                        const int b0 = w0 + (int)((long)(w1 - w0) * k / K), b1 = w0 + (int)((long)(w1 - w0) * (k + 1) / K);
                        cudaGraphExec_t* dst = w ? &p->gwave[(size_t)(w - 1) * K + k] : (k ? &p->graph2[k - 1] : &p->graph);
                        if (b1 == b0) continue;  // (a short last wave)
                        RowArgs ak = row_args_range(a, p, b0, b1 - b0);
                        ColArgs ck = col_args_range(c, p, b0, b1 - b0);
                        // a wave's fields (or a small batch's single-member parts) live in L2
                        if (group || b1 - b0 == 1) ak.l2_hints = ck.l2_hints = BS_L2_HINTS;
                        p->stream = k ? p->stream2[k - 1] : keep;
                        cudaError_t e = cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal);
                        for (int sw = 0; e == cudaSuccess && sw < kGraphSweeps; ++sw) sweep_once(p, plan, ak, ck, nullptr);
                        if (e == cudaSuccess) e = cudaStreamEndCapture(p->stream, &g);
                        if (e == cudaSuccess) {
                            e = cudaGraphInstantiate(dst, g, 0);
                            cudaGraphDestroy(g);
                        }
                        p->stream = keep;
                        CU(e);
                    }
                }
            }
            p->graph_split = split;
            p->graph_group = group;
            p->graph_map_kind = map->kind;
            p->graph_metric = map->metric;
            p->graph_format = cfg->format;
            p->graph_gamma = a.gamma;
            p->graph_max_iters = cfg->max_iters;
            p->graph_rtol = cfg->rtol;
        }
        long launched = 0;
        if (split) {  // the other parts' streams start after everything enqueued so far
            CU(cudaEventRecord(p->ev_join[0], p->stream));
            for (int k = 1; k < split; ++k) CU(cudaStreamWaitEvent(p->stream2[k - 1], p->ev_join[0], 0));
        }
        while (launched < max_launch) {
            for (int w = 0; w < waves; ++w) {
                for (int k = 0; k < std::max(split, 1); ++k) {
                    cudaGraphExec_t ge = w ? p->gwave[(size_t)(w - 1) * split + k] : (k ? p->graph2[k - 1] : p->graph);
                    if (ge) CU(cudaGraphLaunch(ge, k ? p->stream2[k - 1] : p->stream));
                }
            }
            for (int k = 1; k < split; ++k) {
                CU(cudaEventRecord(p->ev_join[k], p->stream2[k - 1]));
                CU(cudaStreamWaitEvent(p->stream, p->ev_join[k], 0));  // every part before the poll
            }
            launched += kGraphSweeps;
            p->stat_launches += (int64_t)kps * kGraphSweeps * std::max(split, 1) * waves;  // every part's graph
            CU(publish_int(p, a.ctl.n_active));
            CU(cudaStreamSynchronize(p->stream));
            if (*p->host_active == 0) break;
        }
    }
    return BP_OK;
}

// bp::run on an any-shape handle: per sweep q = V u^m + f (members still active), z = G q (four
// line-transform launches + the spectral divide), then one element-wise pass (entry sums, u^{m+1})
// and the device-side entry / termination record -- the same Control protocol as the fused
// path (ping-pong u, entry m finalised after u^m, result_buf), polled every kGraphSweeps sweeps.
int run_core_generic(bp_problem* p, const bp_map* map, const bp_iter_config* cfg, bool have_u0,
                     double* snapshots, int n_snap) {
    const int B = p->batch;
    const GenArgs g = gen_args(p);
    Control c = make_control(p);
    c.max_iters = cfg->max_iters;
    c.rtol = cfg->rtol;
    if (int rc = norms(p, p->f, p->fnorm_l2)) return rc;
    if (int rc = gen_spectral(p, true, p->f, p->y)) return rc;
    if (int rc = norms(p, p->y, p->fnorm_reta)) return rc;
    std::vector<double> fn(B);
    if (int rc = read_fnorm(p, fn)) return rc;
    for (int b = 0; b < B; ++b)
        if (!(fn[b] > 0.0)) return set_err(BP_EINVAL, "run: zero source");
    if (!have_u0) CU(cudaMemsetAsync(p->u0, 0, sizeof(double2) * p->alloc, p->stream));
    CU(cudaMemsetAsync(p->u1, 0, sizeof(double2) * p->alloc, p->stream));
    init_control_kernel<<<(B + 127) / 128, 128, 0, p->stream>>>(c, B);
    fill_nan_kernel<<<grid_for((size_t)B * p->trace_cap), 256, 0, p->stream>>>(p->trace_l2, (size_t)B * p->trace_cap);
    fill_nan_kernel<<<grid_for((size_t)B * p->trace_cap), 256, 0, p->stream>>>(p->trace_reta, (size_t)B * p->trace_cap);
    CU(cudaGetLastError());
    const int nchunk = 64;
    const double2 gamma = make_double2(map->gamma_re, map->gamma_im);
    const int direct = cfg->format == BP_FMT_DIRECT;
    const size_t nd = p->dense_pts;
    if (p->gper) {
        // iterate carried in Fourier space as well (U = DFT(u^m) in x, Q in y): per sweep one
        // forward transform (of q^m) and one backward (u^{m+1} for the members still active)
        if (int rc = gen_dst2(p, p->u0, p->x, 1.0)) return rc;
        if (snapshots && n_snap > 0)
            if (int rc = download(p, p->u0, nullptr, nullptr, snapshots)) return rc;
        p->stat_launches = 0;
        const long max_launch = (long)cfg->max_iters + 1;
        for (long k = 1; k <= max_launch; ++k) {
            gen_source_kernel<<<grid_for(p->field * B), 256, 0, p->stream>>>(g, c, p->u0, p->u1, p->f, p->y);
            if (int rc = gen_dst2(p, p->y, p->y, 1.0)) return rc;
            gen_psweep_kernel<<<dim3(nchunk, B), 256, 0, p->stream>>>(g, c, p->y, p->x, gamma, direct, p->gpart, nchunk);
            gen_finalize_kernel<<<(B + 127) / 128, 128, 0, p->stream>>>(c, B, p->gpart, nchunk);
            if (int rc = gen_dst2(p, p->x, (k & 1) ? p->u1 : p->u0, g.gscale, true, c.status)) return rc;
            CU(cudaGetLastError());
            p->stat_launches += 8;
            if (snapshots && k < n_snap)
                if (int rc = download(p, (k & 1) ? p->u1 : p->u0, nullptr, nullptr, snapshots + 2 * nd * B * k)) return rc;
            if ((snapshots && n_snap > 0) || k % kGraphSweeps == 0 || k == max_launch) {
                CU(publish_int(p, c.n_active));
                CU(cudaStreamSynchronize(p->stream));
                if (*p->host_active == 0) break;
            }
        }
        return BP_OK;
    }
    // hx != hy: five_point (hx^2 only, kernels.cpp:56-69) and the two-spacing symbol differ, the
    // key identity ||G r|| = ||G(V u + f) - u|| no longer holds -- apply G to r explicitly
    const bool exact_reta = std::fabs(p->grid.lx / (p->gnx + 1) - p->grid.ly / (p->gny + 1)) >
                            1e-15 * (p->grid.lx / (p->gnx + 1));
    if (snapshots && n_snap > 0)
        if (int rc = download(p, p->u0, nullptr, nullptr, snapshots)) return rc;
    p->stat_launches = 0;
    const long max_launch = (long)cfg->max_iters + 1;
    for (long k = 1; k <= max_launch; ++k) {
        gen_source_kernel<<<grid_for(p->field * B), 256, 0, p->stream>>>(g, c, p->u0, p->u1, p->f, p->y);
        if (int rc = gen_spectral(p, true, p->y, p->y)) return rc;
        gen_sweep_kernel<<<dim3(nchunk, B), 256, 0, p->stream>>>(g, c, p->y, p->f, p->u0, p->u1, p->u0, p->u1,
                                                                 map->kind, gamma, direct, p->gpart, nchunk,
                                                                 exact_reta ? p->x : nullptr);
        if (exact_reta) {  // ||G r^m|| (iterate.cpp:131) by a Green application
            if (int rc = gen_spectral(p, true, p->x, p->x)) return rc;
            gen_part_kernel<<<dim3(nchunk, B), 256, 0, p->stream>>>(g, c, p->x, p->gpart, nchunk);
        }
        gen_finalize_kernel<<<(B + 127) / 128, 128, 0, p->stream>>>(c, B, p->gpart, nchunk);
        CU(cudaGetLastError());
        p->stat_launches += 8;
        if (snapshots && k < n_snap)  // u^k in buffer k & 1 for every member still iterating
            if (int rc = download(p, (k & 1) ? p->u1 : p->u0, nullptr, nullptr, snapshots + 2 * nd * B * k)) return rc;
        if ((snapshots && n_snap > 0) || k % kGraphSweeps == 0 || k == max_launch) {
            CU(publish_int(p, c.n_active));
            CU(cudaStreamSynchronize(p->stream));
            if (*p->host_active == 0) break;
        }
    }
    return BP_OK;
}

// A u on an any-shape handle (dense batch): five-point stencil (Dirichlet, kernels.cpp:56-69) or
// the pseudospectral F^-1(|xi|^2 F u) - k2 u (periodic, helmholtz.cpp:27-32); f != null: f - A u.
// tmp: scratch field (periodic only).  gen_spectral uses p->T.
int gen_apply_A(bp_problem* p, const double2* u, const double2* f, double2* out, double2* tmp) {
    const GenArgs g = gen_args(p);
    const size_t total = p->field * p->batch;
    if (p->gper) {
        if (int rc = gen_spectral(p, false, u, out, 2)) return rc;
        gen_pointwise_kernel<<<grid_for(total), 256, 0, p->stream>>>(g, 5, u, nullptr, tmp);
        combine_kernel<<<grid_for(total), 256, 0, p->stream>>>(out, tmp, f, total);
    } else {
        gen_pointwise_kernel<<<grid_for(total), 256, 0, p->stream>>>(g, f ? 3 : 0, u, f, out);
    }
    CU(cudaGetLastError());
    return BP_OK;
}

// bp::run with OptimalScalarMap (both metrics) or FourierDiagMap on an any-shape handle
// (Dirichlet or periodic): the reference's loop (iterate.cpp:105-150, correction.cpp:22-76)
// operator by operator in physical space -- r = f - A u, G r for the R_eta trace, the direction
// (r, G r, or the Born residual G(V u + f) - u), the map, the update -- with the reductions and
// the termination test on the device.  Generic, not fused: the any-shape path serves shapes the
// fused kernels do not take (run_sweep at an arbitrary n, bench.cpp:140-151).
int run_core_generic_maps(bp_problem* p, const bp_map* map, const bp_iter_config* cfg, bool have_u0,
                          double* snapshots, int n_snap) {
    const int B = p->batch;
    const GenArgs g = gen_args(p);
    const size_t total = p->field * B, fb = sizeof(double2) * total;
    Control c = make_control(p);
    c.max_iters = cfg->max_iters;
    c.rtol = cfg->rtol;
    if (!p->gm0) {
        CU(cudaMalloc(&p->gm0, fb));
        CU(cudaMalloc(&p->gm1, fb));
        CU(cudaMalloc(&p->gm2, fb));
    }
    if (map->kind == BP_MAP_FOURIER_DIAG) {
        if (!p->fd) CU(cudaMalloc(&p->fd, sizeof(double2) * p->field));
        CU(cudaMemcpyAsync(p->fd, map->m, sizeof(double2) * p->field, cudaMemcpyHostToDevice, p->stream));
    }
    if (int rc = norms(p, p->f, p->fnorm_l2)) return rc;
    if (int rc = gen_spectral(p, true, p->f, p->y)) return rc;
    if (int rc = norms(p, p->y, p->fnorm_reta)) return rc;
    std::vector<double> fn(B);
    if (int rc = read_fnorm(p, fn)) return rc;
    for (int b = 0; b < B; ++b)
        if (!(fn[b] > 0.0)) return set_err(BP_EINVAL, "run: zero source");
    if (!have_u0) CU(cudaMemsetAsync(p->u0, 0, fb, p->stream));
    CU(cudaMemsetAsync(p->u1, 0, fb, p->stream));
    init_control_kernel<<<(B + 127) / 128, 128, 0, p->stream>>>(c, B);
    fill_nan_kernel<<<grid_for((size_t)B * p->trace_cap), 256, 0, p->stream>>>(p->trace_l2, (size_t)B * p->trace_cap);
    fill_nan_kernel<<<grid_for((size_t)B * p->trace_cap), 256, 0, p->stream>>>(p->trace_reta, (size_t)B * p->trace_cap);
    CU(cudaGetLastError());
    const int nchunk = 64;
    const size_t nd = p->dense_pts;
    double2 *U = p->gm0, *R = p->x, *GR = p->y, *X = p->gm1, *W = p->gm2, *tmp = p->dense;
    if (snapshots && n_snap > 0)
        if (int rc = download(p, p->u0, nullptr, nullptr, snapshots)) return rc;
    p->stat_launches = 0;
    const long max_launch = (long)cfg->max_iters + 1;
    for (long k = 1; k <= max_launch; ++k) {
        // entry m = k - 1: r^m = f - A u^m, G r^m (iterate.cpp:108-110, 128-132)
        gen_gather_kernel<<<grid_for(total), 256, 0, p->stream>>>(g, c, p->u0, p->u1, U);
        if (int rc = gen_apply_A(p, U, p->f, R, tmp)) return rc;
        if (int rc = gen_spectral(p, true, R, GR)) return rc;
        // direction (iterate.cpp:118-123), before the entry advances the sweep counter
        const double2* D = R;
        if (cfg->format == BP_FMT_CBS) {
            D = GR;
        } else if (cfg->format == BP_FMT_NPBS) {  // born_residual (problem.cpp:41-49)
            gen_pointwise_kernel<<<grid_for(total), 256, 0, p->stream>>>(g, 4, U, p->f, X);
            if (int rc = gen_spectral(p, true, X, X)) return rc;
            gen_sub_kernel<<<grid_for(total), 256, 0, p->stream>>>(X, X, U, (long)total);
            D = X;
        }
        gen_norms_kernel<<<dim3(nchunk, B), 256, 0, p->stream>>>(g, c, R, GR, p->gpart, nchunk);
        gen_finalize_kernel<<<(B + 127) / 128, 128, 0, p->stream>>>(c, B, p->gpart, nchunk);
        // apply_correction (correction.cpp:22-76) for the members still active
        if (map->kind == BP_MAP_OPTIMAL_SCALAR) {
            if (map->metric == BP_METRIC_RETA) {  // w = x - G V x, gamma = <w, x> / <w, w>
                gen_pointwise_kernel<<<grid_for(total), 256, 0, p->stream>>>(g, 1, D, nullptr, W);
                if (int rc = gen_spectral(p, true, W, W)) return rc;
                gen_sub_kernel<<<grid_for(total), 256, 0, p->stream>>>(W, D, W, (long)total);
                gen_dot_kernel<<<dim3(nchunk, B), 256, 0, p->stream>>>(g, c, W, D, p->gpart, nchunk);
            } else {  // w = A x, gamma = <w, r> / <w, w>
                if (int rc = gen_apply_A(p, D, nullptr, W, tmp)) return rc;
                gen_dot_kernel<<<dim3(nchunk, B), 256, 0, p->stream>>>(g, c, W, R, p->gpart, nchunk);
            }
            gen_gamma_kernel<<<(B + 127) / 128, 128, 0, p->stream>>>(c, B, p->gpart, nchunk);
            gen_update_kernel<<<grid_for(total), 256, 0, p->stream>>>(g, c, p->u0, p->u1, D, 1);
        } else {  // FourierDiag: du = T^-1(m T x) (correction.cpp:63-68)
            if (int rc = gen_dst2(p, D, W, 1.0)) return rc;
            gen_modemul_kernel<<<grid_for(total), 256, 0, p->stream>>>(g, W, p->fd);
            if (int rc = gen_dst2(p, W, W, g.gscale, p->gper)) return rc;
            gen_update_kernel<<<grid_for(total), 256, 0, p->stream>>>(g, c, p->u0, p->u1, W, 0);
        }
        CU(cudaGetLastError());
        p->stat_launches += 16;
        if (snapshots && k < n_snap)  // u^k in buffer k & 1 for every member still iterating
            if (int rc = download(p, (k & 1) ? p->u1 : p->u0, nullptr, nullptr, snapshots + 2 * nd * B * k)) return rc;
        if ((snapshots && n_snap > 0) || k % kGraphSweeps == 0 || k == max_launch) {
            CU(publish_int(p, c.n_active));
            CU(cudaStreamSynchronize(p->stream));
            if (*p->host_active == 0) break;
        }
    }
    return BP_OK;
}

int finish_run_periodic(bp_problem* p, double* u_out, bool host_ptr);
int finish_run_cdr(bp_problem* p, double* u_out, bool host_ptr);
int finish_run_traces(bp_problem* p, const bp_iter_config* cfg, double* res_l2, double* res_reta,
                      bp_trace* info);

int finish_run(bp_problem* p, const bp_iter_config* cfg, double* u_out, bool host_ptr,
               double* res_l2, double* res_reta, bp_trace* info) {
    Control c = make_control(p);
    int rc = p->cdr        ? finish_run_cdr(p, u_out, host_ptr)
             : p->periodic ? finish_run_periodic(p, u_out, host_ptr)
                           : download(p, p->u0, p->u1, c.result_buf, u_out, host_ptr);
    if (rc) return rc;
    if (!p->periodic && !p->cdr) p->stat_launches += 1;  // unpack
    return finish_run_traces(p, cfg, res_l2, res_reta, info);
}

// iteration counts, terminations, norms and the trace vectors of the last run -> host
int finish_run_traces(bp_problem* p, const bp_iter_config* cfg, double* res_l2, double* res_reta,
                      bp_trace* info) {
    const int B = p->batch;
    Control c = make_control(p);
    std::vector<int> iters(B), term(B);
    std::vector<double> f1(B), f2(B);
    CU(cudaMemcpyAsync(iters.data(), c.iters, sizeof(int) * B, cudaMemcpyDeviceToHost, p->stream));
    CU(cudaMemcpyAsync(term.data(), c.term, sizeof(int) * B, cudaMemcpyDeviceToHost, p->stream));
    CU(cudaMemcpyAsync(f1.data(), p->fnorm_l2, sizeof(double) * B, cudaMemcpyDeviceToHost, p->stream));
    CU(cudaMemcpyAsync(f2.data(), p->fnorm_reta, sizeof(double) * B, cudaMemcpyDeviceToHost, p->stream));
    const int stride = cfg->max_iters + 1;
    if (res_l2)
        CU(cudaMemcpy2DAsync(res_l2, sizeof(double) * stride, p->trace_l2, sizeof(double) * p->trace_cap,
                             sizeof(double) * stride, B, cudaMemcpyDeviceToHost, p->stream));
    if (res_reta)
        CU(cudaMemcpy2DAsync(res_reta, sizeof(double) * stride, p->trace_reta,
                             sizeof(double) * p->trace_cap, sizeof(double) * stride, B,
                             cudaMemcpyDeviceToHost, p->stream));
    CU(cudaStreamSynchronize(p->stream));
    p->stat_sweeps = 0;
    for (int b = 0; b < B; ++b) {
        if (info) {
            info[b].iters = iters[b];
            info[b].terminated = term[b];
            info[b].fnorm_l2 = f1[b];
            info[b].fnorm_reta = f2[b];
        }
        p->stat_sweeps += iters[b];
    }
    return BP_OK;
}


// ------------------------------------------------------------------ periodic family (host)
PerArgs per_args(const bp_problem* p) {
    PerArgs a{};
    a.batch = p->batch;
    a.k0sq = p->k0sq;
    a.eta = p->eta;
    a.xi2 = p->xi2;
    a.k2 = p->k2;
    a.f = p->f;
    a.T = p->T;
    a.U0 = p->u0;
    a.U1 = p->u1;
    a.fd = p->fd;
    a.tw = p->tw;
    a.scale = 1.0;
    a.inv_npts = 1.0 / ((double)p->n * p->n);
    a.map_kind = MK_SCALAR;
    a.gamma = make_double2(1.0, 0.0);
    a.ctl = make_control(p);
    return a;
}

#define CUP(call) CU(call)

// Green / L_ref / transforms on padded-free periodic fields: in -> out (out - sub)
int periodic_apply(bp_problem* p, int which, const double2* in, double2* out, const double2* sub) {
    PerArgs a = per_args(p);
    const double inv = 1.0 / ((double)p->n * p->n);
    a.in = in;
    switch (which) {
        case 0:  // G q = F^-1(F q / lambda)   (apply_symbol Divide, symbol.cpp:19-39)
        case 1:  // born: G(V u + f) - u
        case 2:  // L_ref
            CUP(launch_periodic(p->log2n, true, which == 1 ? RP_FWD_BORN : RP_FWD, a, p->stream));
            a.scale = inv;
            CUP(launch_periodic(p->log2n, false, which == 2 ? CP_LREF : CP_GREEN, a, p->stream));
            a.out = out;
            a.sub = sub;
            CUP(launch_periodic(p->log2n, true, RP_INV, a, p->stream));
            return BP_OK;
        case 3:  // forward transform (unnormalised DFT, transforms.hpp:16)
            CUP(launch_periodic(p->log2n, true, RP_FWD, a, p->stream));
            a.scale = 1.0;
            CUP(launch_periodic(p->log2n, false, CP_ONE, a, p->stream));
            CUP(cudaMemcpyAsync(out, p->T, sizeof(double2) * p->field * p->batch,
                                cudaMemcpyDeviceToDevice, p->stream));
            return BP_OK;
        case 4:  // inverse transform (backward DFT / (nx ny))
            a.T = const_cast<double2*>(in);
            a.out = out;
            CUP(launch_periodic(p->log2n, true, RP_INV, a, p->stream));
            a.T = out;
            a.scale = inv;
            CUP(launch_periodic(p->log2n, false, CP_INV, a, p->stream));
            return BP_OK;
    }
    return set_err(BP_EINVAL, "bad periodic op");
}

__global__ void select_copy_kernel(const double2* __restrict__ p0, const double2* __restrict__ p1,
                                   const int* __restrict__ select, double2* __restrict__ out,
                                   size_t per, int batch) {
    const size_t total = per * batch;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const size_t b = idx / per;
        out[idx] = (select && select[b]) ? p1[idx] : p0[idx];
    }
}

// bp::run for the periodic family: the iterate lives in Fourier space (U0/U1 ping-pong)
int run_core_periodic(bp_problem* p, const bp_map* map, const bp_iter_config* cfg, bool have_u0,
                      double* snapshots, int n_snap) {
    const int B = p->batch;
    PerArgs a = per_args(p);
    a.ctl.max_iters = cfg->max_iters;
    a.ctl.rtol = cfg->rtol;
    a.map_kind = map->kind == BP_MAP_FOURIER_DIAG ? MK_FOURIER_DIAG : MK_SCALAR;
    a.gamma = make_double2(map->gamma_re, map->gamma_im);
    a.direct = cfg->format == BP_FMT_DIRECT;
    const bool opt = map->kind == BP_MAP_OPTIMAL_SCALAR;
    a.metric_reta = opt && map->metric == BP_METRIC_RETA;
    a.D = p->x;   // OptimalScalar: spectral direction (x is free once the run has started)
    a.T2 = p->y;  // OptimalScalar (Euclidean): second intermediate (snapshots reuse y between sweeps)
    if (map->kind == BP_MAP_FOURIER_DIAG) {
        CU(cudaMemcpyAsync(p->fd, map->m, sizeof(double2) * p->field, cudaMemcpyHostToDevice, p->stream));
    }
    // fnorm_l2 = ||f||, fnorm_reta = ||G f||  (iterate.cpp:93,102)
    if (int rc = norms(p, p->f, p->fnorm_l2)) return rc;
    if (int rc = periodic_apply(p, 0, p->f, p->y, nullptr)) return rc;
    if (int rc = norms(p, p->y, p->fnorm_reta)) return rc;
    std::vector<double> fn(B);
    if (int rc = read_fnorm(p, fn)) return rc;
    for (int b = 0; b < B; ++b)
        if (!(fn[b] > 0.0)) return set_err(BP_EINVAL, "run: zero source");
    // U^0 = F u0 (u0 staged in p->x by the caller) or 0
    if (have_u0) {
        if (int rc = periodic_apply(p, 3, p->x, p->u0, nullptr)) return rc;
    } else {
        CU(cudaMemsetAsync(p->u0, 0, sizeof(double2) * p->alloc, p->stream));
        CU(cudaMemsetAsync(p->x, 0, sizeof(double2) * p->alloc, p->stream));
    }
    CU(cudaMemsetAsync(p->u1, 0, sizeof(double2) * p->alloc, p->stream));
    init_control_kernel<<<(B + 127) / 128, 128, 0, p->stream>>>(a.ctl, B);
    fill_nan_kernel<<<grid_for((size_t)B * p->trace_cap), 256, 0, p->stream>>>(p->trace_l2, (size_t)B * p->trace_cap);
    fill_nan_kernel<<<grid_for((size_t)B * p->trace_cap), 256, 0, p->stream>>>(p->trace_reta, (size_t)B * p->trace_cap);
    CU(cudaGetLastError());
    // T = F_y q^0, q^0 = V u^0 + f (u^0 physical in p->x)
    a.in = p->x;
    CU(launch_periodic(p->log2n, true, RP_FWD_BORN, a, p->stream));
    p->stat_launches = 16 + (have_u0 ? 2 : 0);
    p->stat_row_ms = p->stat_col_ms = 0;
    p->stat_timed = 0;
    const long max_launch = (long)cfg->max_iters + 1;
    const size_t nd = p->dense_pts;
    // launches per sweep: scalar / FourierDiag 2; OptimalScalar 4 (Euclidean) or 5 (R_eta)
    const int per_sweep = opt ? (a.metric_reta ? 5 : 4) : 2;
    auto sweep = [&](cudaEvent_t* ev) -> int {
        if (ev) CU(cudaEventRecord(ev[0], p->stream));
        if (opt) {
            CU(launch_periodic(p->log2n, false, CP_OPT_A, a, p->stream));
            if (a.metric_reta) {
                CU(launch_periodic(p->log2n, true, RP_RETA_B, a, p->stream));
                CU(launch_periodic(p->log2n, false, CP_RETA_C, a, p->stream));
            } else {
                CU(launch_periodic(p->log2n, true, RP_OPT_B, a, p->stream));
            }
            CU(launch_periodic(p->log2n, false, CP_OPT_C, a, p->stream));
        } else {
            CU(launch_periodic(p->log2n, false, CP_SWEEP, a, p->stream));
        }
        if (ev) CU(cudaEventRecord(ev[1], p->stream));
        CU(launch_periodic(p->log2n, true, RP_SWEEP, a, p->stream));
        if (ev) CU(cudaEventRecord(ev[2], p->stream));
        return BP_OK;
    };
    if (snapshots && n_snap > 0) {
        // u^0 = F^-1 U^0
        if (int rc = periodic_apply(p, 4, p->u0, p->y, nullptr)) return rc;
        if (int rc = download(p, p->y, nullptr, nullptr, snapshots)) return rc;
        for (long k = 1; k <= max_launch; ++k) {
            if (int rc = sweep(nullptr)) return rc;
            p->stat_launches += per_sweep;
            if (k < n_snap) {  // u^k = F^-1 U^k, U^k in buffer k&1
                if (int rc = periodic_apply(p, 4, (k & 1) ? p->u1 : p->u0, p->y, nullptr)) return rc;
                if (int rc = download(p, p->y, nullptr, nullptr, snapshots + 2 * nd * B * k)) return rc;
            }
            CU(publish_int(p, a.ctl.n_active));
            CU(cudaStreamSynchronize(p->stream));
            if (*p->host_active == 0) break;
        }
        return BP_OK;
    }
    std::vector<cudaEvent_t> ev;
    if (p->timing) {
        ev.resize(3 * kGraphSweeps);
        for (auto& e : ev) CU(cudaEventCreate(&e));
    }
    long launched = 0;
    int rc = BP_OK;
    while (launched < max_launch && rc == BP_OK) {
        for (int s = 0; s < kGraphSweeps && rc == BP_OK; ++s) rc = sweep(p->timing ? &ev[3 * s] : nullptr);
        if (rc) break;
        launched += kGraphSweeps;
        p->stat_launches += per_sweep * kGraphSweeps;
        CU(publish_int(p, a.ctl.n_active));
        CU(cudaStreamSynchronize(p->stream));
        if (p->timing) {
            for (int s = 0; s < kGraphSweeps; ++s) {
                float c = 0, r = 0;
                cudaEventElapsedTime(&c, ev[3 * s], ev[3 * s + 1]);
                cudaEventElapsedTime(&r, ev[3 * s + 1], ev[3 * s + 2]);
                p->stat_col_ms += c;
                p->stat_row_ms += r;
                ++p->stat_timed;
            }
        }
        if (*p->host_active == 0) break;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    return rc;
}

int finish_run_periodic(bp_problem* p, double* u_out, bool host_ptr) {
    Control c = make_control(p);
    select_copy_kernel<<<grid_for(p->field * p->batch), 256, 0, p->stream>>>(
        p->u0, p->u1, c.result_buf, p->x, p->field, p->batch);
    CU(cudaGetLastError());
    if (int rc = periodic_apply(p, 4, p->x, p->y, nullptr)) return rc;  // u = F^-1 U
    p->stat_launches += 3;
    return download(p, p->y, nullptr, nullptr, u_out, host_ptr);
}

// ------------------------------------------------------------------ CDR family (config c4, host)
// Real fp64 fields, n x n per member, no padding (cell-centred Neumann nodes (i+1/2) h).
CdrArgs cdr_args(const bp_problem* p) {
    CdrArgs a{};
    a.batch = p->batch;
    a.h = p->grid.lx / p->n;
    a.sigma0 = p->sigma0;
    a.bx = p->bx;
    a.by = p->by;
    a.sigma = p->sigma;
    a.f = reinterpret_cast<const double*>(p->f);
    a.T = reinterpret_cast<double*>(p->T);
    a.u0 = reinterpret_cast<double*>(p->u0);
    a.u1 = reinterpret_cast<double*>(p->u1);
    a.rnorm2 = p->rnorm2;
    a.lapn = p->lapn;
    a.tw = p->tw;
    a.w4 = p->w4;
    a.scale = 1.0;
    a.gamma = 1.0;
    a.ctl = make_control(p);
    return a;
}

// members [b0, b0 + nb) of a CDR batch (split-batch graphs): per-member arrays offset, the
// per-pair partials at the crow kernels' own stride (n/2 pairs per member)
CdrArgs cdr_args_range(const CdrArgs& a0, const bp_problem* p, int b0, int nb) {
    CdrArgs a = a0;
    const size_t fo = (size_t)b0 * p->field;
    a.batch = nb;
    a.sigma0 += b0;
    a.bx += fo;
    a.by += fo;
    a.sigma += fo;
    a.f += fo;
    a.T += fo;
    a.u0 += fo;
    a.u1 += fo;
    a.rnorm2 += b0;
    Control c = control_range(a.ctl, p, b0);
    c.partial = a0.ctl.partial + (size_t)b0 * (p->n / 2) * kPartStride;
    a.ctl = c;
    return a;
}

// A u, V u, V^T u, f - A u, V u + f on real fields (ops 0 .. 4): the same upwind stencil as the
// RC_B prologue (cdr_kernels.cuh), elementwise for the operator API; V^T is the role of
// Problem::apply_V_adjoint (problem.hpp:28) for this real family
__global__ void cdr_stencil_kernel(int op, const double* __restrict__ u, const double* __restrict__ f,
                                   const double* __restrict__ bx, const double* __restrict__ by,
                                   const double* __restrict__ sigma, const double* __restrict__ sigma0,
                                   double* __restrict__ out, int batch, int log2n, double h) {
    const int n = 1 << log2n;
    const size_t total = (size_t)batch << (2 * log2n);
    const double ih = 1.0 / h, ih2 = ih * ih;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const int b = (int)(idx >> (2 * log2n));
        const int j = (int)(idx & (n - 1)), i = (int)((idx >> log2n) & (n - 1));
        const double c = u[idx];
        const double w = i > 0 ? u[idx - n] : c, e = i < n - 1 ? u[idx + n] : c;
        const double so = j > 0 ? u[idx - 1] : c, no = j < n - 1 ? u[idx + 1] : c;
        const double lap = (4.0 * c - w - e - so - no) * ih2;
        const double vx = bx[idx], vy = by[idx], sg = sigma[idx];
        const double dx = vx >= 0.0 ? (c - w) * ih : (e - c) * ih;
        const double dy = vy >= 0.0 ? (c - so) * ih : (no - c) * ih;
        const double conv = vx * dx + vy * dy;
        double r;
        switch (op) {
            case 0: r = (lap + conv) + sg * c; break;
            case 1: r = (sigma0[b] - sg) * c - conv; break;
            case 2: {  // V^T u: the transposed upwind stencil (column idx of conv)
                double t = 0.0;
                if (vx >= 0.0 && i > 0) t += vx * ih * c;
                if (vx < 0.0 && i < n - 1) t -= vx * ih * c;
                if (i < n - 1 && bx[idx + n] >= 0.0) t -= bx[idx + n] * ih * e;
                if (i > 0 && bx[idx - n] < 0.0) t += bx[idx - n] * ih * w;
                if (vy >= 0.0 && j > 0) t += vy * ih * c;
                if (vy < 0.0 && j < n - 1) t -= vy * ih * c;
                if (j < n - 1 && by[idx + 1] >= 0.0) t -= by[idx + 1] * ih * no;
                if (j > 0 && by[idx - 1] < 0.0) t += by[idx - 1] * ih * so;
                r = (sigma0[b] - sg) * c - t;
                break;
            }
            case 3: r = f[idx] - ((lap + conv) + sg * c); break;
            default: r = ((sigma0[b] - sg) * c - conv) + f[idx]; break;
        }
        out[idx] = r;
    }
}

int cdr_upload(bp_problem* p, const double* src, double2* dst, bool host_ptr = true) {
    CU(cudaMemcpyAsync(dst, src, sizeof(double) * p->field * p->batch,
                       host_ptr ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, p->stream));
    return BP_OK;
}

int cdr_download(bp_problem* p, const double2* src, double* dst, bool host_ptr = true) {
    CU(cudaMemcpyAsync(dst, src, sizeof(double) * p->field * p->batch,
                       host_ptr ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, p->stream));
    return BP_OK;
}

// CC_GREEN column pass of the CDR family: the Neumann tridiagonal x-solve when the handle has its
// tables (equal to DCT-II -> x scale / lambda -> DCT-III = 2n h^2 scale Tri^-1, the REDFT01
// REDFT10 pair multiplying by 2n), else the DCT route
cudaError_t cdr_green(bp_problem* p, const CdrArgs& ac, int b0 = 0) {
    if (!p->tri) return launch_cdr(p->log2n, false, CC_GREEN, ac, p->stream);
    ColArgs c{};
    c.batch = ac.batch;
    c.T = reinterpret_cast<double2*>(ac.T);
    c.status = ac.ctl.status;
    c.tri = p->tri + (size_t)b0 * (p->n / 2) * (2 * kTriP + p->n / kTriP);
    const double h = p->grid.lx / p->n;
    c.tri_scale = 2.0 * p->n * h * h * ac.scale;
    return launch_tri(p->log2n, CL_CDR, c, p->stream);
}

// G / L_ref / transforms (transforms.cpp:105-148 with REDFT10 / REDFT01, inverse 1/(4 nx ny))
//   which 0 G, 2 L_ref, 3 forward transform, 4 inverse transform; out - sub when sub != null
int cdr_apply(bp_problem* p, int which, const double2* in, double2* out, const double2* sub) {
    CdrArgs a = cdr_args(p);
    // operator applications act on every member: the column kernel's skip of terminated
    // members (ctl.status) belongs to the sweep only -- left set, a member that terminated in
    // the handle's previous run kept its forward transform here (||G f|| of the next run wrong)
    a.ctl.status = nullptr;
    const double inv = 1.0 / (4.0 * (double)p->n * p->n);
    a.in = reinterpret_cast<const double*>(in);
    a.out = reinterpret_cast<double*>(out);
    a.sub = reinterpret_cast<const double*>(sub);
    switch (which) {
        case 0:
        case 2:
            CU(launch_cdr(p->log2n, true, RC_FWD, a, p->stream));
            a.scale = inv;
            CU(which == 0 ? cdr_green(p, a) : launch_cdr(p->log2n, false, CC_LREF, a, p->stream));
            a.scale = 1.0;
            CU(launch_cdr(p->log2n, true, RC_INV, a, p->stream));
            return BP_OK;
        case 3:
            CU(launch_cdr(p->log2n, true, RC_FWD, a, p->stream));
            CU(launch_cdr(p->log2n, false, CC_ONE, a, p->stream));
            CU(cudaMemcpyAsync(out, p->T, sizeof(double) * p->field * p->batch,
                               cudaMemcpyDeviceToDevice, p->stream));
            return BP_OK;
        case 4:
            a.T = const_cast<double*>(a.in);
            a.sub = nullptr;
            CU(launch_cdr(p->log2n, true, RC_INV, a, p->stream));
            a.T = a.out;
            a.scale = inv;
            CU(launch_cdr(p->log2n, false, CC_INV, a, p->stream));
            return BP_OK;
    }
    return set_err(BP_EINVAL, "bad CDR op");
}

int cdr_stencil(bp_problem* p, int op, const double2* u, const double2* f, double2* out) {
    cdr_stencil_kernel<<<grid_for(p->field * p->batch), 256, 0, p->stream>>>(
        op, reinterpret_cast<const double*>(u), reinterpret_cast<const double*>(f), p->bx, p->by,
        p->sigma, p->sigma0, reinterpret_cast<double*>(out), p->batch, p->log2n, p->grid.lx / p->n);
    CU(cudaGetLastError());
    return BP_OK;
}

// bp::run with OptimalScalarMap (both metrics, correction.cpp:22-48) on the CDR family: the
// reference's loop operator by operator on the real fields (as run_core_generic_maps; the real
// arrays are read as pairs, whose complex inner product's real part is the real one), gamma real.
int run_core_cdr_maps(bp_problem* p, const bp_map* map, const bp_iter_config* cfg, bool have_u0,
                      double* snapshots, int n_snap) {
    const int B = p->batch;
    const size_t total = p->field * B / 2, rb = sizeof(double) * p->field * B;  // double2 pairs
    if (!p->gamma) CU(cudaMalloc(&p->gamma, sizeof(double2) * (size_t)B));
    Control c = make_control(p);
    c.max_iters = cfg->max_iters;
    c.rtol = cfg->rtol;
    GenArgs g{};
    g.batch = B;
    g.nx = p->n;
    g.ny = p->n / 2;
    if (!p->gm1) {
        CU(cudaMalloc(&p->gm1, rb));
        CU(cudaMalloc(&p->gm2, rb));
    }
    if (!p->gpart) CU(cudaMalloc(&p->gpart, sizeof(double) * (size_t)B * 64 * 4));
    if (int rc = norms(p, p->f, p->fnorm_l2)) return rc;
    if (int rc = cdr_apply(p, 0, p->f, p->y, nullptr)) return rc;
    if (int rc = norms(p, p->y, p->fnorm_reta)) return rc;
    std::vector<double> fn(B);
    if (int rc = read_fnorm(p, fn)) return rc;
    for (int b = 0; b < B; ++b)
        if (!(fn[b] > 0.0)) return set_err(BP_EINVAL, "run: zero source");
    if (!have_u0) CU(cudaMemsetAsync(p->u0, 0, sizeof(double2) * p->alloc, p->stream));
    CU(cudaMemsetAsync(p->u1, 0, sizeof(double2) * p->alloc, p->stream));
    init_control_kernel<<<(B + 127) / 128, 128, 0, p->stream>>>(c, B);
    fill_nan_kernel<<<grid_for((size_t)B * p->trace_cap), 256, 0, p->stream>>>(p->trace_l2, (size_t)B * p->trace_cap);
    fill_nan_kernel<<<grid_for((size_t)B * p->trace_cap), 256, 0, p->stream>>>(p->trace_reta, (size_t)B * p->trace_cap);
    CU(cudaGetLastError());
    const int nchunk = 64;
    const size_t nd = p->field;
    double2 *R = p->x, *GR = p->y, *X = p->gm1, *W = p->gm2;
    if (snapshots && n_snap > 0)
        if (int rc = cdr_download(p, p->u0, snapshots)) return rc;
    p->stat_launches = 0;
    const long max_launch = (long)cfg->max_iters + 1;
    for (long k = 1; k <= max_launch; ++k) {
        // every member still active is at sweep m = k - 1: u^m in buffer m & 1
        const double2* U = ((k - 1) & 1) ? p->u1 : p->u0;
        if (int rc = cdr_stencil(p, 3, U, p->f, R)) return rc;       // r = f - A u
        if (int rc = cdr_apply(p, 0, R, GR, nullptr)) return rc;      // G r (R_eta trace)
        const double2* D = GR;                                        // CBS
        if (cfg->format == BP_FMT_NPBS) {                             // G(V u + f) - u
            if (int rc = cdr_stencil(p, 4, U, p->f, X)) return rc;
            if (int rc = cdr_apply(p, 0, X, X, U)) return rc;
            D = X;
        }
        gen_norms_kernel<<<dim3(nchunk, B), 256, 0, p->stream>>>(g, c, R, GR, p->gpart, nchunk);
        gen_finalize_kernel<<<(B + 127) / 128, 128, 0, p->stream>>>(c, B, p->gpart, nchunk);
        if (map->metric == BP_METRIC_RETA) {  // w = x - G V x, gamma = <w, x> / <w, w>
            if (int rc = cdr_stencil(p, 1, D, nullptr, W)) return rc;
            if (int rc = cdr_apply(p, 0, W, W, nullptr)) return rc;
            gen_sub_kernel<<<grid_for(total), 256, 0, p->stream>>>(W, D, W, (long)total);
            gen_dot_kernel<<<dim3(nchunk, B), 256, 0, p->stream>>>(g, c, W, D, p->gpart, nchunk);
        } else {  // w = A x, gamma = <w, r> / <w, w>
            if (int rc = cdr_stencil(p, 0, D, nullptr, W)) return rc;
            gen_dot_kernel<<<dim3(nchunk, B), 256, 0, p->stream>>>(g, c, W, R, p->gpart, nchunk);
        }
        gen_gamma_kernel<<<(B + 127) / 128, 128, 0, p->stream>>>(c, B, p->gpart, nchunk, 1);
        gen_update_kernel<<<grid_for(total), 256, 0, p->stream>>>(g, c, p->u0, p->u1, D, 1);
        CU(cudaGetLastError());
        p->stat_launches += 16;
        if (snapshots && k < n_snap)
            if (int rc = cdr_download(p, (k & 1) ? p->u1 : p->u0, snapshots + nd * B * k)) return rc;
        if ((snapshots && n_snap > 0) || k % kGraphSweeps == 0 || k == max_launch) {
            CU(publish_int(p, c.n_active));
            CU(cudaStreamSynchronize(p->stream));
            if (*p->host_active == 0) break;
        }
    }
    return BP_OK;
}

// bp::run for the CDR family: sweep m = RC_A (entry m, u^{m+1}), RC_B (r^{m+1}, q^{m+1}, rows),
// CC_GREEN (columns); the first RC_B + CC_GREEN pair stages q^0.
int run_core_cdr(bp_problem* p, const bp_map* map, const bp_iter_config* cfg, bool have_u0,
                 double* snapshots, int n_snap) {
    const int B = p->batch;
    CdrArgs a = cdr_args(p);
    a.ctl.max_iters = cfg->max_iters;
    a.ctl.rtol = cfg->rtol;
    a.gamma = map->gamma_re;
    CdrArgs ac = a;
    ac.scale = 1.0 / (4.0 * (double)p->n * p->n);
    // fnorm_l2 = ||f||, fnorm_reta = ||G f||  (iterate.cpp:93,102)
    if (int rc = norms(p, p->f, p->fnorm_l2)) return rc;
    if (int rc = cdr_apply(p, 0, p->f, p->y, nullptr)) return rc;
    if (int rc = norms(p, p->y, p->fnorm_reta)) return rc;
    std::vector<double> fn(B);
    if (int rc = read_fnorm(p, fn)) return rc;
    for (int b = 0; b < B; ++b)
        if (!(fn[b] > 0.0)) return set_err(BP_EINVAL, "run: zero source");
    if (!have_u0) CU(cudaMemsetAsync(p->u0, 0, sizeof(double2) * p->alloc, p->stream));
    CU(cudaMemsetAsync(p->u1, 0, sizeof(double2) * p->alloc, p->stream));
    init_control_kernel<<<(B + 127) / 128, 128, 0, p->stream>>>(a.ctl, B);
    fill_nan_kernel<<<grid_for((size_t)B * p->trace_cap), 256, 0, p->stream>>>(p->trace_l2, (size_t)B * p->trace_cap);
    fill_nan_kernel<<<grid_for((size_t)B * p->trace_cap), 256, 0, p->stream>>>(p->trace_reta, (size_t)B * p->trace_cap);
    CU(cudaGetLastError());
    CU(launch_cdr(p->log2n, true, RC_B, a, p->stream));
    CU(cdr_green(p, ac));
    // norms 2x2, G 3, init_control, 2x fill_nan, RC_B + CC_GREEN
    p->stat_launches = 12;
    p->stat_row_ms = p->stat_col_ms = 0;
    p->stat_timed = 0;
    const long max_launch = (long)cfg->max_iters + 1;
    const size_t nd = p->field;  // real values per member
    auto sweep = [&](cudaEvent_t* ev) -> int {
        if (ev) CU(cudaEventRecord(ev[0], p->stream));
        CU(launch_cdr(p->log2n, true, RC_A, a, p->stream));
        CU(launch_cdr(p->log2n, true, RC_B, a, p->stream));
        if (ev) CU(cudaEventRecord(ev[1], p->stream));
        CU(cdr_green(p, ac));
        if (ev) CU(cudaEventRecord(ev[2], p->stream));
        return BP_OK;
    };
    auto poll = [&]() -> int {
        CU(publish_int(p, a.ctl.n_active));
        CU(cudaStreamSynchronize(p->stream));
        return BP_OK;
    };
    if (snapshots && n_snap > 0) {
        if (int rc = cdr_download(p, p->u0, snapshots)) return rc;
        for (long k = 1; k <= max_launch; ++k) {
            if (int rc = sweep(nullptr)) return rc;
            p->stat_launches += 3;
            if (k < n_snap)  // u^k in buffer k & 1
                if (int rc = cdr_download(p, (k & 1) ? p->u1 : p->u0, snapshots + nd * B * k)) return rc;
            if (int rc = poll()) return rc;
            if (*p->host_active == 0) break;
        }
        return BP_OK;
    }
    if (p->timing) {
        std::vector<cudaEvent_t> ev(3 * kGraphSweeps);
        for (auto& e : ev) CU(cudaEventCreate(&e));
        long launched = 0;
        int rc = BP_OK;
        while (launched < max_launch && rc == BP_OK) {
            for (int s = 0; s < kGraphSweeps && rc == BP_OK; ++s) rc = sweep(&ev[3 * s]);
            if (rc) break;
            launched += kGraphSweeps;
            p->stat_launches += 3 * kGraphSweeps;
            if ((rc = poll())) break;
            for (int s = 0; s < kGraphSweeps; ++s) {
                float r = 0, c = 0;
                cudaEventElapsedTime(&r, ev[3 * s], ev[3 * s + 1]);
                cudaEventElapsedTime(&c, ev[3 * s + 1], ev[3 * s + 2]);
                p->stat_row_ms += r;
                p->stat_col_ms += c;
                ++p->stat_timed;
            }
            if (*p->host_active == 0) break;
        }
        for (auto& e : ev) cudaEventDestroy(e);
        return rc;
    }
    // split-batch graphs as the Dirichlet path (run_core): parts replayed concurrently on their
    // own streams (BP_SPLIT=0 disables)
    const char* senv = std::getenv("BP_SPLIT");
    int split = (B >= 2 && !(senv && senv[0] == '0')) ? std::min(split_parts(B, p->log2n), B) : 0;
    // waves as run_core (BP_GROUP = members per wave; off by default for this family)
    const int group = split ? group_members(p, B) : 0;
    if (group) split = wave_parts(group);
    const int waves = group ? (B + group - 1) / group : 1;
    const bool reuse = p->graph && p->graph_split == split && p->graph_group == group &&
                       p->graph_map_kind == map->kind &&
                       p->graph_gamma.x == map->gamma_re && p->graph_max_iters == cfg->max_iters &&
                       p->graph_rtol == cfg->rtol;
    if (!reuse) {
        if (p->graph) cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
        for (auto& g2 : p->graph2) {
            if (g2) cudaGraphExecDestroy(g2);
            g2 = nullptr;
        }
        for (auto gw : p->gwave)
            if (gw) cudaGraphExecDestroy(gw);
        p->gwave.clear();
        cudaGraph_t g;
        if (!split) {
            CU(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
            for (int s = 0; s < kGraphSweeps; ++s) sweep(nullptr);
            CU(cudaStreamEndCapture(p->stream, &g));
            CU(cudaGraphInstantiate(&p->graph, g, 0));
            cudaGraphDestroy(g);
        } else {
            for (int k = 0; k < split; ++k) {
                if (k && !p->stream2[k - 1]) CU(cudaStreamCreateWithFlags(&p->stream2[k - 1], cudaStreamNonBlocking));
                if (!p->ev_join[k]) CU(cudaEventCreateWithFlags(&p->ev_join[k], cudaEventDisableTiming));
            }
            cudaStream_t keep = p->stream;
            p->gwave.assign((size_t)(waves - 1) * split, nullptr);
            for (int w = 0; w < waves; ++w) {
                const int w0 = group ? w * group : 0, w1 = group ? std::min(B, w0 + group) : B;
                for (int k = 0; k < split; ++k) {
                    const int b0 = w0 + (int)((long)(w1 - w0) * k / split), b1 = w0 + (int)((long)(w1 - w0) * (k + 1) / split);
                    cudaGraphExec_t* dst = w ? &p->gwave[(size_t)(w - 1) * split + k] : (k ? &p->graph2[k - 1] : &p->graph);
                    if (b1 == b0) continue;
                    const CdrArgs ak = cdr_args_range(a, p, b0, b1 - b0);
                    CdrArgs ack = cdr_args_range(ac, p, b0, b1 - b0);
                    p->stream = k ? p->stream2[k - 1] : keep;
                    cudaError_t e = cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal);
                    for (int sw = 0; e == cudaSuccess && sw < kGraphSweeps; ++sw) {
                        if (e == cudaSuccess) e = launch_cdr(p->log2n, true, RC_A, ak, p->stream);
                        if (e == cudaSuccess) e = launch_cdr(p->log2n, true, RC_B, ak, p->stream);
                        if (e == cudaSuccess) e = cdr_green(p, ack, b0);
                    }
                    cudaError_t e2 = cudaStreamEndCapture(p->stream, &g);
                    if (e == cudaSuccess) e = e2;
                    if (e == cudaSuccess) {
                        e = cudaGraphInstantiate(dst, g, 0);
                        cudaGraphDestroy(g);
                    }
                    p->stream = keep;
                    CU(e);
                }
            }
        }
        p->graph_split = split;
        p->graph_group = group;
        p->graph_map_kind = map->kind;
        p->graph_metric = map->metric;
        p->graph_gamma = make_double2(map->gamma_re, 0.0);
        p->graph_max_iters = cfg->max_iters;
        p->graph_rtol = cfg->rtol;
    }
    long launched = 0;
    if (split) {
        CU(cudaEventRecord(p->ev_join[0], p->stream));
        for (int k = 1; k < split; ++k) CU(cudaStreamWaitEvent(p->stream2[k - 1], p->ev_join[0], 0));
    }
    while (launched < max_launch) {
        for (int w = 0; w < waves; ++w) {
            for (int k = 0; k < std::max(split, 1); ++k) {
                cudaGraphExec_t ge = w ? p->gwave[(size_t)(w - 1) * split + k] : (k ? p->graph2[k - 1] : p->graph);
                if (ge) CU(cudaGraphLaunch(ge, k ? p->stream2[k - 1] : p->stream));
            }
        }
        for (int k = 1; k < split; ++k) {
            CU(cudaEventRecord(p->ev_join[k], p->stream2[k - 1]));
            CU(cudaStreamWaitEvent(p->stream, p->ev_join[k], 0));
        }
        launched += kGraphSweeps;
        p->stat_launches += 3 * kGraphSweeps * std::max(split, 1) * waves;
        if (int rc = poll()) return rc;
        if (*p->host_active == 0) break;
    }
    return BP_OK;
}

int finish_run_cdr(bp_problem* p, double* u_out, bool host_ptr) {
    Control c = make_control(p);
    // result_buf selects u0 / u1 per member; real fields copied as pairs
    select_copy_kernel<<<grid_for(p->field * p->batch / 2), 256, 0, p->stream>>>(
        p->u0, p->u1, c.result_buf, p->x, p->field / 2, p->batch);
    CU(cudaGetLastError());
    p->stat_launches += 1;
    return cdr_download(p, p->x, u_out, host_ptr);
}

int validate_run(const bp_problem* p, const bp_map* map, const bp_iter_config* cfg) {
    if (int rc = check_problem(p)) return rc;
    if (!map || !cfg) return set_err(BP_EINVAL, "run: null map or config");
    if (!(cfg->rtol > 0.0 && cfg->rtol < 1.0)) return set_err(BP_EINVAL, "run: rtol must lie in (0,1)");
    if (cfg->max_iters < 1) return set_err(BP_EINVAL, "run: max_iters must be >= 1");
    if (cfg->format != BP_FMT_NPBS && cfg->format != BP_FMT_CBS && cfg->format != BP_FMT_DIRECT)
        return set_err(BP_EINVAL, "run: unknown iteration format");
    if (cfg->format == BP_FMT_DIRECT && p->cdr)
        return set_err(BP_ENOTSUP, "run: the Direct format is implemented for the Helmholtz families "
                                   "(Dirichlet, periodic)");
    if (map->kind < BP_MAP_SCALAR || map->kind > BP_MAP_POINTWISE)
        return set_err(BP_EINVAL, "unknown correction map");
    if (map->kind == BP_MAP_FOURIER_DIAG && !map->m)
        return set_err(BP_EINVAL, "FourierDiag correction: shape mismatch");
    if (map->kind == BP_MAP_OPTIMAL_SCALAR && map->metric != BP_METRIC_EUCLIDEAN &&
        map->metric != BP_METRIC_RETA)
        return set_err(BP_EINVAL, "unknown optimal-scalar metric");
    if (p->cdr && !((map->kind == BP_MAP_SCALAR && map->gamma_im == 0.0) || map->kind == BP_MAP_OPTIMAL_SCALAR))
        return set_err(BP_ENOTSUP, "CDR family on the GPU (real fields): real scalar and optimal-scalar maps");
    if ((p->periodic || p->gper) && map->kind == BP_MAP_POINTWISE)
        return set_err(BP_ENOTSUP, "periodic family: the pointwise (i/eta) V map is defined for the "
                                   "Dirichlet family only");
    return BP_OK;
}

}  // namespace

extern "C" {

const char* bp_last_error(void) { return g_err.c_str(); }
int bp_abi_version(void) { return BP_ABI_VERSION; }

// for the host-side pipeline TU (pipeline.cpp): set this thread's bp_last_error() message
int bp_internal_set_error(int code, const char* msg) { return set_err(code, msg ? msg : ""); }
// for pipeline.cpp: hooks run around the sweeps of every later run on this handle (null: none)
int bp_internal_set_compute_hooks(bp_problem* p, void (*pre)(void*), void (*post)(void*), void* ctx) {
    if (int rc = check_problem(p)) return rc;
    if (pre && p->hook_pre)  // one pipeline per handle: a second one would mix the tickets
        return set_err(BP_EINVAL, "pipeline: the handle is already a slot of another pipeline");
    p->hook_pre = pre;
    p->hook_post = post;
    p->hook_ctx = ctx;
    return BP_OK;
}

}  // extern "C"

namespace {

// Shared constructor of the 2-D (dim 2) and 3-D (dim 3, cubic) Dirichlet Helmholtz batches.
// xi_j = 2 pi m_j / L with m_j in FFT order (wavenumbers_1d Periodic, grid.hpp:67-85)
std::vector<double> xi2_table(int n, double len) {
    std::vector<double> xi2(n);
    for (int i = 0; i < n; ++i) {
        const int m = (i < (n + 1) / 2) ? i : i - n;
        const double xi = 2.0 * kPi * m / len;
        xi2[i] = xi * xi;
    }
    return xi2;
}

int check_symbol_periodic(const std::vector<double>& xi2, int batch, const double* k0, const double* eta) {
    const double xmax = *std::max_element(xi2.begin(), xi2.end());
    const double xmin = *std::min_element(xi2.begin(), xi2.end());
    for (int b = 0; b < batch; ++b) {
        double mn = INFINITY, mx = 0.0;
        const double k0sq = k0[b] * k0[b];
        {
            const double mx0 = std::hypot(std::max(std::fabs((xmin + xmin) - k0sq), std::fabs((xmax + xmax) - k0sq)), eta[b]);
            if (std::fabs(eta[b]) >= kSymbolDivGuard * mx0 * (1.0 + 1e-12)) continue;  // see check_symbol
        }
        for (double a : xi2)
            for (double c : xi2) {
                const double v = std::hypot((a + c) - k0sq, -eta[b]);
                mn = std::min(mn, v);
                mx = std::max(mx, v);
            }
        if (mn < kSymbolDivGuard * mx)
            return set_err(BP_ERUNTIME, "symbol has a (near-)zero entry; reference operator not invertible");
    }
    return BP_OK;
}

// Any-shape 2-D Dirichlet handle (generic_kernels.cuh): nx, ny >= 1 up to 4095 each, any lx, ly.
// periodic: the reference's own HelmholtzProblem on any nx x ny <= 4096 (DFT lines, |xi|^2 symbol,
// pseudospectral A; helmholtz.cpp:11-53), scalar maps
int create_generic(const bp_grid* grid, int32_t batch, const double* k2, const double* k0, const double* eta,
                   int32_t device, bp_problem** out, bool periodic = false) {
    const int nx = grid->nx, ny = grid->ny;
    if (nx + (periodic ? 0 : 1) > 4096 || ny + (periodic ? 0 : 1) > 4096)
        return set_err(BP_ENOTSUP, periodic ? "GPU any-shape periodic path: nx, ny <= 4096"
                                            : "GPU any-shape path: nx, ny <= 4095 (power-of-two paths: nx+1 = ny+1 = 2^k <= 4096)");
    for (int b = 0; b < batch; ++b) {
        if (!(eta[b] > 0.0)) return set_err(BP_EINVAL, "HelmholtzProblem: eta must be > 0");
        if (!std::isfinite(k0[b])) return set_err(BP_EINVAL, "HelmholtzProblem: k0 not finite");
    }
    // Dirichlet: h = l/(n+1) (grid.hpp:12-24), DST-I factors; periodic: h = l/n, xi^2 (FFT order)
    const double hx = periodic ? grid->lx / nx : grid->lx / (nx + 1), hy = periodic ? grid->ly / ny : grid->ly / (ny + 1);
    const std::vector<double> ax = periodic ? xi2_table(nx, grid->lx) : gen_lap(nx, hx);
    const std::vector<double> ay = periodic ? xi2_table(ny, grid->ly) : gen_lap(ny, hy);
    if (int rc = check_symbol_generic(ax, ay, batch, k0, eta)) return rc;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return set_err(BP_ECUDA, "no such CUDA device");
    DeviceGuard guard(device);
    auto* p = new bp_problem();
    p->grid = *grid;
    p->batch = batch;
    p->device = device;
    p->dim = 2;
    p->generic = true;
    p->gper = periodic;
    p->gnx = nx;
    p->gny = ny;
    p->field = (size_t)nx * ny;
    p->alloc = p->field * batch;
    p->dense_pts = p->field;
    p->inv_h2 = 1.0 / (hx * hx);  // five_point's single h2 = hx^2 (newton_problem.cpp:41)
    auto fail = [&](int code) {
        bp_problem_destroy(p);
        return code;
    };
#define CUF(call)                                                                                   \
    do {                                                                                            \
        cudaError_t _e = (call);                                                                    \
        if (_e != cudaSuccess) return fail(set_err(BP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e))); \
    } while (0)
    CUF(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    const size_t fb = sizeof(double2) * p->alloc;
    for (double2** buf : {&p->k2, &p->f, &p->u0, &p->u1, &p->T, &p->x, &p->y, &p->dense}) {
        CUF(cudaMalloc(buf, fb));
        CUF(cudaMemsetAsync(*buf, 0, fb, p->stream));
    }
    CUF(cudaMalloc(&p->gamma, sizeof(double2) * (size_t)batch));
    CUF(cudaMalloc(&p->norm_part, sizeof(double) * (size_t)batch * 64));
    CUF(cudaMalloc(&p->gpart, sizeof(double) * (size_t)batch * 64 * 4));
    CUF(cudaMalloc(&p->fnorm_l2, sizeof(double) * batch));
    CUF(cudaMalloc(&p->fnorm_reta, sizeof(double) * batch));
    CUF(cudaMalloc(&p->ctl_int, sizeof(int) * (5 * (size_t)batch + 1)));
    CUF(cudaMalloc(&p->counter, sizeof(unsigned) * batch));
    CUF(cudaMallocHost(&p->host_active, sizeof(int)));
    CUF(cudaMalloc(&p->dflag, sizeof(int)));
    CUF(cudaMalloc(&p->k0sq, sizeof(double) * batch));
    CUF(cudaMalloc(&p->eta, sizeof(double) * batch));
    CUF(cudaMalloc(&p->gax, sizeof(double) * nx));
    CUF(cudaMalloc(&p->gay, sizeof(double) * ny));
    CUF(cudaMemcpyAsync(p->gax, ax.data(), sizeof(double) * nx, cudaMemcpyHostToDevice, p->stream));
    CUF(cudaMemcpyAsync(p->gay, ay.data(), sizeof(double) * ny, cudaMemcpyHostToDevice, p->stream));
    if (int rc = make_gplan(periodic ? nx : nx + 1, p->gplan_x)) return fail(rc);
    if (int rc = make_gplan(periodic ? ny : ny + 1, p->gplan_y)) return fail(rc);
    std::vector<double> k0sq(batch);
    for (int b = 0; b < batch; ++b) k0sq[b] = k0[b] * k0[b];
    CUF(cudaMemcpyAsync(p->k0sq, k0sq.data(), sizeof(double) * batch, cudaMemcpyHostToDevice, p->stream));
    CUF(cudaMemcpyAsync(p->eta, eta, sizeof(double) * batch, cudaMemcpyHostToDevice, p->stream));
    if (int rc = upload_k2_checked(p, k2)) return fail(rc);
    CUF(cudaStreamSynchronize(p->stream));
    if (int rc = ensure_trace(p, 1000)) return fail(rc);
#undef CUF
    *out = p;
    return BP_OK;
}

int create_impl(const bp_grid* grid, int dim, int32_t batch, const double* k2, const double* k0,
                const double* eta, int32_t device, bp_problem** out, bool periodic = false) {
    // Dirichlet: n = nx + 1 cells (interior nx); periodic: n = nx nodes (helmholtz.cpp:11-25)
    const int n = periodic ? grid->nx : grid->nx + 1;
    int log2n = 0;
    while ((1 << log2n) < n) ++log2n;
    const int max_log2 = dim == 3 ? kMaxLog2_3d : kMaxLog2;
    if (dim == 2 &&
        (grid->nx != grid->ny || (1 << log2n) != n || log2n < kMinLog2 || log2n > max_log2 || grid->lx != grid->ly))
        return create_generic(grid, batch, k2, k0, eta, device, out, periodic);
    if (grid->nx != grid->ny || (1 << log2n) != n || log2n < kMinLog2 || log2n > max_log2)
        return set_err(BP_ENOTSUP, periodic ? "GPU periodic path needs square grids with nx = 2^k, 8 <= 2^k <= 4096"
                                   : dim == 3 ? "GPU path needs cubic grids with n+1 = 2^k, 8 <= 2^k <= 512"
                                              : "GPU path needs square grids with nx+1 = 2^k, 8 <= 2^k <= 4096");
    if (grid->lx != grid->ly) return set_err(BP_ENOTSUP, "GPU path needs lx == ly (hx == hy)");
    size_t nd = (size_t)grid->nx * grid->ny;
    if (dim == 3) nd *= grid->nx;
    for (int b = 0; b < batch; ++b) {
        if (!(eta[b] > 0.0)) return set_err(BP_EINVAL, "HelmholtzProblem: eta must be > 0");
        if (!std::isfinite(k0[b])) return set_err(BP_EINVAL, "HelmholtzProblem: k0 not finite");
    }

    const std::vector<double> xi2 = xi2_table(n, grid->lx);
    if (periodic) {
        if (int rc = check_symbol_periodic(xi2, batch, k0, eta)) return rc;
    } else if (int rc = check_symbol(*grid, dim, batch, k0, eta)) {
        return rc;
    }
    const double h = grid->lx / n;
    std::vector<double> lap = lap_table(n, h);

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return set_err(BP_ECUDA, "no such CUDA device");
    DeviceGuard guard(device);
    auto* p = new bp_problem();
    p->grid = *grid;
    p->batch = batch;
    p->device = device;
    p->log2n = log2n;
    p->n = n;
    p->dim = dim;
    p->periodic = periodic;
    p->field = (size_t)1 << (dim * log2n);
    p->alloc = p->field * batch + ((size_t)1 << ((dim - 1) * log2n));
    p->dense_pts = nd;
    p->inv_h2 = 1.0 / (h * h);
    // 2/(n_i+1) per dimension (proj/src/transforms.cpp:99) divided by the gain of the 2*dim
    // engine passes of a Green application (kEngineGain^(2 dim), exact)
    p->green_scale = std::pow(2.0 / n, dim) / std::pow(kEngineGain, 2 * dim);
    auto fail = [&](int code) {
        bp_problem_destroy(p);
        return code;
    };
#define CUF(call)                                                                                   \
    do {                                                                                            \
        cudaError_t _e = (call);                                                                    \
        if (_e != cudaSuccess) return fail(set_err(BP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e))); \
    } while (0)
    CUF(prepare_kernels(log2n, dim));
    CUF(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    const size_t fb = sizeof(double2) * p->alloc;
    CUF(cudaMalloc(&p->k2, fb));
    CUF(cudaMalloc(&p->f, fb));
    CUF(cudaMalloc(&p->u0, fb));
    CUF(cudaMalloc(&p->u1, fb));
    CUF(cudaMalloc(&p->T, fb));
    CUF(cudaMalloc(&p->x, fb));
    CUF(cudaMalloc(&p->y, fb));
    for (double2* buf : {p->k2, p->f, p->u0, p->u1, p->T, p->x, p->y})
        CUF(cudaMemsetAsync(buf, 0, fb, p->stream));
    CUF(cudaMalloc(&p->dense, sizeof(double2) * nd * batch));
    CUF(cudaMalloc(&p->partial, sizeof(double) * (size_t)batch * ((size_t)1 << ((dim - 1) * log2n)) *
                                    kPartStride));
    CUF(cudaMalloc(&p->gamma, sizeof(double2) * (size_t)batch));
    CUF(cudaMalloc(&p->fd, sizeof(double2) * p->field));
    CUF(cudaMalloc(&p->norm_part, sizeof(double) * (size_t)batch * 64));
    CUF(cudaMalloc(&p->fnorm_l2, sizeof(double) * batch));
    CUF(cudaMalloc(&p->fnorm_reta, sizeof(double) * batch));
    CUF(cudaMalloc(&p->ctl_int, sizeof(int) * (5 * (size_t)batch + 1)));
    CUF(cudaMalloc(&p->counter, sizeof(unsigned) * batch));
    CUF(cudaMallocHost(&p->host_active, sizeof(int)));
    CUF(cudaMalloc(&p->dflag, sizeof(int)));
    CUF(cudaMalloc(&p->k0sq, sizeof(double) * batch));
    CUF(cudaMalloc(&p->eta, sizeof(double) * batch));
    CUF(cudaMalloc(&p->tw, sizeof(double2) * n));
    CUF(cudaMalloc(&p->sinp, sizeof(double) * n));
    CUF(cudaMalloc(&p->lap, sizeof(double) * n));
    CUF(cudaMalloc(&p->xi2, sizeof(double) * n));
    CUF(cudaMemcpyAsync(p->xi2, xi2.data(), sizeof(double) * n, cudaMemcpyHostToDevice, p->stream));
    std::vector<double> k0sq(batch), tw(2 * n), sinp(n);
    for (int b = 0; b < batch; ++b) k0sq[b] = k0[b] * k0[b];
    for (int k = 0; k < n; ++k) {
        tw[2 * k] = std::cos(2.0 * kPi * k / n);
        tw[2 * k + 1] = -std::sin(2.0 * kPi * k / n);
        sinp[k] = kSinScale * std::sin(kPi * k / n);
    }
    CUF(cudaMemcpyAsync(p->k0sq, k0sq.data(), sizeof(double) * batch, cudaMemcpyHostToDevice, p->stream));
    CUF(cudaMemcpyAsync(p->eta, eta, sizeof(double) * batch, cudaMemcpyHostToDevice, p->stream));
    CUF(cudaMemcpyAsync(p->tw, tw.data(), sizeof(double2) * n, cudaMemcpyHostToDevice, p->stream));
    CUF(cudaMemcpyAsync(p->sinp, sinp.data(), sizeof(double) * n, cudaMemcpyHostToDevice, p->stream));
    CUF(cudaMemcpyAsync(p->lap, lap.data(), sizeof(double) * n, cudaMemcpyHostToDevice, p->stream));
    {
        // Green column pass: tridiagonal x-solve for the Dirichlet family, n >= 64 (2-D columns,
        // 3-D x-lines; BP_COL_DST=1 keeps the transform route)
        const char* e = std::getenv("BP_COL_DST");
        if (!periodic && log2n >= 6 && !(e && e[0] == '1')) {
            const size_t lines = (size_t)batch << ((dim - 1) * log2n);
            CUF(cudaMalloc(&p->tri, sizeof(double2) * lines * (kTriP + n / kTriP)));
            p->tri_scale = 8.0 * n * h * h * p->green_scale;
            if (int rc = build_tri(p)) return fail(rc);
        }
    }
    if (int rc = upload_k2_checked(p, k2)) return fail(rc);
    CUF(cudaStreamSynchronize(p->stream));
    if (int rc = ensure_trace(p, 1000)) return fail(rc);
#undef CUF
    *out = p;
    return BP_OK;
}

// Config c4 handle: Neumann cell-centred n x n (h = lx/n), L0 = -Lap_N + sigma0 diagonalised by
// DCT-II (symbol.cpp:81-92), V = (sigma0 - sigma) - b . grad_upwind.  Real fields.
int check_cdr_medium(const bp_problem* p, const double* bx, const double* by, const double* sigma,
                     const double* sigma0) {
    const double h = p->grid.lx / p->n;
    std::vector<double> lapn(p->n);
    for (int k = 0; k < p->n; ++k) {
        const double s = std::sin(k * kPi / (2.0 * p->n));
        lapn[k] = 4.0 / (h * h) * s * s;
    }
    for (int b = 0; b < p->batch; ++b) {
        const double s0 = sigma0[b];
        if (!std::isfinite(s0)) return set_err(BP_EINVAL, "CDR: sigma0 not finite");
        // apply_symbol's guard (symbol.cpp:23-31) over lambda_pq = a_p + a_q + sigma0; the a_k
        // are non-negative and increasing, so sigma0 >= 0 puts the extremes at the corners
        double mn, mx;
        if (s0 >= 0.0) {
            mn = s0;
            mx = 2.0 * lapn[p->n - 1] + s0;
        } else {
            mn = INFINITY;
            mx = 0.0;
            for (int i = 0; i < p->n; ++i)
                for (int j = 0; j < p->n; ++j) {
                    const double v = std::fabs(lapn[i] + lapn[j] + s0);
                    mn = std::min(mn, v);
                    mx = std::max(mx, v);
                }
        }
        if (mn < kSymbolDivGuard * mx)
            return set_err(BP_ERUNTIME, "symbol has a (near-)zero entry; reference operator not invertible");
    }
    return BP_OK;
}

int upload_cdr_medium(bp_problem* p, const double* bx, const double* by, const double* sigma,
                      const double* sigma0) {
    // staged through the scratch fields (T, x, y) and validated there, so a rejected medium
    // leaves the handle's current one intact
    const size_t n = p->field * p->batch, bytes = sizeof(double) * n;
    double* st[3] = {reinterpret_cast<double*>(p->T), reinterpret_cast<double*>(p->x),
                     reinterpret_cast<double*>(p->y)};
    const double* src[3] = {bx, by, sigma};
    double* dst[3] = {p->bx, p->by, p->sigma};
    for (int i = 0; i < 3; ++i)
        CU(cudaMemcpyAsync(st[i], src[i], bytes, cudaMemcpyHostToDevice, p->stream));
    bool ok = true;
    for (int i = 0; i < 3 && ok; ++i)
        if (int rc = all_finite(p, st[i], n, &ok)) return rc;
    if (!ok) return set_err(BP_EINVAL, "CDR medium not finite");
    for (int i = 0; i < 3; ++i)
        CU(cudaMemcpyAsync(dst[i], st[i], bytes, cudaMemcpyDeviceToDevice, p->stream));
    CU(cudaMemcpyAsync(p->sigma0, sigma0, sizeof(double) * p->batch, cudaMemcpyHostToDevice, p->stream));
    if (int rc = build_tri(p)) return rc;
    CU(cudaStreamSynchronize(p->stream));
    return BP_OK;
}

int create_cdr_impl(const bp_grid* grid, int32_t batch, const double* bx, const double* by,
                    const double* sigma, const double* sigma0, int32_t device, bp_problem** out) {
    const int n = grid->nx;
    int log2n = 0;
    while ((1 << log2n) < n) ++log2n;
    if (grid->nx != grid->ny || (1 << log2n) != n || log2n < kMinLog2 || log2n > kMaxLog2)
        return set_err(BP_ENOTSUP, "GPU CDR path needs square Neumann grids with nx = 2^k, 8 <= 2^k <= 4096");
    if (grid->lx != grid->ly) return set_err(BP_ENOTSUP, "GPU path needs lx == ly (hx == hy)");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return set_err(BP_ECUDA, "no such CUDA device");
    DeviceGuard guard(device);
    auto* p = new bp_problem();
    p->grid = *grid;
    p->batch = batch;
    p->device = device;
    p->log2n = log2n;
    p->n = n;
    p->dim = 2;
    p->cdr = true;
    p->field = (size_t)n * n;
    p->alloc = p->field * batch / 2;  // in double2 units (real fields)
    p->dense_pts = p->field;
    auto fail = [&](int code) {
        bp_problem_destroy(p);
        return code;
    };
    if (int rc = check_cdr_medium(p, bx, by, sigma, sigma0)) return fail(rc);
#define CUF(call)                                                                                   \
    do {                                                                                            \
        cudaError_t _e = (call);                                                                    \
        if (_e != cudaSuccess) return fail(set_err(BP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e))); \
    } while (0)
    CUF(prepare_kernels(log2n, 2));
    CUF(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    const size_t fb = sizeof(double) * p->field * batch;
    for (double2** buf : {&p->f, &p->u0, &p->u1, &p->T, &p->x, &p->y}) {
        CUF(cudaMalloc(buf, fb));
        CUF(cudaMemsetAsync(*buf, 0, fb, p->stream));
    }
    for (double** buf : {&p->bx, &p->by, &p->sigma}) CUF(cudaMalloc(buf, fb));
    CUF(cudaMalloc(&p->sigma0, sizeof(double) * batch));
    CUF(cudaMalloc(&p->rnorm2, sizeof(double) * batch));
    CUF(cudaMalloc(&p->partial, sizeof(double) * (size_t)batch * n * kPartStride));
    CUF(cudaMalloc(&p->gamma, sizeof(double2) * (size_t)batch));
    CUF(cudaMalloc(&p->norm_part, sizeof(double) * (size_t)batch * 64));
    CUF(cudaMalloc(&p->fnorm_l2, sizeof(double) * batch));
    CUF(cudaMalloc(&p->fnorm_reta, sizeof(double) * batch));
    CUF(cudaMalloc(&p->ctl_int, sizeof(int) * (5 * (size_t)batch + 1)));
    CUF(cudaMalloc(&p->counter, sizeof(unsigned) * batch));
    CUF(cudaMemsetAsync(p->counter, 0, sizeof(unsigned) * batch, p->stream));
    CUF(cudaMallocHost(&p->host_active, sizeof(int)));
    CUF(cudaMalloc(&p->dflag, sizeof(int)));
    CUF(cudaMalloc(&p->tw, sizeof(double2) * n));
    CUF(cudaMalloc(&p->w4, sizeof(double2) * n));
    CUF(cudaMalloc(&p->lapn, sizeof(double) * n));
    const double h = grid->lx / n;
    std::vector<double> tw(2 * n), w4(2 * n), lapn(n);
    for (int k = 0; k < n; ++k) {
        tw[2 * k] = std::cos(2.0 * kPi * k / n);
        tw[2 * k + 1] = -std::sin(2.0 * kPi * k / n);
        w4[2 * k] = std::cos(kPi * k / (2.0 * n));
        w4[2 * k + 1] = -std::sin(kPi * k / (2.0 * n));
        const double s = std::sin(k * kPi / (2.0 * n));
        lapn[k] = 4.0 / (h * h) * s * s;  // symbol.cpp:81-92 (per axis)
    }
    CUF(cudaMemcpyAsync(p->tw, tw.data(), sizeof(double2) * n, cudaMemcpyHostToDevice, p->stream));
    CUF(cudaMemcpyAsync(p->w4, w4.data(), sizeof(double2) * n, cudaMemcpyHostToDevice, p->stream));
    CUF(cudaMemcpyAsync(p->lapn, lapn.data(), sizeof(double) * n, cudaMemcpyHostToDevice, p->stream));
    {
        // Green column pass: the Neumann tridiagonal x-solve on real column pairs, n >= 128
        // (BP_COL_DST=1 keeps the DCT route); tables built by upload_cdr_medium
        const char* e = std::getenv("BP_COL_DST");
        if (log2n >= 7 && !(e && e[0] == '1')) {
            CUF(cudaMalloc(&p->tri, sizeof(double2) * (size_t)batch * (n / 2) * (2 * kTriP + n / kTriP)));
            CUF(launch_tri(log2n, CL_CDR, ColArgs{}, nullptr, true));
        }
    }
    if (int rc = upload_cdr_medium(p, bx, by, sigma, sigma0)) return fail(rc);
    if (int rc = ensure_trace(p, 1000)) return fail(rc);
#undef CUF
    *out = p;
    return BP_OK;
}


// ------------------------------------------------------------------ slab decomposition (host)
// One rank's x-slab of a distributed 2-D Dirichlet grid (config c2 across GPUs, SURVEY.md
// 8(e)).  The driver (paper_2603_18527_b200/slab.py) sequences the stages below with the
// collectives between them: all-to-all of the blocked row-side T (t_rows) into the column-side
// block (t_cols) and back, the u halo-row exchange, and the all-reduce of the two trace sums.

// entry != 0: trace entry m + termination test from sums[0..1]; gamma_off >= 0: the
// optimal-scalar gamma (correction.cpp:10-18) from sums[gamma_off .. gamma_off + 2]
__global__ void slab_finalize_kernel(Control c, const double* sums, int entry, int gamma_off) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && c.status[0] == ST_ACTIVE) {
        if (gamma_off >= 0) finalize_gamma(c, 0, sums[gamma_off], sums[gamma_off + 1], sums[gamma_off + 2]);
        if (entry) finalize_entry(c, 0, c.sweep[0], sums[0], sums[1]);
    }
}

// dense reference rows (nx*ny interior, x slow) -> padded slab rows [row0, row0 + R) (host)
// dense reference layout -> the rank's padded rows (2-D: [R][n]) / x-planes (3-D: [R][n][n])
void pack_slab_host(const double* dense, int n, int row0, int R, std::vector<double2>& out, int dim = 2) {
    const size_t line = dim == 3 ? (size_t)n * n : (size_t)n;
    out.assign((size_t)R * line, make_double2(0.0, 0.0));
    const int nd = n - 1;
    for (int i = 0; i < R; ++i) {
        const int x = row0 + i;
        if (x < 1 || x > nd) continue;
        if (dim == 2) {
            const double* src = dense + 2 * (size_t)(x - 1) * nd;
            for (int y = 1; y < n; ++y) out[(size_t)i * n + y] = make_double2(src[2 * (y - 1)], src[2 * (y - 1) + 1]);
            continue;
        }
        for (int y = 1; y < n; ++y) {
            const double* src = dense + 2 * ((size_t)(x - 1) * nd + (y - 1)) * nd;
            double2* dst = out.data() + ((size_t)i * n + y) * n;
            for (int z = 1; z < n; ++z) dst[z] = make_double2(src[2 * (z - 1)], src[2 * (z - 1) + 1]);
        }
    }
}

// inverse of pack_slab_host for the rank's own rows / planes
void unpack_slab_host(const std::vector<double2>& rows, int n, int row0, int R, double* dense, int dim) {
    const int nd = n - 1;
    for (int i = 0; i < R; ++i) {
        const int x = row0 + i;
        if (x < 1 || x > nd) continue;
        if (dim == 2) {
            double* dst = dense + 2 * (size_t)(x - 1) * nd;
            for (int y = 1; y < n; ++y) {
                dst[2 * (y - 1)] = rows[(size_t)i * n + y].x;
                dst[2 * (y - 1) + 1] = rows[(size_t)i * n + y].y;
            }
            continue;
        }
        for (int y = 1; y < n; ++y) {
            double* dst = dense + 2 * ((size_t)(x - 1) * nd + (y - 1)) * nd;
            const double2* src = rows.data() + ((size_t)i * n + y) * n;
            for (int z = 1; z < n; ++z) {
                dst[2 * (z - 1)] = src[z].x;
                dst[2 * (z - 1) + 1] = src[z].y;
            }
        }
    }
}

size_t slab_halo(const bp_problem* p) { return p->dim == 3 ? (size_t)p->n * p->n : (size_t)p->n; }

// 3-D slabs: the local y-lines of the rank's x-planes in the dest-blocked T layout (CL_YBLK);
// forward = the launch before the exchange (fused: stores into the peers' t_cols)
int slab_ylines(bp_problem* p, const Control& ctl, bool forward = false) {
    ColArgs c = col_args(p);
    c.T = p->T;
    c.batch = 1;
    c.slab_log2 = p->slab_log2;
    c.scale = 1.0;
    c.status = p->slab_running ? ctl.status : nullptr;
    if (forward && p->xchg_on) {
        c.xchg_on = 1;
        c.xchg_rank = p->slab_rank;
        for (int r = 0; r < p->slab_nranks; ++r) c.xchg[r] = p->xchg_cols[r];
    }
    CU(launch_col_pp(p->log2n, 16, CL_YBLK, C_ONE, c, p->stream));
    return BP_OK;
}

RowArgs slab_row_args(const bp_problem* p) {
    RowArgs a = row_args(p);
    a.slab_log2 = p->slab_log2;
    a.row0 = p->row0;
    a.slab_sums = p->slab_sums;
    a.direct = p->slab_direct ? 1 : 0;
    if (p->xchg_on && p->dim == 2) {  // 2-D: the row kernel's forward stores are the exchange
        a.xchg_on = 1;
        a.xchg_rank = p->slab_rank;
        for (int r = 0; r < p->slab_nranks; ++r) a.xchg[r] = p->xchg_cols[r];
    }
    return a;
}

}  // namespace

extern "C" {

int bp_problem_set_stream(bp_problem* p, void* stream) {
    if (int rc = check_problem(p)) return rc;
    DeviceGuard guard(p->device);
    CU(cudaStreamSynchronize(p->stream));
    if (p->own_stream) CU(cudaStreamDestroy(p->stream));
    p->stream = (cudaStream_t)stream;
    p->own_stream = false;
    return BP_OK;
}

static int slab_create_impl(const bp_grid* grid, int dim, int32_t rank, int32_t nranks, const double* k2,
                            double k0, double eta, int32_t device, bp_problem** out) {
    if (!out) return set_err(BP_EINVAL, "null output handle");
    *out = nullptr;
    if (!grid || !k2) return set_err(BP_EINVAL, "null argument");
    if (grid->bc != BP_BC_DIRICHLET) return set_err(BP_ENOTSUP, "slab decomposition: Dirichlet grids only");
    if (nranks < 1 || (nranks & (nranks - 1)) || rank < 0 || rank >= nranks)
        return set_err(BP_EINVAL, "slab decomposition: nranks must be a power of two, 0 <= rank < nranks");
    const int n = grid->nx + 1;
    int log2n = 0;
    while ((1 << log2n) < n) ++log2n;
    if (grid->nx != grid->ny || (1 << log2n) != n || log2n < kMinLog2 || log2n > (dim == 3 ? kMaxLog2_3d : kMaxLog2))
        return set_err(BP_ENOTSUP, dim == 3 ? "GPU 3-D path needs cubic grids with n+1 = 2^k, 8 <= 2^k <= 512"
                                            : "GPU path needs square grids with nx+1 = 2^k, 8 <= 2^k <= 4096");
    if (grid->lx != grid->ly) return set_err(BP_ENOTSUP, "GPU path needs lx == ly (hx == hy)");
    const int R = n / nranks;
    if (R < 8) return set_err(BP_ENOTSUP, "slab decomposition: at least 8 rows per rank");
    if (!(eta > 0.0)) return set_err(BP_EINVAL, "HelmholtzProblem: eta must be > 0");
    if (!std::isfinite(k0)) return set_err(BP_EINVAL, "HelmholtzProblem: k0 not finite");
    if (int rc = check_symbol(*grid, dim, 1, &k0, &eta)) return rc;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return set_err(BP_ECUDA, "no such CUDA device");
    DeviceGuard guard(device);
    auto* p = new bp_problem();
    p->grid = *grid;
    p->batch = 1;
    p->device = device;
    p->log2n = log2n;
    p->n = n;
    p->dim = dim;
    p->slab_nranks = nranks;
    p->slab_rank = rank;
    p->slab_log2 = 0;
    while ((1 << p->slab_log2) < R) ++p->slab_log2;
    p->row0 = rank * R;
    const size_t halo = dim == 3 ? (size_t)n * n : (size_t)n;  // one row / x-plane
    p->field = (size_t)R * halo;
    p->alloc = p->field;
    p->dense_pts = (size_t)grid->nx * grid->ny * (dim == 3 ? grid->nx : 1);
    const double h = grid->lx / n;
    p->inv_h2 = 1.0 / (h * h);
    p->green_scale = std::pow(2.0 / n, dim) / std::pow(kEngineGain, 2 * dim);
    auto fail = [&](int code) {
        bp_problem_destroy(p);
        return code;
    };
#define CUF(call)                                                                                   \
    do {                                                                                            \
        cudaError_t _e = (call);                                                                    \
        if (_e != cudaSuccess) return fail(set_err(BP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e))); \
    } while (0)
    CUF(prepare_kernels(log2n, dim));
    {
        ColArgs c{};
        CUF(launch_col_pp(log2n, 16, CL_SLAB, C_GREEN, c, nullptr, true));
        CUF(launch_col_pp(log2n, 16, CL_SLAB, C_ONE, c, nullptr, true));
        CUF(launch_col_pp(log2n, 16, CL_SLAB, C_FD, c, nullptr, true));
        CUF(launch_col_pp(log2n, 16, CL_SLAB, C_LREF, c, nullptr, true));
        if (dim == 3) CUF(launch_col_pp(log2n, 16, CL_YBLK, C_ONE, c, nullptr, true));
        if (log2n >= 6) CUF(launch_tri(log2n, CL_SLAB, c, nullptr, true));
    }
    CUF(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    const size_t fb = sizeof(double2) * p->field, ub = sizeof(double2) * (p->field + 2 * halo);
    for (double2** buf : {&p->k2, &p->f, &p->T, &p->Tc, &p->x, &p->y}) {
        CUF(cudaMalloc(buf, fb));
        CUF(cudaMemsetAsync(*buf, 0, fb, p->stream));
    }
    for (double2** buf : {&p->u_alloc0, &p->u_alloc1}) {
        CUF(cudaMalloc(buf, ub));
        CUF(cudaMemsetAsync(*buf, 0, ub, p->stream));
    }
    p->u0 = p->u_alloc0 + halo;
    p->u1 = p->u_alloc1 + halo;
    CUF(cudaMalloc(&p->slab_sums, sizeof(double) * 8));
    CUF(cudaMemsetAsync(p->slab_sums, 0, sizeof(double) * 8, p->stream));
    CUF(cudaMalloc(&p->partial, sizeof(double) * (size_t)R * (dim == 3 ? n : 1) * kPartStride));
    CUF(cudaMalloc(&p->gamma, sizeof(double2)));
    CUF(cudaMalloc(&p->norm_part, sizeof(double) * 64));
    CUF(cudaMalloc(&p->fnorm_l2, sizeof(double)));
    CUF(cudaMalloc(&p->fnorm_reta, sizeof(double)));
    CUF(cudaMalloc(&p->ctl_int, sizeof(int) * 6));
    CUF(cudaMemsetAsync(p->ctl_int, 0, sizeof(int) * 6, p->stream));
    CUF(cudaMalloc(&p->counter, sizeof(unsigned)));
    CUF(cudaMemsetAsync(p->counter, 0, sizeof(unsigned), p->stream));
    CUF(cudaMallocHost(&p->host_active, sizeof(int)));
    CUF(cudaMalloc(&p->dflag, sizeof(int)));
    CUF(cudaMalloc(&p->k0sq, sizeof(double)));
    CUF(cudaMalloc(&p->eta, sizeof(double)));
    CUF(cudaMalloc(&p->tw, sizeof(double2) * n));
    CUF(cudaMalloc(&p->sinp, sizeof(double) * n));
    CUF(cudaMalloc(&p->lap, sizeof(double) * n));
    std::vector<double> lap = lap_table(n, h), tw(2 * n), sinp(n);
    for (int k = 0; k < n; ++k) {
        tw[2 * k] = std::cos(2.0 * kPi * k / n);
        tw[2 * k + 1] = -std::sin(2.0 * kPi * k / n);
        sinp[k] = kSinScale * std::sin(kPi * k / n);
    }
    const double k0sq = k0 * k0;
    CUF(cudaMemcpyAsync(p->k0sq, &k0sq, sizeof(double), cudaMemcpyHostToDevice, p->stream));
    CUF(cudaMemcpyAsync(p->eta, &eta, sizeof(double), cudaMemcpyHostToDevice, p->stream));
    CUF(cudaMemcpyAsync(p->tw, tw.data(), sizeof(double2) * n, cudaMemcpyHostToDevice, p->stream));
    CUF(cudaMemcpyAsync(p->sinp, sinp.data(), sizeof(double) * n, cudaMemcpyHostToDevice, p->stream));
    CUF(cudaMemcpyAsync(p->lap, lap.data(), sizeof(double) * n, cudaMemcpyHostToDevice, p->stream));
    {
        // Green column pass on the rank's column block: tridiagonal x-solve (as create_impl)
        const char* e = std::getenv("BP_COL_DST");
        if (log2n >= 6 && !(e && e[0] == '1')) {
            const size_t lines = (size_t)1 << ((dim - 1) * log2n);
            CUF(cudaMalloc(&p->tri, sizeof(double2) * lines * (kTriP + n / kTriP)));
            p->tri_scale = 8.0 * n * h * h * p->green_scale;
            if (int rc = build_tri(p)) return fail(rc);
        }
    }
    std::vector<double2> rows;
    pack_slab_host(k2, n, p->row0, R, rows, dim);
    CUF(cudaMemcpyAsync(p->k2, rows.data(), fb, cudaMemcpyHostToDevice, p->stream));
    bool ok = false;
    if (int rc = all_finite(p, reinterpret_cast<const double*>(p->k2), 2 * p->field, &ok)) return fail(rc);
    if (!ok) return fail(set_err(BP_EINVAL, "HelmholtzProblem: k2 not finite"));
    if (int rc = ensure_trace(p, 1000)) return fail(rc);
#undef CUF
    *out = p;
    return BP_OK;
}

int bp_slab_create(const bp_grid* grid, int32_t rank, int32_t nranks, const double* k2, double k0,
                   double eta, int32_t device, bp_problem** out) {
    return slab_create_impl(grid, 2, rank, nranks, k2, k0, eta, device, out);
}

int bp_slab_create3d(const bp_grid3* grid, int32_t rank, int32_t nranks, const double* k2, double k0,
                     double eta, int32_t device, bp_problem** out) {
    if (!out) return set_err(BP_EINVAL, "null output handle");
    *out = nullptr;
    if (!grid || !k2) return set_err(BP_EINVAL, "null argument");
    if (grid->nx < 2 || grid->ny < 2 || grid->nz < 2) return set_err(BP_EINVAL, "GridSpec: nx,ny,nz must be >= 2");
    if (grid->nz != grid->nx || grid->lz != grid->lx)
        return set_err(BP_ENOTSUP, "GPU 3-D path needs cubic grids (hx == hy == hz)");
    const bp_grid g2{grid->nx, grid->ny, grid->lx, grid->ly, grid->bc};
    return slab_create_impl(&g2, 3, rank, nranks, k2, k0, eta, device, out);
}

int bp_slab_view(const bp_problem* p, bp_slab_view_t* v) {
    if (int rc = check_problem(p)) return rc;
    if (!p->slab_log2 || !v) return set_err(BP_EINVAL, "not a slab problem");
    const int n = p->n, R = 1 << p->slab_log2;
    v->rank = p->slab_rank;
    v->nranks = p->slab_nranks;
    v->rows = R;
    v->row0 = p->row0;
    v->n = n;
    const size_t halo = slab_halo(p);
    v->block_elems = (int64_t)R * R * (p->dim == 3 ? n : 1);
    v->t_rows = p->T;
    v->t_cols = p->Tc;
    v->sums = p->slab_sums;
    for (int k = 0; k < 2; ++k) {
        double2* u = k ? p->u1 : p->u0;
        v->u_first[k] = u;
        v->u_last[k] = u + (size_t)(R - 1) * halo;
        v->u_halo_lo[k] = u - halo;
        v->u_halo_hi[k] = u + (size_t)R * halo;
    }
    v->stream = p->stream;
    v->dim = p->dim;
    v->halo_elems = (int64_t)halo;
    return BP_OK;
}

int bp_slab_set_exchange(bp_problem* p, int32_t enable, void* local_t_rows, void* local_t_cols,
                         void* const* peer_t_cols, void* const* peer_t_rows) {
    if (int rc = check_problem(p)) return rc;
    if (!p->slab_log2) return set_err(BP_EINVAL, "not a slab problem");
    DeviceGuard guard(p->device);
    CU(cudaStreamSynchronize(p->stream));
    if (!p->own_T) {
        p->own_T = p->T;
        p->own_Tc = p->Tc;
    }
    if (!enable) {
        p->xchg_on = false;
        p->T = p->own_T;
        p->Tc = p->own_Tc;
        return BP_OK;
    }
    if (p->slab_nranks > kMaxXchg) return set_err(BP_ENOTSUP, "fused exchange: at most 8 ranks");
    if (!peer_t_cols || !peer_t_rows) return set_err(BP_EINVAL, "fused exchange: null peer pointer arrays");
    for (int r = 0; r < p->slab_nranks; ++r) {
        if (!peer_t_cols[r] || !peer_t_rows[r]) return set_err(BP_EINVAL, "fused exchange: null peer pointer");
        p->xchg_cols[r] = static_cast<double2*>(peer_t_cols[r]);
        p->xchg_rows[r] = static_cast<double2*>(peer_t_rows[r]);
    }
    p->T = local_t_rows ? static_cast<double2*>(local_t_rows) : p->own_T;
    p->Tc = local_t_cols ? static_cast<double2*>(local_t_cols) : p->own_Tc;
    p->xchg_on = true;
    return BP_OK;
}

int bp_slab_set_fields(bp_problem* p, const double* f, const double* u0) {
    if (int rc = check_problem(p)) return rc;
    if (!p->slab_log2 || !f) return set_err(BP_EINVAL, "slab: null field or not a slab problem");
    DeviceGuard guard(p->device);
    const int R = 1 << p->slab_log2;
    const size_t fb = sizeof(double2) * p->field, ub = sizeof(double2) * (p->field + 2 * slab_halo(p));
    std::vector<double2> rows;
    pack_slab_host(f, p->n, p->row0, R, rows, p->dim);
    CU(cudaMemcpyAsync(p->f, rows.data(), fb, cudaMemcpyHostToDevice, p->stream));
    CU(cudaMemsetAsync(p->u_alloc0, 0, ub, p->stream));
    if (u0) {
        pack_slab_host(u0, p->n, p->row0, R, rows, p->dim);
        CU(cudaMemcpyAsync(p->u0, rows.data(), fb, cudaMemcpyHostToDevice, p->stream));
    }
    CU(cudaStreamSynchronize(p->stream));  // the staging vector goes out of scope
    return BP_OK;
}

int bp_slab_set_multiplier(bp_problem* p, const double* m) {
    if (int rc = check_problem(p)) return rc;
    if (!p->slab_log2 || !m) return set_err(BP_EINVAL, "slab: null multiplier or not a slab problem");
    DeviceGuard guard(p->device);
    // the rank's block of m in the t_cols layout: line (row) px = the x mode, column qa = the
    // rank's y mode (2-D) / (y, z) mode pair (3-D); Dirichlet zero modes stay 0
    const int n = p->n, nd = n - 1, R = 1 << p->slab_log2, col0 = p->slab_rank * R;
    const size_t cols = p->dim == 3 ? (size_t)R * n : (size_t)R;
    std::vector<double2> blk((size_t)n * cols, make_double2(0.0, 0.0));
    for (int px = 1; px < n; ++px)
        for (size_t qa = 0; qa < cols; ++qa) {
            const int yq = col0 + (p->dim == 3 ? (int)(qa >> p->log2n) : (int)qa);
            const int zq = p->dim == 3 ? (int)(qa & (size_t)(n - 1)) : 1;
            if (yq == 0 || zq == 0) continue;
            const size_t di = p->dim == 3 ? ((size_t)(px - 1) * nd + (yq - 1)) * nd + (zq - 1)
                                          : (size_t)(px - 1) * nd + (yq - 1);
            blk[(size_t)px * cols + qa] = make_double2(m[2 * di], m[2 * di + 1]);
        }
    if (!p->fd) CU(cudaMalloc(&p->fd, sizeof(double2) * blk.size()));
    CU(cudaMemcpyAsync(p->fd, blk.data(), sizeof(double2) * blk.size(), cudaMemcpyHostToDevice, p->stream));
    CU(cudaStreamSynchronize(p->stream));  // the staging vector goes out of scope
    p->slab_fd = true;
    return BP_OK;
}

int bp_slab_stage(bp_problem* p, int32_t stage, const bp_map* map, const bp_iter_config* cfg,
                  double a0, double a1) {
    if (int rc = check_problem(p)) return rc;
    if (!p->slab_log2) return set_err(BP_EINVAL, "not a slab problem");
    DeviceGuard guard(p->device);
    RowArgs a = slab_row_args(p);
    a.ctl.max_iters = p->slab_max_iters;
    a.ctl.rtol = p->slab_rtol;
    const int dim = p->dim;
    const bool d3 = dim == 3;  // 3-D: local y-lines after the forward / before the inverse rows
    switch (stage) {
        case BP_SLAB_FWD_F:  // T <- y-DST of f (3-D: z then y); sums[0] = local ||f||^2
            a.in = p->f;
            CU(launch_row(p->log2n, dim, R_FWD, a, p->stream));
            if (d3)
                if (int rc = slab_ylines(p, a.ctl, true)) return rc;
            return norms(p, p->f, p->slab_sums, true);
        case BP_SLAB_COL:
        case BP_SLAB_COL_LREF:
        case BP_SLAB_COL_FD: {  // column (x-line) pass on the rank's received block
            ColArgs c = col_args(p);
            if (stage == BP_SLAB_COL_FD && !p->slab_fd)
                return set_err(BP_EINVAL, "slab FourierDiag: bp_slab_set_multiplier first");
            c.T = p->Tc;
            c.slab_cols = (1 << p->slab_log2) * (d3 ? p->n : 1);  // 3-D: (y, z) pairs
            c.col0 = p->slab_rank * (1 << p->slab_log2);
            c.slab3 = d3;
            c.scale = p->green_scale;
            c.status = p->slab_running ? a.ctl.status : nullptr;
            if (p->xchg_on) {  // results straight into the source ranks' t_rows
                c.xchg_on = 1;
                c.xchg_rank = p->slab_rank;
                c.xchg_log2r = p->slab_log2;
                for (int r = 0; r < p->slab_nranks; ++r) c.xchg[r] = p->xchg_rows[r];
            }
            if (stage == BP_SLAB_COL_FD) {  // x-DST, x m (correction.cpp:63-68), inverse x-DST
                c.fd = p->fd;
                CU(launch_col_pp(p->log2n, 16, CL_SLAB, C_FD, c, p->stream));
            } else if (stage == BP_SLAB_COL_LREF) {  // x lambda: L_ref of the direction (Direct + Euclidean)
                CU(launch_col_pp(p->log2n, 16, CL_SLAB, C_LREF, c, p->stream));
            } else if (p->tri && c.slab_cols % tri_cols_per_cta(p->log2n) == 0) {
                CU(launch_tri(p->log2n, CL_SLAB, c, p->stream));
            } else {
                CU(launch_col_pp(p->log2n, 16, CL_SLAB, C_GREEN, c, p->stream));
            }
            return BP_OK;
        }
        case BP_SLAB_INV_NORM:  // y <- inverse y-DST of T; sums[1] = local ||y||^2
            if (d3)
                if (int rc = slab_ylines(p, a.ctl)) return rc;
            a.out = p->y;
            a.sub = nullptr;
            CU(launch_row(p->log2n, dim, R_INV, a, p->stream));
            return norms(p, p->y, p->slab_sums + 1, true);
        case BP_SLAB_INIT: {  // a0 = ||f||, a1 = ||G f|| (global); cfg: rtol / max_iters
            if (!cfg) return set_err(BP_EINVAL, "slab init: null config");
            if (!(cfg->rtol > 0.0 && cfg->rtol < 1.0)) return set_err(BP_EINVAL, "run: rtol must lie in (0,1)");
            if (cfg->max_iters < 1) return set_err(BP_EINVAL, "run: max_iters must be >= 1");
            if (!(a0 > 0.0)) return set_err(BP_EINVAL, "run: zero source");
            if (cfg->format != BP_FMT_NPBS && cfg->format != BP_FMT_CBS && cfg->format != BP_FMT_DIRECT)
                return set_err(BP_EINVAL, "run: unknown iteration format");
            if (int rc = ensure_trace(p, cfg->max_iters)) return rc;
            p->slab_direct = cfg->format == BP_FMT_DIRECT;
            p->slab_max_iters = cfg->max_iters;
            p->slab_rtol = cfg->rtol;
            a = slab_row_args(p);
            CU(cudaMemcpyAsync(p->fnorm_l2, &a0, sizeof(double), cudaMemcpyHostToDevice, p->stream));
            CU(cudaMemcpyAsync(p->fnorm_reta, &a1, sizeof(double), cudaMemcpyHostToDevice, p->stream));
            CU(cudaMemsetAsync(p->u_alloc1, 0, sizeof(double2) * (p->field + 2 * slab_halo(p)), p->stream));
            init_control_kernel<<<1, 128, 0, p->stream>>>(a.ctl, 1);
            fill_nan_kernel<<<grid_for((size_t)p->trace_cap), 256, 0, p->stream>>>(p->trace_l2, p->trace_cap);
            fill_nan_kernel<<<grid_for((size_t)p->trace_cap), 256, 0, p->stream>>>(p->trace_reta, p->trace_cap);
            CU(cudaGetLastError());
            CU(cudaStreamSynchronize(p->stream));  // a0 / a1 are host stack values
            p->slab_running = true;
            return BP_OK;
        }
        case BP_SLAB_FWD_BORN:  // T <- y-DST of V u^0 + f
            a.in = p->u0;
            CU(launch_row(p->log2n, dim, R_FWD_BORN, a, p->stream));
            if (d3) return slab_ylines(p, a.ctl, true);
            return BP_OK;
        case BP_SLAB_SWEEP:  // fused scalar / pointwise sweep; sums[0..1] = local entry sums
            if (!map || (map->kind != BP_MAP_SCALAR && map->kind != BP_MAP_POINTWISE))
                return set_err(BP_EINVAL, "BP_SLAB_SWEEP is the scalar / pointwise sweep (the other maps "
                                          "run BP_SLAB_OPT_* / RETA_* / FD_*)");
            a.map_kind = map->kind;
            a.gamma = make_double2(map->gamma_re, map->gamma_im);
            if (d3)
                if (int rc = slab_ylines(p, a.ctl)) return rc;
            CU(launch_row(p->log2n, dim, p->slab_direct ? R_SWEEP_D : R_SWEEP, a, p->stream));
            if (d3) return slab_ylines(p, a.ctl, true);
            return BP_OK;
        case BP_SLAB_ZERO_U:
            CU(cudaMemsetAsync(p->u_alloc0, 0, sizeof(double2) * (p->field + 2 * slab_halo(p)), p->stream));
            return BP_OK;
        case BP_SLAB_FINALIZE:  // sums hold the all-reduced entry sums (a0 = 1: + gamma from sums[2..4])
            slab_finalize_kernel<<<1, 32, 0, p->stream>>>(a.ctl, p->slab_sums, 1, a0 == 1.0 ? 2 : -1);
            CU(cudaGetLastError());
            return BP_OK;
        case BP_SLAB_GAMMA:  // sums[0..2] hold the all-reduced <w, x> and |w|^2 (R_eta metric)
            slab_finalize_kernel<<<1, 32, 0, p->stream>>>(a.ctl, p->slab_sums, 0, 0);
            CU(cudaGetLastError());
            return BP_OK;
        // OptimalScalar / FourierDiag sweeps (plan_for's row stages; the driver puts the
        // reductions, BP_SLAB_FINALIZE / BP_SLAB_GAMMA and the column passes between them)
        case BP_SLAB_OPT_A:   // entry sums + <w, r>, |w|^2 -> sums[0..4]; x^m -> X
        case BP_SLAB_RETA_A:  // entry sums -> sums[0..1]; x^m -> X; t_rows <- y-DST of V x^m
        case BP_SLAB_RETA_C:  // t_rows = G V x: w = x - G V x; <w, x>, |w|^2 -> sums[0..2]
        case BP_SLAB_OPT_B:   // u^{m+1} = u^m + gamma x^m; t_rows <- y-DST of V u^{m+1} + f
        case BP_SLAB_FD_A:    // entry sums -> sums[0..1]; t_rows <- y-DST of x^m
        case BP_SLAB_FD_B: {  // t_rows = du: u^{m+1} = u^m + du; t_rows <- y-DST of V u^{m+1} + f
            const int mode = stage == BP_SLAB_OPT_A    ? R_OPT_A
                             : stage == BP_SLAB_RETA_A ? R_RETA_A
                             : stage == BP_SLAB_RETA_C ? R_RETA_C
                             : stage == BP_SLAB_OPT_B  ? R_OPT_B
                             : stage == BP_SLAB_FD_A   ? R_FD_A
                                                       : R_FD_B;
            // Direct + Euclidean optimal scalar (a0 = 1 on FD_A / RETA_C): w = A r = L_ref r - V r, the
            // direction kept by FD_A and L_ref r arriving through BP_SLAB_COL_LREF (plan_for)
            a.lw = a0 == 1.0 && (mode == R_FD_A || mode == R_RETA_C);
            const bool inv = mode != R_OPT_B, fwd = mode != R_OPT_A && mode != R_RETA_C;
            if (d3 && inv)
                if (int rc = slab_ylines(p, a.ctl)) return rc;
            CU(launch_row(p->log2n, dim, mode, a, p->stream));
            if (d3 && fwd) return slab_ylines(p, a.ctl, true);
            return BP_OK;
        }
    }
    return set_err(BP_EINVAL, "unknown slab stage");
}

int bp_slab_active(bp_problem* p, int32_t* n_active) {
    if (int rc = check_problem(p)) return rc;
    if (!n_active) return set_err(BP_EINVAL, "null output");
    DeviceGuard guard(p->device);
    Control c = make_control(p);
    CU(publish_int(p, c.n_active));
    CU(cudaStreamSynchronize(p->stream));
    *n_active = *p->host_active;
    return BP_OK;
}

int bp_slab_result(bp_problem* p, double* u_dense, double* res_l2, double* res_reta, bp_trace* info) {
    if (int rc = check_problem(p)) return rc;
    if (!p->slab_log2 || !u_dense) return set_err(BP_EINVAL, "slab: null output or not a slab problem");
    DeviceGuard guard(p->device);
    Control c = make_control(p);
    int rb = 0;
    CU(cudaMemcpyAsync(&rb, c.result_buf, sizeof(int), cudaMemcpyDeviceToHost, p->stream));
    CU(cudaStreamSynchronize(p->stream));
    const int n = p->n, R = 1 << p->slab_log2;
    std::vector<double2> rows(p->field);
    CU(cudaMemcpyAsync(rows.data(), rb ? p->u1 : p->u0, sizeof(double2) * rows.size(), cudaMemcpyDeviceToHost,
                       p->stream));
    bp_iter_config cfg{BP_FMT_NPBS, p->slab_rtol, p->slab_max_iters};
    bp_trace tr{};
    if (int rc = finish_run_traces(p, &cfg, res_l2, res_reta, &tr)) return rc;
    if (info) *info = tr;
    unpack_slab_host(rows, n, p->row0, R, u_dense, p->dim);
    p->slab_running = false;
    return BP_OK;
}

}  // extern "C"

namespace {
}  // namespace

extern "C" {

int bp_problem_create(const bp_grid* grid, int32_t batch, const double* k2, const double* k0,
                      const double* eta, int32_t device, bp_problem** out) {
    if (!out) return set_err(BP_EINVAL, "null output handle");
    *out = nullptr;
    if (!grid || !k2 || !k0 || !eta) return set_err(BP_EINVAL, "null argument");
    if (grid->nx < 2 || grid->ny < 2) return set_err(BP_EINVAL, "GridSpec: nx,ny must be >= 2");
    if (!(grid->lx > 0.0) || !(grid->ly > 0.0)) return set_err(BP_EINVAL, "GridSpec: lx,ly must be > 0");
    if (batch < 1) return set_err(BP_EINVAL, "batch must be >= 1");
    if (grid->bc == BP_BC_PERIODIC)  // the reference's own HelmholtzProblem
        return create_impl(grid, 2, batch, k2, k0, eta, device, out, true);
    if (grid->bc != BP_BC_DIRICHLET)
        return set_err(BP_ENOTSUP, "Neumann grids are not implemented on the GPU");
    return create_impl(grid, 2, batch, k2, k0, eta, device, out);
}

int bp_problem_create3d(const bp_grid3* grid, int32_t batch, const double* k2, const double* k0,
                        const double* eta, int32_t device, bp_problem** out) {
    if (!out) return set_err(BP_EINVAL, "null output handle");
    *out = nullptr;
    if (!grid || !k2 || !k0 || !eta) return set_err(BP_EINVAL, "null argument");
    if (grid->nx < 2 || grid->ny < 2 || grid->nz < 2)
        return set_err(BP_EINVAL, "GridSpec: nx,ny,nz must be >= 2");
    if (!(grid->lx > 0.0) || !(grid->ly > 0.0) || !(grid->lz > 0.0))
        return set_err(BP_EINVAL, "GridSpec: lx,ly,lz must be > 0");
    if (batch < 1) return set_err(BP_EINVAL, "batch must be >= 1");
    if (grid->bc != BP_BC_DIRICHLET)
        return set_err(BP_ENOTSUP, "only DirichletInterior grids are implemented on the GPU");
    if (grid->nz != grid->nx || grid->lz != grid->lx)
        return set_err(BP_ENOTSUP, "GPU 3-D path needs cubic grids (hx == hy == hz)");
    const bp_grid g2{grid->nx, grid->ny, grid->lx, grid->ly, grid->bc};
    return create_impl(&g2, 3, batch, k2, k0, eta, device, out);
}

int bp_problem_create_cdr(const bp_grid* grid, int32_t batch, const double* bx, const double* by,
                          const double* sigma, const double* sigma0, int32_t device, bp_problem** out) {
    if (!out) return set_err(BP_EINVAL, "null output handle");
    *out = nullptr;
    if (!grid || !bx || !by || !sigma || !sigma0) return set_err(BP_EINVAL, "null argument");
    if (grid->nx < 2 || grid->ny < 2) return set_err(BP_EINVAL, "GridSpec: nx,ny must be >= 2");
    if (!(grid->lx > 0.0) || !(grid->ly > 0.0)) return set_err(BP_EINVAL, "GridSpec: lx,ly must be > 0");
    if (batch < 1) return set_err(BP_EINVAL, "batch must be >= 1");
    if (grid->bc != BP_BC_NEUMANN) return set_err(BP_EINVAL, "CDR problems live on Neumann grids");
    return create_cdr_impl(grid, batch, bx, by, sigma, sigma0, device, out);
}

int bp_problem_set_cdr_medium(bp_problem* p, const double* bx, const double* by, const double* sigma,
                              const double* sigma0) {
    if (int rc = check_problem(p)) return rc;
    if (!p->cdr) return set_err(BP_EINVAL, "not a CDR problem");
    if (!bx || !by || !sigma || !sigma0) return set_err(BP_EINVAL, "null argument");
    if (int rc = check_cdr_medium(p, bx, by, sigma, sigma0)) return rc;
    DeviceGuard guard(p->device);
    return upload_cdr_medium(p, bx, by, sigma, sigma0);
}

int bp_problem_destroy(bp_problem* p) {
    if (!p) return BP_OK;
    DeviceGuard guard(p->device);
    if (p->stream) cudaStreamSynchronize(p->stream);
    if (p->graph) cudaGraphExecDestroy(p->graph);
    for (auto gw : p->gwave)
        if (gw) cudaGraphExecDestroy(gw);
    for (auto g2 : p->graph2)
        if (g2) cudaGraphExecDestroy(g2);
    for (auto s2 : p->stream2)
        if (s2) cudaStreamDestroy(s2);
    for (auto ev : p->ev_join)
        if (ev) cudaEventDestroy(ev);
    if (p->u_alloc0) p->u0 = p->u_alloc0;
    if (p->u_alloc1) p->u1 = p->u_alloc1;
    if (p->own_T) {  // external exchange buffers (bp_slab_set_exchange) are not ours to free
        p->T = p->own_T;
        p->Tc = p->own_Tc;
    }
    for (void* q : {(void*)p->k2, (void*)p->f, (void*)p->u0, (void*)p->u1, (void*)p->T, (void*)p->x,
                    (void*)p->y, (void*)p->dense, (void*)p->partial, (void*)p->gamma, (void*)p->fd, (void*)p->norm_part,
                    (void*)p->fnorm_l2, (void*)p->fnorm_reta, (void*)p->ctl_int, (void*)p->counter,
                    (void*)p->trace_l2, (void*)p->trace_reta, (void*)p->k0sq, (void*)p->eta,
                    (void*)p->tw, (void*)p->sinp, (void*)p->lap, (void*)p->xi2,
                    (void*)p->bx, (void*)p->by, (void*)p->sigma, (void*)p->sigma0, (void*)p->lapn,
                    (void*)p->rnorm2, (void*)p->w4, (void*)p->dflag, (void*)p->Tc, (void*)p->slab_sums,
                    (void*)p->tri, (void*)p->gax, (void*)p->gay, (void*)p->gpart, (void*)p->gm0, (void*)p->gm1,
                    (void*)p->gm2})
        if (q) cudaFree(q);
    if (p->host_active) cudaFreeHost(p->host_active);
    if (p->host_fn) cudaFreeHost(p->host_fn);
    free_gplan(p->gplan_x);
    free_gplan(p->gplan_y);
    if (p->stream && p->own_stream) cudaStreamDestroy(p->stream);
    delete p;
    return BP_OK;
}

int bp_problem_batch(const bp_problem* p, int32_t* batch, bp_grid* grid) {
    if (int rc = check_problem(p)) return rc;
    if (batch) *batch = p->batch;
    if (grid) *grid = p->grid;
    return BP_OK;
}

static int pointwise_op(const bp_problem* cp, int op, const double* u, const double* f, double* out) {
    if (int rc = check_problem(cp)) return rc;
    if (!u || !out || (op == 3 && !f)) return set_err(BP_EINVAL, "null field");
    auto* p = const_cast<bp_problem*>(cp);
    DeviceGuard guard(p->device);
    if (p->cdr) {
        if (int rc = cdr_upload(p, u, p->x)) return rc;
        if (op == 3)
            if (int rc = cdr_upload(p, f, p->f)) return rc;
        if (int rc = cdr_stencil(p, op, p->x, p->f, p->y)) return rc;
        if (int rc = cdr_download(p, p->y, out)) return rc;
        CU(cudaStreamSynchronize(p->stream));
        return BP_OK;
    }
    if (int rc = upload(p, u, p->x)) return rc;
    if (op == 3)
        if (int rc = upload(p, f, p->f)) return rc;
    if (p->gper && (op == 0 || op == 3)) {
        // pseudospectral A u = F^-1(|xi|^2 F u) - k2 u (helmholtz.cpp:27-32)
        if (int rc = gen_spectral(p, false, p->x, p->y, 2)) return rc;
        gen_pointwise_kernel<<<grid_for(p->field * p->batch), 256, 0, p->stream>>>(gen_args(p), 5, p->x, p->f, p->T);
        combine_kernel<<<grid_for(p->field * p->batch), 256, 0, p->stream>>>(p->y, p->T, op == 3 ? p->f : nullptr,
                                                                           p->field * p->batch);
        CU(cudaGetLastError());
        if (int rc = download(p, p->y, nullptr, nullptr, out)) return rc;
        CU(cudaStreamSynchronize(p->stream));
        return BP_OK;
    }
    if (p->generic) {
        gen_pointwise_kernel<<<grid_for(p->field * p->batch), 256, 0, p->stream>>>(gen_args(p), op, p->x, p->f, p->y);
        CU(cudaGetLastError());
        if (int rc = download(p, p->y, nullptr, nullptr, out)) return rc;
        CU(cudaStreamSynchronize(p->stream));
        return BP_OK;
    }
    if (p->periodic && (op == 0 || op == 3)) {
        // pseudospectral A = L_ref - V (helmholtz.cpp:27-32 computes F^-1(|xi|^2 F u) - k2 u;
        // equal to roundoff): y = L_ref x, then y -= V x (and f - y for the residual)
        if (int rc = periodic_apply(p, 2, p->x, p->y, nullptr)) return rc;
        pointwise_kernel<<<grid_for(p->field * p->batch), 256, 0, p->stream>>>(
            1, p->x, p->k2, p->f, p->k0sq, p->eta, p->inv_h2, p->T, p->batch, p->log2n, p->dim, 0);
        combine_kernel<<<grid_for(p->field * p->batch), 256, 0, p->stream>>>(
            p->y, p->T, op == 3 ? p->f : nullptr, p->field * p->batch);
    } else {
        pointwise_kernel<<<grid_for(p->field * p->batch), 256, 0, p->stream>>>(
            op, p->x, p->k2, p->f, p->k0sq, p->eta, p->inv_h2, p->y, p->batch, p->log2n, p->dim,
            p->periodic ? 0 : 1);
    }
    CU(cudaGetLastError());
    if (int rc = download(p, p->y, p->y, nullptr, out)) return rc;
    CU(cudaStreamSynchronize(p->stream));
    return BP_OK;
}

int bp_apply_A(const bp_problem* p, const double* u, double* out) { return pointwise_op(p, 0, u, nullptr, out); }
int bp_apply_V(const bp_problem* p, const double* u, double* out) { return pointwise_op(p, 1, u, nullptr, out); }
int bp_apply_V_adjoint(const bp_problem* p, const double* u, double* out) { return pointwise_op(p, 2, u, nullptr, out); }
int bp_residual(const bp_problem* p, const double* u, const double* f, double* out) { return pointwise_op(p, 3, u, f, out); }

static int spectral_op(const bp_problem* cp, int which, const double* in, const double* f, double* out) {
    if (int rc = check_problem(cp)) return rc;
    if (!in || !out || (which == 1 && !f)) return set_err(BP_EINVAL, "null field");
    auto* p = const_cast<bp_problem*>(cp);
    DeviceGuard guard(p->device);
    if (p->cdr) {
        if (int rc = cdr_upload(p, in, p->x)) return rc;
        if (which == 1) {  // born residual G(V u + f) - u
            if (int rc = cdr_upload(p, f, p->f)) return rc;
            if (int rc = cdr_stencil(p, 4, p->x, p->f, p->y)) return rc;
            if (int rc = cdr_apply(p, 0, p->y, p->y, p->x)) return rc;
        } else if (int rc = cdr_apply(p, which, p->x, p->y, nullptr)) {
            return rc;
        }
        if (int rc = cdr_download(p, p->y, out)) return rc;
        CU(cudaStreamSynchronize(p->stream));
        return BP_OK;
    }
    if (int rc = upload(p, in, p->x)) return rc;
    if (p->generic) {
        const GenArgs g = gen_args(p);
        switch (which) {
            case 0: if (int rc = gen_spectral(p, true, p->x, p->y)) return rc; break;
            case 1:  // G(V u + f) - u
                if (int rc = upload(p, f, p->f)) return rc;
                gen_pointwise_kernel<<<grid_for(p->field * p->batch), 256, 0, p->stream>>>(g, 4, p->x, p->f, p->y);
                if (int rc = gen_spectral(p, true, p->y, p->y)) return rc;
                combine_kernel<<<grid_for(p->field * p->batch), 256, 0, p->stream>>>(p->y, p->x, nullptr,
                                                                                   p->field * p->batch);
                break;
            case 2: if (int rc = gen_spectral(p, false, p->x, p->y)) return rc; break;
            case 3: if (int rc = gen_dst2(p, p->x, p->y, 1.0)) return rc; break;
            default: if (int rc = gen_dst2(p, p->x, p->y, g.gscale, p->gper)) return rc; break;
        }
        CU(cudaGetLastError());
        if (int rc = download(p, p->y, nullptr, nullptr, out)) return rc;
        CU(cudaStreamSynchronize(p->stream));
        return BP_OK;
    }
    if (p->periodic) {
        if (which == 1)
            if (int rc = upload(p, f, p->f)) return rc;
        if (int rc = periodic_apply(p, which, p->x, p->y, which == 1 ? p->x : nullptr)) return rc;
        if (int rc = download(p, p->y, nullptr, nullptr, out)) return rc;
        CU(cudaStreamSynchronize(p->stream));
        return BP_OK;
    }
    RowArgs a = row_args(p);
    ColArgs c = col_args(p);
    a.in = p->x;
    switch (which) {
        case 0:  // G
            if (int rc = green(p, p->x, p->y, nullptr, false)) return rc;
            break;
        case 1:  // born residual: G(V u + f) - u
            if (int rc = upload(p, f, p->f)) return rc;
            if (int rc = green(p, p->x, p->y, p->x, true)) return rc;
            break;
        case 2:  // L_ref
            CU(launch_row(p->log2n, p->dim, R_FWD, a, p->stream));
            if (int rc = col_stage_checked(p, c, C_LREF, p->green_scale)) return rc;
            a.out = p->y;
            CU(launch_row(p->log2n, p->dim, R_INV, a, p->stream));
            break;
        case 3:  // forward transform (plain sine sums)
        case 4:  // inverse transform (x prod 2/(n_i+1), proj/src/transforms.cpp:96-103)
            CU(launch_row(p->log2n, p->dim, R_FWD, a, p->stream));
            // dim engine passes (gain 4 each) for a dim-D transform
            if (int rc = col_stage_checked(p, c, C_ONE,
                    (which == 3 ? 1.0 : std::pow(2.0 / p->n, p->dim)) / std::pow(kEngineGain, p->dim)))
                return rc;
            if (int rc = download(p, p->T, p->T, nullptr, out)) return rc;
            CU(cudaStreamSynchronize(p->stream));
            return BP_OK;
    }
    if (int rc = download(p, p->y, p->y, nullptr, out)) return rc;
    CU(cudaStreamSynchronize(p->stream));
    return BP_OK;
}

int bp_apply_G(const bp_problem* p, const double* q, double* out) { return spectral_op(p, 0, q, nullptr, out); }
int bp_born_residual(const bp_problem* p, const double* u, const double* f, double* out) {
    return spectral_op(p, 1, u, f, out);
}
int bp_apply_Lref(const bp_problem* p, const double* u, double* out) { return spectral_op(p, 2, u, nullptr, out); }
int bp_forward_transform(const bp_problem* p, const double* field, double* modes) {
    return spectral_op(p, 3, field, nullptr, modes);
}
int bp_inverse_transform(const bp_problem* p, const double* modes, double* field) {
    return spectral_op(p, 4, modes, nullptr, field);
}

// Holds the handle's compute turn (if hooks are set) from construction to release().
struct ComputeTurn {
    bp_problem* p;
    bool held;
    explicit ComputeTurn(bp_problem* pp) : p(pp), held(pp->hook_pre != nullptr) {
        if (held) p->hook_pre(p->hook_ctx);
    }
    void release() {
        if (held) p->hook_post(p->hook_ctx);
        held = false;
    }
    ~ComputeTurn() { release(); }
};

static int run_impl(const bp_problem* cp, const bp_map* map, const double* f, const bp_iter_config* cfg,
                    const double* u0, double* u_out, double* res_l2, double* res_reta, bp_trace* info,
                    bool host_ptr, double* snapshots, int n_snap) {
    if (int rc = validate_run(cp, map, cfg)) return rc;
    if (!f || !u_out) return set_err(BP_EINVAL, "run: null field");
    auto* p = const_cast<bp_problem*>(cp);
    DeviceGuard guard(p->device);
    if (int rc = ensure_trace(p, cfg->max_iters)) return rc;
    if (p->cdr) {
        if (int rc = cdr_upload(p, f, p->f, host_ptr)) return rc;
        if (u0)
            if (int rc = cdr_upload(p, u0, p->u0, host_ptr)) return rc;
        ComputeTurn turn(p);
        if (int rc = map->kind == BP_MAP_OPTIMAL_SCALAR
                         ? run_core_cdr_maps(p, map, cfg, u0 != nullptr, snapshots, n_snap)
                         : run_core_cdr(p, map, cfg, u0 != nullptr, snapshots, n_snap))
            return rc;
        turn.release();
        return finish_run(p, cfg, u_out, host_ptr, res_l2, res_reta, info);
    }
    if (int rc = upload(p, f, p->f, host_ptr)) return rc;
    if (u0)  // periodic: the physical u0 is transformed into U^0 by run_core_periodic
        if (int rc = upload(p, u0, p->periodic ? p->x : p->u0, host_ptr)) return rc;
    ComputeTurn turn(p);
    const int rc = p->periodic  ? run_core_periodic(p, map, cfg, u0 != nullptr, snapshots, n_snap)
                   : p->generic
                       ? ((map->kind == BP_MAP_OPTIMAL_SCALAR || map->kind == BP_MAP_FOURIER_DIAG)
                              ? run_core_generic_maps(p, map, cfg, u0 != nullptr, snapshots, n_snap)
                              : run_core_generic(p, map, cfg, u0 != nullptr, snapshots, n_snap))
                                : run_core(p, map, cfg, u0 != nullptr, snapshots, n_snap);
    if (rc) return rc;
    turn.release();
    return finish_run(p, cfg, u_out, host_ptr, res_l2, res_reta, info);
}

int bp_run(const bp_problem* p, const bp_map* map, const double* f, const bp_iter_config* cfg,
           const double* u0, double* u_out, double* res_l2, double* res_reta, bp_trace* info) {
    return run_impl(p, map, f, cfg, u0, u_out, res_l2, res_reta, info, true, nullptr, 0);
}

int bp_run_device(const bp_problem* p, const bp_map* map, const double* f_dev,
                  const bp_iter_config* cfg, const double* u0_dev, double* u_out_dev,
                  double* res_l2, double* res_reta, bp_trace* info) {
    return run_impl(p, map, f_dev, cfg, u0_dev, u_out_dev, res_l2, res_reta, info, false, nullptr, 0);
}

int bp_run_snapshots(const bp_problem* p, const bp_map* map, const double* f,
                     const bp_iter_config* cfg, const double* u0, double* u_out, double* res_l2,
                     double* res_reta, bp_trace* info, double* snapshots, int32_t n_snap) {
    return run_impl(p, map, f, cfg, u0, u_out, res_l2, res_reta, info, true, snapshots, n_snap);
}

int bp_problem_stream(const bp_problem* p, void** stream) {
    if (int rc = check_problem(p)) return rc;
    if (!stream) return set_err(BP_EINVAL, "null output");
    *stream = (void*)p->stream;
    return BP_OK;
}

int bp_problem_set_medium(bp_problem* p, const double* k2, const double* k0, const double* eta) {
    if (int rc = check_problem(p)) return rc;
    if (p->cdr) return set_err(BP_EINVAL, "CDR problem: use bp_problem_set_cdr_medium");
    if (!k2 || !k0 || !eta) return set_err(BP_EINVAL, "null argument");
    for (int b = 0; b < p->batch; ++b) {
        if (!(eta[b] > 0.0)) return set_err(BP_EINVAL, "HelmholtzProblem: eta must be > 0");
        if (!std::isfinite(k0[b])) return set_err(BP_EINVAL, "HelmholtzProblem: k0 not finite");
    }
    if (p->gper) {
        if (int rc = check_symbol_generic(xi2_table(p->gnx, p->grid.lx), xi2_table(p->gny, p->grid.ly), p->batch, k0, eta))
            return rc;
    } else if (p->generic) {
        const double hx = p->grid.lx / (p->gnx + 1), hy = p->grid.ly / (p->gny + 1);
        if (int rc = check_symbol_generic(gen_lap(p->gnx, hx), gen_lap(p->gny, hy), p->batch, k0, eta)) return rc;
    } else if (p->periodic) {
        if (int rc = check_symbol_periodic(xi2_table(p->n, p->grid.lx), p->batch, k0, eta)) return rc;
    } else if (int rc = check_symbol(p->grid, p->dim, p->batch, k0, eta)) {
        return rc;
    }
    DeviceGuard guard(p->device);
    if (int rc = upload_k2_checked(p, k2)) return rc;  // validated before anything is replaced
    std::vector<double> k0sq(p->batch);
    for (int b = 0; b < p->batch; ++b) k0sq[b] = k0[b] * k0[b];
    CU(cudaMemcpyAsync(p->k0sq, k0sq.data(), sizeof(double) * p->batch, cudaMemcpyHostToDevice, p->stream));
    CU(cudaMemcpyAsync(p->eta, eta, sizeof(double) * p->batch, cudaMemcpyHostToDevice, p->stream));
    if (int rc = build_tri(p)) return rc;
    CU(cudaStreamSynchronize(p->stream));
    return BP_OK;
}

int bp_set_kernel_timing(bp_problem* p, int32_t enable) {
    if (int rc = check_problem(p)) return rc;
    p->timing = enable != 0;
    return BP_OK;
}

int bp_last_run_stats(const bp_problem* p, int64_t* kernel_launches, int64_t* active_sweeps,
                      double* row_kernel_ms, double* col_kernel_ms, int64_t* timed_sweeps) {
    if (int rc = check_problem(p)) return rc;
    if (kernel_launches) *kernel_launches = p->stat_launches;
    if (active_sweeps) *active_sweeps = p->stat_sweeps;
    if (row_kernel_ms) *row_kernel_ms = p->stat_row_ms;
    if (col_kernel_ms) *col_kernel_ms = p->stat_col_ms;
    if (timed_sweeps) *timed_sweeps = p->stat_timed;
    return BP_OK;
}

}  // extern "C"
