/*
 * bornsweep.h -- C ABI of the B200-native Born-series sweep (libbornsweep.so).
 *
 * Drop-in boundary for the reference's hot path (arxiv 2603.18527, "bornprec"):
 * the operator API of bp::Problem (proj/include/bp/problem.hpp:16-49), the correction-map
 * API of bp::CorrectionMap / apply_correction (proj/include/bp/correction.hpp:16-59) and the
 * driver bp::run (proj/include/bp/iterate.hpp:14-67).  The reference is a C++ library with no
 * FFI of its own; these are the plain-pointer entry points a ctypes / cffi / extern "C"
 * binding of that API would call.  No torch types cross this boundary.
 *
 * Data conventions (identical to the reference):
 *   field    nx*ny complex128, row-major with x slow: data[ix*ny + iy], re/im interleaved
 *            (proj/include/bp/field.hpp:14-26; std::complex<double> is array-compatible
 *            with double[2]).  Batched entry points take `batch` fields back to back.
 *   grid     DirichletInterior, h = lx/(nx+1) (proj/include/bp/grid.hpp:12-24).
 *   DST-I    forward = plain sine sum, inverse carries 4/((nx+1)(ny+1))
 *            (proj/include/bp/transforms.hpp:15-24).
 * Supported on the GPU (2-D Dirichlet): any nx, ny in [2, 4095] and any lx, ly -- square
 * grids with nx+1 = ny+1 = 2^k (8 <= 2^k <= 4096) and lx == ly run the fused kernels, every
 * other shape the any-shape path (radix-2 / Bluestein line transforms; every map and format);
 * the reference accepts any size through FFTW (proj/src/transforms.cpp:39-65).
 * 3-D, periodic and CDR handles: power-of-two sides as stated at their constructors.
 *
 * Errors: every function returns a status; nothing throws across the boundary.
 *   BP_EINVAL   <-> std::invalid_argument (e.g. proj/src/problem.cpp:16, iterate.cpp:90-94,
 *                   helmholtz.cpp:18)
 *   BP_ERUNTIME <-> std::runtime_error (near-zero symbol, proj/src/symbol.cpp:30-31,109-110)
 *   BP_ECUDA / BP_ENCCL for device / collective failures.  bp_last_error() (thread-local)
 *   holds the message.  Numerical failure is NOT an error: it is reported through
 *   bp_trace.terminated exactly like bp::Termination (proj/include/bp/iterate.hpp:20).
 *
 * Threading: concurrent calls on distinct handles are safe, each handle owns its stream and
 * workspaces.  Unlike bp::Problem (problem.hpp:14-15) a handle is NOT reentrant: every call,
 * the bp_apply_* operators included, uses the handle's device workspaces, so one handle must
 * not be used from two threads at once -- nor directly while a pipeline job runs on it
 * (bp_pipeline_*; a direct call between jobs is fine).
 */
#ifndef BORNSWEEP_H
#define BORNSWEEP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BP_ABI_VERSION 1

enum {
    BP_OK = 0,
    BP_EINVAL = 1,
    BP_ERUNTIME = 2,
    BP_ECUDA = 3,
    BP_ENCCL = 4,
    BP_ENOTSUP = 5
};

/* bp::Bc (proj/include/bp/grid.hpp:10) */
enum { BP_BC_PERIODIC = 0, BP_BC_DIRICHLET = 1, BP_BC_NEUMANN = 2 };

/* bp::GridSpec (proj/include/bp/grid.hpp:15-43) */
typedef struct {
    int32_t nx, ny;
    double lx, ly;
    int32_t bc;
} bp_grid;

/* CorrectionMap variants (proj/include/bp/correction.hpp:16-40) plus the diagonal
 * relaxation gamma(x) = (i/eta) V(x) ("scalar/diagonal relaxation").
 * Supported on the GPU (bp_run):
 *   SCALAR          every family and path (CDR: real gamma only)
 *   OPTIMAL_SCALAR  Dirichlet 2-D (any shape) / 3-D, single device and slabs, and periodic (any
 *                   shape), both metrics, every format; CDR (CBS / NPBS)
 *   FOURIER_DIAG    Dirichlet 2-D (any shape) / 3-D, single device and slabs, and periodic (any shape)
 *   POINTWISE       Dirichlet 2-D (any shape) / 3-D, single device and slabs (a Dirichlet-family map)
 * anything else returns BP_ENOTSUP. */
enum {
    BP_MAP_SCALAR = 0,         /* ScalarMap{gamma}                                      */
    BP_MAP_OPTIMAL_SCALAR = 1, /* OptimalScalarMap{metric}                              */
    BP_MAP_FOURIER_DIAG = 2,   /* FourierDiagMap{m}                                     */
    BP_MAP_POINTWISE = 3       /* gamma(x) = (i/eta) V(x), Osnabrugge-style CBS          */
};
enum { BP_METRIC_EUCLIDEAN = 0, BP_METRIC_RETA = 1 }; /* bp::OptMetric */

typedef struct {
    int32_t kind;
    double gamma_re, gamma_im; /* BP_MAP_SCALAR */
    int32_t metric;            /* BP_MAP_OPTIMAL_SCALAR */
    const double* m;           /* BP_MAP_FOURIER_DIAG: nx*ny complex (host) */
} bp_map;

/* bp::IterFormat / IterationConfig (proj/include/bp/iterate.hpp:12-18).  DIRECT (direction
 * = r, iterate.cpp:118-123) runs on the Helmholtz families (Dirichlet incl. slabs, periodic);
 * CDR takes CBS / NPBS only (BP_ENOTSUP). */
enum { BP_FMT_DIRECT = 0, BP_FMT_CBS = 1, BP_FMT_NPBS = 2 };
typedef struct {
    int32_t format;   /* default BP_FMT_NPBS */
    double rtol;      /* default 1e-6 */
    int32_t max_iters;/* default 1000 */
} bp_iter_config;

/* bp::Termination (proj/include/bp/iterate.hpp:20) */
enum { BP_TERM_CONVERGED = 0, BP_TERM_MAX_ITERS = 1, BP_TERM_DIVERGED = 2, BP_TERM_STAGNATED = 3 };

/* bp::IterationTrace scalars (proj/include/bp/iterate.hpp:25-32); the per-step vectors
 * res_l2_rel / res_reta_rel are returned through caller arrays of max_iters+1 entries
 * (entries past iters are set to NaN). */
typedef struct {
    int32_t iters;
    int32_t terminated;
    double fnorm_l2;
    double fnorm_reta;
} bp_trace;

/* 3-D grid (config c3): the reference has no 3-D; the extension keeps the
 * DirichletInterior convention per axis, layout data[(ix*ny + iy)*nz + iz]. */
typedef struct {
    int32_t nx, ny, nz;
    double lx, ly, lz;
    int32_t bc;
} bp_grid3;

typedef struct bp_problem bp_problem;

const char* bp_last_error(void);
int bp_abi_version(void);

/* Dirichlet five-point Helmholtz batch (grid->bc = BP_BC_DIRICHLET; BP_BC_PERIODIC gives the
 * reference's periodic pseudospectral HelmholtzProblem, nx = ny = 2^k): A = L_D - k2, L_ref = L_D - (k0^2 + i eta),
 * V = k2 - (k0^2 + i eta)   (HelmholtzProblem ctor, proj/src/helmholtz.cpp:11-25, with the
 * DirichletInterior five-point pattern of proj/src/newton_problem.cpp:17-44).
 * k2: batch*nx*ny complex (sponge damping already folded in, like make_helmholtz);
 * k0, eta: batch each.  device: CUDA ordinal. */
int bp_problem_create(const bp_grid* grid, int32_t batch, const double* k2, const double* k0,
                      const double* eta, int32_t device, bp_problem** out);
/* 3-D batch: A = L_D - k2 with the seven-point L_D, symbol sum of three DST-I factors.
 * Cubic grids, n+1 = 2^k, 8 <= 2^k <= 512.  All other entry points take the handle. */
int bp_problem_create3d(const bp_grid3* grid, int32_t batch, const double* k2, const double* k0,
                        const double* eta, int32_t device, bp_problem** out);
/* Config c4 (convection-diffusion-reaction; no reference problem family -- the spectral layer's
 * DCT-II/III and Neumann symbol are the reference pieces it uses: transforms.cpp:56-57,120-121,
 * 142-143, symbol.cpp:81-92).  grid->bc must be BP_BC_NEUMANN (cell-centred, h = lx/nx),
 * nx = ny = 2^k, 8 <= 2^k <= 4096.  A = -Lap_N + b . grad_upwind + sigma (reflective ghosts),
 * L_ref = -Lap_N + sigma0, V = L_ref - A.  bx, by, sigma: batch*nx*ny REAL; sigma0: batch.
 * Every field argument of the entry points below is REAL (nx*ny doubles per member) on a CDR
 * handle; maps: real BP_MAP_SCALAR (the fused sweep) and BP_MAP_OPTIMAL_SCALAR (both metrics,
 * CBS / NPBS; a staged sweep); a complex gamma or a mode-space multiplier would leave the real
 * field layout (BP_ENOTSUP).  bp_apply_V_adjoint applies V^T (the transposed upwind stencil). */
int bp_problem_create_cdr(const bp_grid* grid, int32_t batch, const double* bx, const double* by,
                          const double* sigma, const double* sigma0, int32_t device,
                          bp_problem** out);
int bp_problem_set_cdr_medium(bp_problem* p, const double* bx, const double* by,
                              const double* sigma, const double* sigma0);
/* Launch every later call of this handle on `stream` (a cudaStream_t owned by the caller, e.g.
 * the framework's current stream, so collectives issued on it are ordered with the kernels). */
int bp_problem_set_stream(bp_problem* p, void* stream);
int bp_problem_destroy(bp_problem* p);
int bp_problem_batch(const bp_problem* p, int32_t* batch, bp_grid* grid);
/* Replace the media of every member (same grid and batch): equivalent to constructing new
 * problems, without re-allocating device workspace. */
int bp_problem_set_medium(bp_problem* p, const double* k2, const double* k0, const double* eta);
/* The cudaStream_t the handle launches on (for CUDA-event timing by the caller). */
int bp_problem_stream(const bp_problem* p, void** stream);

/* Operator applications on batch fields, host buffers in and out
 * (Problem::apply_* / born_residual, proj/src/problem.cpp:19-49; residual f - A u,
 * proj/src/iterate.cpp:45-50).  The *_device variants take device pointers. */
int bp_apply_A(const bp_problem* p, const double* u, double* out);
int bp_apply_V(const bp_problem* p, const double* u, double* out);
int bp_apply_V_adjoint(const bp_problem* p, const double* u, double* out);
int bp_apply_Lref(const bp_problem* p, const double* u, double* out);
int bp_apply_G(const bp_problem* p, const double* q, double* out);
int bp_born_residual(const bp_problem* p, const double* u, const double* f, double* out);
int bp_residual(const bp_problem* p, const double* u, const double* f, double* out);
/* forward_transform / inverse_transform for the problem's DST-I basis
 * (proj/src/transforms.cpp:105-148) */
int bp_forward_transform(const bp_problem* p, const double* field, double* modes);
int bp_inverse_transform(const bp_problem* p, const double* modes, double* field);

/* bp::run (proj/src/iterate.cpp:88-153) over the whole batch; every member iterates and
 * terminates independently.  f, u0 (nullable), u_out: batch*nx*ny complex host buffers;
 * res_l2, res_reta: batch*(max_iters+1) (nullable); info: batch entries. */
int bp_run(const bp_problem* p, const bp_map* map, const double* f, const bp_iter_config* cfg,
           const double* u0, double* u_out, double* res_l2, double* res_reta, bp_trace* info);

/* Same with device-resident f / u0 / u_out (CUDA device pointers, same dense layout);
 * traces and info are host buffers.  Used by bench.py's device-resident measurement. */
int bp_run_device(const bp_problem* p, const bp_map* map, const double* f_dev,
                  const bp_iter_config* cfg, const double* u0_dev, double* u_out_dev,
                  double* res_l2, double* res_reta, bp_trace* info);

/* Debug / parity hook: like bp_run, and additionally copies the iterates u^m,
 * m = 0..n_snap-1, of every member into snapshots (n_snap x batch x nx x ny complex). */
int bp_run_snapshots(const bp_problem* p, const bp_map* map, const double* f,
                     const bp_iter_config* cfg, const double* u0, double* u_out,
                     double* res_l2, double* res_reta, bp_trace* info, double* snapshots,
                     int32_t n_snap);

/* Instrumentation for bench.py: number of sweep kernels launched by the last run on this
 * handle, total sweeps executed per member (active sweeps), and the summed device time of
 * the fused sweep kernels measured with CUDA events on the handle's stream (ms; 0 unless
 * enabled with bp_set_kernel_timing). */
int bp_set_kernel_timing(bp_problem* p, int32_t enable);
int bp_last_run_stats(const bp_problem* p, int64_t* kernel_launches, int64_t* active_sweeps,
                      double* row_kernel_ms, double* col_kernel_ms, int64_t* timed_sweeps);

/* ---- overlapped solves (serving pattern; the reference solves one batch at a time and waits,
 * proj/src/bench.cpp:143-151).  A pipeline owns `depth` handles of one shape (created by the
 * caller, destroyed by the caller after bp_pipeline_destroy), each driven by its own host worker
 * thread on the handle's own stream.  bp_pipeline_submit enqueues one job on the next slot
 * (round robin) and returns at once; a job is exactly bp_problem_set_medium (k2 != NULL) or
 * bp_problem_set_cdr_medium (bx != NULL) followed by bp_run on that slot, so while one slot
 * sweeps, the next uploads its media/sources and the previous downloads its iterates.  All host
 * buffers of a job must stay valid until bp_pipeline_wait returns; pinned buffers let the copies
 * run under the other slots' sweeps.  bp_pipeline_wait blocks until every submitted job
 * finished and returns the first job error (message in bp_last_error, prefixed by the slot). */
typedef struct {
    const double *k2, *k0, *eta;               /* Dirichlet / periodic Helmholtz media */
    const double *bx, *by, *sigma, *sigma0;    /* CDR media (config c4) */
} bp_medium;
typedef struct bp_pipeline bp_pipeline;
int bp_pipeline_create(bp_problem* const* slots, int32_t depth, bp_pipeline** out);
int bp_pipeline_submit(bp_pipeline* pl, const bp_medium* medium, const bp_map* map, const double* f,
                       const bp_iter_config* cfg, const double* u0, double* u_out, double* res_l2,
                       double* res_reta, bp_trace* info, int32_t* slot_out);
int bp_pipeline_wait(bp_pipeline* pl);
int bp_pipeline_destroy(bp_pipeline* pl);

/* ---- slab decomposition of ONE 2-D Dirichlet grid over nranks GPUs (config c2).
 * Rank r owns padded rows [r R, (r+1) R), R = (nx+1)/nranks.  The y-DSTs (rows) are local; the
 * x-DSTs need full columns, so the row side writes T blocked by destination rank
 * ([nranks][R][R]: the all-to-all send buffer) and the column pass runs on the received
 * [nranks][R][R] = n x R column block.  The driver (paper_2603_18527_b200/slab.py) runs, per
 * sweep: halo exchange of u^m's edge rows -> BP_SLAB_SWEEP -> all-reduce sums[0..1] ->
 * BP_SLAB_FINALIZE (the termination test of iterate.cpp:134-150 on identical sums on every
 * rank) -> all-to-all t_rows -> t_cols -> BP_SLAB_COL -> all-to-all back (scalar and pointwise
 * maps).  The other reference maps (correction.cpp:22-76) run the staged sweeps, "colpass" =
 * all-to-all, BP_SLAB_COL, all-to-all back:
 *   OptimalScalar, Euclidean:  halo -> OPT_A -> all-reduce sums[0..4] -> FINALIZE(a0 = 1: the
 *                              entry and gamma = <w, r>/<w, w>) -> OPT_B -> colpass
 *   OptimalScalar, R_eta:      halo -> RETA_A -> all-reduce sums[0..1] -> FINALIZE -> colpass
 *                              (G V x) -> RETA_C -> all-reduce sums[0..2] -> GAMMA -> OPT_B -> colpass
 *   FourierDiag:               halo -> FD_A -> all-reduce sums[0..1] -> FINALIZE -> all-to-all,
 *                              COL_FD (the rank's block of m, bp_slab_set_multiplier),
 *                              all-to-all back -> FD_B -> colpass
 * IterFormat::Direct (cfg->format at BP_SLAB_INIT): the same sequences with the direction r^m;
 * OptimalScalar-Euclidean + Direct needs w = A r = L_ref r - V r:
 *   halo -> FD_A(a0 = 1: keeps r) -> all-reduce sums[0..1] -> FINALIZE -> all-to-all, COL_LREF,
 *   all-to-all back -> RETA_C(a0 = 1) -> all-reduce sums[0..2] -> GAMMA -> OPT_B -> colpass
 * bp_run semantics otherwise. */
enum {
    BP_SLAB_FWD_F = 0,     /* t_rows <- y-DST of f; sums[0] = local ||f||^2 */
    BP_SLAB_COL = 1,       /* t_cols: x-DST, x Green weights, inverse x-DST (in place) */
    BP_SLAB_INV_NORM = 2,  /* y <- inverse y-DST of t_rows; sums[1] = local ||y||^2 */
    BP_SLAB_INIT = 3,      /* a0 = ||f||, a1 = ||G f|| (global), cfg: control + traces reset */
    BP_SLAB_FWD_BORN = 4,  /* t_rows <- y-DST of V u^0 + f */
    BP_SLAB_SWEEP = 5,     /* fused sweep; sums[0..1] = local entry sums */
    BP_SLAB_FINALIZE = 6,  /* trace entry + termination from the all-reduced sums */
    BP_SLAB_ZERO_U = 7,    /* u^0 <- 0 on the device (a cold start without re-staging f) */
    BP_SLAB_OPT_A = 8,     /* entry sums, <w, r>, |w|^2 (w = A x) -> sums[0..4]; keeps x^m */
    BP_SLAB_OPT_B = 9,     /* u^{m+1} = u^m + gamma x^m; t_rows <- y-DST of V u^{m+1} + f */
    BP_SLAB_RETA_A = 10,   /* entry sums -> sums[0..1]; keeps x^m; t_rows <- y-DST of V x^m */
    BP_SLAB_RETA_C = 11,   /* t_rows = G V x^m: w = x - G V x; <w, x>, |w|^2 -> sums[0..2] */
    BP_SLAB_FD_A = 12,     /* entry sums -> sums[0..1]; t_rows <- y-DST of x^m */
    BP_SLAB_FD_B = 13,     /* t_rows = du: u^{m+1} = u^m + du; t_rows <- y-DST of V u^{m+1} + f */
    BP_SLAB_COL_FD = 14,   /* t_cols: x-DST, x m (FourierDiag multiplier block), inverse x-DST */
    BP_SLAB_GAMMA = 15,    /* gamma from the all-reduced sums[0..2] (R_eta metric) */
    BP_SLAB_COL_LREF = 16  /* t_cols: x-DST, x lambda, inverse x-DST (L_ref of the direction) */
};
typedef struct {
    int32_t rank, nranks, rows, row0, n;
    int64_t block_elems;           /* R*R complex per destination rank */
    void* t_rows;                  /* device [nranks][R][R] complex128 */
    void* t_cols;                  /* device [nranks][R][R] complex128 */
    void* sums;                    /* device double[8] */
    void* u_first[2];              /* device: first / last owned row of u ping (0) and pong (1) */
    void* u_last[2];
    void* u_halo_lo[2];            /* device: halo rows (row0 - 1, row0 + R) */
    void* u_halo_hi[2];
    void* stream;
    int32_t dim;                   /* 2, or 3 for bp_slab_create3d */
    int64_t halo_elems;            /* complex elements of one halo row (2-D) / x-plane (3-D) */
} bp_slab_view_t;
int bp_slab_create(const bp_grid* grid, int32_t rank, int32_t nranks, const double* k2, double k0,
                   double eta, int32_t device, bp_problem** out);
/* 3-D slabs (config c3 over several GPUs; the 3-D extension has no reference counterpart):
 * rank r owns the x-planes [r R, (r+1) R) of the cubic grid, R = n / nranks.  z-lines (the row
 * kernel) and y-lines are local; the x-lines follow an all-to-all over y-blocks: t_rows is
 * [dest][x_local][y_local][z] (R*R*n per destination), t_cols after the exchange the rank's
 * y-block for every x.  The SWEEP / FWD_F / FWD_BORN stages end with the local y-DSTs, SWEEP /
 * INV_NORM start with the inverse ones, so the stage protocol above is unchanged.  k2, and the
 * fields of bp_slab_set_fields / bp_slab_result, are FULL dense nx^3 arrays. */
int bp_slab_create3d(const bp_grid3* grid, int32_t rank, int32_t nranks, const double* k2, double k0,
                     double eta, int32_t device, bp_problem** out);
/* Fused exchange (nranks <= 8): the kernel that produces the forward transform's blocks (2-D:
 * the row kernel; 3-D: the forward y-lines) stores block d straight into rank d's t_cols, and
 * the column kernel stores its results straight into the source ranks' t_rows -- the two
 * all-to-alls become the kernels' own epilogues (same-device parts, or NVLink peer memory
 * mapped into this process).  peer_t_cols / peer_t_rows: nranks device pointers valid on this
 * device (this rank's own entries included).  local_t_rows / local_t_cols (nullable): buffers
 * to use as this rank's t_rows / t_cols instead of its own (e.g. symmetric-memory allocations;
 * block_elems * nranks complex each).  The driver then only orders the stages across ranks
 * (no transposes).  enable = 0 restores the plain exchange. */
int bp_slab_set_exchange(bp_problem* p, int32_t enable, void* local_t_rows, void* local_t_cols,
                         void* const* peer_t_cols, void* const* peer_t_rows);
int bp_slab_view(const bp_problem* p, bp_slab_view_t* v);
/* f, u0: the FULL dense nx*ny fields (host); u0 may be null */
int bp_slab_set_fields(bp_problem* p, const double* f, const double* u0);
/* FourierDiagMap on slabs (correction.cpp:63-68): m is the FULL dense mode-layout multiplier
 * (nx*ny, or nx^3, complex, host); the rank keeps the block of its own columns, i.e. the
 * multiplier lives in the distributed mode layout of t_cols. */
int bp_slab_set_multiplier(bp_problem* p, const double* m);
int bp_slab_stage(bp_problem* p, int32_t stage, const bp_map* map, const bp_iter_config* cfg,
                  double a0, double a1);
int bp_slab_active(bp_problem* p, int32_t* n_active);
/* writes this rank's rows of the dense nx*ny result into u_dense; traces as bp_run */
int bp_slab_result(bp_problem* p, double* u_dense, double* res_l2, double* res_reta, bp_trace* info);

#ifdef __cplusplus
}
#endif

#endif
