/*
 * bp_oracle.h -- CPU ORACLE (test infrastructure only; never the product path).
 *
 * Plain-C restatement of the reference's Born-series hot path, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER for the
 * CUDA path.  Nothing under paper_2603_18527_b200/ links or calls this code.
 *
 * Parity pinning: the restatement is checked against (i) scipy.fft golden vectors
 * (tests/golden/), (ii) the SPEC.md known-answer values, (iii) the reference's own
 * verify-suite properties (proj/src/verify.cpp:82-216) and (iv) trajectories produced
 * by the reference's own L1-L3 sources compiled in place (oracle/_ref, see
 * oracle/ref/Makefile) -- see tests/test_oracle.py.
 *
 * Conventions follow the reference exactly:
 *   layout      row-major, x slow: data[ix*ny + iy]    (proj/include/bp/field.hpp:14-26)
 *   complex     interleaved re/im doubles               (std::complex<double>)
 *   grid        DirichletInterior, h = lx/(nx+1)         (proj/include/bp/grid.hpp:12-24)
 *   DST-I       Y_pq = sum X_ij sin(pi(i+1)(p+1)/(nx+1)) sin(pi(j+1)(q+1)/(ny+1))
 *               inverse carries 4/((nx+1)(ny+1))         (proj/include/bp/transforms.hpp:15-24,
 *                                                          proj/src/transforms.cpp:96-148)
 */
#ifndef BP_ORACLE_H
#define BP_ORACLE_H

#include <complex.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double _Complex bpo_c;

/* Problem: Dirichlet five-point Helmholtz, A = L_D - k2, L_eta = L_D - (k0^2 + i eta),
 * V = k2 - (k0^2 + i eta).  Pattern of proj/src/newton_problem.cpp:17-44 (DST-I symbol,
 * five-point A) combined with proj/src/helmholtz.cpp:11-25 (V, shift). */
typedef struct {
    int nx, ny, nz; /* nz == 1: the reference's 2-D grid; nz > 1: 3-D extension (config c3) */
    int periodic;   /* 1: the reference's own HelmholtzProblem (FFT basis, spectral Laplacian) */
    int cdr;        /* 1: config-c4 convection-diffusion-reaction, Neumann cell-centred, DCT-II */
    double* bx;     /* cdr: velocity (x = first index), real nx*ny */
    double* by;
    double* sigma;  /* cdr: reaction, real nx*ny */
    double sigma0;  /* cdr: reference shift, L0 = -Lap_N + sigma0 */
    double lx, ly;
    double k0, eta;
    bpo_c* k2;      /* nx*ny, damped squared wavenumber */
    bpo_c* v;       /* nx*ny, V coefficient */
    bpo_c* lambda;  /* nx*ny, L_eta symbol in DST-I basis */
} bpo_problem;

enum { BPO_OK = 0, BPO_EINVAL = 1, BPO_ERUNTIME = 2 };
enum { BPO_MAP_SCALAR = 0, BPO_MAP_OPTIMAL_SCALAR = 1, BPO_MAP_FOURIER_DIAG = 2, BPO_MAP_POINTWISE = 3 };
enum { BPO_METRIC_EUCLIDEAN = 0, BPO_METRIC_RETA = 1 };
enum { BPO_FMT_DIRECT = 0, BPO_FMT_CBS = 1, BPO_FMT_NPBS = 2 };
enum { BPO_TERM_CONVERGED = 0, BPO_TERM_MAXITERS = 1, BPO_TERM_DIVERGED = 2, BPO_TERM_STAGNATED = 3 };

const char* bpo_last_error(void);
void bpo_set_threads(int n);

/* 1-D / 2-D transforms (plain sine sums; reference forward convention). */
void bpo_dst1_1d(int n, const double* in_c, double* out_c);
void bpo_forward_dst(int nx, int ny, const double* in_c, double* out_c);
void bpo_inverse_dst(int nx, int ny, const double* in_c, double* out_c);

/* Problem construction / destruction. k2 is complex interleaved nx*ny. */
int bpo_problem_create(int nx, int ny, double lx, double ly, const double* k2_c, double k0,
                       double eta, bpo_problem** out);
/* 3-D extension (config c3; no reference counterpart): DST-I along x, y, z
 * (layout [ix][iy][iz], z contiguous), seven-point stencil, symbol sum of three 1-D factors,
 * inverse scale 8/((nx+1)(ny+1)(nz+1)).  Requires hx == hy == hz (lx = ly = lz). */
int bpo_problem_create3(int nx, int ny, int nz, double l, const double* k2_c, double k0, double eta,
                        bpo_problem** out);
void bpo_forward_dst3(int nx, int ny, int nz, const double* in_c, double* out_c);
void bpo_inverse_dst3(int nx, int ny, int nz, const double* in_c, double* out_c);
/* The reference's periodic pseudospectral HelmholtzProblem (proj/src/helmholtz.cpp:11-53):
 * A u = F^-1(|xi|^2 F u) - k2 u, L_eta symbol |xi|^2 - (k0^2 + i eta), FFT basis with the
 * unnormalized forward / 1/(nx ny) inverse of proj/include/bp/transforms.hpp:16-17. */
int bpo_problem_create_periodic(int nx, int ny, double lx, double ly, const double* k2_c,
                                double k0, double eta, bpo_problem** out);
void bpo_fft2(int nx, int ny, int sign, const double* in_c, double* out_c);
/* Config c4 (no reference counterpart for the upwind term): Neumann
 * cell-centred grid (h = lx/nx, x_i = (i+1/2) h, grid.hpp:13-14,31), reflective ghosts,
 * A u = -Lap_N u + b . grad_upwind u + sigma u, L0 = -Lap_N + sigma0 diagonalised by DCT-II
 * (symbol.cpp:81-91, transforms.cpp:120-121,142-143: REDFT10 forward, REDFT01 / (4 nx ny)
 * inverse), V = L0 - A.  Fields are complex arrays with zero imaginary part. */
int bpo_problem_create_cdr(int nx, int ny, double lx, double ly, const double* bx,
                           const double* by, const double* sigma, double sigma0,
                           bpo_problem** out);
void bpo_dct2(int nx, int ny, int inverse, const double* in_c, double* out_c);
void bpo_problem_destroy(bpo_problem* p);
void bpo_problem_symbol(const bpo_problem* p, double* lambda_c);

/* Operator applications (all complex interleaved, nx*ny). */
void bpo_apply_A(const bpo_problem* p, const double* u, double* out);
void bpo_apply_V(const bpo_problem* p, const double* u, double* out);
void bpo_apply_V_adjoint(const bpo_problem* p, const double* u, double* out);
void bpo_apply_Lref(const bpo_problem* p, const double* u, double* out);
int bpo_apply_G(const bpo_problem* p, const double* q, double* out);
int bpo_born_residual(const bpo_problem* p, const double* u, const double* f, double* out);
void bpo_residual(const bpo_problem* p, const double* u, const double* f, double* out);
double bpo_norm2(int n, const double* x);

/* Iteration driver, restating bp::run (proj/src/iterate.cpp:88-153).
 * res_l2 / res_reta: capacity max_iters+1.  snapshots (optional): n_snap fields, u^m for
 * m = 0..n_snap-1 (entries past the last iterate are left untouched). */
typedef struct {
    int kind;        /* BPO_MAP_* */
    double gamma_re; /* scalar map */
    double gamma_im;
    int metric;      /* optimal scalar */
    const double* m; /* fourier diag multiplier (complex nx*ny) */
} bpo_map;

typedef struct {
    int iters;
    int terminated;
    double fnorm_l2;
    double fnorm_reta;
} bpo_trace;

int bpo_run(const bpo_problem* p, const bpo_map* map, const double* f, int format, double rtol,
            int max_iters, const double* u0, double* u_out, double* res_l2, double* res_reta,
            bpo_trace* info, double* snapshots, int n_snap);

#ifdef __cplusplus
}
#endif

#endif
