// ref_driver.cpp -- C entry points over the REFERENCE's own L1-L3 code (ORACLE infrastructure).
//
// Linked with the reference sources compiled in place from /root/reference/proj/src
// (parallel, kernels, field, transforms, symbol, problem, helmholtz, newton_problem,
// samplers; see oracle/ref/Makefile) and with the project-owned FFTW shim.  The only code
// restated here is what cannot compile without Eigen (proj/src/iterate.cpp and
// proj/src/correction.cpp include <Eigen/Dense> through proj/include/bp/dense.hpp) and the
// Dirichlet five-point Helmholtz family the BASELINE configs use, which the reference
// assembles only as a pattern (NewtonJacobianProblem, proj/src/newton_problem.cpp:17-51 +
// HelmholtzProblem V/shift, proj/src/helmholtz.cpp:11-39).
//
// Used by tests/ (to pin the plain-C oracle and the instance generator), by
// tests/golden/make_golden.py, and as bench.py's "reference" CPU arm.

#include <omp.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "bp/field.hpp"
#include "bp/grid.hpp"
#include "bp/helmholtz.hpp"
#include "bp/kernels.hpp"
#include "bp/parallel.hpp"
#include "bp/problem.hpp"
#include "bp/problem_io.hpp"
#include "bp/rng.hpp"
#include "bp/samplers.hpp"
#include "bp/symbol.hpp"
#include "bp/transforms.hpp"

using bp::cplx;
using bp::ComplexField;
using bp::GridSpec;

namespace {

thread_local std::string g_err;

// Dirichlet five-point Helmholtz: A = L_D - k2 (five_point as in newton_problem.cpp:38-44),
// L_ref = DST-I five-point symbol shifted by -(k0^2 + i eta) (symbol.cpp:69-80,97-100),
// V = k2 - (k0^2 + i eta) pointwise (helmholtz.cpp:22-24,34-39).
class DirichletHelmholtz : public bp::Problem {
  public:
    DirichletHelmholtz(GridSpec g, ComplexField k2, double k0, double eta)
        : Problem(g, bp::shift_symbol(bp::laplacian_symbol(g), -cplx(k0 * k0, eta))),
          k2_(std::move(k2)),
          k0_(k0),
          eta_(eta) {
        if (g.bc != bp::Bc::DirichletInterior)
            throw std::invalid_argument("DirichletHelmholtz: DirichletInterior grid required");
        if (eta <= 0.0) throw std::invalid_argument("HelmholtzProblem: eta must be > 0");
        if (!bp::all_finite(k2_)) throw std::invalid_argument("HelmholtzProblem: k2 not finite");
        v_.resize(k2_.size());
        const cplx shift(k0 * k0, eta);
        for (size_t i = 0; i < k2_.size(); ++i) v_[i] = k2_.data[i] - shift;
    }
    std::string family() const override { return "helmholtz_dirichlet"; }
    ComplexField apply_A(const ComplexField& u) const override {
        check_grid(u);
        ComplexField out(grid_);
        bp::kernels::five_point(u.data, grid_.nx, grid_.ny, grid_.hx() * grid_.hx(), out.data);
        for (size_t i = 0; i < u.size(); ++i) out.data[i] -= k2_.data[i] * u.data[i];
        return out;
    }
    ComplexField apply_V(const ComplexField& u) const override {
        check_grid(u);
        ComplexField out(grid_);
        bp::kernels::mul(u.data, v_, out.data);
        return out;
    }
    ComplexField apply_V_adjoint(const ComplexField& u) const override {
        check_grid(u);
        ComplexField out(grid_);
        for (size_t i = 0; i < u.size(); ++i) out.data[i] = std::conj(v_[i]) * u.data[i];
        return out;
    }
    const std::vector<cplx>& v() const { return v_; }
    double eta() const { return eta_; }

  private:
    ComplexField k2_;
    double k0_, eta_;
    std::vector<cplx> v_;
};

ComplexField field_from(const GridSpec& g, const double* c) {
    ComplexField f(g);
    if (c) std::memcpy(static_cast<void*>(f.data.data()), c, sizeof(cplx) * f.size());
    return f;
}

void field_to(const ComplexField& f, double* c) {
    std::memcpy(c, f.data.data(), sizeof(cplx) * f.size());
}

// ---- correction maps and driver: restated Eigen-free from proj/src/correction.cpp:10-76
// and proj/src/iterate.cpp:45-153 (same operations, same order).
struct MapDesc {
    int kind;  // 0 scalar, 1 optimal scalar, 2 fourier diag, 3 pointwise (i/eta) V
    cplx gamma;
    int metric;  // 0 euclidean, 1 R_eta
    const double* m;
};

ComplexField residual(const bp::Problem& p, const ComplexField& u, const ComplexField& f) {
    ComplexField au = p.apply_A(u);
    ComplexField r(f.grid);
    bp::kernels::sub(f.data, au.data, r.data);
    return r;
}

cplx optimal_scalar(const ComplexField& r, const ComplexField& w) {
    const double denom = bp::kernels::norm2sq(w.data);
    if (denom <= 0.0 || !std::isfinite(denom)) return cplx{0.0, 0.0};
    return bp::kernels::dotc(w.data, r.data) / denom;
}

ComplexField apply_correction(const bp::Problem& p, const MapDesc& map,
                              const ComplexField& x, const ComplexField& euclid_r) {
    ComplexField out(x.grid);
    switch (map.kind) {
        case 0: bp::kernels::scale(x.data, map.gamma, out.data); return out;
        case 1: {
            cplx gamma;
            if (map.metric == 0) {
                ComplexField w = p.apply_A(x);
                gamma = optimal_scalar(euclid_r, w);
            } else {
                ComplexField gv = p.apply_G(p.apply_V(x));
                ComplexField w = x;
                bp::kernels::sub(w.data, gv.data, w.data);
                gamma = optimal_scalar(x, w);
            }
            bp::kernels::scale(x.data, gamma, out.data);
            return out;
        }
        case 2: {
            std::vector<cplx> modes = bp::forward_transform(x, p.kind());
            std::vector<cplx> m(modes.size());
            std::memcpy(static_cast<void*>(m.data()), map.m, sizeof(cplx) * m.size());
            bp::kernels::mul(modes, m, modes);
            return bp::inverse_transform(modes, x.grid, p.kind());
        }
        case 3: {
            const auto* dh = dynamic_cast<const DirichletHelmholtz*>(&p);
            if (!dh) throw std::invalid_argument("pointwise map needs the Dirichlet family");
            const auto& v = dh->v();
            for (size_t i = 0; i < x.size(); ++i)
                out.data[i] = (cplx(0.0, 1.0) / dh->eta() * v[i]) * x.data[i];
            return out;
        }
    }
    throw std::invalid_argument("unknown correction map");
}

struct TraceOut {
    int iters;
    int terminated;  // 0 converged 1 max_iters 2 diverged 3 stagnated
    double fnorm_l2;
    double fnorm_reta;
};

void run(const bp::Problem& p, const MapDesc& map, const ComplexField& f, int format,
         double rtol, int max_iters, const ComplexField* u0, ComplexField& u,
         std::vector<double>& l2, std::vector<double>& reta, TraceOut& tr) {
    constexpr double kDivergenceThreshold = 1e8;
    constexpr double kStagnationTol = 1e-14;
    constexpr int kStagnationWindow = 20;
    if (!(rtol > 0.0 && rtol < 1.0)) throw std::invalid_argument("run: rtol must lie in (0,1)");
    if (max_iters < 1) throw std::invalid_argument("run: max_iters must be >= 1");
    const double fnorm = bp::kernels::norm2(f.data);
    if (fnorm <= 0.0) throw std::invalid_argument("run: zero source");
    u = u0 ? *u0 : ComplexField(p.grid());
    tr.fnorm_l2 = fnorm;
    tr.fnorm_reta = bp::kernels::norm2(p.apply_G(f).data);
    tr.terminated = 1;
    tr.iters = 0;
    auto record = [&](const ComplexField& r, const ComplexField& gr) {
        l2.push_back(bp::kernels::norm2(r.data) / tr.fnorm_l2);
        reta.push_back(bp::kernels::norm2(gr.data) / tr.fnorm_reta);
    };
    ComplexField r = residual(p, u, f);
    ComplexField gr = p.apply_G(r);
    record(r, gr);
    if (l2.back() <= rtol) {
        tr.terminated = 0;
        return;
    }
    for (int it = 0; it < max_iters; ++it) {
        ComplexField direction(p.grid());
        switch (format) {
            case 0: direction = r; break;
            case 1: direction = gr; break;
            default: direction = p.born_residual(u, f); break;
        }
        ComplexField du = apply_correction(p, map, direction, r);
        bp::kernels::add(u.data, du.data, u.data);
        tr.iters = it + 1;
        r = residual(p, u, f);
        gr = p.apply_G(r);
        record(r, gr);
        const double rel = l2.back();
        if (!std::isfinite(rel) || rel > kDivergenceThreshold) {
            tr.terminated = 2;
            return;
        }
        if (rel <= rtol) {
            tr.terminated = 0;
            return;
        }
        const int n = static_cast<int>(l2.size());
        if (n > kStagnationWindow) {
            const double past = l2[static_cast<size_t>(n - 1 - kStagnationWindow)];
            if (std::abs(past - rel) < kStagnationTol * std::max(1.0, past)) {
                tr.terminated = 3;
                return;
            }
        }
    }
}

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

}  // namespace

extern "C" {

const char* bpref_last_error() { return g_err.c_str(); }

// 0 serial, 1 parallel, 2 auto (proj/include/bp/parallel.hpp:10)
void bpref_set_mode(int mode) {
    bp::parallel::set_mode(mode == 0   ? bp::parallel::Mode::Serial
                           : mode == 1 ? bp::parallel::Mode::Parallel
                                       : bp::parallel::Mode::Auto);
}
int bpref_thread_count() { return bp::parallel::thread_count(); }

int bpref_problem_create(int nx, int ny, double lx, double ly, const double* k2, double k0,
                         double eta, void** out) {
    *out = nullptr;
    return guarded([&] {
        GridSpec g = bp::make_grid(nx, ny, lx, ly, bp::Bc::DirichletInterior);
        *out = new DirichletHelmholtz(g, field_from(g, k2), k0, eta);
    });
}

void bpref_problem_destroy(void* p) { delete static_cast<bp::Problem*>(p); }

// The reference's OWN periodic pseudospectral family: bp::HelmholtzProblem (helmholtz.cpp:11-53)
int bpref_periodic_create(int nx, int ny, double lx, double ly, const double* k2, double k0,
                          double eta, void** out) {
    *out = nullptr;
    return guarded([&] {
        GridSpec g = bp::make_grid(nx, ny, lx, ly, bp::Bc::Periodic);
        *out = static_cast<bp::Problem*>(new bp::HelmholtzProblem(g, field_from(g, k2), k0, eta));
    });
}

// Instance of the reference's Helmholtz bench family (make_bench_instance, bench.cpp:25-67,
// restated: bench.cpp needs Eigen): make_layered_helmholtz(n, ppw, contrast,
// RngState(seed).split("medium")) + gaussian_bump source from split("source").
int bpref_periodic_bench_instance(int n, double ppw, double contrast, uint64_t seed, double* k2,
                                  double* f, double* k0, double* eta) {
    return guarded([&] {
        bp::RngState rng(seed);
        bp::RngState rm = rng.split("medium");
        auto p = bp::make_layered_helmholtz(n, ppw, contrast, rm);
        field_to(p->k2(), k2);
        *k0 = p->k0();
        *eta = p->eta();
        const GridSpec& g = p->grid();
        bp::RngState rs = rng.split("source");
        const double cx = rs.uniform() * g.lx;
        const double cy = rs.uniform() * g.ly;
        const double width = (0.05 + 0.10 * rs.uniform()) * g.lx;
        field_to(bp::to_complex(bp::gaussian_bump(g, cx, cy, width, 1.0)), f);
    });
}

int bpref_symbol(void* h, double* out) {
    auto* p = static_cast<bp::Problem*>(h);  // L_ref symbol of either family
    std::memcpy(out, p->reference_symbol().values.data(),
                sizeof(cplx) * p->reference_symbol().values.size());
    return 0;
}

// op: 0 A, 1 V, 2 V^H, 3 Lref, 4 G, 5 forward DST, 6 inverse DST
int bpref_apply(void* h, int op, const double* in, double* out) {
    auto* p = static_cast<bp::Problem*>(h);
    return guarded([&] {
        ComplexField x = field_from(p->grid(), in);
        switch (op) {
            case 0: field_to(p->apply_A(x), out); break;
            case 1: field_to(p->apply_V(x), out); break;
            case 2: field_to(p->apply_V_adjoint(x), out); break;
            case 3: field_to(p->apply_Lref(x), out); break;
            case 4: field_to(p->apply_G(x), out); break;
            case 5: {
                auto m = bp::forward_transform(x, p->kind());
                std::memcpy(out, m.data(), sizeof(cplx) * m.size());
                break;
            }
            case 6: {
                std::vector<cplx> m(x.data);
                field_to(bp::inverse_transform(m, p->grid(), p->kind()), out);
                break;
            }
            default: throw std::invalid_argument("bad op");
        }
    });
}

int bpref_born_residual(void* h, const double* u, const double* f, double* out) {
    auto* p = static_cast<bp::Problem*>(h);
    return guarded([&] {
        field_to(p->born_residual(field_from(p->grid(), u), field_from(p->grid(), f)), out);
    });
}

int bpref_residual(void* h, const double* u, const double* f, double* out) {
    auto* p = static_cast<bp::Problem*>(h);
    return guarded([&] {
        field_to(residual(*p, field_from(p->grid(), u), field_from(p->grid(), f)), out);
    });
}

int bpref_run(void* h, int map_kind, double g_re, double g_im, int metric, const double* m,
              const double* f, int format, double rtol, int max_iters, const double* u0,
              double* u_out, double* res_l2, double* res_reta, TraceOut* info) {
    auto* p = static_cast<bp::Problem*>(h);
    return guarded([&] {
        MapDesc md{map_kind, cplx(g_re, g_im), metric, m};
        ComplexField ff = field_from(p->grid(), f);
        ComplexField uu0 = u0 ? field_from(p->grid(), u0) : ComplexField(p->grid());
        ComplexField u;
        std::vector<double> l2, reta;
        run(*p, md, ff, format, rtol, max_iters, u0 ? &uu0 : nullptr, u, l2, reta, *info);
        field_to(u, u_out);
        std::memcpy(res_l2, l2.data(), sizeof(double) * l2.size());
        std::memcpy(res_reta, reta.data(), sizeof(double) * reta.size());
    });
}

// Batch of independent members, OpenMP over members (the sample-parallel loop of
// proj/src/bench.cpp:143-151).  k2/f/u_out: batch x nx x ny complex; k0/eta: batch.
// res arrays: batch x (max_iters+1).
// NOTE: the kernels' chunked reductions (proj/src/kernels.cpp:124-157) are not safe inside
// the outer OpenMP loop: with nested parallelism off, the inner team has one thread, which
// sums only chunk 0 of thread_count() chunks.  Under Mode::Auto the reference's own
// bench path therefore computes wrong norms for members >= 16384 points; here the members
// run with Mode::Serial (the reference's ground-truth kernels) and the mode is restored.
int bpref_run_batch(int nx, int ny, double lx, double ly, int batch, const double* k2,
                    const double* k0, const double* eta, int map_kind, double g_re,
                    double g_im, int metric, const double* f, int format, double rtol,
                    int max_iters, double* u_out, double* res_l2, double* res_reta,
                    TraceOut* info, int nthreads) {
    const long npts = static_cast<long>(nx) * ny;
    int rc = 0;
    const bp::parallel::Mode saved = bp::parallel::mode();
    if (nthreads > 1) bp::parallel::set_mode(bp::parallel::Mode::Serial);
#pragma omp parallel for schedule(dynamic) num_threads(nthreads)
    for (int b = 0; b < batch; ++b) {
        void* h = nullptr;
        int r = bpref_problem_create(nx, ny, lx, ly, k2 + 2 * npts * b, k0[b], eta[b], &h);
        if (r == 0)
            r = bpref_run(h, map_kind, g_re, g_im, metric, nullptr, f + 2 * npts * b, format,
                          rtol, max_iters, nullptr, u_out + 2 * npts * b,
                          res_l2 + static_cast<long>(max_iters + 1) * b,
                          res_reta + static_cast<long>(max_iters + 1) * b, info + b);
        bpref_problem_destroy(h);
        if (r) {
#pragma omp critical
            rc = r;
        }
    }
    bp::parallel::set_mode(saved);
    return rc;
}

// Pre-created problems (bpref_problem_create), OpenMP over members like bpref_run_batch: the
// bench's reference arm creates its problems once, outside the timed region, and times only
// the runs (problem setup = the reference's Problem constructor, not part of bp::run).
int bpref_run_handles(int batch, void* const* handles, int map_kind, double g_re, double g_im,
                      int metric, const double* f, long member_stride, int format, double rtol,
                      int max_iters, double* u_out, double* res_l2, double* res_reta,
                      TraceOut* info, int nthreads) {
    int rc = 0;
    const bp::parallel::Mode saved = bp::parallel::mode();
    if (nthreads > 1) bp::parallel::set_mode(bp::parallel::Mode::Serial);
#pragma omp parallel for schedule(dynamic) num_threads(nthreads)
    for (int b = 0; b < batch; ++b) {
        const int r = bpref_run(handles[b], map_kind, g_re, g_im, metric, nullptr,
                                f + 2 * member_stride * b, format, rtol, max_iters, nullptr,
                                u_out + 2 * member_stride * b,
                                res_l2 + static_cast<long>(max_iters + 1) * b,
                                res_reta + static_cast<long>(max_iters + 1) * b, info + b);
        if (r) {
#pragma omp critical
            rc = r;
        }
    }
    bp::parallel::set_mode(saved);
    return rc;
}

// ---- the reference's own samplers and RNG (proj/src/samplers.cpp, proj/include/bp/rng.hpp),
// exposed so the project's instance generator can be pinned against them.
int bpref_sponge_profile(int nx, int ny, int bc, int layer, double strength, double* out) {
    return guarded([&] {
        GridSpec g = bp::make_grid(nx, ny, 1.0, 1.0, static_cast<bp::Bc>(bc));
        bp::RealField d = bp::sponge_profile(g, layer, strength);
        std::memcpy(out, d.data.data(), sizeof(double) * d.size());
    });
}

int bpref_gaussian_bump(int nx, int ny, double lx, double ly, int bc, double cx, double cy,
                        double width, double amp, double* out) {
    return guarded([&] {
        GridSpec g = bp::make_grid(nx, ny, lx, ly, static_cast<bp::Bc>(bc));
        bp::RealField d = bp::gaussian_bump(g, cx, cy, width, amp);
        std::memcpy(out, d.data.data(), sizeof(double) * d.size());
    });
}

// normals from RngState(seed).split(index) (index < 0: unsplit stream)
void bpref_rng_normals(uint64_t seed, int64_t index, int count, double* out) {
    bp::RngState root(seed);
    bp::RngState r = index < 0 ? root : root.split(static_cast<uint64_t>(index));
    for (int i = 0; i < count; ++i) out[i] = r.normal();
}

void bpref_rng_uniforms(uint64_t seed, int64_t index, int count, double* out) {
    bp::RngState root(seed);
    bp::RngState r = index < 0 ? root : root.split(static_cast<uint64_t>(index));
    for (int i = 0; i < count; ++i) out[i] = r.uniform();
}

// DST-I symbol vs five-point: the reference's laplacian_symbol (symbol.cpp:52-95)
int bpref_laplacian_symbol(int nx, int ny, double lx, double ly, int bc, double* out) {
    return guarded([&] {
        GridSpec g = bp::make_grid(nx, ny, lx, ly, static_cast<bp::Bc>(bc));
        auto s = bp::laplacian_symbol(g);
        std::memcpy(out, s.values.data(), sizeof(cplx) * s.values.size());
    });
}

// The reference's DCT pair on a Neumann grid (transforms.cpp:105-148: REDFT10 forward,
// REDFT01 x 1/(4 nx ny) inverse)
int bpref_dct(int nx, int ny, int inverse, const double* in, double* out) {
    return guarded([&] {
        GridSpec g = bp::make_grid(nx, ny, 1.0, 1.0, bp::Bc::Neumann);
        ComplexField x = field_from(g, in);
        if (!inverse) {
            auto m = bp::forward_transform(x, bp::TransformKind::DCT);
            std::memcpy(out, m.data(), sizeof(cplx) * m.size());
        } else {
            std::vector<cplx> m(x.data);
            field_to(bp::inverse_transform(m, g, bp::TransformKind::DCT), out);
        }
    });
}

// Reference kernels for the kernel-level CPU baseline (proj/src/kernels.cpp)
void bpref_five_point(const double* u, int nx, int ny, double h2, double* out) {
    const size_t n = static_cast<size_t>(nx) * ny;
    bp::kernels::five_point(std::span<const cplx>(reinterpret_cast<const cplx*>(u), n), nx, ny,
                            h2, std::span<cplx>(reinterpret_cast<cplx*>(out), n));
}

// ---- BPFD field / problem I/O (field.cpp:37-133, problem_io.cpp:16-95): the reference's own
// writers and readers, for the byte-exact pins of the project's native I/O (tests/)
int bpref_save_field(const char* path, int nx, int ny, int dtype, const double* data) {
    return guarded([&] {
        GridSpec g = bp::make_grid(nx, ny, 1.0, 1.0, bp::Bc::Periodic);
        if (dtype == 1) {
            bp::save_field(path, field_from(g, data));
        } else {
            bp::RealField f(g);
            std::memcpy(f.data.data(), data, sizeof(double) * f.data.size());
            bp::save_field(path, f);
        }
    });
}

int bpref_load_field(const char* path, int nx, int ny, int dtype, double* out) {
    return guarded([&] {
        if (dtype == 1) {
            ComplexField f = bp::load_complex_field(path, bp::Bc::Periodic, 1.0, 1.0);
            if (f.grid.nx != nx || f.grid.ny != ny) throw std::invalid_argument("shape");
            field_to(f, out);
        } else {
            bp::RealField f = bp::load_real_field(path, bp::Bc::Periodic, 1.0, 1.0);
            if (f.grid.nx != nx || f.grid.ny != ny) throw std::invalid_argument("shape");
            std::memcpy(out, f.data.data(), sizeof(double) * f.data.size());
        }
    });
}

int bpref_export_csv(const char* path, int nx, int ny, int dtype, const double* data) {
    return guarded([&] {
        GridSpec g = bp::make_grid(nx, ny, 1.0, 1.0, bp::Bc::Periodic);
        if (dtype == 1) {
            bp::export_csv(path, field_from(g, data));
        } else {
            bp::RealField f(g);
            std::memcpy(f.data.data(), data, sizeof(double) * f.data.size());
            bp::export_csv(path, f);
        }
    });
}

// save_problem of the reference's own HelmholtzProblem (periodic) -> manifest + k2 file
int bpref_save_problem_helmholtz(const char* dir, const char* stem, int nx, int ny, double lx,
                                 double ly, const double* k2, double k0, double eta) {
    return guarded([&] {
        GridSpec g = bp::make_grid(nx, ny, lx, ly, bp::Bc::Periodic);
        bp::HelmholtzProblem p(g, field_from(g, k2), k0, eta);
        bp::save_problem(dir, stem, p);
    });
}

// load_problem of a helmholtz manifest -> grid, k0, eta, k2 (nx*ny complex)
int bpref_load_problem_helmholtz(const char* path, int* nx, int* ny, double* lx, double* ly,
                                 double* k0, double* eta, double* k2, int cap) {
    return guarded([&] {
        bp::ProblemPtr p = bp::load_problem(path);
        const auto* h = dynamic_cast<const bp::HelmholtzProblem*>(p.get());
        if (!h) throw std::invalid_argument("not a helmholtz manifest");
        const GridSpec& g = h->grid();
        *nx = g.nx;
        *ny = g.ny;
        *lx = g.lx;
        *ly = g.ly;
        *k0 = h->k0();
        *eta = h->eta();
        if ((long)g.nx * g.ny > cap) throw std::invalid_argument("capacity");
        field_to(h->k2(), k2);
    });
}

}  // extern "C"
