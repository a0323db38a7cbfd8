// bornsweep.hpp -- header-only C++ mirror of the reference's operator / map / driver API
// (bp::Problem, bp::CorrectionMap, bp::run) over the C ABI in bornsweep.h.
//
// A reference user switches by replacing
//     bp::HelmholtzProblem / bp::run(problem, map, f, cfg)          (proj/include/bp/iterate.hpp:62-67)
// with
//     bornsweep::GpuHelmholtzDirichlet / bornsweep::run(problem, map, f, cfg)
// Fields are std::vector<std::complex<double>> in the reference layout (data[ix*ny + iy],
// proj/include/bp/field.hpp:14-26); a batch is `batch` fields back to back.  Errors are
// re-thrown as the reference's exception types: BP_EINVAL -> std::invalid_argument,
// BP_ERUNTIME -> std::runtime_error (proj/src/problem.cpp:16, proj/src/symbol.cpp:30-31).
#pragma once

#include <complex>
#include <stdexcept>
#include <string>
#include <utility>
#include <type_traits>
#include <variant>
#include <vector>

#include "bornsweep.h"

namespace bornsweep {

using cplx = std::complex<double>;
using Field = std::vector<cplx>;

class unsupported_error : public std::logic_error {
  public:
    using std::logic_error::logic_error;
};

inline void check(int rc) {
    if (rc == BP_OK) return;
    const std::string msg = bp_last_error();
    switch (rc) {
        case BP_EINVAL: throw std::invalid_argument(msg);
        case BP_ERUNTIME: throw std::runtime_error(msg);
        case BP_ENOTSUP: throw unsupported_error(msg);
        default: throw std::runtime_error("bornsweep: " + msg);
    }
}

// bp::ScalarMap / bp::OptimalScalarMap / diagonal relaxation (proj/include/bp/correction.hpp:16-40)
struct ScalarMap {
    cplx gamma{1.0, 0.0};
};
struct OptimalScalarMap {
    int metric = BP_METRIC_EUCLIDEAN;
};
struct PointwiseMap {};  // gamma(x) = (i/eta) V(x)
using CorrectionMap = std::variant<ScalarMap, OptimalScalarMap, PointwiseMap>;

enum class IterFormat { Direct = BP_FMT_DIRECT, CBS = BP_FMT_CBS, NPBS = BP_FMT_NPBS };
struct IterationConfig {  // proj/include/bp/iterate.hpp:14-18
    IterFormat format = IterFormat::NPBS;
    double rtol = 1e-6;
    int max_iters = 1000;
};

enum class Termination { Converged = 0, MaxIters = 1, Diverged = 2, Stagnated = 3 };
struct IterationTrace {  // proj/include/bp/iterate.hpp:25-32
    std::vector<double> res_l2_rel;
    std::vector<double> res_reta_rel;
    int iters = 0;
    Termination terminated = Termination::MaxIters;
    double fnorm_l2 = 0.0;
    double fnorm_reta = 0.0;
};

struct RunResult {
    Field u;                            // batch fields back to back
    std::vector<IterationTrace> trace;  // one per member
};

// Batch of Dirichlet five-point Helmholtz problems (A = L_D - k2, V = k2 - (k0^2 + i eta)).
class GpuHelmholtzDirichlet {
  public:
    GpuHelmholtzDirichlet(int n_interior, const Field& k2, const std::vector<double>& k0,
                          const std::vector<double>& eta, double length = 1.0, int device = 0)
        : n_(n_interior), batch_(static_cast<int>(k0.size())) {
        if (k2.size() != static_cast<size_t>(batch_) * n_ * n_ || eta.size() != k0.size())
            throw std::invalid_argument("GpuHelmholtzDirichlet: field grid mismatch");
        bp_grid g{n_, n_, length, length, BP_BC_DIRICHLET};
        check(bp_problem_create(&g, batch_, reinterpret_cast<const double*>(k2.data()), k0.data(),
                                eta.data(), device, &h_));
    }
    GpuHelmholtzDirichlet(const GpuHelmholtzDirichlet&) = delete;
    GpuHelmholtzDirichlet& operator=(const GpuHelmholtzDirichlet&) = delete;
    ~GpuHelmholtzDirichlet() { bp_problem_destroy(h_); }

    int batch() const { return batch_; }
    int n() const { return n_; }
    const bp_problem* handle() const { return h_; }

    // bp::Problem operator applications (proj/include/bp/problem.hpp:26-39)
    Field apply_A(const Field& u) const { return unary(bp_apply_A, u); }
    Field apply_V(const Field& u) const { return unary(bp_apply_V, u); }
    Field apply_V_adjoint(const Field& u) const { return unary(bp_apply_V_adjoint, u); }
    Field apply_Lref(const Field& u) const { return unary(bp_apply_Lref, u); }
    Field apply_G(const Field& q) const { return unary(bp_apply_G, q); }
    Field born_residual(const Field& u, const Field& f) const {
        Field out(u.size());
        check(bp_born_residual(h_, d(u), d(f), d(out)));
        return out;
    }
    Field residual(const Field& u, const Field& f) const {  // proj/src/iterate.cpp:45-50
        Field out(u.size());
        check(bp_residual(h_, d(u), d(f), d(out)));
        return out;
    }

  private:
    using UnaryFn = int (*)(const bp_problem*, const double*, double*);
    Field unary(UnaryFn fn, const Field& x) const {
        if (x.size() != static_cast<size_t>(batch_) * n_ * n_)
            throw std::invalid_argument("field grid mismatch");
        Field out(x.size());
        check(fn(h_, d(x), d(out)));
        return out;
    }
    static const double* d(const Field& f) { return reinterpret_cast<const double*>(f.data()); }
    static double* d(Field& f) { return reinterpret_cast<double*>(f.data()); }

    int n_, batch_;
    bp_problem* h_ = nullptr;
};

// bp::run (proj/src/iterate.cpp:88-153) over every member of the batch
inline RunResult run(const GpuHelmholtzDirichlet& p, const CorrectionMap& map, const Field& f,
                     const IterationConfig& cfg = {}, const Field* u0 = nullptr) {
    bp_map m{};
    std::visit(
        [&](const auto& mm) {
            using T = std::decay_t<decltype(mm)>;
            if constexpr (std::is_same_v<T, ScalarMap>) {
                m.kind = BP_MAP_SCALAR;
                m.gamma_re = mm.gamma.real();
                m.gamma_im = mm.gamma.imag();
            } else if constexpr (std::is_same_v<T, OptimalScalarMap>) {
                m.kind = BP_MAP_OPTIMAL_SCALAR;
                m.metric = mm.metric;
            } else {
                m.kind = BP_MAP_POINTWISE;
            }
        },
        map);
    bp_iter_config c{static_cast<int32_t>(cfg.format), cfg.rtol, cfg.max_iters};
    const int B = p.batch();
    const size_t stride = static_cast<size_t>(cfg.max_iters) + 1;
    std::vector<double> l2(B * stride), reta(B * stride);
    std::vector<bp_trace> info(B);
    RunResult res;
    res.u.resize(f.size());
    check(bp_run(p.handle(), &m, reinterpret_cast<const double*>(f.data()), &c,
                 u0 ? reinterpret_cast<const double*>(u0->data()) : nullptr,
                 reinterpret_cast<double*>(res.u.data()), l2.data(), reta.data(), info.data()));
    for (int b = 0; b < B; ++b) {
        IterationTrace t;
        const size_t k = static_cast<size_t>(info[b].iters) + 1;
        t.res_l2_rel.assign(l2.begin() + b * stride, l2.begin() + b * stride + k);
        t.res_reta_rel.assign(reta.begin() + b * stride, reta.begin() + b * stride + k);
        t.iters = info[b].iters;
        t.terminated = static_cast<Termination>(info[b].terminated);
        t.fnorm_l2 = info[b].fnorm_l2;
        t.fnorm_reta = info[b].fnorm_reta;
        res.trace.push_back(std::move(t));
    }
    return res;
}

}  // namespace bornsweep
