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
#include <memory>
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

    // swap in new media of the same grid / batch (bp_problem_set_medium)
    void set_medium(const Field& k2, const std::vector<double>& k0, const std::vector<double>& eta) {
        if (k2.size() != static_cast<size_t>(batch_) * n_ * n_ || k0.size() != static_cast<size_t>(batch_) ||
            eta.size() != k0.size())
            throw std::invalid_argument("set_medium: field grid mismatch");
        check(bp_problem_set_medium(h_, reinterpret_cast<const double*>(k2.data()), k0.data(), eta.data()));
    }

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

inline bp_map to_c_map(const CorrectionMap& map) {
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
    return m;
}

inline std::vector<IterationTrace> make_traces(int batch, size_t stride, const std::vector<double>& l2,
                                               const std::vector<double>& reta,
                                               const std::vector<bp_trace>& info) {
    std::vector<IterationTrace> out;
    for (int b = 0; b < batch; ++b) {
        IterationTrace t;
        const size_t k = static_cast<size_t>(info[b].iters) + 1;
        t.res_l2_rel.assign(l2.begin() + b * stride, l2.begin() + b * stride + k);
        t.res_reta_rel.assign(reta.begin() + b * stride, reta.begin() + b * stride + k);
        t.iters = info[b].iters;
        t.terminated = static_cast<Termination>(info[b].terminated);
        t.fnorm_l2 = info[b].fnorm_l2;
        t.fnorm_reta = info[b].fnorm_reta;
        out.push_back(std::move(t));
    }
    return out;
}

// bp::run (proj/src/iterate.cpp:88-153) over every member of the batch
inline RunResult run(const GpuHelmholtzDirichlet& p, const CorrectionMap& map, const Field& f,
                     const IterationConfig& cfg = {}, const Field* u0 = nullptr) {
    const bp_map m = to_c_map(map);
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
    res.trace = make_traces(B, stride, l2, reta, info);
    return res;
}

// Overlapped solves over several handles of one shape (bp_pipeline_*; the reference solves one
// batch at a time, proj/src/bench.cpp:143-151): submit() enqueues set_medium (when k2 is given)
// + run on the next slot and returns; wait() returns the results in submission order.  The
// fields passed to submit() must stay alive until wait(); the slots must outlive the pipeline.
class GpuPipeline {
  public:
    explicit GpuPipeline(const std::vector<GpuHelmholtzDirichlet*>& slots) : slots_(slots) {
        std::vector<bp_problem*> hs;
        for (auto* s : slots_) hs.push_back(const_cast<bp_problem*>(s->handle()));
        check(bp_pipeline_create(hs.data(), static_cast<int32_t>(hs.size()), &pl_));
    }
    GpuPipeline(const GpuPipeline&) = delete;
    GpuPipeline& operator=(const GpuPipeline&) = delete;
    ~GpuPipeline() {
        bp_pipeline_wait(pl_);
        bp_pipeline_destroy(pl_);
    }

    size_t submit(const CorrectionMap& map, const Field& f, const IterationConfig& cfg = {},
                  const Field* k2 = nullptr, const std::vector<double>* k0 = nullptr,
                  const std::vector<double>* eta = nullptr) {
        auto j = std::make_unique<Job>();
        const int B = slots_.front()->batch();
        j->stride = static_cast<size_t>(cfg.max_iters) + 1;
        j->l2.resize(B * j->stride);
        j->reta.resize(B * j->stride);
        j->info.resize(B);
        j->u.resize(f.size());
        bp_medium md{};
        if (k2) {
            if (!k0 || !eta) throw std::invalid_argument("pipeline submit: k2 needs k0 and eta");
            md.k2 = reinterpret_cast<const double*>(k2->data());
            md.k0 = k0->data();
            md.eta = eta->data();
        }
        const bp_map m = to_c_map(map);
        const bp_iter_config c{static_cast<int32_t>(cfg.format), cfg.rtol, cfg.max_iters};
        check(bp_pipeline_submit(pl_, &md, &m, reinterpret_cast<const double*>(f.data()), &c, nullptr,
                                 reinterpret_cast<double*>(j->u.data()), j->l2.data(), j->reta.data(),
                                 j->info.data(), &j->slot));
        jobs_.push_back(std::move(j));
        return jobs_.size() - 1;
    }

    std::vector<RunResult> wait() {
        const int rc = bp_pipeline_wait(pl_);
        std::vector<std::unique_ptr<Job>> jobs;
        jobs.swap(jobs_);
        check(rc);
        std::vector<RunResult> out;
        for (auto& j : jobs) {
            RunResult r;
            r.u = std::move(j->u);
            r.trace = make_traces(slots_[j->slot]->batch(), j->stride, j->l2, j->reta, j->info);
            out.push_back(std::move(r));
        }
        return out;
    }

  private:
    struct Job {  // heap-held: the worker threads write into these buffers until wait()
        int32_t slot = 0;
        size_t stride = 0;
        Field u;
        std::vector<double> l2, reta;
        std::vector<bp_trace> info;
    };
    std::vector<GpuHelmholtzDirichlet*> slots_;
    bp_pipeline* pl_ = nullptr;
    std::vector<std::unique_ptr<Job>> jobs_;
};

}  // namespace bornsweep
