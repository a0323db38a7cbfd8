// cpp_api_check.cpp -- exercises the header-only C++ mirror (include/bornsweep.hpp) the way a
// reference user would call bp::run: build a batch, run CBS, print one line per member:
//   member iters termination res_l2_last u_checksum
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bornsweep.hpp"
#include "bornsweep_instances.h"

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 32;
    const int batch = argc > 2 ? std::atoi(argv[2]) : 2;
    bp_instance_spec spec{n, 10.0, 0.3, 3.0, 2.0, 0, 0, -1, 1.0, 1.01};
    const int nd = n - 1;
    bornsweep::Field k2(static_cast<size_t>(batch) * nd * nd), f(k2.size());
    std::vector<double> k0(batch), eta(batch);
    if (bp_make_instances(&spec, 0, batch, reinterpret_cast<double*>(k2.data()),
                          reinterpret_cast<double*>(f.data()), k0.data(), eta.data(), 0))
        return 2;
    try {
        bornsweep::GpuHelmholtzDirichlet p(nd, k2, k0, eta);
        bornsweep::IterationConfig cfg;
        cfg.rtol = 1e-6;
        cfg.max_iters = 5000;
        auto r = bornsweep::run(p, bornsweep::ScalarMap{}, f, cfg);
        for (int b = 0; b < batch; ++b) {
            double s = 0;
            for (int i = 0; i < nd * nd; ++i) s += std::abs(r.u[static_cast<size_t>(b) * nd * nd + i]);
            std::printf("%d %d %d %.17g %.17g\n", b, r.trace[b].iters,
                        static_cast<int>(r.trace[b].terminated), r.trace[b].res_l2_rel.back(), s);
        }
        // overlapped solves: a two-slot pipeline gives the direct run bit for bit
        {
            bornsweep::GpuHelmholtzDirichlet p2(nd, k2, k0, eta);
            bornsweep::GpuPipeline pipe({&p, &p2});
            for (int j = 0; j < 3; ++j) pipe.submit(bornsweep::ScalarMap{}, f, cfg, &k2, &k0, &eta);
            const auto rs = pipe.wait();
            for (size_t j = 0; j < rs.size(); ++j) {
                bool same = rs[j].u == r.u;
                for (int b = 0; b < batch; ++b)
                    same = same && rs[j].trace[b].iters == r.trace[b].iters &&
                           rs[j].trace[b].res_l2_rel == r.trace[b].res_l2_rel &&
                           rs[j].trace[b].res_reta_rel == r.trace[b].res_reta_rel;
                std::printf("pipe %zu %s\n", j, same ? "same" : "DIFFERENT");
            }
        }
        // error mapping: zero source -> std::invalid_argument, like bp::run
        try {
            bornsweep::run(p, bornsweep::ScalarMap{}, bornsweep::Field(f.size()), cfg);
            std::printf("no-throw\n");
            return 3;
        } catch (const std::invalid_argument& e) {
            std::printf("invalid_argument: %s\n", e.what());
        }
    } catch (const std::exception& e) {
        std::printf("error: %s\n", e.what());
        return 1;
    }
    return 0;
}
