"""Small driver for ncu captures of the sweep kernels (config c1 shapes).

    python tools/profile_sweep.py [--members 64] [--sweeps 4]

Runs one bp::run over `members` c1 media with max_iters = `sweeps`; ncu then selects the
row/column kernels with -k regex:'row_kernel|col_kernel'.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_18527_b200 as bs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--members", type=int, default=64)
ap.add_argument("--sweeps", type=int, default=4)
ap.add_argument("--config", default="c1")
args = ap.parse_args()
if args.config == "c4":
    bx, by, sg, s0, f = bs.config_instances("c4", 0, args.members)
    with bs.CdrNeumann(bx, by, sg, s0) as p:
        p.set_kernel_timing(True)
        r = bs.run(p, bs.ScalarMap(1.0), f, bs.IterationConfig(rtol=1e-8, max_iters=args.sweeps))
        print("iters", [t.iters for t in r.traces[:4]], p.last_run_stats())
    sys.exit(0)
k2, f, k0, eta = bs.config_instances(args.config, 0, args.members)
with bs.HelmholtzDirichlet(k2, k0, eta, dim=3 if args.config == "c3" else 2) as p:
    cmap = bs.PointwiseMap() if args.config == "c1" else bs.ScalarMap(1.0)
    p.set_kernel_timing(True)  # plain launches (no graph) so ncu sees each kernel
    r = bs.run(p, cmap, f, bs.IterationConfig(rtol=1e-6, max_iters=args.sweeps))
    print("iters", [t.iters for t in r.traces[:4]], p.last_run_stats())
