"""Quick per-kernel timing for kernel experiments (not the bench contract):
    python tools/kbench.py [--config c1] [--members 64] [--sweeps 32] [--reps 3]
Runs bp::run with per-launch CUDA-event timing (bp_set_kernel_timing) and prints the average
row-stage / column-stage time per sweep."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_18527_b200 as bs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--members", type=int, default=64)
ap.add_argument("--sweeps", type=int, default=47)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--n", type=int, default=0, help="2-D synthetic n x n instead of a config")
args = ap.parse_args()
if args.config == "c4":
    bx, by, sg, s0, f = bs.config_instances("c4", 0, args.members)
    p = bs.CdrNeumann(bx, by, sg, s0)
    cmap, cfg = bs.ScalarMap(1.0), bs.IterationConfig("cbs", 1e-30, args.sweeps)
else:
    if args.n:
        k2, f, k0, eta = bs.make_instances(bs.InstanceSpec(n=args.n, ppw=8.0, contrast=0.5), 0, args.members)
    else:
        k2, f, k0, eta = bs.config_instances(args.config, 0, args.members)
    p = bs.HelmholtzDirichlet(k2, k0, eta, dim=3 if args.config == "c3" else 2)
    cmap = bs.PointwiseMap() if bs.CONFIGS[args.config]["map"] == "pointwise" else bs.ScalarMap(1.0)
    if args.n:
        args.config = f"n{args.n}"
    cfg = bs.IterationConfig(rtol=1e-30, max_iters=args.sweeps)
p.set_kernel_timing(True)
for rep in range(args.reps):
    t0 = time.perf_counter()
    r = bs.run(p, cmap, f, cfg)
    st = p.last_run_stats()
    full = max(st["active_sweeps"], 1) / args.members  # launches over the whole active batch
    print(f"{args.config} x{args.members} rep{rep}: row {st['row_ms'] / full * 1e3:8.1f} us  col "
          f"{st['col_ms'] / full * 1e3:8.1f} us per full sweep ({st['timed_sweeps']} timed, "
          f"{st['active_sweeps']} member-sweeps)  wall {time.perf_counter() - t0:.2f}s")
p.close()
