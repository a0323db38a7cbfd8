"""Diagnostic: OptimalScalar at n = 256 over a full solve -- single-GPU path vs 4 slabs vs the
oracle: how far do the traces of correct runs drift apart late in the solve?"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_2603_18527_b200 as bs
from oracle import MAP_OPTIMAL_SCALAR, OracleProblem
from paper_2603_18527_b200.slab import LocalComm, SlabPart, run_slab

spec = bs.InstanceSpec(n=256, ppw=10.0, contrast=0.3, sigma_cells=3.0, seed=3)
k2, f, k0, eta = bs.make_instances(spec, 0, 1)
cfg = bs.IterationConfig(rtol=1e-7, max_iters=4000)
for metric in ("euclidean", "reta"):
    cmap = bs.OptimalScalarMap(metric)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        one = bs.run(p, cmap, f, cfg)
    parts = [SlabPart(k2[0], float(k0[0]), float(eta[0]), r, 4) for r in range(4)]
    sl = run_slab(parts, LocalComm(), cmap, f[0], cfg)
    ref = OracleProblem(k2[0], float(k0[0]), float(eta[0])).run(
        f[0], map_kind=MAP_OPTIMAL_SCALAR, metric=0 if metric == "euclidean" else 1, rtol=1e-7, max_iters=4000)
    t1, t2, t3 = one.traces[0].res_l2_rel, sl.trace.res_l2_rel, ref.res_l2
    k = min(len(t1), len(t2), ref.iters + 1)
    d12 = np.abs(t1[:k] - t2[:k]) / t1[:k]
    d13 = np.abs(t1[:k] - t3[:k]) / t1[:k]
    print(metric, "iters single/slab/oracle", one.traces[0].iters, sl.trace.iters, ref.iters)
    for m in (10, 40, 100, 200, 300, 400, k - 1):
        if m < k:
            print(f"  m={m}: single-vs-slab {d12[m]:.2e}  single-vs-oracle {d13[m]:.2e}")
