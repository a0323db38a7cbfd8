"""Staggered termination in multi-member launches, other families: batch runs vs every member
alone, repeated (iteration counts and fields must be identical)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_2603_18527_b200 as bs  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 8


def check(name, make, run_one, batch):
    ref = [run_one(make(slice(b, b + 1))) for b in range(batch)]
    bad = 0
    for rep in range(reps):
        r = run_one(make(slice(None)))
        for b in range(batch):
            if r.traces[b].iters != ref[b].traces[0].iters or not np.array_equal(r.u[b], ref[b].u[0]):
                bad += 1
                print(f"  {name} rep {rep} member {b}: batch iters {r.traces[b].iters} alone {ref[b].traces[0].iters}")
    print(f"{name}: iters alone {[x.traces[0].iters for x in ref]}  mismatches {bad} / {reps * batch}", flush=True)


# CDR (c4 family), 256^2 x 6
bx, by, sg, s0, f = bs.make_cdr_instances(bs.CdrSpec(n=256, seed=3), 0, 6)
f[2] *= 5.0
cfgc = bs.IterationConfig("cbs", 1e-3, 200)
check("cdr", lambda sl: (bs.CdrNeumann(bx[sl], by[sl], sg[sl], s0[sl]), f[sl]),
      lambda pf: (lambda p, ff: (lambda r: (p.close(), r)[1])(bs.run(p, bs.ScalarMap(1.0), ff, cfgc)))(*pf), 6)

# periodic 128^2 x 6
rng = np.random.default_rng(1)
n = 128
g = rng.standard_normal((6, n, n))
kk = 2 * np.pi / (10.0 / n) / (1.0 + 0.1 * np.tanh(g))
k2 = (kk * kk) * (1.0 + 0.05j)
k0 = kk.reshape(6, -1).mean(axis=1)
eta = np.array([1.01 * np.abs(k2[b] - k0[b] ** 2).max() for b in range(6)])
fp = np.zeros((6, n, n), complex)
fp[:, n // 2, n // 2] = 1.0
cfgp = bs.IterationConfig("npbs", 0.3, 300)
check("periodic", lambda sl: (bs.HelmholtzPeriodic(k2[sl], k0[sl], eta[sl]), fp[sl]),
      lambda pf: (lambda p, ff: (lambda r: (p.close(), r)[1])(bs.run(p, bs.OptimalScalarMap(), ff, cfgp)))(*pf), 6)

# 3-D 32^3 x 4, and 2-D Dirichlet n = 128 x 12 with the optimal-scalar and FourierDiag plans
k3, f3, k03, eta3 = bs.make_instances(bs.InstanceSpec(n=32, ppw=8.0, contrast=0.4, dim=3, seed=2), 0, 4)
cfg3 = bs.IterationConfig(rtol=0.3, max_iters=300)
check("3d", lambda sl: (bs.HelmholtzDirichlet(k3[sl], k03[sl], eta3[sl], dim=3), f3[sl]),
      lambda pf: (lambda p, ff: (lambda r: (p.close(), r)[1])(bs.run(p, bs.PointwiseMap(), ff, cfg3)))(*pf), 4)
k2d, fd, k0d, etad = bs.make_instances(bs.InstanceSpec(n=128, ppw=8.0, contrast=0.5, seed=5), 0, 12)
cfgd = bs.IterationConfig(rtol=0.3, max_iters=300)
for nm, cmap in (("2d-pointwise", bs.PointwiseMap()), ("2d-optimal", bs.OptimalScalarMap()),
                 ("2d-reta", bs.OptimalScalarMap("reta"))):
    check(nm, lambda sl: (bs.HelmholtzDirichlet(k2d[sl], k0d[sl], etad[sl]), fd[sl]),
          lambda pf, cmap=cmap: (lambda p, ff: (lambda r: (p.close(), r)[1])(bs.run(p, cmap, ff, cfgd)))(*pf), 12)
