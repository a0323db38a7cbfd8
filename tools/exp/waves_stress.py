"""Which path deviates?  19 members at n = 512: waves (default), one graph (BP_SPLIT=0), two parts
(BP_GROUP=0 BP_SPLIT=2), and member 3 alone; repeated."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_2603_18527_b200 as bs  # noqa: E402

batch = 19
k2, f, k0, eta = bs.make_instances(bs.InstanceSpec(n=512, ppw=8.0, contrast=0.5, sigma_cells=2.0, seed=7), 0, batch)
f[3] *= 10.0
cfg = bs.IterationConfig(rtol=0.5, max_iters=200)


def run(env, sl=slice(None)):
    for k in ("BP_GROUP", "BP_SPLIT"):
        os.environ.pop(k, None)
    os.environ.update(env)
    with bs.HelmholtzDirichlet(k2[sl], k0[sl], eta[sl]) as p:
        r = bs.run(p, bs.PointwiseMap(), f[sl], cfg)
    return [t.iters for t in r.traces], r


# churn the allocator / L2 between runs like a test suite does
junk = []
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    a, ra = run({})
    b, rb = run({"BP_SPLIT": "0"})
    c, rc = run({"BP_GROUP": "0", "BP_SPLIT": "2"})
    alone = [run({}, slice(m, m + 1))[0][0] for m in (3, 11)]
    bad = [m for m in range(batch) if not (a[m] == b[m] == c[m])]
    print(f"rep {rep}: waves {a[3]},{a[11]} one {b[3]},{b[11]} two {c[3]},{c[11]} alone {alone}  mismatching members {bad}",
          [(a[m], b[m], c[m]) for m in bad], flush=True)
    with bs.HelmholtzDirichlet(k2[:5], k0[:5], eta[:5]) as p:  # a different shape in between
        bs.run(p, bs.OptimalScalarMap(), f[:5], bs.IterationConfig(rtol=1e-3, max_iters=30))
