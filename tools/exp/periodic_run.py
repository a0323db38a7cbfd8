"""Small periodic-family run (for ncu tail checks): 16 x 512^2 periodic Helmholtz, 8 sweeps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2603_18527_b200 as bs
n, B = 512, 16
rng = np.random.default_rng(0)
k0 = 2 * np.pi * 16.0
k2 = (k0 ** 2) * (1.0 + 0.2 * rng.random((B, n, n))) + 0j
eta = np.full(B, 0.5 * k0 ** 2)
f = np.zeros((B, n, n), complex); f[:, n // 2, n // 2] = 1.0
with bs.HelmholtzPeriodic(k2, np.full(B, k0), eta) as p:
    p.set_kernel_timing(True)
    r = bs.run(p, bs.ScalarMap(1.0), f, bs.IterationConfig(rtol=1e-12, max_iters=8))
    print("periodic", p.last_run_stats())
