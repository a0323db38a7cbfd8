#!/bin/bash
O=gpurun_out/r02p; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_generic.py tests/test_gpu_parity.py -q > $O/generic_tests.log 2>&1; echo "rc=$?" >> $O/generic_tests.log
timeout 300 python -c "
import time, numpy as np, paper_2603_18527_b200 as bs
for nx, ny in [(1000, 1000), (511, 300), (4095, 511)]:
    k2, f, k0, eta = bs.make_instances(bs.InstanceSpec(n=512, ppw=8.0, contrast=0.5), 0, 1)
    rng = np.random.default_rng(0)
    k2 = (400.0 * (1.0 + 0.1 * rng.standard_normal((nx, ny))) * (1.0 + 0.05j))
    eta = 1.01 * float(np.abs(k2 - 400.0).max())
    with bs.HelmholtzDirichlet(k2, 20.0, eta) as p:
        x = rng.standard_normal((nx, ny)) + 0j
        cfg = bs.IterationConfig(rtol=1e-30, max_iters=64)
        bs.run(p, bs.PointwiseMap(), x, cfg)
        t = time.perf_counter(); bs.run(p, bs.PointwiseMap(), x, cfg); dt = time.perf_counter() - t
        print(nx, ny, 'sweeps/s', 65 / dt, 'Gpts/s', 65 * nx * ny / dt / 1e9)
" > $O/generic_perf.log 2>&1
