"""Waves (BP_GROUP members per wave x BP_SPLIT parts) at other member sizes: n = 256 and 1024.
Wall-clock of bs.run (host fields, 255 sweeps: the copies are ~2 % and equal for every setting)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_2603_18527_b200 as bs  # noqa: E402

for n, batch, settings in [(256, 128, ["0 2", "16 8", "16 16", "32 8", "32 16", "24 12", "48 16", "0 2"]),
                           (1024, 16, ["0 4", "2 2", "4 4", "4 2", "8 8", "8 4", "0 4"])]:
    k2, f, k0, eta = bs.make_instances(bs.InstanceSpec(n=n, ppw=8.0, contrast=0.5), 0, batch)
    cfg = bs.IterationConfig(rtol=1e-30, max_iters=255)
    for st in settings:
        g, s = st.split()
        os.environ["BP_GROUP"], os.environ["BP_SPLIT"] = g, s
        with bs.HelmholtzDirichlet(k2, k0, eta) as p:
            bs.run(p, bs.PointwiseMap(), f, cfg)
            best = 1e9
            for _ in range(3):
                t0 = time.perf_counter()
                r = bs.run(p, bs.PointwiseMap(), f, cfg)
                best = min(best, time.perf_counter() - t0)
        sweeps = sum(t.iters for t in r.traces)
        print(f"n={n} batch={batch} GROUP={g} SPLIT={s}: {sweeps * (n - 1) ** 2 / best / 1e9:7.2f} Gpts/s", flush=True)
