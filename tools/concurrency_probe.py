"""Does running two half-batches on two streams (row pass of one overlapping the column pass of
the other) beat one full batch on one stream?  python tools/concurrency_probe.py [groups]"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2603_18527_b200 as bs  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
S = 127
k2, f, k0, eta = bs.config_instances("c1", 0, 64)
cfg = bs.IterationConfig(rtol=1e-6, max_iters=S)


import ctypes as C  # noqa: E402
import torch  # noqa: E402
from paper_2603_18527_b200 import _native as N  # noqa: E402


def timed(probs, fs, reps=5):
    lib = N.lib()
    dev = {}
    for p, ff in zip(probs, fs):
        fd = torch.from_numpy(ff).cuda()
        dev[id(p)] = (fd, torch.empty_like(fd), (N.Trace * p.batch)(), np.empty((p.batch, S + 1)),
                      np.empty((p.batch, S + 1)))
    mp, cc = bs.PointwiseMap()._c(), cfg._c()
    dp = C.POINTER(C.c_double)

    def one(p, ff):
        fd, ud, info, l2, rt = dev[id(p)]
        rc = lib.bp_run_device(p.handle, C.byref(mp), C.c_void_p(fd.data_ptr()), C.byref(cc), None,
                               C.c_void_p(ud.data_ptr()), l2.ctypes.data_as(dp), rt.ctypes.data_as(dp), info)
        assert rc == 0, N.last_error()
    for _ in range(2):
        ths = [threading.Thread(target=one, args=(p, ff)) for p, ff in zip(probs, fs)]
        [t.start() for t in ths]
        [t.join() for t in ths]
    t0 = time.perf_counter()
    for _ in range(reps):
        ths = [threading.Thread(target=one, args=(p, ff)) for p, ff in zip(probs, fs)]
        [t.start() for t in ths]
        [t.join() for t in ths]
    dt = (time.perf_counter() - t0) / reps
    return 64 * S * 511 * 511 / dt / 1e9


full = [bs.HelmholtzDirichlet(k2, k0, eta)]
print("1 group :", timed(full, [f]))
for p in full:
    p.close()
per = 64 // G
parts = [bs.HelmholtzDirichlet(k2[g * per:(g + 1) * per], k0[g * per:(g + 1) * per],
                               eta[g * per:(g + 1) * per]) for g in range(G)]
print(f"{G} groups:", timed(parts, [f[g * per:(g + 1) * per] for g in range(G)]))
