"""Full-length parity fixtures for the BASELINE configs ("next round" item 1).

    python tests/golden/make_long.py [c1 c2 c3]   (from the repo root; needs oracle/_ref built)

Inputs are the configs' own seeded media (paper_2603_18527_b200.config_instances, host-only
synthesis, no GPU); the solves run on the CPU checkers:
  c1  members 2..9 (members 0, 1 are pinned by tests/test_gpu_parity.py) to rtol 1e-6 with the
      pointwise map, through oracle/_ref -- the reference's own proj/src code (bp::run restated
      Eigen-free in oracle/ref/ref_driver.cpp), OpenMP over members;
  c2  the 4095^2 single grid, 20 and 40 sweeps (u^20, u^40 and the 41-entry traces), oracle/_ref;
  c3  the 255^3 grid to rtol 1e-5 (the full solve), the plain-C oracle (the reference has no
      3-D family), OpenMP inside its transforms.
Each fixture keeps iteration counts, terminations, full residual traces, every field's L2
norm, a fixed projection <w, u> with w = exp(2 pi i (3 ix + 5 iy [+ 7 iz]) / n), and u sampled on
a stride-8 (c2: stride-16) sub-lattice -- the full fields (268 MB each) are not committed.
An input checksum (sum of k2, sum of f) guards against drift in the instance synthesis."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2603_18527_b200 as bs  # noqa: E402
from oracle import MAP_POINTWISE, MAP_SCALAR, Oracle, OracleProblem, Reference  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def projection(u):
    """<w, u> = sum conj(w) u, w = exp(2 pi i (3 i0 + 5 i1 [+ 7 i2]) / n) over the last dims."""
    n = u.shape[-1] + 1
    grids = np.meshgrid(*[np.arange(s) for s in u.shape[-u.ndim:]], indexing="ij")
    phase = sum(k * g for k, g in zip((3, 5, 7), grids))
    w = np.exp(2j * np.pi * phase / n)
    return complex(np.vdot(w, u))


def summary(u, stride):
    sl = tuple(slice(0, None, stride) for _ in range(u.ndim))
    return dict(norm=np.linalg.norm(u), proj=projection(u), sample=np.ascontiguousarray(u[sl]))


def checksum(k2, f):
    return np.array([k2.sum(), f.sum()])


def make_c1():
    first, count = 2, 8
    k2, f, k0, eta = bs.config_instances("c1", first, count)
    t0 = time.time()
    u, l2, rt, info = Reference.run_batch(k2, k0, eta, f, map_kind=MAP_POINTWISE, rtol=1e-6,
                                          max_iters=20000, nthreads=os.cpu_count())
    out = dict(first=first, count=count, checksum=checksum(k2, f),
               iters=np.array([i for i, _ in info]), term=np.array([t for _, t in info]))
    for b in range(count):
        k = info[b][0] + 1
        out[f"l2_{b}"], out[f"reta_{b}"] = l2[b, :k], rt[b, :k]
        s = summary(u[b], 8)
        out[f"norm_{b}"], out[f"proj_{b}"], out[f"sample_{b}"] = s["norm"], s["proj"], s["sample"]
    np.savez_compressed(os.path.join(HERE, "long_c1.npz"), **out)
    print("c1", out["iters"], f"{time.time() - t0:.0f}s", flush=True)


def make_c2():
    k2, f, k0, eta = bs.config_instances("c2")
    t0 = time.time()
    out = dict(checksum=checksum(k2, f))
    for m in (20, 40):
        u, l2, rt, info = Reference.run_batch(k2, k0, eta, f, map_kind=MAP_POINTWISE, rtol=1e-30,
                                              max_iters=m, nthreads=os.cpu_count())
        s = summary(u[0], 16)
        out[f"norm_{m}"], out[f"proj_{m}"], out[f"sample_{m}"] = s["norm"], s["proj"], s["sample"]
        out[f"l2_{m}"], out[f"reta_{m}"] = l2[0, :m + 1], rt[0, :m + 1]
        print("c2", m, info, f"{time.time() - t0:.0f}s", flush=True)
    np.savez_compressed(os.path.join(HERE, "long_c2.npz"), **out)


def make_c3():
    k2, f, k0, eta = bs.config_instances("c3")
    Oracle.set_threads(os.cpu_count() or 8)
    t0 = time.time()
    cmap = MAP_POINTWISE if bs.CONFIGS["c3"]["map"] == "pointwise" else MAP_SCALAR
    r = OracleProblem(k2[0], k0[0], eta[0]).run(f[0], map_kind=cmap, rtol=bs.CONFIGS["c3"]["rtol"],
                                                max_iters=20000)
    s = summary(r.u, 8)
    np.savez_compressed(os.path.join(HERE, "long_c3.npz"), checksum=checksum(k2, f), iters=r.iters,
                        term=r.terminated, l2=r.res_l2, reta=r.res_reta, norm=s["norm"],
                        proj=s["proj"], sample=s["sample"])
    print("c3", r.iters, r.terminated, f"{time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2", "c3"]
    for name in which:
        globals()["make_" + name]()
