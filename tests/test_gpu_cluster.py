"""Whole-solve cluster kernel (csrc/cluster_kernels.cuh) for n = 64 / 128 grids (config c0):
the grid resident in one thread-block cluster's distributed shared memory, bp::run's sweep loop
on the device.  Parity as the rest of the suite: iteration counts +-1 (here: equal), same
termination, iterates within 1e-10 relative L2; against the two-launch path (BP_CLUSTER=0) and
the oracle, and the c0 full solve (232 sweeps)."""
import numpy as np
import pytest

import paper_2603_18527_b200 as bs
from oracle import MAP_POINTWISE, MAP_SCALAR, OracleProblem

pytestmark = pytest.mark.gpu
FIELD_TOL = 1e-10


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def solve(monkeypatch, cluster, k2, f, k0, eta, cmap, cfg):
    monkeypatch.setenv("BP_CLUSTER", "1" if cluster else "0")
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        return bs.run(p, cmap, f, cfg)


@pytest.mark.parametrize("n", [64, 128])
@pytest.mark.parametrize("name", ["scalar", "pointwise", "direct"])
def test_cluster_matches_two_launch_path_and_oracle(gpu, monkeypatch, n, name):
    k2, f, k0, eta = bs.make_instances(bs.InstanceSpec(n=n, ppw=10.0, contrast=0.3, seed=n), 0, 3)
    cmap = bs.ScalarMap(1.0) if name == "scalar" else bs.PointwiseMap()
    cfg = bs.IterationConfig("direct" if name == "direct" else "npbs", 1e-9 if name != "direct" else 1e-3, 3000)
    if name == "direct":
        cmap = bs.ScalarMap(2e-5)
    got = solve(monkeypatch, True, k2, f, k0, eta, cmap, cfg)
    ref = solve(monkeypatch, False, k2, f, k0, eta, cmap, cfg)
    for b in range(3):
        assert got.traces[b].iters == ref.traces[b].iters
        assert got.traces[b].terminated == ref.traces[b].terminated
        k = got.traces[b].iters + 1
        np.testing.assert_allclose(got.traces[b].res_l2_rel[:k], ref.traces[b].res_l2_rel[:k], rtol=1e-9, atol=1e-14)
        np.testing.assert_allclose(got.traces[b].res_reta_rel[:k], ref.traces[b].res_reta_rel[:k], rtol=1e-9, atol=1e-14)
        assert rel(got.u[b], ref.u[b]) < FIELD_TOL
    o = OracleProblem(k2[0], k0[0], eta[0]).run(
        f[0], map_kind=MAP_SCALAR if isinstance(cmap, bs.ScalarMap) else MAP_POINTWISE,
        gamma=getattr(cmap, "gamma", 1.0), fmt=0 if name == "direct" else 2, rtol=cfg.rtol, max_iters=3000)
    assert abs(got.traces[0].iters - o.iters) <= 1 and got.traces[0].terminated == o.terminated
    if o.terminated != "diverged":
        assert rel(got.u[0], o.u) < FIELD_TOL


def test_cluster_c0_full_solve(gpu, monkeypatch):
    """BASELINE c0 (127^2, gamma = 1, rtol 1e-6): 232 sweeps in the oracle (round 1 pin)."""
    k2, f, k0, eta = bs.config_instances("c0")
    got = solve(monkeypatch, True, k2, f, k0, eta, bs.ScalarMap(1.0), bs.IterationConfig(rtol=1e-6, max_iters=20000))
    o = OracleProblem(k2[0], k0[0], eta[0]).run(f[0], rtol=1e-6, max_iters=20000)
    assert got.traces[0].iters == o.iters == 232
    assert got.traces[0].terminated == o.terminated == "converged"
    assert rel(got.u[0], o.u) < FIELD_TOL


def test_cluster_max_iters_and_warm_start(gpu, monkeypatch):
    k2, f, k0, eta = bs.make_instances(bs.InstanceSpec(n=128, ppw=10.0, contrast=0.3, seed=5), 0, 2)
    cfg = bs.IterationConfig(rtol=1e-12, max_iters=37)
    a = solve(monkeypatch, True, k2, f, k0, eta, bs.ScalarMap(1.0), cfg)
    b = solve(monkeypatch, False, k2, f, k0, eta, bs.ScalarMap(1.0), cfg)
    for i in range(2):
        assert a.traces[i].iters == b.traces[i].iters == 37 and a.traces[i].terminated == "max_iters"
        assert rel(a.u[i], b.u[i]) < FIELD_TOL
    monkeypatch.setenv("BP_CLUSTER", "1")
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        w = bs.run(p, bs.ScalarMap(1.0), f, bs.IterationConfig(rtol=1e-6, max_iters=3000), u0=a.u)
    monkeypatch.setenv("BP_CLUSTER", "0")
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        w2 = bs.run(p, bs.ScalarMap(1.0), f, bs.IterationConfig(rtol=1e-6, max_iters=3000), u0=a.u)
    assert w.traces[0].iters == w2.traces[0].iters
    assert rel(w.u, w2.u) < FIELD_TOL
