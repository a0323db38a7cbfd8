"""The reference's own family on the GPU: periodic pseudospectral bp::HelmholtzProblem
(helmholtz.cpp:11-53) vs fixtures produced by the reference's own code (oracle/_ref) on the
reference's own bench instance generator, and vs the oracle at larger sizes."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
import paper_2603_18527_b200 as bs
from oracle import MAP_FOURIER_DIAG, MAP_OPTIMAL_SCALAR, MAP_SCALAR, Oracle, OracleProblem

pytestmark = pytest.mark.gpu
FIELD_TOL = 1e-10
OP_TOL = 1e-13


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("n", [32, 64])
def test_periodic_operators_match_reference(gpu, n):
    g = np.load(os.path.join(GOLDEN, f"ref_periodic_n{n}.npz"))
    x, f = g["x"], g["f"]
    with bs.HelmholtzPeriodic(g["k2"], float(g["k0"]), float(g["eta"])) as p:
        assert rel(p.apply_V(x), g["V"]) < 1e-15
        assert rel(p.apply_V_adjoint(x), g["VH"]) < 1e-15
        assert rel(p.apply_A(x), g["A"]) < OP_TOL
        assert rel(p.apply_Lref(x), g["Lref"]) < OP_TOL
        assert rel(p.apply_G(x), g["G"]) < OP_TOL
        assert rel(p.born_residual(x, f), g["born"]) < OP_TOL
        assert rel(p.residual(x, f), g["res"]) < OP_TOL
        assert rel(p.forward_transform(x), g["fwd"]) < OP_TOL
        assert rel(p.inverse_transform(x), g["inv"]) < OP_TOL


@pytest.mark.parametrize("n", [32, 64])
@pytest.mark.parametrize("name", ["scalar", "scalar_relaxed", "fd", "optl2"])
def test_periodic_runs_match_reference(gpu, n, name):
    # optl2: OptimalScalarMap{Euclidean}, the reference's own default CBS map on its own family
    # (proj/src/bench.cpp:140-141, correction.cpp:22-48)
    g = np.load(os.path.join(GOLDEN, f"ref_periodic_n{n}.npz"))
    cmap = {"scalar": bs.ScalarMap(1.0), "scalar_relaxed": bs.ScalarMap(0.9 + 0.05j),
            "fd": bs.FourierDiagMap(g["fd_m"]), "optl2": bs.OptimalScalarMap("euclidean")}[name]
    with bs.HelmholtzPeriodic(g["k2"], float(g["k0"]), float(g["eta"])) as p:
        res = bs.run(p, cmap, g["f"], bs.IterationConfig(rtol=1e-8, max_iters=4000))
    tr, iters = res.trace, int(g[f"run_{name}_iters"])
    assert tr.terminated == str(g[f"run_{name}_term"])
    assert abs(tr.iters - iters) <= 1
    k = min(tr.iters, iters) + 1
    np.testing.assert_allclose(tr.res_l2_rel[:k], g[f"run_{name}_l2"][:k], rtol=1e-8, atol=1e-13)
    np.testing.assert_allclose(tr.res_reta_rel[:k], g[f"run_{name}_reta"][:k], rtol=1e-8, atol=1e-13)
    if tr.iters == iters:
        assert rel(res.u, g[f"run_{name}_u"]) < FIELD_TOL


@pytest.mark.parametrize("n", [8, 128, 512, 2048])
def test_periodic_transforms_and_green_vs_oracle(gpu, n):
    Oracle.set_threads(os.cpu_count() or 8)
    rng = np.random.default_rng(n)
    k2 = (200.0 + 20 * rng.standard_normal((2, n, n))) * (1 + 0.05j)
    k0, eta = np.array([14.0, 14.5]), np.array([60.0, 70.0])
    x = rng.standard_normal(k2.shape) + 1j * rng.standard_normal(k2.shape)
    f = rng.standard_normal(k2.shape) + 0j
    with bs.HelmholtzPeriodic(k2, k0, eta) as p:
        fw, iv, G, born = p.forward_transform(x), p.inverse_transform(x), p.apply_G(x), p.born_residual(x, f)
    for b in range(2):
        o = OracleProblem(k2[b], k0[b], eta[b], periodic=True)
        assert rel(fw[b], np.fft.fft2(x[b])) < OP_TOL
        assert rel(iv[b], np.fft.ifft2(x[b])) < OP_TOL
        assert rel(G[b], o.apply_G(x[b])) < OP_TOL
        assert rel(born[b], o.born_residual(x[b], f[b])) < OP_TOL


def test_periodic_per_iterate_and_warm_start(gpu):
    n = 128
    rng = np.random.default_rng(1)
    k2 = (300.0 + 30 * rng.standard_normal((n, n))) * (1 + 0.03j)
    k0, eta = 17.0, 90.0
    f = np.zeros((n, n), np.complex128)
    f[n // 2, n // 3] = 1.0
    u0 = 1e-4 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    K = 30
    with bs.HelmholtzPeriodic(k2, k0, eta) as p:
        res = bs.run(p, bs.ScalarMap(1.0), f, bs.IterationConfig(rtol=1e-12, max_iters=K), u0=u0,
                     n_snap=K + 1)
    o = OracleProblem(k2, k0, eta, periodic=True)
    ref = o.run(f, map_kind=MAP_SCALAR, gamma=1.0, rtol=1e-12, max_iters=K, u0=u0, n_snap=K + 1)
    assert res.trace.iters == ref.iters == K
    for m in range(0, K + 1):
        assert rel(res.snapshots[m], ref.snapshots[m]) < FIELD_TOL, m
    np.testing.assert_allclose(res.trace.res_l2_rel, ref.res_l2, rtol=1e-8)


@pytest.mark.parametrize("name", ["optreta", "direct_optl2", "direct_scalar"])
def test_periodic_more_runs_match_reference(gpu, name):
    """OptimalScalar with the R_eta metric and the Direct format (direction = r,
    iterate.cpp:118-123) on the reference's periodic family, vs the reference's own run()."""
    g = np.load(os.path.join(GOLDEN, "ref_periodic_n32.npz"))
    h = np.load(os.path.join(GOLDEN, "ref_periodic_more.npz"))
    cmap, cfg = {
        "optreta": (bs.OptimalScalarMap("reta"), bs.IterationConfig(rtol=1e-8, max_iters=4000)),
        "direct_optl2": (bs.OptimalScalarMap("euclidean"),
                         bs.IterationConfig(format="direct", rtol=1e-3, max_iters=300)),
        "direct_scalar": (bs.ScalarMap(2e-5), bs.IterationConfig(format="direct", rtol=1e-3, max_iters=200)),
    }[name]
    with bs.HelmholtzPeriodic(g["k2"], float(g["k0"]), float(g["eta"])) as p:
        res = bs.run(p, cmap, g["f"], cfg)
    tr, iters = res.trace, int(h[f"run_{name}_iters"])
    assert tr.terminated == str(h[f"run_{name}_term"])
    assert abs(tr.iters - iters) <= 1
    k = min(tr.iters, iters) + 1
    np.testing.assert_allclose(tr.res_l2_rel[:k], h[f"run_{name}_l2"][:k], rtol=1e-8, atol=1e-13)
    np.testing.assert_allclose(tr.res_reta_rel[:k], h[f"run_{name}_reta"][:k], rtol=1e-8, atol=1e-13)
    if tr.iters == iters:
        assert rel(res.u, h[f"run_{name}_u"]) < FIELD_TOL


def test_periodic_optimal_scalar_per_iterate_vs_oracle(gpu):
    """Per-iterate u^m of the periodic OptimalScalar runs (both metrics) vs the plain-C oracle."""
    g = np.load(os.path.join(GOLDEN, "ref_periodic_n64.npz"))
    K = 25
    o = OracleProblem(g["k2"], float(g["k0"]), float(g["eta"]), periodic=True)
    for metric, mk in (("euclidean", 0), ("reta", 1)):
        with bs.HelmholtzPeriodic(g["k2"], float(g["k0"]), float(g["eta"])) as p:
            res = bs.run(p, bs.OptimalScalarMap(metric), g["f"], bs.IterationConfig(rtol=1e-12, max_iters=K),
                         n_snap=K + 1)
        ref = o.run(g["f"], map_kind=MAP_OPTIMAL_SCALAR, metric=mk, rtol=1e-12, max_iters=K, n_snap=K + 1)
        assert res.trace.iters == ref.iters == K
        assert not np.any(res.snapshots[0])  # u^0 = 0
        for m in range(1, K + 1):
            assert rel(res.snapshots[m], ref.snapshots[m]) < FIELD_TOL, (metric, m)


def test_periodic_unsupported_maps_raise(gpu):
    g = np.load(os.path.join(GOLDEN, "ref_periodic_n32.npz"))
    with bs.HelmholtzPeriodic(g["k2"], float(g["k0"]), float(g["eta"])) as p:
        with pytest.raises(NotImplementedError):  # a Dirichlet-family map
            bs.run(p, bs.PointwiseMap(), g["f"])
