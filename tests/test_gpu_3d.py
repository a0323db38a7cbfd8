"""3-D extension (BASELINE config c3: 255^3, seven-point stencil, DST-I along x, y, z).
The reference has no 3-D; parity is GPU vs the plain-C oracle's 3-D restatement,
which tests/test_oracle.py pins against scipy's 3-D DST-I and the verify-suite identities."""
import os

import numpy as np
import pytest

import paper_2603_18527_b200 as bs
from oracle import MAP_POINTWISE, MAP_SCALAR, Oracle, OracleProblem

pytestmark = pytest.mark.gpu
FIELD_TOL = 1e-10
OP_TOL = 1e-13


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def inst3(n, batch=1, seed=0, ppw=8.0, contrast=0.4):
    spec = bs.InstanceSpec(n=n, ppw=ppw, contrast=contrast, sigma_cells=3.0, seed=seed, dim=3)
    return bs.make_instances(spec, 0, batch)


@pytest.mark.parametrize("n", [8, 16, 32, 64])
def test_3d_transforms_and_operators(gpu, n):
    Oracle.set_threads(os.cpu_count() or 8)
    k2, f, k0, eta = inst3(n, batch=2, seed=n)
    rng = np.random.default_rng(n)
    u = rng.standard_normal(k2.shape) + 1j * rng.standard_normal(k2.shape)
    with bs.HelmholtzDirichlet(k2, k0, eta, dim=3) as p:
        got = dict(fw=p.forward_transform(u), iv=p.inverse_transform(u), A=p.apply_A(u),
                   V=p.apply_V(u), G=p.apply_G(u), L=p.apply_Lref(u), born=p.born_residual(u, f),
                   res=p.residual(u, f))
    for b in range(2):
        o = OracleProblem(k2[b], k0[b], eta[b])
        assert rel(got["fw"][b], Oracle.forward_dst(u[b])) < OP_TOL
        assert rel(got["iv"][b], Oracle.inverse_dst(u[b])) < OP_TOL
        assert rel(got["A"][b], o.apply_A(u[b])) < 1e-15
        assert rel(got["V"][b], o.apply_V(u[b])) < 1e-15
        assert rel(got["res"][b], o.residual(u[b], f[b])) < 1e-15
        assert rel(got["G"][b], o.apply_G(u[b])) < OP_TOL
        assert rel(got["L"][b], o.apply_Lref(u[b])) < OP_TOL
        assert rel(got["born"][b], o.born_residual(u[b], f[b])) < OP_TOL


@pytest.mark.parametrize("n,kind", [(32, "pointwise"), (64, "scalar")])
def test_3d_per_iterate(gpu, n, kind):
    Oracle.set_threads(os.cpu_count() or 8)
    k2, f, k0, eta = inst3(n, seed=1, contrast=0.3, ppw=10.0)
    K = 25
    cmap = bs.PointwiseMap() if kind == "pointwise" else bs.ScalarMap(1.0)
    with bs.HelmholtzDirichlet(k2, k0, eta, dim=3) as p:
        res = bs.run(p, cmap, f, bs.IterationConfig(rtol=1e-12, max_iters=K), n_snap=K + 1)
    o = OracleProblem(k2[0], k0[0], eta[0])
    ref = o.run(f[0], map_kind=MAP_POINTWISE if kind == "pointwise" else MAP_SCALAR, rtol=1e-12,
                max_iters=K, n_snap=K + 1)
    assert res.trace.iters == ref.iters == K
    for m in range(1, K + 1):
        assert rel(res.snapshots[m], ref.snapshots[m]) < FIELD_TOL, m
    np.testing.assert_allclose(res.trace.res_l2_rel, ref.res_l2, rtol=1e-8)
    np.testing.assert_allclose(res.trace.res_reta_rel, ref.res_reta, rtol=1e-8)


def test_3d_full_solve_small(gpu):
    k2, f, k0, eta = inst3(32, seed=2, contrast=0.3, ppw=10.0)
    with bs.HelmholtzDirichlet(k2, k0, eta, dim=3) as p:
        res = bs.run(p, bs.PointwiseMap(), f, bs.IterationConfig(rtol=1e-5, max_iters=5000))
    ref = OracleProblem(k2[0], k0[0], eta[0]).run(f[0], map_kind=MAP_POINTWISE, rtol=1e-5,
                                                   max_iters=5000)
    assert res.trace.terminated == ref.terminated == "converged"
    assert abs(res.trace.iters - ref.iters) <= 1
    if res.trace.iters == ref.iters:
        assert rel(res.u, ref.u) < FIELD_TOL


def test_config3_first_sweeps(gpu):
    """BASELINE config 3 at full size (255^3): the first sweeps vs the oracle."""
    Oracle.set_threads(os.cpu_count() or 8)
    k2, f, k0, eta = bs.config_instances("c3")
    K = 2
    with bs.HelmholtzDirichlet(k2, k0, eta, dim=3) as p:
        res = bs.run(p, bs.PointwiseMap(), f, bs.IterationConfig(rtol=1e-5, max_iters=K))
    ref = OracleProblem(k2[0], k0[0], eta[0]).run(f[0], map_kind=MAP_POINTWISE, rtol=1e-5,
                                                   max_iters=K)
    assert res.trace.iters == ref.iters == K
    np.testing.assert_allclose(res.trace.res_l2_rel, ref.res_l2, rtol=1e-8)
    assert rel(res.u, ref.u) < FIELD_TOL


@pytest.mark.parametrize("n", [64, 128])
def test_3d_batch_deferred_finalisation(gpu, n):
    """3-D batches: the trace entry is finalised by the first column launch from one partial per
    row CTA (finalize_member3).  Members terminate independently, each bit-identical to its
    single-member run, and the iteration counts / first iterates agree with the oracle."""
    Oracle.set_threads(os.cpu_count() or 8)
    k2, f, k0, eta = inst3(n, batch=3, seed=7, contrast=0.3, ppw=10.0)
    cfg = bs.IterationConfig(rtol=1e-5, max_iters=3000 if n == 64 else 6)
    with bs.HelmholtzDirichlet(k2, k0, eta, dim=3) as p:
        res = bs.run(p, bs.PointwiseMap(), f, cfg)
    for b in range(3):
        with bs.HelmholtzDirichlet(k2[b:b + 1], k0[b:b + 1], eta[b:b + 1], dim=3) as q:
            one = bs.run(q, bs.PointwiseMap(), f[b:b + 1], cfg)
        assert np.array_equal(res.u[b], one.u[0])
        assert res.traces[b].iters == one.traces[0].iters
        assert np.array_equal(res.traces[b].res_l2_rel, one.traces[0].res_l2_rel)
        assert np.array_equal(res.traces[b].res_reta_rel, one.traces[0].res_reta_rel)
    ref = OracleProblem(k2[0], k0[0], eta[0]).run(f[0], map_kind=MAP_POINTWISE, rtol=1e-5,
                                                   max_iters=cfg.max_iters)
    t = res.traces[0]
    assert t.terminated == ref.terminated
    assert abs(t.iters - ref.iters) <= 1
    k = min(t.iters, ref.iters) + 1
    np.testing.assert_allclose(t.res_l2_rel[:k], ref.res_l2[:k], rtol=1e-8)
    np.testing.assert_allclose(t.res_reta_rel[:k], ref.res_reta[:k], rtol=1e-8)
    if t.iters == ref.iters:
        assert rel(res.u[0], ref.u) < FIELD_TOL
